"""Embedding dims other than the kernels' row widths (CAN's 8~200, MMoE's 12~128):
a table of dim D is stored at picasso_kernel_dim(D) with zero padding, and a field's output / dY
column block is that wide.  Checked against the oracle at the true dims: forward bit-exact on the D
real columns and exactly 0 on the padding; after Adagrad / Adam steps the D real columns of every
table equal the oracle's (bit-exact under dyadic dY) and the padding columns of the tables and the
state never change."""
import numpy as np
import pytest
import torch

import oracle
from datagen import configs as dc
from datagen import init_pack_tables_torch, make_batch, make_dy
from harness import assert_close, oracle_model, oracle_tables

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__

    __graft_entry__.build()


def odd_cfg(**kw):
    return dc.Config("odd", 256, np.array([0, 1, 2, 3, 3, 1], np.int32), np.array([500, 300, 200, 400], np.int64),
                     np.array([12, 200, 8, 20], np.int32), [("uniform", 0, 4)] * 6, alpha=1.0).replace(**kw)


def test_kernel_dim_map():
    import paper_2204_04903_b200 as pb

    assert [pb.picasso_kernel_dim(d) for d in (1, 4, 5, 12, 20, 64, 100, 128, 129, 200, 300, 384, 500, 512)] == \
           [4, 4, 8, 16, 32, 64, 128, 128, 256, 256, 384, 384, 512, 512]
    with pytest.raises(pb.PicassoError):
        pb.picasso_kernel_dim(513)


@pytest.mark.parametrize("opt", [0, 1])
def test_odd_dims_parity(opt):
    import paper_2204_04903_b200 as pb

    cfg = odd_cfg(pool=dc.POOL_SUM if opt == 0 else dc.POOL_MEAN)
    emb = pb.PackedEmbedding(cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=cfg.batch,
                             max_ids=cfg.batch * cfg.F * 8, table_salt=cfg.table_salt, pool=cfg.pool,
                             id_mode=cfg.id_mode, opt=opt)
    init_pack_tables_torch(cfg, emb.plan["table_to_pack"], emb.plan["table_base"], emb.n_packs, emb.weights)
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    s1 = [np.full_like(t, 0.1) if opt == 0 else np.zeros_like(t) for t in tabs]
    s2 = None if opt == 0 else [np.zeros_like(t) for t in tabs]
    D, KD = cfg.field_dim, emb.kdims[cfg.field_to_table]
    col, kcol = cfg.field_col, emb.field_col
    lr = 0.05 if opt == 0 else 0.01
    for step in (1, 2, 3):
        b = make_batch(cfg, 0, step)
        dy = make_dy(cfg, 0, step, dyadic=opt == 0)
        ids, off = torch.from_numpy(b.ids).cuda(), torch.from_numpy(b.offsets).cuda()
        out = emb.forward(ids, off, cfg.batch).cpu().numpy()
        ref = oracle.forward(m, oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy), tabs, cfg.out_width)
        dyk = np.zeros((cfg.batch, emb.out_width), np.float32)
        for f in range(cfg.F):
            got = out[:, kcol[f]:kcol[f] + D[f]]
            exp = ref[:, col[f]:col[f] + D[f]]
            if step == 1 or opt == 0:
                assert np.array_equal(got, exp), f"forward field {f} step {step}"
            else:
                assert_close(got, exp, what=f"forward field {f} step {step}")
            assert (out[:, kcol[f] + D[f]:kcol[f] + KD[f]] == 0).all(), f"padding of field {f}"
            dyk[:, kcol[f]:kcol[f] + D[f]] = dy[:, col[f]:col[f] + D[f]]
        emb.backward_update(torch.from_numpy(dyk).cuda(), lr=lr, step=step)
        emb.check()
        oracle.backward_update(m, [oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)], tabs, s1, s2, kind=opt,
                               lr=lr, step=step)
        for t in range(cfg.T):
            p, base, d = int(emb.plan["table_to_pack"][t]), int(emb.plan["table_base"][t]), int(cfg.table_dim[t])
            w = emb.weights[p][base:base + int(cfg.table_rows[t])].cpu().numpy()
            st = emb.state1[p][base:base + int(cfg.table_rows[t])].cpu().numpy()
            if opt == 0:
                assert np.array_equal(w[:, :d], tabs[t]), f"table {t} step {step}"
                assert np.array_equal(st[:, :d], s1[t])
            assert_close(w[:, :d], tabs[t], what=f"table {t}")
            assert (w[:, d:] == 0).all() and (st[:, d:] == (0.1 if opt == 0 else 0.0)).all(), f"padding t{t}"
