"""Test harness: the same seeded inputs fed to the CUDA path (through the C ABI) and to the
CPU oracle.  The oracle never sees a value computed by the CUDA path."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from datagen import configs as dc
from datagen import init_pack_tables_torch, make_batch, make_dy, table_values_np

# north star tolerance for fp32 (BASELINE.json): 1e-5 relative / 1e-6 absolute
RTOL, ATOL = 1e-5, 1e-6


def oracle_model(cfg: dc.Config):
    return oracle.OracleModel(cfg.field_to_table, cfg.table_rows, cfg.table_dim, cfg.field_col,
                              id_mode=cfg.id_mode, pool=cfg.pool, table_salt=cfg.table_salt)


def oracle_tables(cfg: dc.Config):
    return [table_values_np(cfg.seed, t, np.arange(cfg.table_rows[t]), int(cfg.table_dim[t]))
            for t in range(cfg.T)]


def gpu_embedding(cfg: dc.Config, max_batch=None, max_ids=None, opt=0, split=False, plan_tables=None, **kw):
    import paper_2204_04903_b200 as pb

    mb = max_batch or cfg.batch
    mi = max_ids if max_ids is not None else mb * cfg.F * 60
    emb = pb.PackedEmbedding(cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=mb, max_ids=mi,
                             table_salt=cfg.table_salt, field_col=cfg.field_col, pool=cfg.pool,
                             id_mode=cfg.id_mode, opt=opt, split=split, **kw)
    init_pack_tables_torch(cfg, emb.plan["table_to_pack"], emb.plan["table_base"], emb.n_packs, emb.weights)
    torch.cuda.synchronize()
    return emb


def to_dev(batch):
    ids = torch.from_numpy(batch.ids).cuda()
    off = torch.from_numpy(batch.offsets).cuda()
    return ids, off


def gpu_table_rows(emb, cfg, t, which="w"):
    """Rows of table t as stored in the packed GPU tables (world = 1 layout)."""
    p = int(emb.plan["table_to_pack"][t])
    base = int(emb.plan["table_base"][t])
    src = {"w": emb.weights, "s1": emb.state1, "s2": emb.state2}[which][p]
    return src[base:base + int(cfg.table_rows[t])].cpu().numpy()


def assert_close(got, ref, rtol=RTOL, atol=ATOL, what=""):
    got = np.asarray(got, np.float32)
    ref = np.asarray(ref, np.float32)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    bad = np.abs(got - ref) > atol + rtol * np.abs(ref)
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} / {bad.size} mismatches, first at {tuple(i)}: "
                             f"got {got[tuple(i)]!r} ref {ref[tuple(i)]!r}")
