"""Full-size parity at BASELINE.json configs[1] (Criteo-shaped: 26 fields, dim 128, batch
16,384, 46.875M rows = 24 GB fp32 tables) in the launch configuration bench.py times.
The oracle cannot hold the tables, so it checks (a) the whole unique/inverse of the pack
(bit-exact), (b) a random sample of pooled segments (bit-exact), (c) a sample of touched
rows — including the hottest — after the Adagrad step (1e-5/1e-6), and (d) a sample of
untouched rows (bitwise unchanged).  Table rows for the oracle are regenerated on the host
from the same seeded generator."""
import numpy as np
import pytest
import torch

import oracle
from datagen import configs as dc
from datagen import make_batch, make_dy, table_values_np
from harness import assert_close, gpu_embedding, oracle_model, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__

    __graft_entry__.build()


def _rows_values(cfg, t_arr, r_arr, ld):
    vals = np.zeros((len(t_arr), ld), np.float32)
    for t in np.unique(t_arr):
        sel = t_arr == t
        vals[sel, :cfg.table_dim[t]] = table_values_np(cfg.seed, int(t), r_arr[sel], int(cfg.table_dim[t]))
    return vals


@pytest.mark.parametrize("dyadic", [True, False])
def test_criteo_fullsize_sampled(dyadic):
    cfg = dc.criteo()
    b = make_batch(cfg, 0, 7)
    dy = make_dy(cfg, 0, 7, dyadic=dyadic)
    emb = gpu_embedding(cfg, max_ids=b.n_ids)
    m = oracle_model(cfg)
    ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)
    ids, off = to_dev(b)
    out = emb.forward(ids, off, cfg.batch)
    torch.cuda.synchronize()
    # (a) unique / inverse of the single pack, whole stream
    keys = oracle.pack_key_stream(m, emb.plan["field_to_pack"], emb.plan["table_base"], ob, 0)
    u_ref, inv_ref = oracle.unique(keys)
    assert np.array_equal(emb.unique(0).cpu().numpy(), u_ref)
    assert np.array_equal(emb.inverse(0).cpu().numpy(), inv_ref)
    # (b) sampled segments
    rng = np.random.default_rng(0)
    qf = rng.integers(0, cfg.F, 3000).astype(np.int32)
    qs = rng.integers(0, cfg.batch, 3000).astype(np.int32)
    rt, rr = oracle.segment_rows(m, ob, qf, qs)
    ref = oracle.forward_sampled(m, ob, rt, rr, _rows_values(cfg, rt, rr, 128), qf, qs)
    got = out.cpu().numpy()
    for i in range(len(qf)):
        c = int(cfg.field_col[qf[i]])
        assert np.array_equal(got[qs[i], c:c + 128], ref[i]), f"segment {i}"
    # (c) touched rows: hottest 64 + 1000 random; (d) 500 random rows (mostly untouched)
    tb = emb.plan["table_base"]
    allt, allr = oracle.segment_rows(m, ob, np.repeat(np.arange(cfg.F, dtype=np.int32), cfg.batch),
                                     np.tile(np.arange(cfg.batch, dtype=np.int32), cfg.F))
    key = tb[allt] + allr
    uk, cnt = np.unique(key, return_counts=True)
    pick = np.concatenate([uk[np.argsort(-cnt, kind="stable")[:64]], rng.choice(uk, 1000, replace=False),
                           rng.integers(0, int(cfg.table_rows.sum()), 500)])
    pick = np.unique(pick)
    qt = (np.searchsorted(tb, pick, side="right") - 1).astype(np.int32)
    qr = pick - tb[qt]
    w0 = _rows_values(cfg, qt, qr, 128)
    G, n = oracle.row_grads(m, [ob], qt, qr, 128)
    w_ref, s_ref = w0.copy(), np.full_like(w0, 0.1)
    oracle.apply_update(G, n, w_ref, s_ref, lr=0.01)
    emb.backward_update(torch.from_numpy(dy).cuda(), lr=0.01, step=1)
    emb.check()
    idx = torch.from_numpy(pick).cuda()
    w_gpu = emb.weights[0].index_select(0, idx).cpu().numpy()
    s_gpu = emb.state1[0].index_select(0, idx).cpu().numpy()
    assert (n > 0).sum() >= 1064 - 5 and n.max() > 256  # hot rows take the chunked path
    assert_close(w_gpu, w_ref, what="weights")
    if dyadic:
        assert np.array_equal(w_gpu, w_ref) and np.array_equal(s_gpu, s_ref)
    else:
        # fp64 accumulation on both sides: G = fp32(exact sum) except at rounding ties
        assert_close(s_gpu, s_ref, what="state")
        assert (w_gpu == w_ref).all(axis=1).mean() > 0.99
    assert np.array_equal(w_gpu[n == 0], w0[n == 0])


def _sampled_parity(cfg, step=3, dyadic=True, n_seg=2000, n_rand=600, n_hot=32, lr=0.01):
    """Full-size parity of a multi-pack config, row-sampled (SURVEY §8(c) "Full-scale parity
    without a full CPU replay"): whole unique / inverse per pack (bit-exact), a sample of pooled
    segments (bit-exact), and per pack the hottest rows + random touched rows + random rows
    after the Adagrad step (bit-exact under dyadic dY; untouched rows bitwise unchanged)."""
    b = make_batch(cfg, 0, step)
    dy = make_dy(cfg, 0, step, dyadic=dyadic)
    emb = gpu_embedding(cfg, max_ids=b.n_ids)
    m = oracle_model(cfg)
    ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)
    ids, off = to_dev(b)
    out = emb.forward(ids, off, cfg.batch)
    emb.check()
    rng = np.random.default_rng(step)
    f2p, tb = emb.plan["field_to_pack"], emb.plan["table_base"]
    t2p = emb.plan["table_to_pack"]
    picks = []
    for p in range(emb.n_packs):  # (a) whole-stream unique / inverse, and the per-pack row sample
        keys = oracle.pack_key_stream(m, f2p, tb, ob, p)
        u_ref, inv_ref = oracle.unique(keys)
        assert np.array_equal(emb.unique(p).cpu().numpy(), u_ref), f"unique pack {p}"
        assert np.array_equal(emb.inverse(p).cpu().numpy(), inv_ref), f"inverse pack {p}"
        cnt = np.bincount(inv_ref, minlength=len(u_ref))
        hot = u_ref[np.argsort(-cnt, kind="stable")[:n_hot]]
        pick = np.unique(np.concatenate([hot, rng.choice(u_ref, min(n_rand, len(u_ref)), replace=False),
                                         rng.integers(0, int(emb.plan["pack_rows"][p]), n_rand // 2)]))
        picks.append(pick)
        del keys, inv_ref
    # (b) sampled segments (bit-exact)
    ld = int(cfg.table_dim.max())
    qf = rng.integers(0, cfg.F, n_seg).astype(np.int32)
    qs = rng.integers(0, cfg.batch, n_seg).astype(np.int32)
    rt, rr = oracle.segment_rows(m, ob, qf, qs)
    ref = oracle.forward_sampled(m, ob, rt, rr, _rows_values(cfg, rt, rr, ld), qf, qs)
    got = out.cpu().numpy()
    fd = cfg.field_dim
    for i in range(n_seg):
        c, d = int(cfg.field_col[qf[i]]), int(fd[qf[i]])
        assert np.array_equal(got[qs[i], c:c + d], ref[i, :d]), f"segment {i} (field {qf[i]}, sample {qs[i]})"
    del got, out
    # (c)/(d) sampled rows after the update
    emb.backward_update(torch.from_numpy(dy).cuda(), lr=lr, step=1)
    emb.check()
    for p, pick in enumerate(picks):
        tabs_p = np.nonzero(t2p == p)[0]
        tabs_p = tabs_p[np.argsort(tb[tabs_p], kind="stable")]
        ti = np.searchsorted(tb[tabs_p], pick, side="right") - 1
        qt = tabs_p[ti].astype(np.int32)
        qr = pick - tb[qt]
        D = int(emb.plan["pack_dim"][p])
        w0 = _rows_values(cfg, qt, qr, D)
        G, n = oracle.row_grads(m, [ob], qt, qr, D)
        w_ref, s_ref = w0.copy(), np.full_like(w0, 0.1)
        oracle.apply_update(G, n, w_ref, s_ref, lr=lr)
        idx = torch.from_numpy(pick).cuda()
        w_gpu = emb.weights[p].index_select(0, idx).cpu().numpy()
        s_gpu = emb.state1[p].index_select(0, idx).cpu().numpy()
        assert (n > 0).sum() >= min(n_rand, 1) and (n == 0).any()
        assert_close(w_gpu, w_ref, what=f"weights pack {p}")
        if dyadic:
            assert np.array_equal(w_gpu, w_ref), f"weights pack {p} (dyadic: bit-exact)"
            assert np.array_equal(s_gpu, s_ref), f"state pack {p}"
        assert np.array_equal(w_gpu[n == 0], w0[n == 0]), f"untouched rows pack {p}"
    return b.n_ids


def test_wdl_fullsize_sampled():
    """C3 at full size on one GPU (200 fields, 4 packs D = 8/16/32/64, 2M rows per table = 48 GB
    of weights, B = 16,384, ~83.6 M IDs): three radix passes (uids > 2^20), per-table dedup
    regions, the staged k_scatter3 and the transpose beside the pool (> 4 M IDs), every pool and
    segment-sum variant (flat D <= 32, pipe D = 64)."""
    n = _sampled_parity(dc.wdl(), step=3)
    assert n > (1 << 26)


def test_industrial_shape_fullsize_sampled():
    """C4's shape (250 one-hot + 15 x 50 positional fields, half the positions empty, 265 tables)
    at B = 16,384 with the tables at a quarter of their rows (28 GB) so weights + state fit one
    GPU: > 2^22 IDs, 4 packs, empty bags, fields sharing a table (one dedup per pack)."""
    n = _sampled_parity(dc.scaled(dc.industrial(), batch=16384, rows_div=4), step=2)
    assert n > (1 << 22)
