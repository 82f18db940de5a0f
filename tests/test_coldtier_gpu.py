"""HybridHash with a host-DRAM cold tier (Alg. 1), world = 1: the tables and
optimizer state in pinned host memory (Cold-storage), the top-k rows by FCounter in HBM
(Hot-storage).  Checked against the oracle, which has no cache: every forward bit-exact (hot rows
served from HBM, cold rows read over PCIe), the hot set after every refresh = oracle_hot_select
over the oracle's own post-unique FCounter (reading O11-O13), and the host tables after the final
write-back = the oracle's uncached updates (bit-exact under dyadic dY)."""
import numpy as np
import pytest
import torch

import oracle
from datagen import configs as dc
from datagen import make_batch, make_dy
from harness import assert_close, gpu_embedding, gpu_table_rows, oracle_model, oracle_tables

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__

    __graft_entry__.build()


def run_cached(cfg, capacity, steps=5, warmup=2, flush=1, opt=0, dyadic=True, lr=0.05):
    emb = gpu_embedding(cfg, opt=opt, cold_tier=True, cache_max_bytes=max(capacity, 1024))
    assert not emb.weights[0].is_cuda and emb.weights[0].is_pinned()
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    if opt == 0:
        s1, s2 = [np.full_like(t, 0.1) for t in tabs], None
    else:
        s1, s2 = [np.zeros_like(t) for t in tabs], [np.zeros_like(t) for t in tabs]
    plan = emb.plan
    koff = np.concatenate([[0], np.cumsum(plan["pack_rows"])]).astype(np.int64)
    fc = np.zeros(int(koff[-1]), np.uint64)  # the oracle's FCounter, by global key
    nst = 1 if opt == 0 else 2
    cost = [4 * int(d) * (1 + nst) for d in plan["pack_dim"]]
    hits = []
    for itr in range(steps):  # Alg. 1: itr counts from 0; refresh after bwd when itr >= warmup, itr % flush == 0
        b, dy = make_batch(cfg, 0, itr), make_dy(cfg, 0, itr, dyadic=dyadic)
        ids, off = torch.from_numpy(b.ids).cuda(), torch.from_numpy(b.offsets).cuda()
        out = emb.forward(ids, off, cfg.batch)
        ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)
        ref = oracle.forward(m, ob, tabs, cfg.out_width)
        if dyadic and opt == 0 or itr == 0:
            assert np.array_equal(out.cpu().numpy(), ref), f"forward itr {itr}"
        else:
            assert_close(out.cpu().numpy(), ref, what=f"forward itr {itr}")
        for p in range(emb.n_packs):  # post-unique counting (O11)
            keys = oracle.pack_key_stream(m, plan["field_to_pack"], plan["table_base"], ob, p)
            u, _ = oracle.unique(keys)
            oracle.fcounter_add(u + koff[p], fc)
        emb.backward_update(torch.from_numpy(dy).cuda(), lr=lr, step=itr + 1)
        emb.check()
        oracle.backward_update(m, [ob], tabs, s1, s2, kind=opt, lr=lr, step=itr + 1)
        if itr >= warmup and itr % flush == 0:
            st = emb.hot_cache_refresh(capacity)
            hits.append(st["hit_ratio_unique"])
            g = np.nonzero(fc)[0]
            pk = (np.searchsorted(koff, g, side="right") - 1).astype(np.int32)
            sel = oracle.hot_select(pk, g - koff[pk], fc[g], cost, capacity)
            want = sorted(zip(pk[sel].tolist(), (g - koff[pk])[sel].tolist()))
            hp, hk = emb.hot_keys()
            assert sorted(zip(hp.tolist(), hk.tolist())) == want, f"hot set itr {itr}"
            assert st["k"] == len(want) and st["bytes"] <= capacity
    emb.hot_cache_refresh(0)  # write back and drop: the host tables are authoritative again
    emb.check()
    torch.cuda.synchronize()
    for t in range(cfg.T):
        gw = gpu_table_rows(emb, cfg, t)
        if dyadic and opt == 0:
            assert np.array_equal(gw, tabs[t]), f"table {t}"
            assert np.array_equal(gpu_table_rows(emb, cfg, t, "s1"), s1[t])
        assert_close(gw, tabs[t], what=f"weights t{t}")
        assert_close(gpu_table_rows(emb, cfg, t, "s1"), s1[t], what=f"state1 t{t}")
        if s2:
            assert_close(gpu_table_rows(emb, cfg, t, "s2"), s2[t], what=f"state2 t{t}")
    return hits


@pytest.mark.parametrize("capacity", [0, 640, 4096, 10**7])
def test_toy_cold_tier(capacity):
    """0: no hot rows; 640 B: 5 rows of 128 B (ties cut by key); 4 KB; 10 MB: every row (O18)."""
    hits = run_cached(dc.toy(alpha=1.2), capacity)
    if capacity >= 4096:
        assert max(hits[1:]) > 0


def test_multipack_adam_cold_tier():
    run_cached(dc.scaled(dc.wdl(), batch=24, rows_div=1000), 64 * 1024, steps=4, warmup=1, opt=1, dyadic=False,
               lr=0.01)


def test_criteo_pipe_pool_cold_tier():
    """D = 128: the pipelined pool over row offsets (HStore rows in place, cold rows staged)."""
    hits = run_cached(dc.scaled(dc.criteo(), batch=512, rows_div=5000), 256 * 1024, steps=4, warmup=1)
    assert max(hits) > 0.05
