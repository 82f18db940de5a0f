"""HybridHash (Alg. 1) on the row-sharded path, W = 4 loopback ranks on one GPU.

Checked against the oracle: (a) the hot set chosen at each refresh equals oracle_hot_select over
the oracle's FCounter (post-unique counts of every rank-step so far, reading O11) within the
byte capacity (O12); (b) tier transparency — with hot rows served by the replicas and their
gradients summed over the ranks, every step's forward is bit-exact and, after a final write-back
(capacity 0), every shard equals the oracle's uncached updates (dyadic dY: exact); (c) hot
lookups really bypass the exchange (no hot key is in any send list, every cold unique key is)."""
import numpy as np
import pytest
import torch

import oracle
from datagen import configs as dc
from datagen import init_pack_tables_torch, make_batch, make_dy
from harness import assert_close, oracle_model, oracle_tables
from test_multi_gpu import shard_expected

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__

    __graft_entry__.build()


def _oracle_counts(m, plan, obs, counts, pack_key_off):
    for ob in obs:  # each rank-step: every distinct key of the rank counts once
        for p in range(plan["n_packs"]):
            keys = oracle.pack_key_stream(m, plan["field_to_pack"], plan["table_base"], ob, p)
            oracle.fcounter_add(keys + pack_key_off[p], counts)


@pytest.mark.parametrize("cfg_name", ["toy", "wdl"])
def test_hybridhash_transparency_and_topk(cfg_name):
    import paper_2204_04903_b200 as pb

    W = 4
    cfg = (dc.toy(alpha=1.2) if cfg_name == "toy"
           else dc.scaled(dc.wdl(), batch=24, rows_div=4000).replace(alpha=1.2))
    mi = cfg.batch * cfg.F * 60
    cache_max = 1 << 20
    g = pb.LoopbackGroup(W, cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=cfg.batch, max_ids=mi,
                         table_salt=cfg.table_salt, field_col=cfg.field_col, pool=cfg.pool, id_mode=cfg.id_mode,
                         max_recv=W * mi, cache_max_bytes=cache_max)
    for r, e in enumerate(g.ranks):
        init_pack_tables_torch(cfg, e.plan["table_to_pack"], e.plan["table_base"], e.n_packs, e.weights, rank=r,
                               world=W)
    torch.cuda.synchronize()
    plan = g.ranks[0].plan
    pko = np.concatenate([[0], np.cumsum(plan["pack_rows"])])
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    acc = [np.full_like(t, 0.1) for t in tabs]
    counts = np.zeros(int(pko[-1]), np.uint64)
    cost = 4 * plan["pack_dim"].astype(np.int64) * 2  # weights + Adagrad accumulator
    capacity = 8 * 1024 if cfg_name == "toy" else 64 * 1024
    warmup, flush = 2, 2
    for itr in range(1, 7):
        bs = [make_batch(cfg, r, itr) for r in range(W)]
        dys = [make_dy(cfg, r, itr) for r in range(W)]
        outs = g.forward([torch.from_numpy(b.ids).cuda() for b in bs], [torch.from_numpy(b.offsets).cuda() for b in bs],
                         [cfg.batch] * W)
        obs = [oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy) for b, dy in zip(bs, dys)]
        for r in range(W):
            ref = oracle.forward(m, obs[r], tabs, cfg.out_width)
            assert np.array_equal(outs[r].cpu().numpy(), ref), f"forward r{r} itr {itr}"
        if itr > warmup:  # hot keys leave the exchange: no requested key is hot, every cold unique is sent
            for e in g.ranks:
                hp, hk = e.hot_keys()
                for p_ in range(e.n_packs):
                    hot = set(hk[hp == p_].tolist())
                    u = e.unique(p_).cpu().numpy()
                    cold = [k for k in u.tolist() if k not in hot]
                    req = []
                    for o in range(W):
                        req += (e.send_list(o, p_) * W + o).tolist()
                    assert not hot.intersection(req), "a hot key was sent to its owner"
                    assert sorted(req) == sorted(cold), "every cold unique key is requested exactly once"
        g.backward_update([torch.from_numpy(d).cuda() for d in dys], lr=0.05, step=itr)
        for e in g.ranks:
            e.check()
        oracle.backward_update(m, obs, tabs, acc, lr=0.05, step=itr)
        _oracle_counts(m, plan, obs, counts, pko)
        if itr >= warmup and itr % flush == 0:  # Alg. 1 L514-517 (reading O13)
            stats = g.hot_cache_refresh(capacity)
            nz = np.nonzero(counts)[0]
            packs = np.searchsorted(pko, nz, side="right") - 1
            sel = oracle.hot_select(packs, nz - pko[packs], counts[nz], cost, capacity)
            exp = nz[sel]
            exp_pack = np.searchsorted(pko, exp, side="right") - 1
            order = np.argsort(exp, kind="stable")  # slots in ascending global key: grouped by pack
            for e in g.ranks:
                pk, ky = e.hot_keys()
                assert np.array_equal(pk, exp_pack[order]) and np.array_equal(ky, (exp - pko[exp_pack])[order])
            assert stats[0]["k"] == len(exp) > 0 and stats[0]["bytes"] <= capacity
    g.hot_cache_refresh(0)  # write back + drop: the shards are the authoritative copy again
    for r, e in enumerate(g.ranks):
        for p, exp in enumerate(shard_expected(e, cfg, tabs, "w", W, r)):
            assert np.array_equal(e.weights[p][:len(exp)].cpu().numpy(), exp), f"weights r{r} p{p}"
        for p, exp in enumerate(shard_expected(e, cfg, acc, "s1", W, r)):
            assert_close(e.state1[p][:len(exp)].cpu().numpy(), exp, what=f"state r{r} p{p}")
    g.close()
