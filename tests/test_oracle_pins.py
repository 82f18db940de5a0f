"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a worked example from the paper/SPEC
(tests/golden/worked_examples.json), a library routine (torch.nn.functional.embedding_bag,
torch.optim.Adagrad / SparseAdam sparse paths), a float64 closed form (dense incidence
matrix Y = A·W, dW = Aᵀ·dY), brute force on tiny inputs, or an invariant.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from datagen import configs as dc
from datagen import make_batch, make_dy, table_values_np

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


# ---------------------------------------------------------------- row mapping (O4)
def test_mix64_known_answers():
    g = GOLD["splitmix64_seed0_outputs"]
    for x, y in zip(g["inputs"], g["outputs"]):
        assert oracle.mix64(int(x, 16)) == int(y, 16)


def test_row_of_modes():
    assert oracle.row_of(oracle.IDS_ROWS, 7, 0, 10) == 7
    with pytest.raises(RuntimeError):
        oracle.row_of(oracle.IDS_ROWS, 10, 0, 10)
    with pytest.raises(RuntimeError):
        oracle.row_of(oracle.IDS_ROWS, -1, 0, 10)
    # HASH: row = floor(mix64(raw^salt) * V / 2^64) -- check against Python big ints
    for raw, salt, V in [(0, 0, 1000), (123456789, 0xABCDEF, 4), (-5, 77, 22274651), (2**62, 1, 2**40)]:
        h = oracle.mix64((raw & (2**64 - 1)) ^ salt)
        assert oracle.row_of(oracle.IDS_HASH, raw, salt, V) == (h * V) >> 64
    # range + rough uniformity: V buckets, chi-square on 20k hashes
    V = 16
    rows = [oracle.row_of(oracle.IDS_HASH, i, 99, V) for i in range(20000)]
    assert min(rows) >= 0 and max(rows) < V
    cnt = np.bincount(rows, minlength=V)
    chi2 = ((cnt - 1250.0) ** 2 / 1250.0).sum()
    assert chi2 < 50  # 15 dof, p ~ 1e-5


# ---------------------------------------------------------------- unique / partition
def test_unique_spec_examples():
    for ex in GOLD["unique"]:
        u, inv = oracle.unique(np.array(ex["ids"], np.int64))
        assert u.tolist() == ex["unique"] and inv.tolist() == ex["inverse"]


def _brute_unique(keys):
    uniq, inv = [], []
    for k in keys:
        for i, v in enumerate(uniq):
            if v == k:
                inv.append(i)
                break
        else:
            uniq.append(k)
            inv.append(len(uniq) - 1)
    return uniq, inv


@pytest.mark.parametrize("seed", range(5))
def test_unique_brute_force(seed):
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, 40, 300).astype(np.int64)
    u, inv = oracle.unique(keys)
    bu, binv = _brute_unique(keys.tolist())
    assert u.tolist() == bu and inv.tolist() == binv
    assert (u[inv] == keys).all()  # round trip
    assert len(u) == len(set(keys.tolist()))  # |unique| == #distinct (north star invariant)


def test_partition_spec_examples():
    for ex in GOLD["partition"]:
        keys, lrow, counts = oracle.partition(np.array(ex["ids"], np.int64), ex["n"])
        parts, s = [], 0
        for c in counts:
            parts.append(keys[s:s + c].tolist())
            s += c
        assert parts == ex["parts"]
        assert (lrow == keys // ex["n"]).all()


def test_partition_completeness():
    rng = np.random.default_rng(3)
    u = np.unique(rng.integers(0, 10**9, 1000))
    rng.shuffle(u)
    for W in (1, 2, 3, 8):
        keys, lrow, counts = oracle.partition(u, W)
        assert sorted(keys.tolist()) == sorted(u.tolist())
        s = 0
        for w in range(W):
            part = keys[s:s + counts[w]]
            assert (part % W == w).all()
            # stable: owner list keeps unique order
            pos = {k: i for i, k in enumerate(u.tolist())}
            assert [pos[k] for k in part.tolist()] == sorted(pos[k] for k in part.tolist())
            s += counts[w]


# ---------------------------------------------------------------- forward
def _tiny_model(F, T, rows, dims, f2t=None, pool=oracle.POOL_SUM, mode=oracle.IDS_ROWS, salt=None):
    f2t = np.arange(F) if f2t is None else np.asarray(f2t)
    dims = np.asarray(dims)
    col = np.concatenate([[0], np.cumsum(dims[f2t])[:-1]])
    return oracle.OracleModel(f2t, rows, dims, col, id_mode=mode, pool=pool, table_salt=salt), int(dims[f2t].sum())


def test_segment_reduction_spec_examples():
    for ex in GOLD["segment_reduction"]:
        rows = np.array(ex["rows"], np.float32)
        pool = oracle.POOL_SUM if ex["mode"] == "sum" else oracle.POOL_MEAN
        m, width = _tiny_model(1, 1, [3], [2], pool=pool)
        seg = ex["segments"]
        B = max(seg) + 1
        offsets = np.searchsorted(seg, np.arange(B + 1)).astype(np.int32)
        b = oracle.OracleBatch(B, np.arange(3), offsets)
        out = oracle.forward(m, b, [rows], width)
        assert out.tolist() == ex["out"]


def _random_case(seed, F=5, T=3, B=17, V=(11, 7, 23), D=(4, 8, 4), maxlen=6, pool=oracle.POOL_SUM,
                 mode=oracle.IDS_ROWS, ids_seed=None):
    rng = np.random.default_rng(seed)
    f2t = rng.integers(0, T, F)
    f2t[:T] = np.arange(T)  # every table used
    m, width = _tiny_model(F, T, V, D, f2t=f2t, pool=pool, mode=mode,
                           salt=rng.integers(0, 2**63, T).astype(np.uint64))
    if ids_seed is not None:
        rng = np.random.default_rng(ids_seed)
    lengths = rng.integers(0, maxlen + 1, (F, B))
    offsets = np.concatenate([[0], np.cumsum(lengths.reshape(-1))]).astype(np.int32)
    ids = np.empty(offsets[-1], np.int64)
    for f in range(F):
        lo, hi = offsets[f * B], offsets[(f + 1) * B]
        if mode == oracle.IDS_ROWS:
            ids[lo:hi] = rng.integers(0, V[f2t[f]], hi - lo)
        else:
            ids[lo:hi] = rng.integers(-2**62, 2**62, hi - lo)
    tables = [rng.standard_normal((V[t], D[t])).astype(np.float32) for t in range(T)]
    return m, width, B, ids, offsets, tables, f2t, lengths


def _rows_of(m, ids, f2t, f, offsets, B):
    t = f2t[f]
    lo, hi = offsets[f * B], offsets[(f + 1) * B]
    return np.array([oracle.row_of(m.id_mode, int(x), int(m.salt[t]), int(m.rows[t])) for x in ids[lo:hi]], np.int64)


@pytest.mark.parametrize("pool", [oracle.POOL_SUM, oracle.POOL_MEAN])
@pytest.mark.parametrize("mode", [oracle.IDS_ROWS, oracle.IDS_HASH])
def test_forward_vs_embedding_bag(pool, mode):
    """Library routine pin: torch.nn.functional.embedding_bag (CPU) per field, same fp32."""
    for seed in range(4):
        m, width, B, ids, offsets, tables, f2t, lengths = _random_case(seed, pool=pool, mode=mode)
        b = oracle.OracleBatch(B, ids, offsets)
        out = oracle.forward(m, b, tables, width)
        for f in range(m.F):
            rows = _rows_of(m, ids, f2t, f, offsets, B)
            off = torch.tensor(offsets[f * B:(f + 1) * B] - offsets[f * B], dtype=torch.int64)
            ref = torch.nn.functional.embedding_bag(torch.tensor(rows), torch.tensor(tables[f2t[f]]), off,
                                                    mode="sum" if pool == oracle.POOL_SUM else "mean")
            c = int(m.col[f])
            np.testing.assert_allclose(out[:, c:c + tables[f2t[f]].shape[1]], ref.numpy(), rtol=1e-6, atol=1e-6)


def test_forward_dense_incidence_float64():
    """Closed form Y_f = A_f · W_t in float64 (A_f = B x V incidence counts); fp32 sequential
    sums lie within n*eps*sum|terms| of it; with dyadic tables the sums are exact."""
    for seed in range(3):
        m, width, B, ids, offsets, tables, f2t, lengths = _random_case(seed, maxlen=9)
        dy_tabs = [np.round(t * 64).astype(np.float32) / np.float32(64) for t in tables]
        for tabs, exact in ((tables, False), (dy_tabs, True)):
            out = oracle.forward(m, oracle.OracleBatch(B, ids, offsets), tabs, width)
            for f in range(m.F):
                t = f2t[f]
                A = np.zeros((B, m.rows[t]))
                rows = _rows_of(m, ids, f2t, f, offsets, B)
                for bb in range(B):
                    for j in range(offsets[f * B + bb], offsets[f * B + bb + 1]):
                        A[bb, rows[j - offsets[f * B]]] += 1
                Y = A @ tabs[t].astype(np.float64)
                Yabs = A @ np.abs(tabs[t].astype(np.float64))
                c = int(m.col[f])
                got = out[:, c:c + tabs[t].shape[1]].astype(np.float64)
                if exact:
                    assert (got == Y).all()
                else:
                    assert (np.abs(got - Y) <= 10 * 2**-24 * Yabs + 1e-30).all()


def test_forward_empty_bags_are_zero():
    m, width = _tiny_model(2, 2, [5, 5], [4, 4], pool=oracle.POOL_MEAN)
    B = 3
    offsets = np.array([0, 0, 2, 2, 2, 2, 3], np.int32)
    ids = np.array([1, 2, 4], np.int64)
    tabs = [np.ones((5, 4), np.float32), np.full((5, 4), 2.0, np.float32)]
    out = oracle.forward(m, oracle.OracleBatch(B, ids, offsets), tabs, width)
    assert (out[0] == 0).all() and (out[1, :4] == 1).all() and (out[2, :4] == 0).all()
    assert (out[:2, 4:] == 0).all() and (out[2, 4:] == 2).all()


def test_forward_sampled_matches_full():
    m, width, B, ids, offsets, tables, f2t, _ = _random_case(7, mode=oracle.IDS_HASH)
    b = oracle.OracleBatch(B, ids, offsets)
    full = oracle.forward(m, b, tables, width)
    rng = np.random.default_rng(0)
    qf = rng.integers(0, m.F, 30).astype(np.int32)
    qs = rng.integers(0, B, 30).astype(np.int32)
    rt, rr = oracle.segment_rows(m, b, qf, qs)
    ld = int(max(m.dims))
    rv = np.zeros((len(rt), ld), np.float32)
    for i, (t, r) in enumerate(zip(rt, rr)):
        rv[i, :m.dims[t]] = tables[t][r]
    got = oracle.forward_sampled(m, b, rt, rr, rv, qf, qs)
    for i in range(30):
        D = m.dims[f2t[qf[i]]]
        c = int(m.col[qf[i]])
        assert (got[i, :D] == full[qs[i], c:c + D]).all()


# ---------------------------------------------------------------- backward + update
def _grads_via_torch(m, f2t, ids, offsets, B, dy_list, pool):
    """torch EmbeddingBag(sparse) autograd gradient over all ranks' batches (library pin)."""
    T = len(m.rows)
    G = [np.zeros((m.rows[t], m.dims[t]), np.float64) for t in range(T)]
    for (ids_r, off_r, dy) in dy_list:
        for f in range(m.F):
            t = f2t[f]
            rows = _rows_of(m, ids_r, f2t, f, off_r, B)
            W = torch.zeros((int(m.rows[t]), int(m.dims[t])), dtype=torch.float64, requires_grad=True)
            off = torch.tensor(off_r[f * B:(f + 1) * B] - off_r[f * B], dtype=torch.int64)
            y = torch.nn.functional.embedding_bag(torch.tensor(rows), W, off,
                                                  mode="sum" if pool == oracle.POOL_SUM else "mean")
            c = int(m.col[f])
            y.backward(torch.tensor(dy[:, c:c + int(m.dims[t])], dtype=torch.float64))
            G[t] += W.grad.numpy()
    return G


@pytest.mark.parametrize("pool", [oracle.POOL_SUM, oracle.POOL_MEAN])
def test_table_grad_vs_autograd(pool):
    """dW = Aᵀ·dY (float64 autograd through embedding_bag); exact for dyadic dY with sum."""
    R = 2
    m, width, B, ids0, off0, tables, f2t, _ = _random_case(11, pool=pool)
    rng = np.random.default_rng(5)
    batches, dl = [], []
    for r in range(R):
        _, _, _, ids, off, _, _, _ = _random_case(11, pool=pool, ids_seed=100 + r)
        dy = (rng.integers(-7, 8, (B, width)) * 2.0 ** -8).astype(np.float32)
        batches.append(oracle.OracleBatch(B, ids, off, dy))
        dl.append((ids, off, dy))
    ref = _grads_via_torch(m, f2t, None, None, B, dl, pool)
    for t in range(len(m.rows)):
        G, cnt = oracle.table_grad(m, batches, t)
        if pool == oracle.POOL_SUM:
            assert (G.astype(np.float64) == ref[t]).all()
        else:
            np.testing.assert_allclose(G, ref[t], rtol=1e-5, atol=1e-6)
        assert cnt.sum() == sum(int(b.offsets[(f + 1) * B] - b.offsets[f * B])
                                for b in batches for f in range(m.F) if f2t[f] == t)


def _torch_sparse_step(kind, W0, S0, G, touched, lr, step):
    """Apply torch's own sparse optimizer (one step, number `step`) to W0 with sparse grad
    rows `touched`, starting from optimizer state S0."""
    W = torch.nn.Parameter(torch.tensor(W0))
    idx = torch.tensor(np.nonzero(touched)[0], dtype=torch.int64)
    if kind == oracle.OPT_ADAGRAD:
        opt = torch.optim.Adagrad([W], lr=lr, initial_accumulator_value=0.0, eps=1e-10)
        opt.state[W]["sum"] = torch.tensor(S0[0]).clone()
        opt.state[W]["step"] = torch.tensor(float(step - 1))
    else:
        opt = torch.optim.SparseAdam([W], lr=lr, betas=(0.9, 0.999), eps=1e-8)
        st = opt.state[W]
        st["step"] = step - 1
        st["exp_avg"] = torch.tensor(S0[0]).clone()
        st["exp_avg_sq"] = torch.tensor(S0[1]).clone()
    W.grad = torch.sparse_coo_tensor(idx[None], torch.tensor(G[idx.numpy()]), W0.shape)
    opt.step()
    st = opt.state[W]
    if kind == oracle.OPT_ADAGRAD:
        return W.detach().numpy(), [st["sum"].numpy()]
    return W.detach().numpy(), [st["exp_avg"].numpy(), st["exp_avg_sq"].numpy()]


@pytest.mark.parametrize("kind", [oracle.OPT_ADAGRAD, oracle.OPT_ADAM])
@pytest.mark.parametrize("step", [1, 3])
def test_update_vs_torch_sparse_optimizers(kind, step):
    m, width, B, ids, off, tables, f2t, _ = _random_case(21)
    rng = np.random.default_rng(9)
    dy = rng.uniform(-1, 1, (B, width)).astype(np.float32)
    b = oracle.OracleBatch(B, ids, off, dy)
    T = len(m.rows)
    W = [t.copy() for t in tables]
    if kind == oracle.OPT_ADAGRAD:
        S1 = [np.full_like(t, 0.1) for t in tables]
        S2 = None
    else:
        S1 = [rng.uniform(-0.1, 0.1, t.shape).astype(np.float32) for t in tables]
        S2 = [rng.uniform(0.0, 0.1, t.shape).astype(np.float32) for t in tables]
    W0 = [w.copy() for w in W]
    S10 = [s.copy() for s in S1]
    S20 = [s.copy() for s in S2] if S2 else None
    oracle.backward_update(m, [b], W, S1, S2, kind=kind, lr=0.05, step=step)
    for t in range(T):
        G, cnt = oracle.table_grad(m, [b], t)
        touched = cnt > 0
        S0 = [S10[t]] if S2 is None else [S10[t], S20[t]]
        Wt, St = _torch_sparse_step(kind, W0[t], S0, G, touched, 0.05, step)
        np.testing.assert_allclose(W[t], Wt, rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(S1[t], St[0], rtol=1e-5, atol=1e-6)
        if S2:
            np.testing.assert_allclose(S2[t], St[1], rtol=1e-5, atol=1e-6)
        # an update touches only looked-up rows: others bitwise unchanged (north star)
        assert (W[t][~touched] == W0[t][~touched]).all()
        assert (S1[t][~touched] == S10[t][~touched]).all()
        assert (W[t][touched] != W0[t][touched]).any()


def test_row_grads_and_apply_update_match_full():
    m, width, B, ids, off, tables, f2t, _ = _random_case(31, mode=oracle.IDS_HASH)
    dy = np.random.default_rng(1).uniform(-1, 1, (B, width)).astype(np.float32)
    b = oracle.OracleBatch(B, ids, off, dy)
    ld = int(max(m.dims))
    qt = np.array([0, 0, 1, 2, 2, 1], np.int32)
    qr = np.array([0, 3, 5, 22, 7, 1], np.int64)
    G, cnt = oracle.row_grads(m, [b], qt, qr, ld)
    for i in range(len(qt)):
        Gf, cf = oracle.table_grad(m, [b], int(qt[i]))
        assert cnt[i] == cf[qr[i]]
        assert (G[i, :m.dims[qt[i]]] == Gf[qr[i]]).all()
    W = [t.copy() for t in tables]
    S = [np.full_like(t, 0.1) for t in tables]
    oracle.backward_update(m, [b], W, S, lr=0.1)
    for i in range(len(qt)):
        D = int(m.dims[qt[i]])
        w = np.zeros((1, ld), np.float32)
        s = np.zeros((1, ld), np.float32)
        w[0, :D] = tables[qt[i]][qr[i]]
        s[0, :D] = 0.1
        oracle.apply_update(G[i:i + 1], cnt[i:i + 1], w, s, lr=0.1, D=D)
        assert (w[0, :D] == W[qt[i]][qr[i]]).all()


# ---------------------------------------------------------------- Eq. 1 / plan
def test_calc_vparam_spec_example():
    g = GOLD["calc_vparam"]
    assert oracle.calc_vparam(g["dims"], g["freq_sums"], g["N"]) == g["vparam"]
    # linear in N and in t_dim
    assert oracle.calc_vparam([8], [1.0], 50) * 4 == oracle.calc_vparam([32], [1.0], 50)
    assert oracle.calc_vparam([8], [1.0], 100) == 2 * oracle.calc_vparam([8], [1.0], 50)


def test_plan_four_shards_paper_example():
    g = GOLD["four_shards"]
    dims = np.array(g["table_dim"], np.int32)
    T = len(dims)
    p = oracle.pack_plan(np.arange(T), np.full(T, 100), dims, split=True)
    pd = p["pack_dim"]
    assert (pd == 8).sum() == g["packs_for_dim"]["8"] and (pd == 32).sum() == g["packs_for_dim"]["32"]
    for q in np.nonzero(pd == 32)[0]:
        assert (p["table_to_pack"] == q).sum() == g["tables_per_dim32_shard"]
    p0 = oracle.pack_plan(np.arange(T), np.full(T, 100), dims, split=False)
    assert p0["n_packs"] == 2


def test_plan_coverage_and_bases():
    cfg = dc.industrial()
    p = oracle.pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim, split=True)
    t2p, tb = p["table_to_pack"], p["table_base"]
    for q in range(p["n_packs"]):
        tabs = np.nonzero(t2p == q)[0]
        assert (cfg.table_dim[tabs] == p["pack_dim"][q]).all()
        # bases are the running row sum in ascending table order; key ranges tile the pack
        assert (tb[tabs] == np.concatenate([[0], np.cumsum(cfg.table_rows[tabs])[:-1]])).all()
        assert p["pack_rows"][q] == cfg.table_rows[tabs].sum()
    assert (p["field_to_pack"] == t2p[cfg.field_to_table]).all()
    assert sorted(set(t2p.tolist())) == list(range(p["n_packs"]))


# ---------------------------------------------------------------- Alg. 1 hot set
def test_hybridhash_hand_trace():
    g = GOLD["hybridhash_trace"]
    counts = np.zeros(64, np.uint64)
    # itr 0 (warm-up) and itr 1: count post-unique, then flush after itr 1 (itr >= warmup)
    for itr, ids in enumerate(g["iters"][:2]):
        oracle.fcounter_add(np.array(ids, np.int64), counts)
    keys = np.nonzero(counts)[0]
    sel = oracle.hot_select(np.zeros(len(keys)), keys, counts[keys], [16], 16)  # capacity = 1 row
    assert keys[sel].tolist() == g["hot_after_itr1"]
    hot = set(keys[sel].tolist())
    assert [k in hot for k in g["iters"][2]] == [True, False]


def test_hot_select_brute_force():
    rng = np.random.default_rng(0)
    n = 500
    pk = rng.choice(3 * 1000, n, replace=False)  # distinct (pack, key) pairs
    pack, key = pk // 1000, pk % 1000
    count = rng.integers(0, 6, n).astype(np.uint64)
    cost = np.array([32, 64, 128])
    for cap in (0, 100, 1000, 10**6):
        sel = oracle.hot_select(pack, key, count, cost, cap)
        order = sorted([i for i in range(n) if count[i] > 0], key=lambda i: (-int(count[i]), pack[i], key[i]))
        used, ref = 0, []
        for i in order:
            if used + cost[pack[i]] > cap:
                break
            used += cost[pack[i]]
            ref.append(i)
        assert sel.tolist() == ref


# ---------------------------------------------------------------- packed == unpacked (plan invariance)
def test_packed_key_streams_partition_fields():
    cfg = dc.scaled(dc.wdl(), batch=8, rows_div=10**4)
    b = make_batch(cfg, 0, 0)
    m = oracle.OracleModel(cfg.field_to_table, cfg.table_rows, cfg.table_dim, cfg.field_col,
                           id_mode=cfg.id_mode, pool=cfg.pool, table_salt=cfg.table_salt)
    ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets)
    for split in (False, True):
        p = oracle.pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim, split=split)
        total = 0
        for q in range(p["n_packs"]):
            keys = oracle.pack_key_stream(m, p["field_to_pack"], p["table_base"], ob, q)
            assert keys.min() >= 0 and keys.max() < p["pack_rows"][q]
            total += len(keys)
        assert total == b.n_ids


# ---------------------------------------------------------------- generator pins
def test_zipf_head_coverage_closed_form():
    from datagen import ZipfSampler, zipf_head_mass
    for V, a in [(1000, 1.0), (100000, 0.8), (2_000_000, 0.8), (50, 1.4)]:
        r = ZipfSampler(V, a).sample(np.random.default_rng(1), 200_000)
        assert r.min() >= 1 and r.max() <= V
        emp = (r <= int(np.ceil(0.2 * V))).mean()
        assert abs(emp - zipf_head_mass(V, a, 0.2)) < 0.02
    # alpha 0.8 reproduces "20% of IDs cover 70%" at V >= 1e5
    assert 0.69 <= zipf_head_mass(100000, 0.8, 0.2) <= 0.72


def test_table_values_numpy_torch_identical():
    from datagen import table_values_torch
    rows = np.array([0, 1, 5, 2**33 + 7, 46_874_998])
    a = table_values_np(7, 3, rows, 16)
    b = table_values_torch(7, 3, torch.tensor(rows), 16).numpy()
    assert (a == b).all() and a.min() >= -0.05 and a.max() < 0.05


def test_batches_deterministic():
    cfg = dc.toy()
    a, b = make_batch(cfg, 0, 3), make_batch(cfg, 0, 3)
    c = make_batch(cfg, 1, 3)
    assert (a.ids == b.ids).all() and (a.offsets == b.offsets).all()
    assert not np.array_equal(a.ids, c.ids)
    assert (a.lengths == 0).any()  # toy has empty bags
    dy = make_dy(cfg, 0, 0)
    assert (dy * 256 == np.round(dy * 256)).all()


# ---------------------------------------------------------------- reading O2: the pack key stream order
def _o2_model_batch():
    g = GOLD["key_stream_o2"]
    F = len(g["field_to_table"])
    dims = np.array(g["table_dim"], np.int64)
    col = np.concatenate([[0], np.cumsum(dims[g["field_to_table"]])[:-1]])
    m = oracle.OracleModel(g["field_to_table"], g["table_rows"], g["table_dim"], col, id_mode=dc.IDS_ROWS,
                           pool=dc.POOL_SUM)
    ob = oracle.OracleBatch(g["batch"], np.array(g["ids"], np.int64), np.array(g["offsets"], np.int32))
    assert len(g["offsets"]) == F * g["batch"] + 1
    return g, m, ob


def test_o2_key_stream_golden():
    """Hand-derived key stream / unique / inverse of a 2-pack, 4-field batch (fields sharing a
    table dedupe together, fields of another pack are skipped, an empty bag).  Swapping the
    stream to sample-major, or the fields' order, changes the unique order and fails here."""
    g, m, ob = _o2_model_batch()
    for p, exp in enumerate(g["packs"]):
        keys = oracle.pack_key_stream(m, g["field_to_pack"], g["table_base"], ob, p)
        assert keys.tolist() == exp["key_stream"]
        u, inv = oracle.unique(keys)
        assert u.tolist() == exp["unique"] and inv.tolist() == exp["inverse"]
        k, lrow, cnt = oracle.partition(u, 2)
        ex = exp["partition_W2"]
        assert k.tolist() == ex["owner_keys"][0] + ex["owner_keys"][1]
        assert lrow.tolist() == ex["local_rows"][0] + ex["local_rows"][1]
        assert cnt.tolist() == ex["counts"]


def test_o2_plan_reproduces_golden_layout():
    """The oracle planner gives the golden's pack / table_base layout (one pack per dim)."""
    g, m, ob = _o2_model_batch()
    p = oracle.pack_plan(g["field_to_table"], g["table_rows"], g["table_dim"])
    assert p["field_to_pack"].tolist() == g["field_to_pack"]
    assert p["table_base"].tolist() == g["table_base"]


# ---------------------------------------------------------------- reading O12: hot-set tie-break
def test_hot_select_tie_golden():
    g = GOLD["hot_select_ties"]
    pk, ky, ct = np.array(g["pack"]), np.array(g["key"]), np.array(g["count"], np.uint64)
    for c in g["cases"]:
        sel = oracle.hot_select(pk, ky, ct, g["row_cost_bytes"], c["capacity"])
        assert [[int(pk[i]), int(ky[i])] for i in sel] == c["hot"], c


# ---------------------------------------------------------------- reading O6: fp64 accumulation
def test_near_cancelling_gradient_is_the_rounded_exact_sum():
    """A hot row whose gradient nearly cancels: 4001 occurrences of +1 / -1 (+ 2^-20 perturbations)
    and one tiny term.  A fp32 running sum loses the tiny term (and its sign); the oracle's G must be
    fp32(exact rational sum) — reading O6 (fp64 accumulation, rounded once), computed here with
    Python Fractions, independently of the oracle."""
    from fractions import Fraction

    rng = np.random.default_rng(5)
    n = 4001
    vals = rng.uniform(-1, 1, n).astype(np.float32)
    vals[0], vals[1] = np.float32(1e4), np.float32(-1e4)  # a large partial sum early on
    vals[2:2000:2] += np.float32(3e3)
    vals[3:2000:2] -= np.float32(3e3)
    rest = float(sum(Fraction(float(v)) for v in vals[:-1]))
    vals[-1] = np.float32(-rest)  # total = the rounding residue of the last term: tiny
    # one table, one row, one field: sample b holds the row once with dY[b] = vals[b]
    D = 4
    m = oracle.OracleModel([0], [3], [D], [0], id_mode=dc.IDS_ROWS, pool=dc.POOL_SUM)
    ids = np.ones(n, np.int64)
    off = np.arange(n + 1, dtype=np.int32)
    dy = np.repeat(vals[:, None], D, axis=1).astype(np.float32)
    ob = oracle.OracleBatch(n, ids, off, dy)
    G, cnt = oracle.table_grad(m, [ob], 0)
    exact = sum((Fraction(float(v)) for v in vals), Fraction(0))
    ref = np.float32(float(exact))  # float(Fraction) is correctly rounded; the sum is far inside fp64
    assert cnt[1] == n and cnt[0] == 0 and cnt[2] == 0
    assert (G[1] == ref).all(), (G[1], ref)
    run = np.float32(0)
    for v in vals:
        run = np.float32(run + v)
    assert run != ref  # the plain fp32 running sum misses it: the case reading O6 fixes


# ---------------------------------------------------------------- the all-cores baseline build
def test_openmp_build_is_bitwise_the_plain_oracle():
    """bench.py's all-cores CPU baseline runs the oracle built with -fopenmp; its sampled forward,
    row gradients and update must be bitwise those of the plain build (same per-row order)."""
    cfg = dc.scaled(dc.wdl(), batch=64, rows_div=2000)
    b, dy = make_batch(cfg, 0, 0), make_dy(cfg, 0, 0, dyadic=False)
    res = []
    for omp in (False, True):
        oracle.use_openmp(omp)
        try:
            m = oracle.OracleModel(cfg.field_to_table, cfg.table_rows, cfg.table_dim, cfg.field_col,
                                   id_mode=cfg.id_mode, pool=cfg.pool, table_salt=cfg.table_salt)
            ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)
            qf = np.repeat(np.arange(cfg.F, dtype=np.int32), cfg.batch)
            qs = np.tile(np.arange(cfg.batch, dtype=np.int32), cfg.F)
            rt, rr = oracle.segment_rows(m, ob, qf, qs)
            key = np.unique(rt.astype(np.int64) * (1 << 40) + rr)
            ut, ur = (key >> 40).astype(np.int32), key & ((1 << 40) - 1)
            ld = int(cfg.table_dim.max())
            vals = np.zeros((len(key), ld), np.float32)
            for t in np.unique(ut):
                sel = ut == t
                vals[sel, :cfg.table_dim[t]] = table_values_np(cfg.seed, int(t), ur[sel], int(cfg.table_dim[t]))
            out = oracle.forward_sampled(m, ob, ut, ur, vals, qf, qs)
            G, cnt = oracle.row_grads(m, [ob], ut, ur, ld)
            acc = np.full_like(vals, 0.1)
            oracle.apply_update(G, cnt, vals, acc, lr=0.01, D=ld)
            res.append((out, G, cnt, vals, acc))
        finally:
            oracle.use_openmp(False)
    for a, c in zip(*res):
        assert np.array_equal(a, c)


# ---------------------------------------------------------------- K-Interleaving (Eq. 3, reading O22)
def test_eq3_capacity_and_kinterleave_plan_golden():
    g = GOLD["kinterleave_plan"]
    assert oracle.interleave_capacity(g["rbound"], g["rparam"]) == g["capacity"]
    assert oracle.interleave_capacity([5.0, 7.0], [0.0, 0.0]) == float("inf")  # nothing binds
    p = oracle.kinterleave_plan(g["field_to_table"], g["table_rows"], g["table_dim"], g["capacity"], g["excluded"])
    for k in ("table_to_pack", "table_base", "pack_dim", "pack_rows", "pack_group"):
        assert p[k].tolist() == g[k], k
    assert p["n_groups"] == g["n_groups"]
    p40 = oracle.kinterleave_plan(g["field_to_table"], g["table_rows"], g["table_dim"], 40.0, g["excluded"])
    assert p40["table_to_pack"].tolist() == g["capacity_40"]["table_to_pack"]
    assert p40["pack_group"].tolist() == g["capacity_40"]["pack_group"]


def test_kinterleave_plan_invariants():
    """Every pack's volume and every group's volume stay within the capacity unless a single table
    (resp. pack) exceeds it; excluded tables never share a pack with others; no capacity = D-Packing."""
    cfg = dc.scaled(dc.industrial(), batch=8, rows_div=10**4)
    rng = np.random.default_rng(3)
    cnt = rng.integers(1, 1000, cfg.T).astype(np.uint64)
    vol = cfg.table_dim.astype(float) * cnt
    ex = (rng.random(cfg.T) < 0.1).astype(np.uint8)
    for cap in (vol.max() * 0.5, vol.sum() / 7, vol.sum() / 3, float("inf")):
        p = oracle.kinterleave_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim, cap, ex, cnt)
        pv = np.bincount(p["table_to_pack"], weights=vol, minlength=p["n_packs"])
        ntab = np.bincount(p["table_to_pack"], minlength=p["n_packs"])
        pg = p["pack_group"]
        assert (pg[:ex.any() and len(set(cfg.table_dim[ex == 1]))] == -1).all()
        for q in range(p["n_packs"]):
            members = np.nonzero(p["table_to_pack"] == q)[0]
            assert len(set(ex[members])) == 1 and len(set(cfg.table_dim[members])) == 1
            if pg[q] >= 0 and np.isfinite(cap):  # within capacity, or as small as the dealing allows
                assert pv[q] <= cap or ntab[q] == 1 or pv[q] <= np.ceil(vol[members].sum() / cap) * cap
        gv = np.bincount(pg[pg >= 0], weights=pv[pg >= 0])
        gn = np.bincount(pg[pg >= 0])
        assert ((gv <= cap) | (gn == 1)).all()
        assert list(pg[pg >= 0]) == sorted(pg[pg >= 0])  # contiguous, ascending
    pinf = oracle.kinterleave_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim, float("inf"), None, cnt)
    p0 = oracle.pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim, warmup_count=cnt)
    assert pinf["table_to_pack"].tolist() == p0["table_to_pack"].tolist() and pinf["n_groups"] == 1
