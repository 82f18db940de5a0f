"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Bit-exact: row mapping/dedup/inverse, forward pooling (sequential order by design).
fp32 update: within 1e-5 rel / 1e-6 abs (north star), and bit-exact under dyadic dY
(reading O19) for rows whose occurrences are summed in ascending order."""
import numpy as np
import pytest
import torch

import oracle
from datagen import configs as dc
from datagen import make_batch, make_dy, table_values_np
from harness import (assert_close, gpu_embedding, gpu_table_rows, oracle_model, oracle_tables, to_dev)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__

    __graft_entry__.build()


def run_step(cfg, opt=oracle.OPT_ADAGRAD, dyadic=True, steps=1, lr=0.05, split=False, batch_fn=None,
             check_intermediates=True):
    """Run `steps` fwd+bwd steps on both sides; compare every step."""
    emb = gpu_embedding(cfg, opt=opt, split=split)
    m = oracle_model(cfg)
    tabs = oracle_tables(cfg)
    if opt == oracle.OPT_ADAGRAD:
        s1, s2 = [np.full_like(t, 0.1) for t in tabs], None
    else:
        s1, s2 = [np.zeros_like(t) for t in tabs], [np.zeros_like(t) for t in tabs]
    for step in range(1, steps + 1):
        b = batch_fn(step) if batch_fn else make_batch(cfg, 0, step)
        dy = make_dy(cfg, 0, step, dyadic=dyadic)
        ids, off = to_dev(b)
        out = emb.forward(ids, off, cfg.batch)
        ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)
        ref = oracle.forward(m, ob, tabs, cfg.out_width)
        got = out.cpu().numpy()
        assert np.array_equal(got, ref), f"forward not bit-exact at step {step}: max |d| {np.abs(got - ref).max()}"
        if check_intermediates:
            for p in range(emb.n_packs):
                keys = oracle.pack_key_stream(m, emb.plan["field_to_pack"], emb.plan["table_base"], ob, p)
                u_ref, inv_ref = oracle.unique(keys)
                assert np.array_equal(emb.unique(p).cpu().numpy(), u_ref), f"unique pack {p}"
                assert np.array_equal(emb.inverse(p).cpu().numpy(), inv_ref), f"inverse pack {p}"
        emb.backward_update(torch.from_numpy(dy).cuda(), lr=lr, step=step)
        emb.check()
        oracle.backward_update(m, [ob], tabs, s1, s2, kind=opt, lr=lr, step=step)
        for t in range(cfg.T):
            gw = gpu_table_rows(emb, cfg, t, "w")
            if dyadic:  # reading O19: every partial sum is exact, so the update is bit-exact
                assert np.array_equal(gw, tabs[t]), f"table {t} step {step}: dyadic dY must be bit-exact"
                assert np.array_equal(gpu_table_rows(emb, cfg, t, "s1"), s1[t]), f"state1 t{t} step {step}"
            assert_close(gw, tabs[t], what=f"weights t{t} step {step}")
            assert_close(gpu_table_rows(emb, cfg, t, "s1"), s1[t], what=f"state1 t{t}")
            if s2:
                assert_close(gpu_table_rows(emb, cfg, t, "s2"), s2[t], what=f"state2 t{t}")
    return emb, tabs


def test_o2_golden_through_abi():
    """The hand-derived key stream of tests/golden (reading O2) through the C ABI: the GPU's
    per-pack unique and inverse equal the golden values directly (not via the oracle)."""
    import json
    import os

    import paper_2204_04903_b200 as pb

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))["key_stream_o2"]
    emb = pb.PackedEmbedding(g["field_to_table"], g["table_rows"], g["table_dim"], max_batch=g["batch"],
                             max_ids=64, id_mode=dc.IDS_ROWS)
    assert emb.plan["table_base"].tolist() == g["table_base"]
    ids = torch.tensor(g["ids"], dtype=torch.int64, device="cuda")
    off = torch.tensor(g["offsets"], dtype=torch.int32, device="cuda")
    emb.forward(ids, off, g["batch"])
    emb.check()
    for p, exp in enumerate(g["packs"]):
        assert emb.unique(p).cpu().tolist() == exp["unique"], p
        assert emb.inverse(p).cpu().tolist() == exp["inverse"], p


# ------------------------------------------------------------------------------------------
def test_toy_sum_adagrad_bit_exact():
    cfg = dc.toy()
    emb = gpu_embedding(cfg)
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    b, dy = make_batch(cfg, 0, 0), make_dy(cfg, 0, 0)
    ids, off = to_dev(b)
    out = emb.forward(ids, off, cfg.batch).cpu().numpy()
    ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)
    assert np.array_equal(out, oracle.forward(m, ob, tabs, cfg.out_width))
    w0 = [gpu_table_rows(emb, cfg, t) for t in range(cfg.T)]
    emb.backward_update(torch.from_numpy(dy).cuda(), lr=0.05, step=1)
    emb.check()
    acc = [np.full_like(t, 0.1) for t in tabs]
    oracle.backward_update(m, [ob], tabs, acc, lr=0.05)
    for t in range(cfg.T):
        _, cnt = oracle.table_grad(m, [ob], t)
        gw = gpu_table_rows(emb, cfg, t)
        assert np.array_equal(gw, tabs[t]), f"table {t}: dyadic dY must give a bit-exact update"
        assert np.array_equal(gpu_table_rows(emb, cfg, t, "s1"), acc[t])
        # an update touches only looked-up rows
        assert np.array_equal(gw[cnt == 0], w0[t][cnt == 0])
        assert not np.array_equal(gw[cnt > 0], w0[t][cnt > 0])


@pytest.mark.parametrize("pool", [dc.POOL_SUM, dc.POOL_MEAN])
@pytest.mark.parametrize("mode", [dc.IDS_HASH, dc.IDS_ROWS])
def test_toy_pool_modes_three_steps(pool, mode):
    run_step(dc.toy(pool=pool, id_mode=mode), steps=3, dyadic=(pool == dc.POOL_SUM))


def test_toy_continuous_dy():
    run_step(dc.toy(), dyadic=False, steps=2)


@pytest.mark.parametrize("steps", [1, 3])
def test_toy_adam_lazy(steps):
    run_step(dc.toy(), opt=oracle.OPT_ADAM, steps=steps, dyadic=False, lr=0.01)


def test_multipack_wdl_small():
    cfg = dc.scaled(dc.wdl(), batch=48, rows_div=1000)  # 200 fields, 4 packs, bags 1..50
    run_step(cfg, steps=2)


def test_dedup_per_table_regions(monkeypatch):
    """The per-table hash regions of large batches (forced on a small one): same unique / inverse
    (bit-exact, checked per pack) and the same step."""
    monkeypatch.setenv("PICASSO_DEDUP_REGIONS", "1")
    monkeypatch.setenv("PICASSO_INDEX", "hash")
    cfg = dc.scaled(dc.wdl(), batch=40, rows_div=1000)
    run_step(cfg, steps=2)
    run_step(dc.toy(), steps=2)


def test_multipack_split_plan_same_results():
    cfg = dc.scaled(dc.wdl(), batch=32, rows_div=2000)
    b = make_batch(cfg, 0, 1)
    outs = []
    for split in (False, True):
        emb = gpu_embedding(cfg, split=split)
        ids, off = to_dev(b)
        outs.append(emb.forward(ids, off, cfg.batch).cpu().numpy())
        if split:
            assert emb.n_packs > 4
    assert np.array_equal(outs[0], outs[1])


def test_packed_equals_unpacked_per_field():
    """Packed (one fused pass per dim-pack) == unpacked (one context per field: the per-field
    operator chain of PAPER.md Fig. packing a), bit-exact forward; updates agree."""
    cfg = dc.scaled(dc.wdl(), batch=40, rows_div=2000).replace(alpha=1.1)
    b, dy = make_batch(cfg, 0, 2), make_dy(cfg, 0, 2)
    emb = gpu_embedding(cfg)
    ids, off = to_dev(b)
    packed = emb.forward(ids, off, cfg.batch).cpu().numpy()
    emb.backward_update(torch.from_numpy(dy).cuda(), lr=0.05, step=1)
    B = cfg.batch
    import paper_2204_04903_b200 as pb
    for f in range(0, cfg.F, 37):
        t = int(cfg.field_to_table[f])
        e1 = pb.PackedEmbedding([0], cfg.table_rows[[t]], cfg.table_dim[[t]], max_batch=B, max_ids=B * 60,
                                table_salt=cfg.table_salt[[t]], pool=cfg.pool, id_mode=cfg.id_mode)
        w = table_values_np(cfg.seed, t, np.arange(cfg.table_rows[t]), int(cfg.table_dim[t]))
        e1.weights[0].copy_(torch.from_numpy(w))
        lo, hi = int(b.offsets[f * B]), int(b.offsets[(f + 1) * B])
        ids1 = torch.from_numpy(b.ids[lo:hi].copy()).cuda()
        off1 = torch.from_numpy((b.offsets[f * B:(f + 1) * B + 1] - lo).astype(np.int32)).cuda()
        o1 = e1.forward(ids1, off1, B).cpu().numpy()
        c, D = int(cfg.field_col[f]), int(cfg.table_dim[t])
        assert np.array_equal(o1, packed[:, c:c + D]), f"field {f}"
        # the packed update of this field's table equals the unpacked one when t has one field
        e1.backward_update(torch.from_numpy(np.ascontiguousarray(dy[:, c:c + D])).cuda(), lr=0.05, step=1)
        assert_close(e1.weights[0].cpu().numpy(), gpu_table_rows(emb, cfg, t), what=f"update field {f}")


def _long_cfg():
    return dc.toy(batch=1024).replace(table_rows=np.array([3, 5, 2, 7, 1, 4, 6, 3], np.int64),
                                      bags=[("uniform", 0, 8)] * 8)


def test_long_rows_chunked_path_dyadic():
    """Tiny tables make every row hot (> 256 occurrences): the chunked backward path.  Under
    dyadic dY every partial sum is exact, so the chunked order is bit-exact too (O19)."""
    run_step(_long_cfg(), steps=2, dyadic=True)


def test_long_rows_chunked_path_continuous():
    """Continuous dY on rows with ~1000 occurrences: the oracle (sequential) and the chunked
    GPU sum are both within gamma_n * sum|x| of the exact G (Higham, sequential summation
    bound, gamma_n = n u / (1 - n u), u = 2^-24), so they differ by at most 2 gamma_n sum|x|.
    Weights must still meet the north-star 1e-5/1e-6; the accumulator acc = 0.1 + G^2 is
    checked against the propagated bound 2|G| dG + dG^2."""
    cfg = _long_cfg()
    emb = gpu_embedding(cfg)
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    b, dy = make_batch(cfg, 0, 0), make_dy(cfg, 0, 0, dyadic=False)
    ids, off = to_dev(b)
    emb.forward(ids, off, cfg.batch)
    emb.backward_update(torch.from_numpy(dy).cuda(), lr=0.05, step=1)
    emb.check()
    ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)
    oabs = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, np.abs(dy))
    acc = [np.full_like(t, 0.1) for t in tabs]
    G = [oracle.table_grad(m, [ob], t) for t in range(cfg.T)]
    Gabs = [oracle.table_grad(m, [oabs], t)[0] for t in range(cfg.T)]
    oracle.backward_update(m, [ob], tabs, acc, lr=0.05)
    u = 2.0 ** -24
    for t in range(cfg.T):
        assert_close(gpu_table_rows(emb, cfg, t), tabs[t], what=f"weights t{t}")
        n = G[t][1][:, None].astype(np.float64)
        dG = 2 * (n * u / (1 - n * u)) * Gabs[t].astype(np.float64)
        bound = 2 * np.abs(G[t][0]) * dG + dG ** 2 + 4 * u * acc[t]
        got = gpu_table_rows(emb, cfg, t, "s1").astype(np.float64)
        assert (np.abs(got - acc[t]) <= bound + 1e-6).all(), f"state1 t{t}"
        # both sides accumulate in fp64 (reading O6): the north-star tolerance holds too
        assert_close(got, acc[t], what=f"state1 t{t}")


def test_empty_and_degenerate_batches():
    cfg = dc.toy()
    emb = gpu_embedding(cfg)
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    B = cfg.batch
    # every bag empty (N = 0)
    ids = torch.empty(0, dtype=torch.int64, device="cuda")
    off = torch.zeros(cfg.F * B + 1, dtype=torch.int32, device="cuda")
    out = emb.forward(ids, off, B)
    assert (out == 0).all()
    w0 = [w.clone() for w in emb.weights]
    emb.backward_update(torch.ones(B, cfg.out_width, device="cuda"), lr=0.1, step=1)
    emb.check()
    assert all(torch.equal(a, b) for a, b in zip(w0, emb.weights))
    # batch of 1 sample, one id in one field
    off1 = np.zeros(cfg.F + 1, np.int32)
    off1[3 + 1:] = 1
    ids1 = np.array([12345], np.int64)
    out = emb.forward(torch.from_numpy(ids1).cuda(), torch.from_numpy(off1).cuda(), 1).cpu().numpy()
    ref = oracle.forward(m, oracle.OracleBatch(1, ids1, off1), tabs, cfg.out_width)
    assert np.array_equal(out, ref)
    # batch 0
    emb.forward(ids, torch.zeros(1, dtype=torch.int32, device="cuda"), 0)
    emb.check()


def test_capacity_and_state_errors():
    import paper_2204_04903_b200 as pb

    cfg = dc.toy()
    emb = gpu_embedding(cfg, max_ids=100)
    b = make_batch(cfg, 0, 0)
    ids, off = to_dev(b)
    with pytest.raises(pb.PicassoError):
        emb.forward(ids, off, cfg.batch)  # more ids than max_ids
    with pytest.raises(pb.PicassoError):
        emb.backward_update(torch.zeros(cfg.batch, cfg.out_width, device="cuda"), lr=0.1, step=1)


def test_rows_mode_out_of_range_is_latched():
    import paper_2204_04903_b200 as pb

    cfg = dc.toy(id_mode=dc.IDS_ROWS)
    emb = gpu_embedding(cfg)
    b = make_batch(cfg, 0, 0)
    bad = b.ids.copy()
    bad[5] = cfg.table_rows[0] + 7
    ids = torch.from_numpy(bad).cuda()
    off = torch.from_numpy(b.offsets).cuda()
    emb.forward(ids, off, cfg.batch)
    with pytest.raises(pb.PicassoError):
        emb.check()


@pytest.mark.parametrize("kind", ["short", "long", "decreasing", "start"])
def test_bad_offsets_are_latched(kind):
    """offsets that are not a CSR over the ids (total != n_ids, a decreasing field boundary, a
    non-zero start) latch INVALID_ARG in k_field_prep, which then lays the step out on a
    substitute layout: no kernel reads or writes past its buffers (no illegal access, which would
    surface as PICASSO_ERR_CUDA), and the error belongs to that step only."""
    import paper_2204_04903_b200 as pb

    for cfg in (dc.scaled(dc.criteo(), batch=256, rows_div=20000), dc.toy(), dc.scaled(dc.wdl(), batch=16, rows_div=1000)):
        emb = gpu_embedding(cfg)
        b = make_batch(cfg, 0, 0)
        off = b.offsets.copy()
        if kind == "short":
            off[-1] -= 3
        elif kind == "long":
            off[-1] += 1000
        elif kind == "decreasing":
            off[cfg.batch] = off[2 * cfg.batch] + 5
        else:
            off[0] = 2
        ids = torch.from_numpy(b.ids).cuda()
        emb.forward(ids, torch.from_numpy(off).cuda(), cfg.batch)
        emb.backward_update(torch.ones(cfg.batch, cfg.out_width, device="cuda"), lr=0.1, step=1)
        with pytest.raises(pb.PicassoError) as ei:
            emb.check()
        assert ei.value.status == -1 and "CSR" in str(ei.value), str(ei.value)
        # a valid step afterwards runs clean and its forward is the oracle's on the current tables
        b2 = make_batch(cfg, 0, 1)
        i2, o2 = to_dev(b2)
        out = emb.forward(i2, o2, cfg.batch)
        emb.check()
        tabs = [gpu_table_rows(emb, cfg, t) for t in range(cfg.T)]
        ref = oracle.forward(oracle_model(cfg), oracle.OracleBatch(cfg.batch, b2.ids, b2.offsets), tabs, cfg.out_width)
        assert np.array_equal(out.cpu().numpy(), ref)


def test_host_side_argument_checks():
    import paper_2204_04903_b200 as pb

    cfg = dc.toy()
    emb = gpu_embedding(cfg)
    b = make_batch(cfg, 0, 0)
    ids, off = to_dev(b)
    with pytest.raises(pb.PicassoError, match="ids: dtype"):
        emb.forward(ids.to(torch.int32), off, cfg.batch)
    with pytest.raises(pb.PicassoError, match="offsets: .* elements"):
        emb.forward(ids, off[:-1], cfg.batch)
    with pytest.raises(pb.PicassoError, match="not contiguous"):
        emb.forward(torch.stack([ids, ids], 1)[:, 0], off, cfg.batch)
    with pytest.raises(pb.PicassoError, match="not a CUDA tensor"):
        emb.forward(ids.cpu(), off, cfg.batch)
    emb.forward(ids, off, cfg.batch)
    with pytest.raises(pb.PicassoError, match="grad_out: shape"):
        emb.backward_update(torch.zeros(cfg.batch, cfg.out_width + 4, device="cuda"), lr=0.1, step=1)


def test_deterministic_rerun():
    cfg = dc.scaled(dc.wdl(), batch=64, rows_div=5000).replace(alpha=1.3)
    res = []
    for _ in range(2):
        emb = gpu_embedding(cfg)
        b, dy = make_batch(cfg, 0, 0), make_dy(cfg, 0, 0, dyadic=False)
        ids, off = to_dev(b)
        out = emb.forward(ids, off, cfg.batch).clone()
        emb.backward_update(torch.from_numpy(dy).cuda(), lr=0.05, step=1)
        torch.cuda.synchronize()
        res.append((out.cpu().numpy(), [w.cpu().numpy() for w in emb.weights]))
    assert np.array_equal(res[0][0], res[1][0])
    assert all(np.array_equal(a, b) for a, b in zip(res[0][1], res[1][1]))


def test_criteo_small_shape():
    cfg = dc.scaled(dc.criteo(), batch=2048, rows_div=1000)
    run_step(cfg, steps=2, check_intermediates=True)


def test_profile_per_pack():
    """picasso_profile_read_packs: each pack's pool and backward carry their own event time, the
    per-pack pool times sum to no more than the pool phase (they partition it), and the read
    resets with picasso_profile_read."""
    import paper_2204_04903_b200 as pb

    cfg = dc.scaled(dc.wdl(), batch=64, rows_div=1000)
    emb = gpu_embedding(cfg)
    b = make_batch(cfg, 0, 1)
    ids, off = to_dev(b)
    dy = torch.from_numpy(make_dy(cfg, 0, 1)).cuda()
    pb.picasso_profile_enable(emb.ctx, 1)
    pb.picasso_profile_read(emb.ctx)
    emb.forward(ids, off, cfg.batch)
    emb.backward_update(dy, lr=0.05, step=1)
    torch.cuda.synchronize()
    pool, bwd = pb.picasso_profile_read_packs(emb.ctx, emb.n_packs)
    phase, calls = pb.picasso_profile_read(emb.ctx)
    pb.picasso_profile_enable(emb.ctx, 0)
    emb.check()
    assert emb.n_packs > 1 and calls == 1
    assert all(t > 0 for t in pool) and all(t > 0 for t in bwd), (pool, bwd)
    assert sum(pool) <= phase["pool"] * 1.05 + 1e-3, (pool, phase)
    pool2, _ = pb.picasso_profile_read_packs(emb.ctx, emb.n_packs)
    assert all(t == 0 for t in pool2)


def test_dy_staging_same_update(monkeypatch):
    """The backward of a multi-pack step reads dY regrouped pack by pack (k_dy_pack); reading it
    in place (PICASSO_DY_STAGE=0) gives bit-identical tables, and both match the oracle."""
    cfg = dc.scaled(dc.wdl(), batch=96, rows_div=1000)
    b, dy = make_batch(cfg, 0, 1), make_dy(cfg, 0, 1, dyadic=False)
    res = []
    for stage in ("1", "0"):
        monkeypatch.setenv("PICASSO_DY_STAGE", stage)
        emb = gpu_embedding(cfg)
        ids, off = to_dev(b)
        emb.forward(ids, off, cfg.batch)
        emb.backward_update(torch.from_numpy(dy).cuda(), lr=0.05, step=1)
        emb.check()
        res.append([torch.cat([w.flatten(), s.flatten()]).cpu() for w, s in zip(emb.weights, emb.state1)])
    assert all(torch.equal(x, y) for x, y in zip(res[0], res[1]))
    monkeypatch.setenv("PICASSO_DY_STAGE", "1")
    run_step(cfg, steps=2, dyadic=False, check_intermediates=False)
