"""GPU parity of the two index paths of a world == 1 step: the sort-based index (csrc/k_sortidx.cu,
the default, which every other world == 1 parity test exercises) and the hash-table index
(csrc/k_index.cu + the uid transpose; PICASSO_INDEX=hash, also what the row-sharded steps use).
The parity cases are re-run here on the hash path; multi-chunk batches compare both paths
element by element and against the oracle; key widths of one to three LSD passes; one context
switching between the two."""
import numpy as np
import pytest
import torch

import oracle
from datagen import configs as dc
from datagen import make_batch, make_dy
from harness import gpu_embedding, gpu_table_rows, oracle_model, oracle_tables, to_dev

# the parity cases, collected again in this module (under the hash switch below)
from test_parity_gpu import (run_step, test_bad_offsets_are_latched, test_criteo_small_shape,  # noqa: F401
                             test_deterministic_rerun, test_empty_and_degenerate_batches,
                             test_long_rows_chunked_path_continuous, test_long_rows_chunked_path_dyadic,
                             test_multipack_wdl_small, test_o2_golden_through_abi, test_packed_equals_unpacked_per_field,
                             test_toy_adam_lazy, test_toy_continuous_dy, test_toy_pool_modes_three_steps,
                             test_toy_sum_adagrad_bit_exact)
from test_segsum_pipe_gpu import (test_pipe_adam, test_pipe_dims_long_rows_dyadic,  # noqa: F401
                                  test_pipe_one_row_takes_a_whole_field, test_pipe_tiny_packs)
from test_dinterleave_gpu import test_adam_mean, test_multipack_uneven_micro_batches  # noqa: F401
from test_odd_dims_gpu import test_odd_dims_parity  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__

    __graft_entry__.build()


@pytest.fixture(autouse=True)
def _hash_index(monkeypatch):
    monkeypatch.setenv("PICASSO_INDEX", "hash")


def _step(cfg, b, dy, lr=0.05):
    emb = gpu_embedding(cfg)
    ids, off = to_dev(b)
    out = emb.forward(ids, off, cfg.batch).cpu().numpy()
    uniq = [emb.unique(p).cpu().numpy() for p in range(emb.n_packs)]
    inv = [emb.inverse(p).cpu().numpy() for p in range(emb.n_packs)]
    emb.backward_update(torch.from_numpy(dy).cuda(), lr=lr, step=1)
    emb.check()
    return emb, out, uniq, inv


@pytest.mark.parametrize("name", ["criteo", "wdl"])
def test_sort_equals_hash_and_oracle_multi_chunk(name, monkeypatch):
    """Batches of ~1 M IDs: every CTA of the sort walks several tiles (chunk > 2048), keys of 23
    (criteo) / 27 (wdl, 4 packs) bits take three / four LSD passes.  Sort vs hash: forward, Unique,
    inverse, updated tables identical; both against the oracle (unique / inverse / forward)."""
    if name == "criteo":
        cfg = dc.scaled(dc.criteo(), batch=40960, rows_div=8)
    else:
        cfg = dc.scaled(dc.wdl(), batch=200, rows_div=4)
    b, dy = make_batch(cfg, 0, 3), make_dy(cfg, 0, 3)
    assert b.n_ids > 3 * 148 * 2048, b.n_ids  # more than one tile per CTA
    res = {}
    for mode in ("hash", "sort"):
        monkeypatch.setenv("PICASSO_INDEX", mode)
        res[mode] = _step(cfg, b, dy)
    (e_h, o_h, u_h, i_h), (e_s, o_s, u_s, i_s) = res["hash"], res["sort"]
    assert e_s.n_packs == e_h.n_packs
    assert np.array_equal(o_h, o_s)
    m = oracle_model(cfg)
    ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)
    for p in range(e_s.n_packs):
        keys = oracle.pack_key_stream(m, e_s.plan["field_to_pack"], e_s.plan["table_base"], ob, p)
        u_ref, inv_ref = oracle.unique(keys)
        assert np.array_equal(u_s[p], u_ref), f"unique pack {p}"
        assert np.array_equal(i_s[p], inv_ref), f"inverse pack {p}"
        assert np.array_equal(u_h[p], u_ref) and np.array_equal(i_h[p], inv_ref)
    for p in range(e_s.n_packs):
        assert torch.equal(e_h.weights[p], e_s.weights[p]), f"weights pack {p} (dyadic dY: both exact)"
        assert torch.equal(e_h.state1[p], e_s.state1[p]), f"state pack {p}"
    if name == "criteo":  # forward against the oracle at this size too
        tabs = oracle_tables(cfg)
        assert np.array_equal(o_s, oracle.forward(m, ob, tabs, cfg.out_width))


def test_sort_passes_one_two_three(monkeypatch):
    """Key widths of 5, 13 and 20 bits: one, two and three LSD passes of <= 8 bits; all bit-exact
    against the oracle over three steps."""
    monkeypatch.setenv("PICASSO_INDEX", "sort")
    for rows in (np.array([3, 5, 2, 7, 1, 4, 6, 3], np.int64), np.full(8, 1000, np.int64),
                 np.full(8, 120000, np.int64)):
        cfg = dc.toy(batch=512).replace(table_rows=rows, bags=[("uniform", 0, 6)] * 8)
        run_step(cfg, steps=3)


def test_sort_step_then_hash_step_same_ctx(monkeypatch):
    """One context alternating sort-indexed (large) and hash-indexed (small) steps: the backward
    follows each forward's row numbering (run order after a sorted forward, uid order after a
    hashed one)."""
    cfg = dc.scaled(dc.wdl(), batch=48, rows_div=1000)
    n_half = make_batch(cfg, 0, 2, batch=cfg.batch // 2).n_ids
    assert n_half < min(make_batch(cfg, 0, s).n_ids for s in (1, 3))
    monkeypatch.setenv("PICASSO_INDEX", "auto")
    monkeypatch.setenv("PICASSO_SORT_MIN_IDS", str(n_half + 1))
    emb = gpu_embedding(cfg)
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    s1 = [np.full_like(t, 0.1) for t in tabs]
    for step, bsz in ((1, cfg.batch), (2, cfg.batch // 2), (3, cfg.batch)):
        b = make_batch(cfg, 0, step, batch=bsz)
        dy = make_dy(cfg, 0, step, batch=bsz)
        ids, off = to_dev(b)
        out = emb.forward(ids, off, bsz).cpu().numpy()
        ob = oracle.OracleBatch(bsz, b.ids, b.offsets, dy)
        assert np.array_equal(out, oracle.forward(m, ob, tabs, cfg.out_width))
        emb.backward_update(torch.from_numpy(dy).cuda(), lr=0.05, step=step)
        emb.check()
        oracle.backward_update(m, [ob], tabs, s1, None, kind=oracle.OPT_ADAGRAD, lr=0.05, step=step)
        for t in range(0, cfg.T, 7):
            assert np.array_equal(gpu_table_rows(emb, cfg, t), tabs[t]), f"step {step} table {t}"


@pytest.mark.parametrize("mode", ["sort", "hash"])
@pytest.mark.parametrize("seed", range(8))
def test_sort_index_random_shapes(seed, mode, monkeypatch):
    """Random small layouts (1-12 fields sharing 1-6 tables, dims 4-64, 1-5000 rows, batch 1-300,
    bags of 0-6 IDs, some fields always empty): both index paths bit-exact against the oracle
    (forward, Unique / inverse, dyadic updates), two steps each."""
    monkeypatch.setenv("PICASSO_INDEX", mode)
    rng = np.random.default_rng(1000 + seed)
    T = int(rng.integers(1, 7))
    F = int(rng.integers(1, 13))
    dims = rng.choice([4, 8, 16, 32, 64], size=T).astype(np.int32)
    rows = rng.integers(1, 5001, size=T).astype(np.int64)
    f2t = rng.integers(0, T, size=F).astype(np.int32)
    bags = [("uniform", 0, int(rng.integers(0, 7))) for _ in range(F)]
    cfg = dc.toy(batch=int(rng.integers(1, 301))).replace(
        field_to_table=f2t, table_rows=rows, table_dim=dims, bags=bags, alpha=float(rng.uniform(0.6, 1.4)))
    run_step(cfg, steps=2)
