"""GPU parity of the pipelined backward segment-sum (csrc/k_segsum_bulk.cu: equal-cost tiles,
LDGSTS ring, split-row fix-up) for every dimension it serves (64..512), against the oracle and
against the legacy register-staged path (PICASSO_SEGSUM=legacy).  Rows are made to span many
tiles (tiny tables, one 1-row table that takes every occurrence of its field), packs smaller
than the tile count, mean pooling, Adam, and continuous dY."""
import os

import numpy as np
import pytest
import torch

import oracle
from datagen import configs as dc
from datagen import make_batch, make_dy
from harness import assert_close, gpu_embedding, gpu_table_rows, oracle_model, oracle_tables, to_dev
from test_parity_gpu import run_step

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__

    __graft_entry__.build()


def _cfg(D, batch=2048, rows=(3, 50, 2, 700, 1, 4000, 6, 30000), bags=("uniform", 0, 8), **kw):
    F = len(rows)
    return dc.toy(batch=batch).replace(table_rows=np.array(rows, np.int64), table_dim=np.full(F, D, np.int32),
                                       field_to_table=np.arange(F, dtype=np.int32), bags=[bags] * F, **kw)


@pytest.mark.parametrize("D", [64, 128, 256, 384, 512])
def test_pipe_dims_long_rows_dyadic(D):
    """Rows with thousands of occurrences cut by many tile edges: bit-exact under dyadic dY."""
    run_step(_cfg(D), steps=2, dyadic=True, check_intermediates=False)


@pytest.mark.parametrize("D", [4, 8, 16, 32])
def test_narrow_dims_long_rows(D):
    """D <= 32 (k_segsum_flat + the chunked long-row path): dyadic bit-exact, then continuous
    dY with mean pooling."""
    run_step(_cfg(D), steps=2, dyadic=True, check_intermediates=False)
    run_step(_cfg(D, batch=512, pool=dc.POOL_MEAN), steps=1, dyadic=False, check_intermediates=False)


@pytest.mark.parametrize("D", [64, 128])
def test_pipe_continuous(D):
    run_step(_cfg(D), steps=2, dyadic=False, check_intermediates=False)


def test_pipe_mean_pool():
    run_step(_cfg(128, pool=dc.POOL_MEAN), steps=2, dyadic=False, check_intermediates=False)


def test_pipe_adam():
    run_step(_cfg(256), opt=oracle.OPT_ADAM, steps=3, dyadic=False, lr=0.01, check_intermediates=False)


def test_pipe_one_row_takes_a_whole_field():
    """A 1-row table under a one-hot field of 16K samples: one row spans every tile of the pack
    (the fix-up sums ~nt pieces)."""
    run_step(_cfg(128, batch=16384, rows=(1, 100000), bags=("fixed", 1)), steps=1, dyadic=True,
             check_intermediates=False)
    run_step(_cfg(128, batch=16384, rows=(1, 100000), bags=("fixed", 1)), steps=1, dyadic=False,
             check_intermediates=False)


@pytest.mark.parametrize("batch", [1, 3, 37])
def test_pipe_tiny_packs(batch):
    """Fewer (occurrence + row) units than tiles: tiles of one unit, empty tiles at the end."""
    run_step(_cfg(128, batch=batch, rows=(2, 5, 1000)), steps=2, dyadic=True, check_intermediates=False)


@pytest.mark.parametrize("dyadic", [True, False])
def test_pipe_equals_legacy(dyadic):
    """The pipelined and the legacy segment-sum give the same update (bit-exact under dyadic dY;
    within fp64-then-fp32 rounding otherwise)."""
    cfg = _cfg(128, batch=4096)
    res = []
    for mode in ("legacy", None):
        if mode:
            os.environ["PICASSO_SEGSUM"] = mode
        try:
            emb = gpu_embedding(cfg)
        finally:
            os.environ.pop("PICASSO_SEGSUM", None)
        for step in (1, 2):
            b, dy = make_batch(cfg, 0, step), make_dy(cfg, 0, step, dyadic=dyadic)
            ids, off = to_dev(b)
            emb.forward(ids, off, cfg.batch)
            emb.backward_update(torch.from_numpy(dy).cuda(), lr=0.05, step=step)
        emb.check()
        res.append([gpu_table_rows(emb, cfg, t) for t in range(cfg.T)])
    for t in range(cfg.T):
        if dyadic:
            assert np.array_equal(res[0][t], res[1][t]), f"table {t}"
        else:
            assert_close(res[1][t], res[0][t], what=f"table {t}")


# ---- pipelined pool (csrc/k_pool_pipe.cu) -------------------------------------------------------
def _fwd(cfg, env=None, step=1):
    if env:
        os.environ.update(env)
    try:
        emb = gpu_embedding(cfg)
    finally:
        for k in env or {}:
            os.environ.pop(k, None)
    b = make_batch(cfg, 0, step)
    ids, off = to_dev(b)
    return emb.forward(ids, off, cfg.batch).cpu().numpy(), b


@pytest.mark.parametrize("name", ["wdl", "criteo", "mixed"])
def test_pool_pipe_equals_legacy_and_oracle(name):
    """Pipelined pool == legacy pool == oracle, bit-exact (sequential fp32 per segment)."""
    if name == "wdl":
        cfg = dc.scaled(dc.wdl(), batch=96, rows_div=1000)
    elif name == "criteo":
        cfg = dc.scaled(dc.criteo(), batch=512, rows_div=100)
    else:  # D = 64 / 128 / 256 packs, one field of all-empty bags, bags 0..50 elsewhere
        cfg = dc.toy(batch=300).replace(
            table_rows=np.array([50, 7, 900, 3, 20], np.int64), table_dim=np.array([64, 128, 256, 128, 64], np.int32),
            field_to_table=np.arange(5, dtype=np.int32),
            bags=[("uniform", 0, 50), ("fixed", 0), ("uniform", 1, 3), ("fixed", 1), ("uniform", 0, 2)])
    got, b = _fwd(cfg)
    leg, _ = _fwd(cfg, {"PICASSO_POOL": "legacy"})
    assert np.array_equal(got, leg)
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, None)
    assert np.array_equal(got, oracle.forward(m, ob, tabs, cfg.out_width))


def test_pool_pipe_mean_and_all_empty_pack():
    cfg = dc.toy(batch=200, pool=dc.POOL_MEAN).replace(
        table_rows=np.array([10, 10, 500], np.int64), table_dim=np.array([128, 256, 128], np.int32),
        field_to_table=np.arange(3, dtype=np.int32), bags=[("uniform", 0, 9), ("fixed", 0), ("uniform", 0, 1)])
    got, b = _fwd(cfg)
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, None)
    assert np.array_equal(got, oracle.forward(m, ob, tabs, cfg.out_width))


# ---- alternative paths behind environment switches (read when the context is created) ---------
_H = {"PICASSO_INDEX": "hash"}  # the hash-table index path's own switches


@pytest.mark.parametrize("env", [{"PICASSO_EARLY_POOL": "0", **_H}, {"PICASSO_BWD": "split"}, {"PICASSO_POOL": "flat"},
                                 {"PICASSO_OVERLAP": "0", **_H}, {"PICASSO_OVERLAP": "1", **_H},
                                 {"PICASSO_SEGSUM_CFG": "12x4"}, {"PICASSO_DEDUP_REGIONS": "1", **_H},
                                 {"PICASSO_SEGSUM_SMALL": "legacy"}, _H, {"PICASSO_SORT_OVERLAP": "0"},
                                 {"PICASSO_SORT_RESERVE": "100"}, {"PICASSO_BWD": "split", **_H},
                                 {"PICASSO_SORT": "3", **_H}, {"PICASSO_SORT": "2", **_H}])
def test_alternative_paths_match_oracle(env, monkeypatch):
    """Every switchable variant computes the same step: forward bit-exact, update within the
    north-star tolerance of the oracle (bit-exact under dyadic dY)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    run_step(_cfg(128, batch=1024), steps=2, dyadic=True, check_intermediates=False)
    run_step(_cfg(64, batch=512, pool=dc.POOL_MEAN), steps=1, dyadic=False, check_intermediates=False)
    run_step(_cfg(16, batch=1024), steps=2, dyadic=True, check_intermediates=False)
