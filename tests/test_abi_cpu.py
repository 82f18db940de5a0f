"""Host-side checks of the C-ABI library (-m "not gpu"): it loads, exports every symbol
include/picasso.h declares, and its host-only entry points (the Eq. 1 planner, context
creation, workspace sizing, argument validation) behave.  No kernel is launched."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from datagen import configs as dc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pb():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2204_04903_b200 as pb

    return pb


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "picasso.h")).read()
    return sorted(set(re.findall(r"picasso_status\s+(picasso_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(pb):
    L = ctypes.CDLL(pb.lib_path)
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(pb.abi.EXPORTS) == syms


@pytest.mark.parametrize("name", ["toy", "criteo", "wdl", "industrial"])
@pytest.mark.parametrize("split", [False, True])
def test_pack_plan_matches_oracle_bit_exact(pb, name, split):
    cfg = dc.get_config(name)
    rng = np.random.default_rng(len(name))
    for wc in (None, rng.integers(0, 10**6, cfg.T).astype(np.uint64)):
        a = pb.picasso_pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim, wc, split)
        b = oracle.pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim, wc, split)
        for k in ("field_to_pack", "table_to_pack", "table_base", "pack_dim", "pack_rows", "n_packs"):
            assert np.array_equal(a[k], b[k]), k


def test_pack_plan_paper_four_shards(pb):
    dims = np.array([8] * 8 + [32] * 8)
    a = pb.picasso_pack_plan(np.arange(16), np.full(16, 10), dims, None, True)
    assert (a["pack_dim"] == 32).sum() == 4 and (a["pack_dim"] == 8).sum() == 1


def test_pack_plan_rejects_bad_args(pb):
    with pytest.raises(pb.PicassoError):
        pb.picasso_pack_plan([0, 5], [10, 10], [8, 8])
    with pytest.raises(pb.PicassoError):
        pb.picasso_pack_plan([0], [0], [8])


def test_ctx_create_and_workspace(pb):
    cfg = dc.criteo()
    p = pb.picasso_pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim)
    ctx = pb.picasso_ctx_create(p, cfg.field_to_table, cfg.table_rows, cfg.table_dim, cfg.table_salt,
                                cfg.field_col, cfg.out_width, 0, 1, cfg.batch, cfg.batch * cfg.F)
    try:
        ws = pb.picasso_workspace_size(ctx)
        # index scratch (~100 B / id) + the split backward's G buffer (4 * maxD B / id)
        assert 16 * cfg.batch * cfg.F < ws < (200 + 4 * 128) * cfg.batch * cfg.F
        assert pb.picasso_pack_local_rows(ctx, 0) == int(cfg.table_rows.sum())
        with pytest.raises(pb.PicassoError):
            pb.picasso_pack_local_rows(ctx, 1)
    finally:
        pb.picasso_ctx_destroy(ctx)


def test_ctx_create_validation(pb):
    cfg = dc.toy()
    p = pb.picasso_pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim)
    bad_col = cfg.field_col.copy()
    bad_col[1] += 2  # not a multiple of 4
    with pytest.raises(pb.PicassoError):
        pb.picasso_ctx_create(p, cfg.field_to_table, cfg.table_rows, cfg.table_dim, None, bad_col,
                              cfg.out_width, 0, 1, 16, 100)
    with pytest.raises(pb.PicassoError):  # dim 12 unsupported (not a power of two)
        q = pb.picasso_pack_plan([0], [10], [12])
        pb.picasso_ctx_create(q, [0], [10], [12], None, [0], 12, 0, 1, 16, 100)
    with pytest.raises(pb.PicassoError):
        pb.picasso_ctx_create(p, cfg.field_to_table, cfg.table_rows, cfg.table_dim, None, cfg.field_col,
                              cfg.out_width, 0, 1, 0, 100)


def test_kinterleave_plan_matches_oracle(pb):
    """picasso_pack_plan_kinterleave (host C++ of the product) == the oracle's plan, bit-exact,
    on the golden example and on random industrial-shaped configurations."""
    import json

    import numpy as np

    import oracle
    from datagen import configs as dc

    g = json.load(open(os.path.join(ROOT, "tests", "golden", "worked_examples.json")))["kinterleave_plan"]
    assert pb.picasso_interleave_capacity(g["rbound"], g["rparam"]) == g["capacity"]
    cases = [(g["field_to_table"], g["table_rows"], g["table_dim"], g["capacity"], g["excluded"], None)]
    cfg = dc.scaled(dc.industrial(), batch=8, rows_div=10**4)
    rng = np.random.default_rng(11)
    for _ in range(6):
        cnt = rng.integers(1, 5000, cfg.T).astype(np.uint64)
        ex = (rng.random(cfg.T) < 0.15).astype(np.uint8)
        cap = float(rng.uniform(0.02, 0.6) * (cfg.table_dim * cnt).sum())
        cases.append((cfg.field_to_table, cfg.table_rows, cfg.table_dim, cap, ex, cnt))
    for f2t, rows, dims, cap, ex, cnt in cases:
        a = pb.picasso_pack_plan_kinterleave(f2t, rows, dims, cap, ex, cnt)
        b = oracle.kinterleave_plan(f2t, rows, dims, cap, ex, cnt)
        for k in ("table_to_pack", "table_base", "pack_dim", "pack_rows", "pack_group", "field_to_pack"):
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
        assert a["n_groups"] == b["n_groups"] and a["n_packs"] == b["n_packs"]
