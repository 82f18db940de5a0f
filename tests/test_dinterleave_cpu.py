"""D-Interleaving host logic (no GPU): Eq. 2 through the C ABI's
picasso_micro_batch_size, and the micro-batch slicing of a field-major CSR batch."""
import numpy as np
import pytest

import oracle
from datagen import configs as dc
from datagen import make_batch


@pytest.fixture(scope="module")
def pb():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2204_04903_b200 as pb

    return pb


def test_eq2_hand_examples(pb):
    # one op: 1000 B budget, 64 B / instance -> floor(15.6) = 15; batch 100 -> 7 micro-batches of 15
    assert pb.picasso_micro_batch_size([1000.0], [64.0], 100) == (15, 7)
    # min over ops: 4096/32 = 128, 1000/10 = 100 -> 100; batch 250 -> 3 micro-batches, ceil(250/3) = 84
    assert pb.picasso_micro_batch_size([4096.0, 1000.0], [32.0, 10.0], 250) == (84, 3)
    # bound above the batch: one micro-batch of the whole batch
    assert pb.picasso_micro_batch_size([1e12], [1.0], 16384) == (16384, 1)
    # an op with zero cost per instance never binds
    assert pb.picasso_micro_batch_size([5.0, 80.0], [0.0, 8.0], 30) == (10, 3)
    with pytest.raises(pb.PicassoError):  # not one instance fits
        pb.picasso_micro_batch_size([10.0], [64.0], 8)


def test_even_slices_and_slice_concat():
    from paper_2204_04903_b200.dinterleave import even_slices, slice_batch

    assert even_slices(10, 3) == [(0, 4), (4, 7), (7, 10)]
    cfg = dc.scaled(dc.wdl(), batch=37, rows_div=1000)
    b = make_batch(cfg, 0, 0)
    parts = [slice_batch(b.ids, b.offsets, cfg.F, cfg.batch, b0, b1) for b0, b1 in even_slices(cfg.batch, 4)]
    # slice-concat invariant: per field and sample, the bags are unchanged
    for f in range(cfg.F):
        bags = []
        for (b0, b1), (ids, off) in zip(even_slices(cfg.batch, 4), parts):
            n = b1 - b0
            for s in range(n):
                bags.append(ids[off[f * n + s]:off[f * n + s + 1]].tolist())
        ref = [b.ids[b.offsets[f * cfg.batch + s]:b.offsets[f * cfg.batch + s + 1]].tolist() for s in range(cfg.batch)]
        assert bags == ref
    assert sum(len(i) for i, _ in parts) == b.n_ids


def test_oracle_update_is_slice_invariant():
    """The oracle's whole-batch update equals the update over the micro-batches taken as one
    global batch (the backward sums over every occurrence whatever the batch split): the target
    the GPU's accumulated step is compared with."""
    from paper_2204_04903_b200.dinterleave import even_slices, slice_batch
    from datagen import make_dy, table_values_np

    cfg = dc.toy()
    b, dy = make_batch(cfg, 0, 0), make_dy(cfg, 0, 0)
    m = oracle.OracleModel(cfg.field_to_table, cfg.table_rows, cfg.table_dim, cfg.field_col, id_mode=cfg.id_mode,
                           pool=cfg.pool, table_salt=cfg.table_salt)
    tabs = [table_values_np(cfg.seed, t, np.arange(cfg.table_rows[t]), int(cfg.table_dim[t])) for t in range(cfg.T)]
    t1, t2 = [t.copy() for t in tabs], [t.copy() for t in tabs]
    a1, a2 = [np.full_like(t, 0.1) for t in tabs], [np.full_like(t, 0.1) for t in tabs]
    oracle.backward_update(m, [oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)], t1, a1, lr=0.05)
    mbs = []
    for b0, b1 in even_slices(cfg.batch, 3):
        ids, off = slice_batch(b.ids, b.offsets, cfg.F, cfg.batch, b0, b1)
        mbs.append(oracle.OracleBatch(b1 - b0, ids, off, np.ascontiguousarray(dy[b0:b1])))
    oracle.backward_update(m, mbs, t2, a2, lr=0.05)
    for x, y in zip(t1, t2):
        assert np.array_equal(x, y)  # dyadic dY: exact in any order
