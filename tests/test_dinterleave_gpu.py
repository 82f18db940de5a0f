"""D-Interleaving on the GPU: a step's batch sliced into micro-batches,
each forwarded and accumulated through the C ABI, one update at the end — against the oracle's
whole-batch step.  Forward: every micro-batch's rows equal the whole batch's (bit-exact, the
slice-concat invariant); update: bit-exact under dyadic dY, 1e-5 / 1e-6 otherwise."""
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


def run_micro(cfg, n_micro, steps=2, opt=0, dyadic=True, lr=0.05, max_step_unique=None):
    from paper_2204_04903_b200.dinterleave import even_slices, slice_batch

    sl = even_slices(cfg.batch, n_micro)
    mbmax = max(b1 - b0 for b0, b1 in sl)
    msu = max_step_unique or cfg.batch * cfg.F * 60
    emb = gpu_embedding(cfg, max_batch=mbmax, max_ids=mbmax * cfg.F * 60, opt=opt, max_step_unique=msu)
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    if opt == 0:
        s1, s2 = [np.full_like(t, 0.1) for t in tabs], None
    else:
        s1, s2 = [np.zeros_like(t) for t in tabs], [np.zeros_like(t) for t in tabs]
    for step in range(1, steps + 1):
        b, dy = make_batch(cfg, 0, step), make_dy(cfg, 0, step, dyadic=dyadic)
        ob = oracle.OracleBatch(cfg.batch, b.ids, b.offsets, dy)
        ref = oracle.forward(m, ob, tabs, cfg.out_width)
        emb.dinterleave_begin()
        for b0, b1 in sl:
            ids, off = slice_batch(b.ids, b.offsets, cfg.F, cfg.batch, b0, b1)
            # offsets stay alive until the backward: the mean combiner's bag lengths are read there
            ids_d, off_d = torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda()
            out = emb.forward(ids_d, off_d, b1 - b0)
            if dyadic and opt == 0 or step == 1:
                assert np.array_equal(out.cpu().numpy(), ref[b0:b1]), f"forward micro-batch [{b0},{b1}) step {step}"
            else:
                assert_close(out.cpu().numpy(), ref[b0:b1], what=f"forward [{b0},{b1})")
            emb.backward_accumulate(torch.from_numpy(np.ascontiguousarray(dy[b0:b1])).cuda())
        with pytest.raises(Exception):  # the plain backward is refused inside a D-Interleaving step
            emb.backward_update(torch.zeros(1, cfg.out_width, device="cuda"), lr=lr, step=step)
        emb.dinterleave_apply(lr=lr, step=step)
        emb.check()
        oracle.backward_update(m, [ob], tabs, s1, s2, kind=opt, lr=lr, step=step)
        for t in range(cfg.T):
            gw = gpu_table_rows(emb, cfg, t)
            if dyadic and opt == 0:
                assert np.array_equal(gw, tabs[t]), f"table {t} step {step} (dyadic: bit-exact)"
                assert np.array_equal(gpu_table_rows(emb, cfg, t, "s1"), s1[t])
            assert_close(gw, tabs[t], what=f"weights t{t} step {step}")
            assert_close(gpu_table_rows(emb, cfg, t, "s1"), s1[t], what=f"state1 t{t}")
            if s2:
                assert_close(gpu_table_rows(emb, cfg, t, "s2"), s2[t], what=f"state2 t{t}")
    return emb


@pytest.mark.parametrize("n_micro", [1, 3, 4])
def test_toy_micro_batches(n_micro):
    run_micro(dc.toy(), n_micro)


def test_multipack_uneven_micro_batches():
    run_micro(dc.scaled(dc.wdl(), batch=45, rows_div=1000), 4)  # 12/11/11/11 samples, 4 packs


def test_hot_rows_long_path():
    """Rows with > 256 occurrences in a micro-batch (chunked segment-sum) accumulated across 3."""
    cfg = dc.toy(batch=2048).replace(table_rows=np.array([3, 5, 2, 7, 1, 4, 6, 3], np.int64),
                                     bags=[("uniform", 0, 8)] * 8)
    run_micro(cfg, 3)


def test_criteo_pipe_kernels_continuous():
    run_micro(dc.scaled(dc.criteo(), batch=1024, rows_div=2000), 3, dyadic=False)


def test_adam_mean():
    run_micro(dc.toy(pool=dc.POOL_MEAN), 3, opt=1, dyadic=False, lr=0.01)


def test_accumulator_overflow_is_latched():
    import paper_2204_04903_b200 as pb

    cfg = dc.toy()
    with pytest.raises(pb.PicassoError):
        run_micro(cfg, 2, steps=1, max_step_unique=64)
