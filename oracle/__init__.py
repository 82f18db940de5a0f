"""CPU oracle for the PICASSO packed sparse-embedding hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_2204_04903_b200`` never imports it and shares no code with it.

This module is argument marshalling (numpy <-> C) around ``picasso_oracle.cpp``; every
line of arithmetic lives in that file, each function citing the PAPER.md passage it
follows.  Parity status per function is listed in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "picasso_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

IDS_ROWS, IDS_HASH = 0, 1
POOL_SUM, POOL_MEAN = 0, 1
OPT_ADAGRAD, OPT_ADAM = 0, 1


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")


def build(force: bool = False, openmp: bool = False) -> str:
    """Compile the oracle with g++ (-O2, no FMA contraction, no fast-math).  openmp=True builds
    the same source with -fopenmp (liboracle_omp.so): the loops bench.py's all-cores CPU
    baseline times are split over threads with every per-row / per-segment sum in the same
    sequential order, so its results are bitwise those of the plain build (pinned in
    tests/test_oracle_pins.py).  Tests use the plain build."""
    lib_path = _LIB_OMP if openmp else _LIB
    if force or not os.path.exists(lib_path) or os.path.getmtime(lib_path) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-Wall", *(["-fopenmp"] if openmp else []), "-o", lib_path + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(lib_path + ".tmp", lib_path)
    return lib_path


_use_openmp = False


def use_openmp(on: bool = True):
    """Route the wrappers below to the -fopenmp build (bench.py's all-cores baseline) or back."""
    global _use_openmp
    _use_openmp = bool(on)


def set_threads(n: int) -> int:
    """Threads of the OpenMP build's loops (torchrun sets OMP_NUM_THREADS=1 for its workers); returns
    the count the build will use.  The plain build: always 1."""
    L = lib()
    L.oracle_set_threads(int(n))
    return int(L.oracle_get_threads())


class Model(C.Structure):
    _fields_ = [("n_fields", C.c_int32), ("n_tables", C.c_int32),
                ("field_to_table", C.c_void_p), ("table_rows", C.c_void_p),
                ("table_dim", C.c_void_p), ("table_salt", C.c_void_p),
                ("id_mode", C.c_int32), ("pool", C.c_int32), ("field_col", C.c_void_p)]


class Batch(C.Structure):
    _fields_ = [("batch", C.c_int32), ("ids", C.c_void_p), ("offsets", C.c_void_p),
                ("dy", C.c_void_p), ("dy_stride", C.c_int64)]


class Opt(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lr", C.c_float), ("eps", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float)]


_libs = {}


def lib():
    if _use_openmp not in _libs:
        _libs[_use_openmp] = L = C.CDLL(build(openmp=_use_openmp))
        L.oracle_set_threads.argtypes = [C.c_int32]
        L.oracle_get_threads.restype = C.c_int32
        L.oracle_mix64.restype = C.c_uint64
        L.oracle_mix64.argtypes = [C.c_uint64]
        L.oracle_row_of.restype = C.c_int32
        L.oracle_row_of.argtypes = [C.c_int32, C.c_int64, C.c_uint64, C.c_int64, C.POINTER(C.c_int64)]
        L.oracle_calc_vparam.restype = C.c_double
        L.oracle_calc_vparam.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_double]
        L.oracle_pack_plan.restype = C.c_int32
        L.oracle_pack_plan.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]
        L.oracle_forward.restype = C.c_int32
        L.oracle_forward.argtypes = [C.POINTER(Model), C.POINTER(Batch), C.c_void_p, C.c_void_p, C.c_int64]
        L.oracle_segment_rows.restype = C.c_int64
        L.oracle_segment_rows.argtypes = [C.POINTER(Model), C.POINTER(Batch), C.c_int64, C.c_void_p,
                                          C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.oracle_forward_sampled.restype = C.c_int32
        L.oracle_forward_sampled.argtypes = [C.POINTER(Model), C.POINTER(Batch), C.c_int64, C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                             C.c_void_p, C.c_void_p]
        L.oracle_pack_key_stream.restype = C.c_int64
        L.oracle_pack_key_stream.argtypes = [C.POINTER(Model), C.c_void_p, C.c_void_p, C.POINTER(Batch),
                                             C.c_int32, C.c_int64, C.c_void_p]
        L.oracle_unique.restype = C.c_int64
        L.oracle_unique.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_partition.restype = C.c_int32
        L.oracle_partition.argtypes = [C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_backward_update.restype = C.c_int32
        L.oracle_backward_update.argtypes = [C.POINTER(Model), C.c_int32, C.POINTER(Batch), C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.POINTER(Opt), C.c_int64]
        L.oracle_table_grad.restype = C.c_int32
        L.oracle_table_grad.argtypes = [C.POINTER(Model), C.c_int32, C.POINTER(Batch), C.c_int32,
                                        C.c_void_p, C.c_void_p]
        L.oracle_row_grads.restype = C.c_int32
        L.oracle_row_grads.argtypes = [C.POINTER(Model), C.c_int32, C.POINTER(Batch), C.c_int64,
                                       C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.oracle_apply_update.restype = C.c_int32
        L.oracle_apply_update.argtypes = [C.POINTER(Opt), C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_hot_select.restype = C.c_int64
        L.oracle_hot_select.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_uint64, C.c_void_p]
        L.oracle_interleave_capacity.restype = C.c_double
        L.oracle_interleave_capacity.argtypes = [C.c_int32, C.c_void_p, C.c_void_p]
        L.oracle_kinterleave_plan.restype = C.c_int32
        L.oracle_kinterleave_plan.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]
        L.oracle_fcounter_add.restype = C.c_int32
        L.oracle_fcounter_add.argtypes = [C.c_int64, C.c_void_p, C.c_void_p]
    return _libs[_use_openmp]


def _p(a):
    return None if a is None else a.ctypes.data


def _arr(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class _Check(RuntimeError):
    pass


def _ok(st):
    if st != 0:
        raise _Check(f"oracle returned status {st}")


# ---------------------------------------------------------------------------------------
def mix64(x: int) -> int:
    return int(lib().oracle_mix64(C.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def row_of(mode: int, raw: int, salt: int, V: int) -> int:
    r = C.c_int64()
    _ok(lib().oracle_row_of(mode, raw, salt & 0xFFFFFFFFFFFFFFFF, V, C.byref(r)))
    return r.value


def calc_vparam(dims, id_freq_sums, N) -> float:
    d = _arr(dims, np.int32)
    f = _arr(id_freq_sums, np.float64)
    return float(lib().oracle_calc_vparam(len(d), _p(d), _p(f), float(N)))


def pack_plan(field_to_table, table_rows, table_dim, warmup_count=None, split=False):
    f2t = _arr(field_to_table, np.int32)
    rows = _arr(table_rows, np.int64)
    dims = _arr(table_dim, np.int32)
    wc = None if warmup_count is None else _arr(warmup_count, np.uint64)
    F, T = len(f2t), len(rows)
    f2p = np.zeros(F, np.int32)
    t2p = np.zeros(T, np.int32)
    tb = np.zeros(T, np.int64)
    pd = np.zeros(T, np.int32)
    pr = np.zeros(T, np.int64)
    n = C.c_int32()
    _ok(lib().oracle_pack_plan(F, _p(f2t), T, _p(rows), _p(dims), _p(wc), int(bool(split)),
                               _p(f2p), _p(t2p), _p(tb), _p(pd), _p(pr), C.byref(n)))
    P = n.value
    return dict(field_to_pack=f2p, table_to_pack=t2p, table_base=tb, pack_dim=pd[:P].copy(),
                pack_rows=pr[:P].copy(), n_packs=P)


class OracleModel:
    """Keeps the numpy arrays alive behind the C struct."""

    def __init__(self, field_to_table, table_rows, table_dim, field_col, id_mode=IDS_HASH,
                 pool=POOL_SUM, table_salt=None):
        self.f2t = _arr(field_to_table, np.int32)
        self.rows = _arr(table_rows, np.int64)
        self.dims = _arr(table_dim, np.int32)
        self.col = _arr(field_col, np.int64)
        self.salt = _arr(table_salt if table_salt is not None else np.zeros(len(self.rows)), np.uint64)
        self.id_mode, self.pool = int(id_mode), int(pool)
        self.s = Model(len(self.f2t), len(self.rows), _p(self.f2t), _p(self.rows), _p(self.dims),
                       _p(self.salt), self.id_mode, self.pool, _p(self.col))

    @property
    def F(self):
        return len(self.f2t)


class OracleBatch:
    def __init__(self, B, ids, offsets, dy=None):
        self.ids = _arr(ids, np.int64)
        self.offsets = _arr(offsets, np.int32)
        self.dy = None if dy is None else _arr(dy, np.float32)
        stride = 0 if self.dy is None else self.dy.shape[1]
        self.s = Batch(int(B), _p(self.ids), _p(self.offsets), _p(self.dy), stride)


def _ptr_array(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data if a is not None else None for a in arrs])


def forward(model: OracleModel, batch: OracleBatch, tables, out_width):
    tabs = [_arr(t, np.float32) for t in tables]
    out = np.zeros((batch.s.batch, out_width), np.float32)
    _ok(lib().oracle_forward(C.byref(model.s), C.byref(batch.s), _ptr_array(tabs), _p(out), out_width))
    return out


def segment_rows(model, batch, q_field, q_sample):
    qf, qs = _arr(q_field, np.int32), _arr(q_sample, np.int32)
    n = lib().oracle_segment_rows(C.byref(model.s), C.byref(batch.s), len(qf), _p(qf), _p(qs), 0, None, None)
    if n < 0:
        _ok(n)
    t = np.zeros(n, np.int32)
    r = np.zeros(n, np.int64)
    lib().oracle_segment_rows(C.byref(model.s), C.byref(batch.s), len(qf), _p(qf), _p(qs), n, _p(t), _p(r))
    return t, r


def forward_sampled(model, batch, r_table, r_row, r_val, q_field, q_sample):
    rt, rr = _arr(r_table, np.int32), _arr(r_row, np.int64)
    rv = _arr(r_val, np.float32)
    ld = rv.shape[1]
    qf, qs = _arr(q_field, np.int32), _arr(q_sample, np.int32)
    out = np.zeros((len(qf), ld), np.float32)
    _ok(lib().oracle_forward_sampled(C.byref(model.s), C.byref(batch.s), len(rt), _p(rt), _p(rr), _p(rv),
                                     ld, len(qf), _p(qf), _p(qs), _p(out)))
    return out


def pack_key_stream(model, field_to_pack, table_base, batch, pack):
    f2p, tb = _arr(field_to_pack, np.int32), _arr(table_base, np.int64)
    n = lib().oracle_pack_key_stream(C.byref(model.s), _p(f2p), _p(tb), C.byref(batch.s), pack, 0, None)
    if n < 0:
        _ok(n)
    keys = np.zeros(n, np.int64)
    lib().oracle_pack_key_stream(C.byref(model.s), _p(f2p), _p(tb), C.byref(batch.s), pack, n, _p(keys))
    return keys


def unique(keys):
    k = _arr(keys, np.int64)
    u = np.zeros(len(k), np.int64)
    inv = np.zeros(len(k), np.int32)
    U = lib().oracle_unique(len(k), _p(k), _p(u), _p(inv))
    return u[:U].copy(), inv


def partition(uniq, W):
    u = _arr(uniq, np.int64)
    keys = np.zeros(len(u), np.int64)
    lrow = np.zeros(len(u), np.int64)
    counts = np.zeros(W, np.int64)
    _ok(lib().oracle_partition(len(u), _p(u), W, _p(keys), _p(lrow), _p(counts)))
    return keys, lrow, counts


def _opt(kind, lr, eps=None, beta1=0.9, beta2=0.999):
    if eps is None:
        eps = 1e-10 if kind == OPT_ADAGRAD else 1e-8
    return Opt(kind, lr, eps, beta1, beta2)


def backward_update(model, batches, tables, state1, state2=None, kind=OPT_ADAGRAD, lr=0.01, step=1,
                    eps=None, beta1=0.9, beta2=0.999):
    """In-place update of the float32 numpy arrays tables/state1/state2 (lists per table)."""
    arr = (Batch * len(batches))(*[b.s for b in batches])
    o = _opt(kind, lr, eps, beta1, beta2)
    for a in list(tables) + list(state1) + (list(state2) if state2 else []):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    _ok(lib().oracle_backward_update(C.byref(model.s), len(batches), arr, _ptr_array(tables),
                                     _ptr_array(state1), _ptr_array(state2) if state2 else None,
                                     C.byref(o), step))


def table_grad(model, batches, t):
    arr = (Batch * len(batches))(*[b.s for b in batches])
    V, D = int(model.rows[t]), int(model.dims[t])
    G = np.zeros((V, D), np.float32)
    cnt = np.zeros(V, np.int64)
    _ok(lib().oracle_table_grad(C.byref(model.s), len(batches), arr, t, _p(G), _p(cnt)))
    return G, cnt


def row_grads(model, batches, q_table, q_row, ld):
    arr = (Batch * len(batches))(*[b.s for b in batches])
    qt, qr = _arr(q_table, np.int32), _arr(q_row, np.int64)
    G = np.zeros((len(qt), ld), np.float32)
    cnt = np.zeros(len(qt), np.int64)
    _ok(lib().oracle_row_grads(C.byref(model.s), len(batches), arr, len(qt), _p(qt), _p(qr), ld, _p(G), _p(cnt)))
    return G, cnt


def apply_update(G, count, w, s1, s2=None, kind=OPT_ADAGRAD, lr=0.01, step=1, D=None, eps=None,
                 beta1=0.9, beta2=0.999):
    """In-place on w/s1/s2 ([n, ld] float32)."""
    o = _opt(kind, lr, eps, beta1, beta2)
    n, ld = w.shape
    D = ld if D is None else D
    G = _arr(G, np.float32)
    cnt = None if count is None else _arr(count, np.int64)
    _ok(lib().oracle_apply_update(C.byref(o), step, n, D, ld, _p(G), _p(cnt), _p(w), _p(s1), _p(s2)))


def hot_select(pack, key, count, row_cost_bytes, capacity_bytes):
    pk, ky, ct = _arr(pack, np.int32), _arr(key, np.int64), _arr(count, np.uint64)
    rc = _arr(row_cost_bytes, np.int64)
    order = np.zeros(len(pk), np.int64)
    k = lib().oracle_hot_select(len(pk), _p(pk), _p(ky), _p(ct), _p(rc), int(capacity_bytes), _p(order))
    return order[:k].copy()


def fcounter_add(keys, counts):
    k = _arr(keys, np.int64)
    assert counts.dtype == np.uint64
    _ok(lib().oracle_fcounter_add(len(k), _p(k), _p(counts)))


def interleave_capacity(rbound, rparam):
    rb, rp = _arr(rbound, np.float64), _arr(rparam, np.float64)
    return lib().oracle_interleave_capacity(len(rb), _p(rb), _p(rp))


def kinterleave_plan(field_to_table, table_rows, table_dim, capacity, excluded=None, warmup_count=None):
    f2t, rows, dims = _arr(field_to_table, np.int32), _arr(table_rows, np.int64), _arr(table_dim, np.int32)
    T = len(rows)
    wc = None if warmup_count is None else _arr(warmup_count, np.uint64)
    ex = None if excluded is None else _arr(excluded, np.uint8)
    t2p, tb = np.zeros(T, np.int32), np.zeros(T, np.int64)
    pd, pr, pg = np.zeros(T, np.int32), np.zeros(T, np.int64), np.zeros(T, np.int32)
    ng = C.c_int32()
    P = lib().oracle_kinterleave_plan(len(f2t), _p(f2t), T, _p(rows), _p(dims), _p(wc), float(capacity), _p(ex),
                                      _p(t2p), _p(tb), _p(pd), _p(pr), _p(pg), C.byref(ng))
    return dict(table_to_pack=t2p, table_base=tb, pack_dim=pd[:P].copy(), pack_rows=pr[:P].copy(), n_packs=P,
                pack_group=pg[:P].copy(), n_groups=ng.value, field_to_pack=t2p[f2t])
