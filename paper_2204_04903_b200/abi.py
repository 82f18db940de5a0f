"""ctypes binding of include/picasso.h — same names, argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libpicasso.so")

POOL_SUM, POOL_MEAN = 0, 1
OPT_ADAGRAD, OPT_ADAM_LAZY = 0, 1
IDS_ROWS, IDS_HASH = 0, 1

_STATUS = {0: "OK", -1: "INVALID_ARG", -2: "PLAN_MISMATCH", -3: "ID_RANGE", -4: "CAPACITY", -5: "CUDA",
           -6: "NCCL", -7: "STATE"}

EXPORTS = ["picasso_pack_plan", "picasso_ctx_create", "picasso_workspace_size", "picasso_pack_local_rows",
           "picasso_bind", "picasso_ctx_destroy", "picasso_packed_lookup_fwd", "picasso_packed_lookup_bwd_update",
           "picasso_last_error", "picasso_get_unique", "picasso_get_inverse", "picasso_launch_count",
           "picasso_profile_enable", "picasso_profile_read", "picasso_unique_offsets", "picasso_nccl_unique_id",
           "picasso_group_create", "picasso_group_destroy", "picasso_group_fwd", "picasso_group_bwd_update",
           "picasso_get_owner_unique", "picasso_get_send_counts", "picasso_hot_cache_refresh",
           "picasso_group_hot_cache_refresh", "picasso_get_hot_keys", "picasso_p2p_handle", "picasso_p2p_open",
           "picasso_group_p2p", "picasso_get_send_list", "picasso_micro_batch_size", "picasso_dinterleave_begin",
           "picasso_packed_lookup_bwd_accumulate", "picasso_dinterleave_apply", "picasso_dinterleave_stats",
           "picasso_interleave_capacity", "picasso_pack_plan_kinterleave", "picasso_nvls_create", "picasso_nvls_open",
           "picasso_nvls_bind", "picasso_kernel_dim", "picasso_profile_read_packs"]
PHASES = ["unique", "pool", "transpose", "segsum", "owner_gather", "update"]


class PicassoError(RuntimeError):
    def __init__(self, status, where, msg=""):
        super().__init__(f"{where}: PICASSO_ERR_{_STATUS.get(status, status)} {msg}".strip())
        self.status = status


class PlanView(C.Structure):
    _fields_ = [("n_fields", C.c_int32), ("n_tables", C.c_int32), ("n_packs", C.c_int32),
                ("field_to_table", C.c_void_p), ("table_to_pack", C.c_void_p), ("table_base", C.c_void_p),
                ("table_rows", C.c_void_p), ("table_dim", C.c_void_p), ("table_salt", C.c_void_p),
                ("field_col", C.c_void_p), ("out_width", C.c_int64), ("pack_group", C.c_void_p)]


class CtxOpts(C.Structure):
    _fields_ = [("max_batch", C.c_int32), ("max_ids", C.c_int64), ("pool", C.c_int32), ("id_mode", C.c_int32),
                ("opt", C.c_int32), ("eps", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("max_recv", C.c_int64), ("cache_max_bytes", C.c_int64), ("exchange", C.c_int32),
                ("max_step_unique", C.c_int64), ("max_step_floats", C.c_int64), ("cold_tier", C.c_int32)]


class CacheStats(C.Structure):
    _fields_ = [("k", C.c_int64), ("bytes", C.c_int64), ("hot_uniques", C.c_int64), ("uniques", C.c_int64),
                ("hit_ratio_unique", C.c_double), ("refresh_ms", C.c_double), ("propose_ms", C.c_double),
                ("select_ms", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None


def lib():
    """Load libpicasso.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(lib_path):
            raise ImportError(f"{lib_path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(lib_path)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "picasso_pack_plan": [i32, vp, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp],
            "picasso_ctx_create": [C.POINTER(PlanView), i32, i32, vp, C.POINTER(CtxOpts), C.POINTER(vp)],
            "picasso_nccl_unique_id": [vp],
            "picasso_group_create": [vp, i32, C.POINTER(vp)],
            "picasso_group_destroy": [vp],
            "picasso_group_fwd": [vp, vp, vp, vp, vp, vp, vp],
            "picasso_group_bwd_update": [vp, vp, C.c_float, i64, vp],
            "picasso_get_owner_unique": [vp, i32, vp, i64, C.POINTER(i64)],
            "picasso_get_send_counts": [vp, vp],
            "picasso_get_send_list": [vp, i32, i32, vp, i64, C.POINTER(i64)],
            "picasso_hot_cache_refresh": [vp, C.c_size_t, vp, vp],
            "picasso_group_hot_cache_refresh": [vp, C.c_size_t, vp, vp],
            "picasso_get_hot_keys": [vp, vp, vp, i64, C.POINTER(i64)],
            "picasso_workspace_size": [vp, C.POINTER(C.c_size_t)],
            "picasso_pack_local_rows": [vp, i32, C.POINTER(i64)],
            "picasso_bind": [vp, vp, C.c_size_t, vp, vp, vp],
            "picasso_ctx_destroy": [vp],
            "picasso_packed_lookup_fwd": [vp, vp, vp, i32, i64, vp, vp],
            "picasso_packed_lookup_bwd_update": [vp, vp, C.c_float, i64, vp],
            "picasso_last_error": [vp, C.c_char_p, C.c_size_t],
            "picasso_get_unique": [vp, i32, vp, i64, C.POINTER(i64)],
            "picasso_get_inverse": [vp, i32, vp, i64, C.POINTER(i64)],
            "picasso_launch_count": [vp, C.POINTER(i64), C.POINTER(i64)],
            "picasso_profile_enable": [vp, i32],
            "picasso_profile_read": [vp, vp, C.POINTER(i64)],
            "picasso_unique_offsets": [vp, vp, vp],
            "picasso_micro_batch_size": [i32, vp, vp, i32, C.POINTER(i32), C.POINTER(i32)],
            "picasso_dinterleave_begin": [vp, vp],
            "picasso_packed_lookup_bwd_accumulate": [vp, vp, vp],
            "picasso_dinterleave_apply": [vp, C.c_float, i64, vp],
            "picasso_dinterleave_stats": [vp, C.POINTER(i64), C.POINTER(i64)],
            "picasso_interleave_capacity": [i32, vp, vp, C.POINTER(C.c_double)],
            "picasso_nvls_create": [vp, C.POINTER(i32)],
            "picasso_nvls_open": [vp, i32],
            "picasso_nvls_bind": [vp],
            "picasso_kernel_dim": [i32, C.POINTER(i32)],
            "picasso_profile_read_packs": [vp, vp, vp, i32],
            "picasso_pack_plan_kinterleave": [i32, vp, i32, vp, vp, vp, C.c_double, vp, vp, vp, vp, vp, vp, vp,
                                              C.POINTER(i32), C.POINTER(i32)],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        _lib = L
    return _lib


def _chk(st, where, ctx=None):
    if st != 0:
        msg = ""
        if ctx is not None:
            buf = C.create_string_buffer(256)
            lib().picasso_last_error(ctx, buf, 256)
            msg = buf.value.decode(errors="replace")
        raise PicassoError(st, where, msg)


def _np(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


# ------------------------------------------------------------------------------------------
def picasso_pack_plan(field_to_table, table_rows, table_dim, table_warmup_count=None, split=False):
    f2t, rows, dims = _np(field_to_table, np.int32), _np(table_rows, np.int64), _np(table_dim, np.int32)
    wc = None if table_warmup_count is None else _np(table_warmup_count, np.uint64)
    F, T = len(f2t), len(rows)
    f2p, t2p = np.zeros(F, np.int32), np.zeros(T, np.int32)
    tb, pd, pr = np.zeros(T, np.int64), np.zeros(T, np.int32), np.zeros(T, np.int64)
    n = C.c_int32()
    st = lib().picasso_pack_plan(F, f2t.ctypes.data, T, rows.ctypes.data, dims.ctypes.data,
                                 None if wc is None else wc.ctypes.data, int(split), f2p.ctypes.data,
                                 t2p.ctypes.data, tb.ctypes.data, pd.ctypes.data, pr.ctypes.data, C.byref(n))
    _chk(st, "picasso_pack_plan")
    P = n.value
    return dict(field_to_pack=f2p, table_to_pack=t2p, table_base=tb, pack_dim=pd[:P].copy(),
                pack_rows=pr[:P].copy(), n_packs=P)


def picasso_interleave_capacity(rbound, rparam):
    """Eq. 3: Capacity_g = min over ops of rbound / rparam (parameters per step)."""
    rb, rp = _np(rbound, np.float64), _np(rparam, np.float64)
    c = C.c_double()
    _chk(lib().picasso_interleave_capacity(len(rb), rb.ctypes.data, rp.ctypes.data, C.byref(c)),
         "picasso_interleave_capacity")
    return c.value


def picasso_pack_plan_kinterleave(field_to_table, table_rows, table_dim, capacity_g, excluded=None,
                                  table_warmup_count=None):
    """The K-Interleaving plan (include/picasso.h 1b): picasso_pack_plan's dict plus pack_group
    (-1 = preset excluded) and n_groups."""
    f2t, rows, dims = _np(field_to_table, np.int32), _np(table_rows, np.int64), _np(table_dim, np.int32)
    wc = None if table_warmup_count is None else _np(table_warmup_count, np.uint64)
    ex = None if excluded is None else _np(excluded, np.uint8)
    F, T = len(f2t), len(rows)
    f2p, t2p = np.zeros(F, np.int32), np.zeros(T, np.int32)
    tb, pd, pr, pg = np.zeros(T, np.int64), np.zeros(T, np.int32), np.zeros(T, np.int64), np.zeros(T, np.int32)
    n, g = C.c_int32(), C.c_int32()
    st = lib().picasso_pack_plan_kinterleave(F, f2t.ctypes.data, T, rows.ctypes.data, dims.ctypes.data,
                                             None if wc is None else wc.ctypes.data, float(capacity_g),
                                             None if ex is None else ex.ctypes.data, f2p.ctypes.data,
                                             t2p.ctypes.data, tb.ctypes.data, pd.ctypes.data, pr.ctypes.data,
                                             pg.ctypes.data, C.byref(n), C.byref(g))
    _chk(st, "picasso_pack_plan_kinterleave")
    P = n.value
    return dict(field_to_pack=f2p, table_to_pack=t2p, table_base=tb, pack_dim=pd[:P].copy(),
                pack_rows=pr[:P].copy(), n_packs=P, pack_group=pg[:P].copy(), n_groups=g.value)


def picasso_kernel_dim(dim):
    """The padded row width a table of embedding dim `dim` is stored at."""
    k = C.c_int32()
    _chk(lib().picasso_kernel_dim(int(dim), C.byref(k)), "picasso_kernel_dim")
    return k.value


class _Keep:
    """Keeps numpy arrays referenced by a C struct alive."""


def picasso_nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    _chk(lib().picasso_nccl_unique_id(buf), "picasso_nccl_unique_id")
    return bytes(buf)


def picasso_ctx_create(plan, field_to_table, table_rows, table_dim, table_salt, field_col, out_width, rank, world,
                       max_batch, max_ids, pool=POOL_SUM, id_mode=IDS_HASH, opt=OPT_ADAGRAD, eps=None, beta1=0.9,
                       beta2=0.999, nccl_uid=None, max_recv=0, cache_max_bytes=0, exchange="p2p", max_step_unique=0,
                       max_step_floats=0, cold_tier=0):
    k = _Keep()
    k.f2t = _np(field_to_table, np.int32)
    k.t2p = _np(plan["table_to_pack"], np.int32)
    k.tb = _np(plan["table_base"], np.int64)
    k.rows = _np(table_rows, np.int64)
    k.dims = _np(table_dim, np.int32)
    k.salt = _np(np.zeros(len(k.rows)) if table_salt is None else table_salt, np.uint64)
    k.col = _np(field_col, np.int64)
    k.pg = None if plan.get("pack_group") is None else _np(plan["pack_group"], np.int32)
    pv = PlanView(len(k.f2t), len(k.rows), int(plan["n_packs"]), k.f2t.ctypes.data, k.t2p.ctypes.data,
                  k.tb.ctypes.data, k.rows.ctypes.data, k.dims.ctypes.data, k.salt.ctypes.data, k.col.ctypes.data,
                  int(out_width), None if k.pg is None else k.pg.ctypes.data)
    if eps is None:
        eps = 1e-10 if opt == OPT_ADAGRAD else 1e-8
    o = CtxOpts(int(max_batch), int(max_ids), int(pool), int(id_mode), int(opt), float(eps), float(beta1),
                float(beta2), int(max_recv), int(cache_max_bytes), 0 if exchange == "p2p" else 1, int(max_step_unique),
                int(max_step_floats), int(cold_tier))
    ctx = C.c_void_p()
    uid = None if nccl_uid is None else (C.c_uint8 * 128)(*nccl_uid)
    _chk(lib().picasso_ctx_create(C.byref(pv), int(rank), int(world), uid, C.byref(o), C.byref(ctx)),
         "picasso_ctx_create")
    return ctx


def picasso_workspace_size(ctx):
    n = C.c_size_t()
    _chk(lib().picasso_workspace_size(ctx, C.byref(n)), "picasso_workspace_size")
    return n.value


def picasso_pack_local_rows(ctx, pack):
    n = C.c_int64()
    _chk(lib().picasso_pack_local_rows(ctx, int(pack), C.byref(n)), "picasso_pack_local_rows")
    return n.value


def picasso_bind(ctx, workspace, weights, state1, state2=None):
    P = len(weights)
    w = (C.c_void_p * P)(*[t.data_ptr() for t in weights])
    s1 = (C.c_void_p * P)(*[t.data_ptr() for t in state1])
    s2 = None if state2 is None else (C.c_void_p * P)(*[t.data_ptr() for t in state2])
    _chk(lib().picasso_bind(ctx, C.c_void_p(workspace.data_ptr()), workspace.numel() * workspace.element_size(),
                            w, s1, s2), "picasso_bind", ctx)


def picasso_ctx_destroy(ctx):
    lib().picasso_ctx_destroy(ctx)


def _same_device(a, b):
    import torch

    b = torch.device(b)
    if b.index is None:
        b = torch.device(b.type, torch.cuda.current_device())
    return a == b


def _check(t, name, dtype, numel=None, shape=None, device=None):
    """Host-side argument checks (the C ABI takes raw pointers and cannot see them): dtype,
    contiguity, device and size of a tensor argument.  Raises PicassoError(INVALID_ARG)."""
    import torch

    if t is None:
        return
    bad = None
    if t.dtype != dtype:
        bad = f"dtype {t.dtype}, expected {dtype}"
    elif not t.is_contiguous():
        bad = "not contiguous"
    elif not t.is_cuda:
        bad = "not a CUDA tensor"
    elif device is not None and not _same_device(t.device, device):
        bad = f"on {t.device}, expected {device}"
    elif not t.is_cuda:
        bad = "not a CUDA tensor"
    elif numel is not None and t.numel() != numel:
        bad = f"{t.numel()} elements, expected {numel}"
    elif shape is not None and tuple(t.shape) != tuple(shape):
        bad = f"shape {tuple(t.shape)}, expected {tuple(shape)}"
    if bad:
        raise PicassoError(-1, "argument check", f"{name}: {bad}")


def picasso_packed_lookup_fwd(ctx, ids, offsets, batch, out, stream=None, n_fields=None, out_width=None,
                              device=None):
    """ids int64 [N], offsets int32 [F*B+1] (CSR over the N ids, field-major), out fp32 [B, out_width]:
    all contiguous CUDA tensors on the ctx's device.  n_fields / out_width (known to PackedEmbedding)
    enable the size checks; offsets[F*B] == N is checked on the device (latched, picasso_last_error)."""
    import torch

    _check(ids, "ids", torch.int64, device=device)
    _check(offsets, "offsets", torch.int32, numel=None if n_fields is None else int(n_fields) * int(batch) + 1,
           device=device)
    _check(out, "out", torch.float32, shape=None if out_width is None else (int(batch), int(out_width)),
           device=device)
    _chk(lib().picasso_packed_lookup_fwd(ctx, _ptr(ids), _ptr(offsets), int(batch), int(ids.numel()), _ptr(out),
                                         _stream(stream)), "picasso_packed_lookup_fwd", ctx)


def picasso_packed_lookup_bwd_update(ctx, grad_out, lr, step, stream=None, batch=None, out_width=None, device=None):
    """grad_out fp32 [B, out_width] contiguous, the forward's output layout."""
    import torch

    _check(grad_out, "grad_out", torch.float32,
           shape=None if (batch is None or out_width is None) else (int(batch), int(out_width)), device=device)
    _chk(lib().picasso_packed_lookup_bwd_update(ctx, _ptr(grad_out), float(lr), int(step), _stream(stream)),
         "picasso_packed_lookup_bwd_update", ctx)


def picasso_last_error(ctx):
    buf = C.create_string_buffer(512)
    st = lib().picasso_last_error(ctx, buf, 512)
    return st, buf.value.decode(errors="replace")


def picasso_get_unique(ctx, pack, device):
    import torch

    n = C.c_int64()
    _chk(lib().picasso_get_unique(ctx, int(pack), None, 0, C.byref(n)), "picasso_get_unique", ctx)
    out = torch.empty(max(n.value, 1), dtype=torch.int64, device=device)
    _chk(lib().picasso_get_unique(ctx, int(pack), _ptr(out), n.value, C.byref(n)), "picasso_get_unique", ctx)
    return out[:n.value]


def picasso_get_inverse(ctx, pack, device):
    import torch

    n = C.c_int64()
    _chk(lib().picasso_get_inverse(ctx, int(pack), None, 0, C.byref(n)), "picasso_get_inverse", ctx)
    out = torch.empty(max(n.value, 1), dtype=torch.int32, device=device)
    _chk(lib().picasso_get_inverse(ctx, int(pack), _ptr(out), n.value, C.byref(n)), "picasso_get_inverse", ctx)
    return out[:n.value]


def picasso_launch_count(ctx):
    f, b = C.c_int64(), C.c_int64()
    _chk(lib().picasso_launch_count(ctx, C.byref(f), C.byref(b)), "picasso_launch_count")
    return f.value, b.value


def picasso_profile_enable(ctx, on=True):
    """on: False/True, or 2 before capturing the step into a CUDA graph."""
    _chk(lib().picasso_profile_enable(ctx, 2 if on == 2 and not isinstance(on, bool) else int(bool(on))),
         "picasso_profile_enable")


def picasso_profile_read(ctx):
    """{phase: summed ms since the last read}, number of profiled steps."""
    ms = (C.c_float * len(PHASES))()
    n = C.c_int64()
    _chk(lib().picasso_profile_read(ctx, ms, C.byref(n)), "picasso_profile_read", ctx)
    return {PHASES[i]: float(ms[i]) for i in range(len(PHASES))}, n.value


def picasso_profile_read_packs(ctx, n_packs):
    """Per pack: (pool ms, backward ms) summed since the last picasso_profile_read (call before it)."""
    pool = (C.c_float * n_packs)()
    bwd = (C.c_float * n_packs)()
    _chk(lib().picasso_profile_read_packs(ctx, pool, bwd, int(n_packs)), "picasso_profile_read_packs", ctx)
    return list(pool), list(bwd)


# ---- world > 1 ---------------------------------------------------------------------------
def picasso_p2p_handle(ctx):
    buf = (C.c_uint8 * 64)()
    _chk(lib().picasso_p2p_handle(ctx, buf), "picasso_p2p_handle", ctx)
    return bytes(buf)


def picasso_p2p_open(ctx, handles):
    blob = b"".join(handles)
    buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
    _chk(lib().picasso_p2p_open(ctx, buf), "picasso_p2p_open", ctx)


def picasso_group_p2p(group):
    _chk(lib().picasso_group_p2p(group), "picasso_group_p2p")


def picasso_group_create(ctxs):
    arr = (C.c_void_p * len(ctxs))(*[c.value for c in ctxs])
    g = C.c_void_p()
    _chk(lib().picasso_group_create(arr, len(ctxs), C.byref(g)), "picasso_group_create")
    return g


def picasso_group_destroy(group):
    lib().picasso_group_destroy(group)


def _ptrs(ts):
    return (C.c_void_p * len(ts))(*[t.data_ptr() if t.numel() else None for t in ts])


def picasso_group_fwd(group, ids, offsets, batch, out, stream=None):
    W = len(ids)
    b = (C.c_int32 * W)(*[int(x) for x in batch])
    n = (C.c_int64 * W)(*[int(t.numel()) for t in ids])
    _chk(lib().picasso_group_fwd(group, _ptrs(ids), _ptrs(offsets), b, n, _ptrs(out), _stream(stream)),
         "picasso_group_fwd")


def picasso_group_bwd_update(group, grad_out, lr, step, stream=None):
    _chk(lib().picasso_group_bwd_update(group, _ptrs(grad_out), float(lr), int(step), _stream(stream)),
         "picasso_group_bwd_update")


def picasso_get_owner_unique(ctx, pack, device):
    import torch

    n = C.c_int64()
    _chk(lib().picasso_get_owner_unique(ctx, int(pack), None, 0, C.byref(n)), "picasso_get_owner_unique", ctx)
    out = torch.empty(max(n.value, 1), dtype=torch.int64, device=device)
    _chk(lib().picasso_get_owner_unique(ctx, int(pack), _ptr(out), n.value, C.byref(n)), "picasso_get_owner_unique",
         ctx)
    return out[:n.value]


def picasso_get_send_counts(ctx, world):
    arr = (C.c_int64 * world)()
    _chk(lib().picasso_get_send_counts(ctx, arr), "picasso_get_send_counts", ctx)
    return list(arr)


def picasso_get_send_list(ctx, owner, pack):
    """Local rows this rank requested from `owner` for `pack`, send order (numpy int64)."""
    n = C.c_int64()
    _chk(lib().picasso_get_send_list(ctx, int(owner), int(pack), None, 0, C.byref(n)), "picasso_get_send_list", ctx)
    out = np.zeros(max(n.value, 1), np.int64)
    _chk(lib().picasso_get_send_list(ctx, int(owner), int(pack), out.ctypes.data, n.value, C.byref(n)),
         "picasso_get_send_list", ctx)
    return out[:n.value]


def picasso_unique_offsets(ctx, dst, stream=None):
    """Enqueue a copy of the int32 [n_packs+1] uid prefix of the last forward into `dst` (a
    device tensor or a pinned host tensor)."""
    _chk(lib().picasso_unique_offsets(ctx, _ptr(dst), _stream(stream)), "picasso_unique_offsets", ctx)
    return dst


# ---- HybridHash ---------------------------------------------------------------------------
def picasso_hot_cache_refresh(ctx, capacity_bytes, stream=None):
    st = CacheStats()
    _chk(lib().picasso_hot_cache_refresh(ctx, int(capacity_bytes), _stream(stream), C.byref(st)),
         "picasso_hot_cache_refresh", ctx)
    return st.as_dict()


def picasso_group_hot_cache_refresh(group, world, capacity_bytes, stream=None):
    st = (CacheStats * world)()
    _chk(lib().picasso_group_hot_cache_refresh(group, int(capacity_bytes), _stream(stream), st),
         "picasso_group_hot_cache_refresh")
    return [s.as_dict() for s in st]


def picasso_get_hot_keys(ctx):
    n = C.c_int64()
    _chk(lib().picasso_get_hot_keys(ctx, None, None, 0, C.byref(n)), "picasso_get_hot_keys", ctx)
    pk = np.zeros(max(n.value, 1), np.int32)
    ky = np.zeros(max(n.value, 1), np.int64)
    _chk(lib().picasso_get_hot_keys(ctx, pk.ctypes.data, ky.ctypes.data, n.value, C.byref(n)), "picasso_get_hot_keys",
         ctx)
    return pk[:n.value], ky[:n.value]


# ---- D-Interleaving (include/picasso.h section 8) -----------------------------------------
def picasso_micro_batch_size(rbound, rinstance, batch):
    """Eq. 2: (bs_micro, n_micro) from per-op bounds and per-instance costs (sequences of floats)."""
    rb = _np(rbound, np.float64)
    ri = _np(rinstance, np.float64)
    bs, n = C.c_int32(), C.c_int32()
    _chk(lib().picasso_micro_batch_size(len(rb), rb.ctypes.data, ri.ctypes.data, int(batch), C.byref(bs), C.byref(n)),
         "picasso_micro_batch_size")
    return bs.value, n.value


def picasso_dinterleave_begin(ctx, stream=None):
    _chk(lib().picasso_dinterleave_begin(ctx, _stream(stream)), "picasso_dinterleave_begin", ctx)


def picasso_packed_lookup_bwd_accumulate(ctx, grad_out, stream=None, batch=None, out_width=None, device=None):
    import torch

    _check(grad_out, "grad_out", torch.float32,
           shape=None if (batch is None or out_width is None) else (int(batch), int(out_width)), device=device)
    _chk(lib().picasso_packed_lookup_bwd_accumulate(ctx, _ptr(grad_out), _stream(stream)),
         "picasso_packed_lookup_bwd_accumulate", ctx)


def picasso_dinterleave_apply(ctx, lr, step, stream=None):
    _chk(lib().picasso_dinterleave_apply(ctx, float(lr), int(step), _stream(stream)), "picasso_dinterleave_apply", ctx)


def picasso_dinterleave_stats(ctx):
    """(distinct keys, fp64 values) the last D-Interleaving step accumulated."""
    r, f = C.c_int64(), C.c_int64()
    _chk(lib().picasso_dinterleave_stats(ctx, C.byref(r), C.byref(f)), "picasso_dinterleave_stats", ctx)
    return r.value, f.value


# ---- NVLS multicast of the hot-row gradients (include/picasso.h 7b) -----------------------
def picasso_nvls_create(ctx):
    """Rank 0: the multicast object's POSIX file descriptor; other ranks: -1."""
    fd = C.c_int32(-1)
    _chk(lib().picasso_nvls_create(ctx, C.byref(fd)), "picasso_nvls_create", ctx)
    return fd.value


def picasso_nvls_open(ctx, fd):
    _chk(lib().picasso_nvls_open(ctx, int(fd)), "picasso_nvls_open", ctx)


def picasso_nvls_bind(ctx):
    _chk(lib().picasso_nvls_bind(ctx), "picasso_nvls_bind", ctx)
