"""D-Interleaving (Eq. 2): micro-batch sizing and batch slicing — host-side
plumbing around the C ABI's section 8 (every step of the layer still runs in libpicasso).

Eq. 2:  BS_micro = min over ops of RBound_op / RInstance_op, with RInstance measured from
warm-up iterations ("we determine their values empirically or experimentally from warm-up
iterations of training", L419-421).  The ops whose memory grows with the batch are:

  * the pooled output and its gradient (out, dY):       8 * out_width bytes per sample
  * the layer's per-ID scratch (dedup, transpose, G):   ws_per_id * IDs per sample
  * the ID stream itself (ids, offsets):                8 * IDs per sample + 4 * F
"""
from __future__ import annotations

import numpy as np

from . import abi


def workspace_bytes_per_id(emb_kwargs: dict, probe=(1 << 16, 1 << 17)) -> float:
    """Bytes of ctx workspace per ID occurrence, measured as the difference quotient of
    picasso_workspace_size at two max_ids (world 1, no device memory is touched)."""
    sizes = []
    for mi in probe:
        kw = dict(emb_kwargs)
        kw["max_ids"] = mi
        ctx = abi.picasso_ctx_create(**kw)
        sizes.append(abi.picasso_workspace_size(ctx))
        abi.picasso_ctx_destroy(ctx)
    return (sizes[1] - sizes[0]) / float(probe[1] - probe[0])


def micro_batch_plan(batch, out_width, n_fields, ids_per_sample, ws_per_id, budget_bytes):
    """Eq. 2 over the three batch-proportional ops above.  Each op's RBound is its share of the
    device-memory budget in proportion to its cost (so the ops together fit the budget); returns
    (bs_micro, n_micro, {op: (rbound, rinstance)})."""
    rinst = {
        "out_dy": 8.0 * out_width,
        "index_scratch": ws_per_id * ids_per_sample,
        "id_stream": 8.0 * ids_per_sample + 4.0 * n_fields,
    }
    tot = sum(rinst.values())
    rb = {k: budget_bytes * v / tot for k, v in rinst.items()}
    bs, n = abi.picasso_micro_batch_size([rb[k] for k in rinst], [rinst[k] for k in rinst], batch)
    return bs, n, {k: (rb[k], rinst[k]) for k in rinst}


def slice_batch(ids: np.ndarray, offsets: np.ndarray, n_fields: int, batch: int, b0: int, b1: int):
    """Samples [b0, b1) of a field-major CSR batch (ids int64 [N], offsets int32 [F*B+1]) as a
    batch of their own: per field, its bags of those samples, fields concatenated in order."""
    F, B = n_fields, batch
    seg = offsets.astype(np.int64)
    starts = seg[np.arange(F) * B + b0]
    ends = seg[np.arange(F) * B + b1]
    idx = np.concatenate([np.arange(s, e) for s, e in zip(starts, ends)]) if F else np.zeros(0, np.int64)
    lens = np.diff(seg)[(np.arange(F)[:, None] * B + np.arange(b0, b1)[None, :]).reshape(-1)]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    return np.ascontiguousarray(ids[idx]), off


def even_slices(batch: int, n_micro: int):
    """[b0, b1) bounds of n_micro near-equal micro-batches (the paper's default)."""
    n = max(int(n_micro), 1)
    q, r = divmod(batch, n)
    out, b = [], 0
    for i in range(n):
        e = b + q + (1 if i < r else 0)
        out.append((b, e))
        b = e
    return out
