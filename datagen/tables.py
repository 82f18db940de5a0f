"""Initial embedding-table values: W_t[row][d] ~ U[-0.05, 0.05) from an integer counter hash
of (seed, t, row, d).  Two bit-identical implementations of the SAME generator: numpy (host,
for the oracle) and torch (device, to fill the 24-113 GB tables without a host copy).
Pure input generation: no arithmetic of the method lives here."""
from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF


def _lowbias32_np(x):
    x = x & M32
    x ^= x >> np.uint64(16)
    x = (x * np.uint64(0x7FEB352D)) & np.uint64(M32)
    x ^= x >> np.uint64(15)
    x = (x * np.uint64(0x846CA68B)) & np.uint64(M32)
    x ^= x >> np.uint64(16)
    return x


def _lowbias32_t(x):
    x = x & M32
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & M32
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & M32
    x = x ^ (x >> 16)
    return x


def _table_key(seed, t):
    return (int(t) * 2654435761 + int(seed)) & M32


def table_values_np(seed: int, t: int, rows: np.ndarray, D: int) -> np.ndarray:
    """float32 [len(rows), D]."""
    rows = np.asarray(rows, np.int64).astype(np.uint64)
    c = rows[:, None] * np.uint64(D) + np.arange(D, dtype=np.uint64)[None, :]
    k = _lowbias32_np(np.uint64(_table_key(seed, t)))
    h = _lowbias32_np((c & np.uint64(M32)) ^ _lowbias32_np((c >> np.uint64(32)) ^ k))
    v = (h >> np.uint64(8)).astype(np.float32) * np.float32(2.0 ** -24)
    return (v * np.float32(0.1) - np.float32(0.05)).astype(np.float32)


def table_values_torch(seed: int, t, rows, D: int):
    """Same generator on torch int64 tensors (t may be a tensor aligned with rows)."""
    import torch

    rows = rows.to(torch.int64)
    c = rows[:, None] * D + torch.arange(D, device=rows.device, dtype=torch.int64)[None, :]
    if isinstance(t, int):
        k = torch.full_like(rows, _table_key(seed, t))
    else:
        k = (t.to(torch.int64) * 2654435761 + int(seed)) & M32
    k = _lowbias32_t(k)[:, None]
    h = _lowbias32_t((c & M32) ^ _lowbias32_t((c >> 32) ^ k))
    v = (h >> 8).to(torch.float32) * (2.0 ** -24)
    return v * torch.tensor(0.1, dtype=torch.float32) - torch.tensor(0.05, dtype=torch.float32)


def init_pack_tables_torch(cfg, table_to_pack, table_base, n_packs, weights, rank=0, world=1,
                           chunk_rows=1 << 20):
    """Fill each pack's local row shard (torch tensors [rows_local_p, D_p]) in place.
    Local row lr of rank r holds pack key lr*world + r (row-wise sharding, key mod W)."""
    import torch

    t2p = np.asarray(table_to_pack)
    tb = np.asarray(table_base)
    for p in range(n_packs):
        W = weights[p]
        dev = W.device if W.is_cuda else torch.device("cuda", torch.cuda.current_device())  # host tables: made on the GPU
        tabs = np.nonzero(t2p == p)[0]
        tabs = tabs[np.argsort(tb[tabs], kind="stable")]
        bases = torch.tensor(tb[tabs], dtype=torch.int64, device=dev)
        tids = torch.tensor(tabs, dtype=torch.int64, device=dev)
        n, KD = W.shape
        D = int(cfg.table_dim[tabs[0]])  # the tables' own dim; columns D..KD are the kernel-dim padding
        for s in range(0, n, chunk_rows):
            e = min(n, s + chunk_rows)
            lr = torch.arange(s, e, device=dev, dtype=torch.int64)
            key = lr * world + rank
            ti = torch.searchsorted(bases, key, right=True) - 1
            row = key - bases[ti]
            vals = table_values_torch(cfg.seed, tids[ti], row, D).to(W.device)
            if D == KD:
                W[s:e] = vals
            else:
                W[s:e, :D] = vals
                W[s:e, D:] = 0.0
