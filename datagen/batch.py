"""Per-rank, per-step synthetic batches: field-major IDs + int32 offsets, and dY."""
from __future__ import annotations

import dataclasses

import numpy as np

from .configs import IDS_HASH, Config
from .zipf import ZipfSampler

_SCRAMBLE = np.uint64(0xD6E8FEB86659FD93)  # odd => bijective on uint64


@dataclasses.dataclass
class Batch:
    batch: int
    ids: np.ndarray      # int64 [N], field-major
    offsets: np.ndarray  # int32 [F*B+1]
    lengths: np.ndarray  # int32 [F, B]

    @property
    def n_ids(self):
        return int(self.offsets[-1])


def _rng(cfg: Config, *stream):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([cfg.seed, cfg.cfg_id, *stream])))


_SAMPLERS = {}


def _sampler(V, alpha):
    key = (int(V), float(alpha))
    if key not in _SAMPLERS:
        _SAMPLERS[key] = ZipfSampler(V, alpha)
    return _SAMPLERS[key]


def _raw_ids(cfg: Config, t: int, ranks: np.ndarray) -> np.ndarray:
    """Zipf rank (1-based) -> raw categorical ID.  HASH mode: a bijective 64-bit scramble
    (raw IDs look like arbitrary 64-bit feature IDs); ROWS mode: a rotation into [0, V)."""
    if cfg.id_mode == IDS_HASH:
        with np.errstate(over="ignore"):
            u = ranks.astype(np.uint64) * _SCRAMBLE + np.uint64(t) * np.uint64(0x632BE59BD9B4E019)
        return u.view(np.int64)
    V = int(cfg.table_rows[t])
    rot = (t * 7919) % V
    return ((ranks - 1 + rot) % V).astype(np.int64)


def make_batch(cfg: Config, rank: int = 0, step: int = 0, batch: int | None = None) -> Batch:
    B = int(batch or cfg.batch)
    F = cfg.F
    lengths = np.zeros((F, B), np.int32)
    seq_len = {}
    for s in range(cfg.n_seq()):
        seq_len[s] = _rng(cfg, rank, step, 1_000_000 + s).integers(0, cfg.seq_max + 1, B).astype(np.int32)
    for f in range(F):
        bag = cfg.bags[f]
        if bag[0] == "fixed":
            lengths[f] = bag[1]
        elif bag[0] == "uniform":
            lengths[f] = _rng(cfg, rank, step, 2_000_000 + f).integers(bag[1], bag[2] + 1, B)
        elif bag[0] == "seqpos":
            lengths[f] = (seq_len[bag[1]] > bag[2]).astype(np.int32)
        else:
            raise ValueError(bag)
    offsets = np.zeros(F * B + 1, np.int64)
    np.cumsum(lengths.reshape(-1), out=offsets[1:])
    assert offsets[-1] < 2**31, "per-rank ID count must fit int32 offsets"
    ids = np.empty(int(offsets[-1]), np.int64)
    for f in range(F):
        t = int(cfg.field_to_table[f])
        lo, hi = int(offsets[f * B]), int(offsets[(f + 1) * B])
        if hi > lo:
            ranks = _sampler(cfg.table_rows[t], cfg.alpha).sample(_rng(cfg, rank, step, f), hi - lo)
            ids[lo:hi] = _raw_ids(cfg, t, ranks)
    return Batch(B, ids, offsets.astype(np.int32), lengths)


def make_dy(cfg: Config, rank: int = 0, step: int = 0, batch: int | None = None, dyadic: bool = True):
    """Upstream gradient dY [B, out_width] fp32.  dyadic: k*2^-8, k in [-7, 7] (reading O19:
    every partial sum is exact, so G is order independent); else U[-1, 1)."""
    B = int(batch or cfg.batch)
    g = _rng(cfg, rank, step, 3_000_000)
    if dyadic:
        return (g.integers(-7, 8, (B, cfg.out_width)).astype(np.float32) * np.float32(2.0 ** -8))
    return (g.random((B, cfg.out_width), dtype=np.float32) * 2.0 - 1.0).astype(np.float32)
