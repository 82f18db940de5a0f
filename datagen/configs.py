"""Synthetic workload shapes (BASELINE.json "configs"; recipe in DESIGN.md §4).

Shapes follow SURVEY.md §8(d) and the paper's workloads: Criteo (26 fields, dim 128,
PAPER.md tab:dataset L588), sequence features counted as positional fields sharing one
table (L592-593: 1,834 fields = 334 + 30x50), multi-hot length <= 50.
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

import numpy as np

IDS_ROWS, IDS_HASH = 0, 1
POOL_SUM, POOL_MEAN = 0, 1
SEED = 220404903


@dataclasses.dataclass
class Config:
    name: str
    batch: int                     # B per rank
    field_to_table: np.ndarray     # int32 [F]
    table_rows: np.ndarray         # int64 [T]
    table_dim: np.ndarray          # int32 [T]
    bags: List[Tuple]              # per field: ("fixed", L) | ("uniform", lo, hi) | ("seqpos", s, p)
    alpha: float = 0.8
    id_mode: int = IDS_HASH
    pool: int = POOL_SUM
    seq_max: int = 50
    cfg_id: int = 0
    seed: int = SEED

    @property
    def F(self):
        return len(self.field_to_table)

    @property
    def T(self):
        return len(self.table_rows)

    @property
    def field_dim(self):
        return self.table_dim[self.field_to_table]

    @property
    def field_col(self):
        d = self.field_dim.astype(np.int64)
        return np.concatenate([[0], np.cumsum(d)[:-1]]).astype(np.int64)

    @property
    def out_width(self):
        return int(self.field_dim.astype(np.int64).sum())

    @property
    def table_salt(self):
        t = np.arange(1, self.T + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            return (t * np.uint64(0xA24BAED4963EE407)) ^ np.uint64(self.seed)

    def replace(self, **kw):
        return dataclasses.replace(self, **kw)

    def n_seq(self):
        return 1 + max([b[1] for b in self.bags if b[0] == "seqpos"], default=-1)


def toy(**kw) -> Config:
    """C1: 8 fields, 1K-row tables of dim 16, batch 256, multi-hot <= 4 (empty bags occur), sum."""
    F = 8
    return Config("toy", 256, np.arange(F, dtype=np.int32), np.full(F, 1000, np.int64),
                  np.full(F, 16, np.int32), [("uniform", 0, 4)] * F, alpha=1.0, cfg_id=1).replace(**kw)


def criteo(**kw) -> Config:
    """C2: Criteo-shaped DLRM, 26 one-hot fields, dim 128, batch 16K, sum 46.875M rows
    (6B params / 128, PAPER.md tab:dataset L588); V_f = max(4, round(Vmax*10^(-7(25-f)/25)))."""
    F = 26
    w = 10.0 ** (-7.0 * (25 - np.arange(F)) / 25.0)
    vmax = 46_875_000 / w.sum()
    rows = np.maximum(4, np.round(vmax * w)).astype(np.int64)
    return Config("criteo", 16384, np.arange(F, dtype=np.int32), rows, np.full(F, 128, np.int32),
                  [("fixed", 1)] * F, alpha=0.8, cfg_id=2).replace(**kw)


def wdl(**kw) -> Config:
    """C3: W&D/DIN-style, 200 multi-hot fields (L ~ U{1..50}), dims 8/16/32/64 round-robin
    (4 dim-packs x 50), 2M rows per field-table, batch 16K per rank."""
    F = 200
    dims = np.array([8, 16, 32, 64], np.int32)[np.arange(F) % 4]
    return Config("wdl", 16384, np.arange(F, dtype=np.int32), np.full(F, 2_000_000, np.int64), dims,
                  [("uniform", 1, 50)] * F, alpha=0.8, cfg_id=3).replace(**kw)


def industrial(**kw) -> Config:
    """C4: 1000 fields = 250 one-hot attribute fields (tables log-spaced 1e3..1e7 rows) +
    15 sequence features x 50 positional fields (15 tables of 48.3M rows; position p is
    present iff p < L_seq, L_seq ~ U{0..50}); 265 tables, ~1.0B rows; dims round-robin
    {8,16,32,64} over tables; batch 64K per rank."""
    n_attr, n_seq, L = 250, 15, 50
    attr_rows = np.round(10.0 ** np.linspace(3, 7, n_attr)).astype(np.int64)
    rows = np.concatenate([attr_rows, np.full(n_seq, 48_300_000, np.int64)])
    T = n_attr + n_seq
    dims = np.array([8, 16, 32, 64], np.int32)[np.arange(T) % 4]
    f2t = list(range(n_attr))
    bags = [("fixed", 1)] * n_attr
    for s in range(n_seq):
        for p in range(L):
            f2t.append(n_attr + s)
            bags.append(("seqpos", s, p))
    return Config("industrial", 65536, np.array(f2t, np.int32), rows, dims, bags, alpha=0.8,
                  cfg_id=4).replace(**kw)


def skew(alpha=1.2, **kw) -> Config:
    """C5: the C3 shape under a different Zipf exponent (sweep 0.8..1.4)."""
    return wdl(alpha=alpha, cfg_id=5, name=f"skew{alpha}").replace(**kw)


CONFIGS = {"toy": toy, "criteo": criteo, "wdl": wdl, "industrial": industrial, "skew": skew}


def get_config(name: str, **kw) -> Config:
    return CONFIGS[name](**kw)


def scaled(cfg: Config, batch=None, rows_div=1, min_rows=4) -> Config:
    """Same field/dim/bag structure at a smaller batch and smaller tables (parity sizes)."""
    rows = np.maximum(min_rows, cfg.table_rows // rows_div).astype(np.int64)
    return cfg.replace(batch=batch or cfg.batch, table_rows=rows, name=cfg.name + "-small")
