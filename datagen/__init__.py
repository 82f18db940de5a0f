"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This package holds NO arithmetic of the method (no row mapping, dedup, pooling, gradient or
optimizer math).  It only draws inputs: Zipf-distributed categorical IDs with bag offsets,
initial table values, and upstream gradients dY.  Every draw is a pure function of
(seed, config, rank, step, field) through counter-based generators (numpy Philox; the
table-value hash is integer-exact in both numpy and torch), so the oracle and the GPU path
see identical inputs.  The recipe is stated in DESIGN.md §4.
"""
from .zipf import ZipfSampler, zipf_head_mass, resolve_alpha  # noqa: F401
from .configs import CONFIGS, Config, get_config  # noqa: F401
from .batch import make_batch, make_dy, Batch  # noqa: F401
from .tables import table_values_np, table_values_torch, init_pack_tables_torch  # noqa: F401
