"""The row-sharded step indexed by sort (world > 1; csrc/k_sortidx.cu through mfwd_a), no uid
transpose: with the peer-memory exchange the whole step in run order (send lists in ascending local
row, Unique / inverse views built on request); with the NCCL exchange Unique / inverse from the
sort's reading-O1 views and the backward's per-row destinations gathered through run -> uid.  The loopback parity cases of test_multi_gpu.py and
test_hot_cache_gpu.py re-run with every step sort-indexed (PICASSO_SORT_MIN_IDS_W=0): forward,
Unique, send lists, owner uniques and shards against the oracle, as on the hash path."""
import pytest

from test_multi_gpu import (exchange, test_criteo_small_sharded_continuous_dy, test_multipack_sharded,  # noqa: F401
                            test_sharded_adam_mean, test_sharded_hot_rows, test_toy_sharded)
from test_hot_cache_gpu import *  # noqa: F401,F403

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _sorted_row_sharded(monkeypatch):
    monkeypatch.setenv("PICASSO_SORT_MIN_IDS_W", "0")
