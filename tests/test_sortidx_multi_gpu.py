"""The row-sharded step indexed by sort (world > 1; csrc/k_sortidx.cu through mfwd_a): Unique /
inverse from the sort's reading-O1 views, the backward in run order with its per-row destinations
gathered through run -> uid, no uid transpose.  The loopback parity cases of test_multi_gpu.py and
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
