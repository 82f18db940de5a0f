"""B200-native PICASSO packed sparse-embedding hot path (arXiv 2204.04903).

The compute lives in ``libpicasso.so`` (hand-written sm_100a CUDA kernels behind the C ABI
of ``include/picasso.h``).  This package is argument marshalling only: it converts torch
tensors to raw pointers and calls the C entry points of the same names.  There is no CPU
fallback: importing fails loudly if the library is missing.
"""
from .abi import (  # noqa: F401
    PicassoError,
    lib,
    lib_path,
    picasso_bind,
    picasso_ctx_create,
    picasso_ctx_destroy,
    picasso_get_inverse,
    picasso_get_unique,
    picasso_last_error,
    picasso_launch_count,
    picasso_pack_local_rows,
    picasso_pack_plan,
    picasso_packed_lookup_bwd_update,
    picasso_packed_lookup_fwd,
    picasso_workspace_size,
    picasso_profile_enable,
    picasso_profile_read,
    picasso_profile_read_packs,
    picasso_unique_offsets,
    picasso_nccl_unique_id,
    picasso_group_create,
    picasso_group_destroy,
    picasso_group_fwd,
    picasso_group_bwd_update,
    picasso_get_owner_unique,
    picasso_get_send_counts,
    picasso_hot_cache_refresh,
    picasso_group_hot_cache_refresh,
    picasso_get_hot_keys,
    picasso_get_send_list,
    picasso_micro_batch_size,
    picasso_dinterleave_begin,
    picasso_packed_lookup_bwd_accumulate,
    picasso_dinterleave_apply,
    picasso_dinterleave_stats,
    picasso_interleave_capacity,
    picasso_pack_plan_kinterleave,
    picasso_nvls_create,
    picasso_nvls_open,
    picasso_nvls_bind,
    picasso_kernel_dim,
    POOL_SUM, POOL_MEAN, OPT_ADAGRAD, OPT_ADAM_LAZY, IDS_ROWS, IDS_HASH,
)
from .embedding import LoopbackGroup, PackedEmbedding  # noqa: F401
from . import dinterleave  # noqa: F401
