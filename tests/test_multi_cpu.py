"""Host-side logic of the row-sharded path on CPU (-m "not gpu"): two processes over the gloo
backend bootstrap the NCCL id the way bench.py does (rank 0 creates it, broadcast over
torch.distributed), create world = 2 contexts (host only: no device memory is touched before
picasso_bind) and agree on the shard layout: every pack key k lives on rank k mod W at local
row k div W (reading O3), so the local row counts of the ranks tile each pack."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from datagen import configs as dc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2204_04903_b200 as pb

        cfg = dc.wdl()
        obj = [pb.picasso_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        plan = pb.picasso_pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim)
        ctx = pb.picasso_ctx_create(plan, cfg.field_to_table, cfg.table_rows, cfg.table_dim, cfg.table_salt,
                                    cfg.field_col, cfg.out_width, rank, world, 1024, 1024 * cfg.F * 50,
                                    nccl_uid=obj[0])
        rows = [pb.picasso_pack_local_rows(ctx, p) for p in range(plan["n_packs"])]
        ws = pb.picasso_workspace_size(ctx)
        pb.picasso_ctx_destroy(ctx)
        out = [None] * world
        dist.all_gather_object(out, {"rows": rows, "ws": ws, "uid": obj[0]})
        if rank == 0:
            q.put((out, plan["pack_rows"].tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_bootstrap_and_shard_layout():
    import __graft_entry__

    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, pack_rows = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0]["uid"] == out[1]["uid"] and len(out[0]["uid"]) == 128
    for p, R in enumerate(pack_rows):
        assert out[0]["rows"][p] + out[1]["rows"][p] == R  # ceil((R - r) / W) over r tiles the pack
        assert out[0]["rows"][p] - out[1]["rows"][p] in (0, 1)
    assert out[0]["ws"] == out[1]["ws"]


def test_world_argument_validation():
    import paper_2204_04903_b200 as pb

    cfg = dc.toy()
    plan = pb.picasso_pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim)
    for rank, world in ((2, 2), (0, 9), (-1, 2)):
        with pytest.raises(pb.PicassoError):
            pb.picasso_ctx_create(plan, cfg.field_to_table, cfg.table_rows, cfg.table_dim, None, cfg.field_col,
                                  cfg.out_width, rank, world, 16, 100)
    # a loopback rank (no NCCL id) is valid; the single-rank entry points refuse it until a group drives it
    c = pb.picasso_ctx_create(plan, cfg.field_to_table, cfg.table_rows, cfg.table_dim, None, cfg.field_col,
                              cfg.out_width, 1, 4, 16, 100)
    assert pb.picasso_pack_local_rows(c, 0) == int(np.ceil((cfg.table_rows.sum() - 1) / 4))
    pb.picasso_ctx_destroy(c)
