"""One rank of the NCCL row-sharded parity check (launched by tests/test_nccl_gpu.py under
torchrun, one process per GPU).  Every rank regenerates all ranks' seeded batches, runs the
oracle on the global batch itself, and checks its own outputs and table shard."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # PICASSO_XPROC_SAMEDEV=1: every rank on cuda:0, no NCCL communicator (NCCL refuses two ranks
    # on one device): the peer-memory exchange between processes — IPC windows opened by another
    # process, system-scope device barriers — is then testable on a one-GPU box
    samedev = os.environ.get("PICASSO_XPROC_SAMEDEV") == "1"
    local = 0 if samedev else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if samedev:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import oracle
    import paper_2204_04903_b200 as pb
    from datagen import configs as dc
    from datagen import init_pack_tables_torch, make_batch, make_dy
    from harness import assert_close, oracle_model, oracle_tables
    from test_multi_gpu import shard_expected

    name = sys.argv[1] if len(sys.argv) > 1 else "toy"
    cache = name.endswith("_cache")  # HybridHash on: refresh after step 1 (warm-up 1, flush 1)
    graph = name.endswith("_graph")  # one captured step (fixed batch) replayed 3 times
    base = name[:-6] if (cache or graph) else name
    if base == "toy":
        cfg = dc.toy(alpha=1.2)
    elif base in ("criteo", "criteok2"):  # D = 128: pipelined kernels, rows spanning tiles, P2P pushes
        cfg = dc.scaled(dc.criteo(), batch=2048, rows_div=20000)
    elif base == "uneven":  # per-rank batch sizes differ; the last rank has an empty batch
        cfg = dc.scaled(dc.wdl(), batch=32, rows_div=2000)
    else:
        cfg = dc.scaled(dc.wdl(), batch=32, rows_div=2000)
    kplan = None
    if base == "wdlk":  # K-Interleaving plan (Eq. 3): groups of several packs + preset-excluded packs first
        ex = np.zeros(cfg.T, np.uint8)
        ex[::9] = 1
        vol = float((cfg.table_dim.astype(np.float64) * np.bincount(cfg.field_to_table, minlength=cfg.T)).sum())
        kplan = pb.picasso_pack_plan_kinterleave(cfg.field_to_table, cfg.table_rows, cfg.table_dim, vol / 4, ex)
        assert kplan["n_groups"] >= 3 and (kplan["pack_group"] == -1).sum() >= 2
        assert np.bincount(kplan["pack_group"][kplan["pack_group"] >= 0]).max() >= 2  # a group of >= 2 packs
    bsz = [cfg.batch] * world
    if base == "uneven":
        bsz = [max(cfg.batch - 11 * r, 1) for r in range(world)]
        bsz[-1] = 0
    cfgs = [cfg.replace(batch=b) for b in bsz]
    obj = [pb.picasso_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    all_gather = None
    if samedev:
        assert not cache, "HybridHash needs the NCCL AllReduce"
        obj = [None]

        def all_gather(x):
            out = [None] * world
            dist.all_gather_object(out, x)
            return out
    mi = cfg.batch * cfg.F * 60
    e = pb.PackedEmbedding(cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=max(cfg.batch, 1), max_ids=mi,
                           table_salt=cfg.table_salt, field_col=cfg.field_col, pool=cfg.pool, id_mode=cfg.id_mode,
                           rank=rank, world=world, nccl_uid=obj[0], max_recv=world * mi,
                           device=torch.device("cuda", local), cache_max_bytes=(1 << 20) if cache else 0,
                           split=2 if base == "criteok2" else False,  # k2: two K-Interleaving groups
                           all_gather=all_gather, plan=kplan)
    init_pack_tables_torch(cfg, e.plan["table_to_pack"], e.plan["table_base"], e.n_packs, e.weights, rank=rank,
                           world=world)
    m, tabs = oracle_model(cfg), oracle_tables(cfg)
    acc = [np.full_like(t, 0.1) for t in tabs]
    report = {"rank": rank, "world": world, "ok": False, "nvls": bool(getattr(e, "nvls", False))}
    if cache and e.exchange == "p2p" and os.environ.get("PICASSO_NVLS", "1") != "0":
        # the hot-row gradients must go through the NVLS multicast reduce (B200 NVSwitch), not NCCL
        assert e.nvls, "NVLS multicast setup failed on a multicast-capable box"

    gr = None
    for step in (1, 2, 3):
        bstep = 1 if graph else step
        bs = [make_batch(cfgs[r], r, bstep) for r in range(world)]
        dys = [make_dy(cfgs[r], r, bstep) for r in range(world)]
        obs = [oracle.OracleBatch(cfgs[r].batch, b.ids, b.offsets, dy) for r, (b, dy) in enumerate(zip(bs, dys))]
        ref = oracle.forward(m, obs[rank], tabs, cfg.out_width)
        if graph:  # static buffers, captured once; every replay is a full row-sharded step
            if gr is None:
                ids_s = torch.from_numpy(bs[rank].ids).cuda()
                off_s = torch.from_numpy(bs[rank].offsets).cuda()
                dy_s = torch.from_numpy(dys[rank]).cuda()
                out = torch.empty(bsz[rank], e.out_width, device="cuda")
                e.forward(ids_s, off_s, bsz[rank], out)  # warm-up outside the capture (step 1 itself)
                e.backward_update(dy_s, lr=0.05, step=1)
                torch.cuda.synchronize()
                gr = torch.cuda.CUDAGraph()
                cap = torch.cuda.Stream()
                with torch.cuda.graph(gr, stream=cap):
                    e.forward(ids_s, off_s, bsz[rank], out, stream=cap)
                    e.backward_update(dy_s, lr=0.05, step=1, stream=cap)
            else:
                gr.replay()
            torch.cuda.synchronize()
        else:
            out = e.forward(torch.from_numpy(bs[rank].ids).cuda(), torch.from_numpy(bs[rank].offsets).cuda(),
                            bsz[rank])
        if not graph or step == 1:
            assert np.array_equal(out.cpu().numpy(), ref), f"forward step {step}"
        if not graph:
            e.backward_update(torch.from_numpy(dys[rank]).cuda(), lr=0.05, step=step)
        e.check()
        oracle.backward_update(m, obs, tabs, acc, lr=0.05, step=1 if graph else step)
        if cache:  # the shards are authoritative only after a write-back: refresh every step
            stats = e.hot_cache_refresh(8 * 1024 if step < 3 else 0)
            report[f"stats{step}"] = stats
            if step == 2:
                assert stats["hot_uniques"] > 0 and stats["k"] > 0, stats
        for p, exp in enumerate(shard_expected(e, cfg, tabs, "w", world, rank)):
            got = e.weights[p][:len(exp)].cpu().numpy()
            assert np.array_equal(got, exp), f"weights p{p} step {step} (dyadic dY: exact)"
        for p, exp in enumerate(shard_expected(e, cfg, acc, "s1", world, rank)):
            assert_close(e.state1[p][:len(exp)].cpu().numpy(), exp, what=f"state p{p}")
    report["ok"] = True
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    tag = "xproc" if samedev else "nccl"
    with open(os.path.join(ROOT, "gpurun_out", f"{tag}_{name}_rank{rank}.json"), "w") as f:
        json.dump(report, f)
    e.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
