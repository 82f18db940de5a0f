"""One row-sharded step of a (scaled) config on ONE GPU through the loopback group (all W ranks in
this process, peer-memory kernels on plain pointers), between cudaProfilerStart / Stop, for
single-process `ncu --profile-from-start off` launch lists of the owner-side kernels (ncu must not
wrap a multi-rank run).

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/lb.csv python tools/loopback_profile.py --config skew
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="skew")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--rows-div", type=int, default=1)
    ap.add_argument("--batch", type=int, default=None)
    args = ap.parse_args()
    import __graft_entry__

    __graft_entry__.build()
    import paper_2204_04903_b200 as pb
    from datagen import configs as dc
    from datagen import init_pack_tables_torch, make_batch, make_dy

    cfg = dc.get_config(args.config)
    if args.alpha is not None:
        cfg = cfg.replace(alpha=args.alpha)
    cfg = dc.scaled(cfg, batch=args.batch or cfg.batch, rows_div=args.rows_div)
    W = args.world
    bs = [make_batch(cfg, r, 0) for r in range(W)]
    mi = max(b.n_ids for b in bs)
    g = pb.LoopbackGroup(W, cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=cfg.batch, max_ids=mi,
                         table_salt=cfg.table_salt, field_col=cfg.field_col, pool=cfg.pool, id_mode=cfg.id_mode,
                         max_recv=W * mi)
    for r, e in enumerate(g.ranks):
        init_pack_tables_torch(cfg, e.plan["table_to_pack"], e.plan["table_base"], e.n_packs, e.weights, rank=r,
                               world=W)
    ids = [torch.from_numpy(b.ids).cuda() for b in bs]
    offs = [torch.from_numpy(b.offsets).cuda() for b in bs]
    dys = [torch.from_numpy(make_dy(cfg, r, 0, dyadic=False)).cuda() for r in range(W)]

    def step(i):
        g.forward(ids, offs, [cfg.batch] * W)
        g.backward_update(dys, 0.01, i)

    step(1)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    step(2)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    for e in g.ranks:
        e.check()
    print("[loopback_profile] ids per rank", [b.n_ids for b in bs], flush=True)


if __name__ == "__main__":
    main()
