"""Drive the row-sharded step of W ranks in ONE process on one GPU (LoopbackGroup) on a bench
workload, for kernel-level profiling of the W > 1 path with ncu (which must never wrap a
multi-rank command).  Peer traffic is local here, so the NVLink part of the exchange kernels
is not represented; index / partition / pool / segsum kernels are.
  python tools/loopback_run.py [--world 2] [--config criteo] [--steps 3] [--exchange p2p]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--config", default="criteo")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--exchange", default="p2p")
    args = ap.parse_args()
    os.environ["PICASSO_EXCHANGE"] = args.exchange
    import torch

    import __graft_entry__

    __graft_entry__.build()
    import paper_2204_04903_b200 as pb
    from datagen import configs as dc
    from datagen import init_pack_tables_torch, make_batch, make_dy

    cfg = dc.get_config(args.config)
    W, B = args.world, cfg.batch
    bs = [make_batch(cfg, r, 0) for r in range(W)]
    mi = max(b.n_ids for b in bs)
    g = pb.LoopbackGroup(W, cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=B, max_ids=mi,
                         table_salt=cfg.table_salt, field_col=cfg.field_col, pool=cfg.pool, id_mode=cfg.id_mode,
                         max_recv=2 * mi)
    for r, e in enumerate(g.ranks):
        init_pack_tables_torch(cfg, e.plan["table_to_pack"], e.plan["table_base"], e.n_packs, e.weights, rank=r,
                               world=W)
    ids = [torch.from_numpy(b.ids).cuda() for b in bs]
    offs = [torch.from_numpy(b.offsets).cuda() for b in bs]
    dys = [torch.from_numpy(make_dy(cfg, r, 0, dyadic=False)).cuda() for r in range(W)]
    for s in range(args.steps):
        g.forward(ids, offs, [B] * W)
        g.backward_update(dys, 0.01, s + 1)
    torch.cuda.synchronize()
    for e in g.ranks:
        e.check()
    print("ok", W, args.config)


if __name__ == "__main__":
    main()
