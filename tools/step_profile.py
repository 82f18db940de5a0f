"""One eager fwd + bwd step of a bench config between cudaProfilerStart / Stop, for
`ncu --profile-from-start off` launch lists (one step's kernels only, after 2 warm-up steps).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/x.csv python tools/step_profile.py --config wdl
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="wdl")
    ap.add_argument("--time", action="store_true", help="print per-step event time instead of profiling")
    args = ap.parse_args()
    import __graft_entry__

    __graft_entry__.build()
    import paper_2204_04903_b200 as pb
    from datagen import configs as dc
    from datagen import init_pack_tables_torch, make_batch, make_dy

    cfg = dc.get_config(args.config)
    dev = torch.device("cuda", 0)
    b = make_batch(cfg, 0, 0)
    emb = pb.PackedEmbedding(cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=cfg.batch,
                             max_ids=b.n_ids, table_salt=cfg.table_salt, field_col=cfg.field_col, pool=cfg.pool,
                             id_mode=cfg.id_mode, device=dev)
    init_pack_tables_torch(cfg, emb.plan["table_to_pack"], emb.plan["table_base"], emb.n_packs, emb.weights)
    ids, off = torch.from_numpy(b.ids).to(dev), torch.from_numpy(b.offsets).to(dev)
    dy = torch.from_numpy(make_dy(cfg, 0, 0, dyadic=False)).to(dev)
    out = torch.empty(cfg.batch, emb.out_width, device=dev)

    def step(i):
        emb.forward(ids, off, cfg.batch, out)
        emb.backward_update(dy, lr=0.01, step=i)

    for i in range(2):
        step(i + 1)
    torch.cuda.synchronize()
    if args.time:
        ts = []
        for i in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step(i + 3)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"[step_profile] {args.config} ms/step {np.median(ts):.3f} ({', '.join(f'{t:.3f}' for t in ts)})")
    else:
        torch.cuda.cudart().cudaProfilerStart()
        step(3)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    emb.check()


if __name__ == "__main__":
    main()
