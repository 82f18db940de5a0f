"""bench.py — packed embedding fwd + bwd + sparse-Adagrad step on synthetic Zipf batches.

Contract (driver): `python bench.py --gpus N --steps K --warmup W [--impl reference]`; for
N > 1 launched by torchrun (one process per GPU).  Prints ONE JSON line on rank 0.

Workload at N = 1: BASELINE.json configs[1], the Criteo-shaped DLRM embedding layer:
26 one-hot categorical fields, dim 128, batch 16,384 per GPU, 46.875M rows (24 GB fp32 +
24 GB Adagrad state), Zipf(alpha = 0.8) IDs hashed into the tables.  A step = one forward
(hash + Unique + gather/pool) and one backward (transpose + segment-sum + Adagrad update)
over one batch.  Inputs resident in HBM; L2 flushed (256 MiB write) before every timed
step.  Per-phase times come from CUDA events the library records on the launch stream, in a
second pass of K steps after the timed one (inside a CUDA graph the event nodes add gaps).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "packed embedding fwd+bwd samples/sec"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="picasso", choices=["picasso", "reference"])
    ap.add_argument("--config", default="criteo")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--rows-div", type=int, default=1, help="tables at 1/rows_div of their rows (fit one GPU)")
    ap.add_argument("--nbatches", type=int, default=4, help="distinct pre-generated batches, used round robin")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cache-bytes", type=int, default=0,
                    help="HybridHash hot storage per GPU (N > 1, or N = 1 with --cold-tier)")
    ap.add_argument("--cache-warmup", type=int, default=3, help="Alg. 1 warmup_iters")
    ap.add_argument("--cache-flush", type=int, default=10, help="Alg. 1 flush_iters")
    ap.add_argument("--eager", action="store_true", help="N = 1: launch every step eagerly instead of a CUDA graph")
    ap.add_argument("--cold-tier", action="store_true",
                    help="N = 1: HybridHash with a host-DRAM cold tier (tables in pinned host memory, "
                         "--cache-bytes of hot rows in HBM, Alg. 1 with --cache-warmup / --cache-flush); "
                         "prints its own JSON line")
    ap.add_argument("--micro", default=None,
                    help="N = 1: D-Interleaving with this many micro-batches per step, or 'auto' (Eq. 2 "
                         "from --micro-budget-gb); prints its own JSON line")
    ap.add_argument("--micro-budget-gb", type=float, default=16.0,
                    help="device-memory budget (GB) of the batch-proportional buffers for --micro auto")
    ap.add_argument("--kgroups", type=int, default=None,
                    help="K-Interleaving groups (packs per dim) at N > 1 with the peer-memory exchange "
                         "(default 1: measured no gain at C2 with 2 groups, DESIGN.md 7b)")
    return ap.parse_args()


def get_cfg(args):
    from datagen import configs as dc

    cfg = dc.get_config(args.config)
    if args.alpha is not None:
        cfg = cfg.replace(alpha=args.alpha)
    if args.batch is not None:
        cfg = cfg.replace(batch=args.batch)
    if args.rows_div > 1:
        cfg = dc.scaled(cfg, rows_div=args.rows_div)
    return cfg


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock and clock-event (throttle) reasons polled through NVML every ~2 ms during the
    timed region (the same fields as the recipe's nvidia-smi clocks line)."""

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self.stop.set()
        if self.nv:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        nv = self.nv
        names = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({n for _, r in self.rows for n, bit in names.items() if r & bit})
        return {"sm_mhz": float(np.median([sm for sm, _ in self.rows])), "sm_max_mhz": float(self.max),
                "reasons": reasons, "samples": len(self.rows), "source": "nvml, 2 ms poll over the timed region"}


# ------------------------------------------------------------------------------------------
def host_cpu():
    """Cores this process may use and the CPU model (/proc/cpuinfo) of the box."""
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return cores, model


def cpu_oracle_baseline(cfg, seconds, openmp=False, max_steps=50):
    """The oracle (oracle/picasso_oracle.cpp as it stands) on a bounded sample of the same
    workload: whole batches of this config, one rank; forward over every segment
    (oracle_forward_sampled), gradients of every touched row (oracle_row_grads) and the
    Adagrad update (oracle_apply_update).  Table rows the sample touches are materialised
    from the same generator beforehand (not timed).  openmp=True: the -fopenmp build on every
    host core (the same loops split over threads, results bitwise the plain build's)."""
    import oracle
    from datagen import make_batch, make_dy, table_values_np

    oracle.use_openmp(openmp)
    # every host core this process may use (torchrun pins its workers' OMP_NUM_THREADS to 1)
    used = oracle.set_threads(host_cpu()[0]) if openmp else 1
    try:
        m = oracle.OracleModel(cfg.field_to_table, cfg.table_rows, cfg.table_dim, cfg.field_col,
                               id_mode=cfg.id_mode, pool=cfg.pool, table_salt=cfg.table_salt)
        B = cfg.batch
        ld = int(cfg.table_dim.max())
        spent, samples, steps = 0.0, 0, 0
        while steps == 0 or (spent < seconds and steps < max_steps):
            b = make_batch(cfg, 0, 1000 + steps)
            dy = make_dy(cfg, 0, 1000 + steps, dyadic=False)
            ob = oracle.OracleBatch(B, b.ids, b.offsets, dy)
            qf = np.repeat(np.arange(cfg.F, dtype=np.int32), B)
            qs = np.tile(np.arange(B, dtype=np.int32), cfg.F)
            rt, rr = oracle.segment_rows(m, ob, qf, qs)
            key = np.unique(rt.astype(np.int64) * (1 << 40) + rr)
            ut, ur = (key >> 40).astype(np.int32), key & ((1 << 40) - 1)
            vals = np.zeros((len(key), ld), np.float32)
            for t in np.unique(ut):
                sel = ut == t
                D = int(cfg.table_dim[t])
                vals[sel, :D] = table_values_np(cfg.seed, int(t), ur[sel], D)
            acc = np.full_like(vals, 0.1)
            t0 = time.perf_counter()
            oracle.forward_sampled(m, ob, ut, ur, vals, qf, qs)
            G, cnt = oracle.row_grads(m, [ob], ut, ur, ld)
            oracle.apply_update(G, cnt, vals, acc, lr=0.01, D=ld)
            spent += time.perf_counter() - t0
            samples += B
            steps += 1
    finally:
        oracle.use_openmp(False)
    cores, model = host_cpu()
    how = f"OpenMP build on {used} threads ({cores} host cores)" if openmp else "single-threaded"
    return {"value": samples / spent, "unit": UNIT, "cores": used, "kind": "oracle", "cpu_model": model,
            "host_cores": cores,
            "sample": f"{steps} full batch(es) of {cfg.name} (B={B}, {cfg.F} fields): fwd over all segments, "
                      f"grads + Adagrad over all touched rows; {spent:.1f} s, {how} C++ (-O2)"}


def run_reference(args):
    """The reference arm: the oracle (the paper has no code) on every host core, one whole batch
    of the same workload per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = get_cfg(args)
    per = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_oracle_baseline(cfg, seconds=0.0, openmp=True)  # exactly one batch per call
        if i >= args.warmup:
            per.append(cfg.batch / cb["value"])
    tot = float(np.sum(per))
    value = cfg.batch * len(per) / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / len(per),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "global_batch": cfg.batch, "fields": cfg.F,
                       "dims": sorted(set(cfg.table_dim.tolist())), "alpha": cfg.alpha},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb["cores"], "kind": "oracle",
                             "cpu_model": cb["cpu_model"],
                             "sample": f"{len(per)} full batches of {cfg.name}, OpenMP oracle build on "
                                       f"{cb['cores']} threads ({cb['host_cores']} host cores)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def algorithmic_bytes(cfg, B, N, U_by_pack, plan, world=1):
    """Per-kernel algorithmic bytes per step (SURVEY.md §8(d) per-unit figures x
    the units one launch processes): what each kernel must move, index scratch not credited.
    N ids, S = F*B segments, U unique rows (per pack), Adagrad (1 state array)."""
    S = cfg.F * B
    fd = cfg.field_dim.astype(np.int64)
    out_bytes = 4 * B * int(fd.sum())                      # pooled output / dY, [B, sum D]
    rows_bytes = sum(4 * int(plan["pack_dim"][p]) * U_by_pack[p] for p in range(plan["n_packs"]))  # 4*D*U
    U = sum(U_by_pack)
    return {
        # ids + offsets + distinct rows + pooled output
        "pool": 8 * N + 4 * (S + 1) + rows_bytes + out_bytes,
        # dY rows + sorted segment list + row bounds + G rows out
        "segsum": out_bytes + 4 * N + 4 * (U + 1) + rows_bytes,
        # G rows in + row keys + weight and accumulator read + written (W = 1: this rank's uniques)
        "update": rows_bytes + 8 * U + 4 * rows_bytes if world == 1 else None,
        # fused segment-sum + Adagrad (W = 1 default, k_segsum_upd): dY rows + sorted segment list + row
        # bounds + row keys + weight and accumulator read + written — no G row in either direction
        "segsum_update": out_bytes + 4 * N + 4 * (U + 1) + 8 * U + 4 * rows_bytes if world == 1 else None,
        # whole step, fused definition of SURVEY §8(d) (fwd + bwd + Adagrad)
        "step": 8 * N + 4 * (S + 1) + 4 * N + 8 * U + rows_bytes + out_bytes + out_bytes + 4 * N + 4 * rows_bytes,
    }


def run_micro(args):
    """D-Interleaving: the step's batch in micro-batches (Eq. 2 or a fixed
    count), each forwarded + accumulated, one update per step; the whole micro-batched step is
    one CUDA graph.  Reports the step time of the whole batch and the device memory of the
    batch-proportional buffers (ctx workspace + out + dY) against the one-shot step's."""
    import torch

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    import __graft_entry__

    __graft_entry__.build()
    import paper_2204_04903_b200 as pb
    from paper_2204_04903_b200 import dinterleave as di
    from datagen import init_pack_tables_torch, make_batch, make_dy

    cfg = get_cfg(args)
    B = cfg.batch
    batches = [make_batch(cfg, 0, s) for s in range(args.nbatches)]
    max_ids = max(b.n_ids for b in batches)
    kw = dict(pool=cfg.pool, id_mode=cfg.id_mode, table_salt=cfg.table_salt, field_col=cfg.field_col)
    if args.micro == "auto":
        plan = pb.picasso_pack_plan(cfg.field_to_table, cfg.table_rows, cfg.table_dim)
        ctx_kw = dict(plan=plan, field_to_table=cfg.field_to_table, table_rows=cfg.table_rows,
                      table_dim=cfg.table_dim, table_salt=cfg.table_salt, field_col=cfg.field_col,
                      out_width=cfg.out_width, rank=0, world=1, max_batch=B, max_ids=max_ids)
        ws_id = di.workspace_bytes_per_id(ctx_kw)
        ids_ps = max_ids / B  # warm-up measurement: IDs per sample (the largest of the batches)
        bs, n_micro, ops = di.micro_batch_plan(B, cfg.out_width, cfg.F, ids_ps, ws_id, args.micro_budget_gb * 1e9)
    else:
        n_micro, ops = int(args.micro), None
    sl = di.even_slices(B, n_micro)
    mb = max(b1 - b0 for b0, b1 in sl)
    mbs = []  # per batch: per micro-batch (ids, offsets, dY) on the device
    mb_ids = 0
    for k, b in enumerate(batches):
        dy = make_dy(cfg, 0, k, dyadic=False)
        parts = []
        for b0, b1 in sl:
            ids, off = di.slice_batch(b.ids, b.offsets, cfg.F, B, b0, b1)
            mb_ids = max(mb_ids, len(ids))
            parts.append((torch.from_numpy(ids).to(dev), torch.from_numpy(off).to(dev),
                          torch.from_numpy(np.ascontiguousarray(dy[b0:b1])).to(dev), b1 - b0))
        mbs.append(parts)
    lr = 0.01
    stream = torch.cuda.current_stream(dev)
    state = {}

    def step(k, s, stepno):
        emb = state["emb"]
        emb.dinterleave_begin(stream=s)
        for (ids, off, dy, n), o in zip(mbs[k], state["outs"]):
            emb.forward(ids, off, n, o, stream=s)
            emb.backward_accumulate(dy, stream=s)
        emb.dinterleave_apply(lr, step=stepno, stream=s)

    def make(msu, msf):
        e = pb.PackedEmbedding(cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=mb, max_ids=mb_ids,
                               device=dev, max_step_unique=msu, max_step_floats=msf, **kw)
        init_pack_tables_torch(cfg, e.plan["table_to_pack"], e.plan["table_base"], e.n_packs, e.weights)
        state["emb"] = e
        state["outs"] = [torch.empty(n, e.out_width, device=dev) for (_, _, _, n) in mbs[0]]
        return e

    # warm-up measurement of the step accumulator (L419-421): one step per batch with a generous
    # accumulator, then the layer is rebuilt with the measured distinct keys / values (+ 15 %)
    emb = make(max_ids, 0)
    rows = floats = 0
    for k in range(args.nbatches):
        step(k, stream, k + 1)
        r, f = emb.dinterleave_stats()
        rows, floats = max(rows, r), max(floats, f)
    emb.check()
    emb.close()
    del emb, state["emb"]
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    emb = make(int(rows * 1.15) + 64, int(floats * 1.15) + 256)
    for i in range(max(args.warmup, 1)):
        step(i % args.nbatches, stream, i + 1)
    emb.check()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(stream)
    graphs = []
    for k in range(args.nbatches):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            step(k, cap, args.warmup + 1)
        graphs.append(g)
    stream.wait_stream(cap)
    for g in graphs:
        g.replay()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clk = ClockSampler(0)
    with clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            st[i].record(stream)
            graphs[i % args.nbatches].replay()
            en[i].record(stream)
        torch.cuda.synchronize()
    emb.check()
    ms = float(sum(a.elapsed_time(b) for a, b in zip(st, en))) / args.steps
    ws_micro = pb.picasso_workspace_size(emb.ctx)
    io_micro = 2 * 4 * mb * emb.out_width
    # the one-shot step's batch-proportional buffers (not allocated: workspace size only)
    c1 = pb.picasso_ctx_create(emb.plan, cfg.field_to_table, cfg.table_rows, cfg.table_dim, cfg.table_salt,
                               cfg.field_col, emb.out_width, 0, 1, B, max_ids)
    ws_full = pb.picasso_workspace_size(c1)
    pb.picasso_ctx_destroy(c1)
    line = {"metric": METRIC, "value": B / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "global_batch": B, "fields": cfg.F, "rows": int(cfg.table_rows.sum()),
                       "alpha": cfg.alpha, "optimizer": "adagrad", "parallelism": "single",
                       "l2": "flushed (256 MiB write, untimed) before every timed step",
                       "launch": "cuda_graph (one captured micro-batched step per batch)"},
            "dinterleave": {"n_micro": n_micro, "bs_micro": mb, "micro_batch_ids_max": mb_ids,
                            "step_distinct_keys": int(rows), "step_accumulator_values": int(floats),
                            "eq2_ops": ops, "budget_gb": args.micro_budget_gb if args.micro == "auto" else None,
                            "batch_buffers_bytes": {"micro": int(ws_micro + io_micro),
                                                    "one_shot": int(ws_full + 2 * 4 * B * emb.out_width)},
                            "note": "batch-proportional device memory = ctx workspace (incl. the step "
                                    "accumulator in micro mode) + out + dY"},
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def run_coldtier(args):
    """HybridHash with DRAM as Cold-storage: the tables and Adagrad state in
    pinned host memory, --cache-bytes of the hottest rows (FCounter top-k) in HBM.  Alg. 1 schedule:
    FCounter from the first iteration, refresh after the backward of every itr >= warmup with
    itr % flush == 0 (reading O13).  Eager launches (a refresh changes the hot set the kernels are
    launched with); the timed K steps include their refreshes."""
    import torch

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    import __graft_entry__

    __graft_entry__.build()
    import paper_2204_04903_b200 as pb
    from datagen import init_pack_tables_torch, make_batch, make_dy

    cfg = get_cfg(args)
    B = cfg.batch
    batches = [make_batch(cfg, 0, s) for s in range(args.nbatches)]
    max_ids = max(b.n_ids for b in batches)
    t0 = time.time()
    emb = pb.PackedEmbedding(cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=B, max_ids=max_ids,
                             table_salt=cfg.table_salt, field_col=cfg.field_col, pool=cfg.pool, id_mode=cfg.id_mode,
                             device=dev, cold_tier=True, cache_max_bytes=max(args.cache_bytes, 1024))
    init_pack_tables_torch(cfg, emb.plan["table_to_pack"], emb.plan["table_base"], emb.n_packs, emb.weights)
    setup_s = time.time() - t0
    dev_in = [(torch.from_numpy(b.ids).to(dev), torch.from_numpy(b.offsets).to(dev)) for b in batches]
    dys = [torch.from_numpy(make_dy(cfg, 0, s, dyadic=False)).to(dev) for s in range(args.nbatches)]
    out = torch.empty(B, emb.out_width, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    stats = {}
    refresh_ms = []

    def step(itr):
        ids, off = dev_in[itr % args.nbatches]
        emb.forward(ids, off, B, out, stream=stream)
        emb.backward_update(dys[itr % args.nbatches], 0.01, step=itr + 1, stream=stream)
        if args.cache_bytes > 0 and itr >= args.cache_warmup and itr % args.cache_flush == 0:
            st = emb.hot_cache_refresh(args.cache_bytes, stream=stream)
            stats.update(st)
            refresh_ms.append(st["refresh_ms"])

    itr = 0
    warm = max(args.warmup, args.cache_warmup + args.cache_flush + 1) if args.cache_bytes else args.warmup
    for _ in range(warm):
        step(itr)
        itr += 1
    emb.check()
    torch.cuda.synchronize()
    refresh_ms.clear()
    st_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    en_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    hot_hits = []
    clk = ClockSampler(0)
    with clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            st_ev[i].record(stream)
            step(itr)
            itr += 1
            en_ev[i].record(stream)
        torch.cuda.synchronize()
    emb.check()
    ms = float(sum(a.elapsed_time(b) for a, b in zip(st_ev, en_ev))) / args.steps
    U = int(np.diff(np.array(emb.unique_offsets_host(), np.int64)).sum())
    nst = 1
    row_b = [4 * int(d) for d in emb.plan["pack_dim"]]
    hit = stats.get("hit_ratio_unique", 0.0)
    line = {"metric": METRIC, "value": B / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": warm, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "global_batch": B, "fields": cfg.F, "rows": int(cfg.table_rows.sum()),
                       "alpha": cfg.alpha, "optimizer": "adagrad", "parallelism": "single",
                       "tables": "pinned host memory (Cold-storage), device-mapped",
                       "l2": "flushed (256 MiB write, untimed) before every timed step", "launch": "eager"},
            "cold_tier": {"cache_bytes": args.cache_bytes, "warmup_iters": args.cache_warmup,
                          "flush_iters": args.cache_flush, "hot_rows": stats.get("k", 0),
                          "hit_ratio_unique": hit, "unique_per_step": U,
                          "refresh_ms_mean": float(np.mean(refresh_ms)) if refresh_ms else None,
                          "refreshes_in_timed_steps": len(refresh_ms),
                          "pcie_bytes_per_step_est": int(U * (1 - hit) * row_b[0] * (3 + 2 * nst))
                          if len(row_b) == 1 else None,
                          "note": "PCIe estimate: per cold unique row one row read (stage) + w and state read "
                                  "+ written (update)",
                          "setup_s": setup_s},
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.cold_tier:
        run_coldtier(args)
        return
    if args.micro:
        run_micro(args)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    import __graft_entry__

    __graft_entry__.build()
    import paper_2204_04903_b200 as pb
    from datagen import init_pack_tables_torch, make_batch, make_dy

    cfg = get_cfg(args)
    B = cfg.batch
    batches = [make_batch(cfg, rank, s) for s in range(args.nbatches)]
    max_ids = max(b.n_ids for b in batches)
    # every rank processes its own B samples (weak scaling, data parallel over samples); at
    # world > 1 the tables are row-sharded over the ranks (key mod W); keys / rows / gradients are
    # exchanged over NVLink peer memory (PICASSO_EXCHANGE=p2p, default) or NCCL AllToAllv
    uid = None
    if world > 1:
        obj = [pb.picasso_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    kgroups = args.kgroups if args.kgroups is not None else 1
    emb = pb.PackedEmbedding(cfg.field_to_table, cfg.table_rows, cfg.table_dim, max_batch=B, max_ids=max_ids,
                             split=kgroups if kgroups >= 2 else False,
                             table_salt=cfg.table_salt, field_col=cfg.field_col, pool=cfg.pool, id_mode=cfg.id_mode,
                             device=dev, rank=rank, world=world, nccl_uid=uid, max_recv=max_ids,
                             cache_max_bytes=args.cache_bytes if world > 1 else 0)
    init_pack_tables_torch(cfg, emb.plan["table_to_pack"], emb.plan["table_base"], emb.n_packs, emb.weights,
                           rank=rank, world=world)
    dev_in = [(torch.from_numpy(b.ids).to(dev), torch.from_numpy(b.offsets).to(dev)) for b in batches]
    dys_host = [torch.from_numpy(make_dy(cfg, rank, s, dyadic=False)).pin_memory() for s in range(args.nbatches)]
    dys = [d.to(dev) for d in dys_host]
    out = torch.empty(B, emb.out_width, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lr = 0.01
    stream = torch.cuda.current_stream(dev)

    cache_stats = {}

    def step(i, s):
        ids, off = dev_in[i % args.nbatches]
        emb.forward(ids, off, B, out, stream=s)
        emb.backward_update(dys[i % args.nbatches], lr, step=i + 1, stream=s)
        itr = i + 1  # Alg. 1 schedule (reading O13): refresh after bwd when itr >= warmup, itr % flush == 0
        # (--cache-flush 0: one refresh, at itr == warmup — the steady state of a hot set, no refresh cost)
        due = (itr % args.cache_flush == 0) if args.cache_flush > 0 else itr == args.cache_warmup
        if world > 1 and args.cache_bytes > 0 and itr >= args.cache_warmup and due:
            cache_stats.update(emb.hot_cache_refresh(args.cache_bytes, stream=s))

    if world > 1 and args.cache_bytes > 0:  # the first refresh and a hot step happen before timing
        args.warmup = max(args.warmup, max(args.cache_flush, args.cache_warmup) + 1)
    hot_refresh_off = world > 1 and args.cache_bytes > 0 and args.cache_flush == 0
    for i in range(args.warmup):
        step(i, stream)
    emb.check()
    torch.cuda.synchronize()
    lf, lb = emb.launch_count()

    # ---------------- timed region: K steps, L2 flushed before each (flush not timed)
    # The whole step is one CUDA graph when it has no host synchronisation inside: world == 1,
    # and world > 1 with the peer-memory exchange (device-side sizes) and no HybridHash refresh
    # schedule.  The NCCL exchange needs one host sync per step (host-side sizes) and runs eagerly.
    # The per-phase CUDA events (roofline, phase split) are NOT in the timed steps: as graph nodes
    # they cost ~26 us per step of inter-node gaps at C2 (0.320 vs 0.293 ms).  A second pass of K
    # steps records them (same graph without vs with the event nodes; eager: profiling on), and
    # its step time is reported beside the timed one.
    # (a hot set that no longer changes — --cache-flush 0 — keeps the step capturable)
    use_graph = not args.eager and (world == 1 or (emb.exchange == "p2p" and (not args.cache_bytes or hot_refresh_off)))
    graphs, graphs_t = {}, []
    if use_graph:
        # timed pass: one captured step per pre-generated batch (--nbatches), replayed round robin;
        # profiled pass: batch 0's step with the phase-event nodes
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        for k in range(args.nbatches):
            ids_k, off_k = dev_in[k]
            pb.picasso_profile_enable(emb.ctx, 0)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                emb.forward(ids_k, off_k, B, out, stream=cap)
                emb.backward_update(dys[k], lr, step=args.warmup + 1, stream=cap)
            graphs_t.append(g)
        ids0, off0 = dev_in[0]
        pb.picasso_profile_enable(emb.ctx, 2)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            emb.forward(ids0, off0, B, out, stream=cap)
            emb.backward_update(dys[0], lr, step=args.warmup + 1, stream=cap)
        graphs[2] = g
        stream.wait_stream(cap)  # profiling stays in graph mode (2): phase events read after replays
        for _ in range(2):  # warm replays
            for gt in graphs_t:
                gt.replay()
            graphs[2].replay()
        torch.cuda.synchronize()
        pb.picasso_profile_read(emb.ctx)
    next_i = [args.warmup]

    pack_ms = [[0.0] * emb.n_packs, [0.0] * emb.n_packs]  # per pack: pool ms, backward ms (profiled pass)

    def run_pass(profiled, clk=None):
        """K steps, L2 flushed before each; returns (ms per step, phase ms summed, #calls)."""
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if not use_graph:
            pb.picasso_profile_enable(emb.ctx, bool(profiled))
            pb.picasso_profile_read(emb.ctx)
        phase, calls = {}, 0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if clk is not None:
            clk.__enter__()
        if world > 1:
            # align the ranks' streams on the device: the host barrier above returns at different
            # times per rank, and a rank that starts early would absorb the skew in its first step
            dist.all_reduce(align)
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            starts[i].record(stream)
            if use_graph:
                (graphs[2] if profiled else graphs_t[i % len(graphs_t)]).replay()
            else:
                step(next_i[0], stream)
                next_i[0] += 1
            ends[i].record(stream)
            if use_graph and profiled:  # this replay's phase times (the sync is outside the start/end events)
                pp, pw = pb.picasso_profile_read_packs(emb.ctx, emb.n_packs)
                pack_ms[0] = [a + b for a, b in zip(pack_ms[0], pp)]
                pack_ms[1] = [a + b for a, b in zip(pack_ms[1], pw)]
                ph, _ = pb.picasso_profile_read(emb.ctx)
                phase = {k: phase.get(k, 0.0) + v for k, v in ph.items()}
                calls += 1
        torch.cuda.synchronize()
        if clk is not None:
            clk.__exit__(None, None, None)
        if world > 1:
            dist.barrier()
        if not use_graph and profiled:
            pack_ms[0], pack_ms[1] = pb.picasso_profile_read_packs(emb.ctx, emb.n_packs)
            phase, calls = pb.picasso_profile_read(emb.ctx)
        if profiled:
            pb.picasso_profile_enable(emb.ctx, False)
        return float(sum(a.elapsed_time(b) for a, b in zip(starts, ends))) / args.steps, phase, calls

    align = torch.zeros(1, device=dev)
    clk = ClockSampler(local)
    ms, _, _ = run_pass(False, clk)
    ms_prof, phase_ms, ncalls = run_pass(True)
    emb.check()
    print(f"[bench] rank {rank} ms_per_step {ms:.4f} (with phase events {ms_prof:.4f})", file=sys.stderr)
    t = torch.tensor([ms], device=dev)
    ms_ranks = [ms]
    if world > 1:
        allms = [None] * world
        dist.all_gather_object(allms, ms)
        ms_ranks = allms
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    tp_ = torch.tensor([ms_prof], device=dev)
    if world > 1:
        dist.all_reduce(tp_, op=dist.ReduceOp.MAX)
    ms_prof_max = float(tp_.item())

    # unique counts of the last timed step (for algorithmic bytes)
    U_pref = np.array(emb.unique_offsets_host(), np.int64)
    U_by_pack = [int(x) for x in np.diff(U_pref)]
    last_b = batches[0 if use_graph else (next_i[0] - 1) % args.nbatches]
    alg = algorithmic_bytes(cfg, B, last_b.n_ids, U_by_pack, emb.plan, world)
    alg = {k: v for k, v in alg.items() if v is not None}
    # the gather (pool) GB/s per pack dim — algorithmic bytes of pack p's pool (its IDs,
    # offsets, distinct rows, pooled output) over its own CUDA-event time
    gather_by_pack = []
    f2p = np.asarray(emb.plan["field_to_pack"])
    seg_len = np.diff(last_b.offsets.astype(np.int64)).reshape(cfg.F, B)
    for p in range(emb.n_packs):
        fields = np.nonzero(f2p == p)[0]
        Dp = int(emb.plan["pack_dim"][p])
        Np, Sp = int(seg_len[fields].sum()), int(len(fields) * B)
        bytes_p = 8 * Np + 4 * (Sp + 1) + 4 * Dp * U_by_pack[p] + 4 * B * int(cfg.field_dim[fields].sum())
        t_ms = pack_ms[0][p] / max(ncalls, 1)
        gather_by_pack.append({"pack": p, "dim": int(emb.plan["pack_dim"][p]), "fields": int(len(fields)),
                               "pool_ms": t_ms, "alg_bytes": bytes_p,
                               "gbs": bytes_p / (t_ms * 1e-3) / 1e9 if t_ms > 0 else None,
                               "backward_ms": pack_ms[1][p] / max(ncalls, 1) if world == 1 else None})
    per_phase = {k: v / max(ncalls, 1) for k, v in phase_ms.items()}
    per_phase = {k: v for k, v in per_phase.items() if v > 0}
    # The dominant kernel = the longest row kernel on the step's serial path.  At world == 1 the
    # library runs the pool beside the sort-based index chain (runtime.cu fwd_sorted; with the
    # hash index: beside its Unique / transpose chain below 4M IDs): its event time then spans the
    # overlap and it is off the serial path, so it is reported separately ("pool_concurrent") and
    # the roofline object takes the longest of the kernels that run alone.
    env = os.environ.get
    sort_idx = env("PICASSO_INDEX", "sort") != "hash"
    early = world == 1 and not args.eager and (
        env("PICASSO_SORT_OVERLAP", "1") != "0" if sort_idx
        else last_b.n_ids < (1 << 22) and env("PICASSO_EARLY_POOL", "1") != "0")
    fused = world == 1 and "segsum" in per_phase and "update" not in per_phase  # k_segsum_upd: one kernel
    if fused:
        per_phase["segsum_update"] = per_phase.pop("segsum")
    cand = [k for k in ("pool", "segsum", "update", "segsum_update") if k in per_phase and k in alg
            and not (early and k == "pool")]
    dom = max(cand, key=lambda k: per_phase[k])
    peak = None
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak_src = "fallback 6650 GB/s (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        peak = float(json.load(open(peaks_path))["hbm_gbs"])
        peak_src = "MEASURED_PEAKS.json hbm_gbs"
    else:
        peak = 6650.0
    achieved = alg[dom] / (per_phase[dom] * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(cfg.name, {}).get(dom)
    kernel_name = {"pool": "k_pool_pipe (+ k_seg_of)", "segsum": "k_segsum_pipe (+ k_segsum_fix)",
                   "update": "k_update_rows", "segsum_update": "k_segsum_upd (+ k_segsum_fix)"}[dom]
    dom_bytes, dom_ms = alg[dom], per_phase[dom]
    # Several packs (world == 1): the phases mix kernels of different packs, so the dominant kernel
    # is taken per pack — each pack's pool and backward with its own algorithmic bytes (SURVEY
    # §8(d) per-unit figures x that pack's IDs / rows / segments) over its own event time.
    if world == 1 and emb.n_packs > 1 and ncalls > 0:
        fused_ok = env("PICASSO_BWD", "") != "split" and all(
            int(d) in (64, 128) for d in emb.plan["pack_dim"] if int(d) >= 64)
        items = []
        for e in gather_by_pack:
            D, p = e["dim"], e["pack"]
            fields = np.nonzero(f2p == p)[0]
            Np, Up = int(seg_len[fields].sum()), U_by_pack[p]
            out_p, rows_p = 4 * B * int(cfg.field_dim[fields].sum()), 4 * D * Up
            if fused_ok and D in (64, 128):
                e["backward_alg_bytes"] = out_p + 4 * Np + 4 * (Up + 1) + 8 * Up + 4 * rows_p
                blabel = f"k_segsum_upd<{D}> (+ k_segsum_fix), pack {p}"
            else:  # split: segment-sum writes G, the update reads it back
                e["backward_alg_bytes"] = (out_p + 4 * Np + 4 * (Up + 1) + rows_p) + (rows_p + 8 * Up + 4 * rows_p)
                blabel = f"k_segsum<{D}> + k_update_rows<{D}> (+ long rows), pack {p}"
            bms = e["backward_ms"] or 0.0
            e["backward_gbs"] = e["backward_alg_bytes"] / (bms * 1e-3) / 1e9 if bms > 0 else None
            items.append((blabel, bms, e["backward_alg_bytes"]))
            if not early:
                items.append((f"{'k_pool_pipe' if D >= 64 else 'k_pool_flat'}<{D}>, pack {p}", e["pool_ms"],
                              e["alg_bytes"]))
        kernel_name, dom_ms, dom_bytes = max(items, key=lambda x: x[1])
        achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
        traffic = None

    # ---------------- NVLink traffic of the exchange (W > 1): bytes this rank pushed per step
    nvlink = None
    if world > 1:
        sent = emb.send_counts()  # keys this rank requested from each owner, last step
        allsent = [None] * world
        dist.all_gather_object(allsent, sent)
        dims = sorted(set(int(d) for d in emb.plan["pack_dim"]))
        row_b = 4 * dims[0] if len(dims) == 1 else None  # bytes per row (single-dim workloads)
        if row_b:
            rows_out = sum(allsent[q][rank] for q in range(world) if q != rank) * row_b  # owner -> requesters
            g_out = sum(sent[q] for q in range(world) if q != rank) * row_b              # requester -> owners
            tg = per_phase.get("owner_gather", 0.0) * 1e-3
            ts = per_phase.get("segsum", 0.0) * 1e-3
            nvlink = {"rows_push_bytes": int(rows_out), "rows_push_gbs": rows_out / tg / 1e9 if tg else None,
                      "g_push_bytes": int(g_out), "g_push_gbs": g_out / ts / 1e9 if ts else None,
                      "peak_gbs_per_direction": 900.0,
                      "note": "rank 0, last step; GB/s over the phase that issues the peer stores "
                              "(owner gather / segment-sum), so a lower bound on link use"}

    # ---------------- end-to-end through the public API with host buffers
    host_ids = [torch.from_numpy(b.ids).pin_memory() for b in batches]
    host_off = [torch.from_numpy(b.offsets).pin_memory() for b in batches]
    ids_buf = torch.empty(max_ids, dtype=torch.int64, device=dev)
    off_buf = torch.empty(cfg.F * B + 1, dtype=torch.int32, device=dev)
    dy_buf = torch.empty_like(dys[0])
    u_host = torch.empty(emb.n_packs + 1, dtype=torch.int32).pin_memory()
    e_st = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e_en = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    h2d = d2h = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        k = (args.warmup + i) % args.nbatches
        flush.fill_(i & 0xFF)
        e_st[i].record(stream)
        n = host_ids[k].numel()
        ids_buf[:n].copy_(host_ids[k], non_blocking=True)
        off_buf.copy_(host_off[k], non_blocking=True)
        dy_buf.copy_(dys_host[k], non_blocking=True)
        emb.forward(ids_buf[:n], off_buf, B, out, stream=stream)
        emb.backward_update(dy_buf, lr, step=10_000 + i, stream=stream)
        emb.unique_offsets(u_host, stream=stream)
        e_en[i].record(stream)
        h2d = 8 * n + 4 * off_buf.numel() + 4 * dy_buf.numel()
        d2h = 4 * u_host.numel()
    torch.cuda.synchronize()
    e2e_ms = float(sum(s.elapsed_time(e) for s, e in zip(e_st, e_en))) / args.steps
    t = torch.tensor([e2e_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # all host cores (the OpenMP build), and the plain single-threaded oracle beside it
        cpu = cpu_oracle_baseline(cfg, args.cpu_seconds / 2, openmp=True)
        one = cpu_oracle_baseline(cfg, args.cpu_seconds / 2, openmp=False)
        cpu["single_thread"] = {"value": one["value"], "cores": 1, "sample": one["sample"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": world * B / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "global_batch": world * B, "batch_per_gpu": B, "fields": cfg.F,
                       "dims": sorted(set(cfg.table_dim.tolist())), "rows": int(cfg.table_rows.sum()),
                       "alpha": cfg.alpha, "optimizer": "adagrad", "pool": "sum",
                       "parallelism": f"dp{world}+rowshard{world}" if world > 1 else "single",
                       "exchange": emb.exchange if world > 1 else None,
                       "packs": emb.n_packs, "k_interleave_groups": kgroups if world > 1 else None,
                       "l2": "flushed (256 MiB write, untimed) before every timed step",
                       "launch": (f"cuda_graph (one captured step per batch, {args.nbatches} distinct batches "
                                  "replayed round robin)") if use_graph else "eager",
                       "nbatches": args.nbatches,
                       "index": ("sort" if sort_idx else "hash") if world == 1 else (
                           ("sort (row-sharded, run order)" if emb.exchange == "p2p" else "sort (row-sharded)") if sort_idx and last_b.n_ids >= int(
                               env("PICASSO_SORT_MIN_IDS_W", str(1 << 20))) else "hash (row-sharded)"),
                       "ids_per_step": int(last_b.n_ids), "unique_per_step": int(sum(U_by_pack))},
            "e2e": {"value": world * B / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "note": "H2D of ids+offsets+dY from pinned host memory, D2H of the per-pack unique counts"},
            "gpu_launches": int((lf + lb) * args.steps),
            "roofline": {"bound": "hbm", "kernel": kernel_name,
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "algorithmic_bytes_per_launch": dom_bytes, "ms_per_launch": dom_ms,
                         "peak_source": peak_src},
            "gather_by_pack": gather_by_pack,
            "pool_concurrent": ({"achieved": alg["pool"] / (per_phase["pool"] * 1e-3) / 1e9, "unit": "GB/s",
                                 "frac_of_peak": alg["pool"] / (per_phase["pool"] * 1e-3) / 1e9 / peak,
                                 "sms": (f"148 - {env('PICASSO_SORT_RESERVE', '52')} reserved for the sort-based index"
                                         if sort_idx else f"148 - {env('PICASSO_POOL_RESERVE', '74')} reserved for "
                                         "the Unique / transpose chain"),
                                 "note": "k_pool_pipe runs beside the index chain (off the serial path); its "
                                         "event time includes the overlap"}
                                if early and "pool" in per_phase else None),
            "ms_per_step_by_rank": ms_ranks,
            "phases_ms": per_phase,
            "phases_note": "per-phase CUDA events recorded in a second pass of K steps (as graph nodes they "
                           "add inter-node gaps), whose step time is ms_per_step_with_phase_events",
            "ms_per_step_with_phase_events": ms_prof_max,
            "nvlink": nvlink,
            "cache": ({"bytes_per_gpu": args.cache_bytes, "warmup_iters": args.cache_warmup,
                       "flush_iters": args.cache_flush, **cache_stats} if args.cache_bytes and world > 1 else None),
            "outside_phases_ms": ms_prof - sum(per_phase.values()),  # exchanges + host sync (W > 1), launch gaps
            "step_algorithmic_bytes": alg["step"],
            "step_roofline_frac": alg["step"] / (ms_max * 1e-3) / 1e9 / peak,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
