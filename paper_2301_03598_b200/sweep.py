"""Geometry sweep on B200: BASELINE configs 3 (quantisation-limited shapes) and
5 (the paper's 32,824-shape log-sampled corpus), Stream-K vs data-parallel.

    python -m paper_2301_03598_b200.sweep --shapes config3 --out sweep.csv
    python -m paper_2301_03598_b200.sweep --shapes corpus --count 2000 --out sweep.csv
    torchrun --nproc-per-node N -m paper_2301_03598_b200.sweep --shapes corpus ...

Mirrors run_sweep (core/src/sweep.cpp:75-112): shapes in corpus order
(sk_corpus == sweep.cpp:21-28,79-86), one CSV row per (shape, strategy) under a
versioned header, deterministic except the measured columns.  The simulator
columns (utilization, makespan) are replaced by measured device time.

Each (shape, strategy) is timed as a CUDA graph of R launches cycling over R
copies of the operands (R chosen so the copies exceed L2 where memory allows),
best of 3 replays, CUDA events on the capture stream.

Multi-GPU: shape i runs on rank i % world (one problem per GPU, no
collective on the data path); rank 0 merges the per-rank CSV parts in input
order after a barrier.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

import paper_2301_03598_b200 as sk

SCHEMA = "# schema=sk_b200/2"  # /2: + gbps (algorithmic A + B + C bytes / time)
COLUMNS = ["m", "n", "k", "tiles_m", "tiles_n", "t", "iters_per_tile", "strategy", "param", "g",
           "schedule", "variant", "dtype",
           "copies", "l2_cold", "time_us", "tflops", "gbps"]
L2_BYTES = 126 * 1024 * 1024

CONFIG3 = [
    (1024, 1024, 32768), (1280, 3840, 4096), (1280, 3840, 8192), (1024, 4864, 4096),
    (2560, 3840, 4096), (1024, 1024, 8192), (512, 512, 65536), (3072, 3072, 3072),
    (2304, 2304, 8192), (1280, 7680, 4096), (4096, 4096, 4096), (8192, 8192, 8192),
]
# Bandwidth-bound skinny shapes (128 x 8192 x 8192 has ~122
# FLOP/B, below the B200 ridge of ~250): reported in HBM GB/s as well.
SKINNY = [
    (128, 8192, 8192), (256, 8192, 8192), (128, 16384, 8192), (8192, 128, 8192),
    (64, 8192, 16384), (128, 4096, 16384), (512, 8192, 4096), (256, 16384, 2048),
]
# BASELINE config 4: FP64 squares 1024..8192 with the paper's 64x64x16 tile,
# plus shapes whose 64x64 tile count sits just above a multiple of 296 CTAs.
CONFIG4 = [(s, s, s) for s in (1024, 1536, 2048, 3072, 4096, 6144, 8192)] + [
    (1216, 1024, 8192), (1088, 1152, 4096), (512, 512, 32768), (2432, 2048, 2048),
]


def strategies_for(problem, blk, p, names, params=None):
    """Strategy tokens: data_parallel, stream_k (g = p), stream_k:<g>,
    stream_k:auto (model-selected g, cost model in csrc/costmodel.cpp),
    stream_k:cal (calibration set: g in {p, p/2, p/4, p/8, p/16}), two_tile_sk_dp,
    dp_one_tile_sk, fixed_split."""
    out = []
    for name in names:
        if name == "data_parallel":
            out.append(sk.data_parallel(problem, blk))
        elif name == "stream_k":
            out.append(sk.stream_k(problem, blk, p))
        elif name == "stream_k:auto":
            a = sk.auto_stream_k(problem, blk, p, params)
            a.label = "stream_k:auto"
            out.append(a)
        elif name == "stream_k:cal":
            for g in sorted({max(1, p >> i) for i in range(5)}, reverse=True):
                a = sk.stream_k(problem, blk, g)
                a.label = f"stream_k:{g}"
                out.append(a)
        elif name.startswith("stream_k:"):
            a = sk.stream_k(problem, blk, int(name.split(":")[1]))
            a.label = name
            out.append(a)
        elif name == "two_tile_sk_dp":
            out.append(sk.hybrid(problem, blk, p, sk.HybridVariant.TwoTileSkDp))
        elif name == "dp_one_tile_sk":
            out.append(sk.hybrid(problem, blk, p, sk.HybridVariant.DpOneTileSk))
        elif name == "fixed_split":
            out.append(sk.fixed_split(problem, blk, 2))
        else:
            raise ValueError(name)
    return out


class ShapeTimer:
    """Pitched operand copies for one shape + graph-timed launches."""

    def __init__(self, torch, m, n, k, tdt, max_copies=16, mem_budget=4 << 30):
        self.torch = torch
        es = torch.tensor([], dtype=tdt).element_size()
        cdt = torch.float64 if tdt == torch.float64 else torch.float32
        al = 16 // es  # 16-byte rows for TMA
        lda, ldb, ldc = -(-k // al) * al, -(-n // al) * al, -(-n // 2) * 2 if es == 8 else -(-n // 4) * 4
        foot = es * (m * lda + k * ldb)
        self.copies = int(max(1, min(max_copies, math.ceil(2 * L2_BYTES / foot),
                                     mem_budget // max(foot, 1))))
        self.cold = self.copies * foot > L2_BYTES
        g = torch.Generator(device="cuda").manual_seed(m * 131 + n * 7 + k)
        self.A = [torch.empty(m, lda, device="cuda", dtype=tdt)[:, :k] for _ in range(self.copies)]
        self.B = [torch.empty(k, ldb, device="cuda", dtype=tdt)[:, :n] for _ in range(self.copies)]
        for t in self.A + self.B:
            t.copy_(torch.rand(t.shape, device="cuda", generator=g) * 2 - 1)
        self.C = torch.empty(m, ldc, device="cuda", dtype=cdt)[:, :n]

    def time_us(self, gemm, reps=3):
        torch = self.torch
        for i in range(self.copies):  # warm-up + lazy attribute setup outside capture
            gemm.run(self.A[i], self.B[i], self.C)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                for i in range(self.copies):
                    gemm.run(self.A[i], self.B[i], self.C)
        torch.cuda.synchronize()
        best = float("inf")
        r = 0
        # best of `reps` replays; short launches (< 50 us) get 3x more replays
        # because their run-to-run noise is ~10 %
        while r < reps or (best < 50.0 and r < 3 * reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            graph.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / self.copies)
            r += 1
        gemm.check()
        return best


def algorithmic_bytes(m, n, k, dtype):
    """Compulsory traffic: A and B read once, C written once (beta = 0)."""
    es = 8 if dtype == "fp64" else 2
    cs = 8 if dtype == "fp64" else 4
    return es * (m * k + k * n) + cs * m * n


def run(shapes, names, variant, dtype, rank=0, world=1, log_every=0, params=None):
    import torch

    ab = {"bf16": sk.DType.BFloat16, "fp16": sk.DType.Float16, "fp64": sk.DType.Float64}[dtype]
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp64": torch.float64}[dtype]
    blk = sk.kernel_blocking(ab, variant)
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    # p = co-resident persistent CTAs: pairs for 2-SM, 2 DMMA CTAs per SM for FP64
    p = 2 * sms if dtype == "fp64" else sms // (2 if variant == sk.Variant.TwoSM else 1)
    params = params or sk.default_cost_params(ab, variant)
    rows = []
    for idx, (m, n, k) in enumerate(shapes):
        if idx % world != rank:
            continue
        problem = sk.GemmProblem(int(m), int(n), int(k))
        timer = ShapeTimer(torch, int(m), int(n), int(k), tdt)
        for a in strategies_for(problem, blk, p, names, params):
            gemm = sk.Gemm(a, ab, variant)
            t = timer.time_us(gemm)
            rows.append({"idx": idx, "m": m, "n": n, "k": k, "t": a.grid.total_tiles,
                         "iters_per_tile": a.grid.iters_per_tile,
                         "strategy": getattr(a, "label", sk.strategy_name(a.strategy)),
                         "schedule": sk.strategy_name(a.strategy),
                         "param": a.param, "tiles_m": a.grid.tiles_m, "tiles_n": a.grid.tiles_n,
                         "g": a.grid_size,
                         "variant": "dmma" if dtype == "fp64" else (
                             "2sm" if variant == sk.Variant.TwoSM else "1sm"),
                         "dtype": dtype, "copies": timer.copies, "l2_cold": int(timer.cold),
                         "time_us": t, "tflops": 2.0 * m * n * k / (t * 1e-6) / 1e12,
                         "gbps": algorithmic_bytes(m, n, k, dtype) / (t * 1e-6) / 1e9})
        del timer
        if log_every and (idx // world) % log_every == 0:
            print(f"[rank {rank}] {idx}/{len(shapes)} {m}x{n}x{k}", file=sys.stderr, flush=True)
    return rows


def summarise(rows, baseline="data_parallel", tol=0.05):
    """Geomean TFLOP/s speedup of each strategy over data-parallel (per-shape
    time ratio), its range, and the shapes regressing beyond `tol`."""
    by_shape = {}
    for r in rows:
        by_shape.setdefault(r["idx"], {})[r["strategy"]] = r["time_us"]
    labels = sorted({r["strategy"] for r in rows} - {baseline})
    out = {"shapes": len(by_shape)}
    for name in labels:
        sp = [d[baseline] / d[name] for d in by_shape.values() if name in d and baseline in d]
        if sp:
            out[name] = {"geomean_speedup": float(np.exp(np.mean(np.log(sp)))),
                         "min": float(min(sp)), "max": float(max(sp)),
                         "regress_gt_5pct": int(sum(s < 1 - tol for s in sp))}
    gb = {}
    for r in rows:
        if "gbps" in r:
            gb.setdefault(r["strategy"], []).append(r["gbps"])
    if gb:
        out["median_gbps"] = {k: float(np.median(v)) for k, v in sorted(gb.items())}
    return out


def fit_cost_model(rows, p):
    """Calibrate the wave-aware model on measured rows (stream_k:<g> and
    data_parallel) and report its selection quality."""
    samples = []
    for r in rows:
        if r["strategy"] == "data_parallel" or r["strategy"].startswith("stream_k:") and \
                r["strategy"] != "stream_k:auto":
            grid = sk.TileGrid(r["tiles_m"], r["tiles_n"], r["t"], r["iters_per_tile"],
                               r["t"] * r["iters_per_tile"])
            samples.append((grid, r["g"], r["time_us"]))
    # the 16-bit kernels' cooperative fixup is part of what was measured
    params = sk.calibrate(samples, p, coop_peers=sk.default_cost_params().coop_peers)
    return params, len(samples)


def write_csv(path, rows):
    rows = sorted(rows, key=lambda r: (r["idx"], r["strategy"]))
    with open(path, "w") as f:
        f.write(SCHEMA + "\n" + ",".join(COLUMNS) + "\n")
        for r in rows:
            f.write(",".join(f"{r[c]:.6g}" if isinstance(r[c], float) else str(r[c]) for c in COLUMNS)
                    + "\n")


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="config3", choices=["config3", "config4", "corpus", "skinny"])
    ap.add_argument("--count", type=int, default=32824)
    ap.add_argument("--offset", type=int, default=0)
    ap.add_argument("--lo", type=int, default=128)
    ap.add_argument("--hi", type=int, default=8192)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--variant", default="2sm", choices=["1sm", "2sm"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16", "fp64"])
    ap.add_argument("--strategies", default="data_parallel,stream_k,two_tile_sk_dp,dp_one_tile_sk")
    ap.add_argument("--out", default="sweep.csv")
    ap.add_argument("--log-every", type=int, default=0)
    ap.add_argument("--calibrate", action="store_true",
                    help="fit the grid-size model on the measured stream_k:<g>/data_parallel rows")
    args = ap.parse_args(argv)

    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if args.shapes == "config3":
        shapes = CONFIG3
    elif args.shapes == "config4":
        shapes = CONFIG4
    elif args.shapes == "skinny":
        shapes = SKINNY
    else:
        c = sk.corpus(args.seed, args.offset + args.count, args.lo, args.hi)[args.offset:]
        shapes = [tuple(int(x) for x in r[:3]) for r in c]
    names = args.strategies.split(",")
    variant = sk.Variant.TwoSM if args.variant == "2sm" else sk.Variant.OneSM
    rows = run(shapes, names, variant, args.dtype, rank, world, args.log_every)
    part = f"{args.out}.part{rank}.json"
    with open(part, "w") as f:
        json.dump(rows, f)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        dist.barrier()  # control plane only: every part is on disk
    if rank == 0:
        allrows = []
        for r in range(world):
            with open(f"{args.out}.part{r}.json") as f:
                allrows += json.load(f)
            os.remove(f"{args.out}.part{r}.json")
        write_csv(args.out, allrows)
        summary = {"sweep": args.shapes, "variant": args.variant, "dtype": args.dtype,
                   "world": world, **summarise(allrows)}
        if args.calibrate:
            sms = torch.cuda.get_device_properties(0).multi_processor_count
            p = 2 * sms if args.dtype == "fp64" else sms // (2 if args.variant == "2sm" else 1)
            params, n = fit_cost_model(allrows, p)
            summary["cost_params"] = params.as_dict()
            summary["calibration_samples"] = n
        print(json.dumps(summary))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
