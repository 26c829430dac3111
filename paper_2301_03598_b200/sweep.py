"""Geometry sweep on B200: BASELINE configs 3 (quantisation-limited shapes),
4 (FP64) and 5 (the paper's 32,824-shape log-sampled corpus), Stream-K vs
data-parallel, every row verified against the reference's CPU executor.

    python -m paper_2301_03598_b200.sweep --shapes config3 --out sweep.csv
    python -m paper_2301_03598_b200.sweep --shapes corpus --count 2000 --out sweep.csv
    torchrun --nproc-per-node N -m paper_2301_03598_b200.sweep --shapes corpus ...

Mirrors run_sweep (core/src/sweep.cpp:75-112): shapes in corpus order
(sk_corpus == sweep.cpp:21-28,79-86), one CSV row per (shape, strategy) under
the reference's own header

    # schema=1
    m,n,k,t,iters_per_tile,strategy,g,utilization,makespan,measured_time,<GPU columns>

The first nine columns are the reference's, byte-identical to run_sweep's for
the same (shape, strategy, p, blocking): utilization and makespan come from the
reference simulator restated in the library (sk_simulate, simulate.cpp:23-80,
unit cost, p = persistent CTAs).  measured_time is the GPU kernel time in
seconds (the reference records its CPU executor's wall time there).  Appended
columns: policy label, knob, kernel variant, dtype, timing copies / L2 state,
TFLOP/s, GB/s, and the verification of that row's C (below) with the reference
CPU executor's own time on the same WorkAssignment.

Timing: each (shape, strategy) runs as a CUDA graph of L >= 8 launches (a multiple of R)
cycling over R operand copies (R chosen so the copies exceed L2 where memory
allows; a copy is re-read only after the others have streamed through L2), best
of 3 replays, CUDA events on the capture stream.  L >= 8 keeps the graph's own
start-up latency out of the per-launch time of large shapes, where R is 2.  Operands are the reference's
random_matrix<float>(seed), (seed + 1) (matrix.hpp:56-68), generated on the
device (sk_random_matrix) and rounded to the kernel's input type.

Verification (every row, after its shape is timed, so CPU work never overlaps
a timed region):
  * integer pass: operands from the reference's random_matrix<int64_t> band
    [-64, 63] (>> 3 when k > 4096, keeping every partial sum below 2^24), C
    compared BIT-EXACTLY with the exact product (integer fp64 GEMM);
  * float pass: random_matrix<float>(matrix_seed), (matrix_seed + 1) rounded to
    the input type and fed to both sides; C checked under the reference's
    verify bound |c - ref| <= 8 eps k max(|ref|, 1) (executor.hpp:217-239)
    against the reference's own execute<float|double> on the same
    WorkAssignment (all host threads, timed: cpu_time_s) when m n k <= 2^30 or
    the shape set is a named config, otherwise against the reference's
    gemm_reference<T> (executor.hpp:22-54) on a seeded sample of rows.
The reference is oracle/_ref (its sources compiled here); the port restatement
when that library is absent.  The product never imports oracle/.

Multi-GPU: shape i runs on rank i % world (one problem per GPU, no
collective on the data path); rank 0 merges the per-rank CSV parts in input
order after a gloo barrier.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

import paper_2301_03598_b200 as sk

SCHEMA = "# schema=1"  # the reference's run_sweep header (sweep.cpp:77)
REF_COLUMNS = ["m", "n", "k", "t", "iters_per_tile", "strategy", "g", "utilization", "makespan",
               "measured_time"]
GPU_COLUMNS = ["policy", "param", "variant", "dtype", "copies", "l2_cold", "tflops", "gbps",
               "int_exact", "float_check", "max_rel_err", "verified", "cpu_time_s", "cpu_threads",
               "cpu_model"]
COLUMNS = REF_COLUMNS + GPU_COLUMNS
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
        elif name.startswith("fixed_split:"):
            a = sk.fixed_split(problem, blk, int(name.split(":")[1]))
            a.label = name
            out.append(a)
        else:
            raise ValueError(name)
    return out


def fmt9(v: float) -> str:
    """sweep.cpp:64-68 fmt: "%.9g"."""
    return "%.9g" % v


def ref_columns(a, p):
    """The reference's deterministic columns of a sweep row (sweep.cpp:104-107):
    m, n, k, t, iters_per_tile, strategy, g, utilization, makespan of the
    unit-cost simulation on p cores."""
    makespan, util = sk.simulate(a, p)
    return [a.problem.m, a.problem.n, a.problem.k, a.grid.total_tiles, a.grid.iters_per_tile,
            sk.strategy_name(a.strategy), a.grid_size, fmt9(util), fmt9(makespan)]


_AB = {"bf16": "BFloat16", "fp16": "Float16", "fp64": "Float64"}


def _ab(dtype):
    return getattr(sk.DType, _AB[dtype])


class ShapeTimer:
    """Pitched operand copies for one shape (the reference's random_matrix
    inputs, generated on the device) + graph-timed launches."""

    def __init__(self, torch, m, n, k, dtype, seed, max_copies=16, mem_budget=4 << 30, min_launches=8):
        self.torch = torch
        ab = _ab(dtype)
        fp64 = dtype == "fp64"
        es = 8 if fp64 else 2
        cdt = torch.float64 if fp64 else torch.float32
        al = 16 // es  # 16-byte rows for TMA
        lda, ldb = -(-k // al) * al, -(-n // al) * al
        ldc = -(-n // 2) * 2 if fp64 else -(-n // 4) * 4
        foot = es * (m * lda + k * ldb)
        self.copies = int(max(1, min(max_copies, math.ceil(2 * L2_BYTES / foot),
                                     mem_budget // max(foot, 1))))
        self.cold = self.copies * foot > L2_BYTES
        # launches per graph replay, cycling over the copies (a copy comes back
        # only after the others -- more than L2 when cold -- have streamed through)
        self.launches = self.copies * max(1, -(-min_launches // self.copies))
        gen = sk.DType.Float64 if fp64 else sk.DType.Float32
        self.A, self.B = [], []
        for i in range(self.copies):  # copy i: random_matrix(seed + 2i), (seed + 2i + 1)
            self.A.append(sk.random_matrix_device(m, k, seed + 2 * i, gen, ab))
            self.B.append(sk.random_matrix_device(k, n, seed + 2 * i + 1, gen, ab))
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
                for j in range(self.launches):
                    i = j % self.copies
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
            best = min(best, e0.elapsed_time(e1) * 1e3 / self.launches)
            r += 1
        gemm.check()
        return best


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip().replace(",", " ")
    except OSError:
        pass
    return "unknown"


class Verifier:
    """Checks one shape's device results against the reference CPU executor
    (see the module docstring).  Test infrastructure: imports oracle/ lazily,
    only when verification is requested; the timed GEMMs never touch it."""

    def __init__(self, torch, dtype, full_limit=1 << 30, sample_rows=8, force_full=False):
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, os.path.join(root, "oracle"))
        import oracle  # noqa: E402  (the checker)

        self.torch = torch
        self.oracle = oracle
        self.ref = oracle.Oracle("reference" if oracle.have_reference() else "port")
        self.kind = self.ref.kind
        self.dtype = dtype
        self.fp64 = dtype == "fp64"
        self.full_limit = full_limit
        self.force_full = force_full
        self.sample_rows = sample_rows
        self.threads = os.cpu_count() or 1
        self.cpu_model = cpu_model()
        self.eps = float(np.finfo(np.float64 if self.fp64 else np.float32).eps)

    def _operands(self, m, n, k, seed, gen, shift=0):
        ab = _ab(self.dtype)
        A = sk.random_matrix_device(m, k, seed, gen, ab, shift=shift)
        B = sk.random_matrix_device(k, n, seed + 1, gen, ab, shift=shift)
        return A, B

    def _run(self, gemm, A, B, m, n):
        torch = self.torch
        cdt = torch.float64 if self.fp64 else torch.float32
        al = 2 if self.fp64 else 4
        C = torch.full((m, -(-n // al) * al), float("nan"), device="cuda", dtype=cdt)[:, :n]
        gemm.run(A, B, C)
        gemm.check()
        return C

    def shape(self, m, n, k, seed, jobs):
        """jobs: [(label, assignment, gemm)].  Returns {label: verification fields}."""
        torch = self.torch
        blk = jobs[0][1].blocking
        out = {}
        # ---- integer pass: bit-exact against the exact product
        shift = 3 if (k > 4096 and not self.fp64) else 0
        Ai, Bi = self._operands(m, n, k, seed, sk.DType.Int64, shift)
        exact = Ai.double() @ Bi.double()  # integers, every partial sum < 2^24: exact
        for label, a, gemm in jobs:
            out[label] = {"int_exact": int(torch.equal(self._run(gemm, Ai, Bi, m, n).double(), exact))}
        del Ai, Bi, exact
        # ---- float pass: the reference's inputs, checked under its verify bound
        gen = sk.DType.Float64 if self.fp64 else sk.DType.Float32
        Af, Bf = self._operands(m, n, k, seed, gen)
        hdt = torch.float64 if self.fp64 else torch.float32
        full = self.force_full or m * n * k <= self.full_limit
        Bh = Bf.to(hdt).cpu().numpy()
        Ah = Af.to(hdt).cpu().numpy() if full else None
        cpu_cache = {}
        rows = None
        if not full:
            rng = np.random.default_rng(seed & 0xFFFFFFFF)
            rows = np.sort(rng.choice(m, size=min(m, self.sample_rows), replace=False))
            Arows = np.ascontiguousarray(Af[torch.from_numpy(rows).cuda()].to(hdt).cpu().numpy())
            from concurrent.futures import ThreadPoolExecutor

            with ThreadPoolExecutor(max_workers=min(len(rows), self.threads)) as ex:
                parts = list(ex.map(lambda i: self.ref.gemm_reference(
                    np.ascontiguousarray(Arows[i:i + 1]), Bh, blk.blk_m, blk.blk_n, blk.blk_k),
                    range(len(rows))))
            ref_rows = np.concatenate(parts, axis=0)
        for label, a, gemm in jobs:
            C = self._run(gemm, Af, Bf, m, n)
            rec = out[label]
            if full:
                key = (int(a.strategy), a.param)
                if key not in cpu_cache:
                    t0 = time.perf_counter()
                    Cref = self.ref.execute(int(a.strategy), a.param, Ah, Bh, blk.blk_m, blk.blk_n,
                                            blk.blk_k, threads=self.threads)
                    cpu_cache[key] = (Cref, time.perf_counter() - t0)
                Cref, cpu_s = cpu_cache[key]
                ok, _, max_rel = self.oracle.verify(C.cpu().numpy(), Cref, k, self.eps)
                rec.update(float_check="full", cpu_time_s=cpu_s)
            else:
                got = C[torch.from_numpy(rows).cuda()].cpu().numpy()
                ok, _, max_rel = self.oracle.verify(got, ref_rows, k, self.eps)
                rec.update(float_check=f"rows{len(rows)}", cpu_time_s=-1.0)
            rec.update(max_rel_err=max_rel,
                       verified="pass" if (ok and rec["int_exact"]) else "FAIL",
                       cpu_threads=self.threads if full else 1,
                       cpu_model=f"{self.kind}:{self.cpu_model}")
        return out


def algorithmic_bytes(m, n, k, dtype):
    """Compulsory traffic: A and B read once, C written once (beta = 0)."""
    es = 8 if dtype == "fp64" else 2
    cs = 8 if dtype == "fp64" else 4
    return es * (m * k + k * n) + cs * m * n


def run(shapes, names, variant, dtype, rank=0, world=1, log_every=0, params=None, seeds=None,
        verify=False, force_full=False, sample_rows=8):
    """Time (and optionally verify) every (shape, strategy); shape i uses
    matrix seed seeds[i] (the corpus's matrix_seed; 42 for named configs)."""
    import torch

    ab = _ab(dtype)
    blk = sk.kernel_blocking(ab, variant)
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    # p = co-resident persistent CTAs: pairs for 2-SM, 2 DMMA CTAs per SM for FP64
    p = 2 * sms if dtype == "fp64" else sms // (1 if variant == sk.Variant.OneSM else 2)
    params = params or sk.default_cost_params(ab, variant)
    ver = Verifier(torch, dtype, force_full=force_full, sample_rows=sample_rows) if verify else None
    rows = []
    for idx, (m, n, k) in enumerate(shapes):
        if idx % world != rank:
            continue
        m, n, k = int(m), int(n), int(k)
        seed = int(seeds[idx]) if seeds is not None else 42
        problem = sk.GemmProblem(m, n, k)
        timer = ShapeTimer(torch, m, n, k, dtype, seed)
        jobs = []
        for a in strategies_for(problem, blk, p, names, params):
            gemm = sk.Gemm(a, ab, variant)
            t = timer.time_us(gemm)
            label = getattr(a, "label", sk.strategy_name(a.strategy))
            jobs.append((label, a, gemm))
            rows.append({"idx": idx, "m": m, "n": n, "k": k, "t": a.grid.total_tiles,
                         "iters_per_tile": a.grid.iters_per_tile,
                         "strategy": label, "schedule": sk.strategy_name(a.strategy),
                         "param": a.param, "tiles_m": a.grid.tiles_m, "tiles_n": a.grid.tiles_n,
                         "g": a.grid_size, "ref": ref_columns(a, p),
                         "variant": "dmma" if dtype == "fp64" else (
                             {sk.Variant.TwoSM: "2sm", sk.Variant.TwoSMWide: "2smw"}.get(variant, "1sm")),
                         "dtype": dtype, "copies": timer.copies, "l2_cold": int(timer.cold),
                         "time_us": t, "tflops": 2.0 * m * n * k / (t * 1e-6) / 1e12,
                         "gbps": algorithmic_bytes(m, n, k, dtype) / (t * 1e-6) / 1e9})
        del timer
        if ver is not None:
            checks = ver.shape(m, n, k, seed, jobs)
            for r in rows[len(rows) - len(jobs):]:
                r.update(checks[r["strategy"]])
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
    if any("verified" in r for r in rows):
        out["verified_rows"] = sum(r.get("verified") == "pass" for r in rows)
        out["failed_rows"] = sum(r.get("verified") == "FAIL" for r in rows)
        out["float_full_rows"] = sum(r.get("float_check") == "full" for r in rows)
        out["max_rel_err"] = max(float(r.get("max_rel_err", 0.0)) for r in rows)
        cpu = [r for r in rows if r.get("cpu_time_s", -1) > 0]
        if cpu:
            out["cpu_reference"] = {
                "rows": len(cpu), "threads": cpu[0]["cpu_threads"], "model": cpu[0]["cpu_model"],
                "seconds": float(sum(r["cpu_time_s"] for r in cpu)),
                "tflops_geomean": float(np.exp(np.mean(np.log(
                    [2.0 * r["m"] * r["n"] * r["k"] / r["cpu_time_s"] / 1e12 for r in cpu]))))}
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


def csv_line(r) -> str:
    """One sweep row: the reference's columns (sweep.cpp:104-109, measured_time =
    GPU seconds), then the GPU / verification columns."""
    ref = [str(x) for x in r["ref"]] + [fmt9(r["time_us"] * 1e-6)]
    ext = {"policy": r["strategy"], "param": r["param"], "variant": r["variant"],
           "dtype": r["dtype"], "copies": r["copies"], "l2_cold": r["l2_cold"],
           "tflops": "%.6g" % r["tflops"], "gbps": "%.6g" % r["gbps"],
           "int_exact": r.get("int_exact", ""), "float_check": r.get("float_check", ""),
           "max_rel_err": "%.3g" % r["max_rel_err"] if "max_rel_err" in r else "",
           "verified": r.get("verified", ""),
           "cpu_time_s": fmt9(r["cpu_time_s"]) if r.get("cpu_time_s", -1) > 0 else "",
           "cpu_threads": r.get("cpu_threads", ""), "cpu_model": r.get("cpu_model", "")}
    return ",".join(ref + [str(ext[c]) for c in GPU_COLUMNS])


def write_csv(path, rows):
    rows = sorted(rows, key=lambda r: (r["idx"], r["strategy"]))
    with open(path, "w") as f:
        f.write(SCHEMA + "\n" + ",".join(COLUMNS) + "\n")
        for r in rows:
            f.write(csv_line(r) + "\n")


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="config3",
                    help="config3 | config4 | corpus | skinny | file:<path> (lines m,n,k[,seed])")
    ap.add_argument("--count", type=int, default=32824)
    ap.add_argument("--offset", type=int, default=0)
    ap.add_argument("--lo", type=int, default=128)
    ap.add_argument("--hi", type=int, default=8192)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--variant", default="2sm", choices=["1sm", "2sm", "2smw"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16", "fp64"])
    ap.add_argument("--strategies", default="data_parallel,stream_k,two_tile_sk_dp,dp_one_tile_sk")
    ap.add_argument("--out", default="sweep.csv")
    ap.add_argument("--log-every", type=int, default=0)
    ap.add_argument("--calibrate", action="store_true",
                    help="fit the grid-size model on the measured stream_k:<g>/data_parallel rows")
    ap.add_argument("--no-verify", action="store_true", help="time only (no C verification)")
    ap.add_argument("--cpu-full", default="auto", choices=["auto", "all", "subset"],
                    help="full CPU reference run per row: all rows (default for named configs) or "
                         "only m n k <= 2^30 (default for the corpus)")
    ap.add_argument("--sample-rows", type=int, default=8)
    args = ap.parse_args(argv)

    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    seeds = None
    if args.shapes == "config3":
        shapes = CONFIG3
    elif args.shapes == "config4":
        shapes = CONFIG4
    elif args.shapes == "skinny":
        shapes = SKINNY
    elif args.shapes.startswith("file:"):
        with open(args.shapes[5:]) as f:
            recs = [[int(x) for x in line.split(",")] for line in f if line.strip() and line[0].isdigit()]
        shapes = [tuple(r[:3]) for r in recs]
        seeds = [r[3] if len(r) > 3 else 42 for r in recs]
    elif args.shapes == "corpus":
        c = sk.corpus(args.seed, args.offset + args.count, args.lo, args.hi)[args.offset:]
        shapes = [tuple(int(x) for x in r[:3]) for r in c]
        seeds = [int(r[3]) for r in c]  # run_sweep's per-shape matrix_seed (sweep.cpp:86)
    else:
        raise SystemExit(f"unknown --shapes {args.shapes}")
    names = args.strategies.split(",")
    variant = {"2sm": sk.Variant.TwoSM, "2smw": sk.Variant.TwoSMWide}.get(args.variant, sk.Variant.OneSM)
    force_full = args.cpu_full == "all" or (args.cpu_full == "auto" and args.shapes != "corpus")
    rows = run(shapes, names, variant, args.dtype, rank, world, args.log_every, seeds=seeds,
               verify=not args.no_verify, force_full=force_full, sample_rows=args.sample_rows)
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
            p = 2 * sms if args.dtype == "fp64" else sms // (1 if args.variant == "1sm" else 2)
            params, n = fit_cost_model(allrows, p)
            summary["cost_params"] = params.as_dict()
            summary["calibration_samples"] = n
        print(json.dumps(summary))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
