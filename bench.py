#!/usr/bin/env python
"""bench.py -- Stream-K GEMM on B200 (BASELINE.json config 2 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--strategy two_tile_sk_dp|stream_k|data_parallel|fixed_split|dp_one_tile_sk]
                    [--m 8192 --n 8192 --k 8192] [--dtype bf16|fp16] [--no-e2e] [--no-cpu]

A step = one GEMM C(fp32) = A(bf16) x B(bf16), 8192^3, through the hand-written
sm_100a kernel (libskb200.so) under the Stream-K schedule (default: the paper's
evaluated two-tile Stream-K + data-parallel hybrid, p = #SMs).  Inputs are
resident in HBM (A + B = 256 MiB > 126 MB L2, so no flush is needed between
steps).  Rank 0 prints ONE JSON line.

Multi-GPU (torchrun, one process per GPU): weak scaling with no data-path
collective -- rank r computes its own N-column block C[:, r*n:(r+1)*n] of a
GEMM with N*n columns.  No NCCL anywhere: the control plane (the timing
barrier and the max-over-ranks reduction) runs over gloo on host tensors.

--impl reference times the reference's own CPU executor (streamk::execute<float>,
oracle/_ref, built from the reference sources) on rank 0 on a bounded row
sample of the same workload, with all host threads; the product arm's
cpu_baseline times the same sample.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

STRATS = {"data_parallel": 0, "fixed_split": 1, "stream_k": 2, "dp_one_tile_sk": 3,
          "two_tile_sk_dp": 4}
# BASELINE.json "metric"; `value` is the TFLOP/s half, `pct_of_peak` and
# `stream_k_vs_dp` carry the other two.
METRIC = ("GEMM TFLOP/s and % of B200 tensor peak; geomean speedup of Stream-K vs "
          "data-parallel")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strategy", default="two_tile_sk_dp", choices=list(STRATS))
    ap.add_argument("--param", type=int, default=0, help="g / p / s (0 = #SMs, s=2)")
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=8192)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16", "fp64"])
    ap.add_argument("--variant", default="2smw", choices=["auto", "1sm", "2sm", "2smw"])
    ap.add_argument("--sweep-variant", default="2sm", choices=["1sm", "2sm", "2smw"],
                    help="kernel variant of the config-3 / skinny legs (the 256x256 tile by default)")
    ap.add_argument("--tile-group", type=int, default=0,
                    help="sk_gemm_desc.tile_group: 0 = the reference's row-major tile map (default); "
                         "G > 1 / -1 = opt-in grouped layout (experiments)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=0, help="row sample for the CPU legs (0=auto)")
    ap.add_argument("--sustained-s", type=float, default=2.0,
                    help="seconds of back-to-back launches for the sustained figure (0 = skip)")
    return ap.parse_args(argv)


class ControlPlane:
    """Barrier + max-over-ranks over gloo (host tensors): the only inter-rank
    traffic of the bench.  The GEMM data path has no collective and no NCCL."""

    def __init__(self, world: int):
        self.world = world
        self.dist = None
        if world > 1:
            import torch.distributed as dist

            dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.dist:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist:
            self.dist.barrier()
            self.dist.destroy_process_group()


# Row sample of the CPU legs: both the reference arm (per step) and the
# product arm's cpu_baseline time streamk::execute on these many rows of A.
CPU_ROWS = {"bf16": 1024, "fp16": 1024, "fp64": 512}


def fp64_leg(sk, torch, timed, p_dev_fp64, size=8192):
    """8192^3 FP64 on the DMMA kernel: two_tile_sk_dp(p) and data-parallel
    against cuBLAS DGEMM on the same operands (best of 3 bursts of 5 launches
    each), then the config-4 sweep's stream_k:auto vs data-parallel geomean."""
    from paper_2301_03598_b200 import sweep as sw

    ab = sk.DType.Float64
    blk = sk.kernel_blocking(ab)
    pr = sk.GemmProblem(size, size, size)
    A = sk.random_matrix_device(size, size, 42, sk.DType.Float64, ab)
    B = sk.random_matrix_device(size, size, 43, sk.DType.Float64, ab)
    Cd = torch.empty(size, size, device="cuda", dtype=torch.float64)
    flops = 2.0 * size ** 3
    out = {"shape": [size, size, size], "blocking": [blk.blk_m, blk.blk_n, blk.blk_k]}
    for name, a in (("two_tile_sk_dp", sk.hybrid(pr, blk, p_dev_fp64, sk.HybridVariant.TwoTileSkDp)),
                    ("data_parallel", sk.data_parallel(pr, blk))):
        g = sk.Gemm(a, ab)
        ms = min(timed(lambda: g.run(A, B, Cd), 5, 2) for _ in range(3))
        g.check()
        out[name] = {"ms": ms, "tflops": flops / (ms * 1e-3) / 1e12}
    ms_c = min(timed(lambda: torch.matmul(A, B), 5, 2) for _ in range(3))
    out["cublas_dgemm_tflops"] = flops / (ms_c * 1e-3) / 1e12
    out["frac_of_cublas_dgemm"] = out["two_tile_sk_dp"]["tflops"] / out["cublas_dgemm_tflops"]
    del A, B, Cd
    rows = sw.run(sw.CONFIG4, ["data_parallel", "stream_k:auto"], sk.Variant.Auto, "fp64")
    summ = sw.summarise(rows)["stream_k:auto"]
    out["config4"] = {"shapes": len(sw.CONFIG4), "policy": "stream_k:auto",
                      "geomean_sk_vs_dp": summ["geomean_speedup"], "min": summ["min"],
                      "max": summ["max"], "regress_gt_5pct": summ["regress_gt_5pct"]}
    return out


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("hbm_gbs", 6552.3)), "measured"
    except Exception:
        return 1590.0, 6650.0, "fallback"


def load_sustained_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops_sustained"])
    except Exception:
        return None


def load_traffic(workload: str):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(workload)
        return float(e["dram_bytes_per_launch"]) if e else None
    except Exception:
        return None


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: an NVML
    polling thread (~1 ms period), falling back to `nvidia-smi -lms 20`."""

    REASONS = {  # nvmlClocksEventReason bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap",
    }

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop = False
        self.thread = None
        self.max_mhz = None

    def _poll(self, nv, h):
        while not self.stop:
            try:
                mhz = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.samples.append((mhz, bits, pw))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        import sys
        import threading

        # the poller must get the GIL between the launch loop's Python steps
        self._switch = sys.getswitchinterval()
        sys.setswitchinterval(0.0002)
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.thread.start()
            time.sleep(0.01)
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *exc):
        import sys

        self.stop = True
        if self.thread:
            self.thread.join()
        sys.setswitchinterval(self._switch)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        loaded = [x for x in sm if x > 500] or sm
        reasons = sorted({name for _, bits, _ in self.samples for bit, name in self.REASONS.items()
                          if bits & bit})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "power_w_max": max(s[2] for s in self.samples),
                "source": "NVML poll during the timed region"}


def cpu_reference_leg(args, strategy, param, blk, rows=None):
    """The reference's own CPU executor on a row sample of the workload:
    streamk::execute<float> with every host thread.  Returns (tflops, seconds,
    sample description, threads)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np

    import oracle

    kind = "reference" if oracle.have_reference() else "port"
    orc = oracle.Oracle(kind)
    threads = os.cpu_count() or 1
    fp64 = args.dtype == "fp64"
    rows = rows or args.cpu_rows or CPU_ROWS[args.dtype]
    m, n, k = rows, args.n, args.k
    dt_name, tname = ("float64", "double") if fp64 else ("float32", "float")
    A = orc.random_matrix(m, k, 42, dt_name)
    B = orc.random_matrix(k, n, 43, dt_name)
    # same decomposition family on the sampled problem; the grid knob is the CPU's p
    prm = param if strategy != 1 else max(param, 1)
    t0 = time.perf_counter()
    orc.execute(strategy, prm, A, B, blk[0], blk[1], blk[2], threads=threads)
    dt = time.perf_counter() - t0
    tf = 2.0 * m * n * k / dt / 1e12
    sample = (f"streamk::execute<{tname}> ({kind}) {m}x{n}x{k} row sample of {args.m}x{args.n}x{args.k}, "
              f"strategy {list(STRATS)[strategy]}, blk {blk[0]}x{blk[1]}x{blk[2]}")
    return tf, dt, sample, (threads if kind == "reference" else 1), kind


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    # same tile config and grid knob as our arm (kernel_blocking of the variant)
    if args.dtype == "fp64":
        blk, p_dev = (64, 64, 16), 296
    elif args.variant == "2sm":
        blk, p_dev = (256, 256, 64), 74
    elif args.variant == "2smw":
        blk, p_dev = (256, 512, 64), 74
    else:
        blk, p_dev = (128, 256, 64), 148
    strategy = STRATS[args.strategy]
    param = args.param or (2 if strategy == 1 else p_dev)
    vals = []
    last = None
    for i in range(args.warmup + args.steps):
        tf, dt, sample, cores, kind = cpu_reference_leg(args, strategy, param, blk)
        if i >= args.warmup:
            vals.append(tf)
        last = (sample, cores, kind)
    v = statistics.median(vals) if vals else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if args.dtype == "fp64" else "f32",
        "data": "synthetic (reference random_matrix<%s>)" % ("double" if args.dtype == "fp64" else "float"),
        "config": {"workload": f"{args.m}x{args.n}x{args.k} GEMM, {args.strategy}, CPU row sample"},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": last[1], "kind": last[2],
                         "sample": last[0]},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import numpy as np
    import torch

    import paper_2301_03598_b200 as sk

    ndev = torch.cuda.device_count()
    # One rank per GPU (more ranks than GPUs only when the multi-rank path is
    # exercised on a 1-GPU box: ranks then share the device).
    local = local % max(ndev, 1)
    torch.cuda.set_device(local)
    cp = ControlPlane(world)

    ab = {"bf16": sk.DType.BFloat16, "fp16": sk.DType.Float16, "fp64": sk.DType.Float64}[args.dtype]
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp64": torch.float64}[args.dtype]
    cdt = torch.float64 if args.dtype == "fp64" else torch.float32
    variant = {"auto": sk.Variant.Auto, "1sm": sk.Variant.OneSM, "2sm": sk.Variant.TwoSM,
               "2smw": sk.Variant.TwoSMWide}[args.variant]
    blk = sk.kernel_blocking(ab, variant)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    strategy = sk.Strategy(STRATS[args.strategy])
    # p = co-resident persistent CTAs: SM pairs (2-SM), SMs (1-SM), 2 per SM (FP64 DMMA)
    p_dev = 2 * sms if args.dtype == "fp64" else sms // (2 if blk.blk_m == 256 else 1)
    param = args.param or (2 if strategy == sk.Strategy.FixedSplit else p_dev)
    m, n, k = args.m, args.n, args.k  # this rank's column block: n columns of a N*n GEMM
    problem = sk.GemmProblem(m, n, k)
    a = sk._assignment(strategy, problem, blk, param)
    a_dp = sk.data_parallel(problem, blk)

    # The reference's inputs (random_matrix<float>, matrix.hpp:56-68), generated
    # on the device and rounded to the kernel's input type.
    gen = sk.DType.Float64 if args.dtype == "fp64" else sk.DType.Float32
    A = sk.random_matrix_device(m, k, 42 + 2 * rank, gen, ab)
    B = sk.random_matrix_device(k, n, 43 + 2 * rank, gen, ab)
    cal = 2 if args.dtype == "fp64" else 4  # 16-byte rows of C (TMA)
    Cout = torch.empty(m, -(-n // cal) * cal, device="cuda", dtype=cdt)[:, :n]
    gemm = sk.Gemm(a, ab, variant, tile_group=args.tile_group)
    gemm_dp = sk.Gemm(a_dp, ab, variant, tile_group=args.tile_group)
    stream = torch.cuda.current_stream()
    flops = 2.0 * m * n * k

    def timed(run, steps, warmup):
        for _ in range(warmup):
            run()
        torch.cuda.synchronize()
        cp.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        return cp.max(e0.elapsed_time(e1) / steps)

    run_sk = lambda: gemm.run(A, B, Cout)  # noqa: E731
    with ClockSampler(local) as clk:
        ms = timed(run_sk, args.steps, max(args.warmup, 3))
    gemm.check()
    clocks = clk.summary()
    # Cross-check with the clock the kernel itself sees: clock64 / globaltimer
    # stamped by every CTA of a traced launch run back-to-back after the timed
    # region (same power state).
    traced = sk.Gemm(a, ab, variant, trace=True, tile_group=args.tile_group)
    for _ in range(max(3, min(args.steps, 10))):
        traced.run(A, B, Cout)
    torch.cuda.synchronize()
    clocks["kernel_sm_mhz"] = traced.clock_mhz()
    del traced
    ms_dp = timed(lambda: gemm_dp.run(A, B, Cout), max(args.steps // 2, 3), 3)
    gemm_dp.check()

    value = flops * world / (ms * 1e-3) / 1e12  # whole-job TFLOP/s
    per_launch_tflops = flops / (ms * 1e-3) / 1e12
    peak_tf, _, peak_kind = load_peaks()
    peak_kind = f"{peak_kind} bf16_tflops (burst)"
    sustained_peak = load_sustained_peak()
    cublas = None
    if args.dtype == "fp64":
        # no FP64 figure in MEASURED_PEAKS.json: cuBLAS DGEMM of the same shape,
        # measured here (best of 5), is the FP64 denominator
        dg = lambda: torch.matmul(A, B)  # noqa: E731
        ms_d = min(timed(dg, 3, 2) for _ in range(5))
        peak_tf, peak_kind = flops / (ms_d * 1e-3) / 1e12, "measured cuBLAS DGEMM, same shape and harness"
        sustained_peak = None
    esz = A.element_size()
    workload = f"{m}x{n}x{k}_{args.dtype}_{sk.strategy_name(strategy)}_{blk.blk_m}x{blk.blk_n}x{blk.blk_k}"

    # ---- sustained: back-to-back launches for >= sustained_s seconds, own clocks
    sustained = None
    if args.sustained_s > 0:
        reps = max(args.steps, int(math.ceil(args.sustained_s * 1e3 / ms)))
        with ClockSampler(local) as clk2:
            ms_s = timed(run_sk, reps, 3)
        gemm.check()
        tf_s = flops / (ms_s * 1e-3) / 1e12
        sustained = {"tflops": tf_s, "launches": reps, "seconds": reps * ms_s * 1e-3,
                     "clocks": clk2.summary()}
        if sustained_peak:
            sustained.update(peak=sustained_peak, frac=tf_s / sustained_peak,
                             peak_kind="measured bf16_tflops_sustained")
        if args.dtype != "fp64" and rank == 0:
            # the library GEMM on the same operands in the same harness, for context
            mm = lambda: torch.matmul(A, B)  # noqa: E731
            cb = min(timed(mm, 10, 3) for _ in range(3))
            cs = timed(mm, reps, 3)
            cublas = {"burst_tflops": flops / (cb * 1e-3) / 1e12,
                      "sustained_tflops": flops / (cs * 1e-3) / 1e12,
                      "what": "torch.matmul (cuBLAS, bf16 C), same operands, for comparison only"}

    # ---- host cost of one sk_gemm call (descriptor checks, cached tensor maps,
    # launch), outside CUDA graphs, on a short shape
    host = None
    if rank == 0:
        hp = sk.GemmProblem(512, 512, 512)
        ha = sk.auto_stream_k(hp, blk, p_dev)  # the policy's pick for this shape
        hg = sk.Gemm(ha, ab, variant)
        hA = sk.random_matrix_device(512, 512, 1, gen, ab)
        hB = sk.random_matrix_device(512, 512, 2, gen, ab)
        hC = torch.empty(512, 512, device="cuda", dtype=cdt)
        for _ in range(20):
            hg.run(hA, hB, hC)
        torch.cuda.synchronize()
        calls = 500
        t0 = time.perf_counter()
        for _ in range(calls):
            hg.run(hA, hB, hC)
        host_us = (time.perf_counter() - t0) / calls * 1e6
        torch.cuda.synchronize()
        ms_small = timed(lambda: hg.run(hA, hB, hC), 200, 10)
        hg.check()
        host = {"shape": [512, 512, 512],
                "strategy": f"stream_k:auto -> {sk.strategy_name(ha.strategy)}({ha.param})",
                "host_us_per_call": host_us, "device_us_per_launch_back_to_back": ms_small * 1e3,
                "path": "Gemm.run -> sk_gemm (ctypes), no CUDA graph"}

    # ---- end to end through the reference-facing C-ABI call (sk_execute): pinned
    # host A/B in, host C out, copies inside the timed region.
    e2e = None
    if not args.no_e2e:
        Ah = A.cpu().pin_memory()
        Bh = B.cpu().pin_memory()
        Ch = torch.empty(m, n, dtype=cdt).pin_memory()
        if ab == sk.DType.Float64:
            An, Bn = Ah.numpy(), Bh.numpy()
        else:
            An = Ah.view(torch.int16).numpy().view(np.uint16 if ab == sk.DType.BFloat16 else np.float16)
            Bn = Bh.view(torch.int16).numpy().view(np.uint16 if ab == sk.DType.BFloat16 else np.float16)
        Cn = Ch.numpy()
        lib = sk.lib()
        pc, bc = problem._c(), blk._c()

        def e2e_step():
            st = lib.sk_execute(C.byref(pc), C.byref(bc), int(strategy), param, int(ab), int(ab),
                                int(variant), An.ctypes.data_as(C.c_void_p),
                                Bn.ctypes.data_as(C.c_void_p), Cn.ctypes.data_as(C.c_void_p), local)
            sk._check(st, "sk_execute")

        for _ in range(2):
            e2e_step()
        cp.barrier()
        steps_e2e = max(3, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(steps_e2e):
            e2e_step()  # synchronous: H2D + kernel + D2H + status read
        dt = cp.max((time.perf_counter() - t0) / steps_e2e)
        e2e = {"value": flops * world / dt / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(A.numel() * A.element_size() + B.numel() * B.element_size()),
               "d2h_bytes_per_step": int(m * n * Cout.element_size() + 4),
               "ms_per_step": dt * 1e3,
               "path": "sk_execute (C ABI, host buffers, pinned)"}
        sk.lib().sk_execute_release()

    # Live Stream-K vs data-parallel geomean over BASELINE config 3's
    # quantisation-limited shapes (the metric's second half; the full corpus
    # is measured by `python -m paper_2301_03598_b200.sweep`).
    sweep = None
    if rank == 0 and not args.no_sweep:
        from paper_2301_03598_b200 import sweep as sw

        shapes, label = (sw.CONFIG4, "config4") if args.dtype == "fp64" else (sw.CONFIG3, "config3")
        sv = {"1sm": sk.Variant.OneSM, "2sm": sk.Variant.TwoSM,
              "2smw": sk.Variant.TwoSMWide}[args.sweep_variant] if args.dtype != "fp64" else variant
        rows = sw.run(shapes, ["data_parallel", "stream_k:auto"], sv, args.dtype)
        summ = sw.summarise(rows)["stream_k:auto"]
        sweep = {"shapes": "%s (%d)" % (label, len(shapes)), "policy": "stream_k:auto (cost model)",
                 "variant": args.sweep_variant if args.dtype != "fp64" else "dmma",
                 "geomean_sk_vs_dp": summ["geomean_speedup"], "min": summ["min"],
                 "max": summ["max"], "regress_gt_5pct": summ["regress_gt_5pct"]}
        if args.dtype != "fp64":
            # bandwidth-bound skinny shapes (below the ridge): HBM GB/s vs the measured peak
            hbm = load_peaks()[1]
            srows = sw.run(sw.SKINNY[:2] + sw.SKINNY[4:6], ["data_parallel", "stream_k:auto"], sv,
                           args.dtype)
            sweep["skinny_hbm"] = [
                {"shape": [r["m"], r["n"], r["k"]], "strategy": r["strategy"],
                 "schedule": r["schedule"], "g": r["g"],
                 "gbps": round(r["gbps"], 1), "frac_of_hbm_peak": round(r["gbps"] / hbm, 3)}
                for r in srows]
            if args.sweep_variant != "1sm":
                # the same shapes on the 1-SM kernel (m <= 128 fills its 128-row tile;
                # its cluster fixup fits more k-chunks: clusters of up to 8 CTAs)
                srows = sw.run(sw.SKINNY[:2] + sw.SKINNY[4:6], ["data_parallel", "stream_k:auto"],
                               sk.Variant.OneSM, args.dtype)
                sweep["skinny_hbm_1sm"] = [
                    {"shape": [r["m"], r["n"], r["k"]], "strategy": r["strategy"],
                     "schedule": r["schedule"], "g": r["g"],
                     "gbps": round(r["gbps"], 1), "frac_of_hbm_peak": round(r["gbps"] / hbm, 3)}
                    for r in srows]

    # BASELINE config 4 in the default run: FP64 DGEMM on the DMMA kernel (the
    # paper's 64x64x16 tile), 8192^3 hybrid vs data-parallel vs cuBLAS DGEMM in
    # this harness (the FP64 denominator: MEASURED_PEAKS.json has none), and the
    # config-4 shapes' Stream-K policy vs data-parallel.
    fp64 = None
    if rank == 0 and not args.no_sweep and args.dtype != "fp64":
        fp64 = fp64_leg(sk, torch, timed, p_dev_fp64=2 * sms)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        tf, dt, sample, cores, kind = cpu_reference_leg(args, int(strategy), param,
                                                        (blk.blk_m, blk.blk_n, blk.blk_k))
        cpu = {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": kind, "sample": sample,
               "seconds": dt}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic: the reference's random_matrix<float>(42 + 2r), (43 + 2r) rounded to "
                    f"{args.dtype}, generated on the device",
            "config": {"workload": workload, "m": m, "n": n * world, "k": k,
                       "n_per_gpu": n, "strategy": sk.strategy_name(strategy), "param": param,
                       "grid_size": a.grid_size, "blocking": [blk.blk_m, blk.blk_n, blk.blk_k],
                       "tile_map": "row-major (executor.hpp:69-70)" if args.tile_group in (0, 1)
                       else f"grouped (tile_group={args.tile_group}, opt-in)",
                       "parallelism": f"column-blocks x{world}, no collective",
                       "l2": "inputs 256 MiB > 126 MB L2 (no flush needed)"},
            "pct_of_peak": {"measured_cublas_burst": per_launch_tflops / peak_tf,
                            "datasheet_2250": per_launch_tflops / 2250.0},
            "data_parallel": {"ms_per_step": ms_dp, "tflops": flops / (ms_dp * 1e-3) / 1e12,
                              "speedup_sk_over_dp": ms_dp / ms},
            "roofline": {"bound": "tensor", "achieved": per_launch_tflops, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": per_launch_tflops / peak_tf,
                         "peak_kind": peak_kind,
                         "traffic": load_traffic(workload),
                         "algorithmic": {"flops_per_launch": flops,
                                         "bytes_per_launch": esz * (m * k + k * n)
                                         + Cout.element_size() * m * n}},
            "sustained": sustained,
            "cublas_same_harness": cublas,
            "clocks": clocks,
            "gpu_launches": args.steps,
            "host_overhead": host,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "stream_k_vs_dp": sweep,
            "fp64_config4": fp64,
        }
        print(json.dumps(line), flush=True)
    cp.close()


if __name__ == "__main__":
    main()
