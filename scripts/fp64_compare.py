"""Same-harness FP64 comparison: the DMMA Stream-K kernel vs cuBLAS DGEMM (torch.mm
on float64) at one shape, 20 back-to-back launches after warm-up, alternating.

  python scripts/fp64_compare.py [--n 8192] [--rounds 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    n = args.n
    A = torch.rand(n, n, device="cuda", dtype=torch.float64) * 2 - 1
    B = torch.rand(n, n, device="cuda", dtype=torch.float64) * 2 - 1
    C = torch.empty(n, n, device="cuda", dtype=torch.float64)
    blk = sk.kernel_blocking(sk.DType.Float64)
    prob = sk.GemmProblem(n, n, n)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    fns = {
        "sk_data_parallel": sk.Gemm(sk.data_parallel(prob, blk), sk.DType.Float64),
        "sk_two_tile_sk_dp": sk.Gemm(sk.hybrid(prob, blk, 2 * sms, sk.HybridVariant.TwoTileSkDp),
                                     sk.DType.Float64),
    }
    run = {k: (lambda g=g: g.run(A, B, C)) for k, g in fns.items()}
    run["cublas_dgemm"] = lambda: torch.mm(A, B, out=C)
    res = {k: [] for k in run}
    stream = torch.cuda.current_stream()
    for _ in range(args.rounds):
        for k, f in run.items():
            torch.cuda.synchronize()
            time.sleep(0.5)
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                f()
            e1.record(stream)
            torch.cuda.synchronize()
            res[k].append(round(2.0 * n ** 3 / (e0.elapsed_time(e1) / args.steps * 1e-3) / 1e12, 2))
    print(json.dumps({"shape": [n, n, n], "dtype": "fp64", "tflops": res}))


if __name__ == "__main__":
    main()
