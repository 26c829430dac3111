"""Same-harness comparison of the Stream-K kernel with cuBLAS (torch.mm) at one shape.

Both arms are timed exactly like bench.py (W warm-ups, K back-to-back launches
between CUDA events on the launching stream), alternating ROUNDS times on the
same box, so power-cap/clock state is comparable.  cuBLAS is run with an fp32
output (out_dtype) to match C = fp32, and with bf16 output for reference.

  python scripts/cublas_compare.py [--m 8192 --n 8192 --k 8192 --steps 20 --rounds 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    A = (torch.rand(m, k, device="cuda") * 2 - 1).bfloat16()
    B = (torch.rand(k, n, device="cuda") * 2 - 1).bfloat16()
    C = torch.empty(m, n, device="cuda", dtype=torch.float32)
    Cb = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
    prob = sk.GemmProblem(m, n, k)
    arms = {
        "sk_data_parallel": sk.Gemm(sk.data_parallel(prob, blk), sk.DType.BFloat16, sk.Variant.TwoSM),
        "sk_two_tile_sk_dp": sk.Gemm(sk.hybrid(prob, blk, 74, sk.HybridVariant.TwoTileSkDp),
                                     sk.DType.BFloat16, sk.Variant.TwoSM),
    }
    fns = {name: (lambda g=g: g.run(A, B, C)) for name, g in arms.items()}
    fns["cublas_out_fp32"] = lambda: torch.mm(A, B, out_dtype=torch.float32, out=C)
    fns["cublas_out_bf16"] = lambda: torch.mm(A, B, out=Cb)
    stream = torch.cuda.current_stream()
    flops = 2.0 * m * n * k
    res = {name: [] for name in fns}
    for _ in range(args.rounds):
        for name, f in fns.items():
            for _ in range(args.warmup):
                f()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                f()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            res[name].append(round(flops / (ms * 1e-3) / 1e12, 1))
    arms["sk_two_tile_sk_dp"].run(A, B, C)
    ref = torch.mm(A.float(), B.float())
    out = {"shape": [m, n, k], "steps": args.steps, "tflops": res,
           "max_abs_diff_sk_vs_fp32": float((C - ref).abs().max())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
