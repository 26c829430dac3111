"""BASELINE config 1 on the device: 384 x 384 x 128 on an explicit 4-CTA
persistent grid (num_ctas = 4), data-parallel vs stream_k(4), next to the
reference simulator's unit-cost prediction for the same schedules on p = 4
(simulate.cpp:23-80; acceptance c1's 0.75 vs 1.0 utilisation).

  python scripts/config1_echo.py [--out profiles/r02/config1_echo.json]
The device tile is the 1-SM kernel's 128 x 256 x 64: 6 tiles, 2 iterations
each, so DP needs 2 waves on 4 CTAs (quantisation efficiency 0.75) and
stream_k(4) gives every CTA 3 iterations."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--reps", type=int, default=2000)
    args = ap.parse_args()
    V = sk.Variant.OneSM
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    P = sk.GemmProblem(384, 384, 128)
    A = sk.random_matrix_device(384, 128, 42, sk.DType.Float32, sk.DType.BFloat16)
    B = sk.random_matrix_device(128, 384, 43, sk.DType.Float32, sk.DType.BFloat16)
    C = torch.empty(384, 384, device="cuda")
    out = {"shape": [384, 384, 128], "blocking": [blk.blk_m, blk.blk_n, blk.blk_k], "num_ctas": 4, "rows": []}
    for a in (sk.data_parallel(P, blk), sk.stream_k(P, blk, 4)):
        g = sk.Gemm(a, variant=V, num_ctas=4)
        for _ in range(50):
            g.run(A, B, C)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                for _ in range(100):
                    g.run(A, B, C)
        best = 1e9
        for _ in range(args.reps // 100):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            graph.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 10.0)  # us per launch
        g.check()
        makespan, util = sk.simulate(a, 4)
        out["rows"].append({"strategy": sk.strategy_name(a.strategy), "g": a.grid_size,
                            "device_us_per_launch": round(best, 3),
                            "simulated_makespan_iters": makespan, "simulated_utilization": util,
                            "quantization_efficiency": sk.quantization_efficiency(a.grid.total_tiles, 4)})
    print(json.dumps(out))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
