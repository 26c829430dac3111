"""Measured device timelines of a few launches rendered in the reference's
Timeline CSV and Gantt SVG formats (timeline.py), after warm-up launches.

  python scripts/render_timelines.py --out profiles/r01g/timelines
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402
from paper_2301_03598_b200 import timeline as tlm  # noqa: E402

CASES = [((8192, 8192, 8192), "two_tile_sk_dp"), ((8192, 8192, 8192), "data_parallel"),
         ((1024, 1024, 32768), "stream_k"), ((512, 512, 65536), "stream_k"),
         ((128, 8192, 8192), "stream_k")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r01g/timelines")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
    for (m, n, k), strat in CASES:
        A = (torch.rand(m, k, device="cuda") * 2 - 1).bfloat16()
        B = (torch.rand(k, n, device="cuda") * 2 - 1).bfloat16()
        C = torch.empty(m, n, device="cuda")
        P = sk.GemmProblem(m, n, k)
        a = {"two_tile_sk_dp": lambda: sk.hybrid(P, blk, 74, sk.HybridVariant.TwoTileSkDp),
             "data_parallel": lambda: sk.data_parallel(P, blk),
             "stream_k": lambda: sk.stream_k(P, blk, 74)}[strat]()
        plain = sk.Gemm(a, sk.DType.BFloat16, sk.Variant.TwoSM)
        g = sk.Gemm(a, sk.DType.BFloat16, sk.Variant.TwoSM, timeline=True)
        for _ in range(8):
            plain.run(A, B, C)
        g.run(A, B, C)
        torch.cuda.synchronize()
        tl = tlm.from_device(g.timeline())
        base = os.path.join(args.out, f"{m}x{n}x{k}_{strat}")
        with open(base + ".csv", "w") as f:
            tlm.write_timeline_csv(tl, f)
        with open(base + ".svg", "w") as f:
            tlm.render_gantt(tl, f)
        print(base, "makespan_us", round(tl.makespan, 1), "utilization", round(tlm.utilization(tl), 3), flush=True)


if __name__ == "__main__":
    main()
