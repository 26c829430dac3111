"""Device timeline of one stream_k launch with and without the cooperative fixup
(SKB200_COOP=0/1): when mainloops end, when units finish (publish + folds), makespan.

  python scripts/coop_timeline.py --m 1024 --n 1024 --k 32768 --g 74
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1024)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--k", type=int, default=32768)
    ap.add_argument("--g", type=int, default=74)
    ap.add_argument("--strategy", default="stream_k", choices=["stream_k", "data_parallel", "two_tile_sk_dp"])
    ap.add_argument("--variant", default="2sm", choices=["1sm", "2sm"])
    ap.add_argument("--coop", default="0,1")
    ap.add_argument("--csv", default="", help="write the last timeline (reference CSV format) here")
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    A = sk.random_matrix_device(m, k, 42, sk.DType.Float32, sk.DType.BFloat16)  # 16-byte rows
    B = sk.random_matrix_device(k, n, 43, sk.DType.Float32, sk.DType.BFloat16)
    C = torch.empty(m, -(-n // 4) * 4, device="cuda")[:, :n]
    V = sk.Variant.TwoSM if args.variant == "2sm" else sk.Variant.OneSM
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    P = sk.GemmProblem(m, n, k)
    a = {"stream_k": lambda: sk.stream_k(P, blk, args.g), "data_parallel": lambda: sk.data_parallel(P, blk),
         "two_tile_sk_dp": lambda: sk.hybrid(P, blk, args.g, sk.HybridVariant.TwoTileSkDp)}[args.strategy]()
    for coop in args.coop.split(","):
        os.environ["SKB200_COOP"] = coop
        sk.reload_env()
        g = sk.Gemm(a, sk.DType.BFloat16, V, timeline=True)
        for _ in range(10):
            g.run(A, B, C)
        torch.cuda.synchronize()
        r = g.timeline()
        t0 = r[:, 4].min()
        us = lambda x: np.round((x - t0) / 1e3, 2)  # noqa: E731
        kind = r[:, 3].astype(np.int64)
        own = (kind & 2) != 0
        part = (kind & 1) != 0
        out = {"coop": coop, "makespan_us": float(us(r[:, 7].max())),
               "mac_end_us": [float(us(r[:, 5].min())), float(np.median(us(r[:, 5]))), float(us(r[:, 5].max()))],
               "partial_done_us": [float(np.median(us(r[part, 7]))), float(us(r[part, 7].max()))] if part.any() else None,
               "owner_wait_end_us": [float(np.median(us(r[own, 6]))), float(us(r[own, 6].max()))] if own.any() else None,
               "owner_done_us": [float(np.median(us(r[own, 7]))), float(us(r[own, 7].max()))] if own.any() else None}
        out.update(shape=[m, n, k], strategy=args.strategy, g=a.grid_size, variant=args.variant)
        print(json.dumps(out))
        if args.csv:
            from paper_2301_03598_b200 import timeline as tlm

            with open(args.csv, "w") as f:
                tlm.write_timeline_csv(tlm.from_device(r), f)


if __name__ == "__main__":
    main()
