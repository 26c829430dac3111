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
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    A = (torch.rand(m, k, device="cuda") * 2 - 1).bfloat16()
    B = (torch.rand(k, n, device="cuda") * 2 - 1).bfloat16()
    C = torch.empty(m, n, device="cuda")
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
    a = sk.stream_k(sk.GemmProblem(m, n, k), blk, args.g)
    for coop in ("0", "1"):
        os.environ["SKB200_COOP"] = coop
        sk.reload_env()
        g = sk.Gemm(a, sk.DType.BFloat16, sk.Variant.TwoSM, timeline=True)
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
        print(json.dumps(out))


if __name__ == "__main__":
    main()
