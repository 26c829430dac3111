"""Drift of the persistent data-parallel waves (device timeline, one B200).

Runs the 2-SM kernel on one shape with per-segment %globaltimer records after
W warm-up launches (so the power state matches the bench) and reports, per
wave j (each pair's j-th tile), the spread of mainloop start times across the
pairs in us and in k-iterations, plus the per-pair mean tile time spread.

  python scripts/wave_drift.py [--m 8192 --n 8192 --k 8192 --strategy data_parallel]
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
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=8192)
    ap.add_argument("--strategy", default="data_parallel")
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    A = (torch.rand(m, k, device="cuda") * 2 - 1).bfloat16()
    B = (torch.rand(k, n, device="cuda") * 2 - 1).bfloat16()
    C = torch.empty(m, n, device="cuda", dtype=torch.float32)
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
    prob = sk.GemmProblem(m, n, k)
    if args.strategy == "data_parallel":
        a = sk.data_parallel(prob, blk)
    else:
        a = sk.hybrid(prob, blk, 74, sk.HybridVariant.TwoTileSkDp)
    plain = sk.Gemm(a, sk.DType.BFloat16, sk.Variant.TwoSM)
    g = sk.Gemm(a, sk.DType.BFloat16, sk.Variant.TwoSM, timeline=True)
    for _ in range(args.warmup):
        plain.run(A, B, C)
    g.run(A, B, C)
    torch.cuda.synchronize()
    rec = g.timeline()  # [unit, tile, core, kind, t_mac_start, t_mac_end, t_wait_end, t_done]
    rec = rec[np.argsort(rec[:, 4])]
    t0 = rec[:, 4].min()
    cores = int(rec[:, 2].max()) + 1
    per_core = [rec[rec[:, 2] == c] for c in range(cores)]
    per_core = [r[np.argsort(r[:, 4])] for r in per_core]
    tile_us = np.median(np.concatenate([(r[:, 5] - r[:, 4]) for r in per_core])) * 1e-3
    ipt = (k + 63) // 64
    waves = min(len(r) for r in per_core)
    out = {"shape": [m, n, k], "strategy": args.strategy, "cores": cores,
           "median_mainloop_us": round(float(tile_us), 2),
           "makespan_us": round(float((rec[:, 7].max() - t0) * 1e-3), 1), "waves": []}
    for j in range(waves):
        st = np.array([(r[j, 4] - t0) * 1e-3 for r in per_core])
        out["waves"].append({"j": j, "start_min_us": round(float(st.min()), 1),
                             "spread_us": round(float(st.max() - st.min()), 2),
                             "spread_kiters": round(float((st.max() - st.min()) / tile_us * ipt), 1),
                             "p10_p90_us": round(float(np.percentile(st, 90) - np.percentile(st, 10)), 2)})
    sm = (rec[:, 3].astype(np.int64) >> 16) & 0xFFFF
    per_core_mean = np.array([np.mean((r[:, 5] - r[:, 4]) * 1e-3) for r in per_core])
    out["per_pair_mean_mainloop_us"] = {"min": round(float(per_core_mean.min()), 2),
                                        "max": round(float(per_core_mean.max()), 2)}
    # the slowest / fastest pairs and their SM ids (die membership)
    order = np.argsort(per_core_mean)
    out["fastest_pairs"] = [[int(c), int(sm[rec[:, 2] == c][0])] for c in order[:6]]
    out["slowest_pairs"] = [[int(c), int(sm[rec[:, 2] == c][0])] for c in order[-6:]]
    print(json.dumps(out))
    if args.out:
        np.save(args.out, rec)


if __name__ == "__main__":
    main()
