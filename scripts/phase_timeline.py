"""Where the time of one persistent launch goes (device timeline, one B200).

Runs one shape after W warm-up launches (so the power state matches the
bench), then one launch with per-segment %globaltimer records, and reports:
makespan; mainloop ns per k-iteration of data-parallel vs Stream-K segments;
the end of the data-parallel phase; fixup waits and owner folds; the tail from
the last mainloop end to the last store.

  python scripts/phase_timeline.py --variant 2smw --strategy two_tile_sk_dp
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402

VARIANTS = {"1sm": "OneSM", "2sm": "TwoSM", "2smw": "TwoSMWide"}


def analyse(a, rec):
    """rec rows: [unit, tile, core, kind, t_mac_start, t_mac_end, t_wait_end, t_done]."""
    ipt = a.grid.iters_per_tile
    rng = a.range_table()
    t0 = rec[:, 4].min()
    seg_iters = []
    for u, tile in rec[:, :2]:
        b, e = rng[int(u)]
        lo, hi = max(b, tile * ipt), min(e, (tile + 1) * ipt)
        seg_iters.append(hi - lo)
    seg_iters = np.array(seg_iters, np.float64)
    full = seg_iters == ipt
    partial = (rec[:, 3] & 1) == 1
    owner_peers = (rec[:, 3] & 2) == 2
    dp_units = np.zeros(len(rec), bool)
    if a.strategy in (sk.Strategy.DataParallel,):
        dp_units[:] = True
    elif a.strategy == sk.Strategy.TwoTileSkDp:
        dp_units = rec[:, 0] >= min(a.grid_size, 74 if a.blocking.blk_m == 256 else 148)
    mac = (rec[:, 5] - rec[:, 4]).astype(np.float64)
    ns_per_iter = mac / np.maximum(seg_iters, 1)
    out = {
        "makespan_us": round(float((rec[:, 7].max() - t0) * 1e-3), 2),
        "last_mainloop_end_us": round(float((rec[:, 5].max() - t0) * 1e-3), 2),
        "segments": int(len(rec)),
        "dp_ns_per_iter_median": round(float(np.median(ns_per_iter[dp_units])), 1) if dp_units.any() else None,
        "sk_ns_per_iter_median": round(float(np.median(ns_per_iter[~dp_units])), 1) if (~dp_units).any() else None,
        "dp_phase_end_us": round(float((rec[dp_units, 7].max() - t0) * 1e-3), 2) if dp_units.any() else None,
        "sk_phase_start_us": round(float((rec[~dp_units, 4].min() - t0) * 1e-3), 2) if (~dp_units).any() else None,
    }
    if owner_peers.any():
        w = (rec[owner_peers, 6] - rec[owner_peers, 5]) * 1e-3
        f = (rec[owner_peers, 7] - rec[owner_peers, 6]) * 1e-3
        out["owner_wait_us"] = {"median": round(float(np.median(w)), 2), "max": round(float(w.max()), 2)}
        out["owner_fold_store_us"] = {"median": round(float(np.median(f)), 2), "max": round(float(f.max()), 2)}
    if partial.any():
        p = (rec[partial, 7] - rec[partial, 5]) * 1e-3
        out["partial_publish_us"] = {"median": round(float(np.median(p)), 2), "max": round(float(p.max()), 2)}
    plain = ~partial & ~owner_peers
    if plain.any():
        d = (rec[plain, 7] - rec[plain, 5]) * 1e-3
        out["plain_store_us"] = {"median": round(float(np.median(d)), 2), "max": round(float(d.max()), 2)}
    # per core: idle gaps between a segment's mainloop end and the next one's start
    gaps = []
    for c in np.unique(rec[:, 2]):
        r = rec[rec[:, 2] == c]
        r = r[np.argsort(r[:, 4])]
        gaps += list((r[1:, 4] - r[:-1, 5]) * 1e-3)
    if gaps:
        out["mma_gap_us"] = {"median": round(float(np.median(gaps)), 3), "max": round(float(np.max(gaps)), 2)}
    ends = np.array([rec[rec[:, 2] == c, 7].max() for c in np.unique(rec[:, 2])]) - t0
    out["core_end_us"] = {"min": round(float(ends.min() * 1e-3), 2), "max": round(float(ends.max() * 1e-3), 2)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=8192)
    ap.add_argument("--variant", default="2smw", choices=list(VARIANTS))
    ap.add_argument("--strategy", default="two_tile_sk_dp")
    ap.add_argument("--g", type=int, default=0, help="stream_k grid (0 = p)")
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    V = getattr(sk.Variant, VARIANTS[args.variant])
    A = sk.random_matrix_device(m, k, 42, sk.DType.Float32, sk.DType.BFloat16)
    B = sk.random_matrix_device(k, n, 43, sk.DType.Float32, sk.DType.BFloat16)
    C = torch.empty(m, n, device="cuda", dtype=torch.float32)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    p = 148 if V == sk.Variant.OneSM else 74
    prob = sk.GemmProblem(m, n, k)
    a = {"data_parallel": lambda: sk.data_parallel(prob, blk),
         "stream_k": lambda: sk.stream_k(prob, blk, args.g or p),
         "fixed_split": lambda: sk.fixed_split(prob, blk, args.g or 2),
         "stream_k:auto": lambda: sk.auto_stream_k(prob, blk, p),
         "two_tile_sk_dp": lambda: sk.hybrid(prob, blk, p, sk.HybridVariant.TwoTileSkDp),
         "dp_one_tile_sk": lambda: sk.hybrid(prob, blk, p, sk.HybridVariant.DpOneTileSk)}[args.strategy]()
    plain = sk.Gemm(a, sk.DType.BFloat16, V)
    g = sk.Gemm(a, sk.DType.BFloat16, V, timeline=True)
    for _ in range(args.warmup):
        plain.run(A, B, C)
    g.run(A, B, C)
    torch.cuda.synchronize()
    rec = g.timeline()
    out = {"shape": [m, n, k], "variant": args.variant, "strategy": args.strategy,
           "g": a.grid_size, **analyse(a, rec)}
    print(json.dumps(out))
    if args.out:
        np.save(args.out, rec)


if __name__ == "__main__":
    main()
