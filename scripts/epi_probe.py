"""Epilogue phase timing of a probe build (-DSKB200_EPI_PROBE, loaded through
SKB200_LIB): per (CTA, epilogue warp) globaltimer stamps of the warp's LAST
segment: 0 accumulator ready, 15 peer flags seen, then per 64-column step
1+3s TMEM drained, 2+3s fold / publish done, 3+3s C boxes issued, 13 flags
signalled, 14 all TMA stores complete.  Prints medians (us) over warps.

  SKB200_LIB=/tmp/probe.so python scripts/epi_probe.py --m 128 --n 8192 --k 8192 --strategy stream_k
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
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=8192)
    ap.add_argument("--strategy", default="stream_k")
    ap.add_argument("--variant", default="2sm")
    ap.add_argument("--g", type=int, default=0)
    args = ap.parse_args()
    V = {"1sm": sk.Variant.OneSM, "2sm": sk.Variant.TwoSM, "2smw": sk.Variant.TwoSMWide}[args.variant]
    p = 148 if args.variant == "1sm" else 74
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    P = sk.GemmProblem(args.m, args.n, args.k)
    a = {"stream_k": lambda: sk.stream_k(P, blk, args.g or p), "data_parallel": lambda: sk.data_parallel(P, blk),
         "two_tile_sk_dp": lambda: sk.hybrid(P, blk, p, sk.HybridVariant.TwoTileSkDp)}[args.strategy]()
    A = sk.random_matrix_device(args.m, args.k, 1, sk.DType.Float32, sk.DType.BFloat16)
    B = sk.random_matrix_device(args.k, args.n, 2, sk.DType.Float32, sk.DType.BFloat16)
    C = torch.empty(args.m, -(-args.n // 4) * 4, device="cuda")[:, :args.n]
    g = sk.Gemm(a, variant=V, trace=True)
    g.cta_clocks = torch.zeros(148 * 8 * 16, dtype=torch.int64, device="cuda")
    for _ in range(5):
        g.run(A, B, C)
    torch.cuda.synchronize()
    g.cta_clocks.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.run(A, B, C)
    e1.record()
    torch.cuda.synchronize()
    g.check()
    st = g.cta_clocks.view(-1, 16).cpu().numpy().astype(np.float64)
    st = st[st[:, 0] > 0]
    t0 = st[:, 0].min()
    rel = (st - t0) * 1e-3
    rel[st == 0] = np.nan
    out = {"shape": [args.m, args.n, args.k], "strategy": args.strategy, "launch_us": e0.elapsed_time(e1) * 1e3,
           "warps": int(len(st))}
    names = {0: "acc_ready", 15: "peers_seen", 13: "signalled", 14: "stores_done"}
    for s in range(4):
        names[1 + 3 * s], names[2 + 3 * s], names[3 + 3 * s] = f"tmem{s}", f"fold{s}", f"store{s}"
    out["median_us_from_first_acc"] = {names[i]: (None if np.all(np.isnan(rel[:, i])) else
                                                  round(float(np.nanmedian(rel[:, i])), 2)) for i in sorted(names)}
    work = ~np.isnan(rel[:, 3])
    if work.any():
        d = rel[work]
        out["median_phase_us"] = {
            "wait_peers": round(float(np.nanmedian(d[:, 15] - d[:, 0])), 3),
            "tmem_step": round(float(np.nanmedian(d[:, 1] - d[:, 15])), 3),
            "fold_step": round(float(np.nanmedian(d[:, 2] - d[:, 1])), 3),
            "store_step": round(float(np.nanmedian(d[:, 3] - d[:, 2])), 3),
            "step2_total": round(float(np.nanmedian(d[:, 6] - d[:, 3])), 3),
            "signal": round(float(np.nanmedian(d[:, 13] - d[:, 12])), 3) if not np.all(np.isnan(d[:, 12])) else None,
            "drain_stores": round(float(np.nanmedian(d[:, 14] - d[:, 13])), 3),
            "acc_to_end": round(float(np.nanmedian(d[:, 14] - d[:, 0])), 3)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
