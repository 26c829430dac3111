"""In-process A/B of library knobs read from the environment at launch time
(SKB200_DIE_AWARE, SKB200_RASTER_ROWS, SKB200_L2_POLICY, ...), alternating the
settings ROUNDS times on the same box so power/thermal drift hits all arms.

  python scripts/ab_env.py --set SKB200_DIE_AWARE=0 --set SKB200_DIE_AWARE=1 \
      [--strategy data_parallel] [--m 8192 --n 8192 --k 8192] [--steps 30 --rounds 4]
Each --set is one arm: comma-separated VAR=VALUE pairs (TILE_GROUP=G sets the
descriptor's tile_group instead of an environment variable).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", action="append", required=True)
    ap.add_argument("--strategy", default="two_tile_sk_dp")
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--k", type=int, default=8192)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--g", type=int, default=74, help="stream_k grid / hybrid p")
    ap.add_argument("--variant", default="2sm", choices=["1sm", "2sm", "2smw"])
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--no-check", action="store_true",
                    help="arms may legitimately differ in float rounding (e.g. k order)")
    ap.add_argument("--cool", type=float, default=1.0, help="idle seconds before each measurement "
                    "(every arm then starts from the same power/thermal state)")
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    ab = sk.DType.BFloat16 if args.dtype == "bf16" else sk.DType.Float16
    tdt = torch.bfloat16 if args.dtype == "bf16" else torch.float16
    pad = lambda x, q: (x + q - 1) // q * q  # noqa: E731  16-byte rows for TMA
    A = (torch.rand(m, pad(k, 8), device="cuda") * 2 - 1).to(tdt)[:, :k]
    B = (torch.rand(k, pad(n, 8), device="cuda") * 2 - 1).to(tdt)[:, :n]
    C = torch.empty(m, pad(n, 4), device="cuda", dtype=torch.float32)[:, :n]
    V = {"1sm": sk.Variant.OneSM, "2sm": sk.Variant.TwoSM, "2smw": sk.Variant.TwoSMWide}[args.variant]
    blk = sk.kernel_blocking(ab, V)
    prob = sk.GemmProblem(m, n, k)
    if args.strategy == "data_parallel":
        a = sk.data_parallel(prob, blk)
    elif args.strategy == "stream_k":
        a = sk.stream_k(prob, blk, args.g)
    else:
        a = sk.hybrid(prob, blk, args.g, sk.HybridVariant.TwoTileSkDp)
    g = sk.Gemm(a, ab, V)
    stream = torch.cuda.current_stream()
    flops = 2.0 * m * n * k
    def parse_arm(spec):  # VAR=VALUE pairs separated by commas; values may contain commas
        pairs = []
        for tok in spec.split(","):
            if "=" in tok or not pairs:
                pairs.append(tok)
            else:
                pairs[-1] += "," + tok
        return dict(kv.split("=", 1) for kv in pairs)

    arms = [parse_arm(s) for s in args.set]
    res = [[] for _ in arms]
    ref = None
    for _ in range(args.rounds):
        for i, env in enumerate(arms):
            for key in {kk for e in arms for kk in e}:  # each arm sets only its own knobs
                os.environ.pop(key, None)
            os.environ.update({kk: v for kk, v in env.items() if kk != "TILE_GROUP"})
            sk.reload_env()  # the library reads SKB200_* once
            g.desc.tile_group = int(env.get("TILE_GROUP", "0"))  # sk_gemm_desc field, not a knob
            torch.cuda.synchronize()
            time.sleep(args.cool)
            for _ in range(args.warmup):
                g.run(A, B, C)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                g.run(A, B, C)
            e1.record(stream)
            torch.cuda.synchronize()
            g.check()
            ms = e0.elapsed_time(e1) / args.steps
            res[i].append(round(flops / (ms * 1e-3) / 1e12, 1))
            cs = float(C.double().sum())
            if ref is None:
                ref = cs
            elif cs != ref and not args.no_check:  # deterministic: bit-identical C across arms
                raise SystemExit(f"checksum mismatch for {env}: {cs} vs {ref}")
    print(json.dumps({"shape": [m, n, k], "strategy": args.strategy,
                      "arms": [{"env": env, "tflops": r, "median": float(np.median(r))}
                               for env, r in zip(arms, res)]}))


if __name__ == "__main__":
    main()
