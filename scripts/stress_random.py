"""Randomised bit-exactness stress of the device paths (integer-valued operands
vs an fp64 reference product): every decomposition with random knobs, shapes up
to 3000 x 3000 with k up to 16384 (deep-k, few-tile cases exercise the
cooperative fixup), both tcgen05 variants and FP64, pageable and pinned host
buffers (the tile-block transfer pipeline).

  python scripts/stress_random.py [--trials 40] [--seed 5]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2301_03598_b200 as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=40)
    ap.add_argument("--seed", type=int, default=5)
    args = ap.parse_args()
    port = oracle.Oracle("port")
    rng = np.random.default_rng(args.seed)
    bad = runs = 0
    for var in ("2sm", "1sm", "fp64"):
        if var == "fp64":
            ab, V, dt, ht = sk.DType.Float64, sk.Variant.Auto, np.float64, np.float64
        else:
            ab = sk.DType.BFloat16
            V = sk.Variant.TwoSM if var == "2sm" else sk.Variant.OneSM
            dt, ht = np.float32, np.float16
        blk = sk.kernel_blocking(ab, V)
        for trial in range(args.trials):
            m, n = (int(x) for x in rng.integers(1, 3000, 2))
            k = int(rng.integers(1, 16384)) if trial % 3 == 0 else int(rng.integers(1, 2500))
            if var == "fp64":
                m, n, k = max(1, m // 3), max(1, n // 3), max(1, k // 4)
            A = port.random_matrix(m, k, int(rng.integers(1 << 40)), "int64") >> 3
            B = port.random_matrix(k, n, int(rng.integers(1 << 40)), "int64") >> 3
            want = (A.astype(np.float64) @ B.astype(np.float64)).astype(dt)
            P = sk.GemmProblem(m, n, k)
            p = 74 if var == "2sm" else 148
            cands = [sk.data_parallel(P, blk), sk.fixed_split(P, blk, int(rng.integers(1, 6))),
                     sk.stream_k(P, blk, int(rng.integers(1, p + 1))),
                     sk.stream_k(P, blk, int(rng.integers(1, 4 * p))),
                     sk.hybrid(P, blk, p, sk.HybridVariant.TwoTileSkDp),
                     sk.hybrid(P, blk, int(rng.integers(1, p + 1)), sk.HybridVariant.DpOneTileSk)]
            pinned = trial % 2 == 0 and var != "fp64"
            if pinned:
                At = torch.empty((m, k), dtype=torch.float16, pin_memory=True)
                Bt = torch.empty((k, n), dtype=torch.float16, pin_memory=True)
                Ct = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
                At.numpy()[...] = A.astype(ht)
                Bt.numpy()[...] = B.astype(ht)
            for a in cands:
                if pinned:
                    got = sk.execute(a, At.numpy(), Bt.numpy(), compute=sk.DType.Float16, variant=V,
                                     out=Ct.numpy())
                else:
                    got = sk.execute(a, A.astype(dt), B.astype(dt), compute=ab, variant=V)
                runs += 1
                if not np.array_equal(got, want):
                    bad += 1
                    print("MISMATCH", var, m, n, k, sk.strategy_name(a.strategy), a.param, pinned, flush=True)
        print(var, "done", flush=True)
    print(f"stress: {runs} runs, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
