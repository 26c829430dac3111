"""Launch the Stream-K policy's pick for the bench's skinny shapes, R times each
(for an ncu launch list: DRAM bytes per launch vs the algorithmic bytes).

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:sk_gemm --csv python scripts/skinny_launch.py --variant 1sm
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402
from paper_2301_03598_b200 import sweep as sw  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="2sm", choices=["1sm", "2sm"])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    V = sk.Variant.OneSM if args.variant == "1sm" else sk.Variant.TwoSM
    p = 148 if args.variant == "1sm" else 74
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    out = []
    for m, n, k in sw.SKINNY[:2] + sw.SKINNY[4:6]:
        a = sk.auto_stream_k(sk.GemmProblem(m, n, k), blk, p)
        A = sk.random_matrix_device(m, k, 42, sk.DType.Float32, sk.DType.BFloat16)
        B = sk.random_matrix_device(k, n, 43, sk.DType.Float32, sk.DType.BFloat16)
        C = torch.empty(m, n, device="cuda")
        g = sk.Gemm(a, variant=V)
        for _ in range(args.reps):
            g.run(A, B, C)
        g.check()
        out.append({"shape": [m, n, k], "strategy": sk.strategy_name(a.strategy), "param": a.param,
                    "algorithmic_bytes": sw.algorithmic_bytes(m, n, k, "bf16"), "launches": args.reps})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
