"""Validate the cluster fixup's non-power-of-two splits against the policy
they replace, on the corpus shapes whose Stream-K policy pick changes.

For every corpus shape (seed 0, FP16, sk_corpus order) the shipped rule
(largest S in {8, 4, 3, 2} that fits as clusters; --all-s: every S in 8..2) is
compared with the round-2 one (S in {8, 4, 2} only, else the cost model's
pick).  Where they differ, a seeded sample of those shapes (--max 0: all) is
timed -- data-parallel, the previous pick and the new pick, same harness as
sweep.py (graphs of >= 8 launches over L2-cold operand copies) -- and the new
pick's C is verified against the reference executor (integer pass bit-exact,
float pass under 8 eps k).

  python scripts/cluster_s_validate.py --variant 1sm --max 300 --out x.jsonl
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402
from paper_2301_03598_b200 import sweep as sw  # noqa: E402


NEW = (8, 4, 3, 2)  # the shipped rule (costmodel.cpp); --all-s: 8..2


def rule(t, ipt, caps, min_iters, candidates):
    for S in candidates:
        ips = -(-ipt // S)
        if (S - 1) * ips >= ipt or ips < min_iters or t * S > caps[S]:
            continue
        return S
    return None


def token(a):
    name = sk.strategy_name(a.strategy)
    if name == "data_parallel":
        return name
    if name == "two_tile_sk_dp":
        return name
    return f"{name}:{a.param}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="1sm", choices=["1sm", "2sm"])
    ap.add_argument("--dtype", default="fp16", choices=["fp16", "bf16"])
    ap.add_argument("--max", type=int, default=300)
    ap.add_argument("--count", type=int, default=32824)
    ap.add_argument("--out", default="")
    ap.add_argument("--all-s", action="store_true", help="new rule over every S in 8..2 (not shipped)")
    args = ap.parse_args()
    global NEW
    if args.all_s:
        NEW = tuple(range(8, 1, -1))
    V = sk.Variant.OneSM if args.variant == "1sm" else sk.Variant.TwoSM
    ab = sk.DType.Float16 if args.dtype == "fp16" else sk.DType.BFloat16
    blk = sk.kernel_blocking(ab, V)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    p = sms if V == sk.Variant.OneSM else sms // 2
    params = sk.default_cost_params(ab, V)
    caps = {S: sk.cluster_capacity(S, V) for S in range(2, 9)}
    model_only = sk.default_cost_params(ab, V)
    model_only.cluster_min_iters = 0.0
    corpus = sk.corpus(0, args.count, 128, 8192)
    changed = []
    for i, r in enumerate(corpus):
        m, n, k, seed = (int(x) for x in r[:4])
        pr = sk.GemmProblem(m, n, k)
        g = sk.tile_grid(pr, blk)
        t, ipt = g.total_tiles, g.iters_per_tile
        new = rule(t, ipt, caps, params.cluster_min_iters, NEW)
        old = rule(t, ipt, caps, params.cluster_min_iters, (8, 4, 2))
        if new == old:
            continue
        if not args.all_s:  # the library's policy is the rule restated here
            a_new = sk.auto_stream_k(pr, blk, p, params)
            assert (a_new.strategy, a_new.param) == (sk.Strategy.FixedSplit, new), (m, n, k)
        old_tok = f"fixed_split:{old}" if old else token(sk.auto_stream_k(pr, blk, p, model_only))
        changed.append((i, m, n, k, seed, old_tok, f"fixed_split:{new}"))
    print(json.dumps({"caps": caps, "shapes": len(corpus), "changed": len(changed)}), flush=True)
    rng = np.random.default_rng(7)
    size = len(changed) if args.max <= 0 else min(args.max, len(changed))
    pick = sorted(rng.choice(len(changed), size=size, replace=False))
    ver = sw.Verifier(torch, args.dtype)
    out = open(args.out, "w") if args.out else None
    sp_old, sp_dp, fails = [], [], 0
    for j in pick:
        i, m, n, k, seed, old_tok, new_tok = changed[j]
        pr = sk.GemmProblem(m, n, k)
        timer = sw.ShapeTimer(torch, m, n, k, args.dtype, seed)
        times, jobs = {}, []
        names = ["data_parallel", old_tok, new_tok]
        for name, a in zip(names, sw.strategies_for(pr, blk, p, names, params)):
            gemm = sk.Gemm(a, ab, V)
            times[name] = timer.time_us(gemm)
            if name == new_tok:
                jobs.append((name, a, gemm))
        del timer
        chk = ver.shape(m, n, k, seed, jobs)[new_tok]
        fails += chk["verified"] != "pass"
        rec = {"idx": i, "shape": [m, n, k], "old": old_tok, "new": new_tok,
               "us": {kk: round(v, 2) for kk, v in times.items()},
               "new_vs_old": times[old_tok] / times[new_tok],
               "new_vs_dp": times["data_parallel"] / times[new_tok],
               "verified": chk["verified"], "max_rel_err": chk["max_rel_err"]}
        sp_old.append(rec["new_vs_old"])
        sp_dp.append(rec["new_vs_dp"])
        if out:
            out.write(json.dumps(rec) + "\n")
            out.flush()
    gm = lambda x: float(np.exp(np.mean(np.log(x)))) if x else None  # noqa: E731
    print(json.dumps({"variant": args.variant, "dtype": args.dtype, "changed": len(changed),
                      "timed": len(sp_old), "geomean_new_vs_old": gm(sp_old),
                      "min_new_vs_old": min(sp_old, default=None),
                      "new_slower_than_old_gt_5pct": int(sum(s < 0.95 for s in sp_old)),
                      "geomean_new_vs_dp": gm(sp_dp), "min_new_vs_dp": min(sp_dp, default=None),
                      "new_slower_than_dp_gt_5pct": int(sum(s < 0.95 for s in sp_dp)),
                      "verify_failures": fails}), flush=True)


if __name__ == "__main__":
    main()
