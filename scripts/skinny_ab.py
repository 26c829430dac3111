"""Skinny (HBM-bound) shapes: GB/s per (variant, schedule, fixup protocol).

  python scripts/skinny_ab.py [--shapes bench|all] [--coop -1,0,1]
Prints one JSON line per (shape, variant, coop, strategy) with time and the
fraction of the measured HBM peak (algorithmic A + B + C bytes / time)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2301_03598_b200 as sk  # noqa: E402
from paper_2301_03598_b200 import sweep as sw  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="bench")
    ap.add_argument("--coop", default="-1,1")
    ap.add_argument("--variants", default="1sm,2sm")
    ap.add_argument("--strategies", default="data_parallel,stream_k:auto,stream_k")
    args = ap.parse_args()
    shapes = sw.SKINNY[:2] + sw.SKINNY[4:6] if args.shapes == "bench" else sw.SKINNY
    if args.shapes not in ("bench", "all"):
        shapes = [tuple(int(x) for x in s.split("x")) for s in args.shapes.split(",")]
    hbm = 6545.3
    for var in args.variants.split(","):
        V = sk.Variant.OneSM if var == "1sm" else sk.Variant.TwoSM
        p = 148 if var == "1sm" else 74
        names = [n if n != "stream_k:half" else f"stream_k:{p // 2}" for n in args.strategies.split(",")]
        for coop in args.coop.split(","):
            if coop == "-1":
                os.environ.pop("SKB200_COOP", None)
            else:
                os.environ["SKB200_COOP"] = coop
            sk.reload_env()
            rows = sw.run(shapes, names, V, "bf16")
            for r in rows:
                print(json.dumps({"shape": [r["m"], r["n"], r["k"]], "variant": var, "coop": int(coop),
                                  "strategy": r["strategy"], "g": r["g"], "time_us": round(r["time_us"], 2),
                                  "gbps": round(r["gbps"], 1), "frac": round(r["gbps"] / hbm, 3)}), flush=True)


if __name__ == "__main__":
    main()
