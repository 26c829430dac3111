"""Fit the grid-size model (csrc/costmodel.cpp) on a calibration sweep CSV
(`python -m paper_2301_03598_b200.sweep --strategies data_parallel,stream_k:cal`)
and report selection quality over the measured candidates.

    python scripts/fit_costmodel.py <cal.csv> [--p 74] [--margin 0.15] [--out profiles/r01/costmodel.json]
"""
import argparse
import collections
import csv
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03598_b200 as sk  # noqa: E402


def load(path):
    return list(csv.DictReader(l for l in open(path) if not l.startswith("#")))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--p", type=int, default=74)
    ap.add_argument("--margin", type=float, default=0.15)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rows = load(a.csv)
    samples = []
    for r in rows:
        if r["strategy"] == "data_parallel" or r["strategy"].startswith("stream_k:"):
            t, ipt = int(r["t"]), int(r["iters_per_tile"])
            grid = sk.TileGrid(int(r["tiles_m"]), int(r["tiles_n"]), t, ipt, t * ipt)
            samples.append((grid, int(r["g"]), float(r["time_us"]), r))
    params = sk.calibrate([s[:3] for s in samples], a.p, a.margin,
                          coop_peers=sk.default_cost_params().coop_peers)
    by = collections.defaultdict(list)
    for grid, g, t, r in samples:
        by[(r["m"], r["n"], r["k"])].append((sk.predict_time(params, grid, g, a.p), t, r["strategy"]))
    sp, reg, picked = [], 0, 0
    for lst in by.values():
        pdp, tdp = [(x[0], x[1]) for x in lst if x[2] == "data_parallel"][0]
        cand = min(x for x in lst if x[2] != "data_parallel")
        s = tdp / cand[1] if cand[0] < (1 - a.margin) * pdp else 1.0
        picked += s != 1.0
        sp.append(s)
        reg += s < 0.95
    best = [max(1.0, max(l, key=lambda x: -x[1])[1] and min(x[1] for x in l if x[2] == "data_parallel")
                / min(x[1] for x in l)) for l in by.values()]
    out = {"params": params.as_dict(), "samples": len(samples), "shapes": len(by), "p": a.p,
           "selection_over_measured": {"geomean_speedup_vs_dp": float(np.exp(np.mean(np.log(sp)))),
                                       "regress_gt_5pct": int(reg), "picked_stream_k": int(picked)},
           "oracle_best_of_measured_geomean": float(np.exp(np.mean(np.log(best)))),
           "source": a.csv}
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
