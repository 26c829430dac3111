"""Merge sweep CSV parts (e.g. corpus chunks run as --offset/--count calls) into
one gzipped CSV in corpus order and print the summary the sweep prints for a
single run: Stream-K policy vs data-parallel geomean, shapes more than 5 %
slower, verification counts, the reference CPU executor's time.

  python scripts/corpus_merge.py --out profiles/r02/corpus_full.csv.gz part0.csv part1.csv ...
"""
import argparse
import csv
import gzip
import io
import json
import math


def read_rows(path):
    with open(path) as f:
        lines = f.read().splitlines()
    assert lines[0] == "# schema=1", path
    return lines[1], list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--baseline", default="data_parallel")
    ap.add_argument("--policy", default="stream_k:auto")
    ap.add_argument("parts", nargs="+")
    args = ap.parse_args()
    header, rows = None, []
    for p in args.parts:
        h, r = read_rows(p)
        header = header or h
        assert h == header, p
        rows += r
    with gzip.open(args.out, "wt") as f:
        f.write("# schema=1\n" + header + "\n")
        w = csv.DictWriter(f, fieldnames=header.split(","), lineterminator="\n")
        for r in rows:
            w.writerow(r)
    by_shape = {}
    for r in rows:
        by_shape.setdefault((int(r["m"]), int(r["n"]), int(r["k"])), {})[r["policy"]] = float(r["measured_time"])
    sp = [d[args.baseline] / d[args.policy] for d in by_shape.values()
          if args.baseline in d and args.policy in d]
    worst = sorted(((d[args.baseline] / d[args.policy], s) for s, d in by_shape.items()
                    if args.baseline in d and args.policy in d))[:5]
    cpu = [r for r in rows if r.get("cpu_time_s")]
    out = {
        "rows": len(rows), "shapes": len(by_shape),
        args.policy: {"geomean_speedup": math.exp(sum(math.log(x) for x in sp) / len(sp)),
                      "min": min(sp), "max": max(sp), "regress_gt_5pct": sum(x < 0.95 for x in sp),
                      "worst": [[round(x, 4), list(s)] for x, s in worst]},
        "verified_rows": sum(r["verified"] == "pass" for r in rows),
        "failed_rows": sum(r["verified"] == "FAIL" for r in rows),
        "int_exact_rows": sum(r["int_exact"] == "1" for r in rows),
        "float_full_rows": sum(r["float_check"] == "full" for r in rows),
        "float_sampled_rows": sum(r["float_check"].startswith("rows") for r in rows),
        "max_rel_err": max(float(r["max_rel_err"]) for r in rows if r["max_rel_err"]),
        "cpu_reference": {"rows": len(cpu), "seconds": sum(float(r["cpu_time_s"]) for r in cpu),
                          "threads": cpu[0]["cpu_threads"] if cpu else None,
                          "model": cpu[0]["cpu_model"] if cpu else None,
                          "tflops_geomean": math.exp(sum(
                              math.log(2.0 * int(r["m"]) * int(r["n"]) * int(r["k"]) /
                                       float(r["cpu_time_s"]) / 1e12) for r in cpu) / len(cpu))
                          if cpu else None},
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
