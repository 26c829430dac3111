"""DRAM bytes per launch vs algorithmic bytes for the skinny shapes, from the
ncu launch list of scripts/skinny_launch.py (see scripts/closing_run.sh):

  python scripts/skinny_traffic.py profiles/<run>/skinny_ncu_1sm.csv profiles/<run>/skinny_launch_1sm.json

Prints one JSON list: per shape the median ncu duration and DRAM bytes (read +
write) over its launches, and traffic / algorithmic (A + B + C bytes)."""
import csv
import json
import statistics
import sys


def main(csv_path, launch_path):
    with open(launch_path) as f:
        shapes = json.load(f)
    per_launch = {}
    with open(csv_path) as f:
        rows = [r for r in csv.reader(f) if len(r) > 14 and r[0].isdigit()]
    for r in rows:
        per_launch.setdefault(int(r[0]), {})[r[12]] = float(r[14].replace(",", ""))
    ids = sorted(per_launch)
    out, i = [], 0
    for s in shapes:
        got = [per_launch[j] for j in ids[i:i + s["launches"]]]
        i += s["launches"]
        dram = statistics.median(g["dram__bytes_read.sum"] + g["dram__bytes_write.sum"] for g in got)
        t = statistics.median(g["gpu__time_duration.sum"] for g in got)
        out.append({"shape": s["shape"], "strategy": s["strategy"], "param": s["param"],
                    "ncu_time_us": round(t / 1e3, 1), "dram_bytes": dram,
                    "algorithmic_bytes": s["algorithmic_bytes"],
                    "traffic_over_algorithmic": round(dram / s["algorithmic_bytes"], 3)})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
