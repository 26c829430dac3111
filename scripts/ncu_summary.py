"""Summarise ncu captures into profiles/ (committed evidence).

    python scripts/ncu_summary.py <tag> <workload> <rep> [<workload> <rep> ...]

Writes profiles/<tag>/<name>.raw.csv (ncu --page raw), appends/updates
profiles/ncu_summary.json keyed by bench workload (bench.py reads
dram_bytes_per_launch from it for roofline.traffic), and prints a table."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__cluster_size": "cluster",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "smem_st_bank_conflicts",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
         "ms": 1e-3, "s": 1, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                out[KEYS[h]] = v
                continue
            out[KEYS[h]] = x * SCALE.get(u, 1.0)
    return raw, out


def main():
    tag = sys.argv[1]
    pairs = sys.argv[2:]
    os.makedirs(os.path.join(ROOT, "profiles", tag), exist_ok=True)
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(path)) if os.path.exists(path) else {}
    for workload, rep in zip(pairs[0::2], pairs[1::2]):
        raw, s = summarise(rep)
        name = os.path.basename(rep).replace(".ncu-rep", "")
        with open(os.path.join(ROOT, "profiles", tag, name + ".raw.csv"), "w") as f:
            f.write(raw)
        s["dram_bytes_per_launch"] = s.get("dram_read", 0) + s.get("dram_write", 0)
        s["source"] = f"profiles/{tag}/{name}.raw.csv (ncu --set full --clock-control none)"
        summary[workload] = s
        print(workload, json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in s.items()}))
    with open(path, "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
