"""Summarise ncu --set full reports into profiles/ncu_summary.json.

usage: python scripts/ncu_summary.py <key>=<report.ncu-rep>:<algorithmic bytes per launch> ...
(key = bench workload, e.g. c4; `bench.py` reads dram_bytes_per_launch as the
roofline `traffic`)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__time_duration.sum": "ncu_duration",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__block_size": "block_size",
    "launch__grid_size": "grid_size",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def read(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    res = {"kernel": vals[h.index("Kernel Name")], "report": os.path.basename(rep)}
    for k, name in KEYS.items():
        if k not in h:
            continue
        i = h.index(k)
        v = float(vals[i].replace(",", ""))
        u = units[i]
        if name.startswith("dram_bytes"):
            v *= SCALE.get(u, 1)
        if name == "ncu_duration":
            v *= SCALE.get(u, 1)
            name = "ncu_duration_ms"
        res[name] = v
    return res


def main():
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(path)) if os.path.exists(path) else {}
    for arg in sys.argv[1:]:
        key, rest = arg.split("=", 1)
        rep, alg = rest.rsplit(":", 1)
        r = read(rep)
        r["dram_bytes_per_launch"] = r["dram_bytes_read"] + r["dram_bytes_write"]
        r["algorithmic_bytes_per_launch"] = int(alg)
        r["traffic_over_algorithmic"] = r["dram_bytes_per_launch"] / int(alg)
        r["ncu_achieved_gbs"] = r["dram_bytes_per_launch"] / (r["ncu_duration_ms"] * 1e-3) / 1e9
        summary[key] = r
    json.dump(summary, open(path, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
