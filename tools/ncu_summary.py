"""Condense ncu outputs into profiles/ summaries.

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.json> [kernel-regex]
"""
import csv
import json
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "launch__grid_size",
    "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__shared_mem_per_block_dynamic",
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def launches(path, out):
    rows = list(csv.DictReader(line for line in open(path) if line.startswith('"')))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"])[:90]
        v = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else
                                        1.0 if r["Metric Unit"] == "us" else 1e3)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({path}), gpu__time_duration.sum, --clock-control none\n\n")
        f.write("Cold-cache, serialised per-launch times: compare shares, not absolutes.\n\n")
        f.write("| kernel | launches | total us | share |\n|---|---|---|---|\n")
        for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{name}` | {n} | {us:.1f} | {us / tot:.1%} |\n")
    print(open(out).read())


def full(path, out, regex=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, zip(units, vals)))
        name = d.get("Kernel Name", ("", ""))[1]
        if regex and not re.search(regex, name):
            continue
        rec = {"kernel": name}
        for k in KEYS:
            if k in d:
                u, v = d[k]
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                if u in SCALE:
                    x *= SCALE[u]
                    u = "byte"
                rec[k] = x
                rec[k + ".unit"] = u
        rb = rec.get("dram__bytes_read.sum", 0.0) + rec.get("dram__bytes_write.sum", 0.0)
        rec["dram_bytes_per_launch"] = rb
        res.append(rec)
    with open(out, "w") as f:
        json.dump(res[0] if len(res) == 1 else res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
