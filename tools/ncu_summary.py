"""Summarise an ncu report into profiles/: per-kernel duration, DRAM bytes,
throughput %, occupancy, L1/L2 hit rates; and update profiles/ncu_latest.json
(dram bytes per work unit, used by bench.py for the roofline `traffic`).

    python tools/ncu_summary.py REPORT.ncu-rep KERNEL_REGEX UNITS OUT_TXT [CONFIG_KEY]

CONFIG_KEY (e.g. c2:n=1000000:nq=10000) names the workload the capture ran;
bench.py takes `traffic` only from records of its own workload.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def main(rep, pattern, units, out_txt, config=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, unit_row = rows[0], rows[1]
    col = {h: i for i, h in enumerate(head)}
    lines = []
    summary = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        if not re.search(pattern, name):
            continue
        rec = {}
        for w in WANT:
            if w in col:
                v = r[col[w]].replace(",", "")
                try:
                    x = float(v)
                    x *= SCALE.get(unit_row[col[w]], 1)
                except ValueError:
                    x = v
                rec[w] = x
        short = re.sub(r"<.*", "", re.sub(r"\(.*", "", name).split("::")[-1])  # template args dropped
        lines.append(f"{short}: " + ", ".join(f"{k}={v}" for k, v in rec.items()))
        dram = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
        if short in summary and summary[short]["duration_ms"] >= rec.get("gpu__time_duration.sum", 0):
            continue  # several launches of one kernel: keep the longest (the full-size one)
        summary[short] = {"dram_bytes": dram, "duration_ms": rec.get("gpu__time_duration.sum"),
                          "dram_bytes_per_unit": dram / float(units),
                          "source": os.path.basename(out_txt), "config": config}
    # records are kept per (kernel, workload): {kernel: {config: record}}
    with open(out_txt, "w") as f:
        f.write(f"# ncu summary of {os.path.basename(rep)} (units per launch = {units})\n")
        f.write("\n".join(lines) + "\n")
    latest = os.path.join(ROOT, "profiles", "ncu_latest.json")
    cur = {}
    if os.path.exists(latest):
        cur = json.load(open(latest))
    for kname, rec in summary.items():
        cur.setdefault(kname, {})[str(rec["config"])] = rec
    json.dump(cur, open(latest, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else None)
