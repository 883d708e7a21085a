"""Summarise an ncu --set full capture into profiles/ (details CSV + key metrics JSON).

usage: python scripts/export_ncu.py <report.ncu-rep> <out_prefix>
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    summary = {"kernel": d.get("Kernel Name"), "metrics": {}}
    for k in KEYS:
        if k in d:
            summary["metrics"][k] = {"value": d[k], "unit": u.get(k, "")}
    for k in d:  # tensor sub-pipes (UTCIMMA / UTCHMMA activity)
        if "pipe_tensor" in k and ("pct" in k or k.endswith(".avg")):
            summary["metrics"][k] = {"value": d[k], "unit": u.get(k, "")}
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
              for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v}
    tot = sum(stalls.values()) or 1.0
    summary["stall_pct"] = {k: round(100 * v / tot, 1)
                            for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    json.dump(summary, open(out + "_summary.json", "w"), indent=1)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    open(out + "_details.csv", "w").write(det)
    print(json.dumps(summary)[:600])


if __name__ == "__main__":
    main()
