"""Summarise an ncu --set full report and an ncu launch list into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_r01.ncu-rep gpurun_out/launches.csv profiles/r01
writes <prefix>_ncu_full.csv (selected metrics per profiled launch),
<prefix>_launches.csv (per-kernel share of the launch list) and updates
profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep, launches, prefix):
    hdr, units, data = raw_rows(rep)
    sel = []
    for r in data:
        if len(r) != len(hdr):
            continue
        rec = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                rec[m] = r[i]
                if units[i] in SCALE:
                    rec[m + ".bytes"] = float(r[i].replace(",", "")) * SCALE[units[i]]
        sel.append(rec)
    with open(prefix + "_ncu_full.csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=sorted({k for rec in sel for k in rec}, key=lambda k: (k != "kernel", k)))
        w.writeheader()
        w.writerows(sel)
    traffic = [rec.get("dram__bytes_read.sum.bytes", 0) + rec.get("dram__bytes_write.sum.bytes", 0) for rec in sel]
    # launch list shares
    rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
    h = rows[0]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        k = r[h.index("Kernel Name")].split("(")[0]
        tot[k] += float(r[h.index("Metric Value")].replace(",", ""))
        cnt[k] += 1
    total = sum(tot.values())
    with open(prefix + "_launches.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_ns", "mean_ns", "share"])
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            w.writerow([k, cnt[k], int(v), int(v / cnt[k]), f"{v / total:.4f}"])
    summary = {
        "report": os.path.basename(rep),
        "dram_bytes_per_launch": sum(traffic) / len(traffic) if traffic else None,
        "dram_bytes_per_launch_each": traffic,
        "kernels": sel,
        "launch_shares": {k: tot[k] / total for k in tot},
    }
    with open(os.path.join(os.path.dirname(prefix), "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: summary[k] for k in ("dram_bytes_per_launch", "launch_shares")}, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
