"""Per-kernel evidence table from an `ncu --set full` capture of tools/profile_kernels.py.

    python tools/kernel_evidence.py gpurun_out/kernels.ncu-rep profiles/r01d_kernels
writes <prefix>.json and <prefix>.md: duration, DRAM bytes and GB/s, and the
pipe utilisation that bounds each kernel (DMMA / tensor / fp64 / issue).
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
KEEP = [
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum",
]


def main(rep, prefix, peak_gbs=6550.1):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    tensor_cols = [h for h in hdr if ("tensor" in h or "tmem" in h or "utc" in h.lower())
                   and h.endswith("pct_of_peak_sustained_active")]

    def val(r, m):
        i = hdr.index(m)
        v = float(r[i].replace(",", ""))
        return v * SCALE.get(units[i], 1.0)

    recs = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        name = r[hdr.index("Kernel Name")]
        rec = {"kernel": name.split("(")[0]}
        t = val(r, "gpu__time_duration.sum")
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        rec.update({"duration_us": t * 1e6, "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6,
                    "dram_GBps": (rd + wr) / t / 1e9, "dram_frac_of_measured_peak": (rd + wr) / t / 1e9 / peak_gbs})
        for m in KEEP:
            if m in hdr:
                rec[m] = val(r, m)
        rec["tensor_metrics_pct_active"] = {h: val(r, h) for h in tensor_cols if val(r, h) > 0.5}
        recs.append(rec)
    json.dump({"report": rep, "hbm_peak_GBps": peak_gbs, "kernels": recs}, open(prefix + ".json", "w"), indent=1)
    lines = ["| kernel | grid×block | µs | DRAM MB (r+w) | DRAM GB/s (frac of 6550) | DMMA pipe % | tensor pipe % | issue % |",
             "|---|---|---|---|---|---|---|---|"]
    for rec in recs:
        lines.append("| {} | {}×{} | {:.1f} | {:.1f} | {:.0f} ({:.2f}) | {} | {} | {} |".format(
            rec["kernel"].replace("void ", ""), int(rec.get("launch__grid_size", 0)), int(rec.get("launch__block_size", 0)),
            rec["duration_us"], rec["dram_read_MB"] + rec["dram_write_MB"], rec["dram_GBps"],
            rec["dram_frac_of_measured_peak"],
            "%.1f" % rec.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 0),
            "%.1f" % rec.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0),
            "%.1f" % rec.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0)))
    open(prefix + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
