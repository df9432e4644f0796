import csv, sys, subprocess
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d["Kernel Name"][:40], d["gpu__time_duration.sum"])
    for k in sorted(hdr):
        sel = (("tensor" in k and "pct" in k and "avg" in k and "ops_path" not in k)
               or ("stalled" in k and "ratio" in k)
               or ("lts__t" in k and "pct" in k and "avg" in k)
               or ("l1tex__throughput.avg.pct" in k))
        if sel:
            try:
                if float(d[k]) > 0.5:
                    print("   ", k, d[k])
            except ValueError:
                pass
