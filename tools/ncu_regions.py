"""Warp-stall samples of one kernel binned by SASS address, with the notable instructions of
each bin (DMMA count, barriers, TMA, global stores), to tell the main loop from the prologue,
the epilogue and the stream-K fix-up:

    python tools/ncu_regions.py source.csv[.gz] [bin_bytes]
"""
import collections
import csv
import gzip
import io
import re
import sys


def main(path, bin_bytes=0x400):
    raw = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
    for block in re.split(r'^"Kernel Name",', raw, flags=re.M)[1:]:
        name, body = block.split("\n", 1)
        rows = list(csv.reader(io.StringIO(body)))
        h = rows[0]
        i_s = h.index("Warp Stall Sampling (All Samples)")
        i_a = h.index("Address")
        reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        good = [r for r in rows[1:] if len(r) == len(h)]
        tot = sum(int(r[i_s] or 0) for r in good) or 1
        base = int(good[0][i_a], 16)
        bins = collections.OrderedDict()
        for r in good:
            b = (int(r[i_a], 16) - base) // bin_bytes
            e = bins.setdefault(b, {"n": 0, "ops": collections.Counter(), "rs": collections.Counter()})
            s = int(r[i_s] or 0)
            e["n"] += s
            op = r[1].strip().split()
            op = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
            e["ops"][op.split(".")[0] + ("." + op.split(".")[1] if op.startswith(("SYNCS", "UTMA")) else "")] += 1
            for c in reasons:
                e["rs"][c[6:]] += int(r[h.index(c)] or 0)
        print(name[:100], "samples", tot)
        for b, e in bins.items():
            if e["n"] * 200 < tot:
                continue
            notable = {k: v for k, v in e["ops"].items()
                       if k.startswith(("DMMA", "SYNCS", "UTMA", "STG", "LDG", "BAR", "ERRBAR", "MEMBAR", "RED", "ATOM"))}
            print(f"  +{b * bin_bytes:06x} {100 * e['n'] / tot:5.1f}%  {dict(notable)}  "
                  f"{[(k, round(100 * v / max(e['n'], 1))) for k, v in e['rs'].most_common(3)]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2], 0) if len(sys.argv) > 2 else 0x400)
