"""Per-kernel stall summary of an ncu report captured with --import-source on:
stall reasons, samples by opcode, and the hottest non-math instructions.

    python tools/ncu_stalls.py report.ncu-rep [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(rep, top=25):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    for block in re.split(r'^"Kernel Name",', raw, flags=re.M)[1:]:
        name, body = block.split("\n", 1)
        rows = list(csv.reader(io.StringIO(body)))
        h = rows[0]
        i_s = h.index("Warp Stall Sampling (All Samples)")
        reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        good = [r for r in rows[1:] if len(r) == len(h)]
        tot = sum(int(r[i_s] or 0) for r in good) or 1
        rs = collections.Counter()
        ops = collections.Counter()
        for r in good:
            for c in reasons:
                rs[c] += int(r[h.index(c)] or 0)
            op = r[1].strip().split()
            op = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
            ops[op.split(".")[0]] += int(r[i_s] or 0)
        print(name[:110], "samples", tot)
        print("  reasons:", [(k, round(100 * v / tot, 1)) for k, v in rs.most_common(8)])
        print("  opcodes:", [(k, round(100 * v / tot, 1)) for k, v in ops.most_common(10)])
        hot = sorted(good, key=lambda r: -int(r[i_s] or 0))[:top]
        for r in hot:
            stalls = sorted(((int(r[h.index(c)] or 0), c[6:]) for c in reasons), reverse=True)[:2]
            print("   %5.2f%% %-60s %s" % (100 * int(r[i_s]) / tot, r[1].strip()[:60], stalls))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
