"""Print registers / stack per kernel of a .so (cuobjdump -res-usage), demangled."""
import re, subprocess, sys
out = subprocess.run(["cuobjdump", "-res-usage", sys.argv[1]], capture_output=True, text=True).stdout
lines = out.splitlines()
for i, l in enumerate(lines):
    m = re.match(r"\s*Function (\S+):", l)
    if m and i + 1 < len(lines):
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(anonymous namespace\)::|kmb::|El<[^>]*>::T", "", name)
        name = name.split("(")[0]
        r = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+)", lines[i + 1])
        print(f"REG={r.group(1):>3} STACK={r.group(2):>3}  {name}")
