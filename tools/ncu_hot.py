"""Top stalled SASS instructions of one kernel in an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
r = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = r[0]
rows = []
for x in r[1:]:
    if x and x[0] == "Address":
        break
    if len(x) > 5:
        rows.append(x)
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
tot = sum(float(x[si] or 0) for x in rows)
print(f"total stall samples {tot:.0f}, instructions executed {sum(float(x[ei] or 0) for x in rows):.0f}")
rows.sort(key=lambda x: -float(x[si] or 0))
for x in rows[:top]:
    print(f"{float(x[si]) / tot * 100:5.1f}%  exec {x[ei]:>8s}  {x[1].strip()[:90]}")
