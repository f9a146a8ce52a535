"""Stall-reason totals and the top stalled SASS instructions of one kernel in an ncu report
(source page, --print-source sass; needs --import-source / -lineinfo for line mapping).
    python tools/ncu_stalls.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
i = [k for k, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[i]
data = [r for r in rows[i + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]


def num(x):
    try:
        return int(float(x or 0))
    except ValueError:
        return 0


sc = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in data:
    for k in sc:
        tot[hdr[k]] += num(r[k])
allc = sum(tot.values()) or 1
print("stall totals:", ", ".join(f"{k[6:]} {100 * v / allc:.1f}%" for k, v in tot.most_common(8)))
si = hdr.index("Warp Stall Sampling (All Samples)")
data.sort(key=lambda r: -num(r[si]))
for r in data[:top]:
    reasons = sorted(((num(r[k]), hdr[k][6:]) for k in sc), reverse=True)[:3]
    print(f"{num(r[si]):6d} {r[1][:60]:60s} " + " ".join(f"{n}:{v}" for v, n in reasons if v))
