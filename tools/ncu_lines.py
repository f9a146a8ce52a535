"""Per-source-line stall samples / executed instructions of one kernel (ncu --print-source cuda,sass)."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
stats = collections.OrderedDict()
fname, hdr, cur = "?", None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a source line row
        cur = (fname, r[0], r[1].strip()[:90])
        stats.setdefault(cur, [0.0, 0.0])
        continue
    try:
        a = stats.setdefault(cur, [0.0, 0.0])
        a[0] += float(r[4] or 0)
        a[1] += float(r[7] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in stats.values()) or 1
for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}%  inst {v[1]:9.0f}  {k[0]}:{k[1]}: {k[2]}")
