"""Measure the tensor-pipe roofline denominators on this B200 with sampled clocks.

Runs tools/probes/tc_peak (fp64 DMMA and tcgen05 kind::i8 at N = 64 / 128 / 256) while
bench.ClockSampler polls nvidia-smi, and writes profiles/<out>.json. bench.py reads the DMMA
figure as the fp64 peak and the kind::i8 N = 64 figure as the Ozaki GEMM's peak (its MMA shape).

  python tools/tc_peaks.py [--out profiles/r02_tc_peaks.json]
"""
import argparse
import datetime
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_tc_peaks.json"))
    ap.add_argument("--bin", default=os.path.join(ROOT, "tools", "probes", "tc_peak"))
    a = ap.parse_args()
    with ClockSampler(0) as cs:
        r = subprocess.run([a.bin], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    if r.returncode:
        sys.exit(r.returncode)
    dmma = float(re.search(r"DMMA.m8n8k4 ([\d.]+) TFLOP/s", r.stdout).group(1))
    i8 = {f"n{m.group(1)}_acc{m.group(2)}": float(m.group(3))
          for m in re.finditer(r"I8 N=(\d+) accum=(\d+)\s+([\d.]+) TOP/s", r.stdout)}
    n64 = max(v for k, v in i8.items() if k.startswith("n64_"))
    out = {"what": "measured tensor-pipe throughput on one B200 (tools/probes/tc_peak.cu, best of 5 launches "
                   "each; clocks sampled with nvidia-smi every 20 ms over the whole run)",
           "dmma_tflops": dmma, "i8_tops": i8, "i8_n64_tops": n64, "i8_best_tops": max(i8.values()),
           "clocks": cs.summary(), "raw": r.stdout.strip().splitlines(),
           "date": datetime.date.today().isoformat()}
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("dmma_tflops", "i8_n64_tops", "i8_best_tops", "clocks")}))


if __name__ == "__main__":
    main()
