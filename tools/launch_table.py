"""Summarise an ncu --metrics gpu__time_duration.sum launch list: one Newton iteration
(from k_seed_jet to the LU kernel) of the captured graph, per-kernel device time."""
import csv
import io
import sys


def load(path):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    seq = []
    for r in rows:
        n = r["Kernel Name"]
        short = n.split("(")[0].replace("nlrom::", "").replace("void ", "")
        for tag in ["EpiJetOut", "EpiJet", "EpiBwdAct", "EpiStore", "EpiAct"]:
            if tag in n:
                short = "gemm<" + tag + ">"
                break
        seq.append((short, float(r["Metric Value"]) / 1000, r["Grid Size"], r["Block Size"]))
    return seq


def iteration(seq):
    """Last complete Newton iteration: seed/jet-chain ... cubature ... LU."""
    starts = [i for i, s in enumerate(seq) if s[0].endswith("k_seed_jet") or "k_mlp_jet_fwd" in s[0]]
    best = None
    for i0 in starts:
        ends = [i for i in range(i0, len(seq)) if ("k_lu_solve" in seq[i][0] or "k_lu_lookahead" in seq[i][0])]
        # a graph replay is a few dozen launches; the per-stage timing loops after it are not
        if ends and ends[0] - i0 < 48 and any("k_cubature" in s[0] for s in seq[i0:ends[0]]):
            best = (i0, ends[0])
    i0, i1 = best
    return seq[i0:i1 + 1]


if __name__ == "__main__":
    it = iteration(load(sys.argv[1]))
    tot = sum(s[1] for s in it)
    for s in it:
        print(f"{s[0]:26s} {s[1]:8.2f} us {100 * s[1] / tot:5.1f}%  grid {s[2]:14s} block {s[3]}")
    print(f"total {tot:.1f} us over {len(it)} kernels (ncu: serialised, cold caches)")
