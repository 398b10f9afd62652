"""Stall samples and executed instructions per CUDA source line of one ncu report
(source page, cuda+sass view): the hottest lines of the kernel with their top stall reasons.
    python tools/ncu_lines.py report.ncu-rep [n_lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f, hdr, agg = "", None, {}
for r in csv.reader(io.StringIO(raw)):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iA = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        st = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
        continue
    if not hdr or not r or not r[0] or len(r) <= max(iA, iE):
        continue
    try:
        a = float(r[iA] or 0)
    except ValueError:
        continue
    key = (f, int(r[0]))
    e = agg.setdefault(key, [0.0, 0.0, {}, r[1].strip()[:90]])
    e[0] += a
    e[1] += float(r[iE] or 0) if r[iE] not in ("-", "") else 0
    for i in st:
        try:
            e[2][hdr[i]] = e[2].get(hdr[i], 0) + float(r[i] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
tote = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot:.0f}, warp instructions {tote:.0f}")
for (fn, ln), (a, e, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = sorted(s.items(), key=lambda kv: -kv[1])[:2]
    print(f"{100 * a / tot:5.1f}% {100 * e / tote:5.1f}%i {fn}:{ln:<5d} {src:90s} "
          + " ".join(f"{k[6:]}={100 * v / max(a, 1):.0f}" for k, v in top))
