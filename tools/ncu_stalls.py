"""Stall breakdown of an ncu report: by stall reason and by SASS opcode, plus hottest lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
hdr, data = rows[1], rows[2:]
iS, iA = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[iA] or 0) for r in data) or 1.0
agg, op = {}, {}
for r in data:
    for i in stall_cols:
        agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
    parts = r[iS].split()
    o = parts[1] if parts and parts[0].startswith("@") and len(parts) > 1 else (parts[0] if parts else "")
    o = o.split(".")[0]
    op[o] = op.get(o, 0) + float(r[iA] or 0)
print("stalls:", sorted(((round(v / tot * 100, 1), k) for k, v in agg.items()), reverse=True)[:8])
print("opcodes:", sorted(((round(v / tot * 100, 1), k) for k, v in op.items()), reverse=True)[:14])
