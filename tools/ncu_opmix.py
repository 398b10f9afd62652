"""Executed-instruction mix (per opcode) and stall samples of one ncu report (source page, SASS)."""
import csv
import io
import subprocess
import sys
from collections import Counter

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
i_st = hdr.index("Warp Stall Sampling (All Samples)")
ex, st = Counter(), Counter()
for r in rows[2:]:
    if len(r) <= i_ex or not r[i_src].strip():
        continue
    toks = r[i_src].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    ex[op] += int(r[i_ex] or 0)
    st[op] += int(r[i_st] or 0)
tot, tst = sum(ex.values()), max(1, sum(st.values()))
print(f"{sys.argv[1]}: {tot} warp instructions")
for k, v in ex.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"  {k:8s} {v:12d} {100 * v / tot:5.1f}%  stall samples {100 * st[k] / tst:5.1f}%")
