"""Per-kernel static SASS summary of the built sm_100a objects (committed as evidence).

For every kernel function in build/obj/kernels_p*.o and solver.o: registers, stack and
local bytes (cuobjdump -res-usage), and the static count of the opcodes that show which
hardware paths the kernel uses: DMMA (FP64 tensor core), DFMA/DMUL/DADD (FP64 pipe),
UTMALDG/UTMASTG/UBLKCP (TMA / bulk copies), SYNCS (mbarrier), LDGSTS (cp.async),
LDS/STS, LDG/STG, LDL/STL (spills), MUFU.

    python tools/sass_summary.py > profiles/r02_sass_summary.txt
"""
import os
import re
import subprocess
import sys
from collections import Counter, OrderedDict

HERE = os.path.dirname(os.path.abspath(__file__))
OBJ = os.path.join(HERE, "..", "build", "obj")
OPS = ["DMMA", "DFMA", "DMUL", "DADD", "MUFU", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "LDGSTS",
       "LDS", "STS", "LDG", "STG", "LDL", "STL", "SHFL", "BAR"]
KIND = {"0": "vol", "1": "surf", "2": "rhs", "3": "stage"}


def demangle(name):
    m = re.search(r"k_elementILi(\d)ELi(\d)ELi(\d+)E", name)
    if m:
        mode, flux, var = m.groups()
        return f"k_element<{KIND.get(mode, mode)},{'llf' if flux == '0' else 'roe'},var{var}>"
    m = re.search(r"(k_[a-z_0-9]+)", name)
    if m:
        t = re.search(r"k_[a-z_0-9]+I(.*?)EEv", name)
        return m.group(1) + (f"<{','.join(re.findall(r'Li(\d+)E', t.group(1) + 'E'))}>" if t else "")
    return name[:60]


def res_usage(obj):
    out = subprocess.run(["cuobjdump", "-res-usage", obj], capture_output=True, text=True).stdout
    res, fn = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
        if m and fn:
            res[fn] = tuple(int(x) for x in m.groups())
    return res


def sass_counts(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    counts, fn = OrderedDict(), None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            counts[fn] = Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m and fn:
            op = m.group(1)
            counts[fn][op] += 1
    return counts


def main():
    objs = sorted(f for f in os.listdir(OBJ) if f.endswith(".o") and (f.startswith("kernels_") or f == "solver.o"))
    print("# static SASS opcode counts per kernel (cuobjdump -sass, sm_100a), registers/stack/local from -res-usage")
    print("# columns: " + " ".join(OPS))
    for o in objs:
        path = os.path.join(OBJ, o)
        res = res_usage(path)
        cnt = sass_counts(path)
        print(f"\n== {o}")
        for fn, c in cnt.items():
            r = res.get(fn, (0, 0, 0, 0))
            vals = " ".join(f"{op}={c[op]}" for op in OPS if c[op])
            print(f"{demangle(fn):44s} reg={r[0]:3d} stack={r[1]:4d} | {vals}")


if __name__ == "__main__":
    sys.exit(main())
