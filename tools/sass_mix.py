"""Static SASS instruction mix per kernel of libsmallkv.so (cuobjdump -sass).

    python tools/sass_mix.py > profiles/r02_sass_mix.txt

Blackwell evidence columns: UTMALDG = TMA tensor load (cp.async.bulk.tensor),
UBLKCP = cp.async.bulk, LDGSTS = cp.async, HMMA = mma.sync, UTC*MMA =
tcgen05.mma, SYNCS = mbarrier operations.
"""
from __future__ import annotations

import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2508_02751_b200", "libsmallkv.so")
COLS = ["HMMA", "UTMALDG", "UBLKCP", "UTCHMMA", "LDGSTS", "LDSM", "MOVM", "LDG", "STG", "LDS", "STS",
        "ATOMS", "ATOMG", "RED", "SYNCS", "BAR", "SHFL", "MUFU", "FFMA", "FADD", "FMUL", "IMAD", "BRA"]


def demangle_short(name: str) -> str:
    m = re.search(r"(\w+_kernel)I(.*?)E?Ev", name)
    if not m:
        m = re.search(r"(\w+_kernel)", name)
        return m.group(1) if m else name
    base, targs = m.group(1), m.group(2)
    args = re.findall(r"L(b[01]|i-?\d+)E", "L" + (targs + "E").replace("ELb", "E;Lb").replace("ELi", "E;Li").replace(";", ""))
    vals = [("true" if a == "b1" else "false") if a.startswith("b") else a[1:] for a in args]
    return f"{base}<{','.join(vals)}>" if vals else base


def short(k: str) -> str:
    """select_kernel<...> out of the namespace-mangled prefix."""
    m = re.findall(r"\d+([a-z][a-z_]*?_kernel)(<[^>]*>)?$", k)
    return "".join(m[-1]) if m else k


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else LIB
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = demangle_short(m.group(1))
            kernels.setdefault(cur, collections.Counter())
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if cur and m:
            op = m.group(2)
            c = kernels[cur]
            c["total"] += 1
            for col in COLS:
                if op == col or op.startswith(col + "_") or (col == "UTCHMMA" and op.startswith("UTC") and "MMA" in op):
                    c[col] += 1
                    break
            else:
                if op.startswith("SYNCS"):
                    c["SYNCS"] += 1
    print("# SASS instruction mix of libsmallkv.so (static counts per kernel; cuobjdump -sass, sm_100a)")
    print("# UTMALDG = TMA (cp.async.bulk.tensor), UBLKCP = cp.async.bulk, LDGSTS = cp.async, HMMA = mma.sync,")
    print("# UTC*MMA = tcgen05.mma (none: DESIGN.md §8), SYNCS = mbarrier ops; regenerate: python tools/sass_mix.py")
    print(" | ".join(["kernel", "total"] + COLS))
    for k in sorted(kernels, key=short):
        c = kernels[k]
        print(" | ".join([short(k), str(c["total"])] + [str(c[col]) for col in COLS]))


if __name__ == "__main__":
    main()
