"""SASS instruction census of libfairkv.so (cuobjdump, no GPU needed).

For every kernel: the Blackwell-specific instructions that prove which
hardware paths it uses (UTCHMMA/UTCBAR = tcgen05.mma/commit, LDTM/STTM =
tcgen05.ld/st, UTMALDG = TMA tensor load, UBLKCP = cp.async.bulk, SYNCS =
mbarrier ops, HMMA = mma.sync, LDSM = ldmatrix, MUFU.EX2) plus registers
and shared memory from cuobjdump -res-usage.

    python tools/sass_census.py > profiles/r02_sass_census.md
"""

import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_2502_15804_b200" / "libfairkv.so"
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP", "SYNCS", "HMMA", "LDSM",
       "MUFU.EX2", "REDG", "ATOMG", "ST.E.STRONG.SYS", "LDG", "STG", "BAR.SYNC", "FENCE"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


def main():
    cuobj = "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([cuobj, "-sass", str(LIB)], capture_output=True, text=True).stdout
    res = subprocess.run([cuobj, "-res-usage", str(LIB)], capture_output=True, text=True).stdout
    counts = defaultdict(Counter)
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            op = m.group(2)
            for k in OPS:
                if op == k or op.startswith(k + "."):
                    counts[cur][k] += 1
    usage = {}
    name = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"REG:(\d+).*SHARED:(\d+)", line)
        if m and name:
            usage[name] = (int(m.group(1)), int(m.group(2)))
    names = sorted(counts)
    pretty = demangle(names)
    print(f"# SASS census of `{LIB.name}` (sm_100a)\n")
    print("Static instruction counts per kernel from `cuobjdump -sass`; REG / static SHARED "
          "from `cuobjdump -res-usage` (dynamic shared memory is set at launch).\n")
    cols = [k for k in OPS if any(counts[n][k] for n in names)]
    print("| kernel | REG | SHARED | " + " | ".join(cols) + " |")
    print("|---|---|---|" + "---|" * len(cols))
    for n, p in zip(names, pretty):
        r, s = usage.get(n, ("?", "?"))
        short = p.replace("(anonymous namespace)::", "").replace("fkv::", "").replace("void ", "")
        short = short[:short.rfind("(")] if short.endswith(")") else short
        print(f"| `{short}` | {r} | {s} | " + " | ".join(str(counts[n][k]) for k in cols) + " |")


if __name__ == "__main__":
    sys.exit(main())
