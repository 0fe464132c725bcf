"""SASS instruction census per kernel of the built objects (cuobjdump -sass):
opcode counts for the memory-movement and synchronisation families that show
how each hot kernel moves data (LDG/STG/LDS/STS, LDGSTS = cp.async,
UBLKCP = cp.async.bulk (TMA), SYNCS = mbarrier, RED/ATOM(S), BAR, ...).

    python tools/sass_census.py build/obj/*.o > profiles/r02_sass_census.json
"""
import collections
import json
import re
import subprocess
import sys

FAMILIES = ["LDG", "STG", "LDS", "STS", "LD", "ST", "LDGSTS", "UBLKCP", "UTMALDG", "UTMASTG",
            "SYNCS", "RED", "ATOM", "ATOMS", "ATOMG", "BAR", "MEMBAR", "ERRBAR", "VOTE", "SHFL",
            "REDUX", "MATCH", "POPC", "FADD", "FMUL", "FFMA", "BRA", "CCTL", "UCGABAR_ARV",
            "UCGABAR_WAIT"]


def census(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    kernels = {}
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(?:\.[\w.]+)?", line)
        if m and cur:
            op = m.group(1)
            kernels[cur]["total"] += 1
            if op in FAMILIES:
                kernels[cur][op] += 1
    return kernels


def short(name):
    dm = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    dm = re.sub(r"sdl::\(anonymous namespace\)::", "", dm)
    return dm.split("(")[0] + ("<" + dm.split("<", 1)[1].split(">")[0] + ">" if "<" in dm.split("(")[0] else "")


if __name__ == "__main__":
    res = {}
    for obj in sys.argv[1:]:
        for k, c in census(obj).items():
            res[short(k)] = dict(sorted(c.items()))
    json.dump(res, sys.stdout, indent=1)
