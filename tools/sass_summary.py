"""Per-kernel SASS mnemonic counts of libppgpu.so (cuobjdump -sass): memory
access widths, fp64 arithmetic (no DFMA may appear in the coefficient
updates: the reference rounds the product and the sum separately), barriers,
bulk/TMA copies.  usage: python tools/sass_summary.py [lib] > profiles/.../sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2506_13241_b200", "libppgpu.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["LDG.E.64", "LDG.E.128", "STG.E.64", "STG.E.128", "LDS.64", "LDS.128", "STS.64", "STS.128", "DMUL", "DADD",
        "DFMA", "DSETP", "VIADDMNMX", "BAR.SYNC", "ATOMS", "ATOMG", "RED.E", "REDUX", "MATCH", "VOTE", "SHFL", "LDGSTS",
        "UBLKCP", "UTMALDG", "UTMASTG", "LDL", "STL"]
per = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = subprocess.run(["cu++filt", m.group(1)], capture_output=True, text=True).stdout.strip() or m.group(1)
        name = name.replace("void ppgpu::", "").replace("(int)", "")
        i = name.find(">(")
        name = name[:i + 1] if i >= 0 else name.split("(")[0]
        cur = per.setdefault(name, collections.Counter())
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(1)
    cur["total"] += 1
    for k in KEYS:
        if op.startswith(k) or (("." in k) and all(part in op for part in k.split(".")) and op.startswith(k.split(".")[0])):
            cur[k] += 1
print(f"SASS mnemonic counts per kernel, {os.path.basename(lib)} (cuobjdump -sass, static instruction counts)")
cols = ["total"] + KEYS
print(f"{'kernel':44s} " + " ".join(f"{c:>9s}" for c in cols))
for name, c in per.items():
    print(f"{name[:44]:44s} " + " ".join(f"{c[k]:9d}" for k in cols))
