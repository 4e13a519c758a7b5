"""Per-loop-body instruction counts of a kernel's SASS (development aid).
usage: python tools/sass_blocks.py <lib.so> <mangled kernel name>"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", "-fun", sys.argv[2], sys.argv[1]], capture_output=True, text=True).stdout
L = []
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?)\s*;", line)
    if m:
        L.append((m.group(1), m.group(2)))
print("instructions:", len(L))
cur, start = [], 0
for i, (a, b) in enumerate(L):
    cur.append(b)
    if re.search(r"\bBRA\b|EXIT|BAR\.", b):
        dp = sum(1 for x in cur if re.search(r"\b(DADD|DMUL)\b", x))
        if dp > 20:
            st = sum(1 for x in cur if "STG" in x)
            mv = sum(1 for x in cur if re.search(r"IMAD\.MOV|\bMOV\b", x))
            print(f"  [{start:5d},{i:5d}] {len(cur):4d} instrs: DP {dp}, other {len(cur) - dp} (STG {st}, moves {mv})")
        cur, start = [], i + 1
