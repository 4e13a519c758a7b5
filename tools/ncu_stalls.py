"""Stall reasons by SASS opcode (and the hottest instructions) from an ncu source-page CSV (development aid).
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_stalls.py x.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
hot = []
prev = None
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) < len(hdr) or not r[ia].startswith("0x"):
        continue
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc].strip())
    o = m.group(2) if m else "?"
    row = {}
    for h, i in zip(reasons, ri):
        v = int(r[i] or 0)
        tot[h] += v
        byop[h][o] += v
        row[h] = v
    hot.append((sum(row.values()), r[ia][-5:], r[isrc].strip(), max(row, key=row.get), prev))
    prev = r[isrc].strip()
T = sum(tot.values())
for h, v in tot.most_common(8):
    print(f"{h:22s} {100 * v / T:5.1f}%   by opcode: {byop[h].most_common(5)}")
print("hottest instructions (samples, addr, instr, top reason, previous instr):")
for x in sorted(hot, reverse=True)[:25]:
    print(f"  {x[0]:5d} {x[1]} {x[2][:60]:60s} {x[3]:16s} prev: {x[4][:50] if x[4] else ''}")
