#!/usr/bin/env python
"""Summarise an `ncu --page source --csv --print-source sass` export:
instruction mix (executed warp instructions) and the hottest stall sites."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc = h.index("Instructions Executed"), h.index("Source")
ist = h.index("Warp Stall Sampling (All Samples)")
cnt, tot, samples = collections.Counter(), 0, []
for r in rows[2:]:
    if len(r) <= max(ia, ist):
        continue
    n = int(r[ia] or 0)
    op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split(" ")[0]
    cnt[op] += n
    tot += n
    samples.append((int(r[ist] or 0), n, r[isrc].strip()[:90]))
print(rows[0][1] if len(rows[0]) > 1 else "")
print(f"executed warp instructions: {tot}")
for op, n in cnt.most_common(25):
    print(f"  {op:34s} {n:>12d} {100 * n / max(tot, 1):5.1f}%")
st = sum(s for s, _, _ in samples)
print(f"stall samples: {st}; hottest sites:")
for s, n, src in sorted(samples, reverse=True)[:15]:
    print(f"  {100 * s / max(st, 1):5.1f}%  exec {n:>10d}  {src}")
