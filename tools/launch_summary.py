#!/usr/bin/env python
"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`):
per-kernel launch count, total device time and share.

    python tools/launch_summary.py gpurun_out/launches.csv [--skip N]
"""

import collections
import csv
import re
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
        "second": 1e6, "s": 1e6}


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(ek::.*|\(long.*|\(int.*", "", r[kn]).replace("ek::", "")
        out.append((name.strip(), float(r[mv].replace(",", "")) * UNIT.get(r[mu], 1.0)))
    return out


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    launches = load(path)[skip:]
    t, c = collections.Counter(), collections.Counter()
    for name, us in launches:
        t[name] += us
        c[name] += 1
    tot = sum(t.values())
    print(f"{len(launches)} launches, {tot / 1e3:.3f} ms device time (serialised, cold-cache)")
    for name, us in t.most_common():
        print(f"{us / tot * 100:6.1f}%  {us / 1e3:9.3f} ms  n={c[name]:5d}  avg {us / c[name]:9.1f} us  {name}")


if __name__ == "__main__":
    main()
