#!/usr/bin/env python
"""Bandwidth of the fused stage-algebra kernel (ek_lincomb) and the norm
reduction on config-4-sized vectors (2 x 4096^2 doubles)."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2211_08948_b200 import _device as D
    n = 2 * 4096 * 4096
    vs = [torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(5)]
    out = torch.empty_like(vs[0])
    X = D.V
    cases = {
        "scale (1 in, 1 out)": (X(vs[0]) * 3.3e-5, 2),
        "u + c*x (2 in)": (X(vs[0]) + 0.125 * X(vs[1]), 3),
        "(a*x + b*y)*dt (2 in)": ((32.0 * X(vs[0]) - 13.5 * X(vs[1])) * 3.3e-5, 3),
        "u + a*x + b*y + c*z (4 in)": (X(vs[0]) + 0.9 * X(vs[1]) + 1.08 * X(vs[2])
                                       + 5.832 * X(vs[3]), 5),
    }
    res = {}
    for name, (ex, nvec) in cases.items():
        for _ in range(3):
            D.ev(ex, n, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            D.ev(ex, n, out=out)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10 / 1e3
        res[name] = {"ms": t * 1e3, "GBps": nvec * 8 * n / t / 1e9}
    for _ in range(3):
        D.norm2(vs[0])
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for _ in range(10):
        D.norm2(vs[0])
    t = (time.perf_counter() - t0) / 10
    res["norm2 incl. sync"] = {"ms": t * 1e3, "GBps": 8 * n / t / 1e9}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
