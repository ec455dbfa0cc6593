#!/usr/bin/env python
"""Print GPU-vs-oracle whole-run parity numbers for configs 2 and 3."""
import sys, json, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext
from oracle import np_fields as OF, np_integrate as OI, np_phi as OP

def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))

xi = OP.leja_points(400)
runs = [("c2", "allen_cahn_periodic", 256, "exprb43", "leja", 1e-10, 100, None),
        ("c2", "allen_cahn_periodic", 256, "exprb43", "kiops", 1e-10, 100, None),
        ("c3", "burgers2d", 1024, "epirk4s3", "leja", 1e-8, 20, True),
        ("c3", "burgers2d", 1024, "epirk4s3", "lekry", 1e-8, 20, True),
        ("c3", "burgers2d", 256, "epirk4s3", "kiops", 1e-8, 20, True)]
which = sys.argv[1:] or None
for tag, name, n, integ, scheme, tol, ms, jac in runs:
    if which and f"{tag}-{scheme}" not in which:
        continue
    p = ext.make_ext_problem(name, n=n)
    q = getattr(OF, name)(n=n)
    t0 = time.time()
    tr = ek.adaptive_loop(p.rhs, p.u0, 1.0, integ, scheme, tol, jac_factory=p.jac_factory,
                          ctx=ek.EngineContext(xi=xi), max_steps=ms)
    t1 = time.time()
    otr = OI.adaptive(q.rhs, q.u0, 1.0, integ, scheme, tol, jac_factory=q.jac_factory,
                      ctx=OI.Ctx(xi=xi), max_steps=ms)
    t2 = time.time()
    c = lambda r: [r.steps_accepted, r.steps_rejected, r.rhs_evals, r.leja_iters, r.krylov_matvecs, r.substeps]
    nn = min(len(tr.dts), len(otr.dts))
    print(json.dumps({"run": f"{tag} {name} {n} {integ} {scheme}", "gpu": c(tr), "oracle": c(otr),
                      "dts_rel": rel(tr.dts[:nn], otr.dts[:nn]), "u_rel": rel(tr.u, otr.u),
                      "t_gpu": t1 - t0, "t_oracle": t2 - t1, "t": [tr.t, otr.t]}))
