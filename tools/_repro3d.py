import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext
n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
p = ext.make_ext_problem("advdiff3d", n=n)
rhs = ek.CountingRhs(p.rhs)
s = ek.make_linearized(rhs, p.u0, jac_factory=p.jac_factory)
torch.cuda.synchronize()
print("linearized", flush=True)
lam, ok = ek.power_iterate(s.J)
print("lam", lam, ok, flush=True)
