import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext
p = ext.advdiff3d_problem(n=int(sys.argv[1]) if len(sys.argv) > 1 else 512)
u0 = torch.from_numpy(p.u0).cuda()
xi = ek.get_leja_points(400)
def run():
    return ek.adaptive_loop(p.rhs, u0, 1.0, "exprb32", "leja", 1e-10, jac_factory=p.jac_factory,
                            ctx=ek.EngineContext(xi=xi), max_steps=20, stepper=ext.take_step_ext,
                            order=ext.EXT_ORDER["exprb32"])
dts = []
def obs(t, dt, sys_, res):
    dts.append((t, dt, res.stats.leja_iters))
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
tr = ek.adaptive_loop(p.rhs, u0, 1.0, "exprb32", "leja", 1e-10, jac_factory=p.jac_factory,
                      ctx=ek.EngineContext(xi=xi), max_steps=20, stepper=ext.take_step_ext,
                      order=ext.EXT_ORDER["exprb32"], observer=obs)
torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t0, "acc", tr.steps_accepted, "rej", tr.steps_rejected, "leja", tr.leja_iters, "rhs", tr.rhs_evals)
for d in dts: print(d)
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(20)
