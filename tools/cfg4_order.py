"""Dev: cfg4 ensemble (M=64, N=1M, L=224, p=8) pass times per item order
(2 plain slice-major, 3 interleaved; results bitwise equal)."""
import sys, time
sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth
spec = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
x = synth.generate(spec)[0]
dev = edaa.Device.get(0); dev.set_image(x)
T = 2
seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=spec.runs, solver=edaa.SolverConfig(endmembers=spec.endmembers, outer_iters=T)))
fits = {}
for order in (2, 3, 2, 3):
    dev.set_pass_order(order)
    dev.solve(spec.endmembers, T, 5, 5, seeds, gammas)
    dev.profile_enable(True); t0 = time.time(); dev.solve(spec.endmembers, T, 5, 5, seeds, gammas); dt = time.time() - t0
    pr = dev.profile(); dev.profile_enable(False)
    fits[order] = [dev.record(m).fit_l1 for m in range(spec.runs)]
    print("order %d: solve T=%d %.3fs; per launch ms: %s" % (order, T, dt,
          {k: round(v[0] / max(v[1], 1), 3) for k, v in pr.items()}), flush=True)
print("bitwise equal fits:", fits[2] == fits[3])
