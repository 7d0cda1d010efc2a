"""Dev: one cfg4 ensemble (M=64, N=1M, L=224, p=8) solve at small T on one GPU."""
import sys, time
sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth
spec = synth.CONFIGS["cfg4"]
t0 = time.time(); x = synth.generate(spec)[0]; print("gen %.1fs" % (time.time() - t0), x.shape, x.dtype, flush=True)
dev = edaa.Device.get(0); dev.set_image(x)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 2
seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=spec.runs, solver=edaa.SolverConfig(endmembers=8, outer_iters=T)))
dev.solve(8, T, 5, 5, seeds, gammas)
dev.profile_enable(True); t0 = time.time(); dev.solve(8, T, 5, 5, seeds, gammas); dt = time.time() - t0
pr = dev.profile(); dev.profile_enable(False)
print("cfg4 M=64 T=%d solve %.2fs -> %.1f run-iters/s; per launch: %s" % (T, dt, 64 * T / dt,
      {k: round(v[0] / max(v[1], 1), 3) for k, v in pr.items()}))
r = [dev.record(m) for m in range(3)]; print("fit", [round(q.fit_l1, 3) for q in r], "ok", [q.ok for q in r])
