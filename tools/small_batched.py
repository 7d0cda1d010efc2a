import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2209_11002_b200 import edaa, synth
d = edaa.Device.get(0)
for (L, N, p, M) in ((156, 9025, 3, 1), (156, 9025, 3, 50), (50, 2500, 4, 50), (100, 5000, 6, 20)):
    x = synth.small_scene(L, N, p, seed=5)
    d.set_image(x)
    seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=M, solver=edaa.SolverConfig(endmembers=p, outer_iters=50)))
    d.solve(p, 50, 5, 5, seeds, gammas)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter(); d.solve(p, 50, 5, 5, seeds, gammas); best = min(best, time.perf_counter() - t0)
    print("L=%d N=%d p=%d M=%d: %.2f ms per 50 outer iterations -> %.0f run-iterations/s" % (L, N, p, M, best * 1e3, M * 50 / best))
