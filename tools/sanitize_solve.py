"""A small multi-chunk ensemble solve for compute-sanitizer (racecheck / synccheck / memcheck):
13 runs of p = 4 (3 run chunks), 5 pixel slices, T = 2, no CUDA graph, then a p = 12 batch.
Usage: EDAA_NO_GRAPH=1 compute-sanitizer --tool racecheck python tools/sanitize_solve.py"""
import sys

sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth  # noqa: E402

dev = edaa.Device.get(0)
for L, N, p, M in ((41, 600, 4, 13), (24, 300, 12, 3)):
    x = synth.small_scene(L, N, p, seed=5)
    dev.set_image(x)
    seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=M, solver=edaa.SolverConfig(endmembers=p, outer_iters=2)))
    dev.solve(p, 2, 5, 5, seeds, gammas)
    print("ok", L, N, p, M, dev.traces()[0, -1], dev.select(1.05)[1])
