"""Dev probe: A-pass time vs K1 (inner A steps) on cfg1, to split the per-step chain cost from per-tile overhead."""
import sys
sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth  # noqa: E402
spec = synth.CONFIGS["cfg1"]
x = synth.generate(spec)[0]
dev = edaa.Device.get(0)
dev.set_image(x)
seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=spec.runs, solver=edaa.SolverConfig(endmembers=4, outer_iters=5)))
for k1 in (1, 2, 5, 10):
    dev.solve(4, 5, k1, 5, seeds, gammas)
    dev.profile_enable(True)
    dev.solve(4, 5, k1, 5, seeds, gammas)
    pr = dev.profile()
    dev.profile_enable(False)
    print("K1=%2d A %.3f ms/launch  B %.3f" % (k1, pr["A"][0] / pr["A"][1], pr["B"][0] / pr["B"][1]), flush=True)
