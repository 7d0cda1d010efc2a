"""Development: one ensemble solve of a BASELINE config (for ncu captures).
Usage: python tools/one_solve.py cfg1 [T] [f64]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = synth.CONFIGS[name]
x = synth.generate(spec)[0]
if "f64" in sys.argv[3:]:
    x = x.astype(np.float64)
dev = edaa.Device.get(0)
dev.set_image(x)
seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=spec.runs, solver=edaa.SolverConfig(
    endmembers=spec.endmembers, outer_iters=T)))
dev.solve(spec.endmembers, T, 5, 5, seeds, gammas)
print("trace[0,-1]", dev.traces()[0, -1])
