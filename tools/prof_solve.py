"""One short solve for profiling: python tools/prof_solve.py cfg2 [T]"""
import sys
sys.path.insert(0, '.')
from paper_2209_11002_b200 import edaa, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = synth.CONFIGS[cfg]
x, _, _ = synth.generate(spec)
dev = edaa.Device.get(0)
dev.set_image(x)
seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=spec.runs))
dev.solve(spec.endmembers, T, 5, 5, seeds, gammas)
print("ok", dev.record(0).fit_l1)
