"""Per-pass device times of one solve (profiling events): python tools/pass_times.py cfg2 [T]"""
import sys
sys.path.insert(0, '.')
from paper_2209_11002_b200 import edaa, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 5
spec = synth.CONFIGS[cfg]
x, _, _ = synth.generate(spec)
dev = edaa.Device.get(0)
dev.set_image(x)
seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=spec.runs))
dev.solve(spec.endmembers, 1, 5, 5, seeds, gammas)  # warm
dev.profile_enable(True)
dev.solve(spec.endmembers, T, 5, 5, seeds, gammas)
pr = dev.profile()
print(cfg, "T=%d" % T, {k: (round(v[0] / max(v[1], 1), 4), v[1]) for k, v in pr.items()}, "(ms per launch, launches)")
