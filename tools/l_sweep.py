import sys
sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth
dev = edaa.Device.get(0)
N, p, M = 10000, 4, 50
seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=M))
for L in (48, 96, 144, 198, 256, 320):
    x = synth.small_scene(L, N, p, seed=3)
    dev.set_image(x)
    dev.solve(p, 1, 5, 5, seeds, gammas)
    dev.profile_enable(True)
    dev.solve(p, 3, 5, 5, seeds, gammas)
    pr = dev.profile()
    dev.profile_enable(False)
    tiles = -(-N // 32) * 9 / 148.0
    b = pr["B"][0] / pr["B"][1] * 1e3; a = pr["A"][0] / pr["A"][1] * 1e3
    print("L=%3d  B pass %.1f us = %.0f cycles per tile per CTA;  A pass %.1f us = %.0f" % (L, b, b * 1965 / tiles, a, a * 1965 / tiles))
