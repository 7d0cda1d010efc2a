"""Development timing probe: solve time per config with the fp32 image and with
the image widened to fp64 on the host (exactly the same values), plus the
per-pass-kind device times.  Usage: python tools/xp_time.py cfg1 [cfg2 ...]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth  # noqa: E402


def timed(dev, spec, T, reps=3):
    seeds, gammas = edaa.ensemble_plan(edaa.EnsembleConfig(runs=spec.runs, solver=edaa.SolverConfig(
        endmembers=spec.endmembers, outer_iters=T)))
    dev.solve(spec.endmembers, T, 5, 5, seeds, gammas)  # warm (graph capture)
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        dev.solve(spec.endmembers, T, 5, 5, seeds, gammas)
        best = min(best, time.perf_counter() - t0)
    dev.profile_enable(True)
    dev.solve(spec.endmembers, T, 5, 5, seeds, gammas)
    prof = dev.profile()
    dev.profile_enable(False)
    tr = dev.traces()
    return best, prof, tr


def main():
    names = sys.argv[1:] or ["cfg1"]
    modes = [m for m in ("f32", "f64") if m in (sys.argv[0] + " ".join(names)) or True]
    dev = edaa.Device.get(0)
    for name in names:
        spec = synth.CONFIGS[name]
        x = synth.generate(spec)[0]
        T = 20
        res = {}
        for mode in modes:
            dev.set_image(x if mode == "f32" else x.astype(np.float64))
            best, prof, tr = timed(dev, spec, T)
            res[mode] = tr
            ps = " ".join("%s %.3f ms/launch" % (k, v[0] / max(v[1], 1)) for k, v in prof.items())
            print("%s %s: M=%d T=%d solve %.2f ms  (%s)" % (name, mode, spec.runs, T, best * 1e3, ps),
                  flush=True)
        if len(res) == 2:
            d = np.max(np.abs(res["f32"] - res["f64"]) / np.abs(res["f32"]))
            print("%s trace rel diff f32 vs f64 image: %.3e" % (name, d))


if __name__ == "__main__":
    main()
