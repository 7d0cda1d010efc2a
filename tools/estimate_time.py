"""Timing of estimate_abundances on a BASELINE shape, next to the compiled
reference on a pixel prefix: python tools/estimate_time.py cfg2 [iters]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
spec = synth.CONFIGS[cfg]
x, E, _ = synth.generate(spec)
E = np.ascontiguousarray(E, dtype=np.float64)
eta = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0 / np.linalg.eigvalsh(E.T @ E)[-1]   # contractive step
dev = edaa.Device.get(0)
dev.set_image(x)
dev.estimate_abundances(E, 2, eta)
t0 = time.perf_counter()
A = dev.estimate_abundances(E, iters, eta)
dt = time.perf_counter() - t0
print("%s: estimate_abundances L=%d N=%d p=%d iters=%d eta=%.3g: %.1f ms on the GPU (incl. the p×N download)" %
      (cfg, x.shape[0], x.shape[1], E.shape[1], iters, eta, dt * 1e3))
try:
    from oracle import Oracle
    n = min(x.shape[1], 2048)
    xs = np.ascontiguousarray(x[:, :n]).astype(np.float64)
    t0 = time.perf_counter()
    ref = Oracle("reference").estimate_abundances(xs, E, iters, eta)
    dc = time.perf_counter() - t0
    print("  compiled reference, first %d pixels: %.1f ms -> %.0f ms for the image on one core; max |A - ref| on the prefix %.2e"
          % (n, dc * 1e3, dc * 1e3 * x.shape[1] / n, np.abs(A[:, :n] - ref).max()))
except Exception as exc:  # noqa: BLE001
    print("  reference unavailable:", exc)
