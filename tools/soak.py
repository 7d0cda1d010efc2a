"""Soak test of the batched solver on random shapes (race / hang / edge-shape evidence):
every shape is solved twice (bitwise equal), one member is re-solved alone (bitwise equal: batch
independence), simplex and finiteness of the factors are checked, and a small fraction of the
cases is compared with the compiled reference at T = 3.
Usage: python tools/soak.py [seconds=240] [seed=0]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
try:
    from oracle import Oracle
    orc = Oracle("reference")
except Exception:  # noqa: BLE001
    orc = None
dev = edaa.Device.get(0)
t_end = time.time() + budget
cases = checked = 0
worst = 0.0
while time.time() < t_end:
    p = int(rng.integers(2, 17))
    L = int(rng.integers(max(p, 3), 321))
    N = int(rng.choice([1, 2, 31, 32, 33, 63, 64, 65, 127, 128, 129]) if rng.random() < 0.2 else rng.integers(1, 30001))
    M = int(rng.choice([1, 2, 3, 7, 24, 50, 64]))
    T = int(rng.integers(1, 5))
    K1, K2 = int(rng.integers(1, 7)), int(rng.integers(1, 7))
    if L * N * M * p > 4e9:
        continue
    x = synth.small_scene(L, N, p, seed=int(rng.integers(1 << 30)))
    seeds = [int(s) for s in rng.integers(0, 1 << 40, M)]
    gammas = [float(g) for g in rng.choice([0.125, 0.25, 0.5, 1, 2, 4, 8], M)]
    dev.set_image(x)
    dev.solve(p, T, K1, K2, seeds, gammas)
    tr1 = dev.traces().copy()
    m = int(rng.integers(M))
    A1, B1, E1 = dev.factors(m)
    ok = [bool(dev.record(r).ok) for r in range(M)]
    dev.solve(p, T, K1, K2, seeds, gammas)
    assert np.array_equal(tr1, dev.traces()), ("repeat differs", L, N, p, M, T)
    A2, B2, E2 = dev.factors(m)
    assert np.array_equal(A1, A2) and np.array_equal(B1, B2) and np.array_equal(E1, E2)
    if ok[m]:
        assert np.all(np.isfinite(A1)) and np.all(A1 >= 0) and np.abs(A1.sum(axis=0) - 1).max() <= 1e-9, (L, N, p, M)
        assert np.all(np.isfinite(B1)) and np.all(B1 >= 0) and np.abs(B1.sum(axis=0) - 1).max() <= 1e-9, (L, N, p, M)
    dev.solve(p, T, K1, K2, [seeds[m]], [gammas[m]])   # the member alone: same bits
    As, Bs, Es = dev.factors(0)
    assert np.array_equal(As, A1) and np.array_equal(Bs, B1) and np.array_equal(dev.traces()[0], tr1[m]), \
        ("batch dependence", L, N, p, M, m)
    if orc is not None and ok[m] and L * N * p * T * (K1 + K2) < 3e8:
        ref = orc.run(x.astype(np.float64), p, T=T, K1=K1, K2=K2, gamma=gammas[m], seed=seeds[m])
        # absolute differences below 1e-13·½‖X‖² are rounding noise of the expanded-form trace: e.g. N = 1,
        # where X·B·A = x·Σa reproduces the pixel exactly and the reference's objective is 0
        scale = 0.5 * float((x.astype(np.float64) ** 2).sum())
        dev_rel = np.max(np.maximum(np.abs(tr1[m] - ref.trace) - 1e-13 * scale, 0.0) / np.maximum(np.abs(ref.trace), 1e-6 * scale))
        worst = max(worst, float(dev_rel), float(np.abs(A1 - ref.A).max()), float(np.abs(B1 - ref.B).max()))
        # 1e-6: a hundredth of the north-star bar.  Unstable members (large γ with K1 = 1: the objective
        # rises and falls by 2x between iterations) amplify last-bit differences ~100x per outer
        # iteration — observed 2e-8 after 4 iterations at L=15 N=24,195 p=3 γ=4 — typical cases sit at 1e-11.
        assert dev_rel <= 1e-6 and np.abs(A1 - ref.A).max() <= 1e-6, ("reference mismatch", L, N, p, M, T, K1, K2, dev_rel)
        checked += 1
    cases += 1
print("soak ok: %d random shapes in %.0f s (each solved twice + one member alone, bitwise equal); %d compared with the "
      "compiled reference, worst deviation %.1e" % (cases, budget, checked, worst))
