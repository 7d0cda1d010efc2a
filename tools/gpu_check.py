"""Quick GPU-vs-oracle parity probe (development tool)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2209_11002_b200 import edaa, synth
from oracle import Oracle

orc = Oracle()
print("oracle kind", orc.kind)

def cmp_run(x, p, T, gamma, seed):
    t0 = time.time()
    ref = orc.run(x.astype(np.float64), p, T=T, gamma=gamma, seed=seed)
    t1 = time.time()
    got = edaa.run(x, edaa.SolverConfig(endmembers=p, outer_iters=T, gamma=gamma, seed=seed))
    t2 = time.time()
    n50 = min(T, 50) + 1
    rel = np.abs(got.objective_trace[:n50] - ref.trace[:n50]) / np.abs(ref.trace[:n50])
    print(f"L={x.shape[0]} N={x.shape[1]} p={p} T={T} g={gamma} s={seed}: "
          f"obj_rel={rel.max():.3e} A={np.abs(got.abundances-ref.A).max():.3e} "
          f"B={np.abs(got.contributions-ref.B).max():.3e} E={np.abs(got.endmembers-ref.E).max():.3e} "
          f"fit={abs(got.fit_l1-ref.fit_l1)/ref.fit_l1:.3e} mu={abs(got.coherence-ref.coherence):.3e} "
          f"t_ref={t1-t0:.2f}s t_gpu={t2-t1:.2f}s")
    return rel.max()

x = synth.small_scene(24, 500, 3)
for g in (1.0, 8.0):
    cmp_run(x, 3, 30, g, 3)
x = synth.small_scene(40, 2000, 6, alpha=0.5, seed=11)
cmp_run(x, 6, 100, 8.0, 3)
cmp_run(x, 6, 100, 0.5, 13)
x = synth.small_scene(60, 3000, 12, alpha=0.3, seed=5)
cmp_run(x, 12, 60, 4.0, 7)
# ensemble
x = synth.small_scene(20, 500, 3, seed=0)
cfg = edaa.EnsembleConfig(runs=50, solver=edaa.SolverConfig(endmembers=3, outer_iters=100))
t0 = time.time(); res, rep = edaa.run_ensemble(x, cfg); t1 = time.time()
ref = orc.run_ensemble(x.astype(np.float64), 3, M=50, T=100)
t2 = time.time()
fits = np.array([r.fit_l1 for r in rep.per_run]); mus = np.array([r.coherence for r in rep.per_run])
print("ensemble selected gpu", rep.selected, "ref", ref.selected, "cand equal", rep.candidate_set == ref.candidates,
      "fit rel", np.max(np.abs(fits-ref.fits)/ref.fits), "mu", np.max(np.abs(mus-ref.mus)), f"t_gpu={t1-t0:.2f} t_ref={t2-t1:.2f}")
