"""Golden fixtures for the BASELINE configs cfg2-cfg4 and every compiled p bucket.

Companion of make_golden.py (same recipe): the UNMODIFIED reference solver
(oracle/_ref/liboracle_ref.so, built from /root/reference by `make -C oracle
ref`) runs on the seeded synthetic scenes of paper_2209_11002_b200/synth.py and
its outputs are stored; the input image is pinned by the SHA-256 of its fp32
bytes.  These targets take CPU hours (the reference is single-threaded per
run), so each one is a separate invocation:

    python tests/golden/make_golden_big.py pbuckets   # p = 7..15 single runs (minutes)
    python tests/golden/make_golden_big.py cfg2       # M=50, T=100 ensemble (~1.5 h on 8 cores)
    python tests/golden/make_golden_big.py cfg3       # M=50, T=100 ensemble (~1 h)
    python tests/golden/make_golden_big.py cfg4run    # full N=1,048,576 runs, T=50 (~2 h)
    python tests/golden/make_golden_big.py cfg4prefix # 65,536-pixel prefix, 8 runs, T=50

Factor matrices of the big scenes are stored as fp32 (the parity bar is 1e-3
max-abs; fp32 storage adds <= 6e-8), full-N cfg4 factors only on a strided
sample of pixels (every 1024th) to keep the fixtures small.
"""
import concurrent.futures as cf
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle  # noqa: E402
from paper_2209_11002_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
WORKERS = int(os.environ.get("GOLDEN_WORKERS", os.cpu_count() or 1))

# One small single run per compiled p not covered by make_golden.py (p = 2..6,
# 12, 16 are), two per bucket of the pass-kernel instantiations where the
# register layout changes (p = 7, 8: G off registers; 9-16: 24-column chunks
# hold one run).  (name, L, N, p, alpha, snr, scene seed, T, gamma, run seed)
P_BUCKETS = [
    ("run_l40_n1500_p7_g8", 40, 1500, 7, 0.5, 30.0, 31, 50, 8.0, 0),
    ("run_l40_n1500_p7_g05", 40, 1500, 7, 0.5, 30.0, 31, 50, 0.5, 4),
    ("run_l48_n1200_p8_g8", 48, 1200, 8, 0.5, 30.0, 37, 50, 8.0, 0),
    ("run_l48_n1200_p8_g1", 48, 1200, 8, 0.5, 30.0, 37, 50, 1.0, 1),
    ("run_l52_n1000_p9_g4", 52, 1000, 9, 0.4, 35.0, 41, 50, 4.0, 2),
    ("run_l56_n1100_p10_g8", 56, 1100, 10, 0.3, 35.0, 43, 50, 8.0, 6),
    ("run_l60_n900_p11_g2", 60, 900, 11, 0.3, 35.0, 47, 50, 2.0, 8),
    ("run_l64_n800_p13_g8", 64, 800, 13, 0.3, 35.0, 53, 50, 8.0, 10),
    ("run_l70_n700_p14_g025", 70, 700, 14, 0.3, 35.0, 59, 50, 0.25, 12),
    ("run_l72_n650_p15_g1", 72, 650, 15, 0.3, 35.0, 61, 50, 1.0, 14),
]

C4_STRIDE = 1024          # sampled pixel columns of the full-N cfg4 factors
C4_PREFIX = 65536         # pixel prefix of the cfg4 image for the M=8 ensemble
C4_T = 50


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float32).tobytes()).hexdigest()


def scene(L, N, p, alpha, snr, seed):
    return synth.generate(synth.SceneSpec("golden", L, N, p, 1, alpha, snr), seed=seed)[0]


def pbuckets(orc):
    def one(item):
        name, L, N, p, al, snr, sseed, T, g, rseed = item
        x = scene(L, N, p, al, snr, sseed)
        r = orc.run(x.astype(np.float64), p, T=T, gamma=g, seed=rseed)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), kind="run", bands=L, pixels=N, p=p,
                            alpha=al, snr=snr, scene_seed=sseed, T=T, gamma=g, seed=rseed,
                            x_sha=sha(x), trace=r.trace, A=r.A, B=r.B, E=r.E, fit=r.fit_l1,
                            mu=r.coherence)
        return name
    with cf.ThreadPoolExecutor(WORKERS) as ex:
        for name in ex.map(one, P_BUCKETS):
            print("wrote", name, flush=True)


def ensemble(orc, cfg):
    spec = synth.CONFIGS[cfg]
    x = synth.generate(spec)[0]
    t0 = time.time()
    e = orc.run_ensemble(x.astype(np.float64), spec.endmembers, M=spec.runs, T=100,
                         workers=WORKERS)
    np.savez_compressed(os.path.join(OUT, "%s_m%d.npz" % (cfg, spec.runs)), kind="ensemble",
                        config=cfg, T=100, M=spec.runs, x_sha=sha(x), gammas=e.gammas,
                        fits=e.fits, mus=e.mus, ok=e.ok, candidates=np.array(e.candidates),
                        selected=e.selected, fit_min=e.fit_min, trace=e.trace,
                        A=e.A.astype(np.float32), B=e.B.astype(np.float32), E=e.E,
                        factors_dtype="f4", cpu_seconds=time.time() - t0, workers=WORKERS)
    print("wrote", cfg, "in %.0f s" % (time.time() - t0), flush=True)


def cfg4run(orc):
    spec = synth.CONFIGS["cfg4"]
    x = synth.generate(spec)[0]
    xs = sha(x)
    x64 = x.astype(np.float64)
    del x
    seeds = [0, 1]   # ensemble members 0 and 1: γ = 8 and γ = 1 (sample_gamma's first draw)
    gam = [float(orc.sample_gamma(s, 1)[0]) for s in seeds]

    def one(i):
        t0 = time.time()
        r = orc.run(x64, spec.endmembers, T=C4_T, gamma=gam[i], seed=seeds[i])
        cols = np.arange(0, spec.pixels, C4_STRIDE)
        name = "c4run_s%d_t%d.npz" % (seeds[i], C4_T)
        np.savez_compressed(os.path.join(OUT, name), kind="c4run", config="cfg4", T=C4_T,
                            gamma=gam[i], seed=seeds[i], x_sha=xs, trace=r.trace, E=r.E,
                            fit=r.fit_l1, mu=r.coherence, stride=C4_STRIDE, A_cols=r.A[:, cols],
                            B_rows=r.B[cols, :], A_rowsum=r.A.sum(axis=1), B_colmax=r.B.max(axis=0),
                            cpu_seconds=time.time() - t0)
        return name, time.time() - t0
    with cf.ThreadPoolExecutor(len(seeds)) as ex:
        for name, dt in ex.map(one, range(len(seeds))):
            print("wrote", name, "in %.0f s" % dt, flush=True)


def cfg4prefix(orc):
    spec = synth.CONFIGS["cfg4"]
    x = np.ascontiguousarray(synth.generate(spec)[0][:, :C4_PREFIX])
    x64 = x.astype(np.float64)
    M = 8
    seeds = list(range(M))
    gam = [float(orc.sample_gamma(s, 1)[0]) for s in seeds]

    def one(m):
        return orc.run(x64, spec.endmembers, T=C4_T, gamma=gam[m], seed=seeds[m])
    with cf.ThreadPoolExecutor(WORKERS) as ex:
        rs = list(ex.map(one, range(M)))
    fits = np.array([r.fit_l1 for r in rs])
    mus = np.array([r.coherence for r in rs])
    cand, sel, fmin = orc.select_runs(fits, mus, np.ones(M, dtype=bool))
    # full factors for the selected member and the first γ <= 1 member (size)
    keep = [sel] + [m for m in range(M) if gam[m] <= 1.0 and m != sel][:1]
    np.savez_compressed(os.path.join(OUT, "c4pre_n%d_m%d_t%d.npz" % (C4_PREFIX, M, C4_T)),
                        kind="c4prefix", config="cfg4", prefix=C4_PREFIX, T=C4_T, M=M,
                        x_sha=sha(x), seeds=np.array(seeds), gammas=np.array(gam), fits=fits,
                        mus=mus, candidates=np.array(cand), selected=sel, fit_min=fmin,
                        traces=np.stack([r.trace for r in rs]), E=np.stack([r.E for r in rs]),
                        factor_runs=np.array(keep), factors_dtype="f4",
                        A=np.stack([rs[m].A for m in keep]).astype(np.float32),
                        B=np.stack([rs[m].B for m in keep]).astype(np.float32))
    print("wrote c4pre (selected %d, candidates %s)" % (sel, cand), flush=True)


if __name__ == "__main__":
    orc = Oracle("reference")
    for target in sys.argv[1:]:
        {"pbuckets": pbuckets, "cfg2": lambda o: ensemble(o, "cfg2"),
         "cfg3": lambda o: ensemble(o, "cfg3"), "cfg4run": cfg4run,
         "cfg4prefix": cfg4prefix}[target](orc)
