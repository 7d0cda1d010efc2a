"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

Runs the UNMODIFIED reference solver (oracle/_ref/liboracle_ref.so, built by
`make -C oracle ref` from /root/reference) on seeded synthetic scenes and
stores its outputs.  Inputs are regenerated from (generator spec, seed) and
pinned by a SHA-256 of the fp32 image so a drifted generator is detected.

    python tests/golden/make_golden.py [--big]

--big adds the BASELINE cfg0 single run (T=100, ~40 s) and the cfg1 M=50
ensemble (T=100, several minutes on 8 cores).
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle  # noqa: E402
from paper_2209_11002_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, bands, pixels, p, alpha, snr, scene seed, T, gamma, run seed)
SMALL_RUNS = [
    ("run_l24_n500_p3_g1", 24, 500, 3, 1.0, 30.0, 7, 50, 1.0, 3),
    ("run_l24_n500_p3_g8", 24, 500, 3, 1.0, 30.0, 7, 50, 8.0, 3),
    ("run_l40_n2000_p6_g8", 40, 2000, 6, 0.5, 30.0, 11, 60, 8.0, 3),
    ("run_l60_n3000_p12_g4", 60, 3000, 12, 0.3, 35.0, 5, 50, 4.0, 7),
    ("run_l33_n777_p5_g2", 33, 777, 5, 0.7, 40.0, 19, 50, 2.0, 11),   # ragged N, odd L
    ("run_l1_n64_p2_g1", 1, 64, 2, 1.0, None, 2, 20, 1.0, 0),          # single band
    ("run_l16_n1_p2_g1", 16, 1, 2, 1.0, None, 3, 10, 1.0, 5),          # single pixel
    ("run_l300_n200_p16_g05", 300, 200, 16, 0.5, 30.0, 23, 30, 0.5, 9),  # max p, wide L
]
SMALL_ENSEMBLES = [
    ("ens_l20_n500_p3_m50", 20, 500, 3, 1.0, 30.0, 0, 100, 50),
    ("ens_l50_n2500_p4_m50", 50, 2500, 4, 0.7, 40.0, 1, 60, 50),
    ("ens_l30_n1000_p6_m20", 30, 1000, 6, 0.5, 30.0, 4, 50, 20),
]


def scene(bands, pixels, p, alpha, snr, seed):
    spec = synth.SceneSpec("golden", bands, pixels, p, 1, alpha, snr)
    return synth.generate(spec, seed=seed)[0]


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float32).tobytes()).hexdigest()


def main(big=False):
    orc = Oracle("reference")
    for name, L, N, p, al, snr, sseed, T, g, rseed in SMALL_RUNS:
        x = scene(L, N, p, al, snr, sseed)
        r = orc.run(x.astype(np.float64), p, T=T, gamma=g, seed=rseed)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), kind="run", bands=L, pixels=N, p=p,
                            alpha=al, snr=np.nan if snr is None else snr, scene_seed=sseed, T=T,
                            gamma=g, seed=rseed, x_sha=sha(x), trace=r.trace, A=r.A, B=r.B, E=r.E,
                            fit=r.fit_l1, mu=r.coherence)
        print("wrote", name)
    for name, L, N, p, al, snr, sseed, T, M in SMALL_ENSEMBLES:
        x = scene(L, N, p, al, snr, sseed)
        e = orc.run_ensemble(x.astype(np.float64), p, M=M, T=T, workers=os.cpu_count())
        np.savez_compressed(os.path.join(OUT, name + ".npz"), kind="ensemble", bands=L, pixels=N,
                            p=p, alpha=al, snr=snr, scene_seed=sseed, T=T, M=M, x_sha=sha(x),
                            gammas=e.gammas, fits=e.fits, mus=e.mus, ok=e.ok,
                            candidates=np.array(e.candidates), selected=e.selected,
                            fit_min=e.fit_min, trace=e.trace, A=e.A, B=e.B, E=e.E)
        print("wrote", name)
    if big:
        spec = synth.CONFIGS["cfg0"]
        x = synth.generate(spec)[0]
        # cfg0 through the ensemble path, M=1 seed 0 → γ = 8 (test_ensemble.cpp:70-72)
        e = orc.run_ensemble(x.astype(np.float64), 3, M=1, T=100, workers=1)
        np.savez_compressed(os.path.join(OUT, "cfg0_m1.npz"), kind="ensemble", config="cfg0",
                            T=100, M=1, x_sha=sha(x), gammas=e.gammas, fits=e.fits, mus=e.mus,
                            ok=e.ok, candidates=np.array(e.candidates), selected=e.selected,
                            fit_min=e.fit_min, trace=e.trace, A=e.A, B=e.B, E=e.E)
        print("wrote cfg0_m1")
        spec = synth.CONFIGS["cfg1"]
        x = synth.generate(spec)[0]
        e = orc.run_ensemble(x.astype(np.float64), 4, M=50, T=100, workers=os.cpu_count())
        np.savez_compressed(os.path.join(OUT, "cfg1_m50.npz"), kind="ensemble", config="cfg1",
                            T=100, M=50, x_sha=sha(x), gammas=e.gammas, fits=e.fits, mus=e.mus,
                            ok=e.ok, candidates=np.array(e.candidates), selected=e.selected,
                            fit_min=e.fit_min, trace=e.trace, A=e.A, B=e.B, E=e.E)
        print("wrote cfg1_m50")


if __name__ == "__main__":
    main(big="--big" in sys.argv)
