"""Seeded synthetic linear-mixing scenes at the BASELINE.json configs.

The real scenes the paper reports on (Samson, Jasper Ridge, Urban, …) are not
available, so these generators stand in for them with the same shapes:

* endmembers: a 0.05 offset plus a sum of ``bumps`` Gaussians over the band
  index (random centre, width and height), optionally rejected until every
  pair is at least ``min_angle_deg`` apart (cfg3);
* abundances: Dirichlet(α) per pixel; with ``cap`` the largest abundance is set
  to ``cap`` and the excess spread over the others in proportion to their
  mass, repeated until no entry exceeds ``cap`` (cfg2: no pure pixels);
* X = E·A + noise scaled to the SNR exactly as the reference's generator does
  (Frobenius norms of E·A and of the noise, before clamping; synth.cpp:108-124),
  then clamped at 0;
* each pixel is ℓ2-normalised in fp64 and the result stored as fp32.  The
  fp32 array is THE input: the GPU reads it as is and the oracle widens it to
  fp64, so both see bit-identical values.

numpy's PCG64 generator drives everything, so a (config, seed) pair is
reproducible in this image.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


@dataclass(frozen=True)
class SceneSpec:
    name: str
    bands: int
    pixels: int
    endmembers: int
    runs: int
    alpha: float
    snr_db: Optional[float]
    bumps: int = 3
    cap: Optional[float] = None
    min_angle_deg: Optional[float] = None
    height: Optional[int] = None
    width: Optional[int] = None


# BASELINE.json "configs" (the reference metric's workloads).
CONFIGS = {
    "cfg0": SceneSpec("cfg0", 156, 95 * 95, 3, 1, 1.0, 30.0, height=95, width=95),
    "cfg1": SceneSpec("cfg1", 198, 100 * 100, 4, 50, 0.7, 40.0, height=100, width=100),
    "cfg2": SceneSpec("cfg2", 162, 307 * 307, 6, 50, 0.5, 30.0, cap=0.8, height=307, width=307),
    "cfg3": SceneSpec("cfg3", 188, 250 * 190, 12, 50, 0.3, 35.0, bumps=5, min_angle_deg=5.0,
                      height=250, width=190),
    "cfg4": SceneSpec("cfg4", 224, 1024 * 1024, 8, 64, 0.5, 30.0, height=1024, width=1024),
}


def _spectra(rng, L, p, bumps, min_angle_deg):
    idx = np.arange(L, dtype=np.float64)
    out = []
    tries = 0
    while len(out) < p:
        tries += 1
        if tries > 10000:
            raise RuntimeError("could not draw well-separated endmembers")
        s = np.full(L, 0.05)
        for _ in range(bumps):
            c = rng.uniform(0.0, L - 1.0)
            w = rng.uniform(L / 25.0, L / 6.0)
            h = rng.uniform(0.2, 1.0)
            s += h * np.exp(-0.5 * ((idx - c) / w) ** 2)
        if min_angle_deg is not None:
            ok = True
            for q in out:
                cosang = float(s @ q / (np.linalg.norm(s) * np.linalg.norm(q)))
                if np.degrees(np.arccos(min(1.0, cosang))) < min_angle_deg:
                    ok = False
                    break
            if not ok:
                continue
        out.append(s)
    return np.stack(out, axis=1)  # L×p


def _cap_abundances(a, cap):
    a = a.copy()
    for _ in range(64):
        over = a > cap
        if not over.any():
            break
        cols = np.flatnonzero(over.any(axis=0))
        sub = a[:, cols]
        excess = np.where(sub > cap, sub - cap, 0.0).sum(axis=0)
        sub = np.minimum(sub, cap)
        room = np.where(sub < cap, sub, 0.0)
        mass = room.sum(axis=0)
        share = np.where(mass[None, :] > 0, room / np.where(mass > 0, mass, 1.0)[None, :],
                         (sub < cap) / np.maximum((sub < cap).sum(axis=0), 1)[None, :])
        sub = sub + share * excess[None, :]
        a[:, cols] = sub
    return a


def generate(spec: SceneSpec, seed: int = 2209, pixels: Optional[int] = None):
    """Returns (X fp32 L×N, E fp64 L×p, A fp64 p×N)."""
    rng = np.random.default_rng([seed, spec.bands, spec.endmembers])
    L, p = spec.bands, spec.endmembers
    N = spec.pixels if pixels is None else pixels
    E = _spectra(rng, L, p, spec.bumps, spec.min_angle_deg)
    A = rng.dirichlet(np.full(p, spec.alpha), size=N).T  # p×N
    if spec.cap is not None:
        A = _cap_abundances(A, spec.cap)
    X = E @ A
    if spec.snr_db is not None:
        noise = rng.standard_normal(X.shape)
        scale = (np.linalg.norm(X) / np.linalg.norm(noise)) * 10.0 ** (-spec.snr_db / 20.0)
        X = np.maximum(X + scale * noise, 0.0)
    norms = np.linalg.norm(X, axis=0)
    norms[norms == 0.0] = 1.0
    X = (X / norms[None, :]).astype(np.float32)
    return X, E, A


def small_scene(bands=24, pixels=500, endmembers=3, alpha=1.0, snr_db=30.0, seed=7):
    """A small scene for parity tests (oracle finishes in well under a second)."""
    spec = SceneSpec("small", bands, pixels, endmembers, 1, alpha, snr_db)
    return generate(spec, seed=seed)[0]
