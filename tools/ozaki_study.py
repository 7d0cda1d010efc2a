"""Precision study for fixed-point (int8-sliced) B-step contractions.

Question: how many bits of fixed-point precision must the two B-step
contractions keep (g = XᵀZ and Y = X·w, w = e^{ℓ−m} ≤ 1) so that the EDAA
trajectory stays within the parity bars (objective 1e-4 relative over the first
50 iterations, A/B 1e-3 max-abs) of the fp64 reference?  Model: X quantised to
bx fractional bits (X ∈ [0,1]), Z to bz bits relative to a power-of-two bound
of its column max, w to bw fractional bits; products then exact (fp64 stands in
for the int32 accumulators).  Vectorised numpy restatement of solver.cpp:209-230
in the restructured form (Z = XAᵀ − Y·AAᵀ).

usage: python tools/ozaki_study.py [cfg0|cfg1] [T]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_2209_11002_b200 import synth  # noqa: E402


def q_abs(v, bits):
    s = float(2 ** bits)
    return np.round(v * s) / s


def q_col(v, bits):  # per column, relative to the power-of-two bound of max |v|
    m = np.max(np.abs(v), axis=0, keepdims=True)
    e = np.where(m > 0, np.ceil(np.log2(np.where(m > 0, m, 1.0))), 0.0)
    s = 2.0 ** (bits - e)
    return np.round(v * s) / s


def softmax_cols(logits):
    m = logits.max(axis=0, keepdims=True)
    e = np.exp(logits - m)
    return e / e.sum(axis=0, keepdims=True), e, m


def run(X, p, gamma, seed, T, K1=5, K2=5, bits=None):
    L, N = X.shape
    # B0 as the reference (SplitMix64 draws) is not needed for a precision study: seeded uniforms
    rng = np.random.default_rng(seed)
    u = rng.random((N, p))
    B = softmax_cols(0.1 * u)[0]
    A = np.full((p, N), 1.0 / p)
    Y = X @ B
    s = np.linalg.svd(Y, compute_uv=False)[0]
    eta_a = gamma / s ** 2
    eta_b = np.sqrt(p / N) * eta_a
    Xq = q_abs(X, bits[0]) if bits else X
    trace = [0.5 * np.sum((X - Y @ A) ** 2)]
    for t in range(T):
        G = Y.T @ Y
        P = Y.T @ X
        for _ in range(K1):
            u = eta_a * (P - G @ A)
            lg = np.log(np.maximum(A, 1e-30)) + u
            A = softmax_cols(lg)[0]
        XA = X @ A.T
        AA = A @ A.T
        for k in range(K2):
            if k > 0:
                Y = X @ B if not bits else Yq
            Z = XA - Y @ AA
            if bits:
                g = Xq.T @ q_col(Z, bits[1])
            else:
                g = X.T @ Z
            lg = np.log(np.maximum(B, 1e-30)) + eta_b * g
            B, w, m = softmax_cols(lg)
            if bits:
                # Y_next = X·B = (Xq·wq) / S  (w = e^{ℓ−m} ≤ 1 quantised absolutely)
                S = w.sum(axis=0, keepdims=True)
                Yq = (Xq @ q_abs(w, bits[2])) / S
        Y = X @ B if not bits else Yq
        trace.append(0.5 * np.sum((X - Y @ A) ** 2))
    return np.array(trace), A, B


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg0"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    spec = synth.CONFIGS[cfg]
    X = synth.generate(spec, pixels=min(spec.pixels, 10000))[0].astype(np.float64)
    for gamma in (8.0, 1.0, 0.125):
        ref = run(X, spec.endmembers, gamma, 1, T)
        for bits in ((24, 24, 24), (28, 28, 28), (32, 32, 32), (35, 35, 35), (42, 42, 42)):
            got = run(X, spec.endmembers, gamma, 1, T, bits=bits)
            rel = np.max(np.abs(got[0] - ref[0]) / np.abs(ref[0]))
            print(f"{cfg} gamma={gamma:6.3f} bits={bits}: trace rel {rel:.2e}  A {np.max(np.abs(got[1]-ref[1])):.2e}"
                  f"  B {np.max(np.abs(got[2]-ref[2])):.2e}", flush=True)


if __name__ == "__main__":
    main()
