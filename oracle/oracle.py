"""ctypes surface over the two CPU oracle libraries (see __init__ docstring)."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "reference": os.path.join(HERE, "_ref", "liboracle_ref.so"),
    "port": os.path.join(HERE, "_ref", "libedaa_oracle.so"),
}
# Symbol prefix per library; both export the same argument lists.
PREFIX = {"reference": "oref_", "port": "orc_"}
DEFAULT_GAMMAS = (0.125, 0.25, 0.5, 1.0, 2.0, 4.0, 8.0)  # ensemble.hpp:18


class OracleError(RuntimeError):
    """The oracle reported archetype::Error (message preserved)."""


def available_kinds():
    return [k for k, p in LIBS.items() if os.path.exists(p)]


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


@dataclass
class RunOut:
    trace: np.ndarray
    A: np.ndarray
    B: np.ndarray
    E: np.ndarray
    fit_l1: float
    coherence: float


@dataclass
class EnsembleOut:
    seeds: np.ndarray
    gammas: np.ndarray
    fits: np.ndarray
    mus: np.ndarray
    ok: np.ndarray
    candidates: list
    selected: int
    fit_min: float
    trace: np.ndarray
    A: np.ndarray
    B: np.ndarray
    E: np.ndarray
    extra: dict = field(default_factory=dict)


class Oracle:
    def __init__(self, kind: str | None = None):
        if kind is None:
            kinds = available_kinds()
            if not kinds:
                raise FileNotFoundError("no oracle library built; run `make -C oracle`")
            kind = kinds[0]
        self.kind = kind
        self.lib = C.CDLL(LIBS[kind])
        self._p = PREFIX[kind]
        self._err = C.create_string_buffer(512)

    def _f(self, name):
        return getattr(self.lib, self._p + name)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self._err.value.decode("utf-8"))

    # -- ingest -----------------------------------------------------------------
    def l2_normalize(self, x):
        """(normalised L×N, zero pixels) — image.cpp:29-47 (validation included)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        L, N = x.shape
        out = np.zeros((L, N))
        zero = np.zeros(max(N, 1), dtype=np.uint64)
        nz = _sz()
        f = self._f("l2_normalize")
        f.argtypes = [_dp, _sz, _sz, _dp, _u64p, C.POINTER(_sz), C.c_char_p, _sz]
        self._check(f(x, L, N, out, zero, C.byref(nz), self._err, 512))
        return out, [int(v) for v in zero[:nz.value]]

    # -- solver -----------------------------------------------------------------
    def run(self, x, p, T=100, K1=5, K2=5, gamma=1.0, seed=0) -> RunOut:
        x = np.ascontiguousarray(x, dtype=np.float64)
        L, N = x.shape
        trace = np.zeros(T + 1)
        A = np.zeros((p, N))
        B = np.zeros((N, p))
        E = np.zeros((L, p))
        fit = C.c_double()
        mu = C.c_double()
        f = self._f("run")
        f.argtypes = [_dp, _sz, _sz, _sz, _sz, _sz, _sz, C.c_double, C.c_uint64, _dp, _dp, _dp,
                      _dp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_char_p, _sz]
        self._check(f(x, L, N, p, T, K1, K2, gamma, seed, trace, A, B, E, C.byref(fit),
                      C.byref(mu), self._err, 512))
        return RunOut(trace, A, B, E, fit.value, mu.value)

    def run_ensemble(self, x, p, M=50, T=100, K1=5, K2=5, base_seed=0, gammas=DEFAULT_GAMMAS,
                     fit_slack=1.05, workers=0) -> EnsembleOut:
        x = np.ascontiguousarray(x, dtype=np.float64)
        L, N = x.shape
        g = np.ascontiguousarray(gammas, dtype=np.float64)
        if workers == 0:
            workers = os.cpu_count() or 1
        seeds = np.zeros(M, dtype=np.uint64)
        gam = np.zeros(M)
        fits = np.zeros(M)
        mus = np.zeros(M)
        ok = np.zeros(M, dtype=np.uint8)
        cand = np.zeros(M, dtype=np.uint8)
        sel = _sz()
        fmin = C.c_double()
        trace = np.zeros(T + 1)
        A = np.zeros((p, N))
        B = np.zeros((N, p))
        E = np.zeros((L, p))
        f = self._f("run_ensemble")
        f.argtypes = [_dp, _sz, _sz, _sz, _sz, _sz, _sz, _sz, C.c_uint64, _dp, _sz, C.c_double,
                      C.c_uint, _u64p, _dp, _dp, _dp, _u8p, _u8p, C.POINTER(_sz),
                      C.POINTER(C.c_double), _dp, _dp, _dp, _dp, C.c_char_p, _sz]
        self._check(f(x, L, N, p, T, K1, K2, M, base_seed, g, len(g), fit_slack, workers, seeds,
                      gam, fits, mus, ok, cand, C.byref(sel), C.byref(fmin), trace, A, B, E,
                      self._err, 512))
        return EnsembleOut(seeds, gam, fits, mus, ok.astype(bool),
                           [int(i) for i in np.flatnonzero(cand)], int(sel.value), fmin.value,
                           trace, A, B, E)

    # -- primitives ---------------------------------------------------------------
    def select_runs(self, fits, mus, ok, fit_slack=1.05):
        fits = np.ascontiguousarray(fits, dtype=np.float64)
        mus = np.ascontiguousarray(mus, dtype=np.float64)
        okm = np.ascontiguousarray(ok, dtype=np.uint8)
        m = len(fits)
        cand = np.zeros(m, dtype=np.uint8)
        sel = _sz()
        fmin = C.c_double()
        f = self._f("select_runs")
        f.argtypes = [_sz, _dp, _dp, _u8p, C.c_double, _u8p, C.POINTER(_sz),
                      C.POINTER(C.c_double), C.c_char_p, _sz]
        self._check(f(m, fits, mus, okm, fit_slack, cand, C.byref(sel), C.byref(fmin),
                      self._err, 512))
        return [int(i) for i in np.flatnonzero(cand)], int(sel.value), fmin.value

    def spectral_norm(self, m, tol=1e-6, max_iters=1000):
        m = np.ascontiguousarray(m, dtype=np.float64)
        out = C.c_double()
        f = self._f("spectral_norm")
        f.argtypes = [_dp, _sz, _sz, C.c_double, _sz, C.POINTER(C.c_double), C.c_char_p, _sz]
        self._check(f(m, m.shape[0], m.shape[1], tol, max_iters, C.byref(out), self._err, 512))
        return out.value

    def entropic_step(self, z, g, eta):
        z = np.ascontiguousarray(z, dtype=np.float64)
        g = np.ascontiguousarray(g, dtype=np.float64)
        out = np.zeros_like(z)
        f = self._f("entropic_step")
        f.argtypes = [_dp, _dp, _sz, C.c_double, _dp, C.c_char_p, _sz]
        self._check(f(z, g, len(z), eta, out, self._err, 512))
        return out

    def step_sizes(self, x, b0, gamma):
        x = np.ascontiguousarray(x, dtype=np.float64)
        b0 = np.ascontiguousarray(b0, dtype=np.float64)
        ea, eb = C.c_double(), C.c_double()
        f = self._f("step_sizes")
        f.argtypes = [_dp, _sz, _sz, _dp, _sz, C.c_double, C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.c_char_p, _sz]
        self._check(f(x, x.shape[0], x.shape[1], b0, b0.shape[1], gamma, C.byref(ea),
                      C.byref(eb), self._err, 512))
        return ea.value, eb.value

    # -- reference-only primitives (solver.cpp:65-90,166-188,240-259) -------------
    def _need_ref(self, what):
        if self.kind != "reference":
            raise NotImplementedError("%s: exported by the compiled reference only" % what)

    def _xba(self, name, x, b, a, out_shape):
        self._need_ref(name)
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = np.zeros(out_shape)
        f = self._f(name)
        f.argtypes = [_dp, _sz, _sz, _dp, _sz, _dp, _dp, C.c_char_p, _sz]
        self._check(f(x, x.shape[0], x.shape[1], b, b.shape[1], a, out, self._err, 512))
        return out

    def grad_abundances(self, x, b, a):
        return self._xba("grad_abundances", x, b, a, (b.shape[1], x.shape[1]))

    def grad_contributions(self, x, b, a):
        return self._xba("grad_contributions", x, b, a, (x.shape[1], b.shape[1]))

    def objective_l2(self, x, b, a):
        return float(self._xba("objective_l2", x, b, a, (1,))[0])

    def estimate_abundances(self, x, e, iters, eta):
        self._need_ref("estimate_abundances")
        x = np.ascontiguousarray(x, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
        out = np.zeros((e.shape[1], x.shape[1]))
        f = self._f("estimate_abundances")
        f.argtypes = [_dp, _sz, _sz, _dp, _sz, _sz, C.c_double, _dp, C.c_char_p, _sz]
        self._check(f(x, x.shape[0], x.shape[1], e, e.shape[1], int(iters), float(eta), out,
                      self._err, 512))
        return out

    def check_iterate(self, m, outer, which):
        """None if the matrix passes check_iterate, else the reference's message."""
        self._need_ref("check_iterate")
        m = np.ascontiguousarray(m, dtype=np.float64)
        f = self._f("check_iterate")
        f.argtypes = [_dp, _sz, _sz, _sz, C.c_char_p, C.c_char_p, _sz]
        rc = f(m, m.shape[0], m.shape[1], int(outer), which.encode(), self._err, 512)
        return None if rc == 0 else self._err.value.decode("utf-8")

    def fit_l1(self, x, e, a):
        x = np.ascontiguousarray(x, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
        a = np.ascontiguousarray(a, dtype=np.float64)
        if self.kind == "reference":
            out = C.c_double()
            f = self._f("fit_l1")
            f.argtypes = [_dp, _sz, _sz, _dp, _sz, _dp, C.POINTER(C.c_double), C.c_char_p, _sz]
            self._check(f(x, x.shape[0], x.shape[1], e, e.shape[1], a, C.byref(out), self._err,
                          512))
            return out.value
        f = self._f("fit_l1")
        f.argtypes = [_dp, _sz, _sz, _dp, _sz, _dp]
        f.restype = C.c_double
        return f(x, x.shape[0], x.shape[1], e, e.shape[1], a)

    def coherence(self, e, normalized=False):
        e = np.ascontiguousarray(e, dtype=np.float64)
        if self.kind == "reference":
            out = C.c_double()
            f = self._f("coherence")
            f.argtypes = [_dp, _sz, _sz, C.c_int, C.POINTER(C.c_double)]
            f(e, e.shape[0], e.shape[1], int(normalized), C.byref(out))
            return out.value
        f = self._f("coherence")
        f.argtypes = [_dp, _sz, _sz, C.c_int]
        f.restype = C.c_double
        return f(e, e.shape[0], e.shape[1], int(normalized))

    def init_contributions(self, n, p, seed):
        b = np.zeros((n, p))
        if self.kind == "reference":
            f = self._f("init_contributions")
            f.argtypes = [_sz, _sz, C.c_uint64, _dp, C.c_char_p, _sz]
            self._check(f(n, p, seed, b, self._err, 512))
            return b
        st = C.c_uint64(seed)
        f = self._f("init_contributions")
        f.argtypes = [_sz, _sz, C.POINTER(C.c_uint64), _dp]
        f(n, p, C.byref(st), b)
        return b

    def prng_u64(self, seed, count):
        out = np.zeros(count, dtype=np.uint64)
        if self.kind == "reference":
            f = self._f("prng_u64")
            f.argtypes = [C.c_uint64, _sz, _u64p]
            f(seed, count, out)
            return out
        st = C.c_uint64(seed)
        f = self._f("splitmix_next")
        f.argtypes = [C.POINTER(C.c_uint64)]
        f.restype = C.c_uint64
        for i in range(count):
            out[i] = f(C.byref(st))
        return out

    def prng_unit(self, seed, count):
        out = np.zeros(count)
        if self.kind == "reference":
            f = self._f("prng_unit")
            f.argtypes = [C.c_uint64, _sz, _dp]
            f(seed, count, out)
            return out
        st = C.c_uint64(seed)
        f = self._f("splitmix_unit")
        f.argtypes = [C.POINTER(C.c_uint64)]
        f.restype = C.c_double
        for i in range(count):
            out[i] = f(C.byref(st))
        return out

    def sample_gamma(self, seed, draws, gammas=DEFAULT_GAMMAS):
        g = np.ascontiguousarray(gammas, dtype=np.float64)
        out = np.zeros(draws)
        if self.kind == "reference":
            f = self._f("sample_gamma")
            f.argtypes = [C.c_uint64, _dp, _sz, _sz, _dp, C.c_char_p, _sz]
            self._check(f(seed, g, len(g), draws, out, self._err, 512))
            return out
        st = C.c_uint64(seed)
        f = self._f("sample_gamma")
        f.argtypes = [C.POINTER(C.c_uint64), _dp, _sz]
        f.restype = C.c_double
        for i in range(draws):
            out[i] = f(C.byref(st), g, len(g))
        return out
