"""Python surface of the B200 EDAA path, mirroring the reference C++ API.

Names, argument meaning and error behaviour follow
``/root/reference/proj/include/archetype/{solver,ensemble,prng}.hpp``:

=====================  ==========================================================
``SolverConfig``       solver.hpp:15-24 (validate: solver.cpp:103-111)
``RunResult``          solver.hpp:29-38
``run``                solver.hpp:81 / solver.cpp:190-238  → one-run batch on the GPU
``EnsembleConfig``     ensemble.hpp:15-29 (validate: ensemble.cpp:17-27)
``RunRecord``          ensemble.hpp:31-40
``SelectionReport``    ensemble.hpp:42-47
``run_ensemble``       ensemble.hpp:68-69 / ensemble.cpp:108-167 → ONE batched solve
``select_runs``        ensemble.hpp:63 / ensemble.cpp:71-94
``sample_gamma``       ensemble.hpp:58 / ensemble.cpp:62-69
``Prng``               prng.hpp:11-30 (SplitMix64, bit-exact)
=====================  ==========================================================

Every solve runs in the sm_100a kernels behind ``include/edaa_b200.h``; there
is no CPU fallback (a missing library or GPU raises :class:`EdaaError`).
Errors carry the reference's ``archetype::Error`` messages.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import EdaaError, RunRecordC, SolveParams

DEFAULT_GAMMAS = (0.125, 0.25, 0.5, 1.0, 2.0, 4.0, 8.0)  # ensemble.hpp:18
_MASK = (1 << 64) - 1


class Prng:
    """SplitMix64 with the reference's unit mapping (prng.hpp:15-26)."""

    def __init__(self, seed: int):
        self.state = int(seed) & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def next_unit(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53


def sample_gamma(rng: Prng, gamma_set: Sequence[float]) -> float:
    """index = floor(u·|S|), clamped (ensemble.cpp:62-69)."""
    if len(gamma_set) == 0:
        raise EdaaError("step factor set is empty")
    idx = int(rng.next_unit() * float(len(gamma_set)))
    return gamma_set[min(idx, len(gamma_set) - 1)]


@dataclass
class SolverConfig:
    endmembers: int = 0
    outer_iters: int = 100
    inner_iters_a: int = 5
    inner_iters_b: int = 5
    gamma: float = 1.0
    seed: int = 0

    def validate(self):
        if self.endmembers < 2:
            raise EdaaError("solver config: endmember count must be at least 2")
        if self.outer_iters < 1 or self.inner_iters_a < 1 or self.inner_iters_b < 1:
            raise EdaaError("solver config: iteration counts must be at least 1")
        if not (self.gamma > 0.0) or not math.isfinite(self.gamma):
            raise EdaaError("solver config: step factor gamma must be positive")


@dataclass
class EnsembleConfig:
    runs: int = 50
    base_seed: int = 0
    gamma_set: Sequence[float] = DEFAULT_GAMMAS
    fit_slack: float = 1.05
    solver: SolverConfig = field(default_factory=SolverConfig)
    workers: int = 0  # accepted for API parity; the batch runs as one device launch

    def validate(self):
        if self.runs == 0:
            raise EdaaError("ensemble needs at least one run")
        if len(self.gamma_set) == 0:
            raise EdaaError("step factor set is empty")
        for g in self.gamma_set:
            if not math.isfinite(g) or g <= 0.0:
                raise EdaaError("step factors must be finite and positive")
        if not math.isfinite(self.fit_slack) or self.fit_slack < 1.0:
            raise EdaaError("fit slack must be at least 1")
        self.solver.validate()


@dataclass
class RunResult:
    endmembers: np.ndarray      # L×p
    abundances: np.ndarray      # p×N
    contributions: np.ndarray   # N×p
    fit_l1: float
    coherence: float
    seed: int
    gamma: float
    objective_trace: np.ndarray  # T+1


@dataclass
class RunRecord:
    index: int = 0
    seed: int = 0
    gamma: float = 0.0
    fit_l1: float = 0.0
    coherence: float = 0.0
    wall_ms: float = 0.0
    ok: bool = False
    error: str = ""


@dataclass
class SelectionReport:
    per_run: List[RunRecord]
    candidate_set: List[int]
    selected: int
    fit_min: float


def select_runs(per_run: List[RunRecord], fit_slack: float) -> SelectionReport:
    """Algorithm 2's rule on given records (ensemble.cpp:71-94); bookkeeping over
    M scalars.  The device path (run_ensemble) applies the same rule on the GPU."""
    fit_min = math.inf
    for rec in per_run:
        if rec.ok:
            fit_min = min(fit_min, rec.fit_l1)
    if fit_min == math.inf:
        raise EdaaError("every run failed")
    cutoff = fit_slack * fit_min
    cand = [rec.index for rec in per_run if rec.ok and rec.fit_l1 <= cutoff]
    best = cand[0]
    for idx in cand:
        if per_run[idx].coherence < per_run[best].coherence:
            best = idx
    return SelectionReport(per_run, cand, best, fit_min)


def _upload_image(dev: "Device", x) -> None:
    """X onto the device, validated as HsiImage::validate (image.cpp:10-27) does: an
    fp32 L×N host array is checked on the device after the upload
    (edaa_set_image_host_checked); anything else goes through validate_image."""
    arr = np.asarray(x)
    if arr.ndim == 2 and arr.dtype == np.float32 and arr.shape[0] >= 1 and arr.shape[1] >= 1:
        dev.set_image_checked(arr)
    else:
        dev.set_image(validate_image(arr))


def validate_image(x) -> np.ndarray:
    """HsiImage::validate (image.cpp:10-27) on the L×N data.

    Returns the array the device will hold: fp32 when every value is exactly an
    fp32 (the fast path, two CTAs per SM), otherwise fp64 so that results track
    the reference on any fp64 input."""
    arr = np.asarray(x)
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise EdaaError("image: needs at least one band and one pixel")
    # fast path: min/max reductions (NaN propagates through min) settle a clean image
    if arr.dtype.kind == "f" and arr.size:
        lo, hi = arr.min(), arr.max()
        if lo >= 0 and np.isfinite(hi):
            if arr.dtype == np.float32:
                return np.ascontiguousarray(arr)
            a64 = np.ascontiguousarray(arr, dtype=np.float64)
            a32 = a64.astype(np.float32)
            return a32 if np.array_equal(a32.astype(np.float64), a64) else a64
    # the reference throws at the first offending element in row-major order
    flat = arr.ravel()
    nonfin = np.flatnonzero(~np.isfinite(flat))
    neg = np.flatnonzero(np.isfinite(flat) & (flat < 0))
    if nonfin.size or neg.size:
        first_nonfin = nonfin[0] if nonfin.size else flat.size
        first_neg = neg[0] if neg.size else flat.size
        raise EdaaError("image: non-finite reflectance" if first_nonfin < first_neg
                        else "image: negative reflectance")
    if arr.dtype == np.float32:
        return np.ascontiguousarray(arr)
    a64 = np.ascontiguousarray(arr, dtype=np.float64)
    a32 = a64.astype(np.float32)
    if np.array_equal(a32.astype(np.float64), a64):
        return a32
    return a64


class Device:
    """One edaa_ctx (one CUDA device).  Not thread-safe."""

    _cache = {}

    @classmethod
    def get(cls, device: int = 0) -> "Device":
        if device not in cls._cache:
            cls._cache[device] = Device(device)
        return cls._cache[device]

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        rc = self.lib.edaa_create(int(device), C.byref(h))
        if rc != 0:
            raise EdaaError("edaa_create failed on device %d (rc=%d): no usable CUDA device; "
                            "there is no CPU fallback" % (device, rc), rc)
        self.h = h
        self.device = device
        self.L = self.N = 0
        self.M = 0
        self.T = 0
        self.p = 0

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.edaa_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise EdaaError(self.lib.edaa_last_error(self.h).decode("utf-8", "replace"), rc)

    @property
    def stream(self) -> int:
        return int(self.lib.edaa_stream(self.h) or 0)

    # -- image ------------------------------------------------------------------
    def set_image_checked(self, x):
        """fp32 host L×N array: upload, then HsiImage::validate on the device
        (EdaaError with the reference's message on a non-finite or negative value)."""
        xf = np.ascontiguousarray(x, dtype=np.float32)
        self._x_keep = xf
        self._check(self.lib.edaa_set_image_host_checked(self.h, xf.ctypes.data_as(C.c_void_p),
                                                         xf.shape[0], xf.shape[1]))
        self.L, self.N = xf.shape

    def set_image(self, x):
        """x: host L×N array (copied H2D) or a CUDA tensor (copied D2D)."""
        if hasattr(x, "is_cuda") and x.is_cuda:
            import torch
            if x.dtype != torch.float32 or x.dim() != 2 or x.stride(1) != 1:
                raise EdaaError("device image must be a row-contiguous 2-D float32 tensor")
            self._check(self.lib.edaa_set_image_device(self.h, C.c_void_p(x.data_ptr()),
                                                       x.shape[0], x.shape[1], x.stride(0)))
            self.L, self.N = int(x.shape[0]), int(x.shape[1])
            return
        xf = np.ascontiguousarray(x)
        if xf.dtype != np.float64:
            xf = np.ascontiguousarray(xf, dtype=np.float32)
        self._x_keep = xf
        fn = self.lib.edaa_set_image_host_f64 if xf.dtype == np.float64 else self.lib.edaa_set_image_host
        self._check(fn(self.h, xf.ctypes.data_as(C.c_void_p), xf.shape[0], xf.shape[1]))
        self.L, self.N = xf.shape

    def lib_set_image_device_raw(self, x):
        """Test hook: hand a HOST array to edaa_set_image_device (must be rejected)."""
        xf = np.ascontiguousarray(x, dtype=np.float32)
        self._check(self.lib.edaa_set_image_device(self.h, xf.ctypes.data_as(C.c_void_p),
                                                   xf.shape[0], xf.shape[1], xf.shape[1]))

    def ingest(self, x) -> List[int]:
        """Validate + ℓ2-normalise a RAW L×N image on the device (image.cpp:10-47);
        it becomes this device's image.  Returns the zero pixels (left as they are)."""
        xr = np.ascontiguousarray(x, dtype=np.float64)
        if xr.ndim != 2:
            raise EdaaError("image: needs at least one band and one pixel")
        L, N = xr.shape
        zp = np.zeros(max(N, 1), dtype=np.uint64)
        nz = C.c_size_t()
        self._check(self.lib.edaa_ingest_host(self.h, xr.ctypes.data_as(C.c_void_p), L, N,
                                              zp.ctypes.data_as(C.c_void_p), zp.size, C.byref(nz)))
        self.L, self.N = L, N
        return [int(v) for v in zp[:nz.value]]

    def ingest_f32(self, x, pixel_major: bool = False) -> List[int]:
        """The same from an fp32 payload as stored: x is L×N (band-major) or,
        with pixel_major, the N×L payload of an (H, W, L) cube
        (edaa_ingest_host_f32).  Returns the zero pixels."""
        xr = np.ascontiguousarray(x, dtype=np.float32)
        if xr.ndim != 2:
            raise EdaaError("image: needs at least one band and one pixel")
        N, L = xr.shape if pixel_major else xr.shape[::-1]
        zp = np.zeros(max(N, 1), dtype=np.uint64)
        nz = C.c_size_t()
        self._check(self.lib.edaa_ingest_host_f32(self.h, xr.ctypes.data_as(C.c_void_p), L, N,
                                                  1 if pixel_major else 0, zp.ctypes.data_as(C.c_void_p),
                                                  zp.size, C.byref(nz)))
        self.L, self.N = L, N
        return [int(v) for v in zp[:nz.value]]

    def image(self):
        """(the device image as L×N fp64, its storage width in bytes: 4 or 8)."""
        out = np.zeros((self.L, self.N))
        xb = C.c_int()
        self._check(self.lib.edaa_image_get(self.h, out.ctypes.data_as(C.c_void_p), C.byref(xb)))
        return out, xb.value

    # -- solve ------------------------------------------------------------------
    def _params(self, p, T, K1, K2, seeds, gammas):
        self._seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        self._gammas = np.ascontiguousarray(gammas, dtype=np.float64)
        prm = SolveParams(p, T, K1, K2, len(self._seeds),
                          self._seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
                          self._gammas.ctypes.data_as(C.POINTER(C.c_double)))
        self.M, self.T, self.p = len(self._seeds), T, p
        return prm

    def solve_async(self, p, T, K1, K2, seeds, gammas):
        self._prm = self._params(p, T, K1, K2, seeds, gammas)
        self._check(self.lib.edaa_solve_async(self.h, C.byref(self._prm)))

    def finish(self):
        self._check(self.lib.edaa_finish(self.h))

    def solve(self, p, T, K1, K2, seeds, gammas):
        self.solve_async(p, T, K1, K2, seeds, gammas)
        self.finish()

    def solve_observed(self, p, T, K1, K2, seed, gamma, observer: Callable):
        prm = self._params(p, T, K1, K2, [seed], [gamma])
        N = self.N

        def cb(outer, block, inner, a_ptr, b_ptr, pp, n, user):
            a = np.ctypeslib.as_array(a_ptr, shape=(pp * n,)).reshape(pp, n).copy()
            b = np.ctypeslib.as_array(b_ptr, shape=(n * pp,)).reshape(n, pp).copy()
            observer(int(outer), block.decode() if isinstance(block, bytes) else block,
                     int(inner), a, b)

        fn = _lib.OBSERVER_FN(cb)
        self._check(self.lib.edaa_solve_observed(self.h, C.byref(prm), fn, None))
        del N

    # -- pixel sharding (include/edaa_b200.h) -------------------------
    @staticmethod
    def _nccl_first():
        # torch ships its own (newer) NCCL; it must be the copy the process binds
        # libnccl.so.2 to, so load it before the library resolves NCCL lazily.
        try:
            import torch  # noqa: F401
        except ImportError:
            pass

    def nccl_unique_id(self) -> bytes:
        """A fresh NCCL communicator id (rank 0 makes it, every rank joins with it)."""
        self._nccl_first()
        buf = C.create_string_buffer(128)
        rc = self.lib.edaa_nccl_unique_id(buf, 128)
        if rc != 0:
            raise EdaaError("edaa_nccl_unique_id failed (rc=%d): NCCL unavailable" % rc, rc)
        return buf.raw

    def set_pixel_shard(self, uid: Optional[bytes], rank: int, world: int):
        """Join the pixel-sharding communicator (collective over `world` ranks);
        uid None turns sharding off (world 1 with a uid: one-rank self-check)."""
        self._nccl_first()
        buf = C.create_string_buffer(uid, 128) if uid else None
        self._check(self.lib.edaa_set_pixel_shard(self.h, buf, 128 if uid else 0, int(rank), int(world)))

    def shard_pixels(self):
        """[first, end) pixel range this rank owned in the last solve."""
        a, b = C.c_size_t(), C.c_size_t()
        self._check(self.lib.edaa_shard_pixels(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_shard_emulation(self, world: int):
        """Development/test: launch every pass as `world` slice-range launches on this one
        device (the sharded decomposition without a collective); 0 or 1 turns it off."""
        self._check(self.lib.edaa_set_shard_emulation(self.h, int(world)))

    def set_shard_exchange(self, mode: int):
        """Per-pass exchange of a pixel-sharded solve: 0 allreduce of the rank-reduced L×Q / Q×Q /
        2Q blocks (default, north_star), 1 broadcast of every slice partial (bitwise)."""
        self._check(self.lib.edaa_set_shard_exchange(self.h, int(mode)))

    def set_pass_order(self, order: int):
        """Pass work-item order: 0 auto, 1 chunk-major, 2 slice-major, 3 interleaved (results are
        bitwise identical; include/edaa_b200.h)."""
        self._check(self.lib.edaa_set_pass_order(self.h, int(order)))

    # -- instrumentation ---------------------------------------------------------
    def profile_enable(self, on: bool = True):
        self._check(self.lib.edaa_profile_enable(self.h, int(on)))

    def profile(self):
        """Per kind (the init / A / B / obj passes, and the combine kernels between them):
        (summed device ms, launches) of the last solve."""
        pr = _lib.ProfileC()
        self._check(self.lib.edaa_profile_read(self.h, C.byref(pr)))
        return {k: (pr.ms[i], int(pr.launches[i])) for i, k in enumerate(("init", "A", "B", "obj", "combine"))}

    def launch_count(self) -> int:
        return int(self.lib.edaa_launch_count(self.h))

    def fp64_peak_tflops(self) -> float:
        out = C.c_double()
        self._check(self.lib.edaa_probe_fp64_peak(self.h, C.byref(out)))
        return out.value

    # -- results ----------------------------------------------------------------
    def record(self, run: int) -> RunRecordC:
        out = RunRecordC()
        self._check(self.lib.edaa_run_record_get(self.h, run, C.byref(out)))
        return out

    def traces(self) -> np.ndarray:
        out = np.zeros((self.M, self.T + 1))
        self._check(self.lib.edaa_traces(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def factors(self, run: int):
        A = np.zeros((self.p, self.N))
        B = np.zeros((self.N, self.p))
        E = np.zeros((self.L, self.p))
        self._check(self.lib.edaa_factors(self.h, run, A.ctypes.data_as(C.c_void_p),
                                          B.ctypes.data_as(C.c_void_p),
                                          E.ctypes.data_as(C.c_void_p)))
        return A, B, E

    def select(self, fit_slack: float):
        cand = np.zeros(self.M, dtype=np.uint8)
        sel = C.c_size_t()
        fmin = C.c_double()
        rc = self.lib.edaa_select(self.h, fit_slack, cand.ctypes.data_as(C.c_void_p),
                                  C.byref(sel), C.byref(fmin))
        if rc == _lib.EDAA_ERR_ALL_FAILED:
            raise EdaaError("every run failed", rc)
        self._check(rc)
        return [int(i) for i in np.flatnonzero(cand)], int(sel.value), fmin.value

    # -- primitives on the resident image ------------------------------------------
    def fit_l1(self, E, A) -> float:
        E = np.ascontiguousarray(E, dtype=np.float64)
        A = np.ascontiguousarray(A, dtype=np.float64)
        out = C.c_double()
        self._check(self.lib.edaa_fit_l1(self.h, E.ctypes.data_as(C.c_void_p),
                                         A.ctypes.data_as(C.c_void_p), E.shape[1], C.byref(out)))
        return out.value

    def _ba(self, B, A):
        B = np.ascontiguousarray(B, dtype=np.float64)
        A = np.ascontiguousarray(A, dtype=np.float64)
        if B.shape != (self.N, A.shape[0]) or A.shape[1] != self.N:
            raise EdaaError("shape mismatch (B %s, A %s, N %d)" % (B.shape, A.shape, self.N))
        return B, A

    def xb(self, B) -> np.ndarray:
        """X·B (L×p): matmul(x, b), solver.cpp:140."""
        B = np.ascontiguousarray(B, dtype=np.float64)
        y = np.zeros((self.L, B.shape[1]))
        self._check(self.lib.edaa_xb(self.h, B.ctypes.data_as(C.c_void_p), B.shape[1],
                                     y.ctypes.data_as(C.c_void_p)))
        return y

    def objective(self, B, A) -> float:
        """½‖X − XB·A‖² (objective_l2, solver.cpp:184-188)."""
        B, A = self._ba(B, A)
        out = C.c_double()
        self._check(self.lib.edaa_objective(self.h, B.ctypes.data_as(C.c_void_p),
                                            A.ctypes.data_as(C.c_void_p), A.shape[0], C.byref(out)))
        return out.value

    def grad_abundances(self, B, A) -> np.ndarray:
        """−(XB)ᵀ(X − XBA), p×N (solver.cpp:166-172)."""
        B, A = self._ba(B, A)
        g = np.zeros(A.shape)
        self._check(self.lib.edaa_grad_abundances(self.h, B.ctypes.data_as(C.c_void_p),
                                                  A.ctypes.data_as(C.c_void_p), A.shape[0],
                                                  g.ctypes.data_as(C.c_void_p)))
        return g

    def grad_contributions(self, B, A) -> np.ndarray:
        """−Xᵀ((X − XBA)Aᵀ), N×p (solver.cpp:174-182)."""
        B, A = self._ba(B, A)
        g = np.zeros(B.shape)
        self._check(self.lib.edaa_grad_contributions(self.h, B.ctypes.data_as(C.c_void_p),
                                                     A.ctypes.data_as(C.c_void_p), A.shape[0],
                                                     g.ctypes.data_as(C.c_void_p)))
        return g

    def estimate_abundances(self, E, iters: int, eta: float) -> np.ndarray:
        E = np.ascontiguousarray(E, dtype=np.float64)
        A = np.zeros((E.shape[1], self.N))
        self._check(self.lib.edaa_estimate_abundances(self.h, E.ctypes.data_as(C.c_void_p), E.shape[1],
                                                      int(iters), float(eta),
                                                      A.ctypes.data_as(C.c_void_p)))
        return A

    def check_iterate(self, m, outer: int, which: str) -> str:
        """check_iterate (solver.cpp:65-90) on the columns of `m`, on the device: '' if the
        iterate is fine, else the reference's message for the first failing check."""
        m = np.ascontiguousarray(m, dtype=np.float64)
        if which not in ("abundance", "contribution"):
            raise ValueError("which must be 'abundance' or 'contribution'")
        code = C.c_int(0)
        buf = C.create_string_buffer(192)
        self._check(self.lib.edaa_check_iterate(self.h, m.ctypes.data_as(C.c_void_p), m.shape[0], m.shape[1],
                                                int(outer), int(which == "contribution"), C.byref(code),
                                                buf, 192))
        return buf.value.decode() if code.value else ""


def _result(dev: Device, run_idx: int, seed: int, gamma: float, traces) -> RunResult:
    A, B, E = dev.factors(run_idx)
    rec = dev.record(run_idx)
    return RunResult(E, A, B, rec.fit_l1, rec.coherence, seed, gamma, traces[run_idx].copy())


def run(x, config: SolverConfig, observer: Optional[Callable] = None, device: int = 0) -> RunResult:
    """Algorithm 1 for one run (solver.cpp:190-238) on the GPU.

    observer(outer, block, inner, A, B) is called after every inner step, as the
    reference's StepObserver (solver.hpp:69-77)."""
    config.validate()
    dev = Device.get(device)
    _upload_image(dev, x)
    args = (config.endmembers, config.outer_iters, config.inner_iters_a, config.inner_iters_b)
    if observer is not None:
        dev.solve_observed(*args, config.seed, config.gamma, observer)
    else:
        dev.solve(*args, [config.seed], [config.gamma])
    rec = dev.record(0)
    if not rec.ok:
        raise EdaaError(rec.message.decode("utf-8"))
    return _result(dev, 0, config.seed, config.gamma, dev.traces())


def l2_normalize(x, device: int = 0):
    """l2_normalize (image.cpp:29-47) on the GPU, validation included; returns
    (normalised L×N fp64 image, zero pixels).  The image stays resident on the
    device for a following solve."""
    dev = Device.get(device)
    zero = dev.ingest(x)
    img, _ = dev.image()
    return img, zero


def ensemble_plan(config: EnsembleConfig, first: int = 0, count: Optional[int] = None):
    """Seeds and step factors of runs [first, first+count): seed = base + m, γ from
    that seed's first draw (ensemble.cpp:123-127)."""
    count = config.runs - first if count is None else count
    seeds, gammas = [], []
    for m in range(first, first + count):
        s = (config.base_seed + m) & _MASK
        seeds.append(s)
        gammas.append(sample_gamma(Prng(s), config.gamma_set))
    return seeds, gammas


def run_ensemble(x, config: EnsembleConfig, device: int = 0):
    """Algorithm 2 (ensemble.cpp:108-167): all M runs in ONE batched device solve,
    then selection on the device.  Returns (selected RunResult, SelectionReport)."""
    config.validate()
    dev = Device.get(device)
    _upload_image(dev, x)
    seeds, gammas = ensemble_plan(config)
    s = config.solver
    t0 = time.perf_counter()
    dev.solve(s.endmembers, s.outer_iters, s.inner_iters_a, s.inner_iters_b, seeds, gammas)
    wall = (time.perf_counter() - t0) * 1e3
    recs = []
    for m in range(config.runs):
        rc = dev.record(m)
        recs.append(RunRecord(m, seeds[m], gammas[m], rc.fit_l1 if rc.ok else 0.0,
                              rc.coherence if rc.ok else 0.0, wall, bool(rc.ok),
                              rc.message.decode("utf-8")))
    cand, sel, fmin = dev.select(config.fit_slack)
    report = SelectionReport(recs, cand, sel, fmin)
    return _result(dev, sel, seeds[sel], gammas[sel], dev.traces()), report


def fit_l1(x, E, A, device: int = 0) -> float:
    """Σ|X − E·A| (ensemble.cpp:29-39) on the GPU."""
    E = np.asarray(E, dtype=np.float64)
    A = np.asarray(A, dtype=np.float64)
    xf = validate_image(x)
    if E.shape[0] != xf.shape[0] or A.shape != (E.shape[1], xf.shape[1]):
        raise EdaaError("fit_l1: shape mismatch")
    dev = Device.get(device)
    dev.set_image(xf)
    return dev.fit_l1(E, A)


def _column_norm(E, j) -> float:
    s = 0.0  # sequential, as Matrix::column_norm (matrix.cpp:44-51); builtin sum() compensates
    for v in E[:, j]:
        s += float(v) * float(v)
    return float(np.sqrt(s))


def coherence(E, normalized: bool = False) -> float:
    """Largest off-diagonal endmember inner product (ensemble.cpp:41-60); a p×p
    host reduction, like the reference's."""
    E = np.asarray(E, dtype=np.float64)
    p = E.shape[1]
    best = -np.inf
    for i in range(p):
        for j in range(i + 1, p):
            dot = 0.0
            for r in range(E.shape[0]):
                dot += E[r, i] * E[r, j]
            if normalized:
                ni, nj = _column_norm(E, i), _column_norm(E, j)
                if ni == 0.0 or nj == 0.0:
                    continue
                dot /= ni * nj
            best = max(best, dot)
    return 0.0 if best == -np.inf else float(best)


def estimate_abundances(x, E, iters: int, eta: float, device: int = 0) -> np.ndarray:
    """A for fixed endmembers E, `iters` entropic steps from 1/p (solver.cpp:240-259)."""
    E = np.asarray(E, dtype=np.float64)
    xf = validate_image(x)
    if not np.all(np.isfinite(E)):
        raise EdaaError("estimate_abundances: non-finite input")
    if E.shape[0] != xf.shape[0]:
        raise EdaaError("estimate_abundances: band count mismatch")
    if E.ndim != 2 or E.shape[1] < 1:
        raise EdaaError("estimate_abundances: need at least one endmember")
    if not (eta > 0.0) or not np.isfinite(eta):
        raise EdaaError("estimate_abundances: eta must be positive")
    dev = Device.get(device)
    dev.set_image(xf)
    return dev.estimate_abundances(E, iters, eta)
