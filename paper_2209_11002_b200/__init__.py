"""B200-native EDAA (arXiv 2209.11002): entropic-descent archetypal analysis.

The hot path — Algorithm 1 batched over the ensemble plus Algorithm 2's model
selection — runs as hand-written sm_100a kernels behind the C-ABI in
``include/edaa_b200.h``.  The reference's C++ API (``include/archetype/``) is
provided by ``libarchetype_b200.so``; this package is the Python surface of
the same C-ABI (used by the tests and the benchmark).
"""
from .edaa import (  # noqa: F401
    Prng, SolverConfig, EnsembleConfig, RunResult, RunRecord, SelectionReport, EdaaError,
    Device, run, run_ensemble, select_runs, sample_gamma, DEFAULT_GAMMAS,
)

__version__ = "0.1.0"
