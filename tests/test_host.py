"""Host-side logic, the C-ABI surface and the synthetic generator (CPU only)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2209_11002_b200 import edaa, synth
from paper_2209_11002_b200 import _lib

HEADER = os.path.join(ROOT, "include", "edaa_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"EDAA_API\s+[\w\s\*]*?\b(edaa_\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("edaa_create", "edaa_set_image_host", "edaa_solve", "edaa_select",
                 "edaa_solve_observed", "edaa_factors", "edaa_traces", "edaa_run_record_get"):
        assert must in syms


def test_cuda_library_exports_every_declared_symbol():
    assert os.path.exists(_lib.CUDA_LIB), "libedaa_cuda.so not built"
    lib = ctypes.CDLL(_lib.CUDA_LIB)  # loads without a GPU; no compute call is made
    for s in declared_symbols():
        assert hasattr(lib, s), s
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(declared_symbols()) == bound, "ctypes binding out of sync with the header"


def test_capability_probe():
    lib = _lib.load()
    assert lib.edaa_max_endmembers() == 16 and lib.edaa_max_bands() == 320
    assert b"sm_100a" in lib.edaa_version()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(edaa.EdaaError, match="no CPU fallback"):
        edaa.Device(0)


def test_prng_matches_reference_stream():  # prng.hpp:15-26, test_core.cpp:14-35
    r = edaa.Prng(0)
    assert [r.next_u64() for _ in range(3)] == [0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4,
                                                 0x06c45d188009454f]
    r = edaa.Prng(1)
    assert r.next_unit() == 0.5665615751722809


def test_sample_gamma_and_plan():  # ensemble.cpp:62-69,117-139
    assert edaa.sample_gamma(edaa.Prng(0), edaa.DEFAULT_GAMMAS) == 8.0
    cfg = edaa.EnsembleConfig(runs=50, solver=edaa.SolverConfig(endmembers=3))
    seeds, gammas = edaa.ensemble_plan(cfg)
    assert seeds == list(range(50))
    assert gammas[0] == 8.0
    assert [i for i, g in enumerate(gammas) if g == 8.0] == [0, 23, 32, 36, 38, 44, 45]
    s2, g2 = edaa.ensemble_plan(cfg, first=20, count=5)
    assert s2 == seeds[20:25] and g2 == gammas[20:25]
    with pytest.raises(edaa.EdaaError, match="empty"):
        edaa.sample_gamma(edaa.Prng(0), [])


def test_config_validation_messages():  # solver.cpp:103-111, ensemble.cpp:17-27
    with pytest.raises(edaa.EdaaError, match="endmember count must be at least 2"):
        edaa.SolverConfig(endmembers=1).validate()
    with pytest.raises(edaa.EdaaError, match="iteration counts must be at least 1"):
        edaa.SolverConfig(endmembers=2, outer_iters=0).validate()
    with pytest.raises(edaa.EdaaError, match="gamma must be positive"):
        edaa.SolverConfig(endmembers=2, gamma=float("nan")).validate()
    ok = edaa.SolverConfig(endmembers=2)
    for kw, msg in [(dict(runs=0), "at least one run"), (dict(gamma_set=[]), "empty"),
                    (dict(gamma_set=[0.5, -1.0]), "finite and positive"),
                    (dict(fit_slack=0.9), "at least 1")]:
        with pytest.raises(edaa.EdaaError, match=msg):
            edaa.EnsembleConfig(solver=ok, **kw).validate()


def test_image_validation():  # image.cpp:10-27
    with pytest.raises(edaa.EdaaError, match="negative reflectance"):
        edaa.validate_image(np.array([[0.5, -0.1]]))
    with pytest.raises(edaa.EdaaError, match="non-finite"):
        edaa.validate_image(np.array([[0.5, np.nan]]))
    with pytest.raises(edaa.EdaaError, match="at least one band"):
        edaa.validate_image(np.zeros((0, 3)))
    assert edaa.validate_image(np.ones((2, 3))).dtype == np.float32       # fp32-exact → fast path
    assert edaa.validate_image(np.full((2, 3), 0.1)).dtype == np.float64  # kept exact in fp64


def test_select_runs_rule():  # ensemble.cpp:71-94, test_ensemble.cpp:38-65
    R = edaa.RunRecord
    rep = edaa.select_runs([R(0, fit_l1=10.0, coherence=0.9, ok=True),
                            R(1, fit_l1=10.4, coherence=0.8, ok=True),
                            R(2, fit_l1=11.0, coherence=0.1, ok=True)], 1.05)
    assert (rep.candidate_set, rep.selected, rep.fit_min) == ([0, 1], 1, 10.0)
    rep = edaa.select_runs([R(i, fit_l1=10.0 + 0.1 * i, coherence=0.5, ok=True) for i in range(3)],
                           1.05)
    assert rep.selected == 0
    with pytest.raises(edaa.EdaaError, match="every run failed"):
        edaa.select_runs([R(0, fit_l1=1.0, ok=False)], 1.05)


def test_select_rule_matches_oracle_on_random_records(oracle_kinds):
    if not oracle_kinds:
        pytest.skip("oracle not built")
    from oracle import Oracle
    orc = Oracle(oracle_kinds[0])
    rng = np.random.default_rng(0)
    for _ in range(50):
        m = int(rng.integers(1, 30))
        fits = rng.uniform(10, 11, m)
        mus = rng.choice([0.1, 0.2, 0.3], m)  # ties on purpose
        ok = rng.random(m) > 0.2
        if not ok.any():
            continue
        recs = [edaa.RunRecord(i, fit_l1=fits[i], coherence=mus[i], ok=bool(ok[i])) for i in range(m)]
        rep = edaa.select_runs(recs, 1.05)
        cand, sel, fmin = orc.select_runs(fits, mus, ok)
        assert (rep.candidate_set, rep.selected, rep.fit_min) == (cand, sel, fmin)


@pytest.mark.parametrize("name", ["cfg0", "cfg1", "cfg3"])
def test_synthetic_configs(name):
    spec = synth.CONFIGS[name]
    x, e, a = synth.generate(spec, pixels=2000)
    assert x.dtype == np.float32 and x.shape == (spec.bands, 2000)
    assert np.all(x >= 0)
    np.testing.assert_allclose(np.linalg.norm(x.astype(np.float64), axis=0), 1.0, atol=1e-6)
    np.testing.assert_allclose(a.sum(axis=0), 1.0, atol=1e-12)
    if spec.min_angle_deg:
        en = e / np.linalg.norm(e, axis=0)
        cos = np.clip(en.T @ en, -1, 1)
        ang = np.degrees(np.arccos(cos[np.triu_indices(spec.endmembers, 1)]))
        assert ang.min() >= spec.min_angle_deg
    x2 = synth.generate(spec, pixels=2000)[0]
    assert np.array_equal(x, x2)


def test_abundance_cap():
    spec = synth.CONFIGS["cfg2"]
    _, _, a = synth.generate(spec, pixels=5000)
    assert a.max() <= 0.8 + 1e-12
    np.testing.assert_allclose(a.sum(axis=0), 1.0, atol=1e-12)


def test_coherence_matches_oracle(oracle_kinds):  # ensemble.cpp:41-60, test_ensemble.cpp:91-116
    e = np.array([[1.0, 0.0], [0.0, 1.0], [0.8, 0.8]])
    assert edaa.coherence(np.array([[1.0], [2.0]])) == 0.0
    if not oracle_kinds:
        pytest.skip("oracle not built")
    from oracle import Oracle
    orc = Oracle(oracle_kinds[0])
    rng = np.random.default_rng(3)
    for _ in range(10):
        e = rng.random((int(rng.integers(1, 40)), int(rng.integers(2, 9))))
        for norm in (False, True):
            assert edaa.coherence(e, norm) == orc.coherence(e, norm)


def test_validate_image_reports_first_offending_element():
    """edaa.validate_image follows HsiImage::validate's scan order (image.cpp:10-27)."""
    from paper_2209_11002_b200 import edaa
    x = np.ones((3, 5))
    y = x.copy(); y[0, 4] = -1.0; y[2, 0] = np.nan
    with pytest.raises(edaa.EdaaError, match="negative reflectance"):
        edaa.validate_image(y)
    y = x.copy(); y[0, 4] = np.nan; y[2, 0] = -1.0
    with pytest.raises(edaa.EdaaError, match="non-finite reflectance"):
        edaa.validate_image(y)
