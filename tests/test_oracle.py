"""The CPU oracle, pinned before it is trusted (CPU only).

* every golden vector / known-answer test of the reference's own unit tests for
  this path (test_core.cpp, test_solver.cpp, test_ensemble.cpp);
* the C restatement (oracle/edaa_oracle.c) is BITWISE equal to the reference
  built from its sources (oracle/_ref) on run() and run_ensemble();
* the committed golden fixtures (tests/golden/, made by make_golden.py from the
  reference) are reproduced bitwise by the restatement.
"""
import math
import os

import numpy as np
import pytest

from conftest import golden_files, golden_scene, load_golden
from oracle import Oracle, OracleError, available_kinds

KINDS = available_kinds()
pytestmark = pytest.mark.skipif(not KINDS, reason="oracle not built (make -C oracle)")


@pytest.fixture(params=KINDS)
def orc(request):
    return Oracle(request.param)


def test_prng_published_stream(orc):  # test_core.cpp:14-35
    assert list(orc.prng_u64(0, 3)) == [0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4, 0x06c45d188009454f]
    assert list(orc.prng_u64(1, 2)) == [0x910a2dec89025cc1, 0xbeeb8da1658eec67]
    assert list(orc.prng_unit(0, 4)) == [0.8833108082136426, 0.43152799704850997,
                                         0.026433771592597743, 0.9708819781538285]
    assert list(orc.prng_unit(1, 2)) == [0.5665615751722809, 0.7457817572627011]
    u = orc.prng_unit(1234567, 10000)
    assert np.all(u >= 0) and np.all(u < 1)


def test_gamma_sampling(orc):  # test_ensemble.cpp:67-89
    g = orc.sample_gamma(0, 2)
    assert list(g) == [8.0, 1.0]
    draws = orc.sample_gamma(123, 70000)
    counts = [int(np.sum(draws == v)) for v in (0.125, 0.25, 0.5, 1.0, 2.0, 4.0, 8.0)]
    assert sum(counts) == 70000
    assert all(10000 - 600 < c < 10000 + 600 for c in counts)


def test_init_contributions_golden(orc):  # test_solver.cpp:41-61
    b = orc.init_contributions(3, 2, 0)
    u = np.array([0.8833108082136426, 0.43152799704850997, 0.026433771592597743])
    sc = np.exp(0.1 * u - 0.1 * u[0])
    np.testing.assert_allclose(b[:, 0], sc / sc.sum(), rtol=1e-15)
    assert np.all((b > 0.30) & (b < 0.37))
    np.testing.assert_allclose(b.sum(axis=0), 1.0, atol=1e-12)


def test_entropic_step_closed_forms(orc):  # test_solver.cpp:79-127
    out = orc.entropic_step([0.5, 0.5], [1.0, 0.0], 1.0)
    np.testing.assert_allclose(out, [0.2689414213699951, 0.7310585786300049], rtol=1e-15)
    out = orc.entropic_step([0.2, 0.3, 0.5], [0.1, -0.2, 0.3], 2.0)
    np.testing.assert_allclose(out, [0.18487779792018505, 0.5053039670477497, 0.3098182350320652],
                               rtol=1e-14)
    out = orc.entropic_step([0.0, 1.0], [-100.0, 0.0], 1.0)  # floor lifts the zero
    assert np.all(np.isfinite(out)) and out[0] > 0 and abs(out.sum() - 1) < 1e-12
    with pytest.raises(OracleError, match="eta must be positive"):
        orc.entropic_step([0.5, 0.5], [1.0, 0.0], 0.0)


def test_spectral_norm_known_values(orc):  # test_core.cpp:80-107
    m = np.array([1.0, 2.0, 0.5, -1.0, 0.0, 3.0, 1.5, 2.0, -2.0, 0.25, 1.0, 0.0]).reshape(3, 4)
    assert orc.spectral_norm(m) == pytest.approx(4.185922592173704, rel=1e-6)
    u = np.array([1.0, -2.0, 2.0])
    assert orc.spectral_norm(np.outer(u, u)) == pytest.approx(9.0, rel=1e-9)
    assert orc.spectral_norm(np.eye(5)) == pytest.approx(1.0, rel=1e-9)
    with pytest.raises(OracleError, match="finite and nonzero"):
        orc.spectral_norm(np.zeros((3, 2)))


def test_step_sizes_formula(orc):  # test_solver.cpp:63-77
    rng = np.random.default_rng(3)
    x = rng.random((5, 40))
    b0 = orc.init_contributions(40, 4, 9)
    ea, eb = orc.step_sizes(x, b0, 2.0)
    sigma = orc.spectral_norm(x @ b0)
    assert ea == pytest.approx(2.0 / sigma**2, rel=1e-12)
    assert eb == pytest.approx(math.sqrt(4 / 40) * ea, rel=1e-12)
    ea2, eb2 = orc.step_sizes(x, b0, 4.0)
    assert ea2 == pytest.approx(2 * ea, rel=1e-12) and eb2 == pytest.approx(2 * eb, rel=1e-12)


def test_selection_rules(orc):  # test_ensemble.cpp:38-65
    cand, sel, fmin = orc.select_runs([10.0, 10.4, 11.0], [0.9, 0.8, 0.1], [1, 1, 1])
    assert (cand, sel, fmin) == ([0, 1], 1, 10.0)
    cand, sel, _ = orc.select_runs([10.0, 10.1, 10.2], [0.5, 0.5, 0.5], [1, 1, 1])
    assert (cand, sel) == ([0, 1, 2], 0)
    cand, sel, fmin = orc.select_runs([1.0, 10.0, 10.2], [0.0, 0.9, 0.3], [0, 1, 1])
    assert (cand, sel, fmin) == ([1, 2], 2, 10.0)
    with pytest.raises(OracleError, match="every run failed"):
        orc.select_runs([1.0], [0.0], [0])


def test_coherence_and_fit(orc):  # test_ensemble.cpp:91-116
    e = np.zeros((3, 3))
    e[0, 0] = e[1, 1] = 1.0
    e[0, 2], e[1, 2] = 0.6, 0.8
    assert orc.coherence(e) == pytest.approx(0.8, rel=1e-12)
    e2 = e.copy()
    e2[:, 2] *= 2
    assert orc.coherence(e2) == pytest.approx(1.6, rel=1e-12)
    assert orc.coherence(e2, normalized=True) == pytest.approx(0.8, rel=1e-12)
    x = np.array([[1.0, 0.0], [0.0, 1.0]])
    assert orc.fit_l1(x, np.eye(2), np.full((2, 2), 0.5)) == pytest.approx(2.0, rel=1e-12)


def test_run_invariants(orc):  # test_solver.cpp:163-212
    rng = np.random.default_rng(5)
    x = rng.random((6, 30))
    r1 = orc.run(x, 3, T=8, gamma=1.0, seed=17)
    assert len(r1.trace) == 9 and r1.trace[-1] < r1.trace[0]
    np.testing.assert_allclose(r1.A.sum(axis=0), 1, atol=1e-9)
    np.testing.assert_allclose(r1.B.sum(axis=0), 1, atol=1e-9)
    r2 = orc.run(x, 3, T=8, gamma=1.0, seed=17)
    assert np.array_equal(r1.A, r2.A) and np.array_equal(r1.B, r2.B)
    r3 = orc.run(x, 3, T=8, gamma=1.0, seed=18)
    assert not np.array_equal(r1.B, r3.B)
    for bad, msg in [(dict(p=1), "at least 2"), (dict(gamma=0.0), "gamma must be positive"),
                     (dict(T=0), "iteration counts")]:
        kw = dict(p=2, T=3, gamma=1.0)
        kw.update(bad)
        with pytest.raises(OracleError, match=msg):
            orc.run(x, kw["p"], T=kw["T"], gamma=kw["gamma"])


@pytest.mark.skipif(not {"port", "reference"} <= set(KINDS), reason="needs both oracles")
@pytest.mark.parametrize("p,gamma,seed", [(3, 8.0, 5), (4, 0.5, 13), (6, 2.0, 1)])
def test_port_bitwise_equals_reference_run(p, gamma, seed):
    from paper_2209_11002_b200 import synth
    x = synth.small_scene(30, 400, p, seed=seed).astype(np.float64)
    a = Oracle("reference").run(x, p, T=20, gamma=gamma, seed=seed)
    b = Oracle("port").run(x, p, T=20, gamma=gamma, seed=seed)
    for f in ("trace", "A", "B", "E"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.fit_l1 == b.fit_l1 and a.coherence == b.coherence


@pytest.mark.skipif(not {"port", "reference"} <= set(KINDS), reason="needs both oracles")
def test_port_bitwise_equals_reference_ensemble():
    from paper_2209_11002_b200 import synth
    x = synth.small_scene(20, 300, 3, seed=2).astype(np.float64)
    a = Oracle("reference").run_ensemble(x, 3, M=12, T=10, workers=3)
    b = Oracle("port").run_ensemble(x, 3, M=12, T=10, workers=5)
    assert np.array_equal(a.fits, b.fits) and np.array_equal(a.mus, b.mus)
    assert np.array_equal(a.gammas, b.gammas)
    assert (a.candidates, a.selected) == (b.candidates, b.selected)
    assert np.array_equal(a.A, b.A)


@pytest.mark.skipif("port" not in KINDS, reason="port oracle not built")
@pytest.mark.parametrize("name", [f for f in golden_files() if not f.startswith(("cfg", "c4"))])
def test_port_reproduces_golden(name):
    g = load_golden(name)
    x = golden_scene(g).astype(np.float64)
    orc = Oracle("port")
    if str(g["kind"]) == "run":
        r = orc.run(x, int(g["p"]), T=int(g["T"]), gamma=float(g["gamma"]), seed=int(g["seed"]))
        assert np.array_equal(r.trace, g["trace"]) and np.array_equal(r.A, g["A"])
        assert np.array_equal(r.B, g["B"]) and np.array_equal(r.E, g["E"])
    else:
        e = orc.run_ensemble(x, int(g["p"]), M=int(g["M"]), T=int(g["T"]))
        assert np.array_equal(e.fits, g["fits"]) and e.selected == int(g["selected"])
        assert e.candidates == [int(c) for c in g["candidates"]]


@pytest.mark.parametrize("seed", [0, 1])
def test_l2_normalize_restatement_matches_reference(seed):
    """image.cpp:29-47 restated in oracle/edaa_oracle.c: bitwise the reference,
    zero pixels listed and left as they are."""
    from oracle import Oracle
    if "reference" not in available_kinds():
        pytest.skip("reference oracle not built")
    rng = np.random.default_rng(seed)
    x = rng.random((13, 300)) ** 3
    x[:, [0, 77, 299]] = 0.0
    a, za = Oracle("reference").l2_normalize(x)
    b, zb = Oracle("port").l2_normalize(x)
    assert np.array_equal(a, b) and za == zb == [0, 77, 299]
    assert np.array_equal(a[:, 77], x[:, 77])


@pytest.mark.parametrize("kind", ["reference", "port"])
def test_l2_normalize_error_messages_follow_scan_order(kind):
    """HsiImage::validate throws at the first offending element (row-major)."""
    from oracle import Oracle, OracleError
    if kind not in available_kinds():
        pytest.skip("oracle not built")
    x = np.ones((4, 9))
    y = x.copy(); y[1, 2] = -1.0; y[3, 0] = np.nan
    with pytest.raises(OracleError, match="negative reflectance"):
        Oracle(kind).l2_normalize(y)
    y = x.copy(); y[1, 2] = np.inf; y[3, 0] = -2.0
    with pytest.raises(OracleError, match="non-finite reflectance"):
        Oracle(kind).l2_normalize(y)
    with pytest.raises(OracleError, match="degenerate input: all pixels are zero"):
        Oracle(kind).l2_normalize(np.zeros((3, 5)))


@pytest.mark.skipif("reference" not in KINDS, reason="compiled reference not built")
def test_reference_check_iterate_messages_and_scan_order():
    """check_iterate (solver.cpp:65-90), reached through the veneer: per column,
    rows top to bottom, the first non-finite or negative entry wins, the sum
    check comes after the column; the first failing column decides."""
    orc = Oracle("reference")
    a = np.full((3, 4), 1.0 / 3.0)
    assert orc.check_iterate(a, 1, "abundance") is None
    m = a.copy(); m[2, 1] = np.nan
    assert orc.check_iterate(m, 7, "abundance") == "non-finite abundance iterate at outer iteration 7"
    m = a.copy(); m[1, 2] = -1e-300
    assert orc.check_iterate(m, 2, "abundance") == "abundance iterate left the simplex at outer iteration 2"
    m = a.copy(); m[0, 0] += 2e-9
    assert orc.check_iterate(m, 3, "contribution") == "contribution column sum drifted from 1 at outer iteration 3"
    m = a.copy(); m[0, 0] += 1e-10          # within tolerance
    assert orc.check_iterate(m, 3, "abundance") is None
    m = a.copy(); m[0, 1] += 2e-9; m[2, 1] = np.inf   # same column: the entry check comes first
    assert orc.check_iterate(m, 4, "abundance").startswith("non-finite")
    m = a.copy(); m[0, 1] += 2e-9; m[2, 3] = np.inf   # earlier column's drift wins
    assert "drifted" in orc.check_iterate(m, 4, "abundance")


@pytest.mark.skipif("reference" not in KINDS, reason="compiled reference not built")
def test_reference_primitives_follow_their_definitions():
    """The new veneer exports (grad_*, objective_l2, estimate_abundances) against
    their definitions in numpy (solver.cpp:166-188,240-259)."""
    orc = Oracle("reference")
    rng = np.random.default_rng(3)
    x = rng.random((6, 40)); b = rng.dirichlet(np.ones(40), 3).T; a = rng.dirichlet(np.ones(3), 40).T
    r = x - x @ b @ a
    assert abs(orc.objective_l2(x, b, a) - 0.5 * np.sum(r * r)) <= 1e-13
    assert np.abs(orc.grad_abundances(x, b, a) + (x @ b).T @ r).max() <= 1e-13
    assert np.abs(orc.grad_contributions(x, b, a) + x.T @ (r @ a.T)).max() <= 1e-13
    e = rng.random((6, 3))
    est = orc.estimate_abundances(x, e, 5, 0.5)
    assert est.shape == (3, 40) and np.allclose(est.sum(axis=0), 1.0)
    with pytest.raises(OracleError, match="eta must be positive"):
        orc.estimate_abundances(x, e, 5, 0.0)
