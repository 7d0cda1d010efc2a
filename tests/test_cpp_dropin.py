"""The C++ drop-in (include/archetype/*.hpp → libarchetype_b200.so).

CPU: the library exports the reference API's symbols and the test binary links.
GPU: the restated reference unit tests + the A/B against the reference build pass.
"""
import os
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2209_11002_b200", "libarchetype_b200.so")
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")

# The reference's public hot-path API (include/archetype/{solver,ensemble,matrix}.hpp).
API = ["archetype::run(", "archetype::run_ensemble(", "archetype::select_runs(",
       "archetype::fit_l1(", "archetype::coherence(", "archetype::sample_gamma(",
       "archetype::resolve_workers(", "archetype::step_sizes(", "archetype::entropic_step(",
       "archetype::grad_abundances(", "archetype::grad_contributions(",
       "archetype::objective_l2(", "archetype::estimate_abundances(",
       "archetype::init_abundances(", "archetype::init_contributions(",
       "archetype::matmul(", "archetype::matmul_tn(", "archetype::matmul_nt(",
       "archetype::spectral_norm(", "archetype::l2_normalize(",
       "archetype::SolverConfig::validate()", "archetype::EnsembleConfig::validate()",
       "archetype::HsiImage::validate()", "archetype::validate_simplex_columns(",
       # formats, output bundle, scoring, generator, front end
       "archetype::read_npy(", "archetype::write_npy(", "archetype::npy_to_matrix(",
       "archetype::npy_to_image(", "archetype::read_envi(", "archetype::envi_data_path(",
       "archetype::report_to_json(", "archetype::report_from_json(", "archetype::evaluation_to_json(",
       "archetype::write_csv_endmembers(", "archetype::read_csv_endmembers(", "archetype::write_pgm(",
       "archetype::write_outputs(", "archetype::evaluate_unmixing(", "archetype::match_endmembers(",
       "archetype::min_cost_assignment(", "archetype::spectral_angle_deg(", "archetype::rmse_percent(",
       "archetype::sad_degrees(", "archetype::format_evaluation(", "archetype::generate(",
       "archetype::cli_main("]


def test_library_exports_reference_api():
    out = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True).stdout
    out = out.replace("[abi:cxx11]", "")  # functions returning std::string carry the ABI tag
    for sym in API:
        assert sym in out, sym


def test_test_binary_links():
    assert os.path.exists(BIN), "tests/cpp/build/test_dropin missing (make -C tests/cpp)"
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libarchetype_b200.so" in out and "not found" not in out


@pytest.mark.gpu
def test_restated_reference_unit_tests_pass_on_gpu():
    r = subprocess.run([BIN], capture_output=True, text=True, cwd=ROOT, timeout=600)
    print(r.stdout)
    print(r.stderr)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "A/B" in r.stdout


CLI_TEST = os.path.join(ROOT, "tests", "cpp", "build", "test_cli")
CLI_BIN = os.path.join(ROOT, "paper_2209_11002_b200", "archetype")


@pytest.mark.gpu
def test_cli_unmix_pipeline_on_gpu():
    """tests/cpp/test_cli.cpp [gpu] cases (the reference's test_cli.cpp:167-250):
    synth → unmix (one batched GPU solve of 50 runs) → evaluate recovers the
    planted endmembers; report.json replays the selected run bitwise through
    archetype::run; spatial cubes get PGM maps."""
    r = subprocess.run([CLI_TEST, "gpu:"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    print(r.stdout)
    print(r.stderr)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 failures" in r.stdout and "[ ok ] gpu: report fields replay" in r.stdout


@pytest.mark.gpu
def test_cli_binary_runs_unmix_end_to_end(tmp_path):
    """The shipped `archetype` executable (the reference's tools/main.cpp)."""
    run = lambda *a: subprocess.run([CLI_BIN, *map(str, a)], capture_output=True, text=True, timeout=300)
    s = run("synth", "--bands", 16, "--pixels", 300, "--endmembers", 3, "--snr", 40, "--seed", 4,
            "--output", tmp_path / "fx")
    assert s.returncode == 0, s.stderr
    u = run("unmix", "--input", tmp_path / "fx" / "cube.npy", "--endmembers", 3, "--runs", 8,
            "--outer", 30, "--output", tmp_path / "est")
    assert u.returncode == 0, u.stderr
    assert "selected: run" in u.stdout
    for f in ("endmembers.csv", "abundances.npy", "report.json"):
        assert (tmp_path / "est" / f).exists()
    e = run("evaluate", "--est", tmp_path / "est", "--gt-endmembers", tmp_path / "fx" / "endmembers.csv",
            "--gt-abundances", tmp_path / "fx" / "abundances.npy")
    assert e.returncode == 0 and "overall" in e.stdout, e.stderr


ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


@pytest.mark.skipif(not os.path.exists(ACC), reason="oracle/_ref/acceptance_b200 not built "
                    "(make -C oracle acceptance, needs the reference sources)")
def test_reference_acceptance_gate_links_against_dropin():
    out = subprocess.run(["ldd", ACC], capture_output=True, text=True).stdout
    assert "libarchetype_b200.so" in out and "not found" not in out


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(ACC), reason="oracle/_ref/acceptance_b200 not built")
def test_reference_acceptance_gate_passes_on_gpu():
    """The reference's own release gate (proj/tests/acceptance.cpp, built in place
    against include/archetype and libarchetype_b200.so) — every check except the
    absent-dataset Samson check (acceptance.cpp:323-346) must pass on the GPU."""
    r = subprocess.run([ACC], capture_output=True, text=True, cwd=ROOT, timeout=900)
    print(r.stdout)
    print(r.stderr)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "all checks passed" in r.stdout
    assert r.stdout.count("PASS") >= 8


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["<f8", "<f4"])
def test_cli_device_ingest_equals_host_normalisation(tmp_path, dtype):
    """`unmix` normalises through the device ingest; ARCHETYPE_HOST_NORMALIZE=1
    takes the reference's host fp64 route. The bundles are identical (but for
    the measured wall_ms), and the error messages come in the reference's
    order: a bad value before a bad config, a wavelength mismatch before
    "degenerate input"."""
    import json
    import numpy as np

    def unmix(cube, out, *extra, host=False):
        env = dict(os.environ, ARCHETYPE_HOST_NORMALIZE="1" if host else "0")
        return subprocess.run([CLI_BIN, "unmix", "--input", cube, "--endmembers", "3", "--runs", "6",
                               "--outer", "15", "--output", out, *extra], capture_output=True, text=True,
                              env=env, timeout=300)

    rng = np.random.default_rng(11)
    x = rng.random((5, 7, 19)) ** 2 + 0.01   # (H, W, L): not fp32-exact after normalising
    x[2, 3, :] = 0.0                          # one zero pixel, left unnormalised
    x = x.astype(dtype)                       # <f4: the fp32 payload ingest (no host widening)
    np.save(tmp_path / "cube.npy", x)
    a = unmix(str(tmp_path / "cube.npy"), str(tmp_path / "dev"))
    b = unmix(str(tmp_path / "cube.npy"), str(tmp_path / "host"), host=True)
    assert a.returncode == 0 and b.returncode == 0, a.stderr + b.stderr
    for f in ("abundances.npy", "endmembers.csv", "maps/endmember_1.pgm", "maps/endmember_3.pgm"):
        assert (tmp_path / "dev" / f).read_bytes() == (tmp_path / "host" / f).read_bytes(), f
    ra, rb = (json.loads((tmp_path / d / "report.json").read_text()) for d in ("dev", "host"))
    assert ra["zero_pixels"] == rb["zero_pixels"] == 1
    for r in ra["runs"] + rb["runs"]:
        r.pop("wall_ms")
    assert ra == rb

    bad = x.copy()
    bad[1, 1, 4] = -0.5
    np.save(tmp_path / "bad.npy", bad)
    for host in (False, True):
        r = unmix(str(tmp_path / "bad.npy"), str(tmp_path / "o"), "--gamma-set", "0", host=host)
        assert r.returncode == 2 and "image: negative reflectance" in r.stderr, r.stderr
        r = unmix(str(tmp_path / "cube.npy"), str(tmp_path / "o"), "--gamma-set", "0", host=host)
        assert r.returncode == 2 and "step factors must be finite and positive" in r.stderr, r.stderr
    (tmp_path / "z.hdr").write_text("ENVI\nsamples = 2\nlines = 2\nbands = 3\ndata type = 5\n"
                                    "interleave = bsq\nwavelength = {1, 2}\n")
    (tmp_path / "z.img").write_bytes(bytes(8 * 12))
    for host in (False, True):
        r = unmix(str(tmp_path / "z.hdr"), str(tmp_path / "o"), host=host)
        assert r.returncode == 2 and "wavelength list length differs" in r.stderr, r.stderr
    (tmp_path / "z.hdr").write_text("ENVI\nsamples = 2\nlines = 2\nbands = 3\ndata type = 5\ninterleave = bsq\n")
    for host in (False, True):
        r = unmix(str(tmp_path / "z.hdr"), str(tmp_path / "o"), host=host)
        assert r.returncode == 2 and "degenerate input: all pixels are zero" in r.stderr, r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [2, 3])
def test_multi_device_run_ensemble_equals_single_device(tmp_path, devices):
    """run_ensemble's multi-device branch (csrc/host/ensemble.cpp: one host thread
    and one contiguous shard of the runs per device context, records merged, the
    host select_runs, factors fetched from the owner) — the GPU analogue of the
    reference's worker-count determinism (ensemble.cpp:141-162,
    test_ensemble.cpp:118-148).  EDAA_VIRTUAL_DEVICES places that many contexts on
    this one GPU; the bundle must equal the single-context one byte for byte
    (a run's arithmetic does not depend on its batch), but for wall_ms."""
    import json
    run = lambda env, *a: subprocess.run([CLI_BIN, *map(str, a)], capture_output=True, text=True, timeout=300,
                                         env=dict(os.environ, **env))
    s = run({}, "synth", "--bands", 20, "--pixels", 900, "--endmembers", 4, "--snr", 35, "--seed", 9,
            "--output", tmp_path / "fx")
    assert s.returncode == 0, s.stderr
    outs = {}
    for name, env in (("one", {}), ("many", {"EDAA_VIRTUAL_DEVICES": str(devices)})):
        u = run(env, "unmix", "--input", tmp_path / "fx" / "cube.npy", "--endmembers", 4, "--runs", 11,
                "--outer", 25, "--output", tmp_path / name, "--json")
        assert u.returncode == 0, u.stderr
        outs[name] = json.loads(u.stdout)
    for f in ("abundances.npy", "endmembers.csv"):
        assert (tmp_path / "one" / f).read_bytes() == (tmp_path / "many" / f).read_bytes(), f
    for rep in outs.values():
        for r in rep["runs"]:
            r.pop("wall_ms")
    assert outs["one"] == outs["many"]
    assert len(outs["one"]["runs"]) == 11
