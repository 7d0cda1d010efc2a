"""the formats and scoring either side of the solver.

Our npy / envi / csv / report.json / output-bundle / metrics / synth code
(csrc/host/{npy,envi,outputs,metrics,synth}.cpp in libarchetype_b200.so) is
driven by tests/cpp/io_tool.cpp; the same driver compiled against the
UNMODIFIED reference sources is oracle/_ref/io_tool_ref (oracle/Makefile).
Each case runs both on the same inputs and requires identical exit codes,
identical stdout (values printed as hex floats, error messages verbatim) and
byte-identical output files. Pure host work: runs in the CPU suite.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

OURS = os.path.join(ROOT, "tests", "cpp", "build", "io_tool")
REF = os.path.join(ROOT, "oracle", "_ref", "io_tool_ref")
CLI_TEST = os.path.join(ROOT, "tests", "cpp", "build", "test_cli")

pytestmark = pytest.mark.skipif(not (os.path.exists(OURS) and os.path.exists(REF)),
                                reason="io_tool / io_tool_ref not built (build(); needs the reference sources)")


def save(path, arr):
    np.save(path, np.ascontiguousarray(arr))  # C order: the format both readers accept


def both(*args, cwd=None):
    r = subprocess.run([REF, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=120)
    o = subprocess.run([OURS, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=120)
    return r, o


def same(*args, expect_error=None):
    r, o = both(*args)
    assert (o.returncode, o.stdout) == (r.returncode, r.stdout), (args, r.stdout[-800:], o.stdout[-800:])
    if expect_error is not None:
        assert r.returncode == 3 and expect_error in r.stdout, r.stdout
    else:
        assert r.returncode == 0, r.stdout
    return r.stdout


def same_tree(a, b):
    fa = sorted(os.path.relpath(os.path.join(d, f), a) for d, _, fs in os.walk(a) for f in fs)
    fb = sorted(os.path.relpath(os.path.join(d, f), b) for d, _, fs in os.walk(b) for f in fs)
    assert fa == fb
    for f in fa:
        with open(os.path.join(a, f), "rb") as x, open(os.path.join(b, f), "rb") as y:
            assert x.read() == y.read(), f
    return fa


@pytest.mark.parametrize("spec", [
    (12, 40, 3, 1.0, 1, 7, "-"), (20, 500, 3, 0.1, 1, 0, "-"), (8, 60, 2, 1.0, 0, 3, "-"),
    (30, 200, 5, 0.5, 0, 11, "30"), (16, 100, 4, 2.5, 1, 2**63 + 5, "25.5"), (6, 6, 6, 0.05, 0, 1, "0")])
def test_synth_fixture_bytes_match_reference(tmp_path, spec):
    ra, oa = tmp_path / "r", tmp_path / "o"
    ra.mkdir(), oa.mkdir()
    r = subprocess.run([REF, "synth", *map(str, spec), ra], capture_output=True, text=True)
    o = subprocess.run([OURS, "synth", *map(str, spec), oa], capture_output=True, text=True)
    assert r.returncode == o.returncode == 0, (r.stdout, o.stdout)
    assert same_tree(ra, oa) == ["abundances.npy", "cube.npy", "endmembers.csv"]


def test_synth_spec_errors_match_reference(tmp_path):
    for spec in [(2, 10, 5, 1.0, 0, 0, "-"), (10, 10, 1, 1.0, 0, 0, "-"), (10, 3, 4, 1.0, 0, 0, "-"),
                 (10, 10, 3, 0.0, 0, 0, "-"), (10, 10, 3, 1.0, 0, 0, "inf")]:
        same("synth", *spec, tmp_path, expect_error="synth spec")


def _npy_cases(d):
    rng = np.random.default_rng(0)
    cases = {}
    for name, arr in {"f8_2d": rng.random((5, 7)), "f4_2d": rng.random((4, 3)).astype("<f4"),
                      "f8_1d": rng.random(6), "f8_3d": rng.random((2, 3, 4)),
                      "f4_3d": rng.random((3, 2, 5)).astype("<f4"), "empty_rows": np.zeros((0, 3))}.items():
        p = os.path.join(d, name + ".npy")
        save(p, arr)
        cases[name] = p
    p = os.path.join(d, "v2.npy")
    with open(p, "wb") as f:
        np.lib.format.write_array(f, rng.random((3, 2)), version=(2, 0))
    cases["v2"] = p
    raw = {  # hand-made headers: (header dict text, payload bytes, version)
        "fortran": ("{'descr': '<f8', 'fortran_order': True, 'shape': (2, 2), }", bytes(32), 1),
        "int": ("{'descr': '<i4', 'fortran_order': False, 'shape': (2,), }", bytes(8), 1),
        "bigendian": ("{'descr': '>f8', 'fortran_order': False, 'shape': (2,), }", bytes(16), 1),
        "no_descr": ("{'fortran_order': False, 'shape': (2,), }", bytes(16), 1),
        "no_shape": ("{'descr': '<f8', 'fortran_order': False, }", bytes(16), 1),
        "no_order": ("{'descr': '<f8', 'shape': (2,), }", bytes(16), 1),
        "bad_order": ("{'descr': '<f8', 'fortran_order': 0, 'shape': (2,), }", bytes(16), 1),
        "scalar": ("{'descr': '<f8', 'fortran_order': False, 'shape': (), }", bytes(8), 1),
        "bad_shape": ("{'descr': '<f8', 'fortran_order': False, 'shape': (2, x), }", bytes(16), 1),
        "neg_shape": ("{'descr': '<f8', 'fortran_order': False, 'shape': (-2,), }", bytes(16), 1),
        "no_paren": ("{'descr': '<f8', 'fortran_order': False, 'shape': 2, }", bytes(16), 1),
        "blank_items": ("{'descr': '<f8', 'fortran_order': False, 'shape': ( 2 , ,3 ,), }", bytes(48), 1),
        "truncated_data": ("{'descr': '<f8', 'fortran_order': False, 'shape': (4,), }", bytes(24), 1),
        "unterminated": ("{'descr': '<f8, 'fortran_order': False, 'shape': (2,), }", bytes(16), 1),
        "v3": ("{'descr': '<f8', 'fortran_order': False, 'shape': (2,), }", bytes(16), 3),
    }
    for name, (hdr, payload, ver) in raw.items():
        p = os.path.join(d, name + ".npy")
        h = hdr.encode()
        with open(p, "wb") as f:
            f.write(b"\x93NUMPY" + bytes([ver, 0]))
            f.write(len(h).to_bytes(2 if ver == 1 else 4, "little") + h + payload)
        cases[name] = p
    for name, blob in {"bad_magic": b"\x93NUMPX\x01\x00\x10\x00", "short": b"\x93NU",
                       "trunc_header": b"\x93NUMPY\x01\x00\x50\x00{'descr'"}.items():
        p = os.path.join(d, name + ".npy")
        with open(p, "wb") as f:
            f.write(blob)
        cases[name] = p
    cases["absent"] = os.path.join(d, "absent.npy")
    return cases


def test_read_npy_matches_reference_on_good_and_bad_files(tmp_path):
    errors = 0
    for name, path in _npy_cases(str(tmp_path)).items():
        r, o = both("npy", path)
        assert (o.returncode, o.stdout) == (r.returncode, r.stdout), (name, r.stdout[-400:], o.stdout[-400:])
        errors += r.returncode != 0
        if name in ("f8_2d", "f4_3d", "v2", "f8_3d"):
            r, o = both("image", path)
            assert (o.returncode, o.stdout) == (r.returncode, r.stdout), name
    assert errors >= 15  # the bad files really were rejected


@pytest.mark.parametrize("dims", [("f8", 5), ("f4", 5), ("f8", 2, 3), ("f4", 3, 1, 4), ("f8", 0, 3)])
def test_write_npy_bytes_match_reference_and_numpy_reads_them(tmp_path, dims):
    r, o = tmp_path / "r.npy", tmp_path / "o.npy"
    subprocess.run([REF, "writenpy", r, *map(str, dims)], check=True)
    subprocess.run([OURS, "writenpy", o, *map(str, dims)], check=True)
    assert r.read_bytes() == o.read_bytes()
    a = np.load(o)
    assert a.shape == tuple(dims[1:]) and a.dtype == np.dtype("<" + dims[0])
    assert (len(o.read_bytes()) - a.nbytes) % 64 == 0  # payload 64-byte aligned


def _envi(d, name, header, payload=None, data_name=None):
    with open(os.path.join(d, name + ".hdr"), "w") as f:
        f.write(header)
    if payload is not None:
        with open(os.path.join(d, data_name or name + ".img"), "wb") as f:
            f.write(payload)
    return os.path.join(d, name + ".hdr")


def test_read_envi_matches_reference(tmp_path):
    d = str(tmp_path)
    rng = np.random.default_rng(1)
    cube8 = rng.random((3, 4, 5)).tobytes()   # bands, lines, samples (BSQ)
    cube4 = rng.random((2, 3, 2)).astype("<f4").tobytes()
    base = "ENVI\nsamples = 5\nlines = 4\nbands = 3\ndata type = 5\ninterleave = bsq\nbyte order = 0\n"
    cases = [
        _envi(d, "f8", base + "wavelength = {400.5, 500,\n  600.25}\n", cube8),
        _envi(d, "f4", "ENVI\nsamples = 2\nlines = 3\nbands = 2\ndata type = 4\ninterleave = BSQ\n", cube4,
              "f4.dat"),
        _envi(d, "offset", base + "header offset = 16\n", bytes(16) + cube8, "offset.raw"),
        _envi(d, "noext", base, cube8, "noext"),
        _envi(d, "upper", "  envi \nSAMPLES = 5\nLines = 4\nbands=3\ndata type = 5\ninterleave = bsq\n", cube8),
        _envi(d, "nosentinel", "samples = 5\n", cube8),
        _envi(d, "empty", "", cube8),
        _envi(d, "bil", base.replace("bsq", "bil"), cube8),
        _envi(d, "dtype2", base.replace("data type = 5", "data type = 2"), cube8),
        _envi(d, "byteorder", base.replace("byte order = 0", "byte order = 1"), cube8),
        _envi(d, "nosamples", base.replace("samples = 5\n", ""), cube8),
        _envi(d, "nointerleave", base.replace("interleave = bsq\n", ""), cube8),
        _envi(d, "badint", base.replace("lines = 4", "lines = 4.0"), cube8),
        _envi(d, "zero", base.replace("lines = 4", "lines = 0"), cube8),
        _envi(d, "truncated", base, cube8[:-8]),
        _envi(d, "unterminated", base + "wavelength = {400, 500\n", cube8),
        _envi(d, "badwl", base + "wavelength = {400, abc, 600}\n", cube8),
        _envi(d, "partialwl", base + "wavelength = {400, 5e, 600}\n", cube8),
        _envi(d, "nodata", base),
    ]
    for hdr in cases:
        r, o = both("image", hdr)
        assert (o.returncode, o.stdout) == (r.returncode, r.stdout), (hdr, r.stdout[-400:], o.stdout[-400:])
    assert "spatial 4 5" in both("image", cases[0])[1].stdout


def test_read_csv_matches_reference(tmp_path):
    files = {"good": "1,2,3\n0.5,1e-3,2\n-1,0x1p-3,7\n", "crlf": "1,2\r\n1.5,2.5\r\n", "trailing": "1,2\n3,4,\n",
             "ragged": "1,2,3\n1,2\n", "malformed": "1,2\n3,abc\n", "empty_cell": "1,2\n3,,\n",
             "empty": "", "header_only": "1,2,3\n", "blank_mid": "1,2\n3,4\n\n5,6\n", "noeol": "1,2\n3,4"}
    for name, text in files.items():
        p = tmp_path / (name + ".csv")
        p.write_text(text)
        r, o = both("csv", p)
        assert (o.returncode, o.stdout) == (r.returncode, r.stdout), (name, r.stdout, o.stdout)
    r, o = both("csv", tmp_path / "absent.csv")
    assert o.stdout == r.stdout and "cannot open" in r.stdout


def _write_est(d, e, a):
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "endmembers.csv"), "w") as f:
        f.write(",".join(str(k + 1) for k in range(e.shape[1])) + "\n")
        for row in e:
            f.write(",".join(repr(float(v)) for v in row) + "\n")
    save(os.path.join(d, "abundances.npy"), a)


@pytest.mark.parametrize("p,renorm", [(3, False), (4, True), (8, False), (9, False), (12, True)])
def test_evaluate_matches_reference(tmp_path, p, renorm):
    rng = np.random.default_rng(p)
    L, N = 25, 300
    gt_e = rng.random((L, p)) + 0.05
    gt_a = rng.dirichlet(np.ones(p), size=N).T
    if renorm:
        gt_a[:, ::7] *= 1.01
    perm = rng.permutation(p)
    est_e = gt_e[:, perm] + 0.02 * rng.standard_normal((L, p))
    est_a = gt_a[perm] + 0.01 * rng.random((p, N))
    _write_est(str(tmp_path / "est"), est_e, est_a)
    save(tmp_path / "gt_a.npy", gt_a)
    save(tmp_path / "gt_e.npy", gt_e)
    out = same("evaluate", tmp_path / "est", tmp_path / "gt_e.npy", tmp_path / "gt_a.npy")
    assert ('"ground_truth_renormalized": true' in out) == renorm
    # the matching undoes the planted permutation
    res, _ = json.JSONDecoder().raw_decode(out)
    assert res["permutation"] == [int(v) for v in perm]


def test_evaluate_errors_match_reference(tmp_path):
    rng = np.random.default_rng(5)
    gt_e, gt_a = rng.random((10, 3)), rng.dirichlet(np.ones(3), size=20).T
    save(tmp_path / "gt_e.npy", gt_e)
    save(tmp_path / "gt_a.npy", gt_a)
    _write_est(str(tmp_path / "p4"), rng.random((10, 4)), rng.dirichlet(np.ones(4), size=20).T)
    same("evaluate", tmp_path / "p4", tmp_path / "gt_e.npy", tmp_path / "gt_a.npy", expect_error="count mismatch")
    _write_est(str(tmp_path / "n"), rng.random((10, 3)), rng.dirichlet(np.ones(3), size=21).T)
    same("evaluate", tmp_path / "n", tmp_path / "gt_e.npy", tmp_path / "gt_a.npy", expect_error="pixel count")
    z = gt_a.copy()
    z[:, 3] = 0
    save(tmp_path / "gt_z.npy", z)
    _write_est(str(tmp_path / "ok"), rng.random((10, 3)), gt_a)
    same("evaluate", tmp_path / "ok", tmp_path / "gt_e.npy", tmp_path / "gt_z.npy", expect_error="sums to zero")
    e0 = rng.random((10, 3))
    e0[:, 1] = 0
    _write_est(str(tmp_path / "zero_e"), e0, gt_a)
    same("evaluate", tmp_path / "zero_e", tmp_path / "gt_e.npy", tmp_path / "gt_a.npy", expect_error="zero spectrum")


REPORT = """{
  "version": "0.1.0",
  "input": {"path": "scene \\u00e9/cube.npy", "bands": 6, "pixels": 12, "height": 3, "width": 4},
  "zero_pixels": 1,
  "config": {"endmembers": 2, "outer_iters": 7, "inner_iters_a": 5, "inner_iters_b": 4, "runs": 3,
             "base_seed": 18446744073709551615, "gamma_set": [0.125, 1.0, 8.0, 0.1, 1e-300, 3.0e+20],
             "fit_slack": 1.05},
  "runs": [
    {"index": 0, "seed": 18446744073709551615, "gamma": 8.0, "fit_l1": 1.2345678901234567, "coherence": 0.5,
     "wall_ms": 12.25, "ok": true},
    {"index": 1, "seed": 0, "gamma": 0.125, "fit_l1": 0.0, "coherence": 0.0, "wall_ms": 0.0, "ok": false,
     "error": "non-finite abundance iterate at outer iteration 3 \\"q\\""},
    {"index": 2, "seed": 1, "gamma": 1.0, "fit_l1": 1.1e-7, "coherence": 0.9999999999999999, "wall_ms": 1e3,
     "ok": true}
  ],
  "selection": {"candidates": [0, 2], "selected": 2, "fit_min": 1.1e-7, "seed": 1, "gamma": 1.0}
}
"""


def test_bundle_and_report_round_trip_match_reference(tmp_path):
    rng = np.random.default_rng(9)
    (tmp_path / "report.json").write_text(REPORT)
    e = rng.random((6, 2))
    a = rng.dirichlet(np.ones(2), size=12).T
    a[0, 0], a[1, 0] = 1.0, 0.0   # exact corners, and an out-of-range value for the map clamp
    a[0, 5], a[1, 5] = 1.5, -0.5
    a[0, 6] = 0.5 / 255.0         # lround of an exact half
    save(tmp_path / "e.npy", e)
    save(tmp_path / "a.npy", a)
    r = subprocess.run([REF, "bundle", tmp_path / "report.json", tmp_path / "e.npy", tmp_path / "a.npy",
                        tmp_path / "r"], capture_output=True, text=True)
    o = subprocess.run([OURS, "bundle", tmp_path / "report.json", tmp_path / "e.npy", tmp_path / "a.npy",
                        tmp_path / "o"], capture_output=True, text=True)
    assert r.returncode == o.returncode == 0 and r.stdout == o.stdout, (r.stdout, o.stdout)
    files = same_tree(tmp_path / "r", tmp_path / "o")
    assert files == ["abundances.npy", "endmembers.csv", "maps/endmember_1.pgm", "maps/endmember_2.pgm",
                     "report.json"]
    assert np.array_equal(np.load(tmp_path / "o" / "abundances.npy"), a)


def test_report_parse_errors_match_reference(tmp_path):
    bad = {"malformed": "{\"version\": ", "not_json": "hello",
           "missing": REPORT.replace('"zero_pixels": 1,', ""),
           "wrong_type": REPORT.replace('"bands": 6', '"bands": "six"'),
           "spatial_half": REPORT.replace(', "width": 4', "")}
    save(tmp_path / "e.npy", np.ones((6, 2)))
    save(tmp_path / "a.npy", np.full((2, 12), 0.5))
    for name, text in bad.items():
        (tmp_path / (name + ".json")).write_text(text)
        out = same("bundle", tmp_path / (name + ".json"), tmp_path / "e.npy", tmp_path / "a.npy",
                   tmp_path / ("out_" + name), expect_error="")
        assert "report JSON" in out, out


def test_cli_host_cases_pass():
    """tests/cpp/test_cli.cpp host cases: usage / data-error exit codes, synth
    determinism, info over npy and ENVI (the GPU cases run in -m gpu)."""
    assert os.path.exists(CLI_TEST), "tests/cpp/build/test_cli missing"
    r = subprocess.run([CLI_TEST, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.parametrize("p", [3, 10])
def test_evaluate_tie_breaking_matches_reference(tmp_path, p):
    """Duplicate spectra make several matchings optimal: the exhaustive search
    (p ≤ 8, first strict minimum in lexicographic order) and the Hungarian
    method (p > 8, column scan order) must pick the reference's."""
    rng = np.random.default_rng(40 + p)
    gt_e = rng.random((12, p)) + 0.1
    gt_e[:, 1] = gt_e[:, 0]
    gt_e[:, p - 1] = gt_e[:, 0]
    gt_a = rng.dirichlet(np.ones(p), size=50).T
    est_e = np.repeat(gt_e[:, :1], p, axis=1)        # every pairing of the copies costs the same
    est_e[:, 2:p - 1] = gt_e[:, 2:p - 1][:, ::-1]
    _write_est(str(tmp_path / "est"), est_e, gt_a[::-1])
    save(tmp_path / "gt_a.npy", gt_a)
    save(tmp_path / "gt_e.npy", gt_e)
    same("evaluate", tmp_path / "est", tmp_path / "gt_e.npy", tmp_path / "gt_a.npy")
