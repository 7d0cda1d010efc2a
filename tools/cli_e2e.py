"""End-to-end `archetype unmix` timing on a BASELINE config-shaped cube (the
CLI a user of the reference runs: load .npy → validate → ℓ2-normalise →
50-run ensemble on the GPU → selection → output bundle), with the
normalisation on the device (default) and on the host
(ARCHETYPE_HOST_NORMALIZE=1, the reference's order of host passes). Both
bundles must be identical apart from the per-run wall_ms.

    python tools/cli_e2e.py [cfg1|cfg2|cfg3|cfg4] [--reps R]
"""
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_11002_b200 import synth  # noqa: E402

CLI = os.path.join(ROOT, "paper_2209_11002_b200", "archetype")


def strip_wall(text):
    rep = json.loads(text)
    for r in rep["runs"]:
        r.pop("wall_ms")
    return rep


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "cfg1"
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
    spec = synth.CONFIGS[cfg]
    x = synth.generate(spec)[0]
    d = tempfile.mkdtemp()
    # (H, W, L) cube as the reference's tools take it: spatial maps are written too
    cube = os.path.join(d, "cube.npy")
    np.save(cube, np.ascontiguousarray(x.T.reshape(spec.height, spec.width, spec.bands)).astype("<f4"))
    args = [CLI, "unmix", "--input", cube, "--endmembers", str(spec.endmembers), "--runs", str(spec.runs)]
    out = {}
    for mode, env in (("device_ingest", {}), ("host_normalize", {"ARCHETYPE_HOST_NORMALIZE": "1"})):
        times = []
        for r in range(reps + 1):  # first call: context + graph capture, reported apart
            est = os.path.join(d, "%s_%d" % (mode, r))
            t0 = time.perf_counter()
            p = subprocess.run(args + ["--output", est], capture_output=True, text=True,
                               env=dict(os.environ, **env))
            times.append(time.perf_counter() - t0)
            assert p.returncode == 0, p.stderr
        out[mode] = {"first_s": times[0], "median_s": float(np.median(times[1:])), "dir": est}
    a, b = out["device_ingest"]["dir"], out["host_normalize"]["dir"]
    same = all(open(os.path.join(a, f), "rb").read() == open(os.path.join(b, f), "rb").read()
               for f in ("abundances.npy", "endmembers.csv"))
    same &= strip_wall(open(os.path.join(a, "report.json")).read()) == \
        strip_wall(open(os.path.join(b, "report.json")).read())
    T = 100
    res = {"workload": cfg, "bands": spec.bands, "pixels": spec.pixels, "endmembers": spec.endmembers,
           "runs": spec.runs, "outer_iters": T, "bundles_identical": bool(same)}
    for mode in ("device_ingest", "host_normalize"):
        res[mode] = {"process_wall_s": out[mode]["median_s"], "first_call_s": out[mode]["first_s"],
                     "run_iterations_per_s": spec.runs * T / out[mode]["median_s"]}
    # in-process timing (context and graph warm): tools/cli_bench.cpp
    exe = os.path.join(d, "cli_bench")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "cli_bench.cpp"), "-L" + os.path.dirname(CLI),
                    "-larchetype_b200", "-ledaa_cuda", "-Wl,-rpath," + os.path.dirname(CLI), "-o", exe],
                   check=True)
    p = subprocess.run([exe, cube, str(spec.endmembers), str(spec.runs), d, str(max(reps, 3))],
                       capture_output=True, text=True, check=True)
    lines = [json.loads(l) for l in p.stdout.splitlines()]
    for mode, key in ((0, "device_ingest"), (1, "host_normalize")):
        best = min((l for l in lines if l["host_normalize"] == mode), key=lambda l: l["median_ms"])
        res[key]["in_process_median_ms"] = best["median_ms"]
        res[key]["in_process_run_iterations_per_s"] = spec.runs * T / (best["median_ms"] / 1e3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
