"""Observed deviations of the GPU path from every reference fixture in tests/golden (the numbers
behind the pass/fail bars of tests/test_gpu_parity.py): python tools/parity_report.py > profiles/roundN/parity_report.txt"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import golden_files, golden_scene, load_golden  # noqa: E402
from paper_2209_11002_b200 import edaa, synth  # noqa: E402


def relmax(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


print("%-28s %-26s %10s %10s %10s %10s  %s" % ("fixture", "shape", "obj rel", "|A-ref|", "|B-ref|", "fit rel", "selection"))
for name in golden_files("run_"):
    g = load_golden(name)
    x = golden_scene(g)
    r = edaa.run(x, edaa.SolverConfig(endmembers=int(g["p"]), outer_iters=int(g["T"]), gamma=float(g["gamma"]),
                                      seed=int(g["seed"])))
    n = min(len(g["trace"]), 51)
    floor = 1e-12 * 0.5 * float(np.sum(x.astype(np.float64) ** 2))
    rel = float(np.max(np.abs(r.objective_trace[:n] - g["trace"][:n]) / np.maximum(np.abs(g["trace"][:n]), floor)))
    print("%-28s L=%-3d N=%-6d p=%-2d g=%-5g %10.1e %10.1e %10.1e %10.1e" %
          (name[:-4], x.shape[0], x.shape[1], int(g["p"]), float(g["gamma"]), rel,
           np.abs(r.abundances - g["A"]).max(), np.abs(r.contributions - g["B"]).max(),
           abs(r.fit_l1 - float(g["fit"])) / max(float(g["fit"]), 1e-300)))
for name in golden_files("ens_") + golden_files("cfg"):
    g = load_golden(name)
    x = golden_scene(g)
    p = int(g["p"]) if "p" in g else int(g["A"].shape[0])
    res, rep = edaa.run_ensemble(x, edaa.EnsembleConfig(runs=int(g["M"]), solver=edaa.SolverConfig(
        endmembers=p, outer_iters=int(g["T"]))))
    n = min(len(g["trace"]), 51)
    fits = np.array([r.fit_l1 for r in rep.per_run])
    mus = np.array([r.coherence for r in rep.per_run])
    cand = [int(c) for c in g["candidates"]]
    # selection margins of the reference ensemble: μ gap to the runner-up, nearest fit to the cutoff
    cm = sorted(float(g["mus"][c]) for c in cand)
    gap = (cm[1] - cm[0]) / cm[0] if len(cm) > 1 else float("inf")
    cut = 1.05 * float(g["fit_min"])
    near = float(np.min(np.abs(g["fits"] - cut) / cut))
    print("%-28s L=%-3d N=%-6d p=%-2d M=%-5d %10.1e %10.1e %10.1e %10.1e  selected %d == %d, %d candidates %s; "
          "reference margins: mu gap %.1e, fit-to-cutoff %.1e; max |mu-ref| %.1e" %
          (name[:-4], x.shape[0], x.shape[1], p, int(g["M"]), relmax(res.objective_trace[:n], g["trace"][:n]),
           np.abs(res.abundances - g["A"]).max(), np.abs(res.contributions - g["B"]).max(), relmax(fits, g["fits"]),
           rep.selected, int(g["selected"]), len(cand), "identical" if rep.candidate_set == cand else "DIFFER", gap, near,
           float(np.max(np.abs(mus - g["mus"])))))
