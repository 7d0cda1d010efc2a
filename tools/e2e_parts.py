"""Where the end-to-end run_ensemble time goes (dev): python tools/e2e_parts.py [cfg1]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2209_11002_b200 import edaa, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
spec = synth.CONFIGS[cfg]
x = synth.generate(spec)[0]
x = torch.from_numpy(x).pin_memory().numpy()
ecfg = edaa.EnsembleConfig(runs=spec.runs, solver=edaa.SolverConfig(endmembers=spec.endmembers))
edaa.run_ensemble(x, ecfg)
dev = edaa.Device.get(0)
for rep in range(3):
    t = {}
    t0 = time.perf_counter()
    xf = edaa.validate_image(x)
    t["validate"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev.set_image(xf)
    torch.cuda.synchronize()
    t["set_image"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    seeds, gammas = edaa.ensemble_plan(ecfg)
    t["plan"] = time.perf_counter() - t0
    s = ecfg.solver
    t0 = time.perf_counter()
    dev.solve(s.endmembers, s.outer_iters, s.inner_iters_a, s.inner_iters_b, seeds, gammas)
    t["solve"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    recs = [dev.record(m) for m in range(ecfg.runs)]
    t["records"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    cand, sel, fmin = dev.select(ecfg.fit_slack)
    t["select"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    tr = dev.traces()
    A, B, E = dev.factors(sel)
    t["results"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    edaa.run_ensemble(x, ecfg)
    t["run_ensemble total"] = time.perf_counter() - t0
    print(" ".join("%s %.2f ms" % (k, v * 1e3) for k, v in t.items()), flush=True)
