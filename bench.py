#!/usr/bin/env python
"""Benchmark: EDAA run-iterations/s (BASELINE.json "metric") on B200.

A step is ONE full EDAA ensemble of the chosen BASELINE config — M runs × T=100
outer iterations (K1 = K2 = 5) with model selection — batched in one device
solve.  The default workload is cfg1 (Jasper-Ridge shape: L=198, N=100×100,
p=4, M=50), the config the metric is quoted on; synthetic seeded data of that
shape (paper_2209_11002_b200/synth.py).

    python bench.py [--gpus N --steps K --warmup W] [--config cfg1] [--impl ours|reference]
    python bench.py --config cfg4 --strong --gpus N   # north_star sweep: 64 runs split over N GPUs

* ``--gpus N`` outside torchrun (no WORLD_SIZE) re-launches this script under
  ``torch.distributed.run`` with N processes (one per GPU) and fails loudly
  when fewer than N CUDA devices are visible; ``n_gpus`` is the number of
  ranks that actually ran.

* ``value``: run-iterations/s with X resident in HBM, device time (CUDA events
  on the solver stream, L2 flushed with a 256 MB write before every timed
  step), max over ranks; N>1 = weak scaling (each rank its own M runs, the
  records gathered for one selection over all M·N runs).
* ``e2e``: the same metric through the public API ``run_ensemble`` with the
  image in pinned host memory: H2D of X, solve, selection and D2H of the
  selected run's A/B/E inside the timed region.
* ``roofline``: the dominant kernel (the B-step pass) against the fp64
  tensor-pipe (DMMA) peak measured live on this GPU; its HBM side vs
  MEASURED_PEAKS.json is reported alongside.
* ``cpu_baseline``: the reference CPU solver (oracle/_ref, built from
  /root/reference) on this host's cores, bounded sample (rank 0, N=1).
* ``--impl reference``: the reference CPU implementation alone, timed per step
  on a bounded sample of the same workload (all host threads).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EDAA run-iterations/sec (M runs x T outer iterations) at N,L,p"
UNIT = "run-iterations/s"
# Paper (PyTorch, RTX 2080 Ti) end-to-end ensemble times, BASELINE.md §1.
PUBLISHED = {"cfg1": 50 * 100 / 9.6, "cfg2": 50 * 100 / 75.2}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--outer", type=int, default=100, help="T (default: the reference's 100)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: the config's M runs in total, split over the GPUs "
                         "(the north_star cfg4 sweep); default: M runs per GPU (weak)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pass-order", type=int, default=0,
                    help="dev: pass item order (0 auto, 1 chunk-major, 2 slice-major, 3 interleaved)")
    ap.add_argument("--x64", action="store_true",
                    help="re-normalise the cube in fp64 (as l2_normalize does for a real cube, not "
                         "fp32-exact): the fp64-X pass kernels, the `unmix` CLI path; not the headline")
    return ap.parse_args()


def launch_ranks(args, argv):
    """--gpus N > 1 outside torchrun: one process per GPU under torch.distributed.run.
    Returns the exit code of the launcher (None when no re-launch is needed)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if have < args.gpus:
            sys.stderr.write("bench.py: --gpus %d needs %d visible CUDA devices, found %d\n"
                             % (args.gpus, args.gpus, have))
            return 2
    cmd = launcher_cmd(args.gpus, argv)
    return subprocess.call(cmd, env=dict(os.environ, MASTER_ADDR="127.0.0.1"))


def launcher_cmd(n, argv):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
            "--master-addr", "127.0.0.1", "--master-port", str(port),
            os.path.join(ROOT, "bench.py")] + list(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def scene(cfg_name):
    from paper_2209_11002_b200 import synth
    spec = synth.CONFIGS[cfg_name]
    x, _, _ = synth.generate(spec)
    return spec, x


# ----------------------------------------------------------------------------- reference arm
# The reference's cost is ~62·L·N·p flops per run-iteration, linear in N
# (SURVEY §3.2); above this L·N·p the CPU sample runs on the first
# CPU_SAMPLE_LNP/(L·p) pixels and its time is scaled by N/N' (cfg2-cfg4: a
# full cfg4 run-iteration is ~2 min per core, and 16 concurrent runs need
# ~100 GB of host temporaries).
CPU_SAMPLE_LNP = 2.0e7


def cpu_sample_pixels(spec):
    n = int(CPU_SAMPLE_LNP // (spec.bands * spec.endmembers))
    return spec.pixels if spec.bands * spec.pixels * spec.endmembers <= CPU_SAMPLE_LNP else max(n, 64)


def cpu_reference_sample(x, spec, T, runs=None, workers=None):
    """Reference run_ensemble on the host cores: returns (seconds scaled to the
    full N, run-iters done, kind, cores)."""
    from oracle import Oracle, available_kinds
    kind = "reference" if "reference" in available_kinds() else "port"
    orc = Oracle(kind)
    cores = workers or os.cpu_count() or 1
    runs = runs or cores
    n = cpu_sample_pixels(spec)
    xd = np.ascontiguousarray(x[:, :n], dtype=np.float64)
    t0 = time.perf_counter()
    orc.run_ensemble(xd, spec.endmembers, M=runs, T=T, workers=cores)
    return (time.perf_counter() - t0) * (spec.pixels / n), runs * T, kind, cores


def cpu_baseline(x, spec):
    """Bounded sample: M = cores concurrent runs at T=1 and T=4; the difference
    removes the per-run setup, giving steady-state run-iterations/s."""
    t1, _, kind, cores = cpu_reference_sample(x, spec, 1)
    t4, _, _, _ = cpu_reference_sample(x, spec, 4)
    value = cores * 3 / max(t4 - t1, 1e-9)
    return {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": "%s shape, M=%d concurrent runs (one per core), T=4 minus T=1 "
                      "(%.1f s + %.1f s wall)%s" % (spec.name, cores, t4, t1, sample_note(spec))}


def sample_note(spec):
    n = cpu_sample_pixels(spec)
    return "" if n == spec.pixels else (", on the first %d of %d pixels, time scaled by N/N' "
                                        "(reference cost is linear in N)" % (n, spec.pixels))


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    spec, x = scene(args.config)
    cores = os.cpu_count() or 1
    # Bounded sample per step: M = cores concurrent runs at T=4 and at T=1; the
    # difference is 3 steady-state outer iterations per run (the per-run setup —
    # B⁰, step sizes, trace[0], fit, μ — cancels), as in cpu_baseline.
    for _ in range(args.warmup):
        cpu_reference_sample(x, spec, 1)
    times = []
    kind = None
    for _ in range(args.steps):
        t4, _, kind, cores = cpu_reference_sample(x, spec, 4)
        t1, _, _, _ = cpu_reference_sample(x, spec, 1)
        times.append(max(t4 - t1, 1e-9))
    total = sum(times)
    T = 3
    value = cores * T * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(spec, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": "%s shape, M=%d runs (one per core) per step, run_ensemble "
                                   "with %d workers at T=4 minus T=1 (3 steady-state outer "
                                   "iterations per run)%s" % (spec.name, cores, cores,
                                                              sample_note(spec))},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(spec, args, runs=None, T=None, world=1):
    strong = getattr(args, "strong", False)
    total = spec.runs if strong else (runs or spec.runs) * world
    return {"workload": "%s: EDAA ensemble L=%d N=%d p=%d M=%d T=%d K1=K2=5 + model selection"
                        % (spec.name, spec.bands, spec.pixels, spec.endmembers,
                           total, T or args.outer),
            "bands": spec.bands, "pixels": spec.pixels, "endmembers": spec.endmembers,
            "runs_total": total, "runs_per_gpu": (runs or spec.runs) if not strong else
            "%d split over %d GPU(s)" % (spec.runs, world), "outer_iters": T or args.outer,
            "inner_iters": [5, 5], "l2_flush": "256 MB write before every timed step",
            "parallelism": ("ensemble runs split over GPUs (strong scaling: fixed total)" if strong
                            else "ensemble runs sharded over GPUs (weak scaling: M per GPU)"),
            "x_storage": "fp64 (cube re-normalised in fp64: not fp32-exact)" if getattr(args, "x64", False)
                         else "fp32 (fp32-exact normalised cube)"}


# ----------------------------------------------------------------------------- our arm
def selection_margins(fits, mus, oks, slack):
    """How close the selection was: μ gap of the winner to the runner-up candidate
    and the nearest fit to the 1.05·fit_min cutoff (relative), ensemble.cpp:71-94."""
    fits, mus, oks = np.asarray(fits), np.asarray(mus), np.asarray(oks, dtype=bool)
    if not oks.any():
        return None
    fmin = fits[oks].min()
    cut = slack * fmin
    cand = np.flatnonzero(oks & (fits <= cut))
    order = cand[np.argsort(mus[cand], kind="stable")]
    gap = float((mus[order[1]] - mus[order[0]]) / abs(mus[order[0]])) if len(order) > 1 else None
    near = float(np.min(np.abs(fits[oks] - cut)) / cut)
    return {"selected": int(order[0]), "candidates": int(len(cand)),
            "mu_gap_to_runner_up_rel": gap, "nearest_fit_to_cutoff_rel": near}


def main():
    args = parse()
    rc = launch_ranks(args, sys.argv[1:])
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference_arm(args)
    import torch
    from paper_2209_11002_b200 import edaa
    rank, world, local = dist_env()
    if torch.cuda.device_count() < world or (args.gpus > 1 and world != args.gpus):
        raise SystemExit("bench.py: %d ranks for --gpus %d with %d visible CUDA devices"
                         % (world, args.gpus, torch.cuda.device_count()))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    spec, x = scene(args.config)
    L, N, p, T = spec.bands, spec.pixels, spec.endmembers, args.outer
    from paper_2209_11002_b200.distributed import shard_bounds
    if args.strong:   # the config's runs in total, contiguous blocks per rank
        first, M = shard_bounds(spec.runs, world, rank)
        M_total = spec.runs
    else:             # M runs per rank
        M = spec.runs
        first, M_total = rank * M, M * world
    dev = edaa.Device.get(local)
    if args.pass_order:
        dev.set_pass_order(args.pass_order)
    stream = torch.cuda.ExternalStream(dev.stream, device=torch.device("cuda", local))
    if args.x64:
        x = x.astype(np.float64)
        x = x / np.sqrt((x * x).sum(axis=0))[None, :]
    x_dev = torch.from_numpy(x).to(f"cuda:{local}")
    x_img = x if args.x64 else x_dev  # host fp64 upload keeps X in fp64 on the device
    torch.cuda.synchronize()
    dev.set_image(x_img)
    cfg = edaa.EnsembleConfig(runs=M_total, solver=edaa.SolverConfig(endmembers=p, outer_iters=T))
    seeds, gammas = edaa.ensemble_plan(cfg, first=first, count=M)
    if M == 0:
        raise SystemExit("bench.py: rank %d has no runs (%d runs over %d GPUs)" % (rank, M_total, world))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    Mmax = max(shard_bounds(M_total, world, r)[1] for r in range(world))

    def gather_records():
        """(fits, mus, oks) of all M_total runs in global order (all_gather over ranks)."""
        recs = [dev.record(m) for m in range(M)]
        loc = torch.zeros(3, Mmax, dtype=torch.float64, device=x_dev.device)
        loc[0, :M] = torch.tensor([r.fit_l1 for r in recs], dtype=torch.float64)
        loc[1, :M] = torch.tensor([r.coherence for r in recs], dtype=torch.float64)
        loc[2, :M] = torch.tensor([float(r.ok) for r in recs], dtype=torch.float64)
        if world > 1:
            import torch.distributed as dist
            allv = [torch.empty_like(loc) for _ in range(world)]
            dist.all_gather(allv, loc)
        else:
            allv = [loc]
        parts = [allv[r][:, :shard_bounds(M_total, world, r)[1]] for r in range(world)]
        return torch.cat(parts, dim=1).cpu().numpy()

    def gather_select():
        cat = gather_records()
        records = [edaa.RunRecord(i, 0, 0.0, cat[0, i], cat[1, i], 0.0, bool(cat[2, i]), "")
                   for i in range(cat.shape[1])]
        return edaa.select_runs(records, cfg.fit_slack).selected

    def one_step(timed):
        with torch.cuda.stream(stream):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        dev.solve_async(p, T, 5, 5, seeds, gammas)
        dev.finish()
        if world == 1:
            dev.select(cfg.fit_slack)
        else:
            gather_select()
        with torch.cuda.stream(stream):
            e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(max(args.warmup, 3)):
        one_step(False)
    dev.profile_enable(True)
    one_step(False)
    prof = dev.profile()
    dev.profile_enable(False)
    sampler = ClockSampler(local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    n0 = dev.launch_count()
    times = [one_step(True) for _ in range(args.steps)]
    launches = dev.launch_count() - n0
    torch.cuda.synchronize()
    clocks = sampler.stop()
    t_dev = sum(times)  # ms on this rank
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t_dev], dtype=torch.float64, device=x_dev.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev = float(tt.item())
    run_iters = M_total * T * args.steps
    value = run_iters / (t_dev * 1e-3)
    recs_all = gather_records()
    margins = selection_margins(recs_all[0], recs_all[1], recs_all[2], cfg.fit_slack)

    # ---- e2e through the public API (pinned host X; H2D + solve + select + D2H) ----
    e2e = None
    if not args.no_e2e and world > 1:
        # public multi-GPU API: pinned host X per rank, sharded solve, record
        # all-gather, selection, broadcast of the selected run's factors
        import torch.distributed as dist
        from paper_2209_11002_b200 import distributed
        x_pin = torch.from_numpy(x).pin_memory().numpy()
        ecfg = edaa.EnsembleConfig(runs=M_total, solver=edaa.SolverConfig(endmembers=p, outer_iters=T))
        distributed.run_ensemble_sharded(x_pin, ecfg, device=local)  # warm
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            distributed.run_ensemble_sharded(x_pin, ecfg, device=local)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=x_dev.device)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": M_total * T * args.steps / float(dt.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(x.nbytes + 16 * M),
               "d2h_bytes_per_step": int(8 * (2 * p * N + L * p + (T + 1)) + 32 * M)}
        dev.set_image(x_img)
    if not args.no_e2e and world == 1:
        x_pin = torch.from_numpy(x).pin_memory().numpy()
        ecfg = edaa.EnsembleConfig(runs=M, solver=edaa.SolverConfig(endmembers=p, outer_iters=T))
        edaa.run_ensemble(x_pin, ecfg, device=local)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            edaa.run_ensemble(x_pin, ecfg, device=local)
        dt = time.perf_counter() - t0
        e2e = {"value": M * T * args.steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(x.nbytes + 16 * M),
               "d2h_bytes_per_step": int(8 * (2 * p * N + L * p + (T + 1) * M + 4 * M) + M)}
        dev.set_image(x_img)

    # ---- roofline of the dominant kernel (B-step pass) ----
    peak64 = dev.fp64_peak_tflops()
    ms_b, n_b = prof["B"]
    ms_a, n_a = prof["A"]
    launch_ms = ms_b / max(n_b, 1)
    flops_b = 4.0 * L * N * p * M  # g = XᵀZ and Y = X·B, M runs per launch
    bytes_b = (8.0 if args.x64 else 4.0) * L * N + 16.0 * p * N * M  # X once + logits read+write (fp64)
    achieved = flops_b / (launch_ms * 1e-3) / 1e12
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6550.4)
    traffic = None
    try:
        summ = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = summ.get(spec.name, {}).get("pass_b_dram_bytes")
    except Exception:
        pass
    total_ms = sum(v[0] for v in prof.values())
    roofline = {
        "bound": "tensor", "achieved": achieved, "peak": peak64, "unit": "TFLOP/s",
        "frac": achieved / peak64 if peak64 else None, "traffic": traffic,
        "kernel": "B pass: k_pass_b64 (64-pixel logical tiles; fp32 images with L <= 200) or k_pass<B> "
                  "(g = XᵀZ, logits, online max, Y = X·B; fp64 DMMA)",
        "peak_source": "fp64 DMMA microkernel measured live (edaa_probe_fp64_peak); "
                       "MEASURED_PEAKS.json has no fp64 entry",
        "flops_per_launch": flops_b, "launch_ms": launch_ms,
        "share_of_step": ms_b / total_ms if total_ms else None,
        "hbm": {"algorithmic_bytes_per_launch": bytes_b,
                "achieved_gbs": bytes_b / (launch_ms * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                "frac": bytes_b / (launch_ms * 1e-3) / 1e9 / hbm_peak},
        "pass_ms": {k: v[0] for k, v in prof.items()},
    }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": t_dev / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": (value / PUBLISHED[spec.name]) if spec.name in PUBLISHED and T == 100 else None,
        "dtype": "f64", "data": "synthetic", "config": workload_config(spec, args, runs=M, world=world),
        "selection": margins, "roofline": roofline, "gpu_launches": int(launches), "clocks": clocks, "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(x, spec)
        except Exception as exc:  # the oracle is absent on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                    "kind": None, "sample": "unavailable: %s" % exc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
