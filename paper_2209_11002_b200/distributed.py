"""Ensemble sharding over the GPUs of one node (one process per GPU).

Algorithm 2's M runs are independent, so rank r of a ``torch.distributed``
group solves the contiguous block of runs [r·M/W, (r+1)·M/W) on its own GPU
with the batched device solver — no data-path collective.  The only exchange
is the per-run record table (fit, coherence, ok: 3·M doubles, one
``all_gather``) so every rank applies the selection rule
(ensemble.cpp:71-94) to the same table, and one ``broadcast`` of the selected
run's factors from the rank that owns it.

A run's arithmetic does not depend on which batch or GPU it ran in (fixed
pixel slicing, per-column reductions), so the sharded result is bitwise the
single-GPU result — the multi-GPU analogue of the reference's worker-count
independence (ensemble.hpp:23-26, test_ensemble.cpp:118-148).

The per-rank solve is pluggable (``local_solver``) so the sharding, gather and
selection logic can be exercised on CPU ranks with ``gloo`` in the tests.
"""
from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np

from . import edaa


@dataclass
class LocalBatch:
    """What one rank produced for its block of runs [first, first+count)."""
    first: int
    records: List[edaa.RunRecord]              # global indices
    factors: Callable[[int], edaa.RunResult]   # global index → RunResult (owner only)


def shard_bounds(runs: int, world: int, rank: int):
    """Contiguous, balanced block of run indices for `rank` (may be empty)."""
    first = rank * runs // world
    return first, (rank + 1) * runs // world - first


def gpu_local_solver(device: int = 0):
    """The production per-rank solver: one batched solve on this rank's GPU."""

    def solve(x, config: edaa.EnsembleConfig, first: int, count: int) -> LocalBatch:
        seeds, gammas = edaa.ensemble_plan(config, first=first, count=count)
        if count == 0:
            return LocalBatch(first, [], lambda m: None)
        dev = edaa.Device.get(device)
        dev.set_image(edaa.validate_image(x))
        s = config.solver
        t0 = time.perf_counter()
        dev.solve(s.endmembers, s.outer_iters, s.inner_iters_a, s.inner_iters_b, seeds, gammas)
        wall = (time.perf_counter() - t0) * 1e3
        recs = []
        for k in range(count):
            rc = dev.record(k)
            recs.append(edaa.RunRecord(first + k, seeds[k], gammas[k], rc.fit_l1 if rc.ok else 0.0,
                                       rc.coherence if rc.ok else 0.0, wall, bool(rc.ok),
                                       rc.message.decode("utf-8")))
        traces = dev.traces()

        def factors(m: int) -> edaa.RunResult:
            k = m - first
            A, B, E = dev.factors(k)
            rec = recs[k]
            return edaa.RunResult(E, A, B, rec.fit_l1, rec.coherence, rec.seed, rec.gamma,
                                  traces[k].copy())

        return LocalBatch(first, recs, factors)

    return solve


def run_ensemble_sharded(x, config: edaa.EnsembleConfig, group=None,
                         local_solver: Optional[Callable] = None, device: Optional[int] = None):
    """Algorithm 2 over the ranks of `group` (torch.distributed must be initialised).

    Returns (selected RunResult, SelectionReport) on every rank."""
    import torch
    import torch.distributed as dist

    config.validate()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if local_solver is None:
        local_solver = gpu_local_solver(device if device is not None else torch.cuda.current_device())
    first, count = shard_bounds(config.runs, world, rank)
    batch = local_solver(x, config, first, count)

    # ---- all-gather the record table (fixed width: the largest shard) ----
    width = -(-config.runs // world)
    backend = dist.get_backend(group)
    tdev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    mine = torch.full((4, width), float("nan"), dtype=torch.float64, device=tdev)
    for k, rec in enumerate(batch.records):
        mine[0, k] = rec.fit_l1
        mine[1, k] = rec.coherence
        mine[2, k] = 1.0 if rec.ok else 0.0
        mine[3, k] = rec.gamma
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)
    table = [g.cpu().numpy() for g in gathered]
    seeds, gammas = edaa.ensemble_plan(config)
    records = []
    for r in range(world):
        f, c = shard_bounds(config.runs, world, r)
        for k in range(c):
            m = f + k
            ok = bool(table[r][2, k] == 1.0)
            err = ""
            if r == rank:
                err = batch.records[k].error
            records.append(edaa.RunRecord(m, seeds[m], float(table[r][3, k]),
                                          float(table[r][0, k]) if ok else 0.0,
                                          float(table[r][1, k]) if ok else 0.0, 0.0, ok, err))
    report = edaa.select_runs(records, config.fit_slack)

    # ---- the selected run's factors from its owner ----
    sel = report.selected
    owner = next(r for r in range(world) if shard_bounds(config.runs, world, r)[0] <= sel <
                 sum(shard_bounds(config.runs, world, r)))
    L, N = np.asarray(x).shape
    p, T = config.solver.endmembers, config.solver.outer_iters
    flat = torch.zeros(p * N + N * p + L * p + T + 1, dtype=torch.float64, device=tdev)
    if rank == owner:
        res = batch.factors(sel)
        flat.copy_(torch.from_numpy(np.concatenate([res.abundances.ravel(), res.contributions.ravel(),
                                                    res.endmembers.ravel(), res.objective_trace])))
    dist.broadcast(flat, src=dist.get_global_rank(group, owner) if group is not None else owner,
                   group=group)
    v = flat.cpu().numpy()
    o = 0
    A = v[o:o + p * N].reshape(p, N); o += p * N
    B = v[o:o + N * p].reshape(N, p); o += N * p
    E = v[o:o + L * p].reshape(L, p); o += L * p
    trace = v[o:o + T + 1].copy()
    rec = report.per_run[sel]
    return edaa.RunResult(E, A, B, rec.fit_l1, rec.coherence, rec.seed, rec.gamma, trace), report
