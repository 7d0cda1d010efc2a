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
    mine_h = np.full((5, width), np.nan)
    for k, rec in enumerate(batch.records):
        mine_h[:, k] = (rec.fit_l1, rec.coherence, 1.0 if rec.ok else 0.0, rec.gamma, rec.wall_ms)
    mine = torch.from_numpy(mine_h).to(tdev)
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)
    table = [g.cpu().numpy() for g in gathered]
    seeds, gammas = edaa.ensemble_plan(config)
    # Failed runs carry the reference's error text (ensemble.cpp:150-155 →
    # report.json "error"): gathered as objects only when some run failed, so the
    # healthy path stays one tensor all-gather and every rank builds the SAME report.
    errors = [{} for _ in range(world)]
    if any(not bool(np.all(t[2, :shard_bounds(config.runs, world, r)[1]] == 1.0)) for r, t in enumerate(table)):
        dist.all_gather_object(errors, {rec.index: rec.error for rec in batch.records if not rec.ok},
                               group=group)
    records = []
    for r in range(world):
        f, c = shard_bounds(config.runs, world, r)
        for k in range(c):
            m = f + k
            ok = bool(table[r][2, k] == 1.0)
            records.append(edaa.RunRecord(m, seeds[m], float(table[r][3, k]),
                                          float(table[r][0, k]) if ok else 0.0,
                                          float(table[r][1, k]) if ok else 0.0,
                                          float(table[r][4, k]), ok, errors[r].get(m, "")))
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


# ---------------------------------------------------------------------------
# Pixel sharding of one solve: the pixels of a single run (or of a
# whole batch) split over the ranks by pixel SLICE, the partial sums of every
# pass exchanged over NCCL inside the device schedule (include/edaa_b200.h,
# edaa_set_pixel_shard).  The host side here only distributes the communicator
# id and mirrors the device's slice plan.

NP = 32            # pixels per tile (csrc/edaa_internal.cuh kNP)
TILES_PER_SLICE = 4
SMALL_TILES_PER_SLICE = 2
MAX_SLICES = 148


def pixel_slices(pixels: int) -> int:
    """Number of pixel slices of an N-pixel image (a function of N only, as in make_dims)."""
    ntiles = 2 * -(-pixels // (2 * NP))   # Npad is a multiple of 64: an even number of 32-pixel tiles
    tps = SMALL_TILES_PER_SLICE if ntiles <= 2 * MAX_SLICES else TILES_PER_SLICE   # edaa::slice_count
    return min(MAX_SLICES, -(-ntiles // tps))


def pixel_shard_plan(pixels: int, world: int, rank: int):
    """(first slice, end slice, first pixel, end pixel) owned by `rank` — the
    device's shard_slices / slice_pixels, clipped to the image."""
    ntiles = 2 * -(-pixels // (2 * NP))
    ns = pixel_slices(pixels)
    if ns < world:
        raise edaa.EdaaError("image too small to shard its pixels over that many devices")
    s0, s1 = rank * ns // world, (rank + 1) * ns // world
    # edaa::slice_first_tile: slices are made of 64-pixel tile pairs
    j0, j1 = 2 * (s0 * (ntiles // 2) // ns) * NP, 2 * (s1 * (ntiles // 2) // ns) * NP
    return s0, s1, min(j0, pixels), min(j1, pixels)


def share_communicator_id(make_id: Callable[[], bytes], group=None) -> bytes:
    """Rank 0 makes the NCCL id, every rank of `group` receives the same bytes."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def join_pixel_shard(dev: "edaa.Device", group=None) -> int:
    """Make `dev` this rank's member of a pixel-sharding communicator over `group`."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world <= 1:
        dev.set_pixel_shard(None, 0, 1)
        return 1
    uid = share_communicator_id(dev.nccl_unique_id, group)
    dev.set_pixel_shard(uid, rank, world)
    return world


def run_pixel_sharded(x, config: edaa.SolverConfig, group=None, device: Optional[int] = None):
    """Algorithm 1 for ONE run with its pixels split over the ranks of `group`
    (one GPU each).  Every rank returns the full RunResult — bitwise the
    single-GPU `edaa.run` result (the exchange keeps the fixed slice order)."""
    import torch
    config.validate()
    xf = edaa.validate_image(x)
    dev = edaa.Device.get(device if device is not None else torch.cuda.current_device())
    join_pixel_shard(dev, group)
    try:
        dev.set_image(xf)
        dev.solve(config.endmembers, config.outer_iters, config.inner_iters_a, config.inner_iters_b,
                  [config.seed], [config.gamma])
        rec = dev.record(0)
        if not rec.ok:
            raise edaa.EdaaError(rec.message.decode("utf-8"))
        A, B, E = dev.factors(0)
        return edaa.RunResult(E, A, B, rec.fit_l1, rec.coherence, config.seed, config.gamma,
                              dev.traces()[0].copy())
    finally:
        dev.set_pixel_shard(None, 0, 1)
