"""Ensemble sharding across ranks (paper_2209_11002_b200/distributed.py), world_size 2
on CPU with gloo.  The per-rank solve is the CPU oracle here (test infrastructure
standing in for the GPU solve); what is under test is the sharding, the record
all-gather, the selection on every rank and the broadcast of the selected run."""
import os
import socket

import numpy as np
import pytest

from paper_2209_11002_b200 import distributed, edaa, synth


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def oracle_local_solver(x, config, first, count):
    from oracle import Oracle
    orc = Oracle()
    seeds, gammas = edaa.ensemble_plan(config, first=first, count=count)
    recs, results = [], {}
    s = config.solver
    for k in range(count):
        m = first + k
        r = orc.run(np.asarray(x, dtype=np.float64), s.endmembers, T=s.outer_iters,
                    K1=s.inner_iters_a, K2=s.inner_iters_b, gamma=gammas[k], seed=seeds[k])
        recs.append(edaa.RunRecord(m, seeds[k], gammas[k], r.fit_l1, r.coherence, 0.0, True, ""))
        results[m] = edaa.RunResult(r.E, r.A, r.B, r.fit_l1, r.coherence, seeds[k], gammas[k], r.trace)
    return distributed.LocalBatch(first, recs, lambda m: results[m])


def _worker(rank, world, port, runs, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = synth.small_scene(16, 200, 3, seed=4)
    cfg = edaa.EnsembleConfig(runs=runs, solver=edaa.SolverConfig(endmembers=3, outer_iters=6))
    res, rep = distributed.run_ensemble_sharded(x, cfg, local_solver=oracle_local_solver)
    np.savez(out % rank, selected=rep.selected, cand=np.array(rep.candidate_set),
             fits=np.array([r.fit_l1 for r in rep.per_run]), A=res.abundances, B=res.contributions,
             E=res.endmembers, trace=res.objective_trace)
    dist.destroy_process_group()


def test_shard_bounds_cover_every_run_once():
    for runs in (1, 2, 5, 50, 64):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                f, c = distributed.shard_bounds(runs, world, r)
                seen += list(range(f, f + c))
            assert seen == list(range(runs))


@pytest.mark.skipif(not __import__("oracle").available_kinds(), reason="oracle not built")
@pytest.mark.parametrize("runs", [7, 1])
def test_sharded_selection_matches_single_process(tmp_path, runs):
    import torch.multiprocessing as mp
    from oracle import Oracle
    out = str(tmp_path / "rank%d.npz")
    mp.spawn(_worker, args=(2, free_port(), runs, out), nprocs=2, join=True)
    r0, r1 = np.load(out % 0), np.load(out % 1)
    x = synth.small_scene(16, 200, 3, seed=4).astype(np.float64)
    ref = Oracle().run_ensemble(x, 3, M=runs, T=6)
    for r in (r0, r1):  # every rank holds the same answer
        assert int(r["selected"]) == ref.selected
        assert list(r["cand"]) == ref.candidates
        assert np.array_equal(r["fits"], ref.fits)
        assert np.array_equal(r["A"], ref.A) and np.array_equal(r["B"], ref.B)
        assert np.array_equal(r["trace"], ref.trace)


def failing_local_solver(x, config, first, count):
    """The oracle solver, with ensemble member 5 reported as failed (its owner
    is rank 1 at world 2) and a distinct wall time per run."""
    batch = oracle_local_solver(x, config, first, count)
    for rec in batch.records:
        rec.wall_ms = 10.0 + rec.index
        if rec.index == 5:
            rec.ok, rec.fit_l1, rec.coherence = False, 0.0, 0.0
            rec.error = "non-finite abundance iterate at outer iteration 3"
    return batch


def _report_worker(rank, world, port, out):
    import json
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = synth.small_scene(16, 200, 3, seed=4)
    cfg = edaa.EnsembleConfig(runs=7, solver=edaa.SolverConfig(endmembers=3, outer_iters=4))
    _, rep = distributed.run_ensemble_sharded(x, cfg, local_solver=failing_local_solver)
    with open(out % rank, "w") as f:
        json.dump([[r.index, r.seed, r.gamma, r.fit_l1, r.coherence, r.wall_ms, r.ok, r.error]
                   for r in rep.per_run] + [rep.selected, rep.candidate_set], f)
    dist.destroy_process_group()


@pytest.mark.skipif(not __import__("oracle").available_kinds(), reason="oracle not built")
def test_every_rank_builds_the_same_report_including_failed_runs(tmp_path):
    """A failed run's error text (report.json "error", outputs.cpp:33-35) and the
    wall times reach every rank: the SelectionReport is identical on all of them."""
    import json
    import torch.multiprocessing as mp
    out = str(tmp_path / "rep%d.json")
    mp.spawn(_report_worker, args=(2, free_port(), out), nprocs=2, join=True)
    r0, r1 = json.load(open(out % 0)), json.load(open(out % 1))
    assert r0 == r1
    assert r0[5][6] is False and r0[5][7] == "non-finite abundance iterate at outer iteration 3"
    assert [rec[5] for rec in r0[:7]] == [10.0 + i for i in range(7)]
    assert 5 not in r0[-1]


# ---- pixel sharding of one solve (distributed.run_pixel_sharded) -----------------

@pytest.mark.parametrize("pixels", [1, 31, 500, 4000, 10000, 94249, 1048576])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_pixel_shard_plan_partitions_the_image(pixels, world):
    ns = distributed.pixel_slices(pixels)
    if ns < world:
        with pytest.raises(edaa.EdaaError, match="too small"):
            distributed.pixel_shard_plan(pixels, world, 0)
        return
    pix, sl = [], []
    for r in range(world):
        s0, s1, j0, j1 = distributed.pixel_shard_plan(pixels, world, r)
        assert s1 > s0 and j0 % distributed.NP == 0
        sl.append((s0, s1))
        pix += list(range(j0, j1))
    assert pix == list(range(pixels))                       # every pixel owned once, in order
    assert sl[0][0] == 0 and sl[-1][1] == ns
    assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))    # contiguous slice ranges


class _FakeDevice:
    """Records what the launcher asks of the device (the C-ABI needs a GPU)."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []

    def nccl_unique_id(self):
        return bytes([7, self.rank]) + bytes(126)

    def set_pixel_shard(self, uid, rank, world):
        self.calls.append((uid, rank, world))


def _shard_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = _FakeDevice(rank)
    w = distributed.join_pixel_shard(dev)
    plan = distributed.pixel_shard_plan(10000, world, rank)
    np.savez(out % rank, uid=np.frombuffer(dev.calls[0][0], np.uint8), rank=dev.calls[0][1],
             world=dev.calls[0][2], w=w, plan=np.array(plan))
    dist.destroy_process_group()


def test_pixel_shard_join_shares_one_communicator_id(tmp_path):
    """world 2 over gloo: rank 0's NCCL id reaches every rank unchanged, each joins
    with its own rank, and the ranks' pixel plans tile the image."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "shard%d.npz")
    mp.spawn(_shard_worker, args=(2, free_port(), out), nprocs=2, join=True)
    r0, r1 = np.load(out % 0), np.load(out % 1)
    assert bytes(r0["uid"]) == bytes(r1["uid"]) == bytes([7, 0]) + bytes(126)
    assert (int(r0["rank"]), int(r1["rank"])) == (0, 1)
    assert int(r0["world"]) == int(r1["world"]) == 2 == int(r0["w"])
    assert r0["plan"][3] == r1["plan"][2] and r0["plan"][2] == 0 and r1["plan"][3] == 10000


@pytest.mark.parametrize("pixels", [1, 63, 64, 65, 9025, 9472, 9473, 10000, 94249, 1048576])
def test_pixel_slices_are_made_of_64_pixel_tile_pairs(pixels):
    """edaa::slice_count / slice_first_tile (mirrored here): slice boundaries are multiples of 64
    pixels — the B pass's 64-pixel logical tiles never straddle a slice — no slice is empty, and
    small images (at most 296 tiles) take one tile pair per slice."""
    ns = distributed.pixel_slices(pixels)
    ntiles = 2 * -(-pixels // 64)
    assert 1 <= ns <= distributed.MAX_SLICES
    bounds = [2 * (s * (ntiles // 2) // ns) for s in range(ns + 1)]
    assert bounds[0] == 0 and bounds[-1] == ntiles
    assert all(b > a and (b - a) % 2 == 0 for a, b in zip(bounds, bounds[1:]))
    if ntiles <= 2 * distributed.MAX_SLICES:
        assert ns == ntiles // 2
    # the plan of a 1-rank world covers the image
    assert distributed.pixel_shard_plan(pixels, 1, 0) == (0, ns, 0, pixels)
