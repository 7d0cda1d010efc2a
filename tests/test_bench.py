"""bench.py's launcher and bookkeeping (CPU): --gpus N really starts N ranks,
fails loudly without the devices, and the selection-margin summary follows
the reference's rule (ensemble.cpp:71-94)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _env():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return env


def test_gpus_n_without_devices_fails_loudly():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, env=dict(_env(), CUDA_VISIBLE_DEVICES=""),
                       timeout=300)
    assert r.returncode != 0
    assert "needs 2 visible CUDA devices" in r.stderr
    assert r.stdout.strip() == ""


def test_launcher_starts_n_ranks_and_rank0_alone_prints():
    """The reference arm under the launcher (no GPU needed): two ranks start,
    rank 0 alone runs the CPU sample and prints ONE line."""
    cmd = bench.launcher_cmd(2, ["--impl", "reference", "--gpus", "2", "--steps", "1",
                                 "--warmup", "0", "--config", "cfg0"])
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert cmd[cmd.index("--nproc-per-node") + 1] == "2"
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    r = subprocess.run(cmd, capture_output=True, text=True, env=_env(), timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(s) for s in r.stdout.splitlines() if s.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert "T=4 minus T=1" in line["cpu_baseline"]["sample"]


def test_selection_margins_follow_the_reference_rule():
    fits = [10.0, 10.4, 11.0, 9.9]
    mus = [0.9, 0.8, 0.1, 0.85]
    oks = [1, 1, 1, 0]
    m = bench.selection_margins(fits, mus, oks, 1.05)   # test_ensemble.cpp:38-65 case
    assert m["selected"] == 1 and m["candidates"] == 2
    assert np.isclose(m["mu_gap_to_runner_up_rel"], (0.9 - 0.8) / 0.8)
    assert np.isclose(m["nearest_fit_to_cutoff_rel"], abs(10.4 - 10.5) / 10.5)
    assert bench.selection_margins([1.0], [0.5], [0], 1.05) is None


def test_strong_split_covers_every_run_once():
    from paper_2209_11002_b200.distributed import shard_bounds
    for world in (1, 2, 3, 4, 8):
        got = []
        for r in range(world):
            first, count = shard_bounds(64, world, r)
            got.extend(range(first, first + count))
        assert got == list(range(64))
