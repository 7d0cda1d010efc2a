import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a path")


@pytest.fixture(scope="session")
def oracle_kinds():
    from oracle import available_kinds
    return available_kinds()


def golden_files(prefix=""):
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".npz") and f.startswith(prefix))


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def golden_scene(g):
    """Regenerate a golden fixture's input image and check its pinned hash."""
    import hashlib
    from paper_2209_11002_b200 import synth
    if "config" in g:
        x = synth.generate(synth.CONFIGS[str(g["config"])])[0]
    else:
        snr = float(g["snr"])
        spec = synth.SceneSpec("golden", int(g["bands"]), int(g["pixels"]), int(g["p"]), 1,
                               float(g["alpha"]), None if np.isnan(snr) else snr)
        x = synth.generate(spec, seed=int(g["scene_seed"]))[0]
    digest = hashlib.sha256(np.ascontiguousarray(x, dtype=np.float32).tobytes()).hexdigest()
    assert digest == str(g["x_sha"]), "synthetic generator drifted from the golden fixture"
    return x
