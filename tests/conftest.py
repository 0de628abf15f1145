import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def load_npz(name):
    d = np.load(GOLDEN / name, allow_pickle=False)
    out = {k: d[k] for k in d.files}
    for k in ("tree", "scene", "camera", "stats", "report", "root"):
        if k in out:
            out[k] = json.loads(str(out[k]))
    return out


def sampler_fixtures():
    return sorted(p.name for p in GOLDEN.glob("sampler_*.npz"))


def render_fixtures():
    return sorted(p.name for p in GOLDEN.glob("render_*.npz"))


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
