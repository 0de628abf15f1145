"""The checked build (device range checks, VR_CHECK in csrc/common.cuh) over every backward
variant: compute-sanitizer is closed on this GPU pool, so the library is also built with
checks at the hot global accesses (a sample's ray index, the hash-table entry of every
gather and scatter), and a run of small training steps through each variant must count
zero failures (scripts/sanitize.py)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.gpu


def test_checked_build_counts_no_range_failures():
    lib = ROOT / "paper_2404_16221_b200" / "libvolray_b200_checked.so"
    assert lib.exists(), "run __graft_entry__.build() (builds the checked library too)"
    env = dict(os.environ, VR_CHECKED="1")
    r = subprocess.run([sys.executable, str(ROOT / "scripts" / "sanitize.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0
    assert "checked build: 0 range-check failures" in r.stdout


def test_checked_build_detects_a_bad_ray_index():
    """The checks fire: a sample whose ray id is out of range is counted (and skipped)."""
    code = r'''
import numpy as np, torch
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200 import _lib
lib = _lib.load()
assert lib.vr_check_failures() == 0
f = vr.HashGridMLP(vr.HashGridConfig(log2_T=12, max_res=64), vr.Aabb([-1,-1,-1],[1,1,1]), "cuda")
rays = torch.zeros((8, 4), dtype=torch.float64, device="cuda"); rays[3] = 1.0
t0 = torch.zeros(16, dtype=torch.float64, device="cuda"); t1 = t0 + 0.1
rid = torch.full((16,), 7, dtype=torch.int32, device="cuda")  # only 4 rays
out = torch.empty((16, 4), device="cuda")
f.forward(rays, t0, t1, rid, 16, out, _lib.stream_ptr())
print("failures", lib.vr_check_failures())
'''
    env = dict(os.environ, VR_CHECKED="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300, cwd=str(ROOT))
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0
    n = int(r.stdout.split("failures")[-1])
    assert n > 0
