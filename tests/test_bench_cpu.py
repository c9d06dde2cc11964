"""bench.py host logic on CPU: the reference arm's composed sweeps and the multi-rank launch.

* ``RefSweep`` (the reference arm and the b200 line's cpu_baseline) computes output t-windows of
  the full lattice through su3bench's own routines; every window must equal the oracle's rows.
* ``--gpus N`` without torchrun spawns its N ranks itself (gloo on CPU for the reference arm);
  rank 0 alone prints one JSON line.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import sweeps as S  # noqa: E402


def _cfg(kind, dims):
    return {"kind": kind, "global_dims": dims, "name": "test"}


@pytest.mark.parametrize("use_ref", [True, False], ids=["su3bench", "port"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_ref_sweep_windows_equal_the_oracle(use_ref, dtype, monkeypatch):
    if use_ref and bench._su3bench() is None:
        pytest.skip("baseline/_ref (su3bench) not installed")
    if not use_ref:
        monkeypatch.setattr(bench, "_su3bench", lambda: None)
    dims = (4, 3, 2, 6)
    F = 24
    nn = bench.RefSweep(_cfg("nn", dims), dtype)
    assert nn.source == ("reference" if use_ref else "port")
    want = S.nn_sweep(nn.U, nn.v, dims)
    for t0, k in ((0, 2), (2, 3), (4, 2), (5, 1), (0, 6)):
        assert np.array_equal(nn(t0, k), want[t0 * F : (t0 + k) * F]), (t0, k)
    lk = bench.RefSweep(_cfg("link", dims), dtype)
    want = S.link_product(lk.U, dims, 1 / 6)
    for t0, k in ((0, 3), (3, 3), (5, 1)):
        assert np.array_equal(lk(t0, k), want[t0 * F : (t0 + k) * F]), (t0, k)


def test_sample_slices_divide_the_lattice():
    assert bench._sample_slices(_cfg("nn", (64, 64, 64, 16))) == 2
    assert bench._sample_slices(_cfg("link", (48, 48, 48, 48))) == 1
    k = bench._sample_slices(_cfg("nn", (8, 8, 8, 6)))
    assert 6 % k == 0


def test_reference_arm_same_config_single_core():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--dims", "8,8,8,4",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["cores"] == 1
    assert line["config"]["same_config"] is False  # --dims override
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert "upper_bound_aggregate" in line and "upper bound" in line["upper_bound_aggregate"]["label"]


def test_bench_spawns_its_ranks_without_torchrun():
    """`bench.py --gpus 2` (no launcher): two ranks over gloo, one JSON line from rank 0."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "SU3G_BENCH_SPAWNED")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--dims", "8,8,8,4", "--steps", "3", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
    assert line["config"]["lattice"] == [8, 8, 8, 8]  # weak scaling: 16*N slices per rank -> nt = 4 * 2
