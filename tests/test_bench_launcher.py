"""bench.py's own N-rank launcher (no torchrun wrapper): `python bench.py --gpus N` must start N
processes, one per GPU, and refuse to report n_gpus = N from fewer ranks.  Runs on CPU: --dry-launch
goes through the same self_launch / rank bookkeeping / report gather with a gloo group and no kernels."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(*argv, env=None, timeout=240):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, BENCH, *argv], capture_output=True, text=True, env=e, timeout=timeout,
                          cwd=ROOT)


@pytest.mark.parametrize("n", [2, 3])
def test_self_launch_starts_n_ranks(n):
    r = _run("--gpus", str(n), "--dry-launch", "--frames", "4")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout            # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == n and d["ranks"] == list(range(n)) and d["processes"] == n
    assert d["frames"] == 4 * n and d["max_over_ranks"] == float(n)   # MAX over ranks of (1 + rank)


def test_single_rank_dry_launch_needs_no_process_group():
    r = _run("--gpus", "1", "--dry-launch")
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["n_gpus"] == 1


def test_world_size_mismatch_is_refused():
    """Under an external launcher the line must not claim more GPUs than ranks ran."""
    r = _run("--gpus", "4", "--dry-launch", env={"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "refusing to report" in (r.stderr + r.stdout)


def test_more_gpus_than_devices_fails_loudly():
    """No silent N = 1 run: with fewer visible devices than --gpus the bench exits non-zero."""
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:
        have = 0
    r = _run("--gpus", str(have + 2), "--steps", "1")
    assert r.returncode != 0
    assert "refusing to report" in (r.stderr + r.stdout)
    assert not any(l.startswith("{") and '"n_gpus"' in l for l in r.stdout.splitlines())


def test_reference_arm_line_and_numpy_reference_leg():
    """`bench.py --impl reference` (CPU only): the port's line carries the keys of the contract; when the
    unmodified reference package is installed under baseline/_ref (git-ignored) the same run
    also times one frame through it and pins the port against it on that frame."""
    r = _run("--impl", "reference", "--workload", "256_gray_5pct_b16o2", "--steps", "1", "--warmup", "0")
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["gpu_launches"] == 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "diffpaint")):
        n = d["numpy_reference"]
        assert n["kind"] == "reference" and n["value"] > 0
        assert n["v_cycles"] == n["port_v_cycles"]
        assert n["max_abs_port_vs_reference"] <= 1e-9
    else:
        assert "numpy_reference" not in d
