"""bench.py's contract (the driver's JSON line) on a small workload: one GPU, and two ranks sharing
the GPU over gloo (the N > 1 code path the driver's scaling run takes with NCCL: decomposition,
ghost exchange, max-over-ranks timing, the e2e leg)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(out: str) -> dict:
    lines = [ln for ln in out.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def _check_common(d: dict, n: int, timing=True):
    assert d["metric"].startswith("pair interactions/s")
    assert d["n_gpus"] == n and d["unit"] == "pair interactions/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["scaling"] == "weak"
    assert d["gpu_launches"] > 0
    e = d["e2e"]
    assert e and e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    if timing:  # (ranks sharing one GPU over gloo time each other's work: no relation to check)
        assert e["value"] < d["value"] * 1.05  # the copies are inside e2e's timed region
    assert "clocks" in d


@pytest.mark.gpu
def test_bench_one_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--config", "c2z", "--steps", "2", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    _check_common(d, 1)
    assert d["roofline"]["unit"] == "TFLOP/s" and 0 < d["roofline"]["frac"] < 1
    assert set(d["pass_ms"]) == {"build_lists", "gravity", "geometry", "corrections_extras", "accel_dudt"}


@pytest.mark.gpu
@pytest.mark.slow
def test_bench_two_ranks_sharing_the_gpu():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, CRK_DIST_BACKEND="gloo", CRK_SHARE_GPU="1", CRK_OVERLAP="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                        "--config", "c2z", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1500, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _line(r.stdout)
    _check_common(d, 2, timing=False)
    assert d["config"]["ghost_particles_total"] > 0
