"""bench.py contract on the GPU: one JSON line with the driver's keys, at N = 1 and under
torchrun at N = 2 (two ranks sharing the one visible GPU over gloo: SG2V_BENCH_SHARED_GPU=1,
the 8-GPU node runs the same code with NCCL, one rank per GPU).  Small scale, u12-1."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks", "status"}


def _line(out):
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def test_bench_single_gpu_line():
    p = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--scale", "14",
                        "--template", "u12-1", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    d = _line(p.stdout)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0 and d["status"] == "OK"
    assert d["roofline"]["unit"] == "GB/s" and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0


def test_bench_two_ranks_torchrun():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, SG2V_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--scale", "14", "--template", "u12-1", "--no-cpu-baseline"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    d = _line(p.stdout)
    assert d["n_gpus"] == 2 and d["config"]["colourings"] == 4 and d["scaling"] == "weak" and d["value"] > 0
