"""bench.py's contract lines on a real GPU: the single-GPU line (short run) and the
N > 1 sharded path under torchrun (gloo backend, both ranks on the box's one GPU —
a functional run of the code the driver's scaling step uses with NCCL)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"}


def _golden_c2():
    """The bench workload's counts as the oracle computes them on the full scene
    (tests/golden/make_contract_golden.py)."""
    with open(os.path.join(ROOT, "tests", "golden", "contract_C2.json")) as f:
        g = json.load(f)
    return g["summary"]["exact_paths"], g["summary"]["coarse_paths"], g["cone_traces"] + g["transmission_rays"]


def _last_json(out):
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "1", "--warmup", "3", "--no-cpu-baseline"], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert line["roofline"]["kernel"] == "refine" and 0 < line["roofline"]["frac"] < 1
    exact, coarse, rays = _golden_c2()
    assert line["config"]["max_interactions"] == 4 and line["config"]["max_diffractions"] == 1
    assert line["exact_paths"] == exact and line["coarse_paths"] == coarse and line["rays_per_step"] == rays


def test_bench_two_ranks_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "3",
           "--backend", "gloo"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert KEYS <= set(line)
    exact, coarse, rays = _golden_c2()
    assert line["n_gpus"] == 2 and line["exact_paths"] == exact and line["coarse_paths"] == coarse
