"""The multi-GPU host driver (paper_2402_13747_b200/mgpu/pcray_mgpu.cpp: one process per
GPU, every exchange over NCCL) on the box's one GPU: world size 1 runs the NCCL
broadcast / all-gather / all-reduce code path end to end (a communicator of one rank),
in both grid modes (rank 0 builds + ncclBroadcast; sharded parts + ncclAllGather). The
RunSummary and the JSONL must equal the single-process pipeline's from the same files
(pcr_run_pipeline), which the other tests pin to the reference. More ranks than GPUs
cannot share one NCCL communicator; the multi-rank exchange logic is covered by the
gloo tests of shard.py (tests/test_shard_gpu.py, tests/test_voxshard_gpu.py)."""
import json
import os
import socket
import subprocess

import pytest

from paper_2402_13747_b200 import abi, pcray, scenes
from test_io_gpu import _save_edges

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2402_13747_b200", "mgpu", "_build", "pcray_mgpu")


def _files(oracle, tmp_path, name):
    scene, _ = scenes.build_scene(name)
    ply, edges, radios = str(tmp_path / "s.ply"), str(tmp_path / "e.txt"), str(tmp_path / "r.txt")
    oracle.save_point_cloud(ply, oracle.RefScene(scene), True)
    _save_edges(edges, scene)
    with open(radios, "w") as f:
        for p in scene.tx:
            f.write("tx %r %r %r\n" % tuple(float(x) for x in p))
        for p in scene.rx:
            f.write("rx %r %r %r\n" % tuple(float(x) for x in p))
    return scene, ply, edges, radios


@pytest.mark.parametrize("name,mi,md", [("C1", 2, 0), ("C2", 2, 1)])
@pytest.mark.parametrize("mode", ["broadcast", "sharded"])
def test_mgpu_driver_world1_matches_pipeline(oracle, gpu, tmp_path, name, mi, md, mode):
    if not os.path.exists(EXE):
        pytest.skip("pcray_mgpu not built")
    scene, ply, edges, radios = _files(oracle, tmp_path, name)
    out = str(tmp_path / "mgpu.jsonl")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_PORT=str(port),
               PCRAY_NCCL_ID=str(tmp_path / "nccl.id"))
    r = subprocess.run([EXE, "--ply", ply, "--edges", edges, "--radios", radios, "--out", out, "--grid", mode,
                        "--max-interactions", str(mi), "--max-diffractions", str(md)],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    ref_out = str(tmp_path / "ref.jsonl")
    want = pcray.run_pipeline(ply, edges, ref_out, scene.tx, scene.rx, abi.default_run_config(max_interactions=mi,
                                                                                              max_diffractions=md))
    for k in ["point_count", "ie_count", "coarse_paths", "refined_paths", "exact_paths", "cone_traces",
              "transmission_rays", "hash"]:
        assert got[k] == want[k], k
    assert got["rejected"] == list(want["rejected"])
    assert got["world"] == 1 and got["rows_per_rank"][0] > 0
    assert open(out, "rb").read() == open(ref_out, "rb").read()
