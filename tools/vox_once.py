"""Build one C5-geometry grid (development aid for ncu launch lists of stage 1).
Usage: vox_once.py [points] [voxel] [dv]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_13747_b200 import abi, pcray, scenes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30_000_000
vs = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
dv = int(sys.argv[3]) if len(sys.argv) > 3 else 2
base = scenes.config("C3")
scene = scenes.scene_from_planar(base.planar, scenes.scaled_density(base, n), base.seed)
ds = pcray.DeviceScene(scene)
for _ in range(2):
    g = pcray.build_grid(ds, abi.voxel_params(vs, dv))
    del g
if "--time" in sys.argv:
    import torch

    st = torch.cuda.ExternalStream(pcray.stream_ptr(ds.ctx))
    ms = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        g = pcray.build_grid(ds, abi.voxel_params(vs, dv))
        b.record(st)
        b.synchronize()
        ms.append(a.elapsed_time(b))
        del g
    print(f"build_grid {scene.n_points} points: min {min(ms):.3f} ms")
print("done", scene.n_points)
