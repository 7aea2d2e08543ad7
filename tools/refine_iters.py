"""Development aid: refine iterations, outcome counts and stage times of one config
(default C2) after a warm-up run — for A/B of the refine kernel's exact early exits."""
import sys

sys.path.insert(0, ".")
from paper_2402_13747_b200 import abi, pcray, scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
scene, cfg = scenes.build_scene(name)
conf = abi.default_run_config(**cfg.run)
ds = pcray.DeviceScene(scene)
pcray.run_pipeline_device(ds, conf)
s = pcray.run_pipeline_device(ds, conf)
print(name, "iterations", s["refine_iterations"], "rejected", list(s["rejected"]), "exact", s["exact_paths"],
      "hash", s["hash"], {k: round(v, 3) for k, v in s["timings"]})
