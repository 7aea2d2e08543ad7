"""Development aid: the C2 pipeline through the resident-scene call and the host-buffer
call, alternating, with per-stage wall times and (optionally, --kt) per-kernel device
times, to separate host gaps from kernel time."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2402_13747_b200 import abi, pcray, scenes  # noqa: E402

kt = "--kt" in sys.argv
scene, cfg = scenes.build_scene("C2")
conf = abi.default_run_config(**cfg.run)
ctx = pcray.Context.default()
ds = pcray.DeviceScene(scene)
pin = {}
for name in ["position", "normal", "label", "edges", "edge_label", "tx", "tx_id", "rx", "rx_id"]:
    a = np.ascontiguousarray(getattr(scene, name))
    t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    t.numpy()[...] = a
    pin[name] = t.numpy()
hs = abi.Scene(pin["position"], pin["normal"], pin["label"], pin["edges"], pin["edge_label"], pin["tx"], pin["tx_id"],
               pin["rx"], pin["rx_id"], scene.carrier_frequency_hz)
pcray.run_pipeline_device(ds, conf)
for rep in range(3):
    for name, fn in [("device", lambda: pcray.run_pipeline_device(ds, conf)),
                     ("host", lambda: pcray.run_pipeline_on_scene(hs, conf, ctx))]:
        if kt:
            pcray.kernel_times(reset=True, ctx=ctx)
            pcray.set_profiling(1, ctx)
        torch.cuda.synchronize()
        t0 = time.time()
        s = fn()
        t1 = time.time()
        tm = dict(s["timings"])
        line = f"{name} {t1 - t0:.3f} trace {tm['trace']:.3f} refine {tm['refine']:.3f}"
        if kt:
            k = pcray.kernel_times(reset=True, ctx=ctx)
            pcray.set_profiling(0, ctx)
            tr = sum(v[0] for n, v in k.items() if n in ("cone_walk", "visibility", "materialize", "transmission", "kappa_select"))
            line += f" trace-kernels {tr / 1e3:.3f} " + " ".join(f"{n}={v[0] / 1e3:.3f}" for n, v in k.items() if v[0] > 20)
        print(line, flush=True)
