"""Regenerate the golden fixtures of tests/golden from the oracle (the unmodified
reference compiled in oracle/_ref). Run here, where /root/reference exists:

    python tests/golden/make_golden.py

The fixtures let the GPU parity tests run on a box without the oracle, and the CPU
suite checks that the oracle still reproduces them.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from fixtures import box_room, make_scene, voxel_grid_scenes  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2402_13747_b200 import abi, scenes  # noqa: E402

GRID_SCENES = ["single_point", "edge_clip", "reception_points", "partition", "determinism", "oblique_edge"]


def golden_scene(name):
    if name == "box_room":
        return make_scene(box_room((2, 2, 2), 0.05), tx=[(0.6, 0.7, 0.9)], rx=[(1.3, 1.2, 1.1)])
    if name == "c1":
        return scenes.build_scene("C1")[0]
    return voxel_grid_scenes()[name]


def save_dict(path, d, prefix=""):
    flat = {}
    for k, v in d.items():
        if isinstance(v, dict):
            for k2, v2 in v.items():
                flat[f"{k}.{k2}"] = np.asarray(v2)
        else:
            flat[k] = np.asarray(v)
    np.savez_compressed(path, **flat)


def main():
    for name in GRID_SCENES:
        g = ref.build_grid(ref.RefScene(golden_scene(name))).to_dict()
        save_dict(os.path.join(HERE, f"grid_{name}.npz"), g)
    sc = golden_scene("box_room")
    rs = ref.RefScene(sc)
    rg = ref.build_grid(rs)
    tp = abi.trace_params(max_interactions=2, max_diffractions=0)
    los, hits = ref.transmission_phase(rg, rs, 0, tp)
    cands = ref.propagate(rg, rs, 0, hits, tp)
    out = ref.refine_batch(rg, rs, cands)
    save_dict(os.path.join(HERE, "trace_box_room_mi2.npz"), {"los": los, "hits": hits, "cands": cands, "out": out})
    c1, cfg = scenes.build_scene("C1")
    s = ref.run_pipeline_on_scene(ref.RefScene(c1), ref.default_run_config(**cfg.run))
    keep = {k: s[k] for k in ["point_count", "ie_count", "grid_dims", "coarse_paths", "refined_paths", "rejected",
                              "exact_paths", "hash"]}
    keep["paths"] = {"length": s["paths"]["length"].tolist(), "n_inter": s["paths"]["n_inter"].tolist(),
                     "rx_id": s["paths"]["rx_id"].tolist()}
    with open(os.path.join(HERE, "smoke_c1.json"), "w") as f:
        json.dump(keep, f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
