"""Per-shard work of the sharded pipeline (SURVEY 8e load balance): every shard of
run_pipeline_sharded_local runs alone on the one GPU, so its device seconds are its
share of the work at full-GPU speed; max / mean per stage is the imbalance the
cyclic splits (initial hits for trace, candidates for refine) leave at G shards.

  python tools/shard_balance.py [--configs C2,C3] [--shards 2,4,8] [--out profiles/shard_balance_r02.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2402_13747_b200 import abi, pcray, scenes, shard  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2")
    ap.add_argument("--shards", default="2,4,8")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "shard_balance_r02.json"))
    args = ap.parse_args()
    rows = []
    for name in args.configs.split(","):
        scene, cfg = scenes.build_scene(name)
        conf = abi.default_run_config(**cfg.run)
        ref = pcray.run_pipeline_on_scene(scene, conf)
        for g in [int(x) for x in args.shards.split(",")]:
            t = {}
            s = shard.run_pipeline_sharded_local(scene, conf, g, times=t)
            assert s["exact_paths"] == ref["exact_paths"] and s["coarse_paths"] == ref["coarse_paths"]
            row = {"config": name, "run": cfg.run, "shards": g}
            for k in ["trace", "refine"]:
                v = t[k]
                mean = sum(v) / len(v)
                row[k] = {"seconds": v, "max_over_mean": max(v) / mean if mean else None}
            rows.append(row)
            print(json.dumps(row), flush=True)
    with open(args.out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
