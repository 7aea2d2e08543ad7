"""Per-candidate refinement work of a PCR_REFINE_TRACE dump (development aid): the
`.cand` rows (iterations, depth, reflection mask, reason) written by refine_device.

    PCR_REFINE_TRACE=/tmp/rt python tools/profile_stages.py --config C2 --reps 1
    python tools/refine_hist.py /tmp/rt.cand

Prints the iteration distribution, the path-iterations and reflection-node iterations
(the scans a wavefront schedule would launch), and how many paths are still running
after i iterations (the tail a per-iteration launch schedule pays for)."""
import sys

import numpy as np


def main(path):
    a = np.fromfile(path, dtype=np.uint32).reshape(-1, 4)
    it, d, kinds, reason = a[:, 0].astype(np.int64), a[:, 1].astype(np.int64), a[:, 2], a[:, 3].astype(np.int32)
    refl = np.array([bin(int(k)).count("1") for k in kinds]) if len(a) < 200000 else None
    n = len(a)
    print(f"candidates {n}, LOS {int((d == 0).sum())}")
    print(f"iterations: sum {int(it.sum())}  mean {it.mean():.1f}  max {int(it.max())}")
    for q in [0.5, 0.9, 0.99, 0.999]:
        print(f"  p{q * 100:g}: {int(np.quantile(it, q))}")
    print(f"node-iterations (sum it*d): {int((it * d).sum())}")
    # reflection nodes: kinds bit q = 1 for a diffraction (kind & 1) -> reflections = d - popcount
    pc = np.zeros(n, np.int64)
    k = kinds.astype(np.int64)
    for q in range(8):
        pc += (k >> q) & 1
    print(f"reflection-node iterations: {int((it * (d - pc)).sum())}")
    for dd in range(int(d.max()) + 1):
        m = d == dd
        if m.any():
            print(f"  depth {dd}: {int(m.sum())} paths, iterations {int(it[m].sum())}, mean {it[m].mean():.1f}")
    for r in np.unique(reason):
        m = reason == r
        print(f"  reason {r}: {int(m.sum())} paths, iterations {int(it[m].sum())}")
    srt = np.sort(it)
    for i in [1, 2, 5, 10, 20, 50, 100, 200, 500, 1000, 1500, 1999]:
        alive = n - np.searchsorted(srt, i, side="right")
        print(f"  alive after {i:5d} iterations: {alive}")
    del refl


if __name__ == "__main__":
    main(sys.argv[1])
