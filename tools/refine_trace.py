"""Summarise a PCR_REFINE_TRACE dump (per refine thread: start ns, end ns, paths):
how much of the kernel's thread-time is spent before each thread runs out of work
(development aid for the persistent refine kernel's tail)."""
import sys

import numpy as np


def main(path):
    a = np.fromfile(path, dtype=np.uint64).reshape(-1, 3).astype(np.float64)
    a = a[a[:, 1] > 0]
    t0, t1 = a[:, 0].min(), a[:, 1].max()
    span = t1 - t0
    busy = (a[:, 1] - a[:, 0]).sum() / (len(a) * span)
    ends = np.sort((a[:, 1] - t0) / span)
    print(f"threads {len(a)}  kernel {span / 1e6:.1f} ms  thread-busy fraction {busy:.3f}")
    for q in [0.1, 0.25, 0.5, 0.75, 0.9, 0.99]:
        print(f"  {int(q * 100):3d}% of threads done by {ends[int(q * (len(ends) - 1))]:.3f} of the kernel")
    print("  paths per thread: mean %.2f max %d" % (a[:, 2].mean(), a[:, 2].max()))


if __name__ == "__main__":
    main(sys.argv[1])
