"""Summarise a K3-TC CTA-0 timeline written with EXEM_TC_TRACE=<file>.

Slots per tile t (clock64 of CTA 0):
  0  issuer reaches the wait for tile t's accumulator buffer (pipelined path:
     inside tile t-1's issue, before its last two MMAs)
  1  ... buffer free (tempty)      2  ... B stage landed (full)
  3  tile t's MMAs issued + committed
  4  epilogue starts waiting for tile t    5  tfull seen
  6  accumulator drained, buffer released  7  relu-sum done
"""
import sys

import numpy as np

for f in sys.argv[1:]:
    T = np.loadtxt(f).astype(np.int64)[10:200]
    d = lambda a, b: float(np.median(T[:, b] - T[:, a]))
    print(f)
    print(f"  tile period {np.median(np.diff(T[:, 3])):.0f} cycles")
    print(f"  issuer: tempty stall {d(0, 1):.0f}  full stall {d(1, 2):.0f}  "
          f"wait->commit {d(2, 3):.0f}")
    print(f"  epilogue: tfull wait {d(4, 5):.0f}  drain+release {d(5, 6):.0f}  "
          f"relu-sum {d(6, 7):.0f}")
    # commit of tile t -> epilogue sees it; release of t -> issuer gets it (t+2)
    print(f"  commit->tfull seen {float(np.median(T[:, 5] - T[:, 3])):.0f}  "
          f"release->issuer {float(np.median(T[2:, 1] - T[:-2, 6])):.0f}")
