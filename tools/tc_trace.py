"""Summarise a K3-TC CTA-0 timeline written with EXEM_TC_TRACE=<file>."""
import sys

import numpy as np

for f in sys.argv[1:]:
    T = np.loadtxt(f).astype(np.int64)[10:200]
    d = lambda a, b: float(np.median(T[:, b] - T[:, a]))
    print(f)
    print(f"  tile period {np.median(np.diff(T[:, 3])):.0f} cycles (ideal 896 at K=112)")
    print(f"  mma: tempty wait {d(0,1):.0f}  chunk0 full wait {d(1,2):.0f}  "
          f"issue {d(2,3):.0f}  loop {np.median(T[1:,0]-T[:-1,3]):.0f}")
    print(f"  epi: tfull wait {d(4,5):.0f}  load+arrive {d(5,6):.0f}  "
          f"compute {d(6,7):.0f}")
