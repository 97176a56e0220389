"""Summarise a K4-TC CTA-0 timeline written with EXEM_TCB_TRACE=<file>.

Slots per point tile t (clock64 on CTA 0):
  0 issuer acquired tile t's accumulator buffer (tempty)
  1 issuer: tile t's first point chunk landed (full)
  2 issuer committed tile t (tfull)
  3 epilogue (warp 2) saw tfull of tile t     4 ... released its buffer
  5 producer: slot for tile t's first chunk free   6 ... last TMA of tile t issued
  7-11 issuer, chunk 1 of tile t (chunk 0 if one chunk): before head MMAs,
       after head MMAs, after the waits, after tail MMAs, after commit
"""
import sys

import numpy as np

for f in sys.argv[1:]:
    T = np.loadtxt(f).astype(np.int64)[8:240]
    med = lambda x: float(np.median(x))
    print(f)
    print(f"  tile period {med(np.diff(T[:, 2])):.0f} cycles")
    print(f"  issuer: buffer->first chunk {med(T[:, 1] - T[:, 0]):.0f}  "
          f"first chunk->commit {med(T[:, 2] - T[:, 1]):.0f}")
    print(f"  commit->tfull seen {med(T[:, 3] - T[:, 2]):.0f}  "
          f"epilogue {med(T[:, 4] - T[:, 3]):.0f}  "
          f"release(t)->issuer acquires(t+2) {med(T[2:, 0] - T[:-2, 4]):.0f}")
    print(f"  producer: first slot free->last TMA {med(T[:, 6] - T[:, 5]):.0f}  "
          f"last TMA->issuer sees first chunk {med(T[:, 1] - T[:, 6]):.0f}  "
          f"(negative: data early)")
    if T.shape[1] > 11:
        print(f"  chunk: head MMAs {med(T[:, 8] - T[:, 7]):.0f}  waits "
              f"{med(T[:, 9] - T[:, 8]):.0f}  tail MMAs {med(T[:, 10] - T[:, 9]):.0f}"
              f"  commit {med(T[:, 11] - T[:, 10]):.0f}")
