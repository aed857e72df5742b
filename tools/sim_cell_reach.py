"""CPU replay of one image's forward candidate scan (development diagnostic): batches of 32 a
32x16 tile walks with the image-wide support extent alone, and with the per-cell reach bound
(max clipped support right / bottom edge of a cell's Gaussians) trimming each cell row's span.
usage: python tools/sim_cell_reach.py [H W s]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import gsr_synth as S  # noqa: E402
import oracle as O  # noqa: E402

H, W, s = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (170, 255, 8.0)
TW, TH, CELL = 32, 16, int(__import__("os").environ.get("CELL", 16))
c = S.gaussians(H, W, seed=1000)
R = O.rects(c, H, W, s, 0.1, support=True)
ok = (R[:, 2] <= R[:, 3]) & (R[:, 4] <= R[:, 5])
R = R[ok].astype(np.int64)
x0u, y0u, x0, x1, y0, y1 = R.T
Hs, Ws = O.out_dims(H, W, s)
ext_w = int((x1 - x0u + 1).max()); ext_h = int((y1 - y0u + 1).max())
off = ((max(ext_w, ext_h) + CELL - 1) // CELL + 1) * CELL
cx = (x0u + off) // CELL; cy = (y0u + off) // CELL
ncx = (Ws + off) // CELL + 1; ncy = (Hs + off) // CELL + 1
cell = cy * ncx + cx
cnt = np.bincount(cell, minlength=ncx * ncy).reshape(ncy, ncx)
rx = np.full(ncx * ncy, -1); np.maximum.at(rx, cell, x1); rx = rx.reshape(ncy, ncx)
ry = np.full(ncx * ncy, -1); np.maximum.at(ry, cell, y1); ry = ry.reshape(ncy, ncx)
b0 = b1 = c0 = c1 = 0
for Ty0 in range(0, Hs, TH):
    for Tx0 in range(0, Ws, TW):
        Tx1, Ty1 = min(Ws - 1, Tx0 + TW - 1), min(Hs - 1, Ty0 + TH - 1)
        clo = (Tx0 - ext_w + 1 + off) // CELL; chi = min(ncx - 1, (Tx1 + off) // CELL)
        rlo = (Ty0 - ext_h + 1 + off) // CELL; rhi = min(ncy - 1, (Ty1 + off) // CELL)
        for r in range(max(rlo, 0), rhi + 1):
            n = cnt[r, clo:chi + 1].sum()
            b0 += -(-n // 32); c0 += n
            good = np.nonzero((rx[r, clo:chi + 1] >= Tx0) & (ry[r, clo:chi + 1] >= Ty0))[0]
            if len(good):
                n = cnt[r, clo + good[0]:clo + good[-1] + 1].sum()
                b1 += -(-n // 32); c1 += n
print(f"{(H, W, s)} ext {ext_w}x{ext_h}: candidates {c0} -> {c1} ({c1 / c0:.3f}), "
      f"batches {b0} -> {b1} ({b1 / b0:.3f})")
