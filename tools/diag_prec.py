"""Backward precision diagnostics: err/S distribution vs scale (exact vs inexact 1/s)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np, torch
import gsr_synth as S, oracle as O, paper_2501_06838_b200 as gsr
from _util import to_dev, grad_dict, flat9
for s in [4.0, 2.91088506, 3.0, 2.0, 1.80936014]:
    H = W = 48
    c = S.gaussians(H, W, seed=1002)
    Hs, Ws = O.out_dims(H, W, s)
    g = S.grad_out((Hs, Ws, 3), seed=2002)
    got = flat9(grad_dict(gsr.render_bwd(*to_dev(c), H, W, s, torch.from_numpy(g).cuda())))
    ref = O.render_bwd(c, H, W, s, 0.1, g, want_absmass=True)
    w = flat9(ref); A = ref["absmass"]
    rs = np.abs(got - w) / np.maximum(A, 1e-300)
    print(f"s={s:.4f} err/S per column max:", " ".join(f"{x:.1e}" for x in rs.max(0)),
          " p99.99 %.2e" % np.quantile(rs, 0.9999), flush=True)
