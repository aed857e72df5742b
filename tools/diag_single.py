"""Single-Gaussian precision diagnostics: per-pixel relative error of the GPU forward and the
bwd err/S, vs the oracle, for a sweep of sigma / rho / s."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np, torch
import oracle as O, paper_2501_06838_b200 as gsr
from _util import to_dev, grad_dict, flat9
rng = np.random.default_rng(0)
for s in [1.0, 1.81, 2.0, 4.0]:
    for sig in [0.08, 0.2, 0.6]:
        for rho in [0.0, 0.6, -0.95]:
            H = W = 16
            n = 9
            c = dict(alpha=np.full(n, 0.7, np.float32),
                     mu=(np.stack([rng.uniform(4, 12, n), rng.uniform(4, 12, n)], 1)).astype(np.float32),
                     sigma=np.full((n, 2), sig, np.float32) * np.float32([1.0, 1.3]),
                     rho=np.full(n, rho, np.float32), color=np.full((n, 3), 0.5, np.float32))
            got = gsr.render_fwd(*to_dev(c), H, W, s, ratio=1.0).cpu().numpy().astype(np.float64)
            ref = O.render_fwd(c, H, W, s, 1.0)
            m = ref > 1e-6 * ref.max()
            rel = np.abs(got - ref)[m] / ref[m]
            Hs, Ws = ref.shape[:2]
            g = rng.uniform(-1, 1, (Hs, Ws, 3)).astype(np.float32)
            gg = flat9(grad_dict(gsr.render_bwd(*to_dev(c), H, W, s, torch.from_numpy(g).cuda(), ratio=1.0)))
            rb = O.render_bwd(c, H, W, s, 1.0, g, want_absmass=True)
            es = (np.abs(gg - flat9(rb)) / rb["absmass"]).max(0)
            print(f"s={s:<5} sig={sig:<5} rho={rho:<6} fwd rel max {rel.max():.2e} p99 {np.quantile(rel, .99):.2e} "
                  f"| bwd err/S max per col " + " ".join(f"{x:.1e}" for x in es), flush=True)
