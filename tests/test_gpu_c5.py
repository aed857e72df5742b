"""GPU parity at BASELINE.json's full C5 size, in the launch configuration bench.py times: 64
DIV2K-size images (255x170 LR at x8 -> 2040x1360) in one batched call with a private
workspace, the forward's binning reused by the backward moments (GSR_REUSE_BINNING), then the
finalize -- checked on sampled outputs the float64 oracle computes one by one: pixels of three
images (random + corners), and the gradients of sampled Gaussians (oracle idx mode)."""
import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from _util import KEYS, assert_bwd_close, assert_fwd_close

pytestmark = pytest.mark.gpu


def test_c5_full_size_sampled():
    import torch
    import paper_2501_06838_b200 as gsr
    from paper_2501_06838_b200 import ops
    imgs = S.CONFIGS["C5"]["images"]
    assert len(imgs) == 64
    clouds = [S.gaussians(H, W, seed=1000 + k) for k, (H, W, s) in enumerate(imgs)]
    counts = [c["alpha"].shape[0] for c in clouds]
    offs = np.concatenate([[0], np.cumsum(counts)])
    dev = [torch.from_numpy(np.concatenate([c[k] for c in clouds])).cuda() for k in KEYS]
    lay = gsr.layout([gsr.Image(H, W, s, int(offs[k]), counts[k])
                      for k, (H, W, s) in enumerate(imgs)])
    g = torch.empty(lay.out_numel, dtype=torch.float32, device="cuda")
    g.uniform_(-1.0, 1.0, generator=torch.Generator(device="cuda").manual_seed(2000))
    ws = ops.workspace_for(dev[0], lay, 0.1)
    out = gsr.render_fwd_batched(*dev, lay, 0.1, workspace=ws)
    mom = torch.zeros((dev[0].shape[0], 8), dtype=torch.float64, device="cuda")
    gsr.render_bwd_moments_batched(*dev, lay, g, mom, 0.1, workspace=ws, reuse_binning=True)
    grads = dict(zip(KEYS, gsr.finalize_grads(*dev, mom)))
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    H, W, s = imgs[0]
    Hs, Ws = O.out_dims(H, W, s)
    for k in (0, 31, 63):
        img = lay.view(out, k).cpu().numpy()
        px = np.concatenate([rng.integers(0, Ws, 24), [0, Ws - 1, 0, Ws - 1]])
        py = np.concatenate([rng.integers(0, Hs, 24), [0, 0, Hs - 1, Hs - 1]])
        assert_fwd_close(img[py, px], O.render_pixels(clouds[k], H, W, s, 0.1, px, py))
    for k in (0, 63):
        gk = lay.view(g, k).cpu().numpy()
        idx = np.concatenate([rng.choice(counts[k], 14, replace=False), [0, counts[k] - 1]])
        want = O.render_bwd(clouds[k], H, W, s, 0.1, gk, idx=idx, want_absmass=True)
        sel = torch.from_numpy(offs[k] + idx).cuda()
        got = {kk: grads[kk][sel].cpu().numpy().astype(np.float64) for kk in KEYS}
        assert_bwd_close(got, want, want["absmass"])
