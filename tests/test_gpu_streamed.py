"""GPU: the host-memory streamed step (ops.StreamedFwdBwd: image groups with H2D / compute / D2H
overlapped on three streams) gives the same image and gradients as the device-resident batched
calls, and both match the oracle on a sampled image."""
import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from _util import assert_fwd_close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("groups,sizes", [(3, [1, 2, 2]), (4, [1, 1, 2, 1])],
                         ids=["even", "ramped"])
def test_streamed_matches_batched(groups, sizes):
    import torch
    import paper_2501_06838_b200 as gsr
    imgs = [(20, 24, 3.0), (17, 13, 2.5), (24, 24, 4.0), (9, 30, 1.7), (16, 16, 8.0)]
    clouds = [S.gaussians(H, W, m=4, seed=50 + k) for k, (H, W, s) in enumerate(imgs)]
    keys = ("alpha", "mu", "sigma", "rho", "color")
    host = {k: np.concatenate([c[k] for c in clouds]) for k in keys}
    ims, off = [], 0
    for (H, W, s), c in zip(imgs, clouds):
        ims.append(gsr.Image(H, W, s, off, c["alpha"].shape[0]))
        off += c["alpha"].shape[0]
    lay = gsr.layout(ims)
    g = np.random.default_rng(3).uniform(-1, 1, lay.out_numel).astype(np.float32)
    dev = [torch.from_numpy(host[k]).cuda() for k in keys]
    ref_out = gsr.render_fwd_batched(*dev, lay).cpu().numpy()
    ref_grads = [t.cpu().numpy() for t in gsr.render_bwd_batched(*dev, lay, torch.from_numpy(g).cuda())]

    hp = [torch.from_numpy(host[k]).pin_memory() for k in keys]
    hg = torch.from_numpy(g).pin_memory()
    h_out = torch.empty(lay.out_numel, dtype=torch.float32).pin_memory()
    h_grads = [torch.empty_like(t).pin_memory() for t in hp]
    step = gsr.StreamedFwdBwd(lay, 0.1, groups=groups)
    # >= 4 groups: the first and the last hold one image each (ramp)
    assert [len(sub.images) for *_, sub in step.groups] == sizes
    for _ in range(2):                      # reuse of the cached buffers
        step(hp, hg, h_out, h_grads)
        torch.cuda.synchronize()
        np.testing.assert_allclose(h_out.numpy(), ref_out, rtol=1e-5, atol=1e-6)
        for a, b in zip(h_grads, ref_grads):
            scale = np.abs(b).max() + 1e-30
            assert np.abs(a.numpy() - b).max() <= 1e-4 * scale
    # image 2 against the oracle
    k = 2
    H, W, s = imgs[k]
    got = lay.view(torch.from_numpy(h_out.numpy()), k).numpy()
    assert_fwd_close(got, O.render_fwd(clouds[k], H, W, s, 0.1))
