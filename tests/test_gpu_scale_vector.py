"""GPU parity of the scale-vector variant (reading R22, "an
upsampling scale vector"): images rendered with (s_x, s_y), s_x != s_y, through the C-ABI vs the
float64 oracle on the same seeded inputs, with the gates of test_gpu_parity.py (forward max-abs
<= 1e-5, backward 1e-4 relative to max(|g|, 0.1 S))."""
import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from _util import KEYS, assert_bwd_close, assert_fwd_close, cat, grad_dict, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gsr():
    import torch
    import paper_2501_06838_b200 as g
    from paper_2501_06838_b200.build import build
    assert torch.cuda.is_available()
    build()
    g.load()
    return g


# (H, W, (s_x, s_y), r, dist): ragged, narrow (small-tile forward) and wide windows (recurrence
# path: a1/s_x <= 1), strongly anisotropic, s_y = 1, the stress distribution
CASES = [(7, 9, (2.5, 1.0), 0.1, "image"), (13, 11, (1.5, 3.7), 0.3, "image"),
         (20, 16, (4.0, 2.0), 0.1, "image"), (9, 13, (12.0, 30.0), 0.1, "image"),
         (12, 10, (8.0, 3.0), 0.5, "image"), (10, 12, (3.0, 5.5), 0.4, "stress"),
         (16, 24, (6.0, 6.5), 0.1, "image")]


@pytest.mark.parametrize("H,W,sv,r,dist", CASES)
def test_scale_vector_fwd_bwd(gsr, H, W, sv, r, dist):
    import torch
    c = S.gaussians(H, W, seed=int(10 * sv[0] + sv[1]) + H, dist=dist, offset_range=1.0)
    dev = to_dev(c)
    out = gsr.render_fwd(*dev, H, W, sv, ratio=r)
    torch.cuda.synchronize()
    want = O.render_fwd(c, H, W, sv, r)
    assert out.shape == want.shape == (int(np.floor(sv[1] * H)), int(np.floor(sv[0] * W)), 3)
    assert_fwd_close(out.cpu().numpy(), want, dist)
    g = S.grad_out(want.shape, seed=H + W)
    got = grad_dict(gsr.render_bwd(*dev, H, W, sv, torch.from_numpy(g).cuda(), ratio=r))
    ref = O.render_bwd(c, H, W, sv, r, g, want_absmass=True)
    assert_bwd_close(got, ref, ref["absmass"], dist=dist)


def test_scale_vector_pair_counts(gsr):
    """The GPU's window and support rects with s_x != s_y select the oracle's pair sets."""
    H, W, sv = 17, 23, (3.5, 2.25)
    c = S.gaussians(H, W, seed=5, offset_range=1.5)
    lay = gsr.layout([gsr.Image(H, W, sv[0], 0, c["alpha"].shape[0], s_y=sv[1])])
    dev = to_dev(c)
    assert gsr.pair_count(*dev, lay, 0.1) == O.pair_count(c, H, W, sv, 0.1)
    assert gsr.pair_count(*dev, lay, 0.1, support=True) == O.pair_count(c, H, W, sv, 0.1,
                                                                           support=True)


def test_scale_vector_ragged_batch_with_bands(gsr):
    """One batched call mixing isotropic and anisotropic images, whole images and row bands."""
    import torch
    spec = [(48, 48, (4.0, 2.0), 0, -1), (30, 20, (2.5, 2.5), 0, -1), (16, 40, (1.0, 6.0), 17, 70),
            (24, 24, (8.0, 3.0), 0, 40)]
    clouds = [S.gaussians(H, W, seed=300 + k) for k, (H, W, _, _, _) in enumerate(spec)]
    allc = cat(clouds)
    ims, off = [], 0
    for (H, W, sv, rb, re), cl in zip(spec, clouds):
        n = cl["alpha"].shape[0]
        ims.append(gsr.Image(H, W, sv[0], off, n, rb, re, s_y=None if sv[0] == sv[1] else sv[1]))
        off += n
    lay = gsr.layout(ims)
    dev = to_dev(allc)
    out = gsr.render_fwd_batched(*dev, lay, 0.1)
    g = torch.from_numpy(S.grad_out((lay.out_numel,), seed=9)).cuda()
    grads = grad_dict(gsr.render_bwd_batched(*dev, lay, g, 0.1))
    torch.cuda.synchronize()
    off = 0
    for k, ((H, W, sv, _, _), cl) in enumerate(zip(spec, clouds)):
        rows = lay.rows[k]
        want = O.render_fwd(cl, H, W, sv, 0.1, rows=rows)
        assert_fwd_close(lay.view(out, k).cpu().numpy(), want)
        gk = lay.view(g, k).cpu().numpy()
        wb = O.render_bwd(cl, H, W, sv, 0.1, gk, rows=rows, want_absmass=True)
        n = cl["alpha"].shape[0]
        assert_bwd_close({kk: grads[kk][off:off + n] for kk in KEYS}, wb, wb["absmass"])
        off += n
