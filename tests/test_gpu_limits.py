"""GPU parity at the size limits of the ABI (include/gsr.h: Hs, Ws <= 65535; rect coordinates are
packed as 16-bit pairs in the kernels' records): a 4 x 65532 and a 65532 x 4 HR image (x4 of a
1 x 16383 / 16383 x 1 LR strip), checked on sampled pixels and sampled Gaussians' gradients
against the float64 oracle; and the largest output the ABI accepts is 65535 wide."""
import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from _util import KEYS, assert_bwd_close, assert_fwd_close, to_dev

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


@pytest.mark.parametrize("H,W", [(1, 16383), (16383, 1)])
def test_max_extent_strip(gsr, H, W):
    import torch
    s = 4.0
    c = S.gaussians(H, W, m=4, seed=H + 7, offset_range=1.0)
    Hs, Ws = O.out_dims(H, W, s)
    assert max(Hs, Ws) == 65532
    dev = to_dev(c)
    out = gsr.render_fwd(*dev, H, W, s).cpu().numpy()
    assert out.shape == (Hs, Ws, 3)
    rng = np.random.default_rng(1)
    px = np.concatenate([rng.integers(0, Ws, 40), [0, Ws - 1, Ws - 1]])
    py = np.concatenate([rng.integers(0, Hs, 40), [0, Hs - 1, 0]])
    assert_fwd_close(out[py, px], O.render_pixels(c, H, W, s, 0.1, px, py))
    g = S.grad_out((Hs, Ws, 3), seed=3)
    got = gsr.render_bwd(*dev, H, W, s, torch.from_numpy(g).cuda())
    n = c["alpha"].shape[0]
    idx = np.concatenate([rng.choice(n, 30, replace=False), [0, n - 1]])
    want = O.render_bwd(c, H, W, s, 0.1, g, idx=idx, want_absmass=True)
    assert_bwd_close({k: t.cpu().numpy().astype(np.float64)[idx] for k, t in zip(KEYS, got)},
                     want, want["absmass"])


def test_output_limit(gsr):
    """Ws = 65535 is accepted (1 x 3 LR at s = 21845 would be 43690 x 65535: only the size
    query), 65536 is rejected."""
    assert gsr.out_dims(1, 3, 21845.0) == (21845, 65535)
    with pytest.raises(gsr.GsrError):
        gsr.out_dims(1, 65536, 1.0)
