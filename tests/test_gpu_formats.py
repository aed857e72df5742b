"""GPU parity of the NEXT-4 data formats (include/gsr.h GSR_OUT_BF16, GSR_OUT_CHW,
GSR_PARAMS_BF16; the paper trains its HAT-L model "with Automatic Mixed Precision (AMP) in
bfloat16"). The formats change only what is read and written, so each is checked two
ways: against the float32 HWC path on the same inputs (bitwise where the arithmetic is the same,
i.e. the forward; within fp64 atomic reordering for the backward) and against the float64 oracle
with the standard gates, the oracle reading the same (bf16-rounded) values."""
import numpy as np
import pytest

import gsr_synth as S
import oracle as O
from _util import KEYS, assert_bwd_close, assert_fwd_close, grad_dict, to_dev

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


def _bf16_round(a):
    """float32 -> bfloat16 (round to nearest even) -> float32, via torch's cast."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).bfloat16().float().numpy()


def _setup(gsr, H=20, W=26, s=(4.0, 3.0), bands=None, seed=3):
    c = S.gaussians(H, W, seed=seed, offset_range=1.0)
    n = c["alpha"].shape[0]
    if bands is None:
        lay = gsr.layout([gsr.Image(H, W, s[0], 0, n, s_y=s[1])])
    else:
        lay = gsr.layout([gsr.Image(H, W, s[0], 0, n, rb, re, s_y=s[1]) for rb, re in bands])
    return c, lay


def _close(a, b, rtol=1e-6):
    """Same gradients up to the order of the fp64 atomics (a float32 ulp at most)."""
    for x, y in zip(a, b):
        x = x.double().cpu().numpy()
        y = y.double().cpu().numpy()
        assert np.allclose(x, y, rtol=rtol, atol=rtol * max(np.abs(y).max(), 1e-300))


def test_chw_output_and_grad(gsr):
    """Planar blocks: the same values as HWC, element for element, and the same gradients."""
    import torch
    c, lay = _setup(gsr)
    dev = to_dev(c)
    hwc = gsr.render_fwd_batched(*dev, lay, 0.1)
    chw = gsr.render_fwd_batched(*dev, lay, 0.1, chw=True)
    assert torch.equal(lay.view(chw, 0, chw=True), lay.view(hwc, 0).permute(2, 0, 1))
    want = O.render_fwd(c, 20, 26, (4.0, 3.0), 0.1)
    assert_fwd_close(lay.view(chw, 0, chw=True).permute(1, 2, 0).cpu().numpy(), want)
    g = torch.from_numpy(S.grad_out((lay.out_numel,), seed=4)).cuda()
    g_chw = lay.view(g, 0).permute(2, 0, 1).contiguous().reshape(-1)
    _close(gsr.render_bwd_batched(*dev, lay, g_chw, 0.1, chw=True),
           gsr.render_bwd_batched(*dev, lay, g, 0.1))


def test_chw_row_bands(gsr):
    """Planar blocks of row bands (the sharded path's unit): each band is [3, rows, Ws]; band
    moments summed over the bands and finalized give the whole image's gradients."""
    import torch
    c, _ = _setup(gsr)
    n = c["alpha"].shape[0]
    dev = to_dev(c)
    want = O.render_fwd(c, 20, 26, (4.0, 3.0), 0.1)
    g = torch.from_numpy(S.grad_out((60, 104, 3), seed=5)).cuda()
    mom = torch.zeros((n, 8), dtype=torch.float64, device="cuda")
    for rb, re in [(0, 23), (23, 41), (41, 60)]:
        lay = gsr.layout([gsr.Image(20, 26, 4.0, 0, n, rb, re, s_y=3.0)])
        chw = gsr.render_fwd_batched(*dev, lay, 0.1, chw=True)
        assert_fwd_close(lay.view(chw, 0, chw=True).permute(1, 2, 0).cpu().numpy(), want[rb:re])
        gb = g[rb:re].permute(2, 0, 1).contiguous().reshape(-1)
        gsr.render_bwd_moments_batched(*dev, lay, gb, mom, 0.1, chw=True)
    got = grad_dict(gsr.finalize_grads(*dev, mom))
    ref = O.render_bwd(c, 20, 26, (4.0, 3.0), 0.1, g.cpu().numpy(), want_absmass=True)
    assert_bwd_close(got, ref, ref["absmass"])


@pytest.mark.parametrize("chw", [False, True])
def test_bf16_output(gsr, chw):
    """GSR_OUT_BF16: the stored image is the RNE bfloat16 rounding of the float32 sums."""
    import torch
    c, lay = _setup(gsr, H=24, W=18, s=(6.0, 6.0))
    dev = to_dev(c)
    f32 = gsr.render_fwd_batched(*dev, lay, 0.1, chw=chw)
    b16 = gsr.render_fwd_batched(*dev, lay, 0.1, out_dtype=torch.bfloat16, chw=chw)
    assert b16.dtype == torch.bfloat16
    assert torch.equal(b16, f32.bfloat16())
    want = O.render_fwd(c, 24, 18, 6.0, 0.1)
    got = lay.view(b16.float(), 0, chw=chw)
    got = (got.permute(1, 2, 0) if chw else got).cpu().numpy()
    err = np.abs(got - want)
    assert (err <= 1e-5 + 2.0 ** -8 * np.abs(want)).all(), err.max()


def test_bf16_grad_out(gsr):
    """GSR_OUT_BF16 in the backward: a bfloat16 dL/dI is widened exactly, so the gradients are
    those of the float32 path fed the same values, and match the oracle fed them too."""
    import torch
    c, lay = _setup(gsr)
    dev = to_dev(c)
    g = torch.from_numpy(S.grad_out((lay.out_numel,), seed=6)).cuda().bfloat16()
    got = gsr.render_bwd_batched(*dev, lay, g, 0.1)
    _close(got, gsr.render_bwd_batched(*dev, lay, g.float(), 0.1))
    ref = O.render_bwd(c, 20, 26, (4.0, 3.0), 0.1, lay.view(g.float(), 0).cpu().numpy(),
                       want_absmass=True)
    assert_bwd_close(grad_dict(got), ref, ref["absmass"])


def test_bf16_params(gsr):
    """GSR_PARAMS_BF16: bfloat16 parameters are widened exactly where read -- the forward equals
    the float32 path on the rounded values bit for bit; gradients (float32) match too."""
    import torch
    c, lay = _setup(gsr, H=16, W=16, s=(8.0, 8.0))
    cr = {k: _bf16_round(v) for k, v in c.items()}
    d32 = to_dev(cr)
    d16 = [t.bfloat16() for t in d32]
    f16 = gsr.render_fwd_batched(*d16, lay, 0.1)
    assert torch.equal(f16, gsr.render_fwd_batched(*d32, lay, 0.1))
    assert_fwd_close(lay.view(f16, 0).cpu().numpy(), O.render_fwd(cr, 16, 16, 8.0, 0.1))
    g = torch.from_numpy(S.grad_out((lay.out_numel,), seed=7)).cuda()
    got = gsr.render_bwd_batched(*d16, lay, g, 0.1)
    assert all(t.dtype == torch.float32 for t in got)
    _close(got, gsr.render_bwd_batched(*d32, lay, g, 0.1))
    ref = O.render_bwd(cr, 16, 16, 8.0, 0.1, lay.view(g, 0).cpu().numpy(), want_absmass=True)
    assert_bwd_close(grad_dict(got), ref, ref["absmass"])
    assert gsr.pair_count(*d16, lay, 0.1, support=True) == O.pair_count(cr, 16, 16, 8.0, 0.1,
                                                                           support=True)
    mom = torch.zeros((d16[0].shape[0], 8), dtype=torch.float64, device="cuda")
    gsr.render_bwd_moments_batched(*d16, lay, g, mom, 0.1)
    _close(gsr.finalize_grads(*d16, mom), got)


def test_autograd_amp_formats(gsr):
    """The differentiable op with bfloat16 parameters, a bfloat16 planar output and a loss on
    it: the output is [3, Hs, Ws] bf16, the gradients arrive in the parameters' dtype and equal
    the float32 path's gradients on the same values, rounded to bfloat16."""
    import torch
    c, lay = _setup(gsr, H=12, W=14, s=(5.0, 3.5))
    cr = {k: _bf16_round(v) for k, v in c.items()}
    p16 = [t.bfloat16().requires_grad_(True) for t in to_dev(cr)]
    img = gsr.render(*p16, 12, 14, (5.0, 3.5), out_dtype=torch.bfloat16, chw=True)
    assert img.dtype == torch.bfloat16 and img.shape == (3, 42, 70)
    w = torch.from_numpy(S.grad_out((3, 42, 70), seed=8)).cuda().bfloat16()
    (img.float() * w.float()).sum().backward()
    p32 = to_dev(cr)
    ref = gsr.render_bwd_batched(*p32, lay, w.permute(1, 2, 0).contiguous().reshape(-1).float(),
                                 0.1)
    for p, r, k in zip(p16, ref, KEYS):
        assert p.grad.dtype == torch.bfloat16, k
        r = r.double()
        err = (p.grad.double() - r).abs()
        assert (err <= 2.0 ** -8 * r.abs() + 1e-6 * r.abs().max()).all(), k
