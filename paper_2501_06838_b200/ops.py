"""PyTorch binding over the C-ABI (include/gsr.h): argument marshalling only.

Every step of the rasterization runs in libgsr.so's sm_100a kernels; PyTorch provides device
memory (caching allocator), the current CUDA stream and autograd plumbing. There is no CPU or
PyTorch fallback: CPU tensors, a missing library or a launch failure raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import torch

from . import _lib
from ._lib import check

PARAMS = ("alpha", "mu", "sigma", "rho", "color")
WIDTH = {"alpha": 1, "mu": 2, "sigma": 2, "rho": 1, "color": 3}


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _check_param(t: torch.Tensor, name: str, n: Optional[int] = None,
                 dtypes=(torch.float32,)) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype not in dtypes:
        raise TypeError(f"{name} must be one of {dtypes}, got {t.dtype}")
    t = t.contiguous()
    w = WIDTH.get(name, None)
    if w is not None:
        if (w == 1 and t.dim() != 1) or (w > 1 and (t.dim() != 2 or t.shape[1] != w)):
            raise ValueError(f"{name} must have shape [n]" + ("" if w == 1 else f"x{w}"))
        if n is not None and t.shape[0] != n:
            raise ValueError(f"{name} has {t.shape[0]} rows, expected {n}")
    return t


_FLOATS = (torch.float32, torch.bfloat16)


# GSR_DEBUG=1: every render call first runs gsr_validate_params on its parameters
# and raises on a Gaussian outside the domain (synchronises; a debugging aid, off by default)
DEBUG = os.environ.get("GSR_DEBUG", "0") not in ("", "0")


def _params(alpha, mu, sigma, rho, color, validate: bool = True):
    """Checked parameter tensors: float32, or all bfloat16 (GSR_PARAMS_BF16, NEXT-4)."""
    n = alpha.shape[0] if isinstance(alpha, torch.Tensor) else None
    ts = [_check_param(t, k, n, _FLOATS) for t, k in zip((alpha, mu, sigma, rho, color), PARAMS)]
    dev = ts[0].device
    for t in ts:
        if t.device != dev:
            raise ValueError("all parameters must live on the same device")
        if t.dtype != ts[0].dtype:
            raise TypeError("all parameters must have the same dtype")
    if DEBUG and validate and n:
        cnt, first = _validate(ts, n)
        if cnt:
            raise ValueError(f"GSR_DEBUG: {cnt} Gaussian(s) outside the parameter domain "
                             f"(non-finite, sigma <= 0 or |rho| >= 1), first index {first}")
    return ts, n


def _fmt_flags(params, image: Optional[torch.Tensor] = None, out_dtype=None,
               chw: bool = False) -> int:
    """GSR_* data-format flags (include/gsr.h, NEXT-4) of a call."""
    f = _lib.GSR_PARAMS_BF16 if params[0].dtype == torch.bfloat16 else 0
    dt = out_dtype if out_dtype is not None else (image.dtype if image is not None else None)
    if dt == torch.bfloat16:
        f |= _lib.GSR_OUT_BF16
    elif dt is not None and dt != torch.float32:
        raise TypeError(f"image dtype must be float32 or bfloat16, got {dt}")
    if chw:
        f |= _lib.GSR_OUT_CHW
    return f


def _check_image(t: torch.Tensor, name: str, lay: "Layout", device,
                 dtypes=(torch.float32, torch.bfloat16)) -> torch.Tensor:
    """An image buffer of a layout (out, grad_out, gt): lay.out_numel elements of an accepted dtype
    on the parameters' device, contiguous (the kernels index it by raw element offsets)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype not in dtypes:
        raise TypeError(f"{name} must be one of {dtypes}, got {t.dtype}")
    if t.device != torch.device(device):
        raise ValueError(f"{name} is on {t.device}, the parameters on {device}")
    if t.numel() != lay.out_numel:
        raise ValueError(f"{name} has {t.numel()} elements, the layout needs {lay.out_numel}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _ptr(t: torch.Tensor, offset_elems: int = 0) -> int:
    return t.data_ptr() + offset_elems * t.element_size()


@dataclass
class Image:
    """One image of a batch: LR size (H, W), scale s, its Gaussians [g_off, g_off+g_cnt) and the
    HR row band [row_begin, row_end) (row_end = -1: all Hs rows). s_y (> 0) makes the scale a
    vector (s_x, s_y) = (s, s_y) (reading R22); None: isotropic s."""
    H: int
    W: int
    s: float
    g_off: int
    g_cnt: int
    row_begin: int = 0
    row_end: int = -1
    s_y: Optional[float] = None


@dataclass
class Layout:
    images: List[Image]
    dims: List[Tuple[int, int]]          # (Hs, Ws)
    rows: List[Tuple[int, int]]          # resolved band per image
    out_off: List[int]                   # float offsets into the flat output
    out_numel: int

    def view(self, flat: torch.Tensor, k: int, chw: bool = False) -> torch.Tensor:
        """Image k's block of a flat output: [rows, Ws, 3] (HWC) or [3, rows, Ws] (chw)."""
        rb, re = self.rows[k]
        Ws = self.dims[k][1]
        o = self.out_off[k]
        blk = flat[o:o + (re - rb) * Ws * 3]
        return blk.view(3, re - rb, Ws) if chw else blk.view(re - rb, Ws, 3)


def layout(images: Sequence[Image]) -> Layout:
    dims, rows, offs = [], [], []
    off = 0
    for im in images:
        Hs, Ws = _lib.out_dims(im.H, im.W, im.s, im.s_y)
        rb = im.row_begin
        re = Hs if im.row_end is None or im.row_end < 0 else im.row_end
        dims.append((Hs, Ws))
        rows.append((rb, re))
        offs.append(off)
        off += (re - rb) * Ws * 3
    return Layout(list(images), dims, rows, offs, off)


def _chunks(lay: Layout):
    """Split a batch into ABI calls of <= GSR_MAX_IMAGES images; each call sees its own
    contiguous Gaussian range and output range (pointer offsets, g_off/out_off rebased)."""
    ims = lay.images
    for c0 in range(0, len(ims), _lib.MAX_IMAGES):
        sel = list(range(c0, min(c0 + _lib.MAX_IMAGES, len(ims))))
        g0 = min(ims[k].g_off for k in sel)
        g1 = max(ims[k].g_off + ims[k].g_cnt for k in sel)
        o0 = lay.out_off[sel[0]]
        recs = []
        for k in sel:
            im = ims[k]
            rb, re = lay.rows[k]
            recs.append((im.H, im.W, im.s, im.g_off - g0, im.g_cnt, lay.out_off[k] - o0, rb, re,
                         im.s_y))
        yield g0, g1, o0, _lib.images_array(recs), len(sel)


class Workspace:
    """Grow-only device workspace from the caching allocator (the library allocates nothing)."""

    def __init__(self):
        self.buf: Optional[torch.Tensor] = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


_WS = {}


def _workspace(device, nbytes: int) -> torch.Tensor:
    """The implicit workspace of calls made without one: one per (device, stream), so calls on
    different streams never share scratch (gsr.h: concurrent calls need distinct workspaces). It
    is allocated on, and only ever used by, its own stream, so the caching allocator's stream
    ordering makes a regrown buffer safe to free."""
    dev = torch.device(device)
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    ws = _WS.setdefault(key, Workspace())
    return ws.get(nbytes, device)


def _ws_bytes(arr, n_imgs, n_total, ratio) -> int:
    b = _lib.load().gsr_workspace_bytes_batched(arr, n_imgs, n_total, float(ratio))
    if b == 0:
        raise _lib.GsrError("gsr_workspace_bytes_batched: invalid arguments")
    return b


def single_chunk(lay: Layout) -> bool:
    return len(lay.images) <= _lib.MAX_IMAGES


def workspace_for(alpha, lay: Layout, ratio: float = 0.1) -> torch.Tensor:
    """A private workspace for a single-chunk layout (lets a backward reuse the forward's
    binning: GSR_REUSE_BINNING)."""
    g0, g1, o0, arr, m = next(_chunks(lay))
    return torch.empty(_ws_bytes(arr, m, g1 - g0, ratio), dtype=torch.uint8, device=alpha.device)


def _ws_for(dev, nb, workspace):
    if workspace is not None:
        if workspace.numel() < nb:
            raise ValueError("workspace too small")
        return workspace
    return _workspace(dev, nb)


def render_fwd_batched(alpha, mu, sigma, rho, color, lay: Layout, ratio: float = 0.1,
                       out: Optional[torch.Tensor] = None,
                       workspace: Optional[torch.Tensor] = None,
                       out_dtype: Optional[torch.dtype] = None, chw: bool = False) -> torch.Tensor:
    """Forward render of every image of `lay` into one flat buffer: float32 HWC blocks by
    default; out_dtype=torch.bfloat16 and/or chw=True select the NEXT-4 formats (GSR_OUT_BF16,
    GSR_OUT_CHW); bfloat16 parameters are read as such (GSR_PARAMS_BF16)."""
    params, n = _params(alpha, mu, sigma, rho, color)
    alpha, mu, sigma, rho, color = params
    dev = alpha.device
    if out is None:
        out = torch.empty(lay.out_numel, dtype=out_dtype or torch.float32, device=dev)
    out = _check_image(out, "out", lay, dev)
    flags = _fmt_flags(params, out, chw=chw)
    lib = _lib.load()
    st = _stream_ptr(dev)
    for g0, g1, o0, arr, m in _chunks(lay):
        nb = _ws_bytes(arr, m, g1 - g0, ratio)
        ws = _ws_for(dev, nb, workspace)
        check(lib.gsr_render_fwd_batched_ex(_ptr(alpha, g0), _ptr(mu, 2 * g0),
                                            _ptr(sigma, 2 * g0), _ptr(rho, g0),
                                            _ptr(color, 3 * g0), g1 - g0, arr, m, float(ratio),
                                            _ptr(out, o0), ws.data_ptr(), ws.numel(), flags, st),
              "gsr_render_fwd_batched_ex")
    return out


def render_bwd_moments_batched(alpha, mu, sigma, rho, color, lay: Layout, grad_out: torch.Tensor,
                               moments: torch.Tensor, ratio: float = 0.1,
                               workspace: Optional[torch.Tensor] = None,
                               reuse_binning: bool = False, chw: bool = False) -> torch.Tensor:
    """Accumulate (+=) the backward moments [n, 8] (float64) of every image band of `lay`.
    reuse_binning: `workspace` holds this layout's binning from the preceding forward.
    grad_out float32 or bfloat16, HWC or (chw=True) planar blocks."""
    params, n = _params(alpha, mu, sigma, rho, color)
    alpha, mu, sigma, rho, color = params
    dev = alpha.device
    grad_out = _check_image(grad_out.contiguous(), "grad_out", lay, dev)
    if (moments.dtype != torch.float64 or not moments.is_contiguous() or moments.numel() != 8 * n
            or moments.device != dev):
        raise ValueError("moments must be a contiguous float64 [n, 8] tensor on the params' device")
    lib = _lib.load()
    st = _stream_ptr(dev)
    flags = _lib.GSR_REUSE_BINNING if (reuse_binning and workspace is not None and
                                       single_chunk(lay)) else 0
    flags |= _fmt_flags(params, grad_out, chw=chw)
    for g0, g1, o0, arr, m in _chunks(lay):
        nb = _ws_bytes(arr, m, g1 - g0, ratio)
        ws = _ws_for(dev, nb, workspace)
        check(lib.gsr_render_bwd_moments_batched_ex(
            _ptr(alpha, g0), _ptr(mu, 2 * g0), _ptr(sigma, 2 * g0), _ptr(rho, g0),
            _ptr(color, 3 * g0), g1 - g0, arr, m, float(ratio), _ptr(grad_out, o0),
            _ptr(moments, 8 * g0), ws.data_ptr(), ws.numel(), flags, st),
            "gsr_render_bwd_moments_batched_ex")
    return moments


def finalize_grads(alpha, mu, sigma, rho, color, moments: torch.Tensor):
    """Moments [n, 8] (float64) -> (d_alpha, d_mu, d_sigma, d_rho, d_color) (float32)."""
    params, n = _params(alpha, mu, sigma, rho, color)
    dev = params[0].device
    if (moments.dtype != torch.float64 or not moments.is_contiguous() or moments.numel() != 8 * n
            or moments.device != dev):
        raise ValueError("moments must be a contiguous float64 [n, 8] tensor on the params' device")
    grads = [torch.empty(t.shape, dtype=torch.float32, device=dev) for t in params]
    check(_lib.load().gsr_finalize_grads_ex(*[_ptr(t) for t in params], n, _ptr(moments),
                                            *[_ptr(g) for g in grads], _fmt_flags(params),
                                            _stream_ptr(dev)), "gsr_finalize_grads_ex")
    return tuple(grads)


def render_bwd_batched(alpha, mu, sigma, rho, color, lay: Layout, grad_out: torch.Tensor,
                       ratio: float = 0.1, workspace: Optional[torch.Tensor] = None,
                       reuse_binning: bool = False, chw: bool = False):
    """Gradients of sum(grad_out * I) wrt every parameter (float32, input layouts).
    reuse_binning: `workspace` holds this layout's binning from the preceding forward.
    grad_out float32 or bfloat16, HWC or (chw=True) planar blocks."""
    params, n = _params(alpha, mu, sigma, rho, color)
    alpha, mu, sigma, rho, color = params
    dev = alpha.device
    grad_out = _check_image(grad_out.contiguous(), "grad_out", lay, dev)
    grads = [torch.zeros(t.shape, dtype=torch.float32, device=dev) for t in params]
    lib = _lib.load()
    st = _stream_ptr(dev)
    flags = _lib.GSR_REUSE_BINNING if (reuse_binning and workspace is not None and
                                       single_chunk(lay)) else 0
    flags |= _fmt_flags(params, grad_out, chw=chw)
    for g0, g1, o0, arr, m in _chunks(lay):
        nb = _ws_bytes(arr, m, g1 - g0, ratio)
        ws = _ws_for(dev, nb, workspace)
        ga, gm, gs, gr, gc = grads
        check(lib.gsr_render_bwd_batched_ex(
            _ptr(alpha, g0), _ptr(mu, 2 * g0), _ptr(sigma, 2 * g0), _ptr(rho, g0),
            _ptr(color, 3 * g0), g1 - g0, arr, m, float(ratio), _ptr(grad_out, o0),
            _ptr(ga, g0), _ptr(gm, 2 * g0), _ptr(gs, 2 * g0), _ptr(gr, g0), _ptr(gc, 3 * g0),
            ws.data_ptr(), ws.numel(), flags, st), "gsr_render_bwd_batched_ex")
    return tuple(grads)


def validate_params(alpha, mu, sigma, rho, color):
    """(count, first index or -1) of the Gaussians outside the parameter domain (R20:
    non-finite field, sigma <= 0 or |rho| >= 1) -- gsr_validate_params; synchronises."""
    params, n = _params(alpha, mu, sigma, rho, color, validate=False)
    return _validate(params, n)


def _validate(params, n):
    dev = params[0].device
    res = torch.empty(2, dtype=torch.int64, device=dev)
    check(_lib.load().gsr_validate_params(*[_ptr(t) for t in params], n, _fmt_flags(params),
                                          _ptr(res), _stream_ptr(dev)), "gsr_validate_params")
    cnt, first = (int(v) for v in res.cpu())
    return cnt, (first if cnt else -1)


# ------------------------------------------------------------------ subset mode (a rank's halo)
def _check_idx(idx: torch.Tensor, n: int, dev) -> torch.Tensor:
    if not isinstance(idx, torch.Tensor) or idx.dtype != torch.int32 or idx.dim() != 1:
        raise TypeError("idx must be a 1-D int32 tensor (ascending Gaussian indices)")
    if idx.device != torch.device(dev) or not idx.is_contiguous():
        raise ValueError("idx must be contiguous on the parameters' device")
    if idx.numel() > n:
        raise ValueError("idx has more entries than Gaussians")
    return idx


def _single_chunk_call(lay: Layout):
    if not single_chunk(lay):
        raise ValueError(f"subset calls take at most {_lib.MAX_IMAGES} images")
    return next(_chunks(lay))


def subset_workspace_for(alpha, lay: Layout, m: int, ratio: float = 0.1) -> torch.Tensor:
    """A private workspace for the subset calls of one layout and halo size m."""
    g0, g1, o0, arr, k = _single_chunk_call(lay)
    if g0 != 0:
        raise ValueError("subset calls need layouts whose Gaussian ranges start at 0")
    nb = _lib.load().gsr_workspace_bytes_subset(arr, k, int(alpha.shape[0]), int(m), float(ratio))
    if nb == 0:
        raise _lib.GsrError("gsr_workspace_bytes_subset: invalid arguments")
    return torch.empty(nb, dtype=torch.uint8, device=alpha.device)


def render_fwd_subset(alpha, mu, sigma, rho, color, idx: torch.Tensor, lay: Layout,
                      ratio: float = 0.1, out: Optional[torch.Tensor] = None,
                      workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Forward render of the layout's bands from the Gaussians idx only (a rank's halo:
    gsr_render_fwd_subset); float32 HWC blocks."""
    params, n = _params(alpha, mu, sigma, rho, color)
    dev = params[0].device
    idx = _check_idx(idx, n, dev)
    g0, g1, o0, arr, k = _single_chunk_call(lay)
    if out is None:
        out = torch.empty(lay.out_numel, dtype=torch.float32, device=dev)
    out = _check_image(out, "out", lay, dev)
    ws = workspace if workspace is not None else subset_workspace_for(params[0], lay, idx.numel(),
                                                                      ratio)
    check(_lib.load().gsr_render_fwd_subset(*[_ptr(t) for t in params], n, _ptr(idx), idx.numel(),
                                            arr, k, float(ratio), _ptr(out), ws.data_ptr(),
                                            ws.numel(), _fmt_flags(params, out),
                                            _stream_ptr(dev)), "gsr_render_fwd_subset")
    return out


def render_bwd_moments_subset(alpha, mu, sigma, rho, color, idx: torch.Tensor, lay: Layout,
                              grad_out: torch.Tensor, moments: torch.Tensor, ratio: float = 0.1,
                              workspace: Optional[torch.Tensor] = None,
                              reuse_binning: bool = False) -> torch.Tensor:
    """Accumulate (+=) the compact moments [m, 8] (float64; row t = Gaussian idx[t]) of the
    layout's bands (gsr_render_bwd_moments_subset)."""
    params, n = _params(alpha, mu, sigma, rho, color)
    dev = params[0].device
    idx = _check_idx(idx, n, dev)
    m = idx.numel()
    g0, g1, o0, arr, k = _single_chunk_call(lay)
    grad_out = _check_image(grad_out.contiguous(), "grad_out", lay, dev)
    if (moments.dtype != torch.float64 or not moments.is_contiguous() or moments.numel() != 8 * m
            or moments.device != dev):
        raise ValueError("moments must be a contiguous float64 [m, 8] tensor on the device")
    flags = _lib.GSR_REUSE_BINNING if (reuse_binning and workspace is not None) else 0
    ws = workspace if workspace is not None else subset_workspace_for(params[0], lay, m, ratio)
    check(_lib.load().gsr_render_bwd_moments_subset(
        *[_ptr(t) for t in params], n, _ptr(idx), m, arr, k, float(ratio), _ptr(grad_out),
        _ptr(moments), ws.data_ptr(), ws.numel(), flags | _fmt_flags(params, grad_out),
        _stream_ptr(dev)), "gsr_render_bwd_moments_subset")
    return moments


def finalize_grads_subset(alpha, mu, sigma, rho, color, idx: torch.Tensor,
                          moments: torch.Tensor):
    """Compact moments [m, 8] -> compact gradients (d_alpha[m], d_mu[m,2], d_sigma[m,2],
    d_rho[m], d_color[m,3]) of the Gaussians idx (gsr_finalize_grads_subset)."""
    params, n = _params(alpha, mu, sigma, rho, color)
    dev = params[0].device
    idx = _check_idx(idx, n, dev)
    m = idx.numel()
    if (moments.dtype != torch.float64 or not moments.is_contiguous() or moments.numel() != 8 * m
            or moments.device != dev):
        raise ValueError("moments must be a contiguous float64 [m, 8] tensor on the device")
    grads = [torch.empty((m,) + tuple(t.shape[1:]), dtype=torch.float32, device=dev)
             for t in params]
    check(_lib.load().gsr_finalize_grads_subset(*[_ptr(t) for t in params], n, _ptr(idx), m,
                                                _ptr(moments), *[_ptr(g) for g in grads],
                                                _fmt_flags(params), _stream_ptr(dev)),
          "gsr_finalize_grads_subset")
    return tuple(grads)


def pair_count(alpha, mu, sigma, rho, color, lay: Layout, ratio: float = 0.1,
               support: bool = False) -> int:
    """P = number of (Gaussian, pixel) pairs inside the windows (synchronises). support=True:
    the pairs inside the support rects, i.e. the pairs the kernels evaluate (reading R21)."""
    params, n = _params(alpha, mu, sigma, rho, color)
    alpha, mu, sigma, rho, color = params
    dev = alpha.device
    lib = _lib.load()
    st = _stream_ptr(dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    tmp = torch.zeros(1, dtype=torch.int64, device=dev)
    for g0, g1, o0, arr, m in _chunks(lay):
        nb = _ws_bytes(arr, m, g1 - g0, ratio)
        ws = _workspace(dev, nb)
        check(lib.gsr_pair_count_batched_ex(_ptr(alpha, g0), _ptr(mu, 2 * g0),
                                            _ptr(sigma, 2 * g0), _ptr(rho, g0),
                                            _ptr(color, 3 * g0), g1 - g0, arr, m, float(ratio),
                                            (_lib.GSR_SUPPORT if support else 0) |
                                            _fmt_flags(params), tmp.data_ptr(),
                                            ws.data_ptr(), ws.numel(), st),
              "gsr_pair_count_batched_ex")
        total += tmp
    return int(total.item())


# ------------------------------------------------------------------ single image + autograd
def _scale(s):
    """A scale argument: a number s (the paper's scalar) or a scale vector (s_x, s_y) (R22)
    -> (s_x, s_y or None)."""
    if isinstance(s, (tuple, list)):
        return float(s[0]), float(s[1])
    return float(s), None


def _single(n, H, W, s):
    sx, sy = _scale(s)
    return layout([Image(int(H), int(W), sx, 0, int(n), s_y=sy)])


def render_fwd(alpha, mu, sigma, rho, color, H: int, W: int, scale: float,
               ratio: float = 0.1) -> torch.Tensor:
    lay = _single(alpha.shape[0], H, W, scale)
    return lay.view(render_fwd_batched(alpha, mu, sigma, rho, color, lay, ratio), 0)


def render_bwd(alpha, mu, sigma, rho, color, H: int, W: int, scale: float,
               grad_out: torch.Tensor, ratio: float = 0.1):
    lay = _single(alpha.shape[0], H, W, scale)
    return render_bwd_batched(alpha, mu, sigma, rho, color, lay, grad_out.reshape(-1), ratio)


class _RenderFn(torch.autograd.Function):
    """Forward keeps its private workspace so the backward reuses the forward's binning
    (GSR_REUSE_BINNING) -- valid because autograd saves the very same parameter tensors."""

    @staticmethod
    def forward(ctx, alpha, mu, sigma, rho, color, lay, ratio, out_dtype=None, chw=False):
        ctx.lay, ctx.ratio, ctx.chw = lay, ratio, chw
        ctx.save_for_backward(alpha, mu, sigma, rho, color)
        ws = workspace_for(alpha, lay, ratio) if single_chunk(lay) else None
        ctx.ws = ws
        return render_fwd_batched(alpha.detach(), mu.detach(), sigma.detach(), rho.detach(),
                                  color.detach(), lay, ratio, workspace=ws, out_dtype=out_dtype,
                                  chw=chw)

    @staticmethod
    def backward(ctx, g):
        alpha, mu, sigma, rho, color = ctx.saved_tensors
        # float32 gradients; autograd casts them to the dtype of bfloat16 inputs
        grads = render_bwd_batched(alpha, mu, sigma, rho, color, ctx.lay, g.contiguous(),
                                   ctx.ratio, workspace=ctx.ws, reuse_binning=ctx.ws is not None,
                                   chw=ctx.chw)
        ctx.ws = None
        return (*grads, None, None, None, None)


def render_batch(alpha, mu, sigma, rho, color, images: Sequence[Tuple[int, int, float]],
                 counts: Sequence[int], ratio: float = 0.1):
    """Differentiable ragged batch render. images[k] = (H, W, s) owns counts[k] consecutive
    Gaussians; s is a number or a scale vector (s_x, s_y) (R22). Returns (flat output, Layout);
    Layout.view(flat, k) is image k as [Hs, Ws, 3]."""
    ims, off = [], 0
    for (H, W, s), c in zip(images, counts):
        sx, sy = _scale(s)
        ims.append(Image(int(H), int(W), sx, off, int(c), s_y=sy))
        off += int(c)
    lay = layout(ims)
    return _RenderFn.apply(alpha, mu, sigma, rho, color, lay, float(ratio)), lay


def render(alpha, mu, sigma, rho, color, H: int, W: int, scale: float,
           ratio: float = 0.1, out_dtype: Optional[torch.dtype] = None,
           chw: bool = False) -> torch.Tensor:
    """I_SR = Eq. 4 / Alg. 1 as a differentiable op: [floor(s_y H), floor(s_x W), 3] float32
    (scale = s or (s_x, s_y)); out_dtype=torch.bfloat16 and chw=True ([3, Hs, Ws]) select the
    NEXT-4 formats; float32 or bfloat16 parameters."""
    lay = _single(alpha.shape[0], H, W, scale)
    flat = _RenderFn.apply(alpha, mu, sigma, rho, color, lay, float(ratio), out_dtype, chw)
    return lay.view(flat, 0, chw=chw)


# ------------------------------------------------------------------ NEXT-1: fused training step
RAW = ("raw_alpha", "offset", "raw_sigma", "raw_rho", "raw_color")
RAW_WIDTH = {"raw_alpha": 1, "offset": 2, "ref": 2, "raw_sigma": 2, "raw_rho": 1, "raw_color": 3}


def train_step_l1(raw_alpha, offset, ref, raw_sigma, raw_rho, raw_color, lay: Layout,
                  gt: torch.Tensor, ratio: float = 0.1, rho_scale: float = 1.0,
                  inv_numel: float = 0.0, out: Optional[torch.Tensor] = None,
                  workspace: Optional[torch.Tensor] = None):
    """One fused training step of the rasterizer (gsr_train_step_l1_batched): activations of the
    Gaussian Primary Head, forward render, L1 loss against `gt` and the
    gradients wrt the raw head outputs. Returns (out, loss[1] float64, grads dict)."""
    ts = {}
    n = raw_alpha.shape[0]
    for name, t in zip(("raw_alpha", "offset", "ref", "raw_sigma", "raw_rho", "raw_color"),
                       (raw_alpha, offset, ref, raw_sigma, raw_rho, raw_color)):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
            raise TypeError(f"{name} must be a float32 CUDA tensor")
        t = t.contiguous()
        w = RAW_WIDTH[name]
        if t.shape[0] != n or (w == 1 and t.dim() != 1) or (w > 1 and t.shape[1:] != (w,)):
            raise ValueError(f"{name} has shape {tuple(t.shape)}")
        ts[name] = t
    dev = raw_alpha.device
    gt = _check_image(gt.contiguous(), "gt", lay, dev, dtypes=(torch.float32,))
    if not single_chunk(lay):
        raise ValueError(f"train_step_l1 takes at most {_lib.MAX_IMAGES} images per call")
    g0, g1, o0, arr, m = next(_chunks(lay))
    if g0 != 0 or g1 != n:
        raise ValueError("the layout's Gaussian ranges must span the parameter arrays")
    lib = _lib.load()
    nb = lib.gsr_train_workspace_bytes_batched(arr, m, n, float(ratio))
    if nb == 0:
        raise _lib.GsrError("gsr_train_workspace_bytes_batched: invalid arguments")
    ws = _ws_for(dev, nb, workspace)
    if out is None:
        out = torch.empty(lay.out_numel, dtype=torch.float32, device=dev)
    out = _check_image(out, "out", lay, dev, dtypes=(torch.float32,))
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    grads = {k: torch.empty_like(ts[k]) for k in RAW}
    check(lib.gsr_train_step_l1_batched(
        *[_ptr(ts[k]) for k in ("raw_alpha", "offset", "ref", "raw_sigma", "raw_rho", "raw_color")],
        n, arr, m, float(ratio), float(rho_scale), float(inv_numel), _ptr(gt), _ptr(out),
        _ptr(loss), *[_ptr(grads[k]) for k in RAW], ws.data_ptr(), ws.numel(),
        _stream_ptr(dev)), "gsr_train_step_l1_batched")
    return out, loss, grads


def train_workspace_for(n: int, lay: Layout, ratio: float = 0.1, device=None) -> torch.Tensor:
    """A private workspace for train_step_l1 on this layout (single chunk)."""
    g0, g1, o0, arr, m = next(_chunks(lay))
    nb = _lib.load().gsr_train_workspace_bytes_batched(arr, m, int(n), float(ratio))
    if nb == 0:
        raise _lib.GsrError("gsr_train_workspace_bytes_batched: invalid arguments")
    return torch.empty(nb, dtype=torch.uint8, device=device if device is not None else "cuda")


class TrainStepGraph:
    """NEXT-2: the fused training step (train_step_l1) captured once into a CUDA graph for a fixed
    batch layout (image sizes and per-image scales), replayed with new inputs copied into its
    static buffers -- one graph launch instead of ~25 kernel launches and their host-side
    argument checks per step. The graph owns its workspace and outputs; the returned tensors are
    overwritten by the next replay.

        step = TrainStepGraph(lay, n, ratio=0.1)
        out, loss, grads = step(raw_alpha, offset, ref, raw_sigma, raw_rho, raw_color, gt)
    """

    def __init__(self, lay: Layout, n: int, ratio: float = 0.1, rho_scale: float = 1.0,
                 inv_numel: float = 0.0, device=None):
        dev = torch.device(device if device is not None else "cuda")
        self.lay, self.n = lay, int(n)
        shapes = {"raw_alpha": (n,), "offset": (n, 2), "ref": (n, 2), "raw_sigma": (n, 2),
                  "raw_rho": (n,), "raw_color": (n, 3)}
        self.inp = {k: torch.zeros(s, dtype=torch.float32, device=dev) for k, s in shapes.items()}
        self.inp["raw_sigma"].fill_(-0.5)             # valid parameters for the warm-up
        self.gt = torch.zeros(lay.out_numel, dtype=torch.float32, device=dev)
        self.ws = train_workspace_for(n, lay, ratio, dev)
        self.args = dict(ratio=ratio, rho_scale=rho_scale, inv_numel=inv_numel, workspace=self.ws)
        order = ("raw_alpha", "offset", "ref", "raw_sigma", "raw_rho", "raw_color")
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):                 # warm-up: kernel attributes, allocator
            train_step_l1(*[self.inp[k] for k in order], lay, self.gt, **self.args)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out, self.loss, self.grads = train_step_l1(*[self.inp[k] for k in order], lay,
                                                            self.gt, **self.args)

    def __call__(self, raw_alpha, offset, ref, raw_sigma, raw_rho, raw_color, gt):
        for k, v in zip(("raw_alpha", "offset", "ref", "raw_sigma", "raw_rho", "raw_color"),
                        (raw_alpha, offset, ref, raw_sigma, raw_rho, raw_color)):
            self.inp[k].copy_(v, non_blocking=True)
        self.gt.copy_(gt, non_blocking=True)
        self.graph.replay()
        return self.out, self.loss, self.grads


# ------------------------------------------------------------------ host-resident batches
class StreamedFwdBwd:
    """Forward + backward of a batch whose inputs and outputs live in pinned HOST memory, the
    way a data pipeline hands it over: the images are processed in `groups` contiguous image
    groups, and while group k renders on the compute stream, group k+1's parameters and dL/dI
    are copied host->device on one copy stream and group k-1's image and gradients are copied
    device->host on another (B200's copy engines run both directions concurrently with the
    kernels). Each group is one binning + forward + backward (binning reused) + finalize.

        step = StreamedFwdBwd(lay, ratio, groups=16)
        step(host_params, host_grad_out, host_out, host_grads)   # enqueued on the current stream

    host_params: (alpha, mu, sigma, rho, color) pinned float32 CPU tensors (n Gaussians);
    host_grad_out / host_out: pinned flat float32 [lay.out_numel]; host_grads: 5 pinned tensors
    shaped like host_params. The call returns after enqueueing; the current stream waits for all
    work (synchronize it, or record an event, before reading the host outputs)."""

    def __init__(self, lay: Layout, ratio: float = 0.1, groups: int = 16, device=None,
                 ramp: bool = True):
        self.lay, self.ratio = lay, float(ratio)
        self.dev = torch.device(device if device is not None else "cuda")
        ims = lay.images
        n = max((im.g_off + im.g_cnt for im in ims), default=0)
        self.n = n
        G = max(1, min(groups, len(ims)))
        # image-group boundaries; ramp: the first and the last group hold one image each (the
        # first group's host->device copy and the last group's device->host copy are the only
        # ones no kernel hides), the rest split evenly
        N = len(ims)
        if ramp and G >= 4 and N >= G:
            mid = [1 + (q * (N - 2)) // (G - 2) for q in range(G - 1)]
            bounds = [0] + mid + [N]
        else:
            bounds = [(q * N) // G for q in range(G + 1)]
        self.groups = []
        for q in range(G):
            k0, k1 = bounds[q], bounds[q + 1]
            if k0 == k1:
                continue
            g0 = min(ims[k].g_off for k in range(k0, k1))
            g1 = max(ims[k].g_off + ims[k].g_cnt for k in range(k0, k1))
            sub = layout([Image(ims[k].H, ims[k].W, ims[k].s, ims[k].g_off - g0, ims[k].g_cnt,
                                lay.rows[k][0], lay.rows[k][1], ims[k].s_y)
                          for k in range(k0, k1)])
            o0 = lay.out_off[k0]
            self.groups.append((g0, g1, o0, o0 + sub.out_numel, sub))
        dev = self.dev
        widths = (1, 2, 2, 1, 3)
        self.d_par = [torch.empty((n, w) if w > 1 else (n,), dtype=torch.float32, device=dev)
                      for w in widths]
        self.d_grad = [torch.empty_like(t) for t in self.d_par]
        self.d_g = torch.empty(lay.out_numel, dtype=torch.float32, device=dev)
        self.d_out = torch.empty(lay.out_numel, dtype=torch.float32, device=dev)
        self.d_mom = torch.empty((n, 8), dtype=torch.float64, device=dev)
        nb = 256
        for g0, g1, o0, o1, sub in self.groups:
            for c0, c1, _, arr, m in _chunks(sub):
                nb = max(nb, _ws_bytes(arr, m, c1 - c0, self.ratio))
        self.ws = torch.empty(nb, dtype=torch.uint8, device=dev)
        self.s_h2d = torch.cuda.Stream(device=dev)
        self.s_cmp = torch.cuda.Stream(device=dev)
        self.s_d2h = torch.cuda.Stream(device=dev)

    def __call__(self, host_params, host_grad_out, host_out, host_grads):
        cur = torch.cuda.current_stream(self.dev)
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(cur)
        done_h2d, done_cmp = [], []
        for g0, g1, o0, o1, sub in self.groups:
            with torch.cuda.stream(self.s_h2d):
                for d, h in zip(self.d_par, host_params):
                    d[g0:g1].copy_(h[g0:g1], non_blocking=True)
                self.d_g[o0:o1].copy_(host_grad_out[o0:o1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_h2d)
                done_h2d.append(ev)
        for q, (g0, g1, o0, o1, sub) in enumerate(self.groups):
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(done_h2d[q])
                par = [t[g0:g1] for t in self.d_par]
                render_fwd_batched(*par, sub, self.ratio, out=self.d_out[o0:o1],
                                   workspace=self.ws)
                mom = self.d_mom[g0:g1]
                mom.zero_()
                render_bwd_moments_batched(*par, sub, self.d_g[o0:o1], mom, self.ratio,
                                           workspace=self.ws, reuse_binning=True)
                check(_lib.load().gsr_finalize_grads(
                    *[_ptr(t) for t in par], g1 - g0, _ptr(mom),
                    *[_ptr(t[g0:g1]) for t in self.d_grad], self.s_cmp.cuda_stream),
                    "gsr_finalize_grads")
                ev = torch.cuda.Event()
                ev.record(self.s_cmp)
                done_cmp.append(ev)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(ev)
                host_out[o0:o1].copy_(self.d_out[o0:o1], non_blocking=True)
                for h, d in zip(host_grads, self.d_grad):
                    h[g0:g1].copy_(d[g0:g1], non_blocking=True)
        cur.wait_stream(self.s_d2h)
        cur.wait_stream(self.s_cmp)
