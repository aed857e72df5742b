"""Introspection of the binning stage through the C-ABI (gsr_debug_rects / gsr_debug_tile_lists),
used by the bit-exact binning tests. Same kernels as the render path."""
from __future__ import annotations

import torch

from . import _lib
from ._lib import check
from .ops import _params, _ptr, _stream_ptr


def rects(alpha, mu, sigma, rho, color, H, W, s, ratio=0.1, support=False) -> torch.Tensor:
    """[n, 4] int32 (x0, x1, y0, y1) clipped window rects as the GPU computes them
    (support=True: the support rects the kernels evaluate, reading R21)."""
    (alpha, mu, sigma, rho, color), n = _params(alpha, mu, sigma, rho, color)
    out = torch.empty((n, 4), dtype=torch.int32, device=alpha.device)
    check(_lib.load().gsr_debug_rects_ex(_ptr(alpha), _ptr(mu), _ptr(sigma), _ptr(rho),
                                         _ptr(color), n, int(H), int(W), float(s), float(ratio),
                                         _lib.GSR_SUPPORT if support else 0, _ptr(out),
                                         _stream_ptr(alpha.device)), "gsr_debug_rects_ex")
    return out


def tile_lists(alpha, mu, sigma, rho, color, H, W, s, ratio=0.1):
    """(counts[ntiles], ids, cells) as visited by the render kernels (CSR by tile)."""
    (alpha, mu, sigma, rho, color), n = _params(alpha, mu, sigma, rho, color)
    dev = alpha.device
    lib = _lib.load()
    Hs, Ws = _lib.out_dims(H, W, s)
    tw, th, _, _ = _lib.tile_shape()
    ntiles = -(-Ws // tw) * -(-Hs // th)
    nb = lib.gsr_workspace_bytes(n, int(H), int(W), float(s), float(ratio))
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    counts = torch.zeros(ntiles, dtype=torch.int32, device=dev)
    st = _stream_ptr(dev)
    args = (_ptr(alpha), _ptr(mu), _ptr(sigma), _ptr(rho), _ptr(color), n, int(H), int(W),
            float(s), float(ratio))
    check(lib.gsr_debug_tile_lists(*args, _ptr(counts), None, None, ws.data_ptr(), nb, st),
          "gsr_debug_tile_lists(counts)")
    total = int(counts.sum().item())
    ids = torch.zeros(max(total, 1), dtype=torch.int32, device=dev)
    cells = torch.zeros(max(total, 1), dtype=torch.int32, device=dev)
    check(lib.gsr_debug_tile_lists(*args, None, _ptr(ids), _ptr(cells), ws.data_ptr(), nb, st),
          "gsr_debug_tile_lists(ids)")
    return counts, ids[:total], cells[:total]


def fwd_tile_lists(alpha, mu, sigma, rho, color, H, W, s, ratio=0.1):
    """Forward tiles' kept candidates as K4 walks and filters them (gsr_debug_fwd_tile_lists):
    ((ftile_w, ftile_h, ntiles), counts[ntiles], ids, paths), CSR by tile in stream order."""
    import ctypes
    (alpha, mu, sigma, rho, color), n = _params(alpha, mu, sigma, rho, color)
    dev = alpha.device
    lib = _lib.load()
    nb = lib.gsr_workspace_bytes(n, int(H), int(W), float(s), float(ratio))
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    st = _stream_ptr(dev)
    geom = (ctypes.c_int32 * 3)()
    Hs, Ws = _lib.out_dims(H, W, s)
    nmax = -(-Ws // 16) * -(-Hs // 8)                  # the smaller forward tile bounds the count
    counts = torch.zeros(max(nmax, 1), dtype=torch.int32, device=dev)
    args = (_ptr(alpha), _ptr(mu), _ptr(sigma), _ptr(rho), _ptr(color), n, int(H), int(W),
            float(s), float(ratio))
    check(lib.gsr_debug_fwd_tile_lists(*args, ctypes.cast(geom, ctypes.c_void_p), None,
                                       _ptr(counts), None, None, ws.data_ptr(), nb, st),
          "gsr_debug_fwd_tile_lists(counts)")
    tw, th, nt = geom[0], geom[1], geom[2]
    counts = counts[:nt]
    offs = torch.zeros(max(nt, 1), dtype=torch.int32, device=dev)
    if nt > 1:
        offs[1:nt] = torch.cumsum(counts, 0)[:-1].to(torch.int32)
    total = int(counts.sum().item())
    ids = torch.zeros(max(total, 1), dtype=torch.int32, device=dev)
    paths = torch.zeros(max(total, 1), dtype=torch.uint8, device=dev)
    check(lib.gsr_debug_fwd_tile_lists(*args, ctypes.cast(geom, ctypes.c_void_p), _ptr(offs),
                                       None, _ptr(ids), _ptr(paths), ws.data_ptr(), nb, st),
          "gsr_debug_fwd_tile_lists(ids)")
    return (tw, th, nt), counts, ids[:total], paths[:total]
