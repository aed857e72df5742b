"""Multi-GPU row-band sharding: one process per GPU, torch.distributed (NCCL over
NVLink on B200; gloo in the CPU tests) for the two exchange steps of the path.

Partition: every rank renders HR rows [b_r, b_{r+1}) of every image, with the Gaussians whose
window meets those rows (the halo) -- the library bins only band-intersecting Gaussians, so the
replicated parameters cost O(N) preprocessing per rank and nothing else. Boundaries equalise the
per-row pair counts (the work unit), not the row counts.

Exchange steps (the only collectives):
  forward : all-gather of the output bands (each rank's bands padded to the largest) -> every
            rank holds every band, `assemble_image` views/copies out a full image;
  backward: every rank accumulates the pair moments [n, 8] (float64) of its bands and
            finalizes them locally (the closed forms of gsr_finalize_grads are linear in the
            moments, so a band's gradient is the finalize of its moments). Only SEAM Gaussians --
            support rect (R21) spanning a band boundary -- have partial gradients on several
            ranks; they are packed into one compact [n_seam, 9] buffer and sum-reduced
            (`reduce_seam`). Afterwards rank r holds the final gradient of every Gaussian its
            band sees (its halo) and 0 for the others; `reduce_seam(full=True)` all-reduces every
            gradient instead when each rank needs all of them.
  overlap : the output all-gather is issued asynchronously right after the forward and runs on
            NCCL's stream while the backward computes (waited for at the end of the step).

The band renderer is injected (`render_band` / `moments_band` / `finalize`), so this host logic
is tested on CPU with gloo and a CPU stand-in, and runs on B200 with the CUDA path.
"""
from __future__ import annotations

import math
from typing import Callable, List, Sequence

import numpy as np


def out_size(n: int, s: float) -> int:
    return int(math.floor(s * n))


SUPPORT_SIGMAS = 13.5      # reading R21: the kernels' evaluation box, +-13.5 sigma


def row_pair_counts(mu: np.ndarray, valid: np.ndarray, H: int, W: int, s: float, ratio: float,
                    sigma: np.ndarray | None = None) -> np.ndarray:
    """Exact pairs per HR row of one image: rowpairs[y] = sum_i [y0_i <= y <= y1_i] (x1_i-x0_i+1),
    with the integer window rect of reading R2 (fp64, same operation order as the kernels), cut
    to the support box of reading R21 when sigma is given (the pairs the kernels evaluate)."""
    Hs, Ws = out_size(H, s), out_size(W, s)
    mx = mu[:, 0].astype(np.float64)
    my = mu[:, 1].astype(np.float64)
    hx, hy = ratio * W, ratio * H
    lim = float(2 ** 30)
    with np.errstate(invalid="ignore"):
        x0 = np.floor(np.clip(s * (mx - hx), -lim, lim)) + 1
        x1 = np.ceil(np.clip(s * (mx + hx), -lim, lim)) - 1
        y0 = np.floor(np.clip(s * (my - hy), -lim, lim)) + 1
        y1 = np.ceil(np.clip(s * (my + hy), -lim, lim)) - 1
        if sigma is not None:
            tx = SUPPORT_SIGMAS * sigma[:, 0].astype(np.float64)
            ty = SUPPORT_SIGMAS * sigma[:, 1].astype(np.float64)
            x0 = np.maximum(x0, np.floor(np.clip(s * (mx - tx), -lim, lim)))
            x1 = np.minimum(x1, np.ceil(np.clip(s * (mx + tx), -lim, lim)))
            y0 = np.maximum(y0, np.floor(np.clip(s * (my - ty), -lim, lim)))
            y1 = np.minimum(y1, np.ceil(np.clip(s * (my + ty), -lim, lim)))
        x0 = np.maximum(x0, 0); x1 = np.minimum(x1, Ws - 1)
        y0 = np.maximum(y0, 0); y1 = np.minimum(y1, Hs - 1)
        ok = valid & (x0 <= x1) & (y0 <= y1)
    w = (x1 - x0 + 1)[ok].astype(np.int64)
    d = np.zeros(Hs + 1, np.int64)
    np.add.at(d, y0[ok].astype(np.int64), w)
    np.add.at(d, y1[ok].astype(np.int64) + 1, -w)
    return np.cumsum(d[:-1])


def support_rows(mu: np.ndarray, sigma: np.ndarray, valid: np.ndarray, H: int, W: int, s: float,
                 ratio: float, s_y: float | None = None):
    """Clipped HR row range [y0, y1] of every Gaussian's support rect (R2 window cut to the R21
    box, fp64 in the kernels' operation order); ok = the rect is non-empty."""
    sy = s if not s_y else s_y
    Hs, Ws = out_size(H, sy), out_size(W, s)
    mx = mu[:, 0].astype(np.float64)
    my = mu[:, 1].astype(np.float64)
    lim = float(2 ** 30)
    with np.errstate(invalid="ignore"):
        x0 = np.floor(np.clip(s * (mx - ratio * W), -lim, lim)) + 1
        x1 = np.ceil(np.clip(s * (mx + ratio * W), -lim, lim)) - 1
        y0 = np.floor(np.clip(sy * (my - ratio * H), -lim, lim)) + 1
        y1 = np.ceil(np.clip(sy * (my + ratio * H), -lim, lim)) - 1
        tx = SUPPORT_SIGMAS * sigma[:, 0].astype(np.float64)
        ty = SUPPORT_SIGMAS * sigma[:, 1].astype(np.float64)
        x0 = np.maximum(x0, np.floor(np.clip(s * (mx - tx), -lim, lim)))
        x1 = np.minimum(x1, np.ceil(np.clip(s * (mx + tx), -lim, lim)))
        y0 = np.maximum(y0, np.floor(np.clip(sy * (my - ty), -lim, lim)))
        y1 = np.minimum(y1, np.ceil(np.clip(sy * (my + ty), -lim, lim)))
        x0 = np.maximum(x0, 0); x1 = np.minimum(x1, Ws - 1)
        y0 = np.maximum(y0, 0); y1 = np.minimum(y1, Hs - 1)
        ok = valid & (x0 <= x1) & (y0 <= y1)
    return np.where(ok, y0, 0).astype(np.int64), np.where(ok, y1, -1).astype(np.int64), ok


def seam_mask(mu: np.ndarray, sigma: np.ndarray, valid: np.ndarray, H: int, W: int, s: float,
              ratio: float, bounds: Sequence[int], margin: int = 1,
              s_y: float | None = None) -> np.ndarray:
    """Gaussians of one image whose support rows meet more than one band of `bounds` (the seam
    set of SURVEY 8(e)). Conservative: the rows are widened by `margin` -- a Gaussian wrongly
    marked as a seam only costs buffer space (its partials are complete on one rank, 0 on the
    others); a seam Gaussian marked interior would lose gradient."""
    y0, y1, ok = support_rows(mu, sigma, valid, H, W, s, ratio, s_y)
    b = np.asarray(bounds, np.int64)
    first = np.searchsorted(b, y0 - margin, side="right") - 1
    last = np.searchsorted(b, y1 + margin, side="right") - 1
    return ok & (first < last)


def halo_mask(mu: np.ndarray, sigma: np.ndarray, valid: np.ndarray, H: int, W: int, s: float,
              ratio: float, rows, s_y: float | None = None) -> np.ndarray:
    """Gaussians of one image whose support rows meet HR rows [rows[0], rows[1]) (exact)."""
    y0, y1, ok = support_rows(mu, sigma, valid, H, W, s, ratio, s_y)
    return ok & (y1 >= rows[0]) & (y0 < rows[1])


def plan_bands(row_counts: np.ndarray, G: int) -> List[int]:
    """Boundaries b_0 = 0 <= ... <= b_G = Hs splitting the rows into G contiguous bands of
    (nearly) equal pair count; every band gets at least one row when Hs >= G."""
    Hs = int(row_counts.shape[0])
    if G <= 1:
        return [0, Hs]
    cum = np.cumsum(row_counts.astype(np.float64))
    total = float(cum[-1]) if Hs else 0.0
    b = [0]
    for g in range(1, G):
        if total <= 0:
            y = (g * Hs) // G
        else:
            target = g * total / G
            hi = int(np.searchsorted(cum, target, side="left")) + 1   # cum[hi-1] >= target
            lo = hi - 1
            c_lo = cum[lo - 1] if lo >= 1 else 0.0
            y = lo if abs(c_lo - target) <= abs(cum[hi - 1] - target) else hi
        if Hs >= G:
            y = min(max(y, b[-1] + 1), Hs - (G - g))
        else:
            y = min(max(y, b[-1]), Hs)
        b.append(y)
    b.append(Hs)
    return b


def band_imbalance(row_counts: np.ndarray, bounds: Sequence[int]) -> float:
    """max band work / mean band work (1.0 = perfect balance)."""
    w = [float(row_counts[bounds[g]:bounds[g + 1]].sum()) for g in range(len(bounds) - 1)]
    m = float(np.mean(w)) if w else 0.0
    return max(w) / m if m > 0 else 1.0


def rank_numels(bounds: Sequence[Sequence[int]], widths3: Sequence[int], world: int) -> List[int]:
    """Floats of rank r's output: the concatenation of its band of every image."""
    return [sum((b[r + 1] - b[r]) * w3 for b, w3 in zip(bounds, widths3)) for r in range(world)]


def gather_bands(out, numels: Sequence[int], group=None, async_op: bool = False):
    """All-gather every rank's flat band buffer, padded to the largest: -> [world, max]
    (async_op: -> ([world, max], work); the buffer is valid after work.wait())."""
    import torch
    import torch.distributed as dist
    world = len(numels)
    mx = max(numels)
    send = out if out.numel() == mx else torch.cat(
        [out.reshape(-1), out.new_zeros(mx - out.numel())])
    recv = out.new_empty(world * mx)
    if send.is_cuda and dist.get_backend(group) == "gloo":
        # gloo (the 1-GPU functional check of bench.py) gathers CUDA tensors as a list
        work = dist.all_gather(list(recv.view(world, mx).unbind(0)), send.contiguous(),
                               group=group, async_op=async_op)
    else:
        work = dist.all_gather_into_tensor(recv, send.contiguous(), group=group,
                                           async_op=async_op)
    return (recv.view(world, mx), work) if async_op else recv.view(world, mx)


def assemble_image(gathered, bounds: Sequence[Sequence[int]], widths3: Sequence[int], k: int):
    """Full image k ([Hs_k, Ws_k*3]) from the gathered bands of every rank."""
    import torch
    world = gathered.shape[0]
    parts = []
    for r in range(world):
        off = sum((b[r + 1] - b[r]) * w3 for b, w3 in zip(bounds[:k], widths3[:k]))
        rows = bounds[k][r + 1] - bounds[k][r]
        parts.append(gathered[r, off:off + rows * widths3[k]].view(rows, widths3[k]))
    return torch.cat(parts, 0)


def reduce_moments(moments, group=None):
    """Sum the per-rank partial moments [n, 8] (float64) of every Gaussian in place (the
    uncompacted exchange; `reduce_seam` moves only the seam Gaussians' gradients)."""
    import torch.distributed as dist
    dist.all_reduce(moments, op=dist.ReduceOp.SUM, group=group)
    return moments


def reduce_seam(grads, seam_idx, group=None, full: bool = False):
    """Seam reduce of per-rank partial gradients: `grads` is one [n, k] tensor or a sequence of
    [n] / [n, k] tensors (the finalize's d_alpha, d_mu, ...); the rows `seam_idx` (int64 tensor on
    the same device, identical on every rank) are packed into one [n_seam, sum k] buffer,
    all-reduced, and written back. full=True all-reduces every row instead."""
    import torch
    import torch.distributed as dist
    ts = [grads] if isinstance(grads, torch.Tensor) else list(grads)
    n = ts[0].shape[0]
    cols = [t.view(n, -1) for t in ts]
    if full:
        for c in cols:
            dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
        return grads
    if seam_idx.numel() == 0:
        return grads
    buf = torch.cat([c.index_select(0, seam_idx) for c in cols], 1)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    o = 0
    for c in cols:
        k = c.shape[1]
        c.index_copy_(0, seam_idx, buf[:, o:o + k])
        o += k
    return grads


def sharded_step(rank: int, world: int, bounds: Sequence[Sequence[int]], widths3: Sequence[int],
                 render_band: Callable, moments_band: Callable, finalize: Callable, n: int,
                 device, group=None, moment_cols: int = 8, seam_idx=None):
    """One fwd+bwd step of a batch under row-band sharding. render_band(rows) -> this rank's flat
    bands (images in order); moments_band(rows, moments) accumulates its band moments;
    finalize(moments) -> gradients (linear in the moments). seam_idx: the seam Gaussians
    (`seam_mask`); None = all-reduce every gradient. Returns (gathered bands [world, max] or the
    local bands, gradients)."""
    import torch
    rows = [(b[rank], b[rank + 1]) for b in bounds]
    out = render_band(rows)
    gathered, work = out, None
    if world > 1:                      # overlapped with the backward below
        gathered, work = gather_bands(out, rank_numels(bounds, widths3, world), group,
                                      async_op=True)
    moments = torch.zeros((n, moment_cols), dtype=torch.float64, device=device)
    moments_band(rows, moments)
    grads = finalize(moments)
    if world > 1:
        reduce_seam(grads, seam_idx, group, full=seam_idx is None)
        work.wait()
    return gathered, grads
