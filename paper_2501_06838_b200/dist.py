"""Multi-GPU row-band sharding: one process per GPU, torch.distributed (NCCL over
NVLink on B200; gloo in the CPU tests) for the two exchange steps of the path.

Partition: every rank renders HR rows [b_r, b_{r+1}) of every image, with the Gaussians whose
window meets those rows (the halo) -- the library bins only band-intersecting Gaussians, so the
replicated parameters cost O(N) preprocessing per rank and nothing else. Boundaries equalise the
per-row pair counts (the work unit), not the row counts.

Per rank, `RankPlan` holds the halo (the Gaussians whose support meets the rank's bands) and the
neighbour seam sets; the rank bins, renders and finalizes only its halo (libgsr's subset entry
points), so its binning, moment zeroing and finalize scale with N/G + halo, not N.

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

import functools
import math
import os
from typing import Callable, List, Sequence

import numpy as np


PARAM_WIDTH = (1, 2, 2, 1, 3)       # alpha, mu, sigma, rho, color (include/gsr.h layouts)


def _img_tuple(im):
    """(H, W, s, g_off, g_cnt, s_y) of an ops.Image or a tuple (H, W, s, g_off, g_cnt[, s_y])."""
    if hasattr(im, "H"):
        return (int(im.H), int(im.W), float(im.s), int(im.g_off), int(im.g_cnt),
                im.s_y if getattr(im, "s_y", None) else None)
    t = tuple(im)
    return (int(t[0]), int(t[1]), float(t[2]), int(t[3]), int(t[4]),
            t[5] if len(t) > 5 and t[5] else None)


def _plan_calls(params, images):
    """ABI calls of <= GSR_MAX_IMAGES whole images each: (param pointers, n, images array,
    m, [image indices]); params are numpy float32/bfloat16-free host arrays (host variants) or
    CUDA tensors (device variants)."""
    from . import _lib
    ims = [_img_tuple(im) for im in images]
    for c0 in range(0, len(ims), _lib.MAX_IMAGES):
        sel = list(range(c0, min(c0 + _lib.MAX_IMAGES, len(ims))))
        g0 = min(ims[k][3] for k in sel)
        g1 = max(ims[k][3] + ims[k][4] for k in sel)
        recs = [(H, W, s, go - g0, gc, 0, 0, -1, sy) for (H, W, s, go, gc, sy) in
                (ims[k] for k in sel)]
        yield g0, g1, _lib.images_array(recs), len(sel), sel


def _is_host(params):
    return isinstance(params[0], np.ndarray)


def _host_params(params):
    return [np.ascontiguousarray(np.asarray(p, np.float32).reshape(-1, w) if w > 1 else
                                 np.asarray(p, np.float32).reshape(-1))
            for p, w in zip(params, PARAM_WIDTH)]


def _ptrs(params, g0):
    """Parameter pointers of Gaussian g0 on (host numpy or device tensor arrays)."""
    out = []
    for p, w in zip(params, PARAM_WIDTH):
        if isinstance(p, np.ndarray):
            out.append(p.ctypes.data + g0 * w * p.itemsize)
        else:
            out.append(p.data_ptr() + g0 * w * p.element_size())
    return out


def _flags(params, support=False):
    from . import _lib
    f = _lib.GSR_SUPPORT if support else 0
    if not _is_host(params):
        import torch
        if params[0].dtype == torch.bfloat16:
            f |= _lib.GSR_PARAMS_BF16
    return f


def row_pair_counts(params, images, ratio: float = 0.1, support: bool = True) -> List[np.ndarray]:
    """Exact pairs per HR row of every (whole) image: rowpairs[y] = sum_i [y0_i <= y <= y1_i]
    (x1_i - x0_i + 1), with Alg. 1's window rect (support=False) or the support rect of reading
    R21 (support=True: the pairs the kernels evaluate), computed by libgsr's K7 planner
    (gsr_row_pair_counts_*: the render kernels' own rect code). params = (alpha, mu, sigma, rho,
    color) as numpy arrays (host variant) or CUDA tensors (device variant). -> one int64 array
    per image."""
    from . import _lib
    lib = _lib.load()
    host = _is_host(params)
    if host:
        params = _host_params(params)
    res = [None] * len(images)
    for g0, g1, arr, m, sel in _plan_calls(params, images):
        rows = []
        for k in range(m):
            Hs, _ = _lib.out_dims(arr[k].lr_h, arr[k].lr_w, arr[k].scale, arr[k].scale_y or None)
            rows.append(Hs)
        tot = int(sum(rows))
        if host:
            out = np.zeros(tot, np.int64)
            _lib.check(lib.gsr_row_pair_counts_host(*_ptrs(params, g0), g1 - g0, arr, m,
                                                    float(ratio), _flags(params, support),
                                                    out.ctypes.data), "gsr_row_pair_counts_host")
        else:
            import torch
            dev = params[0].device
            d = torch.empty(tot, dtype=torch.int64, device=dev)
            _lib.check(lib.gsr_row_pair_counts_batched(
                *_ptrs(params, g0), g1 - g0, arr, m, float(ratio), _flags(params, support),
                d.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
                "gsr_row_pair_counts_batched")
            out = d.cpu().numpy()
        o = 0
        for k, h in zip(sel, rows):
            res[k] = out[o:o + h]
            o += h
    return res


def band_spans(params, images, bounds: Sequence[Sequence[int]], ratio: float = 0.1,
               margin: int = 0):
    """[n, 2] int16: first and last band of each image's boundaries `bounds[k]` that every
    Gaussian's support rows (R21) meet ({-1, -1}: invalid (R20) or empty), by libgsr's K7 planner
    (gsr_band_span_*). numpy in -> numpy out (host variant); CUDA tensors -> CUDA tensor."""
    from . import _lib
    lib = _lib.load()
    host = _is_host(params)
    if host:
        params = _host_params(params)
        n = params[0].shape[0]
        span = np.full((n, 2), -1, np.int16)
    else:
        import torch
        n = params[0].shape[0]
        span = torch.full((n, 2), -1, dtype=torch.int16, device=params[0].device)
    G = len(bounds[0]) - 1
    for g0, g1, arr, m, sel in _plan_calls(params, images):
        b = np.ascontiguousarray(np.array([list(bounds[k]) for k in sel], np.int32))
        if b.shape[1] != G + 1:
            raise ValueError("every image needs the same number of bands")
        if host:
            _lib.check(lib.gsr_band_span_host(*_ptrs(params, g0), g1 - g0, arr, m, float(ratio),
                                              _flags(params), b.ctypes.data, G, int(margin),
                                              span.ctypes.data + 4 * g0), "gsr_band_span_host")
        else:
            import torch
            dev = params[0].device
            _lib.check(lib.gsr_band_span_batched(
                *_ptrs(params, g0), g1 - g0, arr, m, float(ratio), _flags(params), b.ctypes.data,
                G, int(margin), span.data_ptr() + 4 * g0,
                torch.cuda.current_stream(dev).cuda_stream), "gsr_band_span_batched")
    return span


def seam_mask(span):
    """Seam Gaussians: support rows meeting more than one band."""
    return span[:, 0] < span[:, 1]


def halo_mask(span, r: int):
    """Gaussians whose support rows meet band r (rank r's replicated halo)."""
    return (span[:, 0] <= r) & (span[:, 1] >= r)


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


def _nvtx(fn):
    """NVTX range "gsr:<name>" around an exchange step when GSR_NVTX=1 (libgsr marks
    its kernel phases the same way)."""
    @functools.wraps(fn)
    def wrap(*a, **k):
        if os.environ.get("GSR_NVTX", "0") in ("", "0"):
            return fn(*a, **k)
        import torch
        torch.cuda.nvtx.range_push("gsr:" + fn.__name__)
        try:
            return fn(*a, **k)
        finally:
            torch.cuda.nvtx.range_pop()
    return wrap


@_nvtx
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


@_nvtx
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


class RankPlan:
    """One rank's share of a row-band shard, from the K7 planner's band spans:

      idx   int32 [m]  its halo: the Gaussians whose support rows (R21) meet its bands, ascending
                       -- the subset it bins, renders and finalizes (gsr_*_subset, compact
                       outputs: row t belongs to Gaussian idx[t]);
      up    int64      positions (into idx) of the Gaussians shared exactly with rank + 1
                       (span [rank, rank+1]); `down` likewise with rank - 1 -- the neighbour
                       seam exchange: both sides hold the same Gaussians in the same (ascending)
                       order, so the two buffers line up;
      multi_pos / multi_slot  Gaussians spanning three or more bands (supports taller than a
                       band; rare): positions in idx and slots in a global [n_multi] buffer that
                       every rank all-reduces.

    The band boundaries come from the row pair counts (work-balanced); spans and halos are
    recomputed by `refresh` whenever the parameters change (every training step)."""

    def __init__(self, params, images, world: int, rank: int, ratio: float = 0.1,
                 bounds=None):
        self.world, self.rank, self.ratio = world, rank, ratio
        self.images = [_img_tuple(im) for im in images]
        if bounds is None:
            bounds = [plan_bands(rc, world) for rc in row_pair_counts(params, images, ratio)]
        self.bounds = bounds
        self.refresh(params)

    def refresh(self, params):
        import torch
        r, G = self.rank, self.world
        if not _is_host(params) and len(self.images) <= 64:
            return self._refresh_device(params)
        span = torch.as_tensor(band_spans(params, self.images, self.bounds, self.ratio))
        f, l = span[:, 0].to(torch.int32), span[:, 1].to(torch.int32)
        halo = (f <= r) & (l >= r)
        self.idx = torch.nonzero(halo).reshape(-1).to(torch.int32)
        pos = torch.cumsum(halo.to(torch.int64), 0) - 1            # position within idx
        self.up = pos[torch.nonzero((f == r) & (l == r + 1)).reshape(-1)]
        self.down = pos[torch.nonzero((f == r - 1) & (l == r)).reshape(-1)]
        multi = torch.nonzero(l - f >= 2).reshape(-1)              # identical on every rank
        inh = halo[multi]
        self.n_multi = int(multi.numel())
        self.multi_pos = pos[multi[inh]]
        self.multi_slot = torch.nonzero(inh).reshape(-1)
        self.n_seam_local = int(self.up.numel() + self.down.numel() + self.multi_pos.numel())
        return self

    def _refresh_device(self, params):
        """One fused libgsr pass (gsr_rank_halo) instead of materialising the spans: halo
        compaction and the seam position lists on the device, one sync for the five counts."""
        import torch
        from . import _lib
        lib = _lib.load()
        dev = params[0].device
        n = int(params[0].shape[0])
        if getattr(self, "_buf", None) is None or self._buf[0].numel() < max(n, 1):
            self._buf = [torch.empty(max(n, 1), dtype=torch.int32, device=dev) for _ in range(5)]
            self._hws = torch.empty(max(int(lib.gsr_rank_halo_workspace_bytes(n)), 256),
                                    dtype=torch.uint8, device=dev)
            self._tot = torch.empty(5, dtype=torch.int64, device=dev)
        g0, g1, arr, m, sel = next(_plan_calls(params, self.images))
        if g0 != 0:
            raise ValueError("RankPlan needs images whose Gaussian ranges start at 0")
        b = np.ascontiguousarray(np.array(self.bounds, np.int32))
        _lib.check(lib.gsr_rank_halo(*_ptrs(params, 0), n, arr, m, float(self.ratio),
                                     _flags(params), b.ctypes.data, self.world, 0, self.rank,
                                     *[t.data_ptr() for t in self._buf], self._tot.data_ptr(),
                                     self._hws.data_ptr(), self._hws.numel(),
                                     torch.cuda.current_stream(dev).cuda_stream),
                   "gsr_rank_halo")
        nh, nu, nd, nm, nM = (int(v) for v in self._tot.cpu())
        self.idx = self._buf[0][:nh]
        self.up = self._buf[1][:nu].long()
        self.down = self._buf[2][:nd].long()
        self.multi_pos = self._buf[3][:nm].long()
        self.multi_slot = self._buf[4][:nm].long()
        self.n_multi = nM
        self.n_seam_local = nu + nd + nm
        return self

    @property
    def m(self) -> int:
        return int(self.idx.numel())

    def band_images(self):
        """(H, W, s, g_off, g_cnt, row_begin, row_end, s_y) of this rank's band of every image."""
        return [(H, W, s, go, gc, b[self.rank], b[self.rank + 1], sy)
                for (H, W, s, go, gc, sy), b in zip(self.images, self.bounds)]

    def exchange_bytes(self) -> dict:
        """Bytes this rank sends per step in the seam exchange (float32 [k, 9] rows)."""
        return {"p2p_up": 36 * int(self.up.numel()), "p2p_down": 36 * int(self.down.numel()),
                "multi_allreduce": 36 * self.n_multi}


@_nvtx
def exchange_seams(grads, plan: RankPlan, group=None):
    """Neighbour seam exchange of a rank's COMPACT partial gradients (the finalize of its halo
    moments, rows = plan.idx): the rows shared with rank +- 1 are swapped with that neighbour
    (torch.distributed P2P: NCCL send/recv over NVLink) and added, so both ranks end with the
    full gradient; Gaussians spanning >= 3 bands are summed by one all-reduce of a small
    global buffer. `grads` = one [m, k] tensor or a sequence of [m] / [m, k] tensors."""
    import torch
    import torch.distributed as dist
    ts = [grads] if isinstance(grads, torch.Tensor) else list(grads)
    m = ts[0].shape[0]
    cols = [t.view(m, -1) for t in ts]
    r, G = plan.rank, plan.world
    # gloo (the CPU tests and the 1-GPU functional check of bench.py) has no point-to-point path
    # for CUDA tensors: stage those buffers through host memory; NCCL sends device memory
    host_p2p = ts[0].is_cuda and dist.get_backend(group) == "gloo"
    ops, recv = [], []
    for peer, sel in ((r + 1, plan.up), (r - 1, plan.down)):
        if 0 <= peer < G and sel.numel() > 0:
            send = torch.cat([c.index_select(0, sel) for c in cols], 1).contiguous()
            wire = send.cpu() if host_p2p else send
            rb = torch.empty_like(wire)
            ops.append(dist.P2POp(dist.isend, wire, peer, group))
            ops.append(dist.P2POp(dist.irecv, rb, peer, group))
            recv.append((sel, rb, send))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for sel, rb, send in recv:
        tot = send + rb.to(send.device)
        o = 0
        for c in cols:
            k = c.shape[1]
            c.index_copy_(0, sel, tot[:, o:o + k])
            o += k
    if plan.n_multi:
        width = sum(c.shape[1] for c in cols)
        buf = cols[0].new_zeros((plan.n_multi, width))
        if plan.multi_pos.numel():
            buf.index_copy_(0, plan.multi_slot,
                            torch.cat([c.index_select(0, plan.multi_pos) for c in cols], 1))
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        if plan.multi_pos.numel():
            sel = buf.index_select(0, plan.multi_slot)
            o = 0
            for c in cols:
                k = c.shape[1]
                c.index_copy_(0, plan.multi_pos, sel[:, o:o + k])
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
