"""ctypes wrapper over liboracle.so (gsr_oracle.c). TEST INFRASTRUCTURE ONLY.

Every function takes the same float32 parameter arrays the GPU gets and widens
them exactly to float64 before calling the C oracle ("Oracle
inputs are the same fp32 arrays the GPU gets, widened exactly to fp64").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "gsr_oracle.c"
_LIB = _HERE / "liboracle.so"

_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_dbl = ctypes.c_double
_p = ctypes.c_void_p


def build_oracle(force: bool = False) -> Path:
    """Compile the C oracle (plain loops, no fast-math, no FMA contraction)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(".so.tmp%d" % os.getpid())
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared",
               "-fPIC", "-std=c11", "-o", str(tmp), str(_SRC), "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


class OracleLib:
    _inst = None

    def __init__(self):
        build_oracle()
        lib = ctypes.CDLL(str(_LIB))
        lib.gsr_oracle_out_dims.argtypes = [_i32, _i32, _dbl, _dbl, ctypes.POINTER(_i32),
                                            ctypes.POINTER(_i32)]
        lib.gsr_oracle_set_threads.argtypes = [_i32]
        lib.gsr_oracle_max_threads.restype = _i32
        par = [_i64, _p, _p, _p, _p, _p, _i32, _i32, _dbl, _dbl, _dbl]
        lib.gsr_oracle_rects.argtypes = par + [_i32, _p]
        lib.gsr_oracle_pair_count.argtypes = par + [_i32, _i32, _i32]
        lib.gsr_oracle_pair_count.restype = _i64
        lib.gsr_oracle_render_fwd.argtypes = par + [_i32, _i32, _i32, _p]
        lib.gsr_oracle_render_pixels.argtypes = par + [_i64, _p, _p, _p]
        lib.gsr_oracle_field.argtypes = [_i64, _p, _p, _p, _p, _p, _dbl, _dbl, _i64, _p, _p]
        lib.gsr_oracle_render_bwd.argtypes = par + [_i32, _i32, _i32, _p, _i64, _p, _p, _p, _p,
                                                    _p, _p, _p, _p]
        lib.gsr_oracle_tile_lists.argtypes = par + [_i32, _i32, _i32, _i32, _i32, _p, _p]
        lib.gsr_oracle_tile_lists.restype = _i64
        self.lib = lib

    @classmethod
    def get(cls) -> "OracleLib":
        if cls._inst is None:
            cls._inst = OracleLib()
        return cls._inst


def load() -> OracleLib:
    return OracleLib.get()


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _params(cloud):
    """Widen float32 parameter arrays exactly to contiguous float64."""
    out = []
    for k, shape in (("alpha", (-1,)), ("mu", (-1, 2)), ("sigma", (-1, 2)), ("rho", (-1,)),
                     ("color", (-1, 3))):
        a = np.ascontiguousarray(np.asarray(cloud[k]).reshape(shape), dtype=np.float64)
        out.append(a)
    return out


def set_threads(n: int) -> None:
    load().lib.gsr_oracle_set_threads(int(n))


def max_threads() -> int:
    return int(load().lib.gsr_oracle_max_threads())


def scales(s):
    """Scale argument -> (s_w, s_h): a number s is the paper's isotropic scale (s, s); a pair
    (s_x, s_y) is the NEXT-4 scale vector, s_x along W (x), s_y along H (y), DESIGN R22."""
    if isinstance(s, (tuple, list, np.ndarray)):
        sw, sh = (float(v) for v in s)
        return sw, sh
    return float(s), float(s)


def out_dims(H: int, W: int, s):
    hs, ws = _i32(), _i32()
    load().lib.gsr_oracle_out_dims(int(H), int(W), *scales(s), ctypes.byref(hs), ctypes.byref(ws))
    return hs.value, ws.value


MODES = {"brute": 0, "rect": 1, "none": 2, "support": 3}


def render_fwd(cloud, H, W, s, r=0.1, mode="rect", rows=None) -> np.ndarray:
    """I_SR as float64 [rows, Ws, 3] (all rows unless rows=(begin, end))."""
    a, mu, sg, rh, c = _params(cloud)
    Hs, Ws = out_dims(H, W, s)
    rb, re = (0, Hs) if rows is None else rows
    re = min(re, Hs)
    out = np.zeros((max(re - rb, 0), Ws, 3), np.float64)
    load().lib.gsr_oracle_render_fwd(a.shape[0], _ptr(a), _ptr(mu), _ptr(sg), _ptr(rh), _ptr(c),
                                     int(H), int(W), *scales(s), float(r), MODES[mode], int(rb),
                                     int(re), _ptr(out))
    return out


def render_pixels(cloud, H, W, s, r, px_x, px_y) -> np.ndarray:
    a, mu, sg, rh, c = _params(cloud)
    px_x = np.ascontiguousarray(px_x, np.int32)
    px_y = np.ascontiguousarray(px_y, np.int32)
    out = np.zeros((px_x.shape[0], 3), np.float64)
    load().lib.gsr_oracle_render_pixels(a.shape[0], _ptr(a), _ptr(mu), _ptr(sg), _ptr(rh),
                                        _ptr(c), int(H), int(W), *scales(s), float(r),
                                        px_x.shape[0], _ptr(px_x), _ptr(px_y), _ptr(out))
    return out


def field(cloud, hx, hy, pts) -> np.ndarray:
    a, mu, sg, rh, c = _params(cloud)
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
    out = np.zeros((pts.shape[0], 3), np.float64)
    load().lib.gsr_oracle_field(a.shape[0], _ptr(a), _ptr(mu), _ptr(sg), _ptr(rh), _ptr(c),
                                float(hx), float(hy), pts.shape[0], _ptr(pts), _ptr(out))
    return out


def render_bwd(cloud, H, W, s, r, grad_out, mode="rect", rows=None, idx=None,
               want_absmass=False):
    """Gradients (float64) of L = sum(grad_out * I) wrt every parameter.

    Returns dict alpha[n'], mu[n',2], sigma[n',2], rho[n'], color[n',3] for the Gaussians in idx
    (all if None); want_absmass adds absmass[n',9] (sum of the monomial magnitudes of each
    per-pair term, DESIGN R18) and termabs[n',9] (sum of |term|)."""
    a, mu, sg, rh, c = _params(cloud)
    Hs, Ws = out_dims(H, W, s)
    rb, re = (0, Hs) if rows is None else rows
    g = np.ascontiguousarray(grad_out, np.float64).reshape(re - rb, Ws, 3)
    n = a.shape[0]
    if idx is not None:
        idx = np.ascontiguousarray(idx, np.int64)
        m = idx.shape[0]
    else:
        m = n
    res = dict(alpha=np.zeros(m), mu=np.zeros((m, 2)), sigma=np.zeros((m, 2)), rho=np.zeros(m),
               color=np.zeros((m, 3)))
    am = np.zeros((m, 9)) if want_absmass else None
    ta = np.zeros((m, 9)) if want_absmass else None
    load().lib.gsr_oracle_render_bwd(
        n, _ptr(a), _ptr(mu), _ptr(sg), _ptr(rh), _ptr(c), int(H), int(W), *scales(s), float(r),
        MODES[mode], int(rb), int(re), _ptr(g), m if idx is not None else 0,
        _ptr(idx) if idx is not None else None, _ptr(res["alpha"]), _ptr(res["mu"]),
        _ptr(res["sigma"]), _ptr(res["rho"]), _ptr(res["color"]),
        _ptr(am) if am is not None else None, _ptr(ta) if ta is not None else None)
    if am is not None:
        res["absmass"] = am
        res["termabs"] = ta
    return res


def rects(cloud, H, W, s, r=0.1, support=False) -> np.ndarray:
    """[n,6] int64: x0u, y0u (unclipped starts), x0, x1, y0, y1 (clipped; empty -> x0>x1).
    support=True: the window rect intersected with the +-13.5 sigma box (reading R21)."""
    a, mu, sg, rh, c = _params(cloud)
    out = np.zeros((a.shape[0], 6), np.int64)
    load().lib.gsr_oracle_rects(a.shape[0], _ptr(a), _ptr(mu), _ptr(sg), _ptr(rh), _ptr(c),
                                int(H), int(W), *scales(s), float(r), int(bool(support)), _ptr(out))
    return out


def pair_count(cloud, H, W, s, r=0.1, rows=None, support=False) -> int:
    """Pairs passing the window predicate (support=True: inside the support rect, R21)."""
    a, mu, sg, rh, c = _params(cloud)
    Hs, _ = out_dims(H, W, s)
    rb, re = (0, Hs) if rows is None else rows
    return int(load().lib.gsr_oracle_pair_count(a.shape[0], _ptr(a), _ptr(mu), _ptr(sg),
                                                _ptr(rh), _ptr(c), int(H), int(W), *scales(s),
                                                float(r), int(rb), int(re), int(bool(support))))


def tile_lists(cloud, H, W, s, r, tw, th, rows=None, support=False):
    """Brute-force per-tile Gaussian lists: (counts[nty*ntx], ids) CSR, ascending i."""
    a, mu, sg, rh, c = _params(cloud)
    Hs, Ws = out_dims(H, W, s)
    rb, re = (0, Hs) if rows is None else rows
    ntx = (Ws + tw - 1) // tw
    nty = (min(re, Hs) - rb + th - 1) // th
    counts = np.zeros(ntx * nty, np.int64)
    lib = load().lib
    args = (a.shape[0], _ptr(a), _ptr(mu), _ptr(sg), _ptr(rh), _ptr(c), int(H), int(W), *scales(s),
            float(r), int(tw), int(th), int(rb), int(re), int(bool(support)))
    total = lib.gsr_oracle_tile_lists(*args, _ptr(counts), None)
    ids = np.zeros(max(total, 1), np.int64)
    lib.gsr_oracle_tile_lists(*args, _ptr(counts), _ptr(ids))
    return counts, ids[:total]
