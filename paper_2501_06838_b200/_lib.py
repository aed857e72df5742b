"""ctypes loader for libgsr.so (the C-ABI of include/gsr.h). Argument marshalling only.

There is no fallback: if the library is missing or cannot be loaded the import of the ops fails
loudly (RuntimeError) -- the product path never routes through the oracle or a CPU renderer.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libgsr.so"

GSR_OK, GSR_EINVAL, GSR_EWORKSPACE, GSR_ECUDA = 0, 1, 2, 3
_ERR = {GSR_EINVAL: "GSR_EINVAL (invalid argument)", GSR_EWORKSPACE: "GSR_EWORKSPACE",
        GSR_ECUDA: "GSR_ECUDA (kernel launch failed)"}
MAX_IMAGES = 64

# Every symbol include/gsr.h declares (checked by tests/test_abi.py).
EXPORTS = ["gsr_version", "gsr_out_dims", "gsr_out_dims_v", "gsr_workspace_bytes_batched", "gsr_workspace_bytes",
           "gsr_render_fwd", "gsr_render_bwd", "gsr_render_fwd_batched", "gsr_render_bwd_batched",
           "gsr_render_bwd_moments_batched", "gsr_finalize_grads", "gsr_pair_count_batched",
           "gsr_debug_rects", "gsr_debug_tile_lists", "gsr_tile_shape", "gsr_profile_enable",
           "gsr_profile_collect", "gsr_render_bwd_batched_ex", "gsr_render_bwd_moments_batched_ex",
           "gsr_train_workspace_bytes_batched", "gsr_train_step_l1_batched",
           "gsr_pair_count_batched_ex", "gsr_debug_rects_ex", "gsr_render_fwd_batched_ex",
           "gsr_finalize_grads_ex", "gsr_row_pair_counts_batched", "gsr_row_pair_counts_host",
           "gsr_band_span_batched", "gsr_band_span_host", "gsr_workspace_bytes_subset",
           "gsr_render_fwd_subset", "gsr_render_bwd_moments_subset", "gsr_finalize_grads_subset",
           "gsr_validate_params", "gsr_rank_halo_workspace_bytes", "gsr_rank_halo",
           "gsr_debug_fwd_tile_lists"]
GSR_REUSE_BINNING = 0x1
GSR_SUPPORT = 0x2
GSR_OUT_BF16 = 0x4
GSR_OUT_CHW = 0x8
GSR_PARAMS_BF16 = 0x10


class GsrImage(ctypes.Structure):
    _fields_ = [("lr_h", ctypes.c_int32), ("lr_w", ctypes.c_int32), ("scale", ctypes.c_double),
                ("g_off", ctypes.c_int64), ("g_cnt", ctypes.c_int64), ("out_off", ctypes.c_int64),
                ("row_begin", ctypes.c_int32), ("row_end", ctypes.c_int32),
                ("scale_y", ctypes.c_double)]


class GsrError(RuntimeError):
    pass


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double
_SZ = ctypes.c_size_t
_IMGP = ctypes.POINTER(GsrImage)
_lib = None


def load(path: Path | str | None = None):
    """Load libgsr.so once and declare every signature."""
    global _lib
    if _lib is not None:
        return _lib
    import os
    p = Path(path) if path else Path(os.environ.get("GSR_LIB_PATH", str(LIB_PATH)))
    if not p.exists():
        raise RuntimeError(f"libgsr.so not built ({p}); run __graft_entry__.build() or "
                           f"python -m paper_2501_06838_b200.build")
    lib = ctypes.CDLL(str(p))
    par = [_P, _P, _P, _P, _P]
    sig = {
        "gsr_version": ([], ctypes.c_char_p),
        "gsr_out_dims": ([_I32, _I32, _D, ctypes.POINTER(_I32), ctypes.POINTER(_I32)], None),
        "gsr_out_dims_v": ([_I32, _I32, _D, _D, ctypes.POINTER(_I32), ctypes.POINTER(_I32)],
                           None),
        "gsr_workspace_bytes_batched": ([_IMGP, _I32, _I64, _D], _SZ),
        "gsr_workspace_bytes": ([_I64, _I32, _I32, _D, _D], _SZ),
        "gsr_render_fwd": (par + [_I64, _I32, _I32, _D, _D, _P, _P, _SZ, _P], None),
        "gsr_render_bwd": (par + [_I64, _I32, _I32, _D, _D, _P, _P, _P, _P, _P, _P, _P, _SZ, _P],
                           None),
        "gsr_render_fwd_batched": (par + [_I64, _IMGP, _I32, _D, _P, _P, _SZ, _P], None),
        "gsr_render_bwd_batched": (par + [_I64, _IMGP, _I32, _D, _P, _P, _P, _P, _P, _P, _P, _SZ,
                                          _P], None),
        "gsr_render_bwd_moments_batched": (par + [_I64, _IMGP, _I32, _D, _P, _P, _P, _SZ, _P],
                                           None),
        "gsr_render_bwd_batched_ex": (par + [_I64, _IMGP, _I32, _D, _P, _P, _P, _P, _P, _P, _P,
                                             _SZ, ctypes.c_uint32, _P], None),
        "gsr_render_bwd_moments_batched_ex": (par + [_I64, _IMGP, _I32, _D, _P, _P, _P, _SZ,
                                                     ctypes.c_uint32, _P], None),
        "gsr_finalize_grads": (par + [_I64, _P, _P, _P, _P, _P, _P, _P], None),
        "gsr_finalize_grads_ex": (par + [_I64, _P, _P, _P, _P, _P, _P, ctypes.c_uint32, _P],
                                  None),
        "gsr_render_fwd_batched_ex": (par + [_I64, _IMGP, _I32, _D, _P, _P, _SZ, ctypes.c_uint32,
                                             _P], None),
        "gsr_train_workspace_bytes_batched": ([_IMGP, _I32, _I64, _D], _SZ),
        "gsr_train_step_l1_batched": ([_P] * 6 + [_I64, _IMGP, _I32, _D, ctypes.c_float, _D, _P,
                                                  _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P], None),
        "gsr_pair_count_batched": (par + [_I64, _IMGP, _I32, _D, _P, _P, _SZ, _P], None),
        "gsr_pair_count_batched_ex": (par + [_I64, _IMGP, _I32, _D, ctypes.c_uint32, _P, _P, _SZ,
                                             _P], None),
        "gsr_debug_rects": (par + [_I64, _I32, _I32, _D, _D, _P, _P], None),
        "gsr_debug_rects_ex": (par + [_I64, _I32, _I32, _D, _D, ctypes.c_uint32, _P, _P], None),
        "gsr_debug_tile_lists": (par + [_I64, _I32, _I32, _D, _D, _P, _P, _P, _P, _SZ, _P], None),
        "gsr_debug_fwd_tile_lists": (par + [_I64, _I32, _I32, _D, _D, _P, _P, _P, _P, _P, _P, _SZ,
                                            _P], None),
        "gsr_row_pair_counts_batched": (par + [_I64, _IMGP, _I32, _D, ctypes.c_uint32, _P, _P],
                                        None),
        "gsr_row_pair_counts_host": (par + [_I64, _IMGP, _I32, _D, ctypes.c_uint32, _P], None),
        "gsr_band_span_batched": (par + [_I64, _IMGP, _I32, _D, ctypes.c_uint32, _P, _I32, _I32,
                                         _P, _P], None),
        "gsr_band_span_host": (par + [_I64, _IMGP, _I32, _D, ctypes.c_uint32, _P, _I32, _I32, _P],
                               None),
        "gsr_workspace_bytes_subset": ([_IMGP, _I32, _I64, _I64, _D], _SZ),
        "gsr_render_fwd_subset": (par + [_I64, _P, _I64, _IMGP, _I32, _D, _P, _P, _SZ,
                                         ctypes.c_uint32, _P], None),
        "gsr_render_bwd_moments_subset": (par + [_I64, _P, _I64, _IMGP, _I32, _D, _P, _P, _P, _SZ,
                                                 ctypes.c_uint32, _P], None),
        "gsr_finalize_grads_subset": (par + [_I64, _P, _I64, _P, _P, _P, _P, _P, _P,
                                             ctypes.c_uint32, _P], None),
        "gsr_validate_params": (par + [_I64, ctypes.c_uint32, _P, _P], None),
        "gsr_rank_halo_workspace_bytes": ([_I64], _SZ),
        "gsr_rank_halo": (par + [_I64, _IMGP, _I32, _D, ctypes.c_uint32, _P, _I32, _I32, _I32,
                                 _P, _P, _P, _P, _P, _P, _P, _SZ, _P], None),
        "gsr_tile_shape": ([ctypes.POINTER(_I32)] * 4, "void"),
        "gsr_profile_enable": ([_I32], None),
        "gsr_profile_collect": ([_P, _P, _P, _I32], None),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:                 # an older build (A/B experiments): leave it undeclared
            continue
        fn.argtypes = args
        if res == "void":
            fn.restype = None
        elif res is not None:
            fn.restype = res
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status != GSR_OK:
        raise GsrError(f"{what} failed: {_ERR.get(status, status)}")


def images_array(imgs):
    """[(H, W, s, g_off, g_cnt, out_off, row_begin, row_end[, s_y]), ...] -> ctypes array
    (s_y = 0 or absent: isotropic scale s)."""
    arr = (GsrImage * len(imgs))()
    for k, t in enumerate(imgs):
        H, W, s, go, gc, oo, rb, re = t[:8]
        sy = t[8] if len(t) > 8 and t[8] is not None else 0.0
        arr[k] = GsrImage(int(H), int(W), float(s), int(go), int(gc), int(oo), int(rb), int(re),
                          float(sy))
    return arr


def out_dims(H: int, W: int, s: float, s_y: float | None = None):
    """(Hs, Ws) = (floor(s_y H), floor(s W)) (R4, R22; s_y None or 0: s_y = s)."""
    h, w = _I32(), _I32()
    lib = load()
    if getattr(lib, "gsr_out_dims_v", None) is None and not s_y:     # an older build (A/B runs)
        check(lib.gsr_out_dims(int(H), int(W), float(s), ctypes.byref(h), ctypes.byref(w)),
              "gsr_out_dims")
        return h.value, w.value
    check(lib.gsr_out_dims_v(int(H), int(W), float(s), float(s_y or 0.0), ctypes.byref(h),
                             ctypes.byref(w)), "gsr_out_dims_v")
    return h.value, w.value


def tile_shape():
    v = [_I32() for _ in range(4)]
    load().gsr_tile_shape(*[ctypes.byref(x) for x in v])
    return tuple(x.value for x in v)


PHASES = ("binning", "render_fwd", "render_bwd", "finalize")


def profile_enable(on: bool = True) -> None:
    check(load().gsr_profile_enable(1 if on else 0), "gsr_profile_enable")


def profile_collect(reset: bool = True):
    """-> ({phase: ms}, {phase: calls}, kernel_launches); synchronises the recorded events."""
    ms = (ctypes.c_double * 4)()
    calls = (ctypes.c_int64 * 4)()
    nl = ctypes.c_int64()
    check(load().gsr_profile_collect(ctypes.cast(ms, _P), ctypes.cast(calls, _P),
                                     ctypes.cast(ctypes.byref(nl), _P), 1 if reset else 0),
          "gsr_profile_collect")
    return dict(zip(PHASES, list(ms))), dict(zip(PHASES, list(calls))), nl.value


def version() -> str:
    return load().gsr_version().decode()
