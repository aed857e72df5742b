"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/gsr.h declares,
and rejects host-checkable bad arguments with GSR_EINVAL before launching anything."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2501_06838_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2501_06838_b200.build import build
    build()
    return _lib.load()


def declared_symbols():
    text = (ROOT / "include" / "gsr.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gsr_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_api():
    decl = declared_symbols()
    assert set(decl) == set(_lib.EXPORTS), set(decl) ^ set(_lib.EXPORTS)
    for name in ("gsr_render_fwd", "gsr_render_bwd"):   # north_star names
        assert name in decl


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    import subprocess
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                        text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", nm), name


def test_version_and_tile_shape(lib):
    assert "sm_100a" in _lib.version()
    tw, th, cw, ch = _lib.tile_shape()
    assert tw > 0 and th > 0 and cw > 0 and ch > 0


@pytest.mark.parametrize("H,W,s", [(48, 48, 4.0), (339, 510, 4.0), (45, 68, 30.0), (170, 255, 8.0),
                                   (48, 48, 1.0), (48, 48, 3.9), (7, 3, 1.5), (10, 7, 2.5)])
def test_out_dims_matches_oracle(lib, H, W, s):
    assert _lib.out_dims(H, W, s) == O.out_dims(H, W, s)


def test_out_dims_rejects(lib):
    h, w = ctypes.c_int32(), ctypes.c_int32()
    for args in [(0, 4, 2.0), (4, 0, 2.0), (4, 4, 0.5), (4, 4, float("nan")),
                 (4, 4, float("inf")), (40000, 4, 2.0)]:
        assert lib.gsr_out_dims(*args, ctypes.byref(h), ctypes.byref(w)) == _lib.GSR_EINVAL


def test_workspace_bytes(lib):
    b = lib.gsr_workspace_bytes(36864, 48, 48, 4.0, 0.1)
    assert b > 36864 * 48
    assert lib.gsr_workspace_bytes(0, 48, 48, 4.0, 0.1) > 0
    assert lib.gsr_workspace_bytes(10, 48, 48, 4.0, 0.0) == 0      # bad ratio
    assert lib.gsr_workspace_bytes(10, 48, 48, 4.0, 1.5) == 0
    assert lib.gsr_workspace_bytes(10, 48, 48, 0.9, 0.1) == 0      # s < 1
    assert lib.gsr_workspace_bytes(-1, 48, 48, 2.0, 0.1) == 0


def test_einval_before_any_launch(lib):
    """Host-checkable errors return GSR_EINVAL / GSR_EWORKSPACE without touching the GPU (this
    runs in a container with no GPU)."""
    P = ctypes.c_void_p
    dummy = P(16)
    ps = [dummy] * 5
    # bad dims / scale / ratio
    assert lib.gsr_render_fwd(*ps, 10, 0, 4, 2.0, 0.1, dummy, dummy, 1 << 30, None) == 1
    assert lib.gsr_render_fwd(*ps, 10, 4, 4, 0.5, 0.1, dummy, dummy, 1 << 30, None) == 1
    assert lib.gsr_render_fwd(*ps, 10, 4, 4, 2.0, 0.0, dummy, dummy, 1 << 30, None) == 1
    assert lib.gsr_render_fwd(*ps, -1, 4, 4, 2.0, 0.1, dummy, dummy, 1 << 30, None) == 1
    # null parameter with n > 0
    assert lib.gsr_render_fwd(None, *ps[1:], 10, 4, 4, 2.0, 0.1, dummy, dummy, 1 << 30,
                              None) == 1
    # null output
    assert lib.gsr_render_fwd(*ps, 10, 4, 4, 2.0, 0.1, None, dummy, 1 << 30, None) == 1
    # workspace too small
    assert lib.gsr_render_fwd(*ps, 10, 4, 4, 2.0, 0.1, dummy, dummy, 16, None) == 2
    assert lib.gsr_render_bwd(*ps, 10, 4, 4, 2.0, 0.1, dummy, *ps, dummy, 16, None) == 2
    assert lib.gsr_render_bwd(*ps, 10, 4, 4, 2.0, 0.1, None, *ps, dummy, 1 << 30, None) == 1
    # batched: overlapping / unsorted Gaussian ranges, too many images, bad band
    imgs = _lib.images_array([(4, 4, 2.0, 0, 6, 0, 0, -1), (4, 4, 2.0, 5, 5, 0, 0, -1)])
    assert lib.gsr_render_fwd_batched(*ps, 10, imgs, 2, 0.1, dummy, dummy, 1 << 30, None) == 1
    imgs = _lib.images_array([(4, 4, 2.0, 0, 20, 0, 0, -1)])
    assert lib.gsr_render_fwd_batched(*ps, 10, imgs, 1, 0.1, dummy, dummy, 1 << 30, None) == 1
    imgs = _lib.images_array([(4, 4, 2.0, 0, 5, 0, 3, 2)])
    assert lib.gsr_render_fwd_batched(*ps, 10, imgs, 1, 0.1, dummy, dummy, 1 << 30, None) == 1
    imgs = _lib.images_array([(4, 4, 2.0, 0, 5, 0, 0, 9)])
    assert lib.gsr_render_fwd_batched(*ps, 10, imgs, 1, 0.1, dummy, dummy, 1 << 30, None) == 1
    # scale vector (R22): scale_y in (0, 1) or non-finite is invalid; the band is checked
    # against Hs = floor(scale_y H)
    for sy in (0.5, float("nan"), float("inf"), -2.0):
        imgs = _lib.images_array([(4, 4, 2.0, 0, 5, 0, 0, -1, sy)])
        assert lib.gsr_render_fwd_batched(*ps, 10, imgs, 1, 0.1, dummy, dummy, 1 << 30,
                                          None) == 1, sy
        assert lib.gsr_workspace_bytes_batched(imgs, 1, 10, 0.1) == 0, sy
    imgs = _lib.images_array([(4, 4, 2.0, 0, 5, 0, 0, 13, 3.0)])
    assert lib.gsr_render_fwd_batched(*ps, 10, imgs, 1, 0.1, dummy, dummy, 1 << 30, None) == 1
    assert lib.gsr_workspace_bytes_batched(_lib.images_array([(4, 4, 2.0, 0, 5, 0, 0, 12, 3.0)]),
                                           1, 10, 0.1) > 0
    # data-format flags (NEXT-4): unknown bits and flags an entry point does not take
    imgs = _lib.images_array([(4, 4, 2.0, 0, 5, 0, 0, -1)])
    for fl in (_lib.GSR_REUSE_BINNING, _lib.GSR_SUPPORT, 0x40, 0x80000000):
        assert lib.gsr_render_fwd_batched_ex(*ps, 10, imgs, 1, 0.1, dummy, dummy, 1 << 30, fl,
                                             None) == 1, fl
    for fl in (_lib.GSR_SUPPORT, 0x40):
        assert lib.gsr_render_bwd_batched_ex(*ps, 10, imgs, 1, 0.1, dummy, *ps, dummy, 1 << 30,
                                             fl, None) == 1, fl
    for fl in (_lib.GSR_OUT_BF16, _lib.GSR_OUT_CHW, _lib.GSR_REUSE_BINNING):
        assert lib.gsr_finalize_grads_ex(*ps, 10, dummy, *ps, fl, None) == 1, fl
    assert lib.gsr_render_fwd_batched_ex(*ps, 10, imgs, 1, 0.1, None, dummy, 1 << 30,
                                         _lib.GSR_OUT_BF16, None) == 1
    many = _lib.images_array([(4, 4, 2.0, 0, 0, 0, 0, -1)] * 65)
    assert lib.gsr_render_fwd_batched(*ps, 10, many, 65, 0.1, dummy, dummy, 1 << 30, None) == 1
    assert lib.gsr_finalize_grads(*ps, -1, dummy, *ps, None) == 1


def test_product_path_does_not_import_oracle():
    """The product package never references oracle/ (independence of the two sides)."""
    pkg = ROOT / "paper_2501_06838_b200"
    for f in pkg.rglob("*.py"):
        txt = f.read_text()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
        assert "liboracle" not in txt and "gsr_oracle" not in txt, f
    for f in list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        assert "gsr_oracle" not in f.read_text(), f
