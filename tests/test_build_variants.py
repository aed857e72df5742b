"""Build matrix of the kernels' compile-time knobs: every alternative the
A/B measurements used still compiles for sm_100a (the shipped defaults are built and tested by
every other test). CPU only: nvcc cross-compiles, nothing runs."""
import os
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2501_06838_b200" / "csrc"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

VARIANTS = [
    ("render_fwd.cu", ["-DGSR_FWD_SPLIT=0", "-DGSR_CELL_REACH=0", "-DGSR_BOUNDS_CHECK", "-DGSR_FWD_HALVES=0",
                       "-DGSR_FWD_CUTMASK=0", "-DGSR_FWD_SCAN_D=3", "-DGSR_FWD_SMALL_STRIP=8",
                       "-DGSR_FWD_WARPS_LARGE=4", "-DGSR_FWD_WARPS_SMALL=2"]),
    ("render_bwd.cu", ["-DGSR_BWD_UNROLL=4", "-DGSR_BWD_UNROLL_MASKED=8", "-DGSR_BWD_KQ=8", "-DGSR_BWD_CTASORT=0",
                       "-DGSR_BWD_BATCH=256", "-DGSR_BWD_SCAN_U=2", "-DGSR_BWD_MACC_T=double"]),
    ("gsr_abi.cu", ["-DGSR_SCHED_DENSE=0"]),
]


@pytest.mark.skipif(not (Path(NVCC).exists() or shutil.which("nvcc")), reason="nvcc not found")
@pytest.mark.parametrize("src,flags", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_variant_compiles(src, flags, tmp_path):
    nvcc = NVCC if Path(NVCC).exists() else shutil.which("nvcc")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
           "--expt-relaxed-constexpr", "-I", str(ROOT / "include"), *flags, "-c",
           str(CSRC / src), "-o", str(tmp_path / (src + ".o"))]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
