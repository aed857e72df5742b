"""The C-ABI driven from plain C (tests/c/abi_check.c): no Python binding, no PyTorch in the
process. CPU: version, sizes, workspace, host-checked errors. GPU: gsr_render_fwd/bwd on
cudaMalloc'd buffers vs the float64 C oracle linked into the test program."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CUDA_LIB = Path("/usr/local/cuda/lib64")


@pytest.fixture(scope="module")
def abi_check(tmp_path_factory):
    from paper_2501_06838_b200 import _lib
    if not _lib.LIB_PATH.exists():
        from paper_2501_06838_b200.build import build
        build()
    if shutil.which("gcc") is None or not (CUDA_LIB / "libcudart.so").exists():
        pytest.skip("gcc or libcudart not available")
    exe = tmp_path_factory.mktemp("cabi") / "abi_check"
    libdir = str(_lib.LIB_PATH.parent)
    cmd = ["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
           "-o", str(exe), str(ROOT / "tests/c/abi_check.c"), str(ROOT / "oracle/gsr_oracle.c"),
           f"-L{libdir}", "-l:libgsr.so", f"-Wl,-rpath,{libdir}", f"-L{CUDA_LIB}", "-lcudart",
           f"-Wl,-rpath,{CUDA_LIB}", "-lm"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_abi_host_side(abi_check):
    r = subprocess.run([str(abi_check)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "abi_check: ok" in r.stdout


@pytest.mark.gpu
def test_c_abi_render_parity(abi_check):
    r = subprocess.run([str(abi_check), "gpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "forward max-abs error" in r.stdout and "abi_check: ok" in r.stdout
