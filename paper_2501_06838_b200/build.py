"""Build libgsr.so (sm_100a) in-tree with nvcc. Called by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libgsr.so"
ROOT = PKG.parent
SOURCES = ["binning.cu", "render_fwd.cu", "render_bwd.cu", "train.cu", "plan.cu", "gsr_abi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# host code: no FMA contraction (the K7 planner evaluates the fp64 rect formulas of reading R2 on
# the CPU with the same operation order as the kernels' explicit __dmul_rn/__dadd_rn)
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
         "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
# experiments only (A/B builds into another directory): extra -D flags
EXTRA = os.environ.get("GSR_NVCC_EXTRA", "").split()


def _stale(out: Path, deps) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          objdir: Path | None = None) -> Path:
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "gsr.h"]
    lib = Path(out) if out else LIB
    objdir = Path(objdir) if objdir else PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = objdir / (src + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers]):
            cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", str(s), "-o", str(o)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            log = objdir / (src + ".ptxas.txt")
            log.write_text(r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {src}")
            if verbose:
                sys.stderr.write(r.stderr)
    if force or _stale(lib, objs):
        tmp = lib.with_suffix(".so.tmp%d" % os.getpid())
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
        subprocess.check_call(cmd)
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [--out path.so --objdir dir]  (GSR_NVCC_EXTRA="-D..." for A/B)
    a = sys.argv
    out = a[a.index("--out") + 1] if "--out" in a else None
    od = a[a.index("--objdir") + 1] if "--objdir" in a else None
    print(build(force="--force" in a, verbose=True, out=out, objdir=od))
