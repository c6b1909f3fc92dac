"""Builds libpolar_torch_ops.so (torch_ops.cpp: the C-ABI as torch.ops.polar.*)
in-tree against the installed torch, linked to libpolarcuda.so through
$ORIGIN.  Run by __graft_entry__.build() after the CUDA library."""

import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent
OUT = PKG / "libpolar_torch_ops.so"


def build(force: bool = False) -> Path:
    src = HERE / "torch_ops.cpp"
    lib = PKG / "libpolarcuda.so"
    hdr = PKG.parent / "include" / "polarcuda.h"
    if not force and OUT.exists() and all(OUT.stat().st_mtime >= p.stat().st_mtime for p in (src, lib, hdr)):
        return OUT
    import torch
    from torch.utils.cpp_extension import CUDA_HOME, include_paths, library_paths

    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", str(src), "-o", str(OUT),
           f"-D_GLIBCXX_USE_CXX11_ABI={abi}", f"-I{PKG.parent / 'include'}", f"-I{CUDA_HOME}/include"]
    cmd += [f"-I{p}" for p in include_paths()]
    cmd += [f"-L{p}" for p in library_paths()] + [f"-Wl,-rpath,{p}" for p in library_paths()]
    cmd += ["-ltorch", "-ltorch_cpu", "-lc10", "-lc10_cuda", "-ltorch_cuda",
            f"-L{PKG}", "-l:libpolarcuda.so", "-Wl,-rpath,$ORIGIN"]
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force=len(sys.argv) > 1 and sys.argv[1] == "--force"))
