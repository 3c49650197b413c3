"""Build the in-tree CUDA library libstk.so for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libstk.so")
ROOT = os.path.dirname(HERE)


def nccl_dir() -> str | None:
    try:
        import nvidia.nccl as m  # torch-bundled NCCL (2.28.x)
        d = list(m.__path__)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    except Exception:
        pass
    return None


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))] + [
        os.path.join(ROOT, "include", "stk.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3",
           "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v" if verbose else "-O3",
           "-o", LIB, os.path.join(CSRC, "stk.cu")]
    nd = nccl_dir()
    if nd:
        cmd += ["-DSTK_HAVE_NCCL=1", "-I" + os.path.join(nd, "include"),
                "-L" + os.path.join(nd, "lib"), "-l:libnccl.so.2",
                "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    else:
        cmd += ["-DSTK_HAVE_NCCL=0"]
    extra = os.environ.get("STK_EXTRA_FLAGS", "").split()   # experiments: -D switches
    cmd += extra
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libstk.so")
    if verbose:
        sys.stderr.write(r.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
