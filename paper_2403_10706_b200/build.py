"""Build libhysco.so in-tree for sm_100a (nvcc; no JIT, no torch extension)."""
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "hysco_api.cu")
SRC_IO = os.path.join(PKG, "csrc", "hysco_io.cu")
DEPS = [os.path.join(PKG, "csrc", f) for f in sorted(os.listdir(os.path.join(PKG, "csrc")))] + \
       [os.path.join(ROOT, "include", "hysco.h"), os.path.join(ROOT, "include", "hysco_io.h"),
        os.path.abspath(__file__)]
LIB = os.path.join(PKG, "libhysco.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-shared",
         "-I" + os.path.join(ROOT, "include")]


def nccl_dirs():
    """torch's bundled NCCL (include, lib): libhysco links the same libnccl.so.2
    torch loads, so the process holds one NCCL whichever library loads first.
    Falls back to the system NCCL when the wheel is absent."""
    try:
        import nvidia.nccl as nn
        base = list(nn.__path__)[0]
        inc, libd = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(libd, "libnccl.so.2")) and os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, libd
    except Exception:
        pass
    return None, None


def cufft_dir():
    """torch's bundled cuFFT (one libcufft.so.11 in the process, like NCCL)."""
    try:
        import nvidia.cufft as nf
        d = os.path.join(list(nf.__path__)[0], "lib")
        if os.path.exists(os.path.join(d, "libcufft.so.11")):
            return d
    except Exception:
        pass
    return None


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force=False, verbose=False):
    """Compile csrc/ into paper_2403_10706_b200/libhysco.so; returns the path."""
    if force or needs_build():
        inc, libd = nccl_dirs()
        nccl = ["-I" + inc, "-L" + libd, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libd] if inc else ["-lnccl"]
        fdir = cufft_dir()
        cufft = ["-L" + fdir, "-l:libcufft.so.11", "-Xlinker", "-rpath=" + fdir] if fdir else ["-lcufft"]
        extra = os.environ.get("HYSCO_NVCC_EXTRA", "").split()   # diagnostic variants (tools/ab_bench.sh)
        cmd = [NVCC] + FLAGS + extra + ["-o", LIB + ".tmp", SRC, SRC_IO] + nccl + cufft + ["-lz"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
