"""Builds libautx.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libautx.so")
SOURCES = ["autx_api.cu", "sched_kernels.cu", "swap_kernels.cu", "radix_kernels.cu"]
HEADERS = ["autx_internal.cuh", "block_prims.cuh", "idmap.h", os.path.join("..", "..", "include", "autx.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dirs():
    """NCCL headers and library: the wheel torch itself loads (one libnccl.so.2 per process),
    else the system copy."""
    try:
        import nvidia.nccl as nn
        root = list(nn.__path__)[0]
        inc, lib = os.path.join(root, "include"), os.path.join(root, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    except ImportError:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


NCCL_INC, NCCL_LIB = _nccl_dirs()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "-shared", "-Xptxas", "-v"]


def _extra():
    return os.environ.get("AUTX_NVCC_FLAGS", "").split()  # e.g. -DAUTX_PHASE_SYNC (profiling)


def stale():
    if not os.path.exists(LIB):
        return True
    try:
        if open(LIB + ".flags").read() != " ".join(_extra()):  # built with other extra flags
            return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    extra = _extra()
    cmd = [NVCC, *FLAGS, *extra, "-I", NCCL_INC, "-o", LIB + ".tmp", *[os.path.join(CSRC, f) for f in SOURCES],
           "-L", NCCL_LIB, "-l:libnccl.so.2", "-Xlinker", "-rpath," + NCCL_LIB]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libautx.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    with open(LIB + ".flags", "w") as f:
        f.write(" ".join(extra))
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
