"""Build libsdnn.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2004_10908_b200.build        # or __graft_entry__.build()
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
# SDNN_LIB / SDNN_NVCC_FLAGS: an alternative in-tree build (A/B experiments,
# e.g. SDNN_LIB=.../libsdnn_b.so SDNN_NVCC_FLAGS=-DSDNN_CLAMP3); the binding
# loads the same SDNN_LIB path
SO = os.environ.get("SDNN_LIB") or os.path.join(HERE, "libsdnn.so")
EXTRA = os.environ.get("SDNN_NVCC_FLAGS", "").split()
SOURCES = ["api.cu", "kernels.cu", "pass_wide.cu", "resident.cu", "pack.cpp", "fuse.cpp"]
HEADERS = ["sdnn_internal.h", "device_util.cuh", os.path.join("..", "..", "include", "sdnn.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-pthread",
         "-Xptxas", "-O3", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = SO + ".%d.tmp" % os.getpid()
    cmd = [nvcc, *ARCH, *FLAGS, *EXTRA, "-shared", "-I", os.path.join(ROOT, "include"),
           *[os.path.join(CSRC, f) for f in SOURCES], "-o", tmp, "-lpthread"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
