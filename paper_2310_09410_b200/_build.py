"""Build liblopf.so in-tree for sm_100a (nvcc; host C++ + CUDA in one shared library)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "liblopf.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("setup.cpp", "partition.cpp", "pack.cpp", "pack_resident.cpp", "pack_batch.cpp", "api.cpp", "kernels.cu",
                                                  "resident.cu", "batch.cu")]
HEADERS = [os.path.join(HERE, "csrc", "internal.h"), os.path.join(HERE, "csrc", "device.cuh"), os.path.join(ROOT, "include", "lopf.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS + [__file__])


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile liblopf.so; `out` / `defines` build A/B variants (e.g. defines=["LOPF_BFIRST=1"])."""
    so = out or SO
    if not force and out is None and not _stale():
        return SO
    tmp = so + f".tmp{os.getpid()}"
    cmd = [NVCC, *[f"-D{d}" for d in defines], "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-O3,-Wall",
           "-shared", "-cudart", "static", "-I", os.path.join(ROOT, "include"), "-o", tmp, *SOURCES, "-lpthread", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building liblopf.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, so)
    if out is None:
        with open(os.path.join(HERE, "ptxas_report.txt"), "w") as fh:
            fh.write(res.stderr)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
