"""Build liblopf.so in-tree for sm_100a (nvcc; host C++ + CUDA in one shared library).

Every source compiles to its own object (in parallel, under build/<variant>/), then one nvcc link;
`force` recompiles everything, otherwise an object is rebuilt when its source or a header is newer."""
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

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
    tag = hashlib.sha1(" ".join(sorted(defines)).encode()).hexdigest()[:10] if defines else "default"
    objdir = os.path.join(ROOT, "build", tag)
    os.makedirs(objdir, exist_ok=True)
    flags = [*[f"-D{d}" for d in defines], "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v", "-Xcompiler",
             "-fPIC,-O3,-Wall", "-I", os.path.join(ROOT, "include")]
    hdr_t = max(os.path.getmtime(p) for p in HEADERS + [__file__])

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(hdr_t, os.path.getmtime(src)):
            return obj, None
        res = subprocess.run([NVCC, *flags, "-c", src, "-o", obj + ".tmp"], capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed compiling {os.path.basename(src)}")
        os.replace(obj + ".tmp", obj)
        return obj, res.stderr

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        done = list(ex.map(compile_one, SOURCES))
    tmp = so + f".tmp{os.getpid()}"
    res = subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *[o for o, _ in done], "-lpthread", "-ldl"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking liblopf.so")
    report = "".join(r for _, r in done if r)
    if verbose:
        sys.stderr.write(report)
    os.replace(tmp, so)
    if out is None and report:
        # ptxas lines of the objects rebuilt now; the others keep their previous entries
        path = os.path.join(HERE, "ptxas_report.txt")
        old = open(path).read() if os.path.exists(path) else ""
        rebuilt = {os.path.basename(s) for s, (_, r) in zip(SOURCES, done) if r}
        names = {os.path.basename(s) for s in SOURCES}
        keep = [blk for blk in old.split("\n### ") if blk and blk.split("\n", 1)[0].strip("# ") in names - rebuilt]
        new = [f"{os.path.basename(s)}\n{r}" for s, (_, r) in zip(SOURCES, done) if r]
        with open(path, "w") as fh:
            fh.write("".join("### " + b.lstrip("# ") + ("\n" if not b.endswith("\n") else "") for b in keep + new))
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
