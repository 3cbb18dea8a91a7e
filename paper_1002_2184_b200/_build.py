"""Builds the in-tree C-ABI library libfhwt.so for sm_100a with nvcc (no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["fhwt_api.cu", "haar2d.cu", "haar2d_ana.cu", "haar2d_syn.cu", "haar2d_small.cu", "haar1d.cu", "direct.cu", "lowpass.cu"]
LIB = os.path.join(HERE, "libfhwt.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # IEEE per-operation rounding (R10): no a*b+c contraction across butterfly levels
    # ((x0+x1)*s + (x2+x3)*s would otherwise fuse), so every kernel path rounds identically.
    "-fmad=false",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr", "-diag-suppress", "128",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "fhwt.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile the library.  Several processes (torchrun ranks) may call this at once: the
    build-and-replace runs under an exclusive file lock, each build writes its own per-process
    temporary file, and a process that waited for the lock re-checks staleness instead of
    rebuilding, so no rank can load a half-written library."""
    import fcntl
    lib = out or LIB
    if not force and out is None and not stale():
        return LIB
    with open(lib + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if not force and out is None and not stale():   # another process built it meanwhile
                return LIB
            import tempfile
            from concurrent.futures import ThreadPoolExecutor
            tmp = f"{lib}.{os.getpid()}.tmp"
            with tempfile.TemporaryDirectory(prefix="fhwt_build_") as od:
                # one nvcc per translation unit, in parallel, then one link step
                def compile_one(src):
                    obj = os.path.join(od, os.path.splitext(src)[0] + ".o")
                    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
                           "-c", os.path.join(CSRC, src), "-o", obj]
                    return obj, subprocess.run(cmd, capture_output=True, text=True)

                with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
                    results = list(ex.map(compile_one, SOURCES))
                logs = "".join(r.stdout + r.stderr for _, r in results)
                res = None
                if all(r.returncode == 0 for _, r in results):
                    res = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                                          *[o for o, _ in results], "-o", tmp],
                                         capture_output=True, text=True)
                    logs += res.stdout + res.stderr
                if res is None or res.returncode != 0:
                    sys.stderr.write(logs)
                    if os.path.exists(tmp):
                        os.unlink(tmp)
                    raise RuntimeError("nvcc failed building libfhwt.so")
            if verbose:
                sys.stderr.write(logs)
            os.replace(tmp, lib)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
