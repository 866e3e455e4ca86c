"""Build libholo.so in-tree with nvcc for sm_100a (B200).

``python -m paper_2004_04049_b200.build`` or ``build()``; no GPU needed (nvcc
cross-compiles).  The .so is git-ignored but travels to the GPU box with the
repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libholo.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
]
TUS = ["runtime.cu", "lut.cu", "ospr.cu", "gs.cu", "hooks.cu", "stream.cu"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(ROOT, "include", "holo.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra=()) -> str:
    """Compile every translation unit and link libholo.so (``out``; ``extra`` nvcc flags are
    for experiment variants built next to the product library, e.g. -DHOLO_GS_NORM=0)."""
    if not force and not extra and out == LIB and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(HERE, "build" if out == LIB else "build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    log = os.path.join(HERE, "build.log" if out == LIB else os.path.basename(out) + ".build.log")

    def compile_one(tu):
        obj = os.path.join(objdir, tu.replace(".cu", ".o"))
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, tu), "-o", obj]
        return cmd, subprocess.run(cmd, capture_output=True, text=True), obj

    with ThreadPoolExecutor(max_workers=len(TUS)) as ex:
        results = list(ex.map(compile_one, TUS))
    with open(log, "w") as f:
        for cmd, res, _ in results:
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr + "\n")
    for cmd, res, _ in results:
        if res.returncode != 0:
            sys.stderr.write(res.stderr[-8000:])
            raise RuntimeError(f"nvcc failed (see {log})")
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
           *[obj for _, _, obj in results], "-o", tmp, "-cudart", "static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-8000:])
        raise RuntimeError("nvcc link failed")
    if verbose:
        for _, r, _ in results:
            sys.stderr.write(r.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    a = sys.argv[1:]
    o = a[a.index("--out") + 1] if "--out" in a else LIB
    ex = [x for x in a if x.startswith("-D")]
    print(build(force="--force" in a, verbose="-v" in a, out=os.path.abspath(o), extra=ex))
