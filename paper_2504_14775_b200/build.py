"""Build libgllm.so (sm_100a) in-tree with nvcc.

    python -m paper_2504_14775_b200.build [--force] [-v]
    python -m paper_2504_14775_b200.build --define GLLM_TRACE --out old_lib/libgllm_trace.so   # debug variant

The shared library links the CUDA runtime statically and resolves the driver
API (cuTensorMapEncodeTiled) at run time, so it loads on a CPU-only host (the
symbol-export tests) and on the B200 box alike.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgllm.so")
SOURCES = ["gemm.cu", "gemm_swab.cu", "gemm_skinny.cu", "kernels.cu", "attention.cu", "stage.cu"]
HEADERS = ["common.cuh", "gllm_internal.h"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def flags() -> list[str]:
    return ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
            "-I", os.path.join(ROOT, "include"), "-DNDEBUG"]


def _digest(extra: list[str]) -> str:
    h = hashlib.sha256()
    for name in SOURCES + HEADERS:
        with open(os.path.join(CSRC, name), "rb") as fh:
            h.update(fh.read())
    with open(os.path.join(ROOT, "include", "gllm.h"), "rb") as fh:
        h.update(fh.read())
    h.update(" ".join(flags() + extra).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, defines: tuple[str, ...] = (), out: str | None = None) -> str:
    """Build the library; `defines` / `out` make a debug variant (e.g. GLLM_TRACE) at another path."""
    lib = os.path.abspath(out) if out else LIB
    extra = [f"-D{d}" for d in defines]
    stamp = lib + ".sha256"
    dg = _digest(extra)
    if not force and os.path.exists(lib) and os.path.exists(stamp) and open(stamp).read().strip() == dg:
        return lib
    objdir = os.path.join(PKG, "build" if not defines else "build_" + "_".join(defines).lower())
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for name in SOURCES:
        obj = os.path.join(objdir, name.replace(".cu", ".o"))
        cmd = [nvcc(), *flags(), *extra, "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, name), "-o", obj]
        procs.append((name, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = []
    for name, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        if p.returncode != 0:
            failed.append(name)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    # Export only the C-ABI (gllm_*) symbols.
    vscript = os.path.join(objdir, "exports.map")
    with open(vscript, "w") as fh:
        fh.write("{ global: gllm_*; local: *; };\n")
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib + ".tmp",
            "-Xlinker", f"--version-script={vscript}", "-cudart", "static"]
    subprocess.run(link, check=True)
    os.replace(lib + ".tmp", lib)
    with open(stamp, "w") as fh:
        fh.write(dg + "\n")
    return lib


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--define", action="append", default=[])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, defines=tuple(a.define), out=a.out))
