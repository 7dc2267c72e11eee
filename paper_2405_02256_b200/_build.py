"""Build libeucalc.so in-tree with nvcc for sm_100a (no JIT cache, travels with gpurun).

Each .cu is compiled to an object in parallel, then linked into the shared library."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libeucalc.so")
LIB_CHECKED = os.path.join(HERE, "libeucalc_checked.so")  # device bounds checks (EU_DCHECK), tests only
LIB_DEV = os.path.join(HERE, "libeucalc_dev.so")  # development: K2 for 8-byte records / 32-bit outputs only (fast compile)
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OBJ = os.path.join(HERE, "build")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build(lib=LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "eucalc.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def _nvcc():
    return os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force: bool = False, verbose: bool = False, checked: bool = False, dev: bool = False) -> str:
    """Compile libeucalc.so (or, checked=True, libeucalc_checked.so with the device
    bounds checks of EU_DCHECK compiled in; objects in build/checked)."""
    lib = LIB_CHECKED if checked else LIB_DEV if dev else LIB
    obj_dir = os.path.join(OBJ, "checked") if checked else os.path.join(OBJ, "dev") if dev else OBJ
    extra = ["-DEUCALC_DEVICE_CHECKS"] if checked else ["-DEUCALC_DEV_FAST"] if dev else []
    if dev:  # experiment switches for development builds, e.g. EUCALC_DEV_DEFS="-DEXP_X=1"
        extra += os.environ.get("EUCALC_DEV_DEFS", "").split()
    if not force and not needs_build(lib):
        return lib
    os.makedirs(obj_dir, exist_ok=True)

    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "eucalc.h")]

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        if not force and os.path.exists(obj):  # object newer than its source and every header: reuse
            t = os.path.getmtime(obj)
            if all(os.path.getmtime(p) < t for p in [src, *headers]):
                return obj, subprocess.CompletedProcess([], 0, "", "")
        r = subprocess.run([_nvcc(), *NVCC_FLAGS, *extra, "-I", INCLUDE, "-c", "-o", obj, src], capture_output=True,
                           text=True)
        return obj, r

    with ThreadPoolExecutor(len(sources())) as ex:
        results = list(ex.map(compile_one, sources()))
    logs = []
    for obj, r in results:
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    r = subprocess.run([_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib + ".tmp",
                        *[o for o, _ in results]], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    if verbose:
        print("\n".join(logs))
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    import sys

    print(build(force="--no-force" not in sys.argv, verbose=True, checked="--checked" in sys.argv,
                dev="--dev" in sys.argv))
