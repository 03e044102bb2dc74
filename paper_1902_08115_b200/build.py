"""Builds libpbgpu.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Every CUDA/C++ source under csrc/ is compiled by its own nvcc process (in
parallel, objects cached under _obj/ and rebuilt when the source or any header
changes) with -gencode arch=compute_100a,code=sm_100a -lineinfo, then linked
into paper_1902_08115_b200/libpbgpu.so (cudart static), which travels with the
repo snapshot to the GPU box.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SO = os.path.join(PKG, "libpbgpu.so")
OBJ = os.path.join(PKG, "_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cpp")))


def headers() -> list[str]:
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + glob.glob(os.path.join(PKG, "csrc", "*.h"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(f) <= t for f in sources() + headers() + [__file__])


def _compile(src: str, verbose: bool) -> tuple[str, subprocess.CompletedProcess | None]:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    newest_dep = max(os.path.getmtime(f) for f in [src, *headers(), __file__])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep and not verbose:
        return obj, None
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc"),
           "-Xptxas", "-v" if verbose else "-O3", "-c", "-o", obj + ".tmp", src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode == 0:
        os.replace(obj + ".tmp", obj)
    return obj, r


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return SO
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(f)
    with ThreadPoolExecutor(max_workers=max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
        res = list(ex.map(lambda f: _compile(f, verbose), sources()))
    failed = [r for _, r in res if r is not None and r.returncode != 0]
    for r in res:
        if r[1] is not None and (verbose or r[1].returncode != 0):
            sys.stderr.write(r[1].stdout + r[1].stderr)
    if failed:
        raise RuntimeError("nvcc build of libpbgpu.so failed")
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", SO + ".tmp", *[o for o, _ in res], "-lpthread"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libpbgpu.so failed")
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
