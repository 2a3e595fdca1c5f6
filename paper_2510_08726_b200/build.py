"""Build the sm_100a shared libraries in-tree (no JIT cache, no torch types).

* ``paper_2510_08726_b200/libattn.so`` -- the C-ABI library (include/attn.h)
* ``datagen/libdatagen.so``           -- the device twin of the input generator

Every CUDA source is compiled with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo`` (cross-compiles without a GPU).  Objects are cached under
``build/`` and rebuilt when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2510_08726_b200")
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-diag-suppress", "177"]

LIBS = {
    os.path.join(PKG, "libattn.so"): {
        "sources": [os.path.join(CSRC, f) for f in ("api.cu", "fwd_tc.cu", "fwd_simt.cu", "decode.cu", "softmax_rows.cu")],
        "headers": [os.path.join(CSRC, f) for f in ("ptx.cuh", "kernels.h")] + [os.path.join(ROOT, "include", "attn.h")],
        "link": ["-ldl"],   # NCCL is dlopen'ed (multi-GPU decode), never linked
    },
    os.path.join(ROOT, "datagen", "libdatagen.so"): {
        "sources": [os.path.join(ROOT, "datagen", "gen.cu")],
        "headers": [],
    },
}


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"command failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(verbose: bool = False, extra_flags=()) -> list[str]:
    os.makedirs(BUILD, exist_ok=True)
    built = []
    for lib, spec in LIBS.items():
        objs, jobs = [], []
        for src in spec["sources"]:
            obj = os.path.join(BUILD, os.path.basename(os.path.dirname(src)) + "_" + os.path.basename(src) + ".o")
            objs.append(obj)
            if _stale(obj, [src] + spec["headers"]):
                cmd = [NVCC, *ARCH, *FLAGS, *extra_flags, "-c", src, "-o", obj]
                if verbose:
                    cmd.insert(1, "-Xptxas=-v")
                jobs.append(cmd)
        with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
            for log in ex.map(_run, jobs):
                if verbose and log:
                    sys.stderr.write(log)
        if jobs or _stale(lib, objs):
            _run([NVCC, *ARCH, "-shared", "-o", lib, *objs, *spec.get("link", [])])
        built.append(lib)
    return built


if __name__ == "__main__":
    for p in build(verbose="-v" in sys.argv):
        print(p)
