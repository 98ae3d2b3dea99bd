"""Build librelay_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2402_14808_b200.build      (or __graft_entry__.build())

The shared library is the C-ABI declared in include/relay_b200.h.  It is
built in the package directory (git-ignored, but it travels to the GPU box
with the gpurun snapshot), never into a JIT cache.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "librelay_b200.so")
DIAG_LIB = os.path.join(PKG, "librelay_b200_diag.so")  # -DRB_DIAG=1: timestamp stamps
# diagnostics: RB_VARIANT="name:-DFOO=1 -DBAR=2" builds librelay_b200_<name>.so
# with extra defines (select it at run time with RB_LIB=<path>)
_VARIANT = os.environ.get("RB_VARIANT", "")
SOURCES = ["sys_attn_sm100.cu", "sys_gqa_sm100.cu", "sys_gqa2_sm100.cu", "ctx_attn.cu",
           "rope_append.cu", "capi.cu"]
HEADERS = ["rb_common.cuh", "rb_plan.h", "rb_args.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "relay_b200.h"))
    deps.append(os.path.join(ROOT, "include", "relay_b200_diag.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False):
    if _VARIANT:
        name, defs = _VARIANT.split(":", 1)
        return _build_to(os.path.join(PKG, f"librelay_b200_{name}.so"), defs.split(),
                         os.path.join(PKG, "build", name), verbose)
    if not force and not _stale():
        return LIB
    # the diagnostics build (per-CTA timestamps, profiles/diag_*.py) first:
    # the staleness check keys on the production library's mtime
    _build_to(DIAG_LIB, ["-DRB_DIAG=1"], os.path.join(PKG, "build", "diag"), verbose)
    return _build_to(LIB, [], os.path.join(PKG, "build"), verbose)


def _build_to(lib, defs, objdir, verbose):
    os.makedirs(objdir, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *defs, "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or res.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}")
        return obj

    # independent translation units: compile them concurrently
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
