"""Build recipe for the CPU checkers (test infrastructure, never the product).

1. ``oracle/liboracle.so`` from ``oracle/relay_oracle.c`` (plain C restatement,
   ``-O3 -ffp-contract=off`` like the reference's own build flags,
   /root/reference/pkg/setup.py:37, plus OpenMP over independent heads).
2. ``oracle/_ref/relayserve/*.so``: the UNMODIFIED reference hot-path modules
   compiled from their sources where they lie under /root/reference
   (cython -> gcc).  Only binaries land in oracle/_ref (git-ignored, travels
   to the GPU box); no reference source is copied into the repo.  Modules:
   __init__, errors, kernels, numerics, attention, costmodel, kvcache, model,
   _kernels_py (.py) and _kernels_cy (.pyx) -- everything attention.py and
   the toy decoder (model.py, whose `_attend` is the reference caller of the
   relay path) import -- plus engine and serving, whose scheduler loop drives
   this package's B200 engine in tests/test_gpu_engine.py.

Run:  python oracle/build.py          (idempotent; skips up-to-date outputs)
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src/relayserve"
REF_MODULES = [
    ("__init__", ".py"), ("errors", ".py"), ("kernels", ".py"),
    ("numerics", ".py"), ("attention", ".py"), ("costmodel", ".py"),
    ("_kernels_py", ".py"), ("_kernels_cy", ".pyx"), ("kvcache", ".py"),
    ("model", ".py"), ("engine", ".py"), ("serving", ".py"),
]


def _newer(target, *sources):
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(s) <= t for s in sources)


def build_oracle(verbose=False):
    src = os.path.join(HERE, "relay_oracle.c")
    out = os.path.join(HERE, "liboracle.so")
    if _newer(out, src):
        return out
    cmd = ["gcc", "-O3", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-shared", "-fPIC", src, "-o", out, "-lm"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return out


def build_reference(verbose=False):
    """Compile the reference's own modules into oracle/_ref (if present)."""
    if not os.path.isdir(REF_SRC):
        return None
    import numpy
    out_dir = os.path.join(HERE, "_ref", "relayserve")
    os.makedirs(out_dir, exist_ok=True)
    import tempfile
    tmp_dir = tempfile.mkdtemp(prefix="relay_ref_build_")
    inc = sysconfig.get_paths()["include"]
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    for mod, ext in REF_MODULES:
        src = os.path.join(REF_SRC, mod + ext)
        so = os.path.join(out_dir, mod + suffix)
        if _newer(so, src):
            continue
        cfile = os.path.join(tmp_dir, mod + ".c")
        cy = [sys.executable, "-m", "cython", "-3", "--module-name",
              f"relayserve.{mod}", src, "-o", cfile]
        cc = ["gcc", "-shared", "-fPIC", "-O3", "-ffp-contract=off",
              "-I", inc, "-I", numpy.get_include(), cfile, "-o", so]
        if verbose:
            print(" ".join(cy))
            print(" ".join(cc))
        subprocess.check_call(cy, stdout=subprocess.DEVNULL)
        subprocess.check_call(cc)
    import shutil
    shutil.rmtree(tmp_dir, ignore_errors=True)
    return out_dir


def main():
    print(build_oracle(verbose=True))
    print(build_reference(verbose=True))


if __name__ == "__main__":
    main()
