"""Builds paper_2507_13204_b200/libkrn_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2507_13204_b200.csrc.build [--force] [--verbose]

nvcc cross-compiles without a GPU.  Flags that matter for parity:
``--fmad=false`` (the reference contract is IEEE double without contraction,
SPEC.md:391) and no fast-math.  ``-lineinfo`` keeps ncu's source page usable.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
LIB = os.path.join(PKG, "libkrn_b200.so")
SOURCES = ["krn_context.cu", "krn_builtins.cu", "krn_laplacian.cu", "krn_jit.cu", "krn_ordered.cu", "krn_peer.cu"]
HEADERS = ["krn_common.cuh", "krn_prelude.cuh", os.path.join("..", "..", "include", "krn_b200.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _embed_prelude() -> str:
    """krn_prelude.cuh as a comma-separated byte list, #included by krn_jit.cu
    so generated kernels can `#include "krn_prelude.cuh"` under NVRTC."""
    src = os.path.join(HERE, "krn_prelude.cuh")
    out = os.path.join(HERE, "krn_prelude_embed.inc")
    data = open(src, "rb").read()
    text = ",".join(str(b) for b in data)
    if not os.path.exists(out) or open(out).read() != text:
        with open(out, "w") as f:
            f.write(text)
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = [os.path.join(HERE, f) for f in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    _embed_prelude()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *ARCH, "-O3", "-std=c++17", "-lineinfo", "--fmad=false", "--prec-div=true",
           "--prec-sqrt=true", "--ftz=false", "-Xcompiler", "-fPIC,-Wall", "-shared",
           "-cudart", "static", "-o", LIB]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += [os.path.join(HERE, s) for s in SOURCES] + ["-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libkrn_b200.so")
    if verbose:
        sys.stderr.write(res.stdout + res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
