"""Build libamgp.so in-tree with nvcc for sm_100a.

    python -m paper_2407_09848_b200._build          # incremental
    python -m paper_2407_09848_b200._build --force

Every translation unit is compiled with -fmad=false (no contracted FMA: the
kernels must reproduce the reference's separate multiply/add roundings) and
-lineinfo (ncu source view).  The host side uses -ffp-contract=off for the
same reason (smoother step scalars).
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libamgp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--shared",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-Xptxas", "-warn-spills",
    "-I", os.path.join(REPO, "include"),
]
LIBS = ["-ldl"]  # NCCL is dlopen'ed at run time (csrc/dist.cu)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(REPO, "include", "*.h")))


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in sources() + headers())


def build(force=False, verbose=False, defines=(), lib=None):
    """Compile every csrc/ translation unit and link libamgp.so.  `defines`
    (e.g. ["SPLIT_WARPS=16"]) and `lib` build a tuning variant elsewhere."""
    target = lib or LIB
    if not force and not defines and lib is None and up_to_date():
        return LIB
    objs = []
    odir = os.path.join(PKG, "build", "variant_" + "_".join(d.replace("=", "") for d in defines)
                        if defines else "")
    os.makedirs(odir, exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(odir, os.path.splitext(os.path.basename(src))[0] + ".o")
        cmd = [NVCC, *ARCH, *[f for f in FLAGS if f != "--shared"], *[f"-D{d}" for d in defines],
               "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode != 0:
            failed.append((src, text))
        elif verbose and text.strip():
            print(text)
    if failed:
        msg = "\n".join(f"--- {s}\n{t}" for s, t in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    cmd = [NVCC, *ARCH, "--shared", "-o", target, *objs, *LIBS]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return target


if __name__ == "__main__":
    # python -m paper_2407_09848_b200._build [--force] [-DNAME=VAL ... -o variant.so]
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = sys.argv[sys.argv.index("-o") + 1] if "-o" in sys.argv else None
    print("built", build(force="--force" in sys.argv, verbose=True, defines=defs, lib=out))
