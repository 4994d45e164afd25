"""Build libspconv.so (sm_100a) in-tree with nvcc: one object per .cu, compiled
in parallel, then linked.  No --use_fast_math: the encoder's NZE test must be
IEEE (reading A21)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspconv.so")
OBJ = os.path.join(HERE, "build")
SOURCES = ["api.cu", "encode.cu", "sparse_conv.cu", "im2col.cu", "tcgemm.cu", "validate.cu", "cscc.cu", "stride_aware.cu", "fused_encode.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _git_rev() -> str:
    try:
        return subprocess.check_output(["git", "-C", HERE, "rev-parse", "--short", "HEAD"],
                                       stderr=subprocess.DEVNULL, text=True).strip()
    except Exception:
        return "unknown"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + \
        [os.path.join(HERE, "..", "include", "spconv.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, probes: bool = False, variant: str = "") -> str:
    """variant: a dev A/B build, `name:-DFOO,-DBAR` -> libspconv_<name>.so (loaded via
    SPC_LIB_OVERRIDE by the timing tools only)."""
    vname, vdefs = (variant.split(":", 1) + [""])[:2] if variant else ("", "")
    lib = LIB.replace(".so", "_probe.so") if probes else LIB
    if vname:
        lib = LIB.replace(".so", f"_{vname}.so")
    if not force and not probes and not vname and not stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    obj_dir = OBJ + ("_probe" if probes else "") + (f"_{vname}" if vname else "")
    os.makedirs(obj_dir, exist_ok=True)
    common = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              f"-DSPC_GIT_REV=\"{_git_rev()}\""] + (["-Xptxas=-v"] if verbose else []) + (["-DSPC_PROBES"] if probes else []) + \
        [d for d in vdefs.split(",") if d]

    def compile_one(src: str) -> str:
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        subprocess.check_call([*common, "-c", "-o", obj, os.path.join(CSRC, src)])
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    subprocess.check_call([nvcc, *ARCH, "-shared", "-o", lib + ".tmp", *objs, "-lcudart", "-lcublas"])
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, probes="--probes" in sys.argv, variant=var))
