"""Build libgridcast_b200.so in-tree for sm_100a (explicit nvcc; no JIT cache).

    python -m paper_2603_01122_b200.build [--force] [--checked]

``--checked`` builds _lib/checked/libgridcast_b200.so with device asserts on the hot
kernels' indices (run anything against it with GC_LIB_PATH=<that path>).
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "_lib", "libgridcast_b200.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC",
    # the reference-arithmetic kernels rely on IEEE float32 semantics: keep denormals,
    # IEEE division and sqrt; the explicit __f*_rn intrinsics forbid contraction there
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
]
# per-file extra flags: the reference-arithmetic translation unit forbids FMA contraction
# (ptxas would fuse packed f32x2 mul+add pairs, changing numpy-exact results)
FILE_FLAGS = {"gc_predict_ref.cu": ["--fmad=false"]}
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "shared"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(os.path.join(HERE, "csrc", "*.h"))
    deps.append(os.path.join(ROOT, "include", "gridcast_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


# bounds-checked variant (every hot-kernel index a device assert; GC_LIB_PATH selects it)
CHECKED_OUT = os.path.join(HERE, "_lib", "checked", "libgridcast_b200.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    out = CHECKED_OUT if checked else OUT
    if not checked and not force and not needs_build():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objdir = os.path.join(HERE, "_lib", "obj_checked" if checked else "obj")
    os.makedirs(objdir, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = ["-DGC_CHECKED"] if checked else []
    # GC_EXTRA_NVCC_FLAGS: extra defines for A/B builds of kernel variants (tuning knob)
    extra += os.environ.get("GC_EXTRA_NVCC_FLAGS", "").split()

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra, *FILE_FLAGS.get(os.path.basename(src), []), "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, sources()))
    subprocess.run([nvcc, *LINK_FLAGS, "-o", out + ".tmp", *objs], check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
