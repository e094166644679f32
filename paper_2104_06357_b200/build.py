"""Build libsemidist_b200.so in-tree with nvcc for sm_100a.

Usage: python -m paper_2104_06357_b200.build [--verbose]
The shared library lands next to this file so that it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsemidist_b200.so")
SOURCES = ["api.cu", "prep.cu", "engine.cu", "epilogue.cu", "isect.cu", "isect_f32.cu", "isect_f64.cu", "topk.cu", "hybrid.cu", "hminsum.cu", "dense_tc.cu", "util.cu"]
HEADERS = ["common.cuh", "semiring.cuh", "metric.cuh", "prep.cuh", "topk.cuh", "isect_kernel.cuh", "index.cuh", "hybrid.cuh", "tma.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    # no FMA contraction: products and sums round exactly like the numpy reference
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def _obj(src):
    return os.path.join(CSRC, "build", src.replace(".cu", ".o"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False, variant=None, defines=()):
    """Compile every source and link LIB.  ``variant``/``defines`` build a
    tuning variant (libsemidist_b200_<variant>.so) with extra -D flags."""
    global LIB
    lib_path = LIB if variant is None else os.path.join(HERE, f"libsemidist_b200_{variant}.so")
    obj_dir = os.path.join(CSRC, "build" if variant is None else f"build_{variant}")
    return _build(verbose, force, lib_path, obj_dir, list(defines))


def _build(verbose, force, lib_path, obj_dir, defines):
    os.makedirs(obj_dir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "semidist_b200.h")]

    def compile_one(src):
        path = os.path.join(CSRC, src)
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        if not force and not _stale(obj, [path] + hdrs):
            return obj
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", path, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{res.stderr}")
        if verbose and res.stderr:
            sys.stderr.write(res.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    if force or _stale(lib_path, objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib_path,
               "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    return lib_path


if __name__ == "__main__":
    args = sys.argv[1:]
    variant = next((a.split("=", 1)[1] for a in args if a.startswith("--variant=")), None)
    defines = [a[2:] for a in args if a.startswith("-D")]
    print(build(verbose="--verbose" in args, force="--force" in args, variant=variant, defines=defines))
