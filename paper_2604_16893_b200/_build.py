"""Build libvp.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvp.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# vp_plan.cu carries the bit-exact f64 planning: no FMA contraction there (SURVEY §7 hard parts).
PER_FILE = {"vp_plan.cu": ["--fmad=false"]}
SOURCES = ["vp_abi.cu", "vp_adjacent.cu", "vp_dedup.cu", "vp_plan.cu", "vp_resize.cu", "vp_resize_fast.cu", "vp_resize_team.cu", "vp_resize_u8.cu", "vp_rope.cu", "vp_synth.cu"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "vp_internal.cuh"), os.path.join(CSRC, "vp_k3_common.cuh"), os.path.join(HERE, "..", "include", "vp.h"), __file__]
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(d) for d in deps):
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    extra = os.environ.get("VP_EXTRA_NVCC_FLAGS", "").split()   # experiments only

    def compile_one(s: str):
        o = os.path.join(objdir, s.replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
               "--expt-relaxed-constexpr", *PER_FILE.get(s, []), *extra, "-c", os.path.join(CSRC, s), "-o", o]
        return s, o, subprocess.run(cmd, capture_output=True, text=True)

    # the translation units are independent: compile them in parallel (the team kernels' file dominates)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = []
    for s, o, r in results:
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(o)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
