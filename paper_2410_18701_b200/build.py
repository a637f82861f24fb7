"""Build libbaton.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2410_18701_b200.build [--verbose] [--force] [--experiments]

Compiles every csrc/*.cu with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
and links them (static cudart) into paper_2410_18701_b200/libbaton.so, which the
ctypes binding (_lib.py) loads.  Rebuilds only when a source or header is newer, or
when the build mode changed.  --experiments (or BATON_EXPERIMENTS=1) also compiles
csrc/experiments/*.cu with -DBATON_EXPERIMENTS=1: the round-1 sweep variants
(BATON_MHA_VARIANT / BATON_GQA_VARIANT) and the globaltimer debug timelines used by
scripts/trace_*.py and scripts/sweep_*.sh.  The product build has neither.
"""
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "libbaton")
LIB = os.path.join(PKG, "libbaton.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def _sources(experiments=False):
    srcs = glob.glob(os.path.join(CSRC, "*.cu"))
    if experiments:
        srcs += glob.glob(os.path.join(CSRC, "experiments", "*.cu"))
    return sorted(srcs)


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + glob.glob(os.path.join(CSRC, "experiments", "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths) if paths else 0.0


def build(verbose=False, force=False, experiments=None):
    if experiments is None:
        experiments = os.environ.get("BATON_EXPERIMENTS", "0") == "1"
    mode = "experiments" if experiments else "product"
    stamp = LIB + ".mode"
    old_mode = open(stamp).read().strip() if os.path.exists(stamp) else "product"
    srcs = _sources(experiments)
    hdr_time = _newest(_headers())
    if (not force and os.path.exists(LIB) and old_mode == mode
            and os.path.getmtime(LIB) >= max(_newest(srcs), hdr_time, os.path.getmtime(__file__))):
        return LIB
    build_dir = BUILD + ("-exp" if experiments else "")
    os.makedirs(build_dir, exist_ok=True)
    flags = FLAGS + (["-DBATON_EXPERIMENTS=1"] if experiments else [])

    def compile_one(src):
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_time,
                                                 os.path.getmtime(__file__))):
            return obj, ""
        cmd = [NVCC, *ARCH, *flags, "-Xptxas", "-v", "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(compile_one, srcs))
    if verbose:
        for obj, log in results:
            if log:
                print(f"== {os.path.basename(obj)}\n{log}")
    objs = [o for o, _ in results]
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(mode + "\n")
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv,
                experiments=True if "--experiments" in sys.argv else None))
