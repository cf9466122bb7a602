"""Build the in-tree CUDA library libsdtw.so for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsdtw.so")
SOURCES = (["sdtw_api.cu"] + ["sdtw_dp_c%d%s.cu" % (c, t) for c in (1, 2, 4) for t in ("", "t")]
           + ["sdtw_dpq_c1.cu", "sdtw_dpq_c2.cu", "sdtw_dp16.cu", "sdtw_dp8.cu", "sdtw_dp_c2k.cu"])
HEADERS = ["sdtw_dp.cuh", "sdtw_dpq.cuh", "sdtw_prep.cuh", "sdtw_path.cuh", "sdtw_dp2.cuh", "sdtw_q8.cuh", "sdtw_start.cuh", "sdtw_dp_pick.h"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "sdtw.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str = None, defines=(), extra=()) -> str:
    """Compile each translation unit to an object in parallel, then link libsdtw.so.
    ``out``/``defines`` build an experimental variant elsewhere (A/B runs only)."""
    if out is None and not defines and not extra and not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build" if out is None else
                          "build_variant_" + os.path.splitext(os.path.basename(out))[0])
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + ["-D" + d for d in defines] + list(extra)

    def one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [_nvcc(), *compile_flags, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd, cwd=CSRC)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(one, SOURCES))
    target = LIB if out is None else out
    tmp = target + ".tmp%d" % os.getpid()
    subprocess.check_call([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs])
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    # python build.py [--force] [--out PATH -DNAME=V ... --xflag=FLAG ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    extra = [a[len("--xflag="):] for a in args if a.startswith("--xflag=")]
    print(build(force="--force" in args, verbose=True, out=out, defines=defs, extra=extra))
