"""Build the sm_100a shared library in-tree (paper_2408_01391_b200/_lib/).

nvcc -gencode arch=compute_100a,code=sm_100a (plain -arch=sm_100a would emit
compute_100 PTX and ptxas then rejects tcgen05).  Exact-order kernels are
compiled with --fmad=false so no multiply-add is ever contracted.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libftkb200.so")
ROOT = os.path.dirname(HERE)

SOURCES = {
    "abi.cu": [],
    "exact.cu": ["--fmad=false"],
    "update.cu": ["--fmad=false"],
    "tc.cu": [],
    "tc_pair.cu": [],
    "tc_narrow.cu": [],
    "tc64.cu": [],
    "dscreen.cu": [],
    "kpp.cu": [],
    "h2d.cu": [],
}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]
if os.environ.get("FTK_PROBE"):  # role-timing probes in the CTA-pair kernel (diagnostics)
    COMMON.append("-DFTK_PAIR_PROBE")
# A/B experiments: FTK_VARIANT=name FTK_DEFS="-DX=1 ..." builds _lib/var_<name>/libftkb200.so,
# loaded with FTK_LIB_PATH=<that path>. The default build is untouched.
if os.environ.get("FTK_VARIANT"):
    LIBDIR = os.path.join(LIBDIR, "var_" + os.environ["FTK_VARIANT"])
    LIB = os.path.join(LIBDIR, "libftkb200.so")
    COMMON += os.environ.get("FTK_DEFS", "").split()


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False):
    os.makedirs(os.path.join(LIBDIR, "obj"), exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "ftk_b200.h"))
    objs, jobs = [], []
    for src, extra in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(LIBDIR, "obj", src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append((src, [nvcc(), *ARCH, *COMMON, *extra, "-c", s, "-o", o]))
    # translation units compile in parallel (nvcc is single-threaded)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda j: (j, subprocess.run(j[1], capture_output=True, text=True)),
                              jobs))
    for (src, cmd), r in results:
        if verbose or r.returncode:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}")
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
