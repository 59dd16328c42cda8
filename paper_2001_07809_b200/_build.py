"""In-tree build of the native libraries (sm_100a only).

  libstk_b200.so   : CUDA kernels + the C-ABI (include/stk_b200.h) + the C++
                     stereotk:: drop-in shim (include/stereotk/...).
  libstk_synth.so  : host-side synthetic scene generators (plain C).

Built with nvcc / gcc directly so the .so files live next to this file and
travel with the repo snapshot to the GPU box.  Rebuilds only when a source is
newer than its output.
"""
from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"

LIB = PKG / "libstk_b200.so"
CLI = PKG / "stereotk"  # the reference CLI (tools/main.cpp) on libstk_b200.so
SYNTH = PKG / "libstk_synth.so"

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = [
    "k_lightness.cu",
    "k_kmeans.cu",
    "k_apply.cu",
    "k_bnd.cu",
    "k_sad.cu",
    "k_sad_strip.cu",
    "k_sad_ws.cu",
    "k_reconstruct.cu",
    "k_blur.cu",
    "k_eval.cu",
    "stk_capi.cu",
]
CXX_SOURCES = ["stereotk_shim.cpp", "stk_io.cpp", "stk_video.cpp"]  # C++ stereotk:: drop-in over the C-ABI; file I/O
HEADERS = ["stk_internal.cuh", "stk_device.cuh"]


def _newer(srcs, out: Path) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(Path(s).stat().st_mtime > t for s in srcs if Path(s).exists())


def _run(cmd, verbose):
    if verbose:
        print(" ".join(map(str, cmd)), file=sys.stderr)
    r = subprocess.run(list(map(str, cmd)), capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(map(str, cmd))}\n{r.stdout}\n{r.stderr}")
    return r


def build(verbose: bool = False, force: bool = False) -> None:
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    deps = [CSRC / h for h in HEADERS] + [INCLUDE / "stk_b200.h"]
    deps += list((INCLUDE / "stereotk").glob("*.hpp"))
    objs, jobs = [], []
    for src in CU_SOURCES:
        s = CSRC / src
        o = objdir / (src + ".o")
        objs.append(o)
        if force or _newer([s] + deps, o):
            jobs.append([NVCC, *ARCH, *os.environ.get("STK_NVCC_EXTRA", "").split(), "-O3", "-lineinfo",
                         "-std=c++17", "-Xcompiler", "-fPIC",
                         "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr",
                         "-I", INCLUDE, "-I", CSRC, "-rdc=false", "-c", s, "-o", o])
    for src in CXX_SOURCES:
        s = CSRC / src
        o = objdir / (src + ".o")
        objs.append(o)
        if force or _newer([s] + deps, o):
            jobs.append(["/usr/bin/g++", "-O2", "-std=c++17", "-fPIC", "-Wall", "-pthread", "-I", INCLUDE,
                         "-c", s, "-o", o])
    # independent translation units: compile them concurrently
    with concurrent.futures.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(_run, j, verbose) for j in jobs]:
            f.result()
    if force or _newer(objs, LIB):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lz", "-lrt",
              "-ldl", "-lpthread"], verbose)
    if force or _newer([CSRC / "stereotk_cli.cpp", LIB] + deps, CLI):
        _run(["/usr/bin/g++", "-O2", "-std=c++17", "-Wall", "-I", INCLUDE, CSRC / "stereotk_cli.cpp",
              "-o", CLI, "-L", PKG, "-lstk_b200", "-Wl,-rpath,$ORIGIN"], verbose)
    if force or _newer([CSRC / "synth.c"], SYNTH):
        _run(["/usr/bin/gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-Wall", "-o", SYNTH,
              CSRC / "synth.c"], verbose)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
