"""In-tree build of the native libraries (no torch JIT cache, nothing under site-packages).

* ``librmgpu.so``        -- CUDA kernels + the C-ABI of ``include/rmgpu.h`` (sm_100a only).
* ``librectmorph_b200.so`` -- the C++ drop-in host library (namespace ``rectmorph``, the
  reference's entry points) layered on the C-ABI.

Run ``python -m paper_2002_09474_b200.build`` or call ``build()``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "librmgpu.so")
HOSTLIB = os.path.join(PKG, "librectmorph_b200.so")
CLI = os.path.join(PKG, "rectmorph_b200")  # the reference CLI (apply | bench | calibrate) on the GPU

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + (["-DRMGPU_TRACE"] if os.environ.get("RMGPU_TRACE") else []) + \
    os.environ.get("RMGPU_EXTRA_DEFS", "").split() + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr",
                     "-I", os.path.join(ROOT, "include")]
CU_SOURCES = ["capi.cu", "morph_generic.cu", "morph_stream.cu", "morph_phase.cu",
              "morph_phase_u8_min.cu", "morph_phase_u8_max.cu", "morph_phase_u16_min.cu", "morph_phase_u16_max.cu",
              "morph_col.cu", "morph_col_u8_min.cu", "morph_col_u8_max.cu", "morph_col_u16_min.cu",
              "morph_col_u16_max.cu", "morph_col_u8_grad.cu", "morph_col_u16_grad.cu", "morph_sep.cu",
              "morph_sep_h_u8_min.cu", "morph_sep_h_u8_max.cu", "morph_sep_h_u16_min.cu", "morph_sep_h_u16_max.cu",
              "transpose.cu",
              "generate.cu", "morph_fuse.cu"]
# K4 instantiations: morph_fuse_inst.cu compiled once per (pixel size, mode, block size B)
FUSE_VARIANTS = [(sz, mx, b) for sz in (1, 2) for mx in (0, 1) for b in ((12, 20) if sz == 1 else (8, 12))]
HOST_SOURCES = [os.path.join("host", "rectmorph_b200.cpp"), os.path.join("host", "pgm_b200.cpp")]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _headers() -> list[str]:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "rmgpu.h"))
    return hs


def _deps(path: str, seen: set | None = None) -> set:
    """Local headers a source includes, transitively (#include "..." resolved in csrc/ or include/)."""
    seen = set() if seen is None else seen
    try:
        lines = open(path).read().splitlines()
    except OSError:
        return seen
    for ln in lines:
        ln = ln.strip()
        if ln.startswith("#include") and '"' in ln:
            name = ln.split('"')[1]
            for d in (os.path.dirname(path), CSRC, os.path.join(ROOT, "include")):
                h = os.path.normpath(os.path.join(d, name))
                if os.path.exists(h):
                    if h not in seen:
                        seen.add(h)
                        _deps(h, seen)
                    break
    return seen


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build step failed:\n  " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.stderr.strip() and os.environ.get("RMGPU_BUILD_VERBOSE"):
        print(r.stderr, file=sys.stderr)


def build(force: bool = False, verbose: bool = False) -> str:
    if shutil.which(NVCC) is None and not os.path.exists(NVCC):
        raise RuntimeError("nvcc not found; the CUDA path cannot be built")
    os.makedirs(OBJ, exist_ok=True)
    headers = _headers()
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _newer(o, [s] + sorted(_deps(s))):
            jobs.append([NVCC] + NVCC_FLAGS + ["-c", s, "-o", o])
    fsrc = os.path.join(CSRC, "morph_fuse_inst.cu")
    fdeps = [fsrc] + sorted(_deps(fsrc))
    for sz, mx, b in FUSE_VARIANTS:
        o = os.path.join(OBJ, f"morph_fuse_u{8 * sz}_{'max' if mx else 'min'}_b{b}.o")
        objs.append(o)
        if force or _newer(o, fdeps):
            jobs.append([NVCC] + NVCC_FLAGS + [f"-DFUSE_SZ={sz}", f"-DFUSE_MAX={mx}", f"-DFUSE_B={b}", "-c", fsrc, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(_run, jobs))
    if force or jobs or _newer(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"])
    host_srcs = [os.path.join(CSRC, s) for s in HOST_SOURCES]
    host_hdr = os.path.join(ROOT, "include", "rectmorph_b200.hpp")
    if force or _newer(HOSTLIB, host_srcs + [host_hdr, LIB, os.path.join(ROOT, "include", "rmgpu.h")]):
        _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
              "-o", HOSTLIB] + host_srcs + ["-L", PKG, "-lrmgpu", "-Wl,-rpath,$ORIGIN"])
    cli_src = os.path.join(CSRC, "host", "rectmorph_cli_b200.cpp")
    if force or _newer(CLI, [cli_src, host_hdr, HOSTLIB, LIB, os.path.join(ROOT, "include", "rmgpu.h")]):
        _run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
              "-o", CLI, cli_src, "-L", PKG, "-lrectmorph_b200", "-lrmgpu", "-L", "/usr/local/cuda/lib64", "-lcudart",
              "-Wl,-rpath,$ORIGIN", "-Wl,-rpath,/usr/local/cuda/lib64"])
    if verbose:
        print("built", LIB, HOSTLIB, CLI)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
