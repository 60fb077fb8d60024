"""Builds the in-tree native library ``paper_2303_12753_b200/lib/libseghdc_b200.so``.

nvcc cross-compiles for sm_100a (B200) only; the same .so travels to the GPU box with the
repo snapshot. No JIT cache, no torch extension machinery: the library is a plain C-ABI
shared object (include/seghdc_cuda.h) that Python loads with ctypes and C/C++ callers link.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libseghdc_b200.so")

SOURCES = ["seghdc_kernels.cu", "seghdc_tc.cu", "seghdc_closed.cu", "seghdc_capi.cu", "seghdc_host.cpp", "seghdc_dropin.cpp",
           "seghdc_metrics.cpp", "seghdc_image_io.cpp"]
HEADERS = ["kernels.cuh", "launch.h", "host_internal.h"]
PUBLIC_HEADERS = [os.path.join(ROOT, "include", "seghdc_cuda.h"),
                  os.path.join(ROOT, "include", "seghdc", "seghdc.hpp"),
                  os.path.join(ROOT, "include", "seghdc", "metrics.hpp"),
                  os.path.join(ROOT, "include", "seghdc", "image_io.hpp")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++20", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-Wall", "-Xptxas", "-v,-warn-spills"] + os.environ.get("SEGHDC_NVCC_EXTRA", "").split()


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra: list[str] | None = None) -> str:
    """Compile + link the library to ``out`` (default: the product path). ``extra`` adds nvcc
    flags to the .cu compiles (e.g. -DSEGHDC_TRACE for a diagnostic build)."""
    extra = list(extra or [])
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + PUBLIC_HEADERS + [__file__]
    if not force and not _stale(out, deps):
        return out
    def compile_one(src):
        obj = out + "." + os.path.basename(src) + ".o"
        cmd = [nvcc()] + ARCH + NVCC_FLAGS + extra + ["-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [nvcc()] + ARCH + ["-O3", "-std=c++20", "-Xcompiler", "-fPIC", "-x", "c++",
                                     "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max(1, min(len(srcs), os.cpu_count() or 1))) as pool:  # one nvcc per source
        results = list(pool.map(compile_one, srcs))
    objs, logs = [], []
    for src, obj, r in results:
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = out + ".tmp"
    r = subprocess.run([nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart", "-lz"], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, out)
    for o in objs:
        os.remove(o)
    with open(out + ".ptxas.log", "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return out


CLI = os.path.join(LIBDIR, "seghdc")
CLI_SRC = os.path.join(ROOT, "tools", "seghdc_cli.cpp")


def build_cli(force: bool = False) -> str:
    """The reference's command-line tool over the drop-in (tools/seghdc_cli.cpp) as lib/seghdc."""
    build()
    if not force and not _stale(CLI, [CLI_SRC, LIB] + PUBLIC_HEADERS):
        return CLI
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cuda_lib = os.path.join(os.path.dirname(os.path.dirname(nvcc())), "lib64")
    cmd = [cxx, "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), CLI_SRC, "-o", CLI, "-L", LIBDIR,
           "-lseghdc_b200", "-L", cuda_lib, "-lcudart", "-lz", "-Wl,-rpath,$ORIGIN", "-Wl,-rpath," + cuda_lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("seghdc CLI build failed")
    return CLI


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=LIB)
    ap.add_argument("extra", nargs="*", help="extra nvcc flags, e.g. -DSEGHDC_TRACE")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=a.out, extra=a.extra))
