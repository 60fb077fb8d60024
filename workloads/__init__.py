"""Benchmark / test workloads: the five BASELINE.json configurations and their seeded
synthetic images.

This package is neither the product nor the oracle. It exists so that bench.py's GPU arm,
its ``--impl reference`` arm, the golden generators and the tests all read the SAME input
bytes without the reference arm loading the product library (or the product loading the
oracle). The generator is a small C++ file (``synth.cpp``) compiled by ``build()`` into
``workloads/lib/libseghdc_synth.so``; image bytes are pinned by SHA-256 in
tests/golden/configs.json.
"""
from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "synth.cpp")
LIB = os.path.join(HERE, "lib", "libseghdc_synth.so")

# BASELINE.json configs. C3/C4 use alpha = 1.0: the default 0.2 fails the reference's flip-unit
# validation at 2048^2 / 4096^2 (position_encoder.cpp:29-38).
CONFIGS = {
    0: dict(name="C0", cid=0, dim=10000, k=2, iterations=10, alpha=0.2),
    1: dict(name="C1", cid=1, dim=10000, k=2, iterations=10, alpha=0.2),
    2: dict(name="C2", cid=2, dim=10000, k=2, iterations=10, alpha=0.2),
    3: dict(name="C3", cid=3, dim=10000, k=4, iterations=20, alpha=1.0),
    4: dict(name="C4", cid=4, dim=16384, k=8, iterations=20, alpha=1.0),
}
WORKLOAD_TEXT = {
    0: "C0: 256x256x3 synthetic nuclei (20 ellipses), D=10000, K=2, 10 iterations",
    1: "C1: 520x696x1 synthetic nuclei (60 ellipses, blur 1.5), D=10000, K=2, 10 iterations",
    2: "C2: 64 x 256x256x3 synthetic nuclei images, D=10000, K=2, 10 iterations each",
    3: "C3: 2048x2048x3 synthetic nuclei (1500 ellipses, 3 classes), D=10000, K=4, 20 iterations",
    4: "C4: 4096x4096x3 synthetic nuclei (6000 ellipses, 7 classes), D=16384, K=8, 20 iterations",
}
BETA, GAMMA, CB_SEED = 26, 1, 0  # RunConfig defaults (pipeline.hpp:18-35)
C2_IMAGES = 64  # config 2: a batch of 64 independent images (seeds 0..63)


def _cxx() -> str:
    for cand in ("/usr/bin/g++", shutil.which("g++")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("g++ not found")


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        subprocess.run([_cxx(), "-std=c++17", "-O2", "-fPIC", "-shared", "-o", LIB, SRC], check=True)
    return LIB


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.seghdc_synth_image.argtypes = [C.c_int, C.c_uint64, C.c_void_p, C.POINTER(C.c_size_t),
                                         C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        L.seghdc_synth_image.restype = C.c_int
        _lib = L
    return _lib


def synth_image(config_id: int, seed: int = 0) -> np.ndarray:
    """Seeded synthetic nuclei image of config ``config_id`` (0..4) as (h, w, c) uint8."""
    h, w, c = C.c_size_t(), C.c_size_t(), C.c_size_t()
    if lib().seghdc_synth_image(config_id, seed, None, C.byref(h), C.byref(w), C.byref(c)):
        raise ValueError(f"synthetic config id must be 0..4, got {config_id}")
    out = np.zeros((h.value, w.value, c.value), np.uint8)
    lib().seghdc_synth_image(config_id, seed, out.ctypes.data, C.byref(h), C.byref(w), C.byref(c))
    return out
