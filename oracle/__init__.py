"""TEST INFRASTRUCTURE ONLY — CPU checkers for the SegHDC hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker or the timed
CPU baseline. The product (``paper_2303_12753_b200``) never imports it.

Two checkers, both ctypes over shared objects built by ``oracle/Makefile``:

* ``Port``  — ``lib/libseghdc_oracle.so``: the plain-C restatement (seghdc_oracle.c),
  each function citing the reference file:line it follows.
* ``Ref``   — ``_ref/libseghdc_ref.so``: the UNMODIFIED reference sources from
  /root/reference/proj/src compiled with the reference's own flags, behind an
  extern "C" shim (ref_shim.cpp). Built only where /root/reference exists; the
  prebuilt .so travels to the GPU box.

Both use the reference layout: a grid is ``n_pixels x ceil(dim/64)`` u64 words.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "lib", "libseghdc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libseghdc_ref.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(force: bool = False) -> None:
    """Compile the checkers (the port always; the reference only if its sources exist)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets += ["ref", "suites"]
    subprocess.run(["make", "-s", "-C", HERE] + (["-B"] if force else []) + targets, check=True)


def words_for(dim: int) -> int:
    return (dim + 63) // 64


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self._err = getattr(self.lib, self.prefix + "last_error")
        self._err.restype = C.c_char_p

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise OracleError(rc, self._err().decode())

    # --- shared wrappers (identical argument conventions in both libraries) ---
    def build_codebooks(self, dim, h, w, c, alpha=0.2, beta=26, gamma=1, seed=0, encoder=0):
        wph = words_for(dim)
        row = np.zeros(h * wph, np.uint64)
        col = np.zeros(w * wph, np.uint64)
        wid = np.zeros(c * 256 * wph, np.uint64)
        f = getattr(self.lib, self.prefix + "build_codebooks")
        f.argtypes = [_sz, _sz, _sz, _sz, C.c_double, _sz, _sz, C.c_uint64, C.c_int, _u64p, _u64p, _u64p]
        self._check(f(dim, h, w, c, alpha, beta, gamma, seed, encoder, row, col, wid))
        return row.reshape(h, wph), col.reshape(w, wph), wid.reshape(c, 256, wph)

    def select_seeds(self, img: np.ndarray, k: int) -> np.ndarray:
        h, w, c = img.shape
        out = np.zeros(k, np.uint64)
        f = getattr(self.lib, self.prefix + "select_seeds")
        f.argtypes = [_u8p, _sz, _sz, _sz, _sz, _u64p]
        self._check(f(np.ascontiguousarray(img), h, w, c, k, out))
        return out


class Port(_Lib):
    """The plain-C restatement (oracle/seghdc_oracle.c)."""

    prefix = "so_"

    def __init__(self, path: str = PORT_SO):
        super().__init__(path)

    def last_wraps(self) -> list:
        """Per-round count of 128-bit-wrapping strictly_closer comparisons of the last
        assign / cluster / cluster_stream call (so_last_wraps; diagnostic, not reference API)."""
        out = np.zeros(4096, np.uint64)
        f = self.lib.so_last_wraps
        f.argtypes = [_u64p, _sz]
        f.restype = _sz
        n = f(out, out.size)
        return [int(x) for x in out[:n]]

    def set_threads(self, n: int) -> None:
        self.lib.so_set_threads(C.c_int(n))

    def threads(self) -> int:
        return int(self.lib.so_get_threads())

    def mt64(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self.lib.so_mt64_stream.argtypes = [C.c_uint64, _sz, _u64p]
        self.lib.so_mt64_stream(seed, n, out)
        return out

    def encode(self, img: np.ndarray, dim: int, row, col, wid) -> np.ndarray:
        h, w, c = img.shape
        grid = np.zeros(h * w * words_for(dim), np.uint64)
        f = self.lib.so_encode
        f.argtypes = [_u8p, _sz, _sz, _sz, _sz, _u64p, _u64p, _u64p, _u64p]
        self._check(f(np.ascontiguousarray(img), h, w, c, dim, np.ascontiguousarray(row).ravel(),
                      np.ascontiguousarray(col).ravel(), np.ascontiguousarray(wid).ravel(), grid))
        return grid.reshape(h * w, words_for(dim))

    def assign(self, grid: np.ndarray, dim: int, z: np.ndarray) -> np.ndarray:
        k = z.shape[0]
        n = grid.shape[0]
        out = np.zeros(n, np.uint32)
        f = self.lib.so_assign
        f.argtypes = [_u64p, _sz, _sz, _u32p, _sz, _u32p]
        self._check(f(np.ascontiguousarray(grid).ravel(), n, dim, np.ascontiguousarray(z, np.uint32).ravel(), k, out))
        return out

    def update(self, grid: np.ndarray, dim: int, labels: np.ndarray, prev: np.ndarray):
        k = prev.shape[0]
        n = grid.shape[0]
        z = np.zeros((k, dim), np.uint32)
        counts = np.zeros(k, np.uint64)
        f = self.lib.so_update
        f.argtypes = [_u64p, _sz, _sz, _u32p, _u32p, _sz, _u32p, _u64p]
        self._check(f(np.ascontiguousarray(grid).ravel(), n, dim, np.ascontiguousarray(labels, np.uint32),
                      np.ascontiguousarray(prev, np.uint32).ravel(), k, z.ravel(), counts))
        return z, counts

    def cluster(self, grid, img, dim, k, iterations, early_stop=False, per_round=False):
        h, w, c = img.shape
        n = h * w
        rounds_buf = np.zeros(iterations * n, np.uint32) if per_round else None
        labels = np.zeros(n, np.uint32)
        z = np.zeros((k, dim), np.uint32)
        counts = np.zeros(k, np.uint64)
        rounds = _sz(0)
        f = self.lib.so_cluster
        f.argtypes = [_u64p, _u8p, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int, C.c_void_p, _u32p, _u32p, _u64p,
                      C.POINTER(_sz)]
        self._check(f(np.ascontiguousarray(grid).ravel(), np.ascontiguousarray(img), h, w, c, dim, k, iterations,
                      int(early_stop), None if rounds_buf is None else rounds_buf.ctypes.data, labels, z.ravel(),
                      counts, C.byref(rounds)))
        res = {"labels": labels, "centroids": z, "counts": counts, "rounds": rounds.value}
        if per_round:
            res["labels_rounds"] = rounds_buf.reshape(iterations, n)[: rounds.value]
        return res


    def cluster_stream(self, img, dim, row, col, widened, k, iterations, early_stop=False, per_round=False):
        """cluster() without a stored grid: pixels re-encoded from the tables every pass
        (so_cluster_stream) — for grids that do not fit host memory (C4)."""
        h, w, c = img.shape
        n = h * w
        rounds_buf = np.zeros(iterations * n, np.uint32) if per_round else None
        labels = np.zeros(n, np.uint32)
        z = np.zeros((k, dim), np.uint32)
        counts = np.zeros(k, np.uint64)
        rounds = _sz(0)
        f = self.lib.so_cluster_stream
        f.argtypes = [_u8p, _sz, _sz, _sz, _sz, _u64p, _u64p, _u64p, _sz, _sz, C.c_int, C.c_void_p, _u32p, _u32p,
                      _u64p, C.POINTER(_sz)]
        self._check(f(np.ascontiguousarray(img), h, w, c, dim, np.ascontiguousarray(row).ravel(),
                      np.ascontiguousarray(col).ravel(), np.ascontiguousarray(widened).ravel(), k, iterations,
                      int(early_stop), None if rounds_buf is None else rounds_buf.ctypes.data, labels, z.ravel(),
                      counts, C.byref(rounds)))
        res = {"labels": labels, "centroids": z, "counts": counts, "rounds": rounds.value}
        if per_round:
            res["labels_rounds"] = rounds_buf.reshape(iterations, n)[: rounds.value]
        return res


class Ref(_Lib):
    """The unmodified reference library (oracle/_ref/libseghdc_ref.so)."""

    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)

    def encode(self, img: np.ndarray, dim: int, alpha=0.2, beta=26, gamma=1, seed=0, encoder=0) -> np.ndarray:
        h, w, c = img.shape
        grid = np.zeros(h * w * words_for(dim), np.uint64)
        f = self.lib.ref_encode
        f.argtypes = [_u8p, _sz, _sz, _sz, _sz, C.c_double, _sz, _sz, C.c_uint64, C.c_int, _u64p]
        self._check(f(np.ascontiguousarray(img), h, w, c, dim, alpha, beta, gamma, seed, encoder, grid))
        return grid.reshape(h * w, words_for(dim))

    def _cluster(self, fname, grid, img, dim, k, iterations, early_stop, per_round, with_centroids):
        h, w, c = img.shape
        n = h * w
        rounds_buf = np.zeros(iterations * n, np.uint32) if per_round else None
        labels = np.zeros(n, np.uint32)
        rounds = _sz(0)
        f = getattr(self.lib, fname)
        args = [np.ascontiguousarray(grid).ravel(), np.ascontiguousarray(img), h, w, c, dim, k, iterations,
                int(early_stop), None if rounds_buf is None else rounds_buf.ctypes.data, labels]
        types = [_u64p, _u8p, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int, C.c_void_p, _u32p]
        res = {"labels": labels}
        if with_centroids:
            z = np.zeros((k, dim), np.uint32)
            counts = np.zeros(k, np.uint64)
            args += [z.ravel(), counts]
            types += [_u32p, _u64p]
            res.update(centroids=z, counts=counts)
        f.argtypes = types + [C.POINTER(_sz)]
        self._check(f(*args, C.byref(rounds)))
        res["rounds"] = rounds.value
        if per_round:
            res["labels_rounds"] = rounds_buf.reshape(iterations, n)[: rounds.value]
        return res

    def cluster(self, grid, img, dim, k, iterations, early_stop=False, per_round=False):
        """The reference's own cluster() (labels only; it does not expose centroids)."""
        return self._cluster("ref_cluster", grid, img, dim, k, iterations, early_stop, per_round, False)

    def cluster_replay(self, grid, img, dim, k, iterations, early_stop=False, per_round=False):
        """cluster()'s loop replayed through the public API, exporting the final centroid set."""
        return self._cluster("ref_cluster_replay", grid, img, dim, k, iterations, early_stop, per_round, True)

    def assign(self, grid, h, w, dim, z):
        k = z.shape[0]
        out = np.zeros(h * w, np.uint32)
        f = self.lib.ref_assign
        f.argtypes = [_u64p, _sz, _sz, _sz, _u32p, _sz, _u32p]
        self._check(f(np.ascontiguousarray(grid).ravel(), h, w, dim, np.ascontiguousarray(z, np.uint32).ravel(), k, out))
        return out

    def update(self, grid, h, w, dim, labels, prev, prev_counts=None):
        k = prev.shape[0]
        z = np.zeros((k, dim), np.uint32)
        counts = np.zeros(k, np.uint64)
        pc = np.ones(k, np.uint64) if prev_counts is None else np.ascontiguousarray(prev_counts, np.uint64)
        f = self.lib.ref_update
        f.argtypes = [_u64p, _sz, _sz, _sz, _u32p, _u32p, _u64p, _sz, _u32p, _u64p]
        self._check(f(np.ascontiguousarray(grid).ravel(), h, w, dim, np.ascontiguousarray(labels, np.uint32),
                      np.ascontiguousarray(prev, np.uint32).ravel(), pc, k, z.ravel(), counts))
        return z, counts

    # parallel execution of the reference's own assign+update (CPU baseline)
    def par_create(self, grid, h, w, dim, row_begin, row_end, nthreads):
        f = self.lib.ref_par_create
        f.argtypes = [_u64p, _sz, _sz, _sz, _sz, _sz, C.c_int]
        f.restype = C.c_void_p
        return f(np.ascontiguousarray(grid).ravel(), h, w, dim, row_begin, row_end, nthreads)

    def par_round(self, handle, z, counts):
        k, dim = z.shape
        nz = np.zeros_like(z)
        nc = np.zeros(k, np.uint64)
        f = self.lib.ref_par_round
        f.argtypes = [C.c_void_p, _u32p, _u64p, _sz, _u32p, _u64p]
        self._check(f(handle, np.ascontiguousarray(z).ravel(), np.ascontiguousarray(counts, np.uint64), k,
                      nz.ravel(), nc))
        return nz, nc

    # reference-pure full-length loop whose shard grids come from the reference's own
    # encode_image (ref_pare_*: peak host memory one grid; C4 = 34.4 GB)
    def cluster_encoded(self, img, dim, k, iterations, alpha=0.2, beta=26, gamma=1, seed=0, nthreads=None,
                        on_round=None):
        """cluster() (clusterer.cpp:190-218, early stop off) on the reference's own encode_image,
        rows split over threads. Returns labels per round (via on_round(r, labels) if given),
        the final labels, the centroid set used by the final assignment and its counts."""
        h, w, c = img.shape
        n = h * w
        nthreads = nthreads or os.cpu_count() or 1
        f = self.lib.ref_pare_create
        f.argtypes = [_u8p, _sz, _sz, _sz, _sz, C.c_double, _sz, _sz, C.c_uint64, C.c_int, C.c_int]
        f.restype = C.c_void_p
        hnd = f(np.ascontiguousarray(img), h, w, c, dim, alpha, beta, gamma, seed, 0, nthreads)
        if not hnd:
            raise OracleError(2, self._err().decode())
        try:
            seeds = self.select_seeds(img, k)
            z = np.zeros((k, dim), np.uint32)
            fs = self.lib.ref_pare_seed
            fs.argtypes = [C.c_void_p, _u64p, _sz, _u32p]
            self._check(fs(hnd, seeds, k, z.ravel()))
            counts = np.ones(k, np.uint64)
            fr = self.lib.ref_pare_round
            fr.argtypes = [C.c_void_p, _u32p, _u64p, _sz, C.c_int, _u32p, _u32p, _u64p]
            labels = np.zeros(n, np.uint32)
            for r in range(1, iterations + 1):
                upd = r < iterations
                nz = np.zeros_like(z)
                nc = np.zeros(k, np.uint64)
                self._check(fr(hnd, z.ravel(), counts, k, int(upd), labels, nz.ravel(), nc))
                if on_round:
                    on_round(r, labels)
                if upd:
                    z, counts = nz, nc
            return {"labels": labels, "centroids": z, "counts": counts, "rounds": iterations, "seeds": seeds}
        finally:
            self.lib.ref_pare_destroy.argtypes = [C.c_void_p]
            self.lib.ref_pare_destroy(hnd)

    def par_destroy(self, handle):
        self.lib.ref_par_destroy.argtypes = [C.c_void_p]
        self.lib.ref_par_destroy(handle)


def have_ref() -> bool:
    return os.path.exists(REF_SO)
