"""SegHDC encode + cluster hot path on B200 — Python host API over the C-ABI.

Mirrors the reference's ``seghdc::`` operator interface (/root/reference/proj/include/seghdc):
same names, same argument meaning, same errors (:class:`ConfigError` where the reference
throws ``seghdc::ConfigError``). Every call goes through ``lib/libseghdc_b200.so``
(include/seghdc_cuda.h); there is no CPU fallback — without the native library or a
B200 the calls raise.

Layouts are the reference's: a grid is ``(h*w, ceil(dim/64))`` uint64, centroids are
``(k, dim)`` uint32 raw member sums, labels are ``(h*w,)`` uint32 row-major.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import threading
import weakref
from typing import Callable, Optional

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# SEGHDC_LIB selects a diagnostic build of the same library (trace / hang-debug variants)
LIB_PATH = os.environ.get("SEGHDC_LIB") or os.path.join(PKG, "lib", "libseghdc_b200.so")

SEGHDC_OK, SEGHDC_ECONFIG, SEGHDC_ERUNTIME = 0, 1, 2
ENCODERS = {"manhattan": 0, "rpos": 1, "rcolor": 2}


class ConfigError(ValueError):
    """Invalid configuration (reference ``seghdc::ConfigError``, errors.hpp:9-12)."""


class RuntimeFailure(RuntimeError):
    """CUDA/device failure (no reference analogue)."""


_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t
ROUND_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.POINTER(C.c_uint32))

# every symbol include/seghdc_cuda.h declares, with its ctypes signature
SIGNATURES = {
    "seghdc_create": ([C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "seghdc_destroy": ([C.c_void_p], None),
    "seghdc_last_error": ([C.c_void_p], C.c_char_p),
    "seghdc_set_stream": ([C.c_void_p, C.c_void_p], C.c_int),
    "seghdc_set_sm_budget": ([C.c_void_p, C.c_int], C.c_int),
    "seghdc_synchronize": ([C.c_void_p], C.c_int),
    "seghdc_kernel_launches": ([C.c_void_p], C.c_uint64),
    "seghdc_round_kernel": ([C.c_void_p], C.c_char_p),
    "seghdc_build_codebooks": ([_sz, _sz, _sz, _sz, C.c_double, _sz, _sz, C.c_uint64, C.c_int, _u64p, _u64p, _u64p],
                               C.c_int),
    "seghdc_validate_run": ([_sz, _sz, _sz, _sz, C.c_double, _sz, _sz, _sz, _sz], C.c_int),
    "seghdc_encode": ([C.c_void_p, _u8p, _sz, _sz, _sz, _sz, _u64p, _u64p, _u64p, C.c_void_p], C.c_int),
    "seghdc_select_seeds": ([C.c_void_p, _u8p, _sz, _sz, _sz, _sz, _u64p], C.c_int),
    "seghdc_assign": ([C.c_void_p, C.c_void_p, _sz, _sz, _sz, _u32p, _sz, _u32p], C.c_int),
    "seghdc_update": ([C.c_void_p, C.c_void_p, _sz, _sz, _sz, _u32p, _u32p, _sz, _u32p, _u64p], C.c_int),
    "seghdc_cluster": ([C.c_void_p, C.c_void_p, _u8p, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int, ROUND_CB, C.c_void_p,
                        _u32p, C.c_void_p, C.c_void_p, C.POINTER(_sz)], C.c_int),
    "seghdc_run_pipeline": ([C.c_void_p, _u8p, _sz, _sz, _sz, _sz, C.c_double, _sz, _sz, _sz, _sz, C.c_uint64, C.c_int,
                             C.c_int, ROUND_CB, C.c_void_p, _u32p, C.POINTER(_sz), C.c_void_p], C.c_int),
    "seghdc_run_pipeline_batch": ([C.c_void_p, C.c_void_p, _sz, _sz, _sz, _sz, _sz, C.c_double, _sz, _sz, _sz, _sz,
                                   C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "seghdc_run_pipeline_closed": ([C.c_void_p, _u8p, _sz, _sz, _sz, _sz, C.c_double, _sz, _sz, _sz, _sz, C.c_uint64,
                                    C.c_int, _u32p, _u32p, _u64p, C.POINTER(_sz)], C.c_int),
    "seghdc_load_image": ([C.c_void_p, C.c_void_p, _sz, _sz, _sz], C.c_int),
    "seghdc_load_codebooks": ([C.c_void_p, _sz, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "seghdc_encode_async": ([C.c_void_p, _sz, _sz], C.c_int),
    "seghdc_load_grid": ([C.c_void_p, _u64p, _sz, _sz, _sz, _sz, _sz], C.c_int),
    "seghdc_store_grid": ([C.c_void_p, _u64p], C.c_int),
    "seghdc_cluster_async": ([C.c_void_p, _sz, _sz, C.c_int], C.c_int),
    "seghdc_fetch_results": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_sz)], C.c_int),
    "seghdc_shard_begin": ([C.c_void_p, _sz, _sz, C.c_int], C.c_int),
    "seghdc_exchange_buffer": ([C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(_sz)], C.c_int),
    "seghdc_exchange_download": ([C.c_void_p, C.c_void_p], C.c_int),
    "seghdc_exchange_upload": ([C.c_void_p, C.c_void_p], C.c_int),
    "seghdc_shard_init_finish": ([C.c_void_p], C.c_int),
    "seghdc_shard_assign": ([C.c_void_p, _sz], C.c_int),
    "seghdc_shard_round_needs_exchange": ([C.c_void_p, _sz], C.c_int),
    "seghdc_shard_finish": ([C.c_void_p, _sz], C.c_int),
    "seghdc_nccl_get_unique_id": ([C.c_void_p], C.c_int),
    "seghdc_nccl_init": ([C.c_void_p, C.c_void_p, C.c_int, C.c_int], C.c_int),
    "seghdc_set_allreduce": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int], C.c_int),
    "seghdc_shard_rows": ([_sz, C.c_int, C.c_int, C.POINTER(_sz), C.POINTER(_sz)], C.c_int),
    "seghdc_shard_row_range": ([C.c_void_p, _sz, C.POINTER(_sz), C.POINTER(_sz)], C.c_int),
    "seghdc_cluster_sharded_async": ([C.c_void_p, _sz, _sz, C.c_int], C.c_int),
    "seghdc_run_pipeline_sharded": ([C.c_void_p, _u8p, _sz, _sz, _sz, _sz, C.c_double, _sz, _sz, _sz, _sz, C.c_uint64,
                                     C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_sz), C.c_void_p],
                                    C.c_int),
    "seghdc_set_wrap_counting": ([C.c_void_p, C.c_int], C.c_int),
    "seghdc_round_wraps": ([C.c_void_p, C.c_void_p, _sz, C.POINTER(_sz)], C.c_int),
    "seghdc_best_foreground_iou": ([_u32p, _u8p, _sz, _sz, _sz, C.POINTER(C.c_double), C.POINTER(C.c_uint32)],
                                   C.c_int),
    "seghdc_profile_rounds": ([C.c_void_p, C.c_int], C.c_int),
    "seghdc_profile_read": ([C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64)], C.c_int),
    "seghdc_profile_read_each": ([C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_void_p, _sz], C.c_int),
    "seghdc_pinned_alloc": ([_sz, C.POINTER(C.c_void_p)], C.c_int),
    "seghdc_pinned_free": ([C.c_void_p], C.c_int),
}

_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Load the native library (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeFailure(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                 "(python -m paper_2303_12753_b200.build)")
        L = C.CDLL(LIB_PATH)
        for name, (argtypes, restype) in SIGNATURES.items():
            if os.environ.get("SEGHDC_LIB") and not hasattr(L, name):
                continue  # a diagnostic / older build selected for an A/B run
            f = getattr(L, name)
            f.argtypes = argtypes
            f.restype = restype
        _lib = L
    return _lib


def _check(rc: int, ctx_handle=None) -> None:
    if rc == SEGHDC_OK:
        return
    msg = lib().seghdc_last_error(ctx_handle).decode()
    if rc == SEGHDC_ECONFIG:
        raise ConfigError(msg)
    raise RuntimeFailure(msg)


def words_for(dim: int) -> int:
    """Hypervector::words_for (hypervector.hpp:37)."""
    return (dim + 63) // 64


def _img3(img: np.ndarray) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.ndim == 2:
        img = img[:, :, None]
    if img.ndim != 3:
        raise ConfigError("image must be (h, w) or (h, w, channels) uint8")
    return img


# ------------------------------------------------------------------------------------------
# Host-side codebooks (position_encoder.hpp:45, color_encoder.hpp:42, pipeline.cpp:43-59)
# ------------------------------------------------------------------------------------------
def build_codebooks(dim: int, h: int, w: int, channels: int, alpha: float = 0.2, beta: int = 26, gamma: int = 1,
                    seed: int = 0, encoder: str = "manhattan"):
    """Position + colour codebooks from one ``mt19937_64(seed)`` in run_pipeline's order.

    Returns ``(row[h, wph], col[w, wph], widened[channels, 256, wph])`` uint64; the colour
    tables are widened to full dim at their concatenation offsets.
    """
    wph = words_for(dim)
    row = np.zeros(h * wph, np.uint64)
    col = np.zeros(w * wph, np.uint64)
    wid = np.zeros(channels * 256 * wph, np.uint64)
    _check(lib().seghdc_build_codebooks(dim, h, w, channels, float(alpha), beta, gamma, seed, ENCODERS[encoder], row,
                                        col, wid))
    return row.reshape(h, wph), col.reshape(w, wph), wid.reshape(channels, 256, wph)


_pinned_free: dict = {}  # nbytes -> [pointers]: page-locked buffers returned by dead arrays
_pinned_lock = threading.Lock()


def _return_pinned(nbytes: int, ptr: int) -> None:
    with _pinned_lock:
        _pinned_free.setdefault(nbytes, []).append(ptr)


def pinned_empty(shape, dtype=np.uint32) -> np.ndarray:
    """An uninitialised array in page-locked host memory (seghdc_pinned_alloc), recycled
    through a process-wide pool once every view of it is gone."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    ptr = None
    with _pinned_lock:  # callers on several host threads (one per context)
        free = _pinned_free.get(nbytes)
        if free:
            ptr = free.pop()
    if ptr is None:
        p = C.c_void_p()
        _check(lib().seghdc_pinned_alloc(nbytes, C.byref(p)))
        ptr = p.value
    raw = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(max(nbytes, 1),))
    weakref.finalize(raw.base, _return_pinned, nbytes, ptr)
    return raw[:nbytes].view(dtype).reshape(shape)


# (user, device int32 buffer, n, cudaStream_t) -> 0 on success: seghdc_allreduce_fn
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, _sz, C.c_void_p)


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0), to be shipped to the other ranks out of band."""
    buf = C.create_string_buffer(128)
    _check(lib().seghdc_nccl_get_unique_id(buf))
    return buf.raw


def shard_rows(h: int, rank: int, nranks: int) -> tuple[int, int]:
    """Rows [r0, r1) of rank ``rank``: contiguous blocks differing by at most one row."""
    r0, r1 = _sz(), _sz()
    _check(lib().seghdc_shard_rows(h, rank, nranks, C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


def best_foreground_iou(labels: np.ndarray, gt: np.ndarray, k: int):
    """best_foreground_iou (metrics.hpp:33-36): (iou, subset of labels) for a mask of cluster
    labels and a ground truth (nonzero = foreground) of the same shape; k <= 4."""
    lab = np.ascontiguousarray(labels, np.uint32).ravel()
    g = (np.ascontiguousarray(gt).reshape(lab.shape[0], -1) != 0).any(axis=1).astype(np.uint8)
    if g.size != lab.size:
        raise ConfigError("best_foreground_iou: mask shapes differ")
    v, m = C.c_double(), C.c_uint32()
    rc = lib().seghdc_best_foreground_iou(lab, g, 1, lab.size, k, C.byref(v), C.byref(m))
    if rc == SEGHDC_ECONFIG:
        raise ConfigError(f"best_foreground_iou: k = {k} must be 1..4 and every label < k")
    _check(rc)
    return v.value, [c for c in range(k) if m.value >> c & 1]


def synth_image(config_id: int, seed: int = 0) -> np.ndarray:
    """Seeded synthetic nuclei image of BASELINE.json config ``config_id``; the
    generator lives in the repo's ``workloads`` package, outside the product library."""
    import workloads

    return workloads.synth_image(config_id, seed)


# ------------------------------------------------------------------------------------------
# Device context
# ------------------------------------------------------------------------------------------
class Context:
    """One CUDA device context (``seghdc_ctx``): stream + resident HVs in HBM."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib().seghdc_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self) -> None:
        if self.h:
            lib().seghdc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def check(self, rc: int) -> None:
        _check(rc, self.h)

    def set_stream(self, stream_handle: int) -> None:
        self.check(lib().seghdc_set_stream(self.h, C.c_void_p(stream_handle)))

    def set_sm_budget(self, sms: int) -> None:
        """Size this context's grids for ``sms`` SMs (0 = all): contexts on separate streams then
        run side by side (batches of small images). Results do not depend on it."""
        self.check(lib().seghdc_set_sm_budget(self.h, sms))

    def synchronize(self) -> None:
        self.check(lib().seghdc_synchronize(self.h))

    @property
    def kernel_launches(self) -> int:
        return int(lib().seghdc_kernel_launches(self.h))

    @property
    def round_kernel(self) -> str:
        """Round kernel of the current clustering plan (k_round_tc / k_round_fused / k_round)."""
        return lib().seghdc_round_kernel(self.h).decode()

    def set_wrap_counting(self, enable: bool) -> None:
        """Opt in to counting 128-bit comparator wraps (seghdc_set_wrap_counting)."""
        self.check(lib().seghdc_set_wrap_counting(self.h, int(enable)))

    def round_wraps(self) -> list:
        """Per-round count of 128-bit-wrapping strictly_closer comparisons in the last clustering
        run (seghdc_round_wraps; diagnostic, compared with the oracle's so_last_wraps)."""
        out = np.zeros(4096, np.uint64)
        n = _sz()
        self.check(lib().seghdc_round_wraps(self.h, out.ctypes.data, out.size, C.byref(n)))
        return [int(x) for x in out[:min(n.value, out.size)]]

    def profile_rounds(self, enable: bool) -> None:
        self.check(lib().seghdc_profile_rounds(self.h, int(enable)))

    def profile_read(self):
        """(summed round-kernel milliseconds, launches) since the last read."""
        t, n = C.c_double(), C.c_uint64()
        self.check(lib().seghdc_profile_read(self.h, C.byref(t), C.byref(n)))
        return t.value, n.value

    def profile_read_each(self, cap: int = 4096) -> np.ndarray:
        """Per-launch round-kernel milliseconds (launch order) since the last read."""
        t, n = C.c_double(), C.c_uint64()
        out = np.zeros(cap, np.float64)
        self.check(lib().seghdc_profile_read_each(self.h, C.byref(t), C.byref(n), out.ctypes.data, cap))
        return out[:min(n.value, cap)].copy()

    # ---- reference API ------------------------------------------------------------------
    def encode_image(self, img: np.ndarray, dim: int, row, col, widened, download: bool = True):
        """encode_image (pixel_pipeline.hpp:74-75). The grid also stays resident."""
        img = _img3(img)
        h, w, c = img.shape
        grid = np.zeros((h * w, words_for(dim)), np.uint64) if download else None
        self.check(lib().seghdc_encode(self.h, img, h, w, c, dim, np.ascontiguousarray(row, np.uint64).ravel(),
                                       np.ascontiguousarray(col, np.uint64).ravel(),
                                       np.ascontiguousarray(widened, np.uint64).ravel(),
                                       None if grid is None else grid.ctypes.data))
        return grid

    def select_initial_centroids(self, img: np.ndarray, k: int) -> np.ndarray:
        """select_initial_centroids (clusterer.hpp:54-55): seed pixels as linear indices."""
        img = _img3(img)
        h, w, c = img.shape
        out = np.zeros(k, np.uint64)
        self.check(lib().seghdc_select_seeds(self.h, img, h, w, c, k, out))
        return out

    def assign_labels(self, grid: Optional[np.ndarray], h: int, w: int, dim: int, centroids: np.ndarray) -> np.ndarray:
        """assign_labels (clusterer.hpp:60). ``grid=None`` uses the resident grid."""
        z = np.ascontiguousarray(centroids, np.uint32)
        k = z.shape[0]
        if z.ndim != 2 or z.shape[1] != dim:
            raise ConfigError("assign_labels: dimension mismatch")
        labels = np.zeros(h * w, np.uint32)
        gp = None if grid is None else np.ascontiguousarray(grid, np.uint64).ctypes.data
        self.check(lib().seghdc_assign(self.h, gp, h, w, dim, z.ravel(), k, labels))
        return labels

    def update_centroids(self, grid: Optional[np.ndarray], h: int, w: int, dim: int, labels: np.ndarray,
                         prev: np.ndarray):
        """update_centroids (clusterer.hpp:65-66) -> (centroids[k, dim], member_counts[k])."""
        z = np.ascontiguousarray(prev, np.uint32)
        k = z.shape[0]
        lab = np.ascontiguousarray(labels, np.uint32).ravel()
        if lab.size != h * w:
            raise ConfigError("update_centroids: mask shape does not match grid")
        out = np.zeros((k, dim), np.uint32)
        counts = np.zeros(k, np.uint64)
        gp = None if grid is None else np.ascontiguousarray(grid, np.uint64).ctypes.data
        self.check(lib().seghdc_update(self.h, gp, h, w, dim, lab, z.ravel(), k, out.ravel(), counts))
        return out, counts

    def cluster(self, grid: Optional[np.ndarray], img: np.ndarray, dim: int, k: int, iterations: int = 10,
                early_stop: bool = True, on_iteration: Optional[Callable[[int, np.ndarray], None]] = None):
        """cluster (clusterer.hpp:79-80) + the final centroid set.

        Returns dict(labels, centroids, counts, rounds); ``on_iteration(round, labels)`` mirrors
        IterationCallback (called after every assignment round)."""
        img = _img3(img)
        h, w, c = img.shape
        labels = np.zeros(h * w, np.uint32)
        z = np.zeros((k, dim), np.uint32)
        counts = np.zeros(k, np.uint64)
        rounds = _sz(0)
        cb = ROUND_CB(0)
        if on_iteration is not None:
            def _cb(_user, r, ptr):
                on_iteration(int(r), np.ctypeslib.as_array(ptr, shape=(h * w,)).copy())
            cb = ROUND_CB(_cb)
        gp = None if grid is None else np.ascontiguousarray(grid, np.uint64).ctypes.data
        self.check(lib().seghdc_cluster(self.h, gp, img, h, w, c, dim, k, iterations, int(early_stop), cb, None, labels,
                                        z.ctypes.data, counts.ctypes.data, C.byref(rounds)))
        return {"labels": labels, "centroids": z, "counts": counts, "rounds": rounds.value}

    def run_pipeline(self, img: np.ndarray, config: "RunConfig",
                     on_iteration: Optional[Callable[[int, np.ndarray], None]] = None) -> "PipelineResult":
        """run_pipeline (pipeline.hpp:55-56)."""
        img = _img3(img)
        h, w, c = img.shape
        labels = pinned_empty(h * w, np.uint32)  # page-locked: the label download runs at PCIe rate
        rounds = _sz(0)
        timings = (C.c_double * 5)()
        cb = ROUND_CB(0)
        if on_iteration is not None:
            def _cb(_user, r, ptr):
                on_iteration(int(r), np.ctypeslib.as_array(ptr, shape=(h * w,)).copy())
            cb = ROUND_CB(_cb)
        self.check(lib().seghdc_run_pipeline(self.h, img, h, w, c, config.dim, float(config.alpha), config.beta,
                                             config.gamma, config.clusters, config.iterations, config.seed,
                                             ENCODERS[config.encoder], int(config.early_stop), cb, None, labels,
                                             C.byref(rounds), C.cast(timings, C.c_void_p)))
        names = ("encode_position", "encode_color", "produce_pixels", "cluster", "total")
        return PipelineResult(labels.reshape(h, w), rounds.value, dict(zip(names, list(timings))))

    def run_pipeline_batch(self, imgs, config: "RunConfig"):
        """run_pipeline over a list of same-shape images in one call (seghdc_run_pipeline_batch):
        returns (labels[n, h, w], rounds[n])."""
        imgs = [_img3(i) for i in imgs]
        h, w, c = imgs[0].shape
        if any(i.shape != (h, w, c) for i in imgs):
            raise ConfigError("run_pipeline_batch: images must share one shape")
        n = len(imgs)
        labels = pinned_empty((n, h, w), np.uint32)
        rounds = np.zeros(n, np.uint64)
        px = (C.c_void_p * n)(*[i.ctypes.data for i in imgs])
        outs = (C.c_void_p * n)(*[labels[j].ctypes.data for j in range(n)])
        self.check(lib().seghdc_run_pipeline_batch(self.h, px, n, h, w, c, config.dim, float(config.alpha),
                                                   config.beta, config.gamma, config.clusters, config.iterations,
                                                   config.seed, ENCODERS[config.encoder], int(config.early_stop),
                                                   outs, rounds.ctypes.data))
        return labels, rounds

    def run_pipeline_closed(self, img: np.ndarray, config: "RunConfig") -> dict:
        """Closed-form Manhattan variant of run_pipeline (SURVEY.md §7 hard part 4): the pixel
        HVs are never materialised. Returns labels (h*w), centroids (k x dim, the set used by
        the final assignment), counts and rounds, like cluster()."""
        if config.encoder != "manhattan":
            raise ConfigError("closed-form variant: Manhattan codebooks only")
        img = _img3(img)
        h, w, c = img.shape
        labels = np.empty(h * w, np.uint32)
        cents = np.empty((config.clusters, config.dim), np.uint32)
        counts = np.empty(config.clusters, np.uint64)
        rounds = _sz(0)
        self.check(lib().seghdc_run_pipeline_closed(self.h, img, h, w, c, config.dim, float(config.alpha), config.beta,
                                                    config.gamma, config.clusters, config.iterations, config.seed,
                                                    int(config.early_stop), labels, cents.reshape(-1), counts,
                                                    C.byref(rounds)))
        return {"labels": labels, "centroids": cents, "counts": counts, "rounds": rounds.value}

    # ---- device-resident staging (bench / sharding) ----------------------------------------
    def load_image(self, img: np.ndarray) -> None:
        img = _img3(img)
        h, w, c = img.shape
        self.check(lib().seghdc_load_image(self.h, img.ctypes.data, h, w, c))

    def load_image_ptr(self, ptr: int, h: int, w: int, c: int) -> None:
        self.check(lib().seghdc_load_image(self.h, C.c_void_p(ptr), h, w, c))

    def load_codebooks(self, dim: int, row, col, widened) -> None:
        self._cb_keep = [np.ascontiguousarray(a, np.uint64) for a in (row, col, widened)]
        self.check(lib().seghdc_load_codebooks(self.h, dim, *[a.ctypes.data for a in self._cb_keep]))

    def encode_async(self, row_begin: int, row_end: int) -> None:
        self.check(lib().seghdc_encode_async(self.h, row_begin, row_end))

    def load_grid(self, grid: np.ndarray, h: int, w: int, dim: int, row_begin: int = 0, row_end: Optional[int] = None):
        g = np.ascontiguousarray(grid, np.uint64).ravel()
        self.check(lib().seghdc_load_grid(self.h, g, h, w, dim, row_begin, h if row_end is None else row_end))

    def store_grid(self, n_pixels: int, dim: int) -> np.ndarray:
        out = np.zeros((n_pixels, words_for(dim)), np.uint64)
        self.check(lib().seghdc_store_grid(self.h, out.ravel()))
        return out

    def cluster_async(self, k: int, iterations: int, early_stop: bool = False) -> None:
        self.check(lib().seghdc_cluster_async(self.h, k, iterations, int(early_stop)))

    def fetch_results(self, n_pixels: int, k: int, dim: int, labels: bool = True, centroids: bool = True):
        lab = np.zeros(n_pixels, np.uint32) if labels else None
        z = np.zeros((k, dim), np.uint32) if centroids else None
        counts = np.zeros(k, np.uint64)
        rounds = _sz(0)
        self.check(lib().seghdc_fetch_results(self.h, None if lab is None else lab.ctypes.data,
                                              None if z is None else z.ctypes.data, counts.ctypes.data,
                                              C.byref(rounds)))
        return {"labels": lab, "centroids": z, "counts": counts, "rounds": rounds.value}

    # ---- row-block sharding with the collective inside the library -------------------------
    def nccl_init(self, unique_id: bytes, rank: int, nranks: int) -> None:
        """NCCL communicator for this rank (seghdc_nccl_init); the sharded calls then all-reduce
        the exchange buffer with ncclAllReduce on the context's stream."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self.check(lib().seghdc_nccl_init(self.h, buf, rank, nranks))
        self.rank, self.nranks = rank, nranks

    def set_allreduce(self, fn: Optional[Callable[[int, int, int], None]], rank: int, nranks: int) -> None:
        """Any other collective: ``fn(device_ptr, n_int32, cuda_stream)`` must leave the int32
        buffer equal to the SUM over ranks (seghdc_set_allreduce). ``fn=None`` clears it."""
        if fn is None:
            self._ar_cb = None
            self.check(lib().seghdc_set_allreduce(self.h, None, None, rank, nranks))
        else:
            def _cb(_user, ptr, n, stream):
                try:
                    fn(int(ptr), int(n), int(stream or 0))
                    return 0
                except Exception:  # noqa: BLE001 - reported to the library as a failed collective
                    import traceback
                    traceback.print_exc()
                    return 1
            self._ar_cb = ALLREDUCE_FN(_cb)  # keep alive while the context may call it
            self.check(lib().seghdc_set_allreduce(self.h, C.cast(self._ar_cb, C.c_void_p), None, rank, nranks))
        self.rank, self.nranks = rank, nranks

    def cluster_sharded_async(self, k: int, iterations: int, early_stop: bool = False) -> None:
        self.check(lib().seghdc_cluster_sharded_async(self.h, k, iterations, int(early_stop)))

    def run_pipeline_sharded(self, img: np.ndarray, config: "RunConfig") -> dict:
        """run_pipeline over this rank's rows (seghdc_run_pipeline_sharded): labels of rows
        shard_rows(h, rank, nranks), and the final centroids/counts (identical on every rank)."""
        img = _img3(img)
        h, w, c = img.shape
        r0, r1 = shard_rows(h, getattr(self, "rank", 0), getattr(self, "nranks", 1))
        labels = np.empty((r1 - r0) * w, np.uint32)
        cents = np.empty((config.clusters, config.dim), np.uint32)
        counts = np.empty(config.clusters, np.uint64)
        rounds = _sz(0)
        timings = (C.c_double * 5)()
        self.check(lib().seghdc_run_pipeline_sharded(
            self.h, img, h, w, c, config.dim, float(config.alpha), config.beta, config.gamma, config.clusters,
            config.iterations, config.seed, ENCODERS[config.encoder], int(config.early_stop), labels.ctypes.data,
            cents.ctypes.data, counts.ctypes.data, C.byref(rounds), C.cast(timings, C.c_void_p)))
        names = ("encode_position", "encode_color", "produce_pixels", "cluster", "total")
        return {"labels": labels, "rows": (r0, r1), "centroids": cents, "counts": counts, "rounds": rounds.value,
                "timings": dict(zip(names, list(timings)))}

    # ---- row-block sharding: the caller all-reduces exchange_buffer() -------------------
    def shard_begin(self, k: int, iterations: int, early_stop: bool = False) -> None:
        self.check(lib().seghdc_shard_begin(self.h, k, iterations, int(early_stop)))

    def exchange_buffer(self):
        """(device pointer, number of int32) of the buffer to all-reduce (SUM) now."""
        p, n = C.c_void_p(), _sz()
        self.check(lib().seghdc_exchange_buffer(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def exchange_download(self) -> np.ndarray:
        _, n = self.exchange_buffer()
        out = np.zeros(n, np.int32)
        self.check(lib().seghdc_exchange_download(self.h, out.ctypes.data))
        return out

    def exchange_upload(self, data: np.ndarray) -> None:
        data = np.ascontiguousarray(data, np.int32)
        self.check(lib().seghdc_exchange_upload(self.h, data.ctypes.data))

    def shard_init_finish(self) -> None:
        self.check(lib().seghdc_shard_init_finish(self.h))

    def shard_assign(self, r: int) -> None:
        self.check(lib().seghdc_shard_assign(self.h, r))

    def shard_needs_exchange(self, r: int) -> bool:
        return bool(lib().seghdc_shard_round_needs_exchange(self.h, r))

    def shard_finish(self, r: int) -> None:
        self.check(lib().seghdc_shard_finish(self.h, r))


# ------------------------------------------------------------------------------------------
# run_pipeline configuration (pipeline.hpp:18-35)
# ------------------------------------------------------------------------------------------
@dataclasses.dataclass
class RunConfig:
    dim: int = 10000
    alpha: float = 0.2
    beta: int = 26
    gamma: int = 1
    clusters: int = 2
    iterations: int = 10
    seed: int = 0
    encoder: str = "manhattan"
    early_stop: bool = True

    def validate(self, h: int, w: int, channels: int) -> None:
        """RunConfig::validate (pipeline.cpp:25-30)."""
        if self.encoder not in ENCODERS:
            raise ConfigError(f"unknown encoder kind '{self.encoder}' (expected manhattan, rpos or rcolor)")
        _check(lib().seghdc_validate_run(self.dim, h, w, channels, float(self.alpha), self.beta, self.gamma,
                                         self.clusters, self.iterations))


@dataclasses.dataclass
class PipelineResult:
    mask: np.ndarray
    iterations_run: int
    timings: dict


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# module-level forms of the reference free functions (use the default device context)
def encode_image(img, dim, row, col, widened):
    return default_context().encode_image(img, dim, row, col, widened)


def select_initial_centroids(img, k):
    return default_context().select_initial_centroids(img, k)


def assign_labels(grid, h, w, dim, centroids):
    return default_context().assign_labels(grid, h, w, dim, centroids)


def update_centroids(grid, h, w, dim, labels, prev):
    return default_context().update_centroids(grid, h, w, dim, labels, prev)


def cluster(grid, img, dim, k, iterations=10, early_stop=True, on_iteration=None):
    return default_context().cluster(grid, img, dim, k, iterations, early_stop, on_iteration)


def run_pipeline(img, config: RunConfig = RunConfig(), on_iteration=None):
    return default_context().run_pipeline(img, config, on_iteration)
