"""Row-block sharding of one image across ranks (one process per GPU).

Each rank holds the full image (50 MB at 4096^2x3) and the codebooks, encodes only its
contiguous slab of pixel rows (the grid is row-major, so a shard is one contiguous slab) and
runs seed selection redundantly on the full image, so seeding needs no communication. The
only collective is one SUM all-reduce per round of the exchange buffer
``[k*Dp centroid sums | k member counts | changed]`` (plus the column sums once at init).
Integer sums are order independent, so every rank finalises bit-identical centroids, and
the result equals the single-device run bit for bit (tests/test_sharding*.py).

The collective is injected: :func:`nccl_allreduce` (torch.distributed over NCCL/NVLink,
zero-copy on the context's exchange buffer) for real multi-GPU runs, or a host-staged sum
for gloo / single-device emulation.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from . import Context


def row_ranges(h: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks, sizes differing by at most one row (earlier ranks larger)."""
    if world < 1 or world > h:
        raise ValueError(f"cannot split {h} rows over {world} ranks")
    base, extra = divmod(h, world)
    out, r = [], 0
    for i in range(world):
        n = base + (1 if i < extra else 0)
        out.append((r, r + n))
        r += n
    return out


def cluster_row_sharded(ctxs: Sequence[Context], k: int, iterations: int, early_stop: bool,
                        allreduce: Callable[[Sequence[Context]], None]) -> None:
    """Drive the split-phase C-ABI on ``ctxs`` (this process's shards) in lock step.

    ``allreduce(ctxs)`` must leave every shard's current exchange buffer equal to the SUM over
    all shards of all ranks. Results stay on the devices (Context.fetch_results)."""
    for c in ctxs:
        c.shard_begin(k, iterations, early_stop)
    allreduce(ctxs)
    for c in ctxs:
        c.shard_init_finish()
    for r in range(1, iterations + 1):
        for c in ctxs:
            c.shard_assign(r)
        if ctxs[0].shard_needs_exchange(r):
            allreduce(ctxs)
            for c in ctxs:
                c.shard_finish(r)


def host_sum_allreduce(ctxs: Sequence[Context]) -> None:
    """All shards live in this process: sum their exchange buffers on the host (int32 wraps
    exactly like the device's u32 arithmetic) and write the sum back to each."""
    total = None
    for c in ctxs:
        buf = c.exchange_download()
        total = buf.copy() if total is None else (total + buf).astype(np.int32)
    for c in ctxs:
        c.exchange_upload(total)


class _CudaArray:
    """Minimal __cuda_array_interface__ view of a device buffer (zero-copy into torch)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False), "version": 3}


def _sum_local(ctxs: Sequence[Context]) -> np.ndarray:
    """Exchange buffers of this process's shards, summed on the host (int32 wraps exactly like
    the device's u32 arithmetic)."""
    total = None
    for c in ctxs:
        buf = c.exchange_download()
        total = buf.copy() if total is None else (total + buf).astype(np.int32)
    return total


def nccl_allreduce(group=None) -> Callable[[Sequence[Context]], None]:
    """torch.distributed all-reduce (SUM) of the exchange buffer. One shard per process (the
    normal case): zero-copy on the context's buffer, on its stream (set it to torch's current
    stream with Context.set_stream first). Several shards in one process: their buffers are
    summed locally first, all-reduced once, and the total written back to every shard, so the
    result is the SUM over all shards of all ranks."""
    import torch
    import torch.distributed as dist

    def _ar(ctxs: Sequence[Context]) -> None:
        if len(ctxs) == 1:
            c = ctxs[0]
            ptr, n = c.exchange_buffer()
            t = torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{c.device}")
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            return
        total = torch.from_numpy(_sum_local(ctxs)).to(f"cuda:{ctxs[0].device}")
        dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)
        host = total.cpu().numpy()
        for c in ctxs:
            c.exchange_upload(host)

    return _ar


def gloo_allreduce(group=None) -> Callable[[Sequence[Context]], None]:
    """Host-staged all-reduce over a CPU process group (gloo); local shards summed first."""
    import torch
    import torch.distributed as dist

    def _ar(ctxs: Sequence[Context]) -> None:
        buf = torch.from_numpy(_sum_local(ctxs))
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        for c in ctxs:
            c.exchange_upload(buf.numpy())

    return _ar


def gloo_collective(group=None) -> Callable[[int, int, int], None]:
    """A seghdc_allreduce_fn for Context.set_allreduce: the library's own sharded loop
    (seghdc_run_pipeline_sharded / seghdc_cluster_sharded_async) with a host-staged gloo
    all-reduce — device buffer to host, SUM over the CPU process group, back to the device."""
    import torch
    import torch.distributed as dist

    def _fn(ptr: int, n: int, stream: int) -> None:
        dev = torch.cuda.current_device()
        t = torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{dev}")
        torch.cuda.synchronize(dev)  # the context's stream produced the buffer
        host = t.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        t.copy_(host)
        torch.cuda.synchronize(dev)

    return _fn
