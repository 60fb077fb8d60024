"""CPU, world_size 2 over gloo: the row-block sharding protocol of the multi-GPU path.

paper_2303_12753_b200.sharded.cluster_row_sharded (the product driver) runs unchanged with
gloo_allreduce (the product's host-staged collective) on two processes. The per-rank device
context is replaced by `ModelShard`, a numpy model of the device exchange semantics (seed bits
+ column sums at init; per round the sums of every cluster but the largest, member counts and
the change count; the skipped cluster derived as colsum - others, empty clusters keep their
centroid, early stop on an unchanged round). The merged result must equal the unsharded CPU
oracle bit for bit — the same property tests/test_gpu_sharding.py checks on the device."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle


def _bits(grid, dim):
    return np.unpackbits(np.ascontiguousarray(grid).view(np.uint8), axis=1, bitorder="little")[:, :dim].astype(np.int64)


class ModelShard:
    """numpy stand-in for Context's split-phase shard API on rows [r0, r1)."""

    def __init__(self, img, grid_rows, r0, dim):
        self.img, self.r0, self.dim = img, r0, dim
        self.w = img.shape[1]
        self.grid = grid_rows
        self.bits = _bits(grid_rows, dim)
        self.port = oracle.Port()
        self.device = 0

    def shard_begin(self, k, iterations, early_stop):
        self.k, self.iterations, self.early_stop = k, iterations, early_stop
        n_local = self.bits.shape[0]
        p0 = self.r0 * self.w
        seeds = self.port.select_seeds(self.img, k)
        seedbits = np.zeros((k, self.dim), np.int64)
        for c, s in enumerate(seeds):
            if p0 <= s < p0 + n_local:
                seedbits[c] = self.bits[s - p0]
        self.xchg = np.concatenate([seedbits.ravel(), np.zeros(k + 1, np.int64), self.bits.sum(0)]).astype(np.int32)
        self.labels = np.full(n_local, 0xFFFFFFFF, np.uint32)
        self.done, self.rounds = False, 0

    def exchange_download(self):
        return self.xchg.copy()

    def exchange_upload(self, data):
        self.xchg = np.asarray(data, np.int32).copy()

    def shard_init_finish(self):
        k, d = self.k, self.dim
        self.Z = self.xchg[: k * d].reshape(k, d).astype(np.uint32)
        self.colsum = self.xchg[k * d + k + 1:].astype(np.int64)
        self.cur = np.ones(k, np.uint32)
        self.xchg = self.xchg[: k * d + k + 1].copy()

    def shard_assign(self, r):
        if self.done:
            return
        k, d = self.k, self.dim
        self.rounds = r
        new = self.port.assign(self.grid, d, self.Z)
        skip = int(np.argmax(self.cur))  # largest current cluster, ties to the lowest index
        sums = np.zeros((k, d), np.int64)
        for c in range(k):
            if c != skip:
                sums[c] = self.bits[new == c].sum(0)
        counts = np.bincount(new, minlength=k)
        changed = int((new != self.labels).sum())
        self.labels = new
        self.skip = skip
        self.xchg = np.concatenate([sums.ravel(), counts, [changed]]).astype(np.int32)

    def shard_needs_exchange(self, r):
        return 1 <= r < self.iterations

    def shard_finish(self, r):
        if self.done:
            return
        k, d = self.k, self.dim
        sums = self.xchg[: k * d].reshape(k, d).astype(np.int64)
        counts = self.xchg[k * d: k * d + k].astype(np.int64)
        changed = int(self.xchg[k * d + k])
        if self.early_stop and r > 1 and changed == 0:
            self.done = True
            return
        others = sum(sums[c] for c in range(k) if c != self.skip)
        for c in range(k):
            if counts[c] == 0:
                continue
            self.Z[c] = (self.colsum - others) if c == self.skip else sums[c]
        self.cur = counts.astype(np.uint32)


def _worker(rank, world, port, cfg, q):
    import torch.distributed as dist

    from paper_2303_12753_b200.sharded import cluster_row_sharded, gloo_allreduce, row_ranges

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    img, grid, dim, k, iterations, early_stop = cfg
    h, w, _ = img.shape
    r0, r1 = row_ranges(h, world)[rank]
    shard = ModelShard(img, grid[r0 * w: r1 * w], r0, dim)
    cluster_row_sharded([shard], k, iterations, early_stop, gloo_allreduce())
    q.put((rank, shard.labels, shard.Z, shard.cur, shard.rounds))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("k,iterations,early_stop,seed", [(2, 6, False, 0), (3, 5, False, 1), (2, 12, True, 2),
                                                          (4, 4, False, 3)])
def test_gloo_row_sharding_matches_oracle(port, k, iterations, early_stop, seed):
    rng = np.random.default_rng(seed)
    h, w, dim = 12, 9, 1000
    img = (rng.integers(0, 4, (h, w, 3)) * 60).astype(np.uint8)
    cb = port.build_codebooks(dim, h, w, 3, 1.0, 2, 1, seed)
    grid = port.encode(img, dim, *cb)
    ref = port.cluster(grid, img, dim, k, iterations, early_stop)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pport = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, pport, (img, grid, dim, k, iterations, early_stop), q))
             for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    labels = np.concatenate([o[1] for o in out])
    assert (labels == ref["labels"]).all()
    for o in out:
        assert (o[2] == ref["centroids"]).all()
        assert (o[3] == ref["counts"]).all()
        assert o[4] == ref["rounds"]
