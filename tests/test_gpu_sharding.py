"""GPU: row-block sharding (the multi-GPU path) emulated on one device.

G contexts each hold one contiguous slab of pixel rows, run the split-phase C-ABI
(shard_begin / shard_assign / shard_finish) in lock step, and exchange through a host-staged
SUM (host_sum_allreduce) instead of NCCL. Kernels never wait on each other (each launch runs
to completion before the host sums), so this is legal on one GPU. The merged result must
equal the single-device run bit for bit: integer sums are order independent."""
import numpy as np
import pytest

import paper_2303_12753_b200 as S
from paper_2303_12753_b200.sharded import cluster_row_sharded, host_sum_allreduce, row_ranges

pytestmark = pytest.mark.gpu


def _sharded(img, dim, alpha, k, iterations, early_stop, world):
    h, w, c = img.shape
    cb = S.build_codebooks(dim, h, w, c, alpha, 26, 1, 0)
    ctxs = []
    for r0, r1 in row_ranges(h, world):
        ctx = S.Context(0)
        ctx.load_image(img)
        ctx.load_codebooks(dim, *cb)
        ctx.encode_async(r0, r1)
        ctxs.append(ctx)
    cluster_row_sharded(ctxs, k, iterations, early_stop, host_sum_allreduce)
    parts = [c.fetch_results((r1 - r0) * w, k, dim) for c, (r0, r1) in zip(ctxs, row_ranges(h, world))]
    for c in ctxs:
        c.close()
    labels = np.concatenate([p["labels"] for p in parts])
    for p in parts[1:]:
        assert (p["centroids"] == parts[0]["centroids"]).all()
        assert (p["counts"] == parts[0]["counts"]).all() and p["rounds"] == parts[0]["rounds"]
    return labels, parts[0]


@pytest.mark.parametrize("cid,dim,alpha,k,iterations,world", [
    (0, 10000, 0.2, 2, 10, 2), (0, 10000, 0.2, 2, 10, 3), (1, 10000, 0.2, 2, 6, 4),
    (0, 10000, 0.2, 4, 5, 2), (0, 16384, 1.0, 8, 3, 2), (0, 2048, 1.0, 1, 3, 2),
])
def test_row_sharded_equals_single_device(ctx, cid, dim, alpha, k, iterations, world):
    img = S.synth_image(cid, 0)
    h, w, c = img.shape
    cb = S.build_codebooks(dim, h, w, c, alpha, 26, 1, 0)
    ctx.encode_image(img, dim, *cb, download=False)
    ref = ctx.cluster(None, img, dim, k, iterations, False)
    labels, part = _sharded(img, dim, alpha, k, iterations, False, world)
    assert (labels == ref["labels"]).all()
    assert (part["centroids"] == ref["centroids"]).all()
    assert (part["counts"] == ref["counts"]).all() and part["rounds"] == ref["rounds"]


def test_row_sharded_early_stop(ctx):
    img = S.synth_image(0, 5)
    h, w, c = img.shape
    cb = S.build_codebooks(10000, h, w, c, 0.2, 26, 1, 0)
    ctx.encode_image(img, 10000, *cb, download=False)
    ref = ctx.cluster(None, img, 10000, 2, 10, True)
    labels, part = _sharded(img, 10000, 0.2, 2, 10, True, 2)
    assert part["rounds"] == ref["rounds"] < 10
    assert (labels == ref["labels"]).all() and (part["centroids"] == ref["centroids"]).all()
