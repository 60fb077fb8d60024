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


# ------------------------------------------- the library's own sharded loop (C++, C-ABI)
def _pipeline_ref(ctx, port, img, cfg):
    """single-GPU run_pipeline + the oracle's labels/centroids of the same inputs"""
    h, w, c = img.shape
    single = ctx.run_pipeline(img, cfg)
    cb = S.build_codebooks(cfg.dim, h, w, c, cfg.alpha, cfg.beta, cfg.gamma, cfg.seed)
    exp = port.cluster(port.encode(img, cfg.dim, *cb), img, cfg.dim, cfg.clusters, cfg.iterations, cfg.early_stop)
    assert (single.mask.reshape(-1) == exp["labels"]).all()
    return exp


def test_nccl_single_rank_pipeline(ctx, port):
    """seghdc_nccl_init (libnccl.so.2 loaded at run time) with one rank: the library's sharded
    run_pipeline (one ncclAllReduce per round on the context's stream) equals the oracle."""
    img = S.synth_image(0, 3)[:120].copy()
    cfg = S.RunConfig(dim=10000, alpha=0.2, clusters=3, iterations=6, early_stop=False)
    exp = _pipeline_ref(ctx, port, img, cfg)
    c1 = S.Context(0)
    c1.nccl_init(S.nccl_unique_id(), 0, 1)
    for _ in range(3):  # eager, captured into a CUDA graph, replayed
        res = c1.run_pipeline_sharded(img, cfg)
        assert res["rows"] == (0, img.shape[0])
        assert (res["labels"] == exp["labels"]).all()
        assert (res["centroids"] == exp["centroids"]).all() and (res["counts"] == exp["counts"]).all()
        assert res["rounds"] == exp["rounds"]
    c1.close()


@pytest.mark.parametrize("world,k,dim", [(2, 2, 10000), (3, 4, 10000), (2, 8, 16384)])
def test_callback_collective_threads(ctx, port, world, k, dim):
    """`world` contexts on one device, each driven by its own host thread through
    seghdc_run_pipeline_sharded, with a host-staged all-reduce callback (seghdc_set_allreduce)
    that meets the other ranks at a barrier: the library's C++ round loop with a real exchange
    between independent callers. Kernels never wait on each other (the callback synchronises
    before the barrier). Labels of all row blocks together and the centroids on every rank
    equal the oracle's."""
    import threading

    import torch

    img = S.synth_image(0, 7)[:150].copy()
    cfg = S.RunConfig(dim=dim, alpha=1.0, clusters=k, iterations=5, early_stop=False)
    exp = _pipeline_ref(ctx, port, img, cfg)
    barrier = threading.Barrier(world)
    slots = [None] * world
    total = {}

    def make_fn(rank):
        def fn(ptr, n, stream):
            t = torch.as_tensor(_Dev(ptr, n), device="cuda:0")
            torch.cuda.synchronize()
            slots[rank] = t.cpu().numpy()
            if barrier.wait() == 0:
                total["sum"] = np.sum(np.stack(slots).astype(np.int64), axis=0).astype(np.uint32).view(np.int32)
            barrier.wait()
            t.copy_(torch.from_numpy(total["sum"].copy()))
            torch.cuda.synchronize()
            barrier.wait()  # nobody overwrites slots/total before every rank copied the sum back
        return fn

    ctxs = [S.Context(0) for _ in range(world)]
    for r, c in enumerate(ctxs):
        c.set_allreduce(make_fn(r), r, world)
    out = [None] * world

    def run(r):
        out[r] = ctxs[r].run_pipeline_sharded(img, cfg)

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    labels = np.concatenate([out[r]["labels"] for r in range(world)])
    assert (labels == exp["labels"]).all()
    for r in range(world):
        assert out[r]["rows"] == S.shard_rows(img.shape[0], r, world)
        assert (out[r]["centroids"] == exp["centroids"]).all() and (out[r]["counts"] == exp["counts"]).all()
    for c in ctxs:
        c.close()


class _Dev:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False), "version": 3}


_WORKER = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["SEGHDC_ROOT"])
import paper_2303_12753_b200 as S
from paper_2303_12753_b200.sharded import gloo_collective
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
img = S.synth_image(1, 0)[:160].copy()
cfg = S.RunConfig(dim=10000, alpha=0.2, clusters=2, iterations=6, early_stop=True)
ctx = S.Context(0)
ctx.set_allreduce(gloo_collective(), rank, world)
res = ctx.run_pipeline_sharded(img, cfg)
np.savez(os.path.join(os.environ["SEGHDC_OUT"], f"rank{rank}.npz"), labels=res["labels"], rows=np.array(res["rows"]),
         centroids=res["centroids"], counts=res["counts"], rounds=res["rounds"])
ctx.close()
dist.destroy_process_group()
"""


def test_two_processes_gloo(port, tmp_path):
    """Two processes on cuda:0, each with its own real Context, run the library's sharded
    run_pipeline with a host-staged gloo all-reduce between them (world_size 2): labels of
    the two row blocks together, and both ranks' centroids, equal the oracle's."""
    import os
    import socket
    import subprocess
    import sys

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no),
                   SEGHDC_ROOT=root, SEGHDC_OUT=str(tmp_path))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env))
    for p in procs:
        assert p.wait(timeout=600) == 0
    img = S.synth_image(1, 0)[:160].copy()
    h, w, c = img.shape
    cb = S.build_codebooks(10000, h, w, c, 0.2, 26, 1, 0)
    exp = port.cluster(port.encode(img, 10000, *cb), img, 10000, 2, 6, True)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    assert (np.concatenate([p["labels"] for p in parts]) == exp["labels"]).all()
    for p in parts:
        assert (p["centroids"] == exp["centroids"]).all() and (p["counts"] == exp["counts"]).all()
        assert int(p["rounds"]) == exp["rounds"]


def test_cpp_dropin_sharded_pipeline(tmp_path):
    """A C++ caller of the drop-in's run_pipeline_sharded (NCCL, one rank) against run_pipeline."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2303_12753_b200", "lib")
    exe = tmp_path / "sharded_pipeline"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "sharded_pipeline.cpp"), "-o", str(exe), "-L", lib,
                    "-lseghdc_b200", "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}",
                    "-Wl,-rpath,/usr/local/cuda/lib64"], check=True)
    out = subprocess.run([str(exe), "96", "130", "3", "3", "5"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().splitlines()[-1] == "ok", out.stdout + out.stderr  # NCCL may print a banner


def test_c3_row_sharded_library_loop_matches_reference_golden(golden_configs):
    """BASELINE config C3 at full size (2048^2 x 3, D = 10000, K = 4, 20 rounds) row-sharded over
    3 callers of seghdc_run_pipeline_sharded (host-staged callback collective): the row blocks
    together and every rank's centroids equal the reference's golden."""
    import hashlib
    import threading

    import torch

    g, spec = golden_configs["C3"], golden_configs["_meta"]["configs"]["C3"]
    img = S.synth_image(3, 0)
    cfg = S.RunConfig(dim=spec["dim"], alpha=spec["alpha"], clusters=spec["k"], iterations=spec["iterations"],
                      early_stop=False)
    world = 3
    barrier = threading.Barrier(world)
    slots, total = [None] * world, {}

    def make_fn(rank):
        def fn(ptr, n, stream):
            t = torch.as_tensor(_Dev(ptr, n), device="cuda:0")
            torch.cuda.synchronize()
            slots[rank] = t.cpu().numpy()
            if barrier.wait() == 0:
                total["sum"] = np.sum(np.stack(slots).astype(np.int64), axis=0).astype(np.uint32).view(np.int32)
            barrier.wait()
            t.copy_(torch.from_numpy(total["sum"].copy()))
            torch.cuda.synchronize()
            barrier.wait()
        return fn

    ctxs = [S.Context(0) for _ in range(world)]
    for r, c in enumerate(ctxs):
        c.set_allreduce(make_fn(r), r, world)
    out = [None] * world
    ths = [threading.Thread(target=lambda r=r: out.__setitem__(r, ctxs[r].run_pipeline_sharded(img, cfg)))
           for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    labels = np.concatenate([out[r]["labels"] for r in range(world)]).astype(np.uint32)
    assert hashlib.sha256(labels.tobytes()).hexdigest() == g["labels_sha256"]
    for r in range(world):
        assert hashlib.sha256(out[r]["centroids"].astype(np.uint32).tobytes()).hexdigest() == g["centroids_sha256"]
        assert out[r]["counts"].tolist() == g["counts"]
    for c in ctxs:
        c.close()
