"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the reference's goldens.

Bit-exact for everything (labels, centroids, member counts, rounds, seeds, grid words): the
path is integer-only (no floating point anywhere in assignment)."""
import hashlib

import numpy as np
import pytest

import paper_2303_12753_b200 as S
from conftest import instance_arrays

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- reference suites' instances
def test_bruteforce_instances(ctx, golden_instances):
    """test_clusterer.cpp:211-235 and acceptance criterion 5: per-round labels of 60 tiny
    instances (<= 16 px, d <= 32, k <= 3) equal the reference's brute-force oracle."""
    for inst in golden_instances:
        img, grid = instance_arrays(inst)
        rounds = []
        res = ctx.cluster(grid, img, inst["dim"], inst["k"], inst["iterations"], False,
                          on_iteration=lambda r, lab: rounds.append(lab.tolist()))
        assert rounds == inst["expected_rounds"], (inst["suite"], inst["instance"])
        assert res["rounds"] == inst["iterations"]
        assert ctx.select_initial_centroids(img, inst["k"]).tolist() == inst["seeds"]


# ---------------------------------------------------------------- encode
@pytest.mark.parametrize("dim,h,w,c,enc,beta", [
    (10000, 40, 37, 3, "manhattan", 26), (10000, 23, 50, 1, "manhattan", 3), (16384, 20, 21, 3, "manhattan", 26),
    (999, 9, 13, 3, "rpos", 2), (1001, 7, 5, 3, "rcolor", 1), (2048, 8, 8, 3, "manhattan", 2), (600, 1, 1, 1, "manhattan", 1),
    (4096, 16, 16, 1, "manhattan", 1), (31000, 6, 7, 3, "manhattan", 2),
])
def test_encode_matches_reference(ctx, port, dim, h, w, c, enc, beta):
    rng = np.random.default_rng(dim + h)
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    cb = S.build_codebooks(dim, h, w, c, 1.0, beta, 1, 7, enc)
    grid = ctx.encode_image(img, dim, *cb)
    assert (grid == port.encode(img, dim, *cb)).all()


@pytest.mark.parametrize("dim,h,w,c,overlap", [
    (1000, 9, 70, 3, "all"),      # every channel non-zero in every word: three lookups per word (nl = 3)
    (2100, 5, 3, 3, "pairs"),     # channels 0/1 share the low words, 1/2 the high ones (nl = 2 everywhere)
    (4200, 130, 9, 3, "disjoint"),  # the reference's structure; rows beyond one staged batch, a ragged 9-column tile
    (777, 3, 131, 1, "all"),      # one channel, three column tiles, the last ragged
])
def test_encode_with_arbitrary_caller_tables(ctx, port, dim, h, w, c, overlap):
    """seghdc_encode takes the caller's tables as they are: the kernel's one-lookup-per-word fast
    path must stay exact when the widened colour tables are NOT channel-disjoint (it derives the
    channel set of every word from the tables). Checked against a direct numpy XOR, and the fused
    column sums (cluster 0 = column sums - cluster 1) through two rounds on the resident grid."""
    rng = np.random.default_rng(dim + w)
    wph = (dim + 63) // 64
    tail = np.uint64((1 << (dim % 64)) - 1) if dim % 64 else np.uint64(0xFFFFFFFFFFFFFFFF)

    def rand(n):
        t = rng.integers(0, 1 << 63, (n, wph), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, (n, wph), dtype=np.uint64)
        t[:, -1] &= tail
        return t

    row, col, wid = rand(h), rand(w), rand(c * 256).reshape(c, 256, wph)
    if overlap != "all" and c == 3:
        third = wph // 3
        keep = np.zeros((3, wph), bool)
        if overlap == "pairs":
            keep[0, : wph // 2], keep[1, :], keep[2, wph // 2:] = True, True, True
        else:
            keep[0, :third], keep[1, third: 2 * third], keep[2, 2 * third:] = True, True, True
        wid = wid * keep[:, None, :].astype(np.uint64)
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    grid = ctx.encode_image(img, dim, row, col, wid)
    exp = (row[:, None, :] ^ col[None, :, :]).reshape(h * w, wph)
    for ch in range(c):
        exp = exp ^ wid[ch][img[:, :, ch].reshape(-1)]
    assert (grid == exp).all()
    res = ctx.cluster(None, img, dim, 2, 2, False)
    ref = port.cluster(exp, img, dim, 2, 2, False)
    assert (res["labels"] == ref["labels"]).all() and (res["centroids"] == ref["centroids"]).all()
    assert (res["counts"] == ref["counts"]).all()


# ---------------------------------------------------------------- assign / update
def _rand_grid(rng, n, dim, density=0.5):
    bits = (rng.random((n, dim)) < density).astype(np.uint8)
    pad = (-dim) % 64
    bits = np.concatenate([bits, np.zeros((n, pad), np.uint8)], axis=1)
    return np.packbits(bits.reshape(n, -1, 8)[:, :, ::-1], axis=2).reshape(n, -1).view("<u8").copy()


@pytest.mark.parametrize("dim,k,zmax", [(10000, 2, 1 << 19), (10000, 2, 3), (333, 1, 10), (10000, 4, 1 << 22),
                                         (16384, 8, 1 << 24), (777, 3, 1000), (64, 9, 50), (40000, 2, 1 << 20),
                                         (10000, 17, 1 << 16), (5000, 5, (1 << 32) - 1)])
def test_assign_matches_oracle(ctx, port, dim, k, zmax):
    rng = np.random.default_rng(dim * 31 + k)
    h, w = 37, 41
    grid = _rand_grid(rng, h * w, dim)
    z = rng.integers(0, zmax, (k, dim), dtype=np.uint64).astype(np.uint32)
    if k > 2:
        z[1] = z[0]          # exact tie: lower index wins
        z[2] = z[0] * 3      # magnitude invariance (clusterer.hpp:27-28)
    lab = ctx.assign_labels(grid, h, w, dim, z)
    assert (lab == port.assign(grid, dim, z)).all()
    # how often the reference's unsigned __int128 comparison wrapped (zmax = 2^32 - 1 wraps)
    assert ctx.round_wraps() == port.last_wraps()


def test_assign_zero_centroid_and_ties(ctx, port):
    # strictly_closer edge rules (clusterer.cpp:43-44) and test_clusterer.cpp:82-104
    dim = 8
    grid = np.array([[0b00000011], [0b00001100]], np.uint64)
    z = np.array([[1, 1, 0, 0, 0, 0, 0, 0], [0, 0, 1, 1, 0, 0, 0, 0]], np.uint32)
    assert ctx.assign_labels(grid, 1, 2, dim, z).tolist() == [0, 1]
    tie = np.array([[1, 0, 1, 0, 0, 0, 0, 0]] * 2, np.uint32)
    assert ctx.assign_labels(grid, 1, 2, dim, tie).tolist() == [0, 0]
    zero = np.zeros((3, dim), np.uint32)
    zero[2, 0] = 5
    assert (ctx.assign_labels(grid, 1, 2, dim, zero) == port.assign(grid, dim, zero)).all()


@pytest.mark.parametrize("dim,k", [(10000, 2), (10000, 4), (16384, 8), (100, 3), (40000, 2), (7, 1)])
def test_update_matches_oracle(ctx, port, dim, k):
    rng = np.random.default_rng(dim + k)
    h, w = 53, 61
    grid = _rand_grid(rng, h * w, dim, density=0.3)
    labels = rng.integers(0, max(1, k - 1), h * w, dtype=np.uint32)  # cluster k-1 stays empty
    prev = rng.integers(0, 1000, (k, dim), dtype=np.uint32)
    z, counts = ctx.update_centroids(grid, h, w, dim, labels, prev)
    z2, c2 = port.update(grid, dim, labels, prev)
    assert (z == z2).all() and (counts == c2).all()
    # update example of test_clusterer.cpp:124-149 ({1100,1010} -> (2,1,1,0), empty keeps previous)
    g = np.array([[0b0011], [0b0101]], np.uint64)
    zz, cc = ctx.update_centroids(g, 1, 2, 4, np.array([0, 0], np.uint32), np.array([[0, 0, 0, 1], [1, 1, 1, 1]], np.uint32))
    assert zz.tolist() == [[2, 1, 1, 0], [1, 1, 1, 1]] and cc.tolist() == [2, 0]


def test_update_rejects_rogue_label(ctx):
    g = np.array([[0b0011], [0b0101]], np.uint64)
    with pytest.raises(S.ConfigError):
        ctx.update_centroids(g, 1, 2, 4, np.array([0, 7], np.uint32), np.zeros((2, 4), np.uint32))


# ---------------------------------------------------------------- seeds
def test_seed_selection(ctx, port):
    img = np.zeros((1, 4, 1), np.uint8)
    img[0, :, 0] = [0, 100, 255, 120]
    assert ctx.select_initial_centroids(img, 3).tolist() == [0, 2, 3]  # test_clusterer.cpp:70-80
    uni = np.full((3, 4, 3), 128, np.uint8)
    assert ctx.select_initial_centroids(uni, 5).tolist() == [0, 3, 8, 11, 1]  # :51-61
    img2 = np.full((2, 2, 1), 50, np.uint8)
    img2[0, 1] = img2[1, 0] = 7
    assert ctx.select_initial_centroids(img2, 1).tolist() == [1]  # :41-49
    rng = np.random.default_rng(3)
    for t in range(8):
        im = rng.integers(0, 6 if t % 2 else 256, (31, 29, 3 if t < 4 else 1), dtype=np.uint8)
        for k in (1, 2, 3, 7, 12):
            assert (ctx.select_initial_centroids(im, k) == port.select_seeds(im, k)).all(), (t, k)
    with pytest.raises(S.ConfigError):
        ctx.select_initial_centroids(uni, 13)


# ---------------------------------------------------------------- full loop, random
@pytest.mark.parametrize("case", range(12))
def test_cluster_random_vs_oracle(ctx, port, case):
    rng = np.random.default_rng(1000 + case)
    h, w = int(rng.integers(5, 90)), int(rng.integers(5, 90))
    c = int(rng.choice([1, 3]))
    dim = int(rng.choice([800, 1024, 2000, 10000, 16384]))
    k = int(rng.integers(1, 7))
    iterations = int(rng.integers(1, 9))
    es = bool(case % 2)
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    if case % 3 == 0:
        img = (img // 64) * 64  # many colour ties
    alpha = 1.0
    beta = int(rng.integers(1, 5))
    cb = S.build_codebooks(dim, h, w, c, alpha, beta, 1, case)
    grid = port.encode(img, dim, *cb)
    got_rounds = []
    res = ctx.cluster(grid, img, dim, k, iterations, es, on_iteration=lambda r, lab: got_rounds.append(lab))
    exp = port.cluster(grid, img, dim, k, iterations, es, per_round=True)
    assert res["rounds"] == exp["rounds"]
    assert len(got_rounds) == exp["rounds"]
    for r in range(exp["rounds"]):
        assert (got_rounds[r] == exp["labels_rounds"][r]).all(), r
    assert (res["labels"] == exp["labels"]).all()
    assert (res["centroids"] == exp["centroids"]).all()
    assert (res["counts"] == exp["counts"]).all()
    # the same call without a callback runs with no host synchronisation between rounds
    res2 = ctx.cluster(None, img, dim, k, iterations, es)
    assert res2["rounds"] == exp["rounds"] and (res2["labels"] == exp["labels"]).all()
    assert (res2["centroids"] == exp["centroids"]).all()
    assert ctx.round_wraps() == port.last_wraps()


# ------------------------------------------------- K <= 8: 4-CTA dimension-split tcgen05 layout
@pytest.mark.parametrize("dim,k,h,w,c,its,es", [
    (3300, 8, 40, 37, 3, 4, False),     # 4 chunks: one per CTA of the cluster
    (5000, 7, 61, 53, 1, 5, True),      # 5 chunks: 1, 1, 1, 2
    (10000, 5, 97, 131, 3, 6, False),   # 10 chunks: 2, 3, 2, 3; ~100 tiles
    (16384, 8, 120, 150, 3, 4, False),  # the C4 shape: 16 chunks, 4 per CTA
    (16384, 2, 9, 11, 3, 3, True),      # K = 2 too wide for the one-CTA layout; fewer tiles than clusters
    (16384, 3, 50, 40, 1, 3, False),
])
def test_cluster_split_layout_vs_oracle(ctx, port, dim, k, h, w, c, its, es):
    """The K <= 8 layout (72 digit columns, a cluster of 4 CTAs each owning a quarter of the HV
    dimensions, partial dots combined in distributed shared memory) against the oracle."""
    rng = np.random.default_rng(dim + 31 * k + h)
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    img[: h // 2] //= 4
    cb = S.build_codebooks(dim, h, w, c, 1.0, 3, 1, k)
    grid = port.encode(img, dim, *cb)
    got = []
    res = ctx.cluster(grid, img, dim, k, its, es, on_iteration=lambda r, lab: got.append(lab))
    assert ctx.round_kernel == "k_round_tc"
    exp = port.cluster(grid, img, dim, k, its, es, per_round=True)
    assert res["rounds"] == exp["rounds"]
    for r in range(exp["rounds"]):
        assert (got[r] == exp["labels_rounds"][r]).all(), r
    assert (res["centroids"] == exp["centroids"]).all()
    assert (res["counts"] == exp["counts"]).all()


@pytest.mark.parametrize("k,dim", [(2, 10000), (8, 16384)])
def test_sm_budget_and_concurrent_contexts(port, k, dim):
    """Contexts with an SM budget on separate streams (bench --config 2) give the oracle's results."""
    import torch
    rng = np.random.default_rng(k)
    imgs = [rng.integers(0, 256, (48, 57, 3), dtype=np.uint8) for _ in range(3)]
    cb = S.build_codebooks(dim, 48, 57, 3, 1.0, 2, 1, 0)
    ctxs, streams = [], []
    for j in range(3):
        c = S.Context(0)
        st = torch.cuda.Stream()
        c.set_stream(st.cuda_stream)
        c.set_sm_budget(13 + 20 * j)
        c.load_image(imgs[j])
        c.load_codebooks(dim, *cb)
        ctxs.append(c)
        streams.append(st)
    for c, im in zip(ctxs, imgs):
        c.encode_async(0, 48)
        c.cluster_async(k, 4, False)
    for c, im in zip(ctxs, imgs):
        res = c.fetch_results(48 * 57, k, dim)
        exp = port.cluster(port.encode(im, dim, *cb), im, dim, k, 4, False)
        assert (res["labels"] == exp["labels"]).all()
        assert (res["centroids"] == exp["centroids"]).all()
    with pytest.raises(S.ConfigError):
        ctxs[0].set_sm_budget(-1)
    for c in ctxs:
        c.close()


def test_k1_stops_at_round_two(ctx, port):
    # test_clusterer.cpp:168-174
    img = np.full((2, 2, 1), 10, np.uint8)
    grid = _rand_grid(np.random.default_rng(10), 4, 16)
    res = ctx.cluster(grid, img, 16, 1, 10, True)
    assert res["rounds"] == 2 and res["labels"].tolist() == [0, 0, 0, 0]


def test_cluster_validation(ctx):
    img = np.zeros((2, 2, 1), np.uint8)
    grid = np.zeros((4, 1), np.uint64)
    with pytest.raises(S.ConfigError):
        ctx.cluster(grid, img, 16, 5, 10, True)
    with pytest.raises(S.ConfigError):
        ctx.cluster(grid, img, 16, 1, 0, True)


# ---------------------------------------------------------------- BASELINE.json configs
def _config_run(ctx, golden_configs, name, image_seed=0, iterations=None, early_stop=False):
    spec = golden_configs["_meta"]["configs"][name]
    img = S.synth_image(spec["cid"], image_seed)
    h, w, c = img.shape
    cb = S.build_codebooks(spec["dim"], h, w, c, spec["alpha"], 26, 1, 0)
    ctx.encode_image(img, spec["dim"], *cb, download=False)
    rounds = []
    res = ctx.cluster(None, img, spec["dim"], spec["k"], iterations or spec["iterations"], early_stop,
                      on_iteration=lambda r, lab: rounds.append(sha(lab)))
    return img, res, rounds


@pytest.mark.parametrize("name", ["C0", "C1"])
def test_config_golden_reference(ctx, golden_configs, name):
    """C0/C1 goldens come from the reference library itself (tests/golden/make_golden.py)."""
    g = golden_configs[name]
    img, res, rounds = _config_run(ctx, golden_configs, name)
    assert sha(img) == g["image_sha256"]
    assert rounds == g["round_labels_sha256"]
    assert sha(res["labels"]) == g["labels_sha256"]
    assert sha(res["centroids"]) == g["centroids_sha256"]
    assert res["counts"].tolist() == g["counts"] and res["rounds"] == g["rounds"]
    _, es, _ = _config_run(ctx, golden_configs, name, early_stop=True)
    assert es["rounds"] == g["early_stop_rounds"] and sha(es["labels"]) == g["early_stop_labels_sha256"]


def test_config_c2_batch(ctx, golden_configs):
    spec = golden_configs["_meta"]["configs"]["C2"]
    for s, g in enumerate(golden_configs["C2"]["images"]):
        img = S.synth_image(2, s)
        h, w, c = img.shape
        cb = S.build_codebooks(spec["dim"], h, w, c, spec["alpha"], 26, 1, 0)
        ctx.encode_image(img, spec["dim"], *cb, download=False)
        res = ctx.cluster(None, img, spec["dim"], spec["k"], spec["iterations"], False)
        assert sha(res["labels"]) == g["labels_sha256"], s
        assert sha(res["centroids"]) == g["centroids_sha256"], s
        assert res["counts"].tolist() == g["counts"], s


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_config_large_golden(ctx, golden_configs, name):
    """C3 / C4 at their full 20 rounds against the reference itself (make_golden_full.py): every
    round's labels, the final centroids and counts, and the per-round number of comparisons
    whose 128-bit products wrapped (C4 wraps: clusters of millions of pixels)."""
    g = golden_configs[name]
    img, res, rounds = _config_run(ctx, golden_configs, name, iterations=g["iterations"])
    assert sha(img) == g["image_sha256"]
    assert rounds == g["round_labels_sha256"]
    assert sha(res["centroids"]) == g["centroids_sha256"]
    assert res["counts"].tolist() == g["counts"]
    if "round_wraps" in g:
        assert ctx.round_wraps() == g["round_wraps"]


# ---------------------------------------------------------------- run_pipeline (closed-form codebooks)
@pytest.mark.parametrize("dim,h,w,c,enc,alpha,beta,gamma,k,its,seed", [
    (10000, 30, 41, 1, "manhattan", 1.0, 26, 1, 2, 6, 0), (10000, 64, 80, 3, "manhattan", 1.0, 26, 1, 2, 5, 3),
    (2003, 17, 19, 3, "manhattan", 1.0, 3, 2, 3, 4, 11), (4096, 12, 9, 1, "manhattan", 0.5, 1, 4, 2, 7, 5),
    (1500, 10, 11, 3, "rpos", 1.0, 2, 1, 2, 4, 9), (1500, 10, 11, 3, "rcolor", 1.0, 2, 1, 2, 4, 9),
    (16384, 21, 23, 3, "manhattan", 1.0, 5, 1, 4, 3, 1),
])
def test_run_pipeline_matches_oracle(ctx, port, dim, h, w, c, enc, alpha, beta, gamma, k, its, seed):
    """run_pipeline (pipeline.cpp:40-75): the Manhattan codebooks are expanded on the device from
    their bases; labels and rounds equal the oracle's encode + cluster of the host-built tables."""
    rng = np.random.default_rng(dim + h * w + seed)
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    img[: h // 2] //= 4  # a dark half: two clear clusters
    cfg = S.RunConfig(dim=dim, alpha=alpha, beta=beta, gamma=gamma, clusters=k, iterations=its, seed=seed,
                      encoder=enc, early_stop=False)
    res = ctx.run_pipeline(img, cfg)
    cb = S.build_codebooks(dim, h, w, c, alpha, beta, gamma, seed, enc)
    exp = port.cluster(port.encode(img, dim, *cb), img, dim, k, its, False)
    assert res.iterations_run == exp["rounds"]
    assert (res.mask.reshape(-1) == exp["labels"]).all()


def test_run_pipeline_c1_golden(ctx, golden_configs):
    """The bench's end-to-end call on config C1 reproduces the reference's golden labels."""
    g, spec = golden_configs["C1"], golden_configs["_meta"]["configs"]["C1"]
    img = S.synth_image(1, 0)
    cfg = S.RunConfig(dim=spec["dim"], alpha=spec["alpha"], beta=26, gamma=1, clusters=spec["k"],
                      iterations=spec["iterations"], seed=0, early_stop=False)
    res = ctx.run_pipeline(img, cfg)
    assert sha(res.mask.astype(np.uint32).reshape(-1)) == g["labels_sha256"] and res.iterations_run == g["rounds"]
    cfg.early_stop = True
    res = ctx.run_pipeline(img, cfg)
    assert sha(res.mask.astype(np.uint32).reshape(-1)) == g["early_stop_labels_sha256"]
    assert res.iterations_run == g["early_stop_rounds"]


@pytest.mark.parametrize("enc,n", [("manhattan", 11), ("rpos", 3)])
def test_run_pipeline_batch_equals_single_calls(ctx, golden_configs, enc, n):
    """seghdc_run_pipeline_batch (images side by side on child streams, one host sync) gives
    every image the labels and rounds of its own run_pipeline call; C2 images 0-3 also match
    the reference's goldens."""
    imgs = [S.synth_image(2, s) for s in range(n)]
    cfg = S.RunConfig(dim=10000, alpha=0.2, clusters=2, iterations=10, early_stop=False, encoder=enc)
    for _ in range(2):  # second call: every child context replays its CUDA graph
        labels, rounds = ctx.run_pipeline_batch(imgs, cfg)
        for j, im in enumerate(imgs):
            one = ctx.run_pipeline(im, cfg)
            assert (labels[j] == one.mask).all() and rounds[j] == one.iterations_run, j
            if enc == "manhattan" and j < 4:
                assert sha(labels[j].astype(np.uint32).reshape(-1)) == golden_configs["C2"]["images"][j]["labels_sha256"]


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_run_pipeline_large_golden(ctx, golden_configs, name):
    """The end-to-end call (run_pipeline: device codebooks, encode, seeds, 20 rounds as one CUDA
    graph from the second call on) at BASELINE sizes against the reference's goldens."""
    g, spec = golden_configs[name], golden_configs["_meta"]["configs"][name]
    img = S.synth_image(spec["cid"], 0)
    cfg = S.RunConfig(dim=spec["dim"], alpha=spec["alpha"], beta=26, gamma=1, clusters=spec["k"],
                      iterations=spec["iterations"], seed=0, early_stop=False)
    for _ in range(2):  # eager, then captured
        res = ctx.run_pipeline(img, cfg)
        assert sha(res.mask.astype(np.uint32).reshape(-1)) == g["labels_sha256"]
        assert res.iterations_run == g["rounds"]


def test_run_pipeline_graph_switches(ctx, port):
    """run_pipeline's CUDA-graph cache across changing call signatures: shape A (eager, then
    captured, then replayed), shape B, back to A, then A with a per-round callback (eager path,
    labels of every round) and with a pageable label buffer — every result equals the oracle."""
    def case(h, w, c, k, its, seed):
        rng = np.random.default_rng(seed)
        img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
        img[: h // 2] //= 4
        cfg = S.RunConfig(dim=4096, alpha=1.0, beta=3, gamma=1, clusters=k, iterations=its, seed=seed,
                          early_stop=False)
        cb = S.build_codebooks(4096, h, w, c, 1.0, 3, 1, seed)
        exp = port.cluster(port.encode(img, 4096, *cb), img, 4096, k, its, False, per_round=True)
        return img, cfg, exp

    a, b = case(60, 70, 3, 3, 5, 1), case(33, 90, 1, 2, 4, 2)
    for img, cfg, exp in (a, a, a, b, b, a, b, a):
        res = ctx.run_pipeline(img, cfg)
        assert (res.mask.reshape(-1) == exp["labels"]).all() and res.iterations_run == exp["rounds"]
    img, cfg, exp = a
    rounds = []
    res = ctx.run_pipeline(img, cfg, on_iteration=lambda r, lab: rounds.append(lab.reshape(-1).copy()))
    assert len(rounds) == exp["rounds"]
    for r in range(exp["rounds"]):
        assert (rounds[r] == exp["labels_rounds"][r]).all(), r
    labels = np.zeros(img.shape[0] * img.shape[1], np.uint32)  # pageable: staged, not zero-copy
    rc = ctx.run_pipeline(img, cfg)  # replayed graph (zero-copy into the pinned buffer)
    assert (rc.mask.reshape(-1) == exp["labels"]).all()
    lib = S.lib()
    rounds_c = S._sz()
    import ctypes as C
    h, w, c = img.shape
    ctx.check(lib.seghdc_run_pipeline(ctx.h, img, h, w, c, cfg.dim, float(cfg.alpha), cfg.beta, cfg.gamma,
                                      cfg.clusters, cfg.iterations, cfg.seed, 0, 0, S.ROUND_CB(0), None, labels,
                                      C.byref(rounds_c), None))
    assert (labels == exp["labels"]).all() and rounds_c.value == exp["rounds"]


@pytest.mark.parametrize("dim,k,kernel", [
    (32, 2, "k_round_tc"), (700, 3, "k_round_tc"), (1024, 1, "k_round_tc"),  # one chunk, padded to two
    (3000, 7, "k_round_tc"), (4096, 8, "k_round_tc"),     # K <= 8 on one CTA per tile (N = 64)
    (16384, 5, "k_round_tc"),                              # K <= 8, split over 4 CTAs
    (2000, 9, "k_round"), (40000, 2, "k_round"),           # the IMMA-only shapes: K > 8, very long HVs
])
def test_round_kernel_layouts(ctx, port, dim, k, kernel):
    """Which round kernel serves which shape (tcgen05 everywhere a layout fits; the IMMA kernels
    only for K > 8 and HVs too long for any tcgen05 B image), each bit-exact against the oracle
    for four full rounds."""
    rng = np.random.default_rng(dim + 17 * k)
    h, w, c = 37, 45, 3
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    img[: h // 2] //= 3
    if dim >= 2048:
        grid = port.encode(img, dim, *S.build_codebooks(dim, h, w, c, 1.0, 2, 1, k))
    else:  # too short for the codebooks' flip units at this size: random HVs
        grid = _rand_grid(rng, h * w, dim)
    got = []
    res = ctx.cluster(grid, img, dim, k, 4, False, on_iteration=lambda r, lab: got.append(lab))
    assert ctx.round_kernel == kernel
    exp = port.cluster(grid, img, dim, k, 4, False, per_round=True)
    for r in range(exp["rounds"]):
        assert (got[r] == exp["labels_rounds"][r]).all(), r
    assert (res["centroids"] == exp["centroids"]).all() and (res["counts"] == exp["counts"]).all()
