"""CPU: pin the oracle (C restatement) to the reference — its own known answers, its own
brute-force test instances, and the compiled reference library itself."""
import numpy as np
import pytest

from conftest import instance_arrays


def test_mt19937_64_known_answer(port):
    # [rand.predef]: the 10000th consecutive output of a default-constructed mt19937_64
    assert int(port.mt64(5489, 10000)[-1]) == 9981545732273789042


def _ham(a, b):
    return sum(bin(int(x) ^ int(y)).count("1") for x, y in zip(a, b))


@pytest.mark.parametrize("dim,h,w,alpha,beta,x_row,x_col", [
    # reference tests/test_position_encoder.cpp:25-28 (x = block-to-block Hamming distance)
    (10000, 100, 100, 0.2, 1, 10, 10), (10000, 64, 32, 0.2, 4, 15, 31),
])
def test_flip_unit_known_answers(port, dim, h, w, alpha, beta, x_row, x_col):
    row, col, _ = port.build_codebooks(dim, h, w, 1, alpha, beta, 1, 1)
    assert _ham(row[0], row[beta]) == x_row and _ham(row[0], row[2 * beta]) == 2 * x_row
    assert _ham(col[0], col[beta]) == x_col
    assert _ham(row[0], row[beta - 1]) == 0  # rows inside a block share one HV


def test_flip_unit_zero_rejected(port):
    import oracle
    with pytest.raises(oracle.OracleError, match="dimension too small for image size"):
        port.build_codebooks(10000, 2048, 2048, 3, 0.2, 26, 1, 0)  # C3 needs alpha >= 0.4096


def test_color_known_answers(port):
    # reference tests/test_color_encoder.cpp:47-48: table distances 510 and 6 at d=512
    _, _, wid = port.build_codebooks(512, 2, 2, 1, 1.0, 1, 1, 11)
    ham = lambda a, b: sum(bin(int(x) ^ int(y)).count("1") for x, y in zip(a, b))
    assert ham(wid[0, 0], wid[0, 255]) == 510
    assert ham(wid[0, 10], wid[0, 13]) == 6


def test_update_known_answer(port):
    # reference tests/test_clusterer.cpp:124-149: {1100, 1010} -> (2,1,1,0); empty keeps previous
    grid = np.array([[0b0011], [0b0101]], np.uint64)  # bit i is LSB-first: "1100" -> 0b0011
    prev = np.array([[0, 0, 0, 1], [1, 1, 1, 1]], np.uint32)
    z, counts = port.update(grid, 4, np.array([0, 0], np.uint32), prev)
    assert z[0].tolist() == [2, 1, 1, 0] and counts.tolist() == [2, 0]
    assert z[1].tolist() == [1, 1, 1, 1]


def test_oracle_matches_bruteforce_instances(port, golden_instances):
    """The reference suites' own brute-force oracle (reference_clusterer.hpp) per round."""
    assert len(golden_instances) == 60
    for inst in golden_instances:
        img, grid = instance_arrays(inst)
        res = port.cluster(grid, img, inst["dim"], inst["k"], inst["iterations"], False, per_round=True)
        assert res["labels_rounds"].tolist() == inst["expected_rounds"], (inst["suite"], inst["instance"])
        assert port.select_seeds(img, inst["k"]).tolist() == inst["seeds"]


def _random_case(rng, h, w, c, dim):
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    return img


@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_compiled_reference(port, ref, seed):
    rng = np.random.default_rng(100 + seed)
    h, w = int(rng.integers(3, 24)), int(rng.integers(3, 24))
    c = int(rng.choice([1, 3]))
    dim = int(rng.integers(800, 3000))
    enc = int(rng.integers(0, 3))
    img = _random_case(rng, h, w, c, dim)
    beta = 2
    a = port.build_codebooks(dim, h, w, c, 1.0, beta, 1, seed, enc)
    b = ref.build_codebooks(dim, h, w, c, 1.0, beta, 1, seed, enc)
    for x, y in zip(a, b):
        assert (x == y).all()
    grid = port.encode(img, dim, *a)
    assert (grid == ref.encode(img, dim, 1.0, beta, 1, seed, enc)).all()
    for k in (1, 2, 3, 5):
        k = min(k, h * w)
        for es in (False, True):
            r1 = port.cluster(grid, img, dim, k, 6, es, per_round=True)
            r2 = ref.cluster_replay(grid, img, dim, k, 6, es, per_round=True)
            r3 = ref.cluster(grid, img, dim, k, 6, es, per_round=True)
            assert r1["rounds"] == r2["rounds"] == r3["rounds"]
            assert (r1["labels_rounds"] == r2["labels_rounds"]).all()
            assert (r2["labels_rounds"] == r3["labels_rounds"]).all()
            assert (r1["centroids"] == r2["centroids"]).all()
            assert (r1["counts"] == r2["counts"]).all()


def test_seeds_greedy_and_uniform(port, ref):
    # reference tests/test_clusterer.cpp:32-80
    img = np.zeros((1, 4, 1), np.uint8)
    img[0, :, 0] = [0, 100, 255, 120]
    assert port.select_seeds(img, 3).tolist() == [0, 2, 3]
    uni = np.full((3, 4, 3), 128, np.uint8)
    assert port.select_seeds(uni, 5).tolist() == [0, 3, 8, 11, 1]
    rng = np.random.default_rng(5)
    for _ in range(5):
        im = rng.integers(0, 4, (7, 9, 3), dtype=np.uint8)
        for k in (1, 2, 4, 9):
            assert (port.select_seeds(im, k) == ref.select_seeds(im, k)).all()


def test_golden_configs_pinned_to_reference(golden_configs):
    """configs.json C0/C1/C2[0:4] were produced by the reference library itself."""
    for name in ("C0", "C1"):
        assert golden_configs[name]["source"].startswith("reference")
    imgs = golden_configs["C2"]["images"]
    assert all(r["source"].startswith("reference") for r in imgs[:4])


@pytest.mark.parametrize("seed", range(4))
def test_streaming_cluster_equals_stored_grid(port, seed):
    """so_cluster_stream (used for the C4 golden, whose grid does not fit host memory) gives the
    same per-round labels, centroids, counts and rounds as so_cluster on the stored grid."""
    rng = np.random.default_rng(50 + seed)
    h, w, c = int(rng.integers(4, 40)), int(rng.integers(4, 40)), int(rng.choice([1, 3]))
    dim, k, its = int(rng.choice([800, 1024, 3000])) * c, int(rng.integers(1, 9)), int(rng.integers(1, 6))
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    cb = port.build_codebooks(dim, h, w, c, 1.0, int(rng.integers(1, 4)), 1, seed)
    exp = port.cluster(port.encode(img, dim, *cb), img, dim, k, its, bool(seed % 2), per_round=True)
    got = port.cluster_stream(img, dim, *cb, k, its, bool(seed % 2), per_round=True)
    assert got["rounds"] == exp["rounds"]
    assert (got["labels_rounds"] == exp["labels_rounds"]).all()
    assert (got["centroids"] == exp["centroids"]).all() and (got["counts"] == exp["counts"]).all()


def test_wrap_counter_matches_bigint(port):
    """so_last_wraps counts strictly_closer comparisons whose unsigned __int128 products exceed
    2^128 (clusterer.cpp:41-50; norm_squared is u64 and wraps too, hypervector.cpp:123-127).
    Checked against Python big integers, labels included."""
    rng = np.random.default_rng(1)
    n, dim, k = 200, 200, 3
    grid = rng.integers(0, 2**63, (n, (dim + 63) // 64), dtype=np.uint64)
    grid[:, -1] &= np.uint64((1 << (dim % 64)) - 1)
    z = rng.integers(0, 2**32, (k, dim), dtype=np.uint64).astype(np.uint32)
    z[0] //= 1 << 20
    lab = port.assign(grid, dim, z)
    bits = np.unpackbits(grid.view(np.uint8), axis=1, bitorder="little")[:, :dim].astype(object)
    dots = bits.dot(z.astype(object).T)
    n2 = [sum(int(v) * int(v) for v in z[c]) % (1 << 64) for c in range(k)]
    M, wraps, exp = 1 << 128, 0, []
    for p in range(n):
        best = 0
        for c in range(1, k):
            dc, db = int(dots[p, c]), int(dots[p, best])
            if n2[c] and n2[best]:
                lhs, rhs = dc * dc * n2[best], db * db * n2[c]
                wraps += lhs >= M or rhs >= M
                if lhs % M > rhs % M:
                    best = c
            elif n2[c] and not n2[best] and dc > 0:
                best = c
        exp.append(best)
    assert port.last_wraps() == [wraps] and wraps > 0
    assert lab.tolist() == exp


def test_reference_encoded_loop_equals_replay(ref):
    """ref_pare_* (row shards encoded by the reference's own encode_image, used for the
    full-length C3/C4 goldens) equals the single-grid replay of cluster()."""
    import workloads
    img = workloads.synth_image(0, 0)[:48, :60].copy()
    for k, it in ((2, 4), (4, 3)):
        grid = ref.encode(img, 2000, 0.5)
        a = ref.cluster_replay(grid, img, 2000, k, it, False, per_round=True)
        rounds = []
        b = ref.cluster_encoded(img, 2000, k, it, alpha=0.5, nthreads=3, on_round=lambda r, l: rounds.append(l.copy()))
        assert (a["labels_rounds"] == np.array(rounds)).all()
        assert (a["centroids"] == b["centroids"]).all() and (a["counts"] == b["counts"]).all()
