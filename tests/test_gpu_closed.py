"""GPU parity of the closed-form Manhattan variant (seghdc_run_pipeline_closed, SURVEY.md §7
hard part 4 / §8f rank 1) against the oracle and the reference's goldens.

The variant never materialises the pixel HVs; its dots and centroid sums are exact integers,
so labels, centroids, member counts and rounds must equal the reference's bit for bit."""
import hashlib

import numpy as np
import pytest

import paper_2303_12753_b200 as S

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CASES = [  # dim, h, w, c, alpha, beta, gamma, k, its, seed, early_stop
    (10000, 30, 41, 1, 1.0, 26, 1, 2, 6, 0, False),
    (10000, 64, 80, 3, 1.0, 26, 1, 2, 5, 3, True),
    (2003, 17, 19, 3, 1.0, 3, 2, 3, 4, 11, False),
    (4096, 12, 9, 1, 0.5, 1, 4, 2, 7, 5, True),
    (16384, 21, 23, 3, 1.0, 5, 1, 4, 3, 1, False),
    (16384, 40, 37, 3, 1.0, 4, 1, 8, 6, 2, False),
    (1500, 25, 30, 3, 1.0, 2, 1, 5, 8, 7, True),
    (777, 9, 13, 1, 1.0, 1, 1, 1, 3, 4, True),  # k = 1: stops at round 2
    (10000, 50, 50, 3, 1.0, 26, 1, 12, 4, 9, False),  # k > 5: several cluster groups in accumulate
]


@pytest.mark.parametrize("case", CASES)
def test_closed_matches_oracle(ctx, port, case):
    dim, h, w, c, alpha, beta, gamma, k, its, seed, es = case
    rng = np.random.default_rng(dim + h * w + seed)
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    img[: h // 2] //= 4  # a dark half: two clear clusters
    cfg = S.RunConfig(dim=dim, alpha=alpha, beta=beta, gamma=gamma, clusters=k, iterations=its, seed=seed,
                      encoder="manhattan", early_stop=es)
    res = ctx.run_pipeline_closed(img, cfg)
    cb = S.build_codebooks(dim, h, w, c, alpha, beta, gamma, seed)
    exp = port.cluster(port.encode(img, dim, *cb), img, dim, k, its, es)
    assert ctx.round_wraps() == port.last_wraps()
    assert res["rounds"] == exp["rounds"]
    assert (res["labels"] == exp["labels"]).all()
    assert (res["centroids"] == exp["centroids"]).all()
    assert res["counts"].tolist() == exp["counts"].tolist()


def test_closed_uniform_image_and_empty_clusters(ctx, port):
    """A uniform image: seeds from the corners (clusterer.cpp:112-128), every pixel ties, the
    other clusters empty and kept (clusterer.cpp:183-185)."""
    img = np.full((16, 20, 3), 77, np.uint8)
    cfg = S.RunConfig(dim=3000, alpha=1.0, beta=4, gamma=1, clusters=3, iterations=4, seed=6, early_stop=False)
    res = ctx.run_pipeline_closed(img, cfg)
    cb = S.build_codebooks(3000, 16, 20, 3, 1.0, 4, 1, 6)
    exp = port.cluster(port.encode(img, 3000, *cb), img, 3000, 3, 4, False)
    assert (res["labels"] == exp["labels"]).all() and (res["centroids"] == exp["centroids"]).all()
    assert res["counts"].tolist() == exp["counts"].tolist()


@pytest.mark.parametrize("name", ["C0", "C1"])
def test_closed_config_golden(ctx, golden_configs, name):
    """C0/C1 goldens were made by the reference library itself (tests/golden/make_golden.py)."""
    g, spec = golden_configs[name], golden_configs["_meta"]["configs"][name]
    img = S.synth_image(spec["cid"], 0)
    cfg = S.RunConfig(dim=spec["dim"], alpha=spec["alpha"], beta=26, gamma=1, clusters=spec["k"],
                      iterations=spec["iterations"], seed=0, early_stop=False)
    res = ctx.run_pipeline_closed(img, cfg)
    assert sha(res["labels"]) == g["labels_sha256"]
    assert sha(res["centroids"]) == g["centroids_sha256"]
    assert res["counts"].tolist() == g["counts"] and res["rounds"] == g["rounds"]
    cfg.early_stop = True
    es = ctx.run_pipeline_closed(img, cfg)
    assert es["rounds"] == g["early_stop_rounds"] and sha(es["labels"]) == g["early_stop_labels_sha256"]


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_closed_config_large_golden(ctx, golden_configs, name):
    """C3 / C4 at their full 20 rounds against the reference (make_golden_full.py), including
    the per-round count of 128-bit comparator wraps."""
    g, spec = golden_configs[name], golden_configs["_meta"]["configs"][name]
    img = S.synth_image(spec["cid"], 0)
    cfg = S.RunConfig(dim=spec["dim"], alpha=spec["alpha"], beta=26, gamma=1, clusters=spec["k"],
                      iterations=g["iterations"], seed=0, early_stop=False)
    res = ctx.run_pipeline_closed(img, cfg)
    assert sha(res["labels"]) == g["labels_sha256"]
    assert sha(res["centroids"]) == g["centroids_sha256"]
    assert res["counts"].tolist() == g["counts"]
    if "round_wraps" in g:
        assert ctx.round_wraps() == g["round_wraps"]


def test_closed_validation(ctx):
    img = np.zeros((8, 8, 3), np.uint8)
    with pytest.raises(S.ConfigError):
        ctx.run_pipeline_closed(img, S.RunConfig(dim=1000, alpha=1.0, clusters=33, iterations=2))
    with pytest.raises(S.ConfigError):
        ctx.run_pipeline_closed(img, S.RunConfig(dim=1000, alpha=1.0, clusters=2, iterations=2, encoder="rpos"))
    with pytest.raises(S.ConfigError):  # x_row = 0 (position_encoder.cpp:29-38)
        ctx.run_pipeline_closed(np.zeros((4096, 1, 1), np.uint8), S.RunConfig(dim=1000, alpha=0.2, clusters=2))


@pytest.mark.parametrize("case", [CASES[1], CASES[5], CASES[8]])
def test_closed_position_tables_match(ctx, port, case, monkeypatch):
    """The full-position tables (SEGHDC_CLOSED_POSITIONS, used when the compressed endpoint
    tables do not fit shared memory) give the same results."""
    monkeypatch.setenv("SEGHDC_CLOSED_POSITIONS", "1")
    test_closed_matches_oracle(ctx, port, case)


@pytest.mark.parametrize("case", [CASES[0], CASES[5], (30000, 20, 23, 3, 1.0, 3, 1, 3, 4, 12, False)])
def test_closed_global_finish_matches(ctx, port, case, monkeypatch):
    """The global-memory finish (k_closed_finish: forced by SEGHDC_CLOSED_FIN_GLOBAL, and taken
    whenever the shared-memory rows exceed 200 KB, i.e. dim above ~25k) gives the same results."""
    if case[0] < 25000:
        monkeypatch.setenv("SEGHDC_CLOSED_FIN_GLOBAL", "1")
    test_closed_matches_oracle(ctx, port, case)


@pytest.mark.parametrize("case", [CASES[0], CASES[4], CASES[8]])
def test_closed_one_cta_shared_memory_finish_matches(ctx, port, case, monkeypatch):
    """The one-CTA shared-memory finish (SEGHDC_CLOSED_FIN=smem; the default is the cluster
    finish, k_closed_finish_cl) gives the same results."""
    monkeypatch.setenv("SEGHDC_CLOSED_FIN", "smem")
    test_closed_matches_oracle(ctx, port, case)
