"""CPU: the C-ABI library loads, exports every symbol include/seghdc_cuda.h declares, and its
host-side pieces (validation, codebooks, synthetic inputs) match the reference. No compute
call touches a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2303_12753_b200 as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "seghdc_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(seghdc_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = S.lib()
    names = declared_symbols()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    # and the Python binding covers exactly the declared surface
    assert set(names) == set(S.SIGNATURES)


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(S.RuntimeFailure):
        S.Context(0)


@pytest.mark.parametrize("dim,h,w,c,alpha,beta,gamma,enc", [
    (10000, 256, 256, 3, 0.2, 26, 1, "manhattan"), (10000, 520, 696, 1, 0.2, 26, 1, "manhattan"),
    (10000, 2048, 2048, 3, 1.0, 26, 1, "manhattan"), (16384, 64, 64, 3, 1.0, 26, 1, "manhattan"),
    (1600, 5, 7, 1, 1.0, 1, 3, "manhattan"), (777, 9, 5, 3, 1.0, 2, 1, "rpos"), (800, 9, 5, 3, 1.0, 2, 1, "rcolor"),
])
def test_codebooks_match_reference(ref, dim, h, w, c, alpha, beta, gamma, enc):
    mine = S.build_codebooks(dim, h, w, c, alpha, beta, gamma, 5, enc)
    theirs = ref.build_codebooks(dim, h, w, c, alpha, beta, gamma, 5, S.ENCODERS[enc])
    for a, b in zip(mine, theirs):
        assert (a == b).all()


@pytest.mark.parametrize("args,msg", [
    ((10000, 2048, 2048, 3, 0.2, 26, 1, 2, 10), "dimension too small for image size"),
    ((255, 4, 4, 1, 1.0, 1, 1, 2, 10), "dimension too small for color resolution"),
    ((1000, 4, 4, 2, 1.0, 1, 1, 2, 10), "channels must be 1 or 3"),
    ((1000, 4, 4, 1, 0.0, 1, 1, 2, 10), "alpha must be in"),
    ((1000, 4, 4, 1, 1.0, 0, 1, 2, 10), "beta must be >= 1"),
    ((1000, 4, 4, 1, 1.0, 1, 1, 0, 10), "k must be >= 1"),
    ((1000, 4, 4, 1, 1.0, 1, 1, 17, 10), "exceeds pixel count"),
    ((1000, 4, 4, 1, 1.0, 1, 1, 2, 0), "iterations must be >= 1"),
])
def test_run_config_validation(args, msg):
    # RunConfig::validate (pipeline.cpp:25-30) -> ConfigError, before any device work
    dim, h, w, c, alpha, beta, gamma, k, it = args
    with pytest.raises(S.ConfigError, match=msg):
        S.RunConfig(dim=dim, alpha=alpha, beta=beta, gamma=gamma, clusters=k, iterations=it).validate(h, w, c)


def test_synthetic_images_are_seeded_and_shaped():
    shapes = {0: (256, 256, 3), 1: (520, 696, 1), 2: (256, 256, 3), 3: (2048, 2048, 3)}
    for cid, shape in shapes.items():
        a = S.synth_image(cid, 0)
        assert a.shape == shape
        assert (a == S.synth_image(cid, 0)).all()
    assert (S.synth_image(2, 1) != S.synth_image(2, 2)).any()
    a = S.synth_image(0, 0).astype(float)
    bright = (a.mean(axis=2) > 120).mean()
    assert 0.02 < bright < 0.3  # 20 bright ellipses over a dark background
    with pytest.raises(ValueError):
        S.synth_image(7, 0)
    # the bench's reference arm reads the same bytes without loading the product library
    import workloads
    assert (workloads.synth_image(1, 0) == S.synth_image(1, 0)).all()


def test_row_ranges():
    from paper_2303_12753_b200.sharded import row_ranges
    assert row_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert row_ranges(4096, 8)[-1] == (3584, 4096)
    with pytest.raises(ValueError):
        row_ranges(2, 3)


def test_best_foreground_iou_matches_reference_rules():
    """best_foreground_iou (metrics.cpp:42-101) through the C-ABI, host-only: the reference
    suite's cases plus a brute-force comparison with the per-subset definition."""
    lab = np.array([0, 1, 2, 0, 1, 2], np.uint32)
    assert S.best_foreground_iou(lab, np.array([0, 1, 1, 0, 1, 1]), 3) == (1.0, [1, 2])
    v, sub = S.best_foreground_iou(np.array([0, 1], np.uint32), np.array([1, 1]), 2)
    assert sub == [0] and abs(v - 0.5) < 1e-12  # tie -> smaller label
    with pytest.raises(S.ConfigError):
        S.best_foreground_iou(lab, np.ones(6), 5)
    with pytest.raises(S.ConfigError):
        S.best_foreground_iou(lab, np.ones(6), 2)  # label 2 out of range
    rng = np.random.default_rng(0)
    for t in range(50):
        k = int(rng.integers(1, 5))
        n = int(rng.integers(1, 40))
        l = rng.integers(0, k, n).astype(np.uint32)
        g = rng.integers(0, 2, n)
        best = None
        for s in range(1, 1 << k):
            if k > 1 and s == (1 << k) - 1:
                continue
            p = (s >> l) & 1
            inter, uni = int((p & g).sum()), int((p | g).sum())
            score = 1.0 if uni == 0 else inter / uni
            labs = [c for c in range(k) if s >> c & 1]
            if best is None or score > best[0] or (score == best[0] and (len(labs), labs) < (len(best[1]), best[1])):
                best = (score, labs)
        assert S.best_foreground_iou(l, g, k) == best, (t, k)
