"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) and for the
checked build (-DSEGHDC_CHECKED, SEGHDC_LIB=...; compute-sanitizer is closed on the GPU pool),
each case re-run 5 times (a race shows up as run-to-run differences): every
round-kernel layout (tcgen05 one-CTA K <= 2 and K <= 4, the 4-CTA dimension split for K <= 8,
the IMMA kernels), encode, seeds, fold lists, finish, and the closed-form variant. Each case
is checked against the oracle so a sanitizer run also proves the results did not change."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2303_12753_b200 as S  # noqa: E402

port = oracle.Port()
ctx = S.Context(0)
rng = np.random.default_rng(5)
cases = [  # dim, h, w, c, k, its, expected round kernel
    (10000, 40, 50, 3, 2, 3, "k_round_tc"),   # one CTA per tile, N = 16, fold warps
    (10000, 40, 50, 3, 4, 3, "k_round_tc"),   # N = 32, fold lists
    (16384, 30, 40, 3, 8, 3, "k_round_tc"),   # 4-CTA cluster, dimension split, DSMEM exchange
    (1000, 30, 40, 3, 2, 3, "k_round_fused"),  # D <= 1024: IMMA
    (4000, 20, 30, 1, 12, 3, "k_round"),      # K > 8: IMMA
]
for dim, h, w, c, k, its, kern in cases:
    img = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    img[: h // 2] //= 4
    cb = S.build_codebooks(dim, h, w, c, 1.0, 3, 1, 1)
    grid = ctx.encode_image(img, dim, *cb)
    res = ctx.cluster(None, img, dim, k, its, False)
    for _ in range(5):  # determinism: identical labels and centroids on every re-run
        again = ctx.cluster(None, img, dim, k, its, False)
        assert (again["labels"] == res["labels"]).all() and (again["centroids"] == res["centroids"]).all()
    exp = port.cluster(grid, img, dim, k, its, False)
    assert (grid == port.encode(img, dim, *cb)).all()
    assert (res["labels"] == exp["labels"]).all() and (res["centroids"] == exp["centroids"]).all(), (dim, k)
    print(f"dim={dim} k={k}: {ctx.round_kernel} ok", flush=True)
    cfg = S.RunConfig(dim=dim, alpha=1.0, beta=3, gamma=1, clusters=min(k, 8), iterations=its, seed=1, early_stop=False)
    cl = ctx.run_pipeline_closed(img, cfg)
    ex = port.cluster(port.encode(img, dim, *S.build_codebooks(dim, h, w, c, 1.0, 3, 1, 1)), img, dim, min(k, 8), its, False)
    assert (cl["labels"] == ex["labels"]).all() and (cl["centroids"] == ex["centroids"]).all()
    print(f"closed dim={dim} k={min(k, 8)} ok", flush=True)
L = S.lib()
if hasattr(L, "seghdc_debug_check"):
    import ctypes
    line = ctypes.c_uint(0)
    assert L.seghdc_debug_check(ctypes.byref(line)) == 0
    print("checked build: first violated device-side check at line", line.value, "(0 = none)")
    assert line.value == 0
print("sanitize cases ok")
