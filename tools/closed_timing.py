"""Time the closed-form Manhattan variant (seghdc_run_pipeline_closed) end to end on the
BASELINE configs: host wall clock around the synchronous C-ABI call (H2D image, codebook
bases, seeds, all rounds, D2H labels + centroids), early stop off. Prints one JSON line per
config. Not the bench metric: the packed-bit path is (SURVEY.md §7 hard part 4)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2303_12753_b200 as S  # noqa: E402

CFG = {0: (10000, 0.2, 2, 10), 1: (10000, 0.2, 2, 10), 3: (10000, 1.0, 4, 20), 4: (16384, 1.0, 8, 20)}
ctx = S.Context(0)
for cid in [int(a) for a in sys.argv[1:]] or [0, 1, 3, 4]:
    dim, alpha, k, its = CFG[cid]
    img = S.synth_image(cid, 0)
    h, w, c = img.shape
    cfg = S.RunConfig(dim=dim, alpha=alpha, beta=26, gamma=1, clusters=k, iterations=its, seed=0, early_stop=False)
    for _ in range(2):
        ctx.run_pipeline_closed(img, cfg)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        res = ctx.run_pipeline_closed(img, cfg)
        ts.append(time.perf_counter() - t)
    ms = float(np.median(ts)) * 1e3
    print(json.dumps({"variant": "closed-form manhattan", "config": f"C{cid}", "h": h, "w": w, "c": c, "dim": dim,
                      "k": k, "iterations": its, "ms_per_run": ms, "px_iter_per_s": h * w * its / (ms / 1e3),
                      "counts": res["counts"].tolist()}), flush=True)
