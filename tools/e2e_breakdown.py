"""Where the end-to-end seghdc_run_pipeline time goes (C1): host codebooks, device stages, total."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_12753_b200 as S
img = S.synth_image(1, 0)
pin = torch.from_numpy(img).pin_memory().numpy()
ctx = S.Context(0)
cfg = S.RunConfig(dim=10000, alpha=0.2, beta=26, gamma=1, clusters=2, iterations=10, seed=0, early_stop=False)
for _ in range(3):
    ctx.run_pipeline(pin, cfg)
rows, walls = [], []
for _ in range(20):
    t0 = time.perf_counter()
    r = ctx.run_pipeline(pin, cfg)
    walls.append((time.perf_counter() - t0) * 1e3)
    rows.append([r.timings[k] for k in ("encode_position", "encode_color", "produce_pixels", "cluster", "total")])
m = np.median(np.array(rows), axis=0)
print("median ms: pos %.3f col %.3f encode(dev) %.3f cluster(dev) %.3f total(C) %.3f wall(py) %.3f" % (*m, np.median(walls)))
