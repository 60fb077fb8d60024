"""Where the end-to-end seghdc_run_pipeline time goes (C1 by default): host codebook bases, device
stages (CUDA events inside the call), the C++ total, the Python wall clock, and the device-only
step of the same work (encode + cluster on resident inputs) for comparison."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_12753_b200 as S
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
img = S.synth_image(cid, 0)
spec = {0: (10000, 2, 10, 0.2), 1: (10000, 2, 10, 0.2), 3: (10000, 4, 20, 1.0)}[cid]
dim, k, its, alpha = spec
h, w, c = img.shape
ctx = S.Context(0)
cfg = S.RunConfig(dim=dim, alpha=alpha, beta=26, gamma=1, clusters=k, iterations=its, seed=0, early_stop=False)
pin = torch.from_numpy(img).pin_memory().numpy()
for name, src in (("pageable", img), ("pinned", pin)):
    for _ in range(3):
        ctx.run_pipeline(src, cfg)
    rows, walls = [], []
    for _ in range(30):
        t0 = time.perf_counter()
        r = ctx.run_pipeline(src, cfg)
        walls.append((time.perf_counter() - t0) * 1e3)
        rows.append([r.timings[q] for q in ("encode_position", "encode_color", "produce_pixels", "cluster", "total")])
    m = np.median(np.array(rows), axis=0)
    print(f"{name:9s} median ms: bases {m[0]:.3f}  encode(dev) {m[2]:.3f}  cluster(dev) {m[3]:.3f}  "
          f"total(C++) {m[4]:.3f}  wall(py) {np.median(walls):.3f}  -> outside device stages {m[4] - m[2] - m[3]:.3f}")
# device-only step on resident inputs (what bench's `value` times)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
ctx.load_image(img); ctx.load_codebooks(dim, *S.build_codebooks(dim, h, w, c, alpha, 26, 1, 0))
for _ in range(3):
    ctx.encode_async(0, h); ctx.cluster_async(k, its, False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(30):
    ctx.encode_async(0, h); ctx.cluster_async(k, its, False)
e1.record(st); torch.cuda.synchronize()
print(f"device-only step: {e0.elapsed_time(e1) / 30:.3f} ms")
