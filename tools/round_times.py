"""Per-round kernel times (CUDA events on the context stream) for one config: which rounds are slow?"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_12753_b200 as S
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
spec = {0: (10000, 2, 0.2), 1: (10000, 2, 0.2), 3: (10000, 4, 1.0), 4: (16384, 8, 1.0)}[cid]
img = S.synth_image(cid, 0)
h, w, c = img.shape
ctx = S.Context(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
ctx.load_image(img)
ctx.load_codebooks(spec[0], *S.build_codebooks(spec[0], h, w, c, spec[2], 26, 1, 0))
for _ in range(3):
    ctx.encode_async(0, h); ctx.cluster_async(spec[1], iters, False)
ctx.profile_rounds(True)
for _ in range(5):
    ctx.encode_async(0, h); ctx.cluster_async(spec[1], iters, False)
t = ctx.profile_read_each().reshape(5, -1) * 1e3
print("per-round kernel us (median of 5 steps):", " ".join(f"{x:.1f}" for x in np.median(t, axis=0)))
