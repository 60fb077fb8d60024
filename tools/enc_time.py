"""Encode kernel time (CUDA events around encode_async, median of 20) for configs 0, 1, 3, 4."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_12753_b200 as S
only = [int(a) for a in sys.argv[1:]]  # optional config filter, e.g. "1 3" (used under ncu)
for cid, dim, alpha in ((0, 10000, 0.2), (1, 10000, 0.2), (3, 10000, 1.0), (4, 16384, 1.0)):
    if only and cid not in only:
        continue
    img = S.synth_image(cid, 0)
    h, w, c = img.shape
    ctx = S.Context(0)
    st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
    ctx.load_image(img); ctx.load_codebooks(dim, *S.build_codebooks(dim, h, w, c, alpha, 26, 1, 0))
    ts = []
    for i in range(23):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); ctx.encode_async(0, h); e1.record(st); torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    s32 = ((dim + 31) // 32 + 31) // 32 * 32
    print(f"C{cid}: encode {ms * 1e3:.1f} us, {h * w * s32 * 4 / ms / 1e6:.0f} GB/s written")
    ctx.close()
