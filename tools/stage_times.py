"""Diagnostic: device time of each stage of one bench step (encode, cluster loop, single
round kernels) measured with CUDA events on the context stream, steady state, C1."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_12753_b200 as S
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
spec = {0: (10000, 2, 10, 0.2), 1: (10000, 2, 10, 0.2), 3: (10000, 4, 20, 1.0), 4: (16384, 8, 20, 1.0)}[cid]
dim, k, iters, alpha = spec
img = S.synth_image(cid, 0)
h, w, c = img.shape
ctx = S.Context(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
ctx.load_image(img)
ctx.load_codebooks(dim, *S.build_codebooks(dim, h, w, c, alpha, 26, 1, 0))
def timed(fn, n=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st)
    for _ in range(n): fn()
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
t_enc = timed(lambda: ctx.encode_async(0, h))
t_all = timed(lambda: (ctx.encode_async(0, h), ctx.cluster_async(k, iters, False)))
t_c1 = timed(lambda: (ctx.encode_async(0, h), ctx.cluster_async(k, 1, False)))
t_c2 = timed(lambda: (ctx.encode_async(0, h), ctx.cluster_async(k, 2, False)))
print(json.dumps({"config": cid, "encode_ms": t_enc, "step_ms": t_all, "cluster_ms": t_all - t_enc,
                  "per_round_ms(2it-1it)": t_c2 - t_c1, "one_round_cluster_ms": t_c1 - t_enc,
                  "px": h * w, "gbs_round": h * w * ((dim + 7) // 8) / ((t_c2 - t_c1) * 1e-3) / 1e9}))
