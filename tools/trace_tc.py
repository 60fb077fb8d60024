"""Diagnostic: per-tile timeline of the tcgen05 round kernel from a -DSEGHDC_TRACE build.
Events (clock64 per CTA): 0 producer issues the tile's first chunk, 1 unpack warp 0 starts
chunk 0, 2 unpack warp 0 done with the last chunk, 3 MMA thread committed the tile, 4 epilogue
sees D, 5 epilogue list ready, 6 fold starts, 7 fold done."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_12753_b200 as S
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
img = S.synth_image(cid, 0)
h, w, c = img.shape
ctx = S.Context(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
ctx.load_image(img)
ctx.load_codebooks(10000, *S.build_codebooks(10000, h, w, c, 0.2, 26, 1, 0))
sleep = len(sys.argv) > 2 and sys.argv[2] == "sleep"
ITERS = int(sys.argv[3]) if len(sys.argv) > 3 else 3
for i in range(3):
    if i == 2:
        ctx.profile_rounds(True)
        if sleep:  # park the GPU so the host enqueues the whole cluster ahead of it
            torch.cuda._sleep(20_000_000)
    ctx.encode_async(0, h); ctx.cluster_async(2, ITERS, False)
torch.cuda.synchronize()
kms, kn = ctx.profile_read()
print(f"round kernel, CUDA events: {kms / kn * 1e3:.1f} us avg over {kn} launches")
buf = np.zeros(148 * 64 * 8, np.uint64)
if not hasattr(S.lib(), "seghdc_debug_trace_tc"): sys.exit(0)
S.lib().seghdc_debug_trace_tc(buf.ctypes.data_as(ctypes.c_void_p))  # (read once to size; counters accumulate across launches)
S.lib().seghdc_debug_trace_tc(buf.ctypes.data_as(ctypes.c_void_p))
t = buf.reshape(148, 64, 8).astype(np.int64)
g = t[:, 63, :].copy(); g = g - g[:, 0].min()
print("events (us): [stamp0] %.2f  [round kernel] %.2f  [stamp1] %.2f" % tuple(t[0, 60, :3] / 1e3))
st = t[:, 61, :].copy()
print(f"stamp kernel before -> first CTA entry: {(t[:, 63, 0].min() - st[:, 0].max()) / 1e3:.2f} us; "
      f"last CTA dealloc -> stamp kernel after: {(st[:, 2].min() - st[:, 1].max()) / 1e3:.2f} us; "
      f"first entry -> last dealloc {(st[:, 1].max() - t[:, 63, 0].min()) / 1e3:.2f} us")
print("kernel-level (us, globaltimer, rel. to earliest CTA entry): median / max over CTAs")
for e, nm in enumerate(["entry", "setup_done", "B_landed", "chunk0_landed", "epi_loop_done", "fold_loop_done", "final_sync", "flush_done"]):
    print(f"  {nm:15s} {np.median(g[:, e]) / 1e3:8.2f} {g[:, e].max() / 1e3:8.2f}")
acc = t[:, 62, :].copy()
print("accumulated cycles per CTA (median):", ", ".join(f"{n}={int(np.median(acc[:, i]))}" for i, n in enumerate(["unp_slotfull", "unp_afree", "mma_afull", "mma_issue", "prod_slotfree", "epi_dfull"])))
t[:, 60:, :] = t[:, 59:60, :]
t = t - t[:, :1, 0:1]
names = ["prod_issue", "unpack_beg", "unpack_end", "mma_commit", "epi_D", "epi_list", "fold_beg", "fold_end"]
print("tile " + " ".join(f"{n:>10s}" for n in names))
for it in list(range(0, 6)) + [10, 11, 15, 16, 17]:
    print(f"{it:4d} " + " ".join(f"{int(np.median(t[:, it, e])):10d}" for e in range(8)))
d = lambda a, b: np.median(t[:, 4:16, b] - t[:, 4:16, a])
print("tile period (unpack_beg)", np.median(np.diff(t[:, 4:16, 1], axis=1)))
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7)]:
    print(f"  {names[a]:>10s} -> {names[b]:<10s} {d(a, b):8.0f}")
