"""Diagnostic: per-role wait cycles and per-tile timeline of the 4-CTA dimension-split tcgen05
round kernel (K = 8, D = 16384, the C4 shape on a smaller image) from a -DSEGHDC_TRACE build
selected by SEGHDC_LIB. Same event slots as tools/trace_tc.py."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_12753_b200 as S
side = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4  # 4: D = 16384, K = 8 (split layout); 3: D = 10000, K = 4
dim, k = (16384, 8) if cfg == 4 else (10000, 4)
img = S.synth_image(cfg, 0)[:side, :side].copy()
h, w, c = img.shape
ctx = S.Context(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
ctx.load_image(img)
ctx.load_codebooks(dim, *S.build_codebooks(dim, h, w, c, 1.0, 26, 1, 0))
for i in range(3):
    if i == 2:
        ctx.profile_rounds(True)
    ctx.encode_async(0, h); ctx.cluster_async(k, 4, False)
torch.cuda.synchronize()
kms, kn = ctx.profile_read()
tiles = (h * w + 127) // 128
print(f"{ctx.round_kernel}: {kms / kn * 1e3:.1f} us avg over {kn} launches; {tiles} tiles, "
      f"{h * w * ((dim + 7) // 8) / (kms / kn / 1e3) / 1e9:.0f} GB/s algorithmic")
if not hasattr(S.lib(), "seghdc_debug_trace_tc"): sys.exit(0)
buf = np.zeros(148 * 64 * 8, np.uint64)
S.lib().seghdc_debug_trace_tc(buf.ctypes.data_as(ctypes.c_void_p))
S.lib().seghdc_debug_trace_tc(buf.ctypes.data_as(ctypes.c_void_p))
t = buf.reshape(148, 64, 8).astype(np.int64)
acc = t[:, 62, :].copy()
# with SEGHDC_TRACE_ROUND=r the accumulators cover round r of the 3 runs above
ncta = 33 if cfg == 4 else 148
nchunk = 3 * ((tiles + ncta - 1) // ncta) * (((dim + 31) // 32 + 31) // 32 // (4 if cfg == 4 else 1))
print("cycles per chunk (median over CTAs):", ", ".join(f"{n}={np.median(acc[:, i]) / nchunk:.0f}" for i, n in enumerate(
    ["unp_slotfull", "unp_afree", "mma_afull", "mma_issue", "prod_slotfree", "epi_dfull", "mma_dfree", "epi_xfree"])))
acc2 = t[1:, 60, :].copy()
print("more cycles per TILE (median over CTAs):", ", ".join(f"{n}={np.median(acc2[:, i]) / (nchunk / 4):.0f}" for i, n in enumerate(
    ["epi_ld+combine", "-", "epi_remote_st", "fin_xfull_wait(2 warps)", "-", "-"])))
t[:, 60:, :] = t[:, 59:60, :]
t = t - t[:, :1, 0:1]
names = ["prod_issue", "unpack_beg", "unpack_end", "mma_commit", "epi_D", "epi_list"]
print("tile " + " ".join(f"{n:>10s}" for n in names))
for it in list(range(0, 6)) + [10, 20, 30]:
    print(f"{it:4d} " + " ".join(f"{int(np.median(t[:, it, e])):10d}" for e in range(6)))
print("tile period (unpack_beg)", np.median(np.diff(t[:, 4:40, 1], axis=1)))
d = lambda a, b: np.median(t[:, 4:40, b] - t[:, 4:40, a])
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5)]:
    print(f"  {names[a]:>10s} -> {names[b]:<10s} {d(a, b):8.0f}")
