"""Diagnostic: per-tile timeline of the fused round kernel from a -DSEGHDC_TRACE build.

  SEGHDC_NVCC_EXTRA=-DSEGHDC_TRACE python paper_2303_12753_b200/build.py --force
  python tools/trace_round.py [config]
Events (clock64 per CTA): 0 TMA issue, 1 tile landed (MMA warp 0), 2 k-loop end (warp 0),
3 epilogue start, 4 epilogue end, 5 buffer freed (seen by the role warp), 6 fold end,
7 k-loop end (last MMA warp). Prints medians over CTAs of the steady-state tiles.
"""
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
for _ in range(3):
    ctx.encode_async(0, h); ctx.cluster_async(2, 3, False)
torch.cuda.synchronize()
NE = 48
buf = np.zeros(148 * 64 * NE, np.uint64)
S.lib().seghdc_debug_trace(buf.ctypes.data_as(ctypes.c_void_p))
t = buf.reshape(148, 64, NE).astype(np.int64)
t = t - t[:, :1, 0:1]  # relative to the CTA's first TMA issue
names = ["issue", "landed", "kloop_end0", "epi_start", "epi_end", "buf_freed", "fold_end", "kloop_endL"]
print("per-tile medians over CTAs (cycles, relative to the CTA's first issue):")
print("tile " + " ".join(f"{n:>10s}" for n in names))
for it in list(range(0, 8)) + [20, 21, 40, 41, 60]:
    print(f"{it:4d} " + " ".join(f"{int(np.median(t[:, it, e])):10d}" for e in range(8)))
d = lambda a, b, it0=8, it1=60: np.median(t[:, it0:it1, b] - t[:, it0:it1, a])
print("steady state (tiles 8..59) median deltas:")
print("  tile period (landed->landed)      ", np.median(np.diff(t[:, 8:60, 1], axis=1)))
print("  issue -> landed (TMA latency)      ", d(0, 1))
print("  landed -> kloop_end (warp 0)       ", d(1, 2))
print("  landed -> kloop_end (last warp)    ", d(1, 7))
print("  kloop_endL -> epi_start            ", d(7, 3))
print("  epi_start -> epi_end               ", d(3, 4))
print("  epi_end -> fold_end                ", d(4, 6))
print("  fold_end -> buf_freed              ", d(6, 5))
nmw = int(os.environ.get("SEGHDC_FUSED", "12,4").split(",")[0])
print("per MMA warp (SMSP = w % 4): median k-loop start rel. to warp 0 start, k-loop duration")
for wq in range(nmw):
    st_, en_ = t[:, 8:60, 8 + 2 * wq], t[:, 8:60, 9 + 2 * wq]
    print(f"  warp {wq:2d} (SMSP {wq % 4}): start {np.median(st_ - t[:, 8:60, 8]):8.0f}  dur {np.median(en_ - st_):8.0f}")
