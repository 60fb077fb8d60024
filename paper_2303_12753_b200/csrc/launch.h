// Internal launcher interface between the C-ABI layer (seghdc_capi.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace seghdc_dev {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) costs host microseconds per call; the
// launchers raise each kernel's limit once per (function, device) instead of per launch.
cudaError_t ensure_dynamic_smem(const void* func, size_t bytes);

// Launch with programmatic dependent launch allowed: the kernel may start before the previous
// kernel in the stream completes and must execute griddepcontrol.wait before reading anything
// that kernel wrote.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

struct RoundState;

struct EncodeArgs {
    const uint8_t* img;  // full image, h*w*c
    uint32_t w, c;
    uint64_t pix_begin, pix_end;  // global pixel range encoded into grid[0..)
    const uint32_t *row, *col, *wid;
    const uint8_t* sup;  // [wref] channel set per HV word (bit ch: wid[ch][*] may be non-zero there)
    uint32_t nl_max;     // most channels any word has
    uint32_t wref;  // u32 words per table entry (2 * ceil(dim/64))
    uint32_t S32, W32;
    uint32_t* grid;
    uint32_t* colsum;  // zeroed by the caller; receives the column sums of the encoded rows
    uint32_t sms;
};
void launch_encode(const EncodeArgs& a, cudaStream_t s);

struct SeedArgs {
    const uint8_t* img;
    uint64_t n;
    uint32_t h, w, c, K;
    uint16_t* min_dist;
    uint64_t* seeds;
    unsigned long long* slots;
    RoundState* hdr;
    bool slots_cleared;  // the caller already set the slots to all ones (launch_init_clear)
    bool defer_post;     // K <= 2: k_init_seeds decides the seeds from the slots (InitSeedArgs::post_slots)
};
void launch_init_clear(void* state, size_t state_bytes, void* run1, size_t run1_bytes, unsigned long long* slots,
                       uint32_t nslots, uint32_t* list_counts, uint32_t nlists, cudaStream_t s);
void launch_select_seeds(const SeedArgs& a, cudaStream_t s);

struct InitSeedArgs {
    const uint32_t* grid;
    uint32_t S32;
    uint64_t pix_begin, n_local;
    uint64_t* seeds;
    uint32_t K, W32, Dp;
    int32_t* xchg;
    const unsigned long long* post_slots;  // nullable (K <= 2): derive the seeds here (see SeedArgs::defer_post)
    uint32_t h, w;
    RoundState* hdr;
    const int32_t* colsum_src;  // nullable: local column sums, copied to colsum_dst (the exchange tail)
    int32_t* colsum_dst;
};
void launch_init_seeds(const InitSeedArgs& a, cudaStream_t s);

struct AccumulateArgs {
    const uint32_t* grid;
    uint32_t S32, W32;
    uint64_t n;
    const uint32_t* labels;  // nullptr: every pixel counts for "cluster 0" (column sums)
    uint32_t K;
    int skip_mode;  // -1 none, -2 largest current cluster, >= 0 explicit
    void* state;    // may be nullptr when skip_mode != -2
    uint32_t parity;
    uint32_t* dst;         // sums land in dst[c * Dp + i] (atomically added)
    uint32_t Dp;
    uint32_t* counts_dst;  // nullable: member counts atomically added to counts_dst[c]
    uint32_t sms;
};
void launch_accumulate(const AccumulateArgs& a, cudaStream_t s);

struct FinishArgs {
    int mode;  // 0 round, 1 init, 2 given centroids, 3 standalone update
    uint32_t K, P, D, W32, W32P, Dp;
    const int32_t* xchg;
    const int32_t* colsum;
    uint32_t* Z;
    uint32_t* run;  // incremental K > 2: running member sums [2 parities][K][Dp] (row 0 unused); else null
    uint8_t* bfrag;
    void* state;
    uint32_t round;
    int early_stop;
};
void launch_prep_finish(void* state, uint32_t K, uint32_t np, cudaStream_t s);
void launch_finish(const FinishArgs& a, cudaStream_t s);

struct RoundPlan {
    uint32_t nwarp_words = 0;  // 32-word blocks per HV
    uint32_t nwarps = 0;       // (MMA) warps per CTA
    uint32_t mt = 0;           // m-tiles of 16 pixels per tile
    uint32_t ntg = 0;          // n-tiles per group
    uint32_t nt = 0;           // n-tiles in total: ceil(K * planes / 8)
    uint32_t wpw = 32;         // HV words per warp (split-K)
    uint32_t w32p = 0;         // words covered by the B-fragment layout (>= W32)
    bool fused = false;        // one n-tile: warp-specialised kernel (+ fused accumulation when K == 2)
    uint32_t nrw = 0;          // fused: dedicated re-bundling warps (0: the MMA warps re-bundle)
    bool tc = false;           // tcgen05 kernel (seghdc_tc.cu) instead of the IMMA kernels
};
struct RoundArgs {
    const uint32_t* grid;
    uint64_t n;
    uint32_t S32, SS, W32, W32P, nwarp_words, K, P, NT;
    const uint64_t* bfrag;
    uint32_t* labels;
    void* state;
    uint32_t round;
    int do_update;
    int32_t* xchg;  // [K*Dp sums | K counts | changed], zeroed before the round
    uint32_t Dp;
    uint32_t ctas;
    // tcgen05 kernel only
    const void* tmap;     // CUtensorMap of the grid (tc_make_grid_map)
    const uint8_t* bimg;  // centroid B image (launch_build_bimg)
    uint32_t nks;         // k-steps of 64 HV dims (tc_ksteps)
    uint32_t* flist;        // non-null: append changed pixels to per-cluster lists (k_fold_list folds them)
    uint32_t* flist_count;  // entries appended per tracked cluster 1..K-1 (zeroed before the round)
    uint32_t serpentine;     // odd rounds walk the tiles backwards
    uint32_t pf;             // L2 prefetch distance of the producer, in chunks (0: none)
    bool wraps;              // a 128-bit comparator wrap is possible: use the wrap-counting kernels
    const unsigned long long* labels_host_slot;  // tcgen05, last round: device slot holding a mapped host
                                                 // label pointer (0: none) that also receives the labels
};
size_t round_smem_bytes(uint32_t MT, uint32_t NTG, uint32_t SS, uint32_t nwarps, uint32_t K, uint32_t NT);
bool plan_round(uint32_t K, uint32_t P, uint32_t W32, uint32_t SS, RoundPlan& p, size_t smem_limit);
cudaError_t launch_round(const RoundArgs& a, const RoundPlan& p, cudaStream_t s);

// tcgen05 round kernel (seghdc_tc.cu)
bool tc_supported(uint32_t K, uint32_t W32);
uint32_t tc_ksteps(uint32_t W32);
size_t tc_smem_bytes(uint32_t K, uint32_t W32);
size_t tc_bimg_bytes(uint32_t K, uint32_t W32);
uint32_t tc_tile_pixels();
bool tc_make_grid_map(void* map, const uint32_t* grid, uint64_t rows, uint32_t S32);
struct ExpandArgs {  // closed-form Manhattan codebooks (seghdc_host::manhattan_bases)
    uint32_t dim, h, w, c, beta, x_row, x_col, wref;
    uint32_t off[3], unit[3];
};
void launch_expand_codebooks(const uint32_t* bases, const ExpandArgs& a, uint32_t* row, uint32_t* col, uint32_t* wid,
                             uint8_t* sup, cudaStream_t s);
// Channels whose dimension segment [off[ch], off[ch + 1] or dim) overlaps HV word q (a superset
// of the support of the widened Manhattan tables, pixel_pipeline.cpp:66-88), as a bit set.
#ifdef __CUDACC__
__host__ __device__
#endif
inline uint8_t manhattan_word_channels(uint32_t dim, uint32_t c, const uint32_t* off, uint32_t q) {
    uint8_t m = 0;
    for (uint32_t ch = 0; ch < c && ch < 3; ++ch) {
        const uint32_t lo = off[ch], hi = (ch + 1 < c && ch + 1 < 3) ? off[ch + 1] : dim;
        if (lo < hi && lo < 32 * q + 32 && hi > 32 * q) m |= uint8_t(1u << ch);
    }
    return m;
}
uint64_t tc_max_value(uint32_t K, uint32_t W32);
uint32_t tc_ncol(uint32_t K, uint32_t W32);  // 16 / 32 (one CTA), 64 (4-CTA dimension split), 0
// incremental K == 2 schedule of the tcgen05 kernel: xchg row 1 holds the round's delta of
// cluster 1's member sums, run1[parity][Dp] the running sums (read p, write p ^ 1)
// lists: nlists tracked clusters, list l at list + l * max_rows (count[l] entries), folded as
// signed deltas into dst + l * dst_stride
void launch_fold_list(const uint32_t* list, const uint32_t* count, uint64_t max_rows, uint32_t nlists,
                      const uint32_t* grid, uint32_t S32, uint32_t W32, int32_t* dst, uint32_t dst_stride,
                      uint32_t sms, cudaStream_t s);
void launch_finish_tc(uint32_t D, uint32_t W32, uint32_t Dp, int32_t* xchg, const int32_t* colsum, uint32_t* Z,
                      uint32_t* run1, uint8_t* bimg, void* state, uint32_t round, int early_stop, uint32_t* ticket,
                      cudaStream_t s);  // centroid entries above this need the IMMA kernels
void launch_build_bimg(const uint32_t* Z, uint32_t K, uint32_t D, uint32_t W32, uint8_t* bimg, const void* state,
                       cudaStream_t s,
                       uint32_t* clear = nullptr, uint32_t clear_n = 0);
cudaError_t launch_round_tc(const RoundArgs& a, cudaStream_t s);
#ifdef SEGHDC_CHECKED
unsigned int check_line_tc();       // first violated SG_CHECK line per translation unit (0: none)
unsigned int check_line_kernels();
unsigned int check_line_closed();
#endif

}  // namespace seghdc_dev
