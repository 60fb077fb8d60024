// C-ABI of the SegHDC B200 hot path (include/seghdc_cuda.h): device context, resident buffers,
// the round schedule and the reference-API entry points. No exception crosses the boundary.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the symbols are resolved at run time (nccl_api below)

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "../../include/seghdc_cuda.h"
#include "closed.h"
#include "host_internal.h"
#include "kernels.cuh"
#include "launch.h"

using seghdc_host::Error;
using namespace seghdc_dev;

namespace seghdc_dev {
cudaError_t ensure_dynamic_smem(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = done[{func, dev}];
    if (cur >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e == cudaSuccess) cur = bytes;
    return e;
}
}  // namespace seghdc_dev

namespace {

thread_local std::string g_thread_err;

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(SEGHDC_ERUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}

// bumped whenever any device buffer is (re)allocated: a captured CUDA graph bakes in device
// pointers, so a graph recorded under an older epoch is re-captured (seghdc_run_pipeline)
std::atomic<uint64_t> g_realloc_epoch{0};

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    // grow-only; contents are not preserved when it grows
    void ensure(size_t count, bool zero = false) {
        if (count > n) {
            if (p) cudaFree(p);
            p = nullptr;
            n = 0;
            ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
            n = count;
            g_realloc_epoch.fetch_add(1);
            if (zero) ck(cudaMemset(p, 0, count * sizeof(T)), "cudaMemset");
        }
    }
    size_t bytes() const { return n * sizeof(T); }
};

// NCCL, resolved with dlopen("libnccl.so.2") on first use: the library has no link-time NCCL
// dependency, and a process that already loaded one (torch's bundled NCCL) shares that copy.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string err;
};

const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown error");
            return a;
        }
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.get_unique_id || !a.comm_init_rank || !a.all_reduce || !a.comm_destroy || !a.error_string)
            a.err = "libnccl.so.2 lacks ncclGetUniqueId / ncclCommInitRank / ncclAllReduce / ncclCommDestroy";
        return a;
    }();
    if (!api.err.empty()) throw Error(SEGHDC_ERUNTIME, api.err);
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(SEGHDC_ERUNTIME, std::string(what) + ": " + nccl_api().error_string(r));
}

// page-locked host staging (grow-only): pageable caller buffers pass through it, so every
// host<->device copy of the pipeline runs as a true async DMA at PCIe rate
struct PinnedBuf {
    uint8_t* p = nullptr;
    size_t n = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
    uint8_t* ensure(size_t bytes) {
        if (bytes > n) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            n = 0;
            ck(cudaHostAlloc(reinterpret_cast<void**>(&p), bytes, cudaHostAllocPortable), "cudaHostAlloc");
            n = bytes;
        }
        return p;
    }
};

bool is_pinned(const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

struct Geometry {
    uint32_t D = 0, W32 = 0, S32 = 0, SS = 0, nwarp_words = 0, W32P = 0, Dp = 0;
    void set(size_t dim) {
        D = uint32_t(dim);
        W32 = uint32_t((dim + 31) / 32);
        // rows padded to whole 128-byte lines: the encode's 128-byte stores never straddle two
        // lines (0.135 -> 0.126 ms at C1), and a short HV's row is one full TMA box of 32 words
        S32 = (W32 + 31) / 32 * 32;
        SS = S32 + ((S32 % 32 == 0) ? 4 : 0);  // keep LDS.128 of adjacent rows on distinct banks
        nwarp_words = (W32 + 31) / 32;
        W32P = nwarp_words * 32;
        Dp = W32 * 32;
    }
    size_t wph() const { return (D + 63) / 64; }
};

}  // namespace

struct seghdc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sms = 148;
    size_t smem_optin = 0;
    size_t l2_bytes = 126u << 20;
    std::string err;
    uint64_t launches = 0;

    // image (full image on every rank)
    DevBuf<uint8_t> img;
    size_t h = 0, w = 0, c = 0;
    // codebooks
    DevBuf<uint32_t> row, col, wid;
    bool slots_cleared = false;         // cluster_begin's clear kernel already reset the seed slots
    bool flist_cleared = false;         // ... and round 1's changed-pixel list counts
    DevBuf<uint8_t> wid_sup;            // channel set per HV word of wid (EncodeArgs::sup)
    std::vector<uint8_t> wid_sup_host;  // its host copy while an upload may be in flight
    uint32_t enc_nl = 1;                // most channels any HV word has
    DevBuf<uint64_t> cb_bases;  // closed-form Manhattan codebooks: bases expanded on the device
    size_t cb_dim = 0, cb_h = 0, cb_w = 0, cb_c = 0;
    // grid (rows [row_begin,row_end) of an h_total x w image)
    DevBuf<uint32_t> grid;
    Geometry g;
    size_t g_h = 0, g_w = 0, row_begin = 0, row_end = 0;
    bool grid_valid = false, colsum_valid = false;
    uint64_t n_local() const { return uint64_t(row_end - row_begin) * g_w; }
    uint64_t pix_begin() const { return uint64_t(row_begin) * g_w; }
    // clustering state
    size_t K = 0, iterations = 0;
    uint32_t planes = kPlanes;  // 6-bit centroid planes per cluster (planes_for)
    int early_stop = 0;
    RoundPlan plan;
    uint32_t round_ctas = 0;
    DevBuf<uint8_t> state, bfrag;
    DevBuf<uint8_t> bimg;                     // tcgen05 kernel: centroid B image
    alignas(64) unsigned char tmap[128] = {};  // tcgen05 kernel: CUtensorMap of the grid
    DevBuf<uint32_t> labels, Z;
    DevBuf<uint32_t> run1;    // tcgen05 K == 2: running member sums of cluster 1, [2][Dp] by parity
    DevBuf<uint32_t> ticket;  // k_finish_tc: last-block detection
    DevBuf<uint32_t> flist;   // round 1 of the incremental schedule: changed pixels, then their count
    bool xchg_clean = false;  // the fused finish left the exchange buffer zeroed
    DevBuf<int32_t> xchg;
    DevBuf<int32_t> colsum;  // this rank's column sums of its grid (valid while colsum_valid)
    DevBuf<uint64_t> seeds;
    DevBuf<unsigned long long> slots;
    DevBuf<uint16_t> min_dist;
    // closed-form Manhattan variant (seghdc_run_pipeline_closed), grow-only
    struct {
        DevBuf<long long> Q;
        DevBuf<unsigned long long> P, n2, cnt, counts, changed;
        DevBuf<uint32_t> Z, labels;
        DevBuf<int32_t> diff, diffc;
        DevBuf<uint8_t> bf;
    } cf;
    int exchange_phase = 0;  // 0: rounds, 1: init (includes colsums)
    // row-block sharding across ranks (seghdc_nccl_init / seghdc_set_allreduce): this rank's
    // collective for the per-round SUM all-reduce of the exchange buffer
    int rank = 0, nranks = 1;
    ncclComm_t nccl_comm = nullptr;
    seghdc_allreduce_fn ar_fn = nullptr;
    void* ar_user = nullptr;
    // per-round counts of 128-bit-wrapping comparisons of the last clustering run (diagnostic):
    // the packed path keeps them behind its round state, the closed-form variant in wraps_hist
    DevBuf<unsigned long long> wraps_hist;
    const unsigned long long* wraps_src = nullptr;
    size_t wraps_rounds = 0;
    bool assign_vmax_wraps = false;  // seghdc_assign with caller centroids large enough to wrap
    bool count_wraps = false;        // seghdc_set_wrap_counting: the tcgen05 kernels' counting variant
    // run_pipeline: device slot with the caller's mapped label pointer for the last round
    DevBuf<unsigned long long> zc_slot;
    unsigned long long zc_host = 0;
    bool in_pipeline = false;  // launches belong to run_pipeline's device part (may arm zc_slot)
    // run_pipeline: staging buffers, stage events (created once) and the CUDA graph of the
    // device part (codebook expansion, encode, seeds, every round) for the last signature
    PinnedBuf stage_in, stage_out;
    cudaEvent_t stage_ev[3] = {nullptr, nullptr, nullptr};
    struct Graph {
        std::vector<uint64_t> sig;
        uint64_t epoch = 0;
        int seen = 0;  // eager runs with this signature (capture on the second)
        cudaGraphExec_t exec = nullptr;
        uint64_t launches = 0;
        bool failed = false;
    } graph;
    // seghdc_run_pipeline_batch: child contexts, each on its own stream with a share of the SMs
    std::vector<seghdc_ctx*> batch;
    // optional CUDA-event timing of every round kernel (bench.py's roofline)
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    size_t prof_used = 0;

    void use() { ck(cudaSetDevice(device), "cudaSetDevice"); }
    size_t xchg_round_ints() const { return K * g.Dp + K + 1; }
    // the tcgen05 round kernel re-bundles incrementally (deltas of clusters 1..K-1): K == 2
    // with the fused k_finish_tc, K = 3, 4 with k_fold_list every round and k_finish
    bool incremental() const { return plan.tc && K >= 2 && K <= 8; }
    // K == 2 on the one-CTA 16-column layout: fold warps in the round kernel + fused k_finish_tc
    bool fold_warps() const { return plan.tc && K == 2 && seghdc_dev::tc_ncol(2, g.W32) == 16; }
    int32_t* colsum_ptr() { return xchg.p + xchg_round_ints(); }
    void count(uint64_t k = 1) { launches += k; }
    void check_launch() { ck(cudaGetLastError(), "kernel launch"); }
};

namespace {

template <class F>
int guarded(seghdc_ctx* ctx, F&& f) {
    try {
        if (ctx) ctx->use();
        f();
        return SEGHDC_OK;
    } catch (const Error& e) {
        (ctx ? ctx->err : g_thread_err) = e.what();
        return e.code;
    } catch (const std::exception& e) {
        (ctx ? ctx->err : g_thread_err) = e.what();
        return SEGHDC_ERUNTIME;
    }
}

void require(bool cond, const std::string& msg) {
    if (!cond) throw Error(SEGHDC_ECONFIG, msg);
}

// ---- resident data ---------------------------------------------------------------------------
void load_image(seghdc_ctx& x, const uint8_t* px, size_t h, size_t w, size_t c) {
    seghdc_host::validate_image(h, w, c);
    x.img.ensure(h * w * c + 64);  // the encode kernel reads whole 4-pixel groups (up to 16 bytes past a ragged row end)
    // host or device pointer (unified addressing): a batch kept resident in HBM loads D2D
    ck(cudaMemcpyAsync(x.img.p, px, h * w * c, cudaMemcpyDefault, x.stream), "upload image");
    x.h = h;
    x.w = w;
    x.c = c;
}

void load_codebooks(seghdc_ctx& x, size_t dim, size_t h, size_t w, size_t c, const uint64_t* row,
                    const uint64_t* col, const uint64_t* wid) {
    const size_t wph = (dim + 63) / 64, wref = 2 * wph;
    x.row.ensure(h * wref);
    x.col.ensure(w * wref);
    x.wid.ensure(c * 256 * wref);
    ck(cudaMemcpyAsync(x.row.p, row, h * wph * 8, cudaMemcpyHostToDevice, x.stream), "upload rows");
    ck(cudaMemcpyAsync(x.col.p, col, w * wph * 8, cudaMemcpyHostToDevice, x.stream), "upload cols");
    ck(cudaMemcpyAsync(x.wid.p, wid, c * 256 * wph * 8, cudaMemcpyHostToDevice, x.stream), "upload colour tables");
    // channel set per 32-bit HV word, from the tables themselves (any caller tables stay exact)
    ck(cudaStreamSynchronize(x.stream), "sync");  // a previous upload may still read wid_sup_host
    x.wid_sup_host.assign(wref, 0);
    for (size_t ch = 0; ch < c && ch < 3; ++ch)
        for (size_t q = 0; q < wph; ++q) {
            uint64_t any = 0;
            for (size_t v = 0; v < 256; ++v) any |= wid[(ch * 256 + v) * wph + q];
            if (uint32_t(any)) x.wid_sup_host[2 * q] |= uint8_t(1u << ch);
            if (any >> 32) x.wid_sup_host[2 * q + 1] |= uint8_t(1u << ch);
        }
    x.enc_nl = 1;
    for (uint8_t m : x.wid_sup_host) x.enc_nl = std::max<uint32_t>(x.enc_nl, uint32_t(__builtin_popcount(m)));
    x.wid_sup.ensure(wref);
    ck(cudaMemcpyAsync(x.wid_sup.p, x.wid_sup_host.data(), wref, cudaMemcpyHostToDevice, x.stream), "upload support");
    x.cb_dim = dim;
    x.cb_h = h;
    x.cb_w = w;
    x.cb_c = c;
}

// Manhattan codebooks from their bases: only (2 + C) HVs cross PCIe, the tables are expanded
// on the device (k_expand_codebooks); same tables as load_codebooks of the host-built ones.
void upload_bases(seghdc_ctx& x, const seghdc_host::ManhattanParams& p, const uint64_t* bases) {
    const size_t wph = (p.dim + 63) / 64, wref = 2 * wph;
    x.row.ensure(size_t(p.h) * wref);
    x.col.ensure(size_t(p.w) * wref);
    x.wid.ensure(size_t(p.c) * 256 * wref);
    x.cb_bases.ensure((2 + p.c) * wph);
    x.wid_sup.ensure(wref);  // written by the expansion kernel
    x.enc_nl = 1;
    for (size_t q = 0; q < wref; ++q)
        x.enc_nl = std::max<uint32_t>(
            x.enc_nl, uint32_t(__builtin_popcount(manhattan_word_channels(p.dim, p.c, p.off, uint32_t(q)))));
    ck(cudaMemcpyAsync(x.cb_bases.p, bases, (2 + p.c) * wph * 8, cudaMemcpyHostToDevice, x.stream), "upload bases");
    x.cb_dim = p.dim;
    x.cb_h = p.h;
    x.cb_w = p.w;
    x.cb_c = p.c;
}

void expand_codebooks(seghdc_ctx& x, const seghdc_host::ManhattanParams& p) {
    const size_t wph = (p.dim + 63) / 64, wref = 2 * wph;
    ExpandArgs a{};
    a.dim = p.dim;
    a.h = p.h;
    a.w = p.w;
    a.c = p.c;
    a.beta = p.beta;
    a.x_row = p.x_row;
    a.x_col = p.x_col;
    a.wref = uint32_t(wref);
    for (int i = 0; i < 3; ++i) {
        a.off[i] = p.off[i];
        a.unit[i] = p.unit[i];
    }
    launch_expand_codebooks(reinterpret_cast<const uint32_t*>(x.cb_bases.p), a, x.row.p, x.col.p, x.wid.p, x.wid_sup.p,
                            x.stream);
    x.count();
    x.check_launch();
}

void set_grid_shape(seghdc_ctx& x, size_t h, size_t w, size_t dim, size_t r0, size_t r1) {
    require(dim >= 1, "hypervector dimension must be >= 1");
    require(dim <= 65536, "dim > 65536 exceeds the exact-integer range of the IMMA similarity kernel");
    require(r0 < r1 && r1 <= h, "row range out of bounds");
    x.g.set(dim);
    x.g_h = h;
    x.g_w = w;
    x.row_begin = r0;
    x.row_end = r1;
    x.grid.ensure(size_t(x.n_local()) * x.g.S32);
    x.colsum_valid = false;
}

void encode_rows(seghdc_ctx& x, size_t r0, size_t r1) {
    require(x.cb_dim > 0 && x.cb_h == x.h && x.cb_w == x.w && x.cb_c == x.c,
            "codebooks do not match the loaded image");
    set_grid_shape(x, x.h, x.w, x.cb_dim, r0, r1);
    EncodeArgs a{};
    a.img = x.img.p;
    a.w = uint32_t(x.w);
    a.c = uint32_t(x.c);
    a.pix_begin = uint64_t(r0) * x.w;
    a.pix_end = uint64_t(r1) * x.w;
    a.row = x.row.p;
    a.col = x.col.p;
    a.wid = x.wid.p;
    a.sup = x.wid_sup.p;
    a.nl_max = x.enc_nl;
    a.wref = uint32_t(2 * x.g.wph());
    a.S32 = x.g.S32;
    a.W32 = x.g.W32;
    a.grid = x.grid.p;
    x.colsum.ensure(x.g.Dp);
    ck(cudaMemsetAsync(x.colsum.p, 0, x.g.Dp * 4, x.stream), "clear colsum");
    a.colsum = reinterpret_cast<uint32_t*>(x.colsum.p);
    a.sms = uint32_t(x.sms);
    launch_encode(a, x.stream);
    x.count();
    x.check_launch();
    x.grid_valid = true;
    x.colsum_valid = true;  // the encode kernel accumulates the column sums as it writes
}

void load_grid(seghdc_ctx& x, const uint64_t* grid, size_t h, size_t w, size_t dim, size_t r0, size_t r1) {
    set_grid_shape(x, h, w, dim, r0, r1);
    ck(cudaMemsetAsync(x.grid.p, 0, size_t(x.n_local()) * x.g.S32 * 4, x.stream), "clear grid");
    const size_t wph = x.g.wph();
    ck(cudaMemcpy2DAsync(x.grid.p, x.g.S32 * 4, grid + size_t(r0) * w * wph, wph * 8, wph * 8, x.n_local(),
                         cudaMemcpyHostToDevice, x.stream),
       "upload grid");
    x.grid_valid = true;
}

void store_grid(seghdc_ctx& x, uint64_t* out) {
    require(x.grid_valid, "no resident grid");
    const size_t wph = x.g.wph();
    ck(cudaMemcpy2DAsync(out, wph * 8, x.grid.p, x.g.S32 * 4, wph * 8, x.n_local(), cudaMemcpyDeviceToHost,
                         x.stream),
       "download grid");
    ck(cudaStreamSynchronize(x.stream), "sync");
}

// ---- clustering schedule ----------------------------------------------------------------------
// planes of kPlaneBits bits needed for centroid entries <= vmax (at least kPlanes)
uint32_t planes_for(uint64_t vmax) {
    uint32_t p = kPlanes;
    while (p * kPlaneBits < 64 && (vmax >> (p * kPlaneBits)) != 0) ++p;
    return p;
}

// vmax: largest centroid entry the round kernels must represent (0: member counts, i.e. the
// image's pixel count)
void alloc_cluster(seghdc_ctx& x, size_t K, uint64_t vmax = 0) {
    require(x.grid_valid, "no resident grid: encode or load a grid first");
    // centroid entries are member counts <= pixels; the IMMA kernels split them into 6-bit
    // planes (kernels.cuh): 4 planes below 2^24 pixels, 5 below 2^30
    require(uint64_t(x.g_h) * x.g_w < (1ull << 28), "images of 2^28 pixels or more are not supported");
    if (vmax == 0) vmax = uint64_t(x.g_h) * x.g_w;
    const uint32_t planes = planes_for(vmax);
    const Geometry& g = x.g;
    x.planes = planes;
    if (!plan_round(uint32_t(K), planes, g.W32, g.SS, x.plan, x.smem_optin))
        throw Error(SEGHDC_ERUNTIME, "dim " + std::to_string(g.D) + " does not fit the round kernel's shared memory");
    if (x.plan.tc && vmax > tc_max_value(uint32_t(K), g.W32)) x.plan.tc = false;  // beyond the layout's digits
    x.K = K;
    const uint64_t n = x.n_local();
    if (x.plan.tc && !tc_make_grid_map(x.tmap, x.grid.p, n, g.S32)) x.plan.tc = false;  // no driver entry point
    const uint64_t tp = x.plan.tc ? tc_tile_pixels() : 16ull * x.plan.mt;
    // balanced waves: as few CTAs as give every CTA the same number of tiles as with x.sms
    // (C0: 512 tiles -> 128 CTAs x 4 instead of 148 CTAs with 3 or 4)
    {
        const uint64_t tiles = std::max<uint64_t>(1, (n + tp - 1) / tp);
        const uint64_t per = (tiles + x.sms - 1) / x.sms;
        x.round_ctas = uint32_t(std::max<uint64_t>(1, (tiles + per - 1) / per));
    }
    const uint32_t NT = x.plan.nt;
    x.state.ensure(StateView::bytes(uint32_t(K), x.iterations));
    x.labels.ensure(n + 4);  // +4: the fused kernel's TMA of a tile's labels rounds up to 16 B
    x.Z.ensure(K * g.D);
    // B fragments: entries of words >= W32 must stay zero -> clear on every (re)plan
    x.bfrag.ensure(size_t(NT) * x.plan.w32p * 32 * 8);
    ck(cudaMemsetAsync(x.bfrag.p, 0, x.bfrag.bytes(), x.stream), "clear bfrag");
    if (x.plan.tc) x.bimg.ensure(tc_bimg_bytes(uint32_t(K), g.W32));
    x.xchg.ensure(x.xchg_round_ints() + g.Dp);
    if (x.incremental()) {
        x.run1.ensure(2 * K * size_t(g.Dp));  // [2][Dp] (K == 2) or [2][K][Dp]
        x.flist.ensure((K - 1) * (n + 1));
        x.ticket.ensure(1);
        ck(cudaMemsetAsync(x.ticket.p, 0, 4, x.stream), "clear ticket");
    }
    x.xchg_clean = false;
    x.colsum.ensure(g.Dp);
    x.seeds.ensure(std::max<size_t>(K, 1));
    x.slots.ensure(2 + K);
    x.min_dist.ensure(x.h * x.w);
}

// Column sums of a grid that did not come from encode (encode computes them on the fly):
// every pixel counts as "cluster 0" of a Harley-Seal accumulation.
void compute_colsum(seghdc_ctx& x) {
    x.colsum.ensure(x.g.Dp);
    ck(cudaMemsetAsync(x.colsum.p, 0, x.g.Dp * 4, x.stream), "clear colsum");
    AccumulateArgs a{};
    a.grid = x.grid.p;
    a.S32 = x.g.S32;
    a.W32 = x.g.W32;
    a.n = x.n_local();
    a.labels = nullptr;
    a.K = 1;
    a.skip_mode = -1;
    a.state = nullptr;
    a.parity = 0;
    a.dst = reinterpret_cast<uint32_t*>(x.colsum.p);
    a.Dp = x.g.Dp;
    a.counts_dst = nullptr;
    a.sms = uint32_t(x.sms);
    launch_accumulate(a, x.stream);
    x.count();
    x.check_launch();
    x.colsum_valid = true;
}

void select_seeds_dev(seghdc_ctx& x, size_t K) {
    SeedArgs a{};
    a.img = x.img.p;
    a.n = uint64_t(x.h) * x.w;
    a.h = uint32_t(x.h);
    a.w = uint32_t(x.w);
    a.c = uint32_t(x.c);
    a.K = uint32_t(K);
    a.min_dist = x.min_dist.p;
    a.seeds = x.seeds.p;
    a.slots = x.slots.p;
    a.hdr = reinterpret_cast<RoundState*>(x.state.p);
    a.slots_cleared = x.slots_cleared;
    a.defer_post = x.slots_cleared;  // inside cluster_begin: k_init_seeds follows
    x.slots_cleared = false;
    launch_select_seeds(a, x.stream);
    x.count((a.defer_post && K <= 2 ? 1 : 2) + (K > 2 ? (K - 2) + 1 : 0));
    x.check_launch();
}

void finish(seghdc_ctx& x, int mode, uint32_t round) {
    if (mode == 0 && x.fold_warps()) {  // one fused kernel per round
        launch_finish_tc(x.g.D, x.g.W32, x.g.Dp, x.xchg.p, x.colsum_ptr(), x.Z.p, x.run1.p, x.bimg.p, x.state.p,
                         round, x.early_stop, x.ticket.p, x.stream);
        x.count();
        x.check_launch();
        x.xchg_clean = true;
        return;
    }
    const uint32_t np = (round & 1) ^ 1;
    // (init: cluster_begin has just cleared the whole state, norm2 included)
    if (mode != 1) launch_prep_finish(x.state.p, uint32_t(x.K), np, x.stream);
    FinishArgs f{};
    f.mode = mode;
    f.K = uint32_t(x.K);
    f.P = x.planes;
    f.D = x.g.D;
    f.W32 = x.g.W32;
    f.W32P = x.plan.w32p;
    f.Dp = x.g.Dp;
    f.xchg = x.xchg.p;
    f.colsum = x.colsum_ptr();
    f.Z = x.Z.p;
    f.bfrag = x.bfrag.p;
    f.state = x.state.p;
    f.round = round;
    f.early_stop = x.early_stop;
    f.run = (mode == 0 && x.incremental()) ? x.run1.p : nullptr;
    launch_finish(f, x.stream);
    x.count(mode != 1 ? 2 : 1);
    if (x.plan.tc) {
        // init (mode 1): the same kernel zeroes the exchange buffer k_finish has just consumed
        launch_build_bimg(x.Z.p, uint32_t(x.K), x.g.D, x.g.W32, x.bimg.p, mode == 0 ? x.state.p : nullptr, x.stream,
                          mode == 1 ? reinterpret_cast<uint32_t*>(x.xchg.p) : nullptr,
                          mode == 1 ? uint32_t(x.xchg_round_ints()) : 0u);
        x.count();
        if (mode == 1) x.xchg_clean = true;
    }
    x.check_launch();
}

// Everything up to (not including) the all-reduce of the init exchange.
void cluster_begin(seghdc_ctx& x, size_t K, size_t iterations, int early_stop) {
    require(x.h > 0 && x.w == x.g_w && x.h == x.g_h, "image and grid shapes differ");
    seghdc_host::validate_cluster(K, iterations, x.h * x.w);
    x.iterations = iterations;
    alloc_cluster(x, K);
    x.early_stop = early_stop;
    // one launch clears the round state, the running sums and the seed slots (was three memsets)
    launch_init_clear(x.state.p, StateView::bytes(uint32_t(K), iterations), x.run1.p,
                      x.incremental() ? 2 * x.K * size_t(x.g.Dp) * 4 : 0, x.slots.p, uint32_t(2 + K),
                      x.incremental() ? x.flist.p + (x.K - 1) * x.n_local() : nullptr,
                      x.incremental() ? uint32_t(x.K - 1) : 0u, x.stream);
    x.count();
    x.slots_cleared = true;
    x.flist_cleared = x.incremental();  // round 1's list counts are zero already
    x.wraps_src = StateView::at(x.state.p, uint32_t(K)).wraps;
    x.wraps_rounds = 0;
    // labels start at 0xFFFFFFFF ("no cluster"); the tcgen05 round kernel takes that as given in
    // round 1 instead of reading them, so only the other kernels need the buffer cleared
    if (!x.plan.tc) ck(cudaMemsetAsync(x.labels.p, 0xFF, x.n_local() * 4, x.stream), "clear labels");
    select_seeds_dev(x, K);
    if (!x.colsum_valid) compute_colsum(x);
    InitSeedArgs a{};
    a.grid = x.grid.p;
    a.S32 = x.g.S32;
    a.pix_begin = x.pix_begin();
    a.n_local = x.n_local();
    a.seeds = x.seeds.p;
    a.K = uint32_t(K);
    a.W32 = x.g.W32;
    a.Dp = x.g.Dp;
    a.xchg = x.xchg.p;
    // local column sums into the exchange tail (inside the same kernel); the init all-reduce
    // makes them global
    a.post_slots = K <= 2 ? x.slots.p : nullptr;
    a.h = uint32_t(x.h);
    a.w = uint32_t(x.w);
    a.hdr = reinterpret_cast<RoundState*>(x.state.p);
    a.colsum_src = reinterpret_cast<const int32_t*>(x.colsum.p);
    a.colsum_dst = reinterpret_cast<int32_t*>(x.colsum_ptr());
    launch_init_seeds(a, x.stream);
    x.count();
    x.check_launch();
    x.exchange_phase = 1;
}

void init_finish(seghdc_ctx& x) {
    finish(x, 1, 0);
    x.exchange_phase = 0;
}

void round_assign(seghdc_ctx& x, uint32_t r) {
    const bool do_update = r < x.iterations;
    RoundArgs a{};
    a.grid = x.grid.p;
    a.n = x.n_local();
    a.S32 = x.g.S32;
    a.SS = x.g.SS;
    a.W32 = x.g.W32;
    a.W32P = x.plan.w32p;
    a.nwarp_words = x.g.nwarp_words;
    a.K = uint32_t(x.K);
    a.P = x.planes;
    a.NT = x.plan.nt;
    a.bfrag = reinterpret_cast<const uint64_t*>(x.bfrag.p);
    a.labels = x.labels.p;
    a.state = x.state.p;
    a.round = r;
    a.do_update = do_update ? 1 : 0;
    a.xchg = x.xchg.p;
    a.Dp = x.g.Dp;
    a.ctas = x.round_ctas;
    a.tmap = x.tmap;
    a.bimg = x.bimg.p;
    a.nks = tc_ksteps(x.g.W32);
    // round 1 of the incremental schedule folds every member of cluster 1 through a global list
    // and the whole-GPU k_fold_list instead of the per-CTA fold warps (whose load follows the
    // nuclei's layout). Later rounds change few pixels and fold in the round kernel.
    // SEGHDC_FLIST: 0 = fold warps in every round, 1 = list in round 1 (default), 2 = always.
    static const char* fe = getenv("SEGHDC_FLIST");
    const int flist_mode = fe ? atoi(fe) : 1;  // measured: lists in every round cost +5 us per round
    const bool use_flist =
        do_update && x.incremental() && (!x.fold_warps() || flist_mode == 2 || (flist_mode == 1 && r == 1));
    {
        static const char* se = getenv("SEGHDC_SERPENTINE");
        a.serpentine = (se && *se == '0') ? 0u : 1u;
        // L2 prefetch distance (chunks) of the producer, SEGHDC_PF; default off: measured slower
        // for every layout (round 2: C3 1050 vs 1100 us per round at 8, C4 12.2 vs 12.6 ms)
        static const char* pe = getenv("SEGHDC_PF");
        a.pf = pe ? uint32_t(atoi(pe)) : 0u;
    }
    // entries are member sums <= the image's pixel count n, so norm2 <= D n^2 and every
    // cross product of strictly_closer is below D^3 n^4: no wrap possible under 2^128
    {
        const double n_img = double(x.g_h) * double(x.g_w), D = double(x.g.D);
        a.wraps = x.count_wraps &&
                  (std::log2(D) * 3 + std::log2(std::max(n_img, 1.0)) * 4 >= 127.0 || x.assign_vmax_wraps);
    }
    a.labels_host_slot = (x.in_pipeline && r == x.iterations) ? x.zc_slot.p : nullptr;
    a.flist = use_flist ? x.flist.p : nullptr;
    a.flist_count = use_flist ? x.flist.p + (x.K - 1) * x.n_local() : nullptr;
    if (use_flist && !(r == 1 && x.flist_cleared))
        ck(cudaMemsetAsync(a.flist_count, 0, (x.K - 1) * 4, x.stream), "clear fold lists");
    x.flist_cleared = false;
    // the round's CTAs fold their exact sums, member counts and changes into the exchange buffer
    if (!x.xchg_clean) ck(cudaMemsetAsync(x.xchg.p, 0, x.xchg_round_ints() * 4, x.stream), "clear exchange");
    x.xchg_clean = false;
    cudaEvent_t ev_end = nullptr;
    if (x.profiling) {
        if (x.prof_used == x.prof_events.size()) {
            cudaEvent_t e0, e1;
            ck(cudaEventCreate(&e0), "event");
            ck(cudaEventCreate(&e1), "event");
            x.prof_events.emplace_back(e0, e1);
        }
        ck(cudaEventRecord(x.prof_events[x.prof_used].first, x.stream), "event");
        ev_end = x.prof_events[x.prof_used++].second;
    }
    ck(launch_round(a, x.plan, x.stream), "round kernel");
    if (ev_end) ck(cudaEventRecord(ev_end, x.stream), "event");
    x.count();
    if (use_flist) {
        launch_fold_list(a.flist, a.flist_count, x.n_local(), uint32_t(x.K - 1), x.grid.p, x.g.S32, x.g.W32,
                         x.xchg.p + x.g.Dp, x.g.Dp, uint32_t(x.sms), x.stream);
        x.count();
        x.check_launch();
    }
    if (do_update && !x.plan.fused && !x.incremental()) {  // K >= 3: separate single-read accumulation pass
        AccumulateArgs u{};
        u.grid = x.grid.p;
        u.S32 = x.g.S32;
        u.W32 = x.g.W32;
        u.n = x.n_local();
        u.labels = x.labels.p;
        u.K = uint32_t(x.K);
        u.skip_mode = -2;
        u.state = x.state.p;
        u.parity = r & 1;
        u.dst = reinterpret_cast<uint32_t*>(x.xchg.p);
        u.Dp = x.g.Dp;
        u.counts_dst = nullptr;  // member counts come from the round kernel
        u.sms = uint32_t(x.sms);
        launch_accumulate(u, x.stream);
        x.count();
        x.check_launch();
    }
}

struct HostState {
    RoundState hdr;
    std::vector<uint32_t> cur[2];
};

HostState read_state(seghdc_ctx& x) {
    std::vector<uint8_t> buf(StateView::bytes(uint32_t(x.K)));
    ck(cudaMemcpyAsync(buf.data(), x.state.p, buf.size(), cudaMemcpyDeviceToHost, x.stream), "read state");
    ck(cudaStreamSynchronize(x.stream), "sync");
    StateView v = StateView::at(buf.data(), uint32_t(x.K));
    HostState h;
    h.hdr = *v.hdr;
    for (int p = 0; p < 2; ++p) h.cur[p].assign(v.cur + p * x.K, v.cur + (p + 1) * x.K);
    return h;
}

void run_rounds(seghdc_ctx& x, seghdc_round_cb cb, void* user) {
    std::vector<uint32_t> host_labels;
    if (cb) host_labels.resize(x.n_local());
    for (uint32_t r = 1; r <= x.iterations; ++r) {
        round_assign(x, r);
        if (cb) {
            ck(cudaMemcpyAsync(host_labels.data(), x.labels.p, x.n_local() * 4, cudaMemcpyDeviceToHost, x.stream),
               "download labels");
            ck(cudaStreamSynchronize(x.stream), "sync");
            cb(user, r, host_labels.data());
        }
        if (r < x.iterations) {
            finish(x, 0, r);
            if (cb && x.early_stop && read_state(x).hdr.done) break;
        }
    }
}

void fetch(seghdc_ctx& x, uint32_t* labels, uint32_t* centroids, uint64_t* counts, size_t* rounds) {
    if (labels)
        ck(cudaMemcpyAsync(labels, x.labels.p, x.n_local() * 4, cudaMemcpyDeviceToHost, x.stream), "download labels");
    if (centroids)
        ck(cudaMemcpyAsync(centroids, x.Z.p, x.K * x.g.D * 4, cudaMemcpyDeviceToHost, x.stream), "download centroids");
    const HostState h = read_state(x);  // synchronises
    if (rounds) *rounds = h.hdr.rounds_run;
    if (counts)
        for (size_t c = 0; c < x.K; ++c) counts[c] = h.cur[h.hdr.rounds_run & 1][c];
}

// ---- row-block sharding with the collective inside the library ---------------------------------
// rank r of n owns rows [r0, r1): contiguous blocks, sizes differing by at most one row
void shard_rows(size_t h, int rank, int nranks, size_t& r0, size_t& r1) {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "shard: rank out of range");
    require(size_t(nranks) <= h, "shard: more ranks than image rows");
    const size_t base = h / size_t(nranks), extra = h % size_t(nranks), r = size_t(rank);
    r0 = r * base + std::min(r, extra);
    r1 = r0 + base + (r < extra ? 1 : 0);
}

// SUM all-reduce of the current exchange buffer ([K*Dp sums | K counts | changed], plus the
// column sums at init) over the ranks, ordered on the context's stream
void allreduce_exchange(seghdc_ctx& x) {
    const size_t n = x.xchg_round_ints() + (x.exchange_phase == 1 ? x.g.Dp : 0);
    if (x.nccl_comm) {
        nck(nccl_api().all_reduce(x.xchg.p, x.xchg.p, n, ncclInt32, ncclSum, x.nccl_comm, x.stream), "ncclAllReduce");
    } else if (x.ar_fn) {
        if (x.ar_fn(x.ar_user, x.xchg.p, n, x.stream) != 0) throw Error(SEGHDC_ERUNTIME, "all-reduce callback failed");
    } else {
        require(x.nranks == 1, "sharded clustering needs a collective (seghdc_nccl_init or seghdc_set_allreduce)");
    }
}

// cluster() (clusterer.cpp:190-218) over this rank's rows: the seeds come from the full image
// on every rank (no communication), the only exchange is one all-reduce per round. Integer
// sums are order independent, so every rank finalises bit-identical centroids and the labels
// equal the single-GPU run's. No host synchronisation.
void cluster_sharded(seghdc_ctx& x, size_t K, size_t iterations, int early_stop) {
    size_t r0, r1;
    shard_rows(x.h, x.rank, x.nranks, r0, r1);
    require(x.grid_valid && x.row_begin == r0 && x.row_end == r1 && x.g_h == x.h,
            "sharded cluster: the resident grid must hold exactly this rank's rows (seghdc_shard_rows)");
    cluster_begin(x, K, iterations, early_stop);
    allreduce_exchange(x);
    init_finish(x);
    for (uint32_t r = 1; r <= iterations; ++r) {
        round_assign(x, r);
        if (r < iterations) {
            allreduce_exchange(x);
            finish(x, 0, r);
        }
    }
}

void cluster_full(seghdc_ctx& x, size_t K, size_t iterations, int early_stop, seghdc_round_cb cb, void* user) {
    cluster_begin(x, K, iterations, early_stop);
    init_finish(x);
    run_rounds(x, cb, user);
}

// ---- run_pipeline (pipeline.cpp:40-75) ---------------------------------------------------------
struct PipelineCall {
    const uint8_t* pixels;
    size_t h, w, c, dim;
    double alpha;
    size_t beta, gamma, k, iterations;
    uint64_t seed;
    int encoder, early_stop;
};

// The device part of the pipeline, everything between the input upload and the result
// download: codebook expansion (Manhattan), encode of rows [r0, r1), seeds, every round.
// capturing: the stage events become event-record nodes of the graph (cudaEventRecordExternal)
void pipeline_device(seghdc_ctx& x, const PipelineCall& pc, const seghdc_host::ManhattanParams* mp, size_t r0,
                     size_t r1, bool sharded, seghdc_round_cb cb, void* user, bool capturing) {
    auto stamp = [&](int i) {
        ck(capturing ? cudaEventRecordWithFlags(x.stage_ev[i], x.stream, cudaEventRecordExternal)
                     : cudaEventRecord(x.stage_ev[i], x.stream),
           "event");
    };
    if (mp) expand_codebooks(x, *mp);
    stamp(0);
    encode_rows(x, r0, r1);
    stamp(1);
    if (sharded)
        cluster_sharded(x, pc.k, pc.iterations, pc.early_stop);
    else
        cluster_full(x, pc.k, pc.iterations, pc.early_stop, cb, user);
    stamp(2);
}

// The device part of one pipeline call on x's stream: eager on the first call with a given
// signature, captured into a CUDA graph on the second, replayed from then on.
// zc_labels (nullable): device-mapped caller label buffer; returns whether the last round was
// armed to write it (tcgen05 plan of this same signature, early stop off, no callback)
bool run_device_part(seghdc_ctx& x, const PipelineCall& pc, const seghdc_host::ManhattanParams* mpp, size_t r0,
                     size_t r1, bool sharded, seghdc_round_cb cb, void* user, void* zc_labels = nullptr) {
    const size_t h = pc.h, w = pc.w, c = pc.c, dim = pc.dim;
    const bool manhattan = mpp != nullptr;
    const seghdc_host::ManhattanParams mp = mpp ? *mpp : seghdc_host::ManhattanParams{};
    for (auto& e : x.stage_ev)
        if (!e) ck(cudaEventCreate(&e), "event");
    // the device part: eager, or one graph launch
    static const char* ge = getenv("SEGHDC_GRAPH");
    // (a host-staged all-reduce callback synchronises, so it cannot live inside a graph)
    const bool graphs = !cb && !x.ar_fn && !(ge && *ge == '0');
    std::vector<uint64_t> sig = {h, w, c, dim, pc.k, pc.iterations, uint64_t(pc.encoder), uint64_t(pc.early_stop),
                                 r0, r1, uint64_t(sharded), uint64_t(x.sms), uint64_t(x.nranks),
                                 reinterpret_cast<uint64_t>(x.nccl_comm), reinterpret_cast<uint64_t>(x.ar_fn)};
    if (manhattan)
        for (uint64_t v : {uint64_t(mp.beta), uint64_t(mp.x_row), uint64_t(mp.x_col), uint64_t(mp.off[1]),
                           uint64_t(mp.off[2]), uint64_t(mp.unit[0]), uint64_t(mp.unit[1]), uint64_t(mp.unit[2])})
            sig.push_back(v);
    auto& G = x.graph;
    const bool same = G.sig == sig && G.epoch == g_realloc_epoch.load();
    if (!same) {
        if (G.exec) cudaGraphExecDestroy(G.exec);
        G = {};
        G.sig = sig;
        G.epoch = g_realloc_epoch.load();
    }
    // a plan for this signature exists once it ran eagerly; only tcgen05 plans write host labels
    const bool zc = zc_labels && !cb && !pc.early_stop && G.seen > 0 && x.plan.tc;
    x.zc_slot.ensure(1);
    x.zc_host = zc ? reinterpret_cast<unsigned long long>(zc_labels) : 0ull;
    ck(cudaMemcpyAsync(x.zc_slot.p, &x.zc_host, 8, cudaMemcpyHostToDevice, x.stream), "label slot");
    x.in_pipeline = true;
    struct Reset {
        seghdc_ctx& x;
        ~Reset() { x.in_pipeline = false; }
    } reset{x};
    bool ran = false;
    if (graphs && G.exec) {
        ck(cudaGraphLaunch(G.exec, x.stream), "cudaGraphLaunch");
        x.count(G.launches);
        ran = true;
    } else if (graphs && G.seen >= 1 && !G.failed) {
        // capture the device part (every buffer is already allocated by the eager run)
        const uint64_t l0 = x.launches;
        cudaGraph_t graph = nullptr;
        bool ok = cudaStreamBeginCapture(x.stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            try {
                pipeline_device(x, pc, mpp, r0, r1, sharded, nullptr, nullptr, true);
            } catch (const Error&) {
                ok = false;
            }
            ok = (cudaStreamEndCapture(x.stream, &graph) == cudaSuccess) && ok && graph;
        }
        if (ok && g_realloc_epoch.load() == G.epoch &&
            cudaGraphInstantiateWithFlags(&G.exec, graph, 0) == cudaSuccess) {
            G.launches = x.launches - l0;
            x.launches = l0;
        } else {
            G.exec = nullptr;
            G.failed = true;
            x.launches = l0;
        }
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();  // a failed capture leaves a sticky-free error; clear it
        if (G.exec) {
            ck(cudaGraphLaunch(G.exec, x.stream), "cudaGraphLaunch");
            x.count(G.launches);
            ran = true;
        }
    }
    if (!ran) {
        pipeline_device(x, pc, mpp, r0, r1, sharded, cb, user, false);
        G.seen++;
    }
    return zc;
}

// run_pipeline: validation and codebooks on the host (one Rng, position then colour), then the
// device part. Without a per-round callback the device part is one CUDA graph per call
// signature (captured on the second call with the same shapes, replayed afterwards); inputs
// and labels cross PCIe through page-locked staging when the caller's buffers are pageable.
void run_pipeline_impl(seghdc_ctx& x, const PipelineCall& pc, seghdc_round_cb cb, void* user, uint32_t* labels_out,
                       uint32_t* centroids_out, uint64_t* counts_out, size_t* rounds_out, double* timings,
                       bool sharded) {
    using Clock = std::chrono::steady_clock;
    auto ms = [](Clock::time_point t0) { return std::chrono::duration<double, std::milli>(Clock::now() - t0).count(); };
    const size_t h = pc.h, w = pc.w, c = pc.c, dim = pc.dim;
    // RunConfig::validate before any work (pipeline.cpp:25-30, 42)
    seghdc_host::validate_image(h, w, c);
    seghdc_host::validate_position(dim, h, w, pc.alpha, pc.beta);
    seghdc_host::validate_color(dim, c, pc.gamma);
    seghdc_host::validate_cluster(pc.k, pc.iterations, h * w);
    size_t r0 = 0, r1 = h;
    if (sharded) shard_rows(h, x.rank, x.nranks, r0, r1);
    const auto t_total = Clock::now();
    const size_t wph = (dim + 63) / 64, img_bytes = h * w * c;
    const bool manhattan = pc.encoder == SEGHDC_ENCODER_MANHATTAN;
    for (auto& e : x.stage_ev)
        if (!e) ck(cudaEventCreate(&e), "event");
    std::mt19937_64 rng(pc.seed);  // one stream: position codebook, then colour (pipeline.cpp:43-59)
    double t_pos = 0, t_col = 0;
    // inputs: the image (and the Manhattan bases) staged together, one H2D each
    const size_t nb = manhattan ? (2 + c) * wph : 0;
    const bool px_pinned = is_pinned(pc.pixels);
    uint8_t* stage = x.stage_in.ensure((px_pinned ? 0 : (img_bytes + 7) / 8 * 8) + nb * 8);
    uint64_t* bases = reinterpret_cast<uint64_t*>(stage + (px_pinned ? 0 : (img_bytes + 7) / 8 * 8));
    ck(cudaStreamSynchronize(x.stream), "sync");  // the staging buffer is free (previous call's copies done)
    seghdc_host::ManhattanParams mp{};
    if (manhattan) {  // closed form: bases on the host, tables expanded on the device
        auto t = Clock::now();
        mp = seghdc_host::manhattan_bases(dim, h, w, c, pc.alpha, pc.beta, pc.gamma, rng, bases);
        t_pos = ms(t);
    }
    const uint8_t* src = pc.pixels;
    if (!px_pinned) {
        std::memcpy(stage, pc.pixels, img_bytes);
        src = stage;
    }
    load_image(x, src, h, w, c);
    if (manhattan) {
        upload_bases(x, mp, bases);
    } else {
        std::vector<uint64_t> row(h * wph), col(w * wph), wid(c * 256 * wph);
        auto t = Clock::now();
        seghdc_host::build_position(dim, h, w, pc.alpha, pc.beta, pc.encoder, rng, row.data(), col.data());
        t_pos = ms(t);
        t = Clock::now();
        seghdc_host::build_color(dim, c, pc.gamma, pc.encoder, rng, wid.data());
        t_col = ms(t);
        load_codebooks(x, dim, h, w, c, row.data(), col.data(), wid.data());
        ck(cudaStreamSynchronize(x.stream), "sync");  // the host tables go out of scope
    }
    // zero-copy labels: a page-locked caller buffer can be written by the last round kernel
    // itself (armed inside run_device_part once this signature's plan is known)
    void* lab_dev = nullptr;
    if (labels_out && !cb && !pc.early_stop && cudaHostGetDevicePointer(&lab_dev, labels_out, 0) != cudaSuccess)
        lab_dev = nullptr;
    cudaGetLastError();
    const bool zc = run_device_part(x, pc, manhattan ? &mp : nullptr, r0, r1, sharded, cb, user, lab_dev);
    // results: labels (this rank's rows) + round state, through the staging buffer unless the
    // caller's label buffer is page-locked
    const size_t n_loc = (r1 - r0) * w, sbytes = StateView::bytes(uint32_t(pc.k));
    const bool lab_pinned = labels_out && is_pinned(labels_out);
    uint8_t* out = x.stage_out.ensure(sbytes + (lab_pinned || !labels_out ? 0 : n_loc * 4));
    if (labels_out && !zc)
        ck(cudaMemcpyAsync(lab_pinned ? static_cast<void*>(labels_out) : static_cast<void*>(out + sbytes), x.labels.p,
                           n_loc * 4, cudaMemcpyDeviceToHost, x.stream),
           "download labels");
    ck(cudaMemcpyAsync(out, x.state.p, sbytes, cudaMemcpyDeviceToHost, x.stream), "read state");
    if (centroids_out)
        ck(cudaMemcpyAsync(centroids_out, x.Z.p, pc.k * dim * 4, cudaMemcpyDeviceToHost, x.stream), "download centroids");
    ck(cudaStreamSynchronize(x.stream), "sync");
    if (labels_out && !lab_pinned) std::memcpy(labels_out, out + sbytes, n_loc * 4);
    const StateView v = StateView::at(out, uint32_t(pc.k));
    if (rounds_out) *rounds_out = v.hdr->rounds_run;
    if (counts_out)
        for (size_t q = 0; q < pc.k; ++q) counts_out[q] = v.cur[size_t(v.hdr->rounds_run & 1) * pc.k + q];
    if (timings) {
        float enc_ms = 0, clu_ms = 0;
        cudaEventElapsedTime(&enc_ms, x.stage_ev[0], x.stage_ev[1]);
        cudaEventElapsedTime(&clu_ms, x.stage_ev[1], x.stage_ev[2]);
        timings[0] = t_pos;
        timings[1] = t_col;
        timings[2] = enc_ms;
        timings[3] = clu_ms;
        timings[4] = ms(t_total);
    }
}

// ---- a batch of same-shape images (the reference CLI's `batch`, seghdc_main.cpp:180-225) -------
// One call runs every image's run_pipeline. The images are dealt round-robin to G child
// contexts, each on its own stream with 1/G of the SMs, so small images run side by side
// (a 256 x 256 image has 512 tiles: one full-GPU grid per image would leave the last wave of
// every round half empty). Each child replays one CUDA graph per image; inputs and labels move
// through page-locked staging; the host synchronises once, at the end.
void run_pipeline_batch(seghdc_ctx& x, const uint8_t* const* pixels, size_t n_img, const PipelineCall& pc,
                        uint32_t* const* labels_out, size_t* rounds_out) {
    const size_t h = pc.h, w = pc.w, c = pc.c, dim = pc.dim;
    require(n_img >= 1, "run_pipeline_batch: no images");
    seghdc_host::validate_image(h, w, c);
    seghdc_host::validate_position(dim, h, w, pc.alpha, pc.beta);
    seghdc_host::validate_color(dim, c, pc.gamma);
    seghdc_host::validate_cluster(pc.k, pc.iterations, h * w);
    static const char* ge = getenv("SEGHDC_BATCH_GROUPS");
    const size_t G = std::min<size_t>(n_img, ge ? std::max(1, atoi(ge)) : 4);
    while (x.batch.size() < G) {
        seghdc_ctx* child = nullptr;
        if (seghdc_create(x.device, &child) != SEGHDC_OK) throw Error(SEGHDC_ERUNTIME, seghdc_last_error(nullptr));
        x.batch.push_back(child);
    }
    for (size_t g = 0; g < G; ++g) {
        x.batch[g]->sms = std::max(1, x.sms / int(G));
        x.batch[g]->count_wraps = x.count_wraps;
    }
    const size_t wph = (dim + 63) / 64, img_bytes = h * w * c, img_slot = (img_bytes + 15) / 16 * 16;
    const bool manhattan = pc.encoder == SEGHDC_ENCODER_MANHATTAN;
    const size_t nb = manhattan ? (2 + c) * wph : 0;
    const size_t n = h * w, sbytes = (StateView::bytes(uint32_t(pc.k)) + 15) / 16 * 16, out_slot = n * 4 + sbytes;
    for (size_t g = 0; g < G; ++g) ck(cudaStreamSynchronize(x.batch[g]->stream), "sync");  // staging free
    uint8_t* in = x.stage_in.ensure(n_img * img_slot + nb * 8);
    uint8_t* out = x.stage_out.ensure(n_img * out_slot);
    uint64_t* bases = reinterpret_cast<uint64_t*>(in + n_img * img_slot);
    std::mt19937_64 rng(pc.seed);  // same shape and seed: one codebook set for every image
    seghdc_host::ManhattanParams mp{};
    std::vector<uint64_t> row, col, wid;
    if (manhattan) {
        mp = seghdc_host::manhattan_bases(dim, h, w, c, pc.alpha, pc.beta, pc.gamma, rng, bases);
    } else {
        row.resize(h * wph);
        col.resize(w * wph);
        wid.resize(c * 256 * wph);
        seghdc_host::build_position(dim, h, w, pc.alpha, pc.beta, pc.encoder, rng, row.data(), col.data());
        seghdc_host::build_color(dim, c, pc.gamma, pc.encoder, rng, wid.data());
    }
    for (size_t g = 0; g < G; ++g) {
        seghdc_ctx& ch = *x.batch[g];
        ch.use();
        if (manhattan) {
            upload_bases(ch, mp, bases);
        } else {
            ch.h = h, ch.w = w, ch.c = c;
            load_codebooks(ch, dim, h, w, c, row.data(), col.data(), wid.data());
        }
    }
    for (size_t i = 0; i < n_img; ++i) {
        seghdc_ctx& ch = *x.batch[i % G];
        ch.use();
        std::memcpy(in + i * img_slot, pixels[i], img_bytes);  // host copy overlaps earlier images' device work
        load_image(ch, in + i * img_slot, h, w, c);
        run_device_part(ch, pc, manhattan ? &mp : nullptr, 0, h, false, nullptr, nullptr);
        uint8_t* o = out + i * out_slot;
        ck(cudaMemcpyAsync(o, ch.labels.p, n * 4, cudaMemcpyDeviceToHost, ch.stream), "download labels");
        ck(cudaMemcpyAsync(o + n * 4, ch.state.p, StateView::bytes(uint32_t(pc.k)), cudaMemcpyDeviceToHost, ch.stream),
           "read state");
    }
    for (size_t g = 0; g < G; ++g) {
        x.batch[g]->use();
        ck(cudaStreamSynchronize(x.batch[g]->stream), "sync");
        x.launches += x.batch[g]->launches;
        x.batch[g]->launches = 0;
    }
    x.use();
    for (size_t i = 0; i < n_img; ++i) {
        const uint8_t* o = out + i * out_slot;
        if (labels_out && labels_out[i]) std::memcpy(labels_out[i], o, n * 4);
        if (rounds_out) rounds_out[i] = StateView::at(const_cast<uint8_t*>(o + n * 4), uint32_t(pc.k)).hdr->rounds_run;
    }
}

}  // namespace

// ================================ C-ABI ========================================================
extern "C" {

int seghdc_create(int device, seghdc_ctx** out) {
    auto ctx = std::make_unique<seghdc_ctx>();
    ctx->device = device;
    const int rc = guarded(nullptr, [&] {
        ck(cudaSetDevice(device), "cudaSetDevice");
        ck(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device), "attr");
        int optin = 0;
        ck(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device), "attr");
        ctx->smem_optin = size_t(optin);
        int l2 = 0;
        ck(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device), "attr");
        if (l2 > 0) ctx->l2_bytes = size_t(l2);
        int major = 0;
        ck(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device), "attr");
        if (major != 10) throw Error(SEGHDC_ERUNTIME, "this build targets sm_100a (B200); device is sm_" + std::to_string(major) + "x");
        ck(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
        ctx->own_stream = true;
    });
    if (rc != SEGHDC_OK) return rc;
    *out = ctx.release();
    return SEGHDC_OK;
}

void seghdc_destroy(seghdc_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->nccl_comm) nccl_api().comm_destroy(ctx->nccl_comm);
    for (seghdc_ctx* child : ctx->batch) seghdc_destroy(child);
    if (ctx->graph.exec) cudaGraphExecDestroy(ctx->graph.exec);
    for (auto& e : ctx->stage_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->prof_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    delete ctx;
}

const char* seghdc_last_error(const seghdc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_thread_err.c_str(); }

int seghdc_set_sm_budget(seghdc_ctx* ctx, int sms) {
    return guarded(ctx, [&] {
        require(sms >= 0, "SM budget must be >= 0");
        int dev_sms = 0;
        ck(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->device), "attr");
        ctx->sms = (sms == 0 || sms > dev_sms) ? dev_sms : sms;
    });
}

int seghdc_set_stream(seghdc_ctx* ctx, void* stream) {
    return guarded(ctx, [&] {
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        if (stream) {
            ctx->stream = static_cast<cudaStream_t>(stream);
            ctx->own_stream = false;
        } else {
            ck(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
            ctx->own_stream = true;
        }
    });
}

int seghdc_synchronize(seghdc_ctx* ctx) {
    return guarded(ctx, [&] { ck(cudaStreamSynchronize(ctx->stream), "sync"); });
}

uint64_t seghdc_kernel_launches(const seghdc_ctx* ctx) { return ctx ? ctx->launches : 0; }

#ifdef SEGHDC_CHECKED
// checked build only: source line of the first violated device-side index check (0: none),
// then reset
extern "C" int seghdc_debug_check(unsigned int* line_out) {
    return guarded(nullptr, [&] {
        ck(cudaDeviceSynchronize(), "sync");
        unsigned int v = seghdc_dev::check_line_tc();
        if (!v) v = seghdc_dev::check_line_kernels();
        if (!v) v = seghdc_dev::check_line_closed();
        *line_out = v;
    });
}
#endif

int seghdc_set_wrap_counting(seghdc_ctx* ctx, int enable) {
    return guarded(ctx, [&] { ctx->count_wraps = enable != 0; });
}

int seghdc_round_wraps(seghdc_ctx* ctx, uint64_t* out, size_t cap, size_t* rounds_out) {
    return guarded(ctx, [&] {
        require(ctx->count_wraps, "wrap counting is off: enable it with seghdc_set_wrap_counting before the run");
        require(ctx->wraps_src != nullptr, "no clustering run on this context yet");
        size_t rounds = ctx->wraps_rounds;
        const bool packed = ctx->K && ctx->state.p && ctx->wraps_src == StateView::at(ctx->state.p, uint32_t(ctx->K)).wraps;
        if (packed) rounds = read_state(*ctx).hdr.rounds_run;  // synchronises
        const size_t nc = std::min(rounds, cap);
        if (nc) ck(cudaMemcpyAsync(out, ctx->wraps_src, nc * 8, cudaMemcpyDeviceToHost, ctx->stream), "download wraps");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        if (rounds_out) *rounds_out = rounds;
    });
}

const char* seghdc_round_kernel(const seghdc_ctx* ctx) {
    if (!ctx || ctx->K == 0) return "";
    return ctx->plan.tc ? "k_round_tc" : ctx->plan.fused ? "k_round_fused" : "k_round";
}

int seghdc_build_codebooks(size_t dim, size_t h, size_t w, size_t c, double alpha, size_t beta, size_t gamma,
                           uint64_t seed, int encoder, uint64_t* row_out, uint64_t* col_out, uint64_t* widened_out) {
    return guarded(nullptr, [&] {
        seghdc_host::validate_position(dim, h, w, alpha, beta);
        seghdc_host::validate_color(dim, c, gamma);
        std::mt19937_64 rng(seed);  // pipeline.cpp:43: one generator, position first, then colour
        seghdc_host::build_position(dim, h, w, alpha, beta, encoder, rng, row_out, col_out);
        seghdc_host::build_color(dim, c, gamma, encoder, rng, widened_out);
    });
}

int seghdc_validate_run(size_t dim, size_t h, size_t w, size_t c, double alpha, size_t beta, size_t gamma, size_t k,
                        size_t iterations) {
    return guarded(nullptr, [&] {  // RunConfig::validate, pipeline.cpp:25-30
        seghdc_host::validate_image(h, w, c);
        seghdc_host::validate_position(dim, h, w, alpha, beta);
        seghdc_host::validate_color(dim, c, gamma);
        seghdc_host::validate_cluster(k, iterations, h * w);
    });
}

int seghdc_encode(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c, size_t dim,
                  const uint64_t* row_words, const uint64_t* col_words, const uint64_t* widened_words,
                  uint64_t* grid_out) {
    return guarded(ctx, [&] {
        load_image(*ctx, pixels, h, w, c);
        load_codebooks(*ctx, dim, h, w, c, row_words, col_words, widened_words);
        encode_rows(*ctx, 0, h);
        if (grid_out) store_grid(*ctx, grid_out);
        ck(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int seghdc_select_seeds(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c, size_t k,
                        uint64_t* seeds_out) {
    return guarded(ctx, [&] {
        load_image(*ctx, pixels, h, w, c);
        require(k >= 1 && k <= h * w, "select_initial_centroids: k = " + std::to_string(k) + " out of range for " +
                                          std::to_string(h * w) + " pixels");
        ctx->K = k;
        ctx->state.ensure(StateView::bytes(uint32_t(k)));
        ctx->seeds.ensure(k);
        ctx->slots.ensure(2 + k);
        ctx->min_dist.ensure(h * w);
        select_seeds_dev(*ctx, k);
        ck(cudaMemcpyAsync(seeds_out, ctx->seeds.p, k * 8, cudaMemcpyDeviceToHost, ctx->stream), "download seeds");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int seghdc_assign(seghdc_ctx* ctx, const uint64_t* grid, size_t h, size_t w, size_t dim, const uint32_t* centroids,
                  size_t k, uint32_t* labels_out) {
    return guarded(ctx, [&] {
        require(k >= 1, "assign_labels: empty centroid set");
        if (grid) load_grid(*ctx, grid, h, w, dim, 0, h);
        require(ctx->g.D == dim && ctx->g_h == h && ctx->g_w == w, "assign_labels: dimension mismatch");
        // caller centroids may hold any u32 (the reference's IntVector): up to 6 planes
        uint32_t zmax = 0;
        for (size_t i = 0; i < k * dim; ++i) zmax = std::max(zmax, centroids[i]);
        ctx->iterations = 1;
        ctx->early_stop = 0;
        alloc_cluster(*ctx, k, std::max<uint64_t>(zmax, 1));
        // caller centroids are arbitrary u32: dot^2 * norm2 <= (D zmax)^2 * D zmax^2 = D^3 zmax^4
        ctx->assign_vmax_wraps = std::log2(double(dim)) * 3 + std::log2(std::max(double(zmax), 1.0)) * 4 >= 127.0;
        ck(cudaMemcpyAsync(ctx->Z.p, centroids, k * dim * 4, cudaMemcpyHostToDevice, ctx->stream), "upload centroids");
        ck(cudaMemsetAsync(ctx->state.p, 0, StateView::bytes(uint32_t(k), 1), ctx->stream), "clear state");
        ctx->wraps_src = StateView::at(ctx->state.p, uint32_t(k)).wraps;
        ck(cudaMemsetAsync(ctx->labels.p, 0xFF, ctx->n_local() * 4, ctx->stream), "clear labels");
        finish(*ctx, 2, 0);  // norm2 + B fragments of the given set (parity 1)
        round_assign(*ctx, 1);
        ck(cudaMemcpyAsync(labels_out, ctx->labels.p, ctx->n_local() * 4, cudaMemcpyDeviceToHost, ctx->stream),
           "download labels");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        ctx->assign_vmax_wraps = false;
    });
}

int seghdc_update(seghdc_ctx* ctx, const uint64_t* grid, size_t h, size_t w, size_t dim, const uint32_t* labels,
                  const uint32_t* prev_centroids, size_t k, uint32_t* centroids_out, uint64_t* counts_out) {
    return guarded(ctx, [&] {
        if (grid) load_grid(*ctx, grid, h, w, dim, 0, h);
        require(ctx->g_h == h && ctx->g_w == w, "update_centroids: mask shape does not match grid");
        require(ctx->g.D == dim, "update_centroids: dimension mismatch");
        for (size_t p = 0; p < h * w; ++p)  // clusterer.cpp:176-179
            if (labels[p] >= k)
                throw Error(SEGHDC_ECONFIG, "update_centroids: label " + std::to_string(labels[p]) +
                                                " out of range for k = " + std::to_string(k));
        alloc_cluster(*ctx, k);
        ck(cudaMemcpyAsync(ctx->labels.p, labels, h * w * 4, cudaMemcpyHostToDevice, ctx->stream), "upload labels");
        ck(cudaMemcpyAsync(ctx->Z.p, prev_centroids, k * dim * 4, cudaMemcpyHostToDevice, ctx->stream), "upload prev");
        ck(cudaMemsetAsync(ctx->state.p, 0, StateView::bytes(uint32_t(k)), ctx->stream), "clear state");
        AccumulateArgs u{};
        u.grid = ctx->grid.p;
        u.S32 = ctx->g.S32;
        u.W32 = ctx->g.W32;
        u.n = ctx->n_local();
        u.labels = ctx->labels.p;
        u.K = uint32_t(k);
        u.skip_mode = -1;
        u.state = ctx->state.p;
        u.parity = 1;
        ck(cudaMemsetAsync(ctx->xchg.p, 0, ctx->xchg_round_ints() * 4, ctx->stream), "clear exchange");
        u.dst = reinterpret_cast<uint32_t*>(ctx->xchg.p);
        u.Dp = ctx->g.Dp;
        u.counts_dst = reinterpret_cast<uint32_t*>(ctx->xchg.p) + k * ctx->g.Dp;
        u.sms = uint32_t(ctx->sms);
        launch_accumulate(u, ctx->stream);
        ctx->count();
        ctx->check_launch();
        finish(*ctx, 3, 1);
        ck(cudaMemcpyAsync(centroids_out, ctx->Z.p, k * dim * 4, cudaMemcpyDeviceToHost, ctx->stream),
           "download centroids");
        const HostState hs = read_state(*ctx);
        for (size_t c = 0; c < k; ++c) counts_out[c] = hs.cur[0][c];
    });
}

int seghdc_cluster(seghdc_ctx* ctx, const uint64_t* grid, const uint8_t* pixels, size_t h, size_t w, size_t c,
                   size_t dim, size_t k, size_t iterations, int early_stop, seghdc_round_cb on_round, void* user,
                   uint32_t* labels_out, uint32_t* centroids_out, uint64_t* counts_out, size_t* rounds_out) {
    return guarded(ctx, [&] {
        seghdc_host::validate_cluster(k, iterations, h * w);  // clusterer.cpp:192 validates first
        load_image(*ctx, pixels, h, w, c);
        if (grid) load_grid(*ctx, grid, h, w, dim, 0, h);
        require(ctx->grid_valid && ctx->g_h == h && ctx->g_w == w && ctx->g.D == dim,
                "cluster: grid shape does not match image");
        cluster_full(*ctx, k, iterations, early_stop, on_round, user);
        fetch(*ctx, labels_out, centroids_out, counts_out, rounds_out);
    });
}

int seghdc_run_pipeline(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c, size_t dim, double alpha,
                        size_t beta, size_t gamma, size_t k, size_t iterations, uint64_t seed, int encoder,
                        int early_stop, seghdc_round_cb on_round, void* user, uint32_t* labels_out, size_t* rounds_out,
                        double* timings) {
    return guarded(ctx, [&] {
        PipelineCall pc{pixels, h, w, c, dim, alpha, beta, gamma, k, iterations, seed, encoder, early_stop};
        run_pipeline_impl(*ctx, pc, on_round, user, labels_out, nullptr, nullptr, rounds_out, timings, false);
    });
}

int seghdc_run_pipeline_batch(seghdc_ctx* ctx, const uint8_t* const* pixels, size_t n_images, size_t h, size_t w,
                              size_t c, size_t dim, double alpha, size_t beta, size_t gamma, size_t k, size_t iterations,
                              uint64_t seed, int encoder, int early_stop, uint32_t* const* labels_out,
                              size_t* rounds_out) {
    return guarded(ctx, [&] {
        PipelineCall pc{nullptr, h, w, c, dim, alpha, beta, gamma, k, iterations, seed, encoder, early_stop};
        run_pipeline_batch(*ctx, pixels, n_images, pc, labels_out, rounds_out);
    });
}

int seghdc_nccl_get_unique_id(void* id_out) {
    return guarded(nullptr, [&] {
        require(id_out != nullptr, "nccl_get_unique_id: null output");
        nck(nccl_api().get_unique_id(static_cast<ncclUniqueId*>(id_out)), "ncclGetUniqueId");
    });
}

int seghdc_nccl_init(seghdc_ctx* ctx, const void* unique_id, int rank, int nranks) {
    return guarded(ctx, [&] {
        require(unique_id != nullptr, "nccl_init: null unique id");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "nccl_init: rank out of range");
        if (ctx->nccl_comm) {
            nccl_api().comm_destroy(ctx->nccl_comm);
            ctx->nccl_comm = nullptr;
        }
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof(id));
        nck(nccl_api().comm_init_rank(&ctx->nccl_comm, nranks, id, rank), "ncclCommInitRank");
        ctx->rank = rank;
        ctx->nranks = nranks;
        ctx->ar_fn = nullptr;
        ctx->ar_user = nullptr;
    });
}

int seghdc_set_allreduce(seghdc_ctx* ctx, seghdc_allreduce_fn fn, void* user, int rank, int nranks) {
    return guarded(ctx, [&] {
        require(nranks >= 1 && rank >= 0 && rank < nranks, "set_allreduce: rank out of range");
        if (ctx->nccl_comm) {
            nccl_api().comm_destroy(ctx->nccl_comm);
            ctx->nccl_comm = nullptr;
        }
        ctx->ar_fn = fn;
        ctx->ar_user = user;
        ctx->rank = rank;
        ctx->nranks = nranks;
    });
}

int seghdc_shard_rows(size_t h, int rank, int nranks, size_t* row_begin, size_t* row_end) {
    return guarded(nullptr, [&] { shard_rows(h, rank, nranks, *row_begin, *row_end); });
}

int seghdc_shard_row_range(const seghdc_ctx* ctx, size_t h, size_t* row_begin, size_t* row_end) {
    return guarded(nullptr, [&] {
        require(ctx != nullptr, "shard_row_range: null context");
        shard_rows(h, ctx->rank, ctx->nranks, *row_begin, *row_end);
    });
}

int seghdc_cluster_sharded_async(seghdc_ctx* ctx, size_t k, size_t iterations, int early_stop) {
    return guarded(ctx, [&] { cluster_sharded(*ctx, k, iterations, early_stop); });
}

int seghdc_run_pipeline_sharded(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c, size_t dim,
                                double alpha, size_t beta, size_t gamma, size_t k, size_t iterations, uint64_t seed,
                                int encoder, int early_stop, uint32_t* labels_out, uint32_t* centroids_out,
                                uint64_t* counts_out, size_t* rounds_out, double* timings_ms_out) {
    return guarded(ctx, [&] {
        PipelineCall pc{pixels, h, w, c, dim, alpha, beta, gamma, k, iterations, seed, encoder, early_stop};
        run_pipeline_impl(*ctx, pc, nullptr, nullptr, labels_out, centroids_out, counts_out, rounds_out, timings_ms_out,
                          true);
    });
}

int seghdc_run_pipeline_closed(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c, size_t dim,
                               double alpha, size_t beta, size_t gamma, size_t k, size_t iterations, uint64_t seed,
                               int early_stop, uint32_t* labels_out, uint32_t* centroids_out, uint64_t* counts_out,
                               size_t* rounds_out) {
    return guarded(ctx, [&] {
        // RunConfig::validate before any work (pipeline.cpp:25-30, 42)
        seghdc_host::validate_image(h, w, c);
        seghdc_host::validate_position(dim, h, w, alpha, beta);
        seghdc_host::validate_color(dim, c, gamma);
        seghdc_host::validate_cluster(k, iterations, h * w);
        require(k <= 32, "closed-form variant: k = " + std::to_string(k) + " > 32");
        const size_t wph = (dim + 63) / 64;
        std::mt19937_64 rng(seed);  // pipeline.cpp:43-59, Manhattan codebooks only
        std::vector<uint64_t> bases((2 + c) * wph);
        const auto mp = seghdc_host::manhattan_bases(dim, h, w, c, alpha, beta, gamma, rng, bases.data());
        std::vector<uint8_t> bflag(dim);  // B = XOR of the bases: every run empty (row 0, col 0, value 0)
        for (size_t i = 0; i < dim; ++i) {
            uint64_t x = 0;
            for (size_t b = 0; b < 2 + c; ++b) x ^= bases[b * wph + (i >> 6)];
            bflag[i] = uint8_t((x >> (i & 63)) & 1);
        }
        load_image(*ctx, pixels, h, w, c);
        ctx->K = k;  // select_initial_centroids on the device, as seghdc_select_seeds
        ctx->state.ensure(StateView::bytes(uint32_t(k)));
        ctx->seeds.ensure(k);
        ctx->slots.ensure(2 + k);
        ctx->min_dist.ensure(h * w);
        select_seeds_dev(*ctx, k);

        const size_t n = h * w, stride = dim + 1;
        // per-position member counts (diff, diffc) are int32
        require(n < (size_t(1) << 31), "closed-form variant: 2^31 pixels or more");
        auto& Q = ctx->cf.Q;
        auto &P = ctx->cf.P, &n2 = ctx->cf.n2, &cnt = ctx->cf.cnt, &counts = ctx->cf.counts, &changed = ctx->cf.changed;
        auto &Z = ctx->cf.Z, &labels = ctx->cf.labels;
        auto& diff = ctx->cf.diff;
        auto& bf = ctx->cf.bf;
        Q.ensure(k * stride);
        P.ensure(k);
        n2.ensure(k);
        cnt.ensure(k);
        counts.ensure(k);
        changed.ensure(1);
        Z.ensure(k * dim);
        labels.ensure(n);
        diff.ensure(k * stride);
        bf.ensure(dim);
        ck(cudaMemcpyAsync(bf.p, bflag.data(), dim, cudaMemcpyHostToDevice, ctx->stream), "upload B");
        ck(cudaMemsetAsync(diff.p, 0, k * stride * 4, ctx->stream), "clear diff");
        ck(cudaMemsetAsync(cnt.p, 0, k * 8, ctx->stream), "clear counts");
        ck(cudaMemsetAsync(labels.p, 0xFF, n * 4, ctx->stream), "clear labels");
        ClosedArgs a{};
        a.img = ctx->img.p;
        a.n = n;
        a.w = uint32_t(w);
        a.c = uint32_t(c);
        a.dim = uint32_t(dim);
        a.beta = mp.beta;
        a.x_row = mp.x_row;
        a.x_col = mp.x_col;
        a.K = uint32_t(k);
        for (int i = 0; i < 3; ++i) a.off[i] = mp.off[i], a.unit[i] = mp.unit[i];
        a.nr = uint32_t((h - 1) / beta + 1);
        a.nc = uint32_t((w - 1) / beta + 1);
        a.L = a.nr + a.nc + 256 * uint32_t(c) + 1;
        // compressed endpoint indices when they fit (keys pos << 15 | index, [K][L] tables in smem)
        const bool compressed = a.L < (1u << 15) && dim < (1u << 17) && size_t(a.L) * k * 8 <= (160u << 10) &&
                                !getenv("SEGHDC_CLOSED_POSITIONS");
        // the position-table accumulate keeps one [dim + 1] int32 difference row per cluster
        // group in shared memory (k_closed_accumulate, at least one cluster per group)
        require(compressed || (dim + 1) * 4 + 4 <= ctx->smem_optin,
                "closed-form variant: dim = " + std::to_string(dim) +
                    " needs the position tables, whose difference row exceeds shared memory");
        auto& diffc = ctx->cf.diffc;
        if (compressed) {
            diffc.ensure(k * a.L);
            ck(cudaMemsetAsync(diffc.p, 0, k * a.L * 4, ctx->stream), "clear diffc");
        }
        ClosedState st{Q.p, P.p, n2.p, Z.p, diff.p, cnt.p, counts.p, bf.p, labels.p, changed.p,
                       compressed ? diffc.p : nullptr, nullptr};
        ctx->wraps_hist.ensure(iterations + 1);
        ck(cudaMemsetAsync(ctx->wraps_hist.p, 0, (iterations + 1) * 8, ctx->stream), "clear wraps");
        launch_closed_seed(a, ctx->seeds.p, st, ctx->stream);
        launch_closed_finish(a, st, ctx->stream);
        ctx->count(2);
        ctx->check_launch();
        size_t rounds = 0;
        for (size_t r = 1; r <= iterations; ++r) {  // clusterer.cpp:208-216
            ck(cudaMemsetAsync(changed.p, 0, 8, ctx->stream), "clear changed");
            st.wraps = ctx->count_wraps ? ctx->wraps_hist.p + (r - 1) : nullptr;  // opt-in counting
            launch_closed_assign(a, st, ctx->sms, ctx->stream);
            ctx->count();
            ctx->check_launch();
            rounds = r;
            if (early_stop && r > 1) {
                unsigned long long ch = 0;
                ck(cudaMemcpyAsync(&ch, changed.p, 8, cudaMemcpyDeviceToHost, ctx->stream), "download changed");
                ck(cudaStreamSynchronize(ctx->stream), "sync");
                if (ch == 0) break;
            }
            if (r < iterations) {
                launch_closed_accumulate(a, st, ctx->sms, ctx->stream);
                launch_closed_finish(a, st, ctx->stream);
                ctx->count(2);
                ctx->check_launch();
            }
        }
        ck(cudaMemcpyAsync(labels_out, labels.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream), "download labels");
        if (centroids_out)
            ck(cudaMemcpyAsync(centroids_out, Z.p, k * dim * 4, cudaMemcpyDeviceToHost, ctx->stream), "download Z");
        if (counts_out)
            ck(cudaMemcpyAsync(counts_out, counts.p, k * 8, cudaMemcpyDeviceToHost, ctx->stream), "download counts");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        if (rounds_out) *rounds_out = rounds;
        ctx->wraps_src = ctx->wraps_hist.p;
        ctx->wraps_rounds = rounds;
    });
}

int seghdc_load_image(seghdc_ctx* ctx, const uint8_t* pixels, size_t h, size_t w, size_t c) {
    return guarded(ctx, [&] { load_image(*ctx, pixels, h, w, c); });
}

int seghdc_load_codebooks(seghdc_ctx* ctx, size_t dim, const uint64_t* row, const uint64_t* col,
                          const uint64_t* wid) {
    return guarded(ctx, [&] {
        require(ctx->h > 0, "load the image before its codebooks");
        load_codebooks(*ctx, dim, ctx->h, ctx->w, ctx->c, row, col, wid);
    });
}

int seghdc_encode_async(seghdc_ctx* ctx, size_t row_begin, size_t row_end) {
    return guarded(ctx, [&] { encode_rows(*ctx, row_begin, row_end); });
}

int seghdc_load_grid(seghdc_ctx* ctx, const uint64_t* grid, size_t h, size_t w, size_t dim, size_t row_begin,
                     size_t row_end) {
    return guarded(ctx, [&] { load_grid(*ctx, grid, h, w, dim, row_begin, row_end); });
}

int seghdc_store_grid(seghdc_ctx* ctx, uint64_t* grid_out) {
    return guarded(ctx, [&] { store_grid(*ctx, grid_out); });
}

int seghdc_cluster_async(seghdc_ctx* ctx, size_t k, size_t iterations, int early_stop) {
    return guarded(ctx, [&] { cluster_full(*ctx, k, iterations, early_stop, nullptr, nullptr); });
}

int seghdc_fetch_results(seghdc_ctx* ctx, uint32_t* labels_out, uint32_t* centroids_out, uint64_t* counts_out,
                         size_t* rounds_out) {
    return guarded(ctx, [&] { fetch(*ctx, labels_out, centroids_out, counts_out, rounds_out); });
}

int seghdc_shard_begin(seghdc_ctx* ctx, size_t k, size_t iterations, int early_stop) {
    return guarded(ctx, [&] { cluster_begin(*ctx, k, iterations, early_stop); });
}

int seghdc_exchange_buffer(seghdc_ctx* ctx, void** device_ptr, size_t* n_int32) {
    return guarded(ctx, [&] {
        require(ctx->xchg.p != nullptr, "no clustering in progress");
        *device_ptr = ctx->xchg.p;
        *n_int32 = ctx->xchg_round_ints() + (ctx->exchange_phase == 1 ? ctx->g.Dp : 0);
    });
}

int seghdc_exchange_download(seghdc_ctx* ctx, int32_t* host) {
    return guarded(ctx, [&] {
        void* p;
        size_t n;
        if (seghdc_exchange_buffer(ctx, &p, &n) != SEGHDC_OK) throw Error(SEGHDC_ECONFIG, ctx->err);
        ck(cudaMemcpyAsync(host, p, n * 4, cudaMemcpyDeviceToHost, ctx->stream), "download exchange");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int seghdc_exchange_upload(seghdc_ctx* ctx, const int32_t* host) {
    return guarded(ctx, [&] {
        void* p;
        size_t n;
        if (seghdc_exchange_buffer(ctx, &p, &n) != SEGHDC_OK) throw Error(SEGHDC_ECONFIG, ctx->err);
        ck(cudaMemcpyAsync(p, host, n * 4, cudaMemcpyHostToDevice, ctx->stream), "upload exchange");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int seghdc_shard_init_finish(seghdc_ctx* ctx) {
    return guarded(ctx, [&] { init_finish(*ctx); });
}

int seghdc_shard_assign(seghdc_ctx* ctx, size_t round) {
    return guarded(ctx, [&] {
        require(round >= 1 && round <= ctx->iterations, "round out of range");
        round_assign(*ctx, uint32_t(round));

    });
}

int seghdc_shard_round_needs_exchange(const seghdc_ctx* ctx, size_t round) {
    return ctx && round >= 1 && round < ctx->iterations ? 1 : 0;
}

int seghdc_shard_finish(seghdc_ctx* ctx, size_t round) {
    return guarded(ctx, [&] { finish(*ctx, 0, uint32_t(round)); });
}

int seghdc_profile_rounds(seghdc_ctx* ctx, int enable) {
    return guarded(ctx, [&] {
        ctx->profiling = enable != 0;
        ctx->prof_used = 0;
    });
}

int seghdc_profile_read(seghdc_ctx* ctx, double* total_ms, uint64_t* count) {
    return seghdc_profile_read_each(ctx, total_ms, count, nullptr, 0);
}

int seghdc_profile_read_each(seghdc_ctx* ctx, double* total_ms, uint64_t* count, double* each_ms, size_t cap) {
    return guarded(ctx, [&] {
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        double t = 0;
        for (size_t i = 0; i < ctx->prof_used; ++i) {
            float ms = 0;
            ck(cudaEventElapsedTime(&ms, ctx->prof_events[i].first, ctx->prof_events[i].second), "elapsed");
            t += ms;
            if (each_ms && i < cap) each_ms[i] = ms;
        }
        *total_ms = t;
        *count = ctx->prof_used;
        ctx->prof_used = 0;
    });
}

int seghdc_pinned_alloc(size_t bytes, void** out) {
    return guarded(nullptr, [&] {
        require(out != nullptr, "pinned_alloc: null output pointer");
        ck(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable), "cudaHostAlloc");
    });
}

int seghdc_pinned_free(void* p) {
    return guarded(nullptr, [&] { ck(cudaFreeHost(p), "cudaFreeHost"); });
}

}  // extern "C"

#ifdef SEGHDC_TRACE
namespace seghdc_dev {
void read_trace(void* dst);
}
// diagnostic build only: 148 x 64 x 8 u64 clock64() stamps of the fused round kernel
extern "C" void seghdc_debug_trace(void* dst) { seghdc_dev::read_trace(dst); }
namespace seghdc_dev {
void read_trace_tc(void* dst);
}
extern "C" void seghdc_debug_trace_tc(void* dst) { seghdc_dev::read_trace_tc(dst); }
#endif

#ifdef SEGHDC_HANGDBG
namespace seghdc_dev {
void* setup_hang();
}
// diagnostic build only: host-mapped log of timed-out barrier waits of the tcgen05 kernel
extern "C" void* seghdc_debug_hang_setup() { return seghdc_dev::setup_hang(); }
#endif
