// C-ABI layer (include/psplat_b200.h): device-resident state, batching, CUB
// scan for the tile CSR, NCCL gradient all-reduce. Host code only orchestrates;
// every per-plane / per-pixel operation runs in the kernels of psg_binning.cu and
// psg_raster.cu. There is no CPU fallback: every call fails with PSG_ECUDA when
// no device is usable.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is bound lazily with dlopen (see nccl_api())
#include <nvtx3/nvToolsExt.h>  // header-only; the ranges cost a pointer test without a tool attached

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/psplat_b200.h"
#include "psg_internal.h"

namespace {
// NVTX range for the tools (nsys / ncu --nvtx): one per API entry point and step phase
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};
}  // namespace

using namespace psg;

namespace {

thread_local std::string g_err;

// pixel rects are short4 and packed into 16-bit halves of the scan records
constexpr int kMaxSide = 32767;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define PSG_CUDA(expr)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(PSG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));     \
    } while (0)

template <typename T>
int grow(T*& p, size_t& cap, size_t need) {
    if (need <= cap && p) return PSG_OK;
    size_t nc = std::max<size_t>(need, cap + cap / 2);
    nc = std::max<size_t>(nc, 256);
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    PSG_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), nc * sizeof(T)));
    cap = nc;
    return PSG_OK;
}

// NCCL is resolved at first use, preferring an already-loaded libnccl.so.2 (the
// one torch.distributed brought in), so the library never forces a second NCCL
// build into a process.
struct NcclApi {
    bool ok = false;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy && a.error_string;
        return a;
    }();
    return api;
}

}  // namespace

struct psg_context {
    // calls on one context from several host threads are serialised (each entry
    // point holds it for its host-side duration; launches stay asynchronous)
    std::recursive_mutex mu;
    int device = 0;
    int precision = PSG_FP32;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // H2D of streamed targets (psg_step_host)
    psg::AuxStream aux;                  // crowded-tile launch, overlapped with the rest
    psg_render_config cfg{};

    // planes
    int64_t P = 0;
    std::vector<int64_t> ids;
    double* d_center = nullptr;
    double* d_rot = nullptr;
    double* d_radii = nullptr;
    size_t plane_cap = 0, plane_cap_r = 0, plane_cap_q = 0;
    PlaneGeo* d_geo = nullptr;
    size_t geo_cap = 0;
    PlaneF* d_geof = nullptr;
    size_t geof_cap = 0;
    double* d_grads = nullptr;  // P*11 + 2: gradients, the step loss, the step-window guard count
    size_t grads_cap = 0;

    // registered views
    std::vector<ViewDev> h_views;
    ViewDev* d_views = nullptr;
    size_t views_cap = 0;
    float* d_td = nullptr;
    float* d_tn = nullptr;
    size_t td_cap = 0, tn_cap = 0;
    long long total_px = 0;

    // batch scratch. The vid[n] + tile_base[n+1] uploads go through a ring of pinned
    // buffers, each reused only after its copy's event completed (no step sync).
    static constexpr int kStage = 4;
    int* h_ring[kStage] = {};
    size_t ring_cap[kStage] = {};
    cudaEvent_t ring_ev[kStage] = {};
    int ring_i = 0;
    int* d_vid = nullptr;
    size_t vid_cap = 0;
    int* d_counts = nullptr;
    int* d_offsets = nullptr;
    int* d_cursor = nullptr;
    size_t counts_cap = 0, offsets_cap = 0, cursor_cap = 0;
    int* d_items = nullptr;
    size_t items_cap = 0;
    short4* d_rects = nullptr;
    size_t rects_cap = 0;
    int2* d_big = nullptr;
    size_t big_cap = 0;
    unsigned char* d_recs = nullptr;  // prebuilt record blocks of the resident tiles
    size_t recs_cap = 0;
    psg::TileDesc* d_desc = nullptr;  // per work item (block offset / 16, n)
    size_t desc_cap = 0;
    long long* d_units = nullptr;  // [T+1] record units per tile, then its exclusive scan
    size_t units_cap = 0;
    int* d_pair_tile = nullptr;  // [pairs] tile of each bin entry
    size_t pair_tile_cap = 0;
    int* d_tile_slot = nullptr;  // [T] slot of each batch tile
    size_t tile_slot_cap = 0;
    void* d_cub = nullptr;
    size_t cub_cap = 0;
    double* d_view_loss = nullptr;
    size_t view_loss_cap = 0;
    // [0] first_bad, [1..2] loss counts, [3] crowded-tile counter, [4] n_big, [5] work counter, [6] checksum,
    // [7] step abort flag, [8] 64-bit bin-entry total, [9..10] sizes an aborted step needs
    unsigned long long* d_misc = nullptr;
    Stats* d_stats = nullptr;
    int64_t* h_total = nullptr;  // pinned

    // single-view scratch (drop-in API)
    ViewDev* d_view1 = nullptr;
    double* d_maps = nullptr;
    size_t maps_cap = 0;
    int* d_rec_prim = nullptr;
    size_t rec_prim_cap = 0;
    unsigned short* d_rec_count = nullptr;
    size_t rec_count_cap = 0;
    float* d_t1 = nullptr;
    size_t t1_cap = 0;
    double* d_sums = nullptr;
    double* d_g1 = nullptr;
    size_t g1_cap = 0;

    // fused-step map outputs
    float* d_smaps = nullptr;
    size_t smaps_cap = 0;
    long long smaps_stride = 0;

    // last step
    std::vector<int> last_vids;
    double last_view_scale = 1.0;
    psg_stats stats{};

    // NCCL
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;

    // device optimiser state (OptimState, optimizer.hpp:63-70), valid after the
    // first psg_optim_* call on the current plane set
    bool optim_ready = false;
    double* d_m = nullptr;
    double* d_v = nullptr;
    long long* d_step = nullptr;
    double* d_rgs = nullptr;
    long long* d_rgc = nullptr;
    double* d_pow = nullptr;  // [2 * pow_len]: pow(beta1, s) then pow(beta2, s)
    int64_t pow_len = 0;
    double pow_b1 = 0.0, pow_b2 = 0.0;
    int64_t max_step = 0;  // upper bound of the per-primitive Adam step counters
    int64_t iteration = 0;
    int64_t next_id = 0;
    int* d_split = nullptr;  // axis[P], cnt[P], pos[P]
    size_t split_cap = 0;
    std::vector<int64_t> epoch_order;
    int64_t epoch_cached = -1;
    uint64_t epoch_seed = 0;

    // optional per-launch timing of the rasteriser
    bool timing = false;
    bool targets_tma = false;  // every view width % 4 == 0: target rows are TMA-copyable
    // deterministic mode: per-(bin entry, warp) gradient and
    // per-(tile, warp) loss partials, reduced in a fixed order after the launch
    bool deterministic = false;
    double* d_det = nullptr;
    size_t det_cap = 0;
    int* d_det_sort = nullptr;  // pid keys out, pair values in, pair values out
    size_t det_sort_cap = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;

    // Step window. psg_step never synchronises: bins and record blocks use the
    // capacities earlier steps needed, and k_bin_guard aborts a step that does not
    // fit (counted in the gradient buffer's guard slot, so an all-reduce carries it
    // to every rank). The next call that reads results (finalize, read_grads, ...)
    // checks the guard once; after an abort it restores the gradients and
    // statistics of the window start and replays the window's steps with exact
    // sizes, splitting a view group whose bin entries exceed pair_limit.
    struct Pending {
        std::vector<int> vids;  // this pass: slots [slot0, slot0 + |vids|) of its step
        double lambda, view_scale;
        int flags, slot0;
        std::vector<int> outs;  // the whole step's views on its first pass (output sizing)
    };
    std::vector<Pending> pending;
    bool window_open = false;
    bool window_allreduced = false;
    double* d_snap = nullptr;  // d_grads (P*11 + 2) at the window start
    size_t snap_cap = 0;
    Stats* d_stats_snap = nullptr;
    psg_stats host_stats_snap{};
    long long pair_limit = 2147483647LL;  // int32 CSR offsets; psg_set_pair_limit lowers it (tests)
    int smaps_n = 0;                      // views the map buffers of the last step hold
    bool host_inv_stale = false;          // streamed targets: 1/count normalisers only on the device
    unsigned long long* d_cnt = nullptr;  // per-view target counts of streamed targets
    size_t cnt_cap = 0;
    double* d_runlog = nullptr;  // deferred Optimizer::run: losses of the issued block
    size_t runlog_cap = 0;
    // drop-in calls: pinned staging for the host buffers, live-record packing
    unsigned char* h_big = nullptr;
    size_t h_big_cap = 0;
    const unsigned long long* run_halt = nullptr;  // set while a deferred run queues a block
    int* d_pack = nullptr;  // live records, pixel-major
    size_t pack_cap = 0;
    long long* d_pack_off = nullptr;  // [np + 1] exclusive scan of the record counts
    size_t pack_off_cap = 0;
};

namespace {

int settle(psg_context* ctx);

void default_cfg(psg_render_config* c) {  // renderer.hpp:10-21
    c->max_records = 30;
    c->normalize_by_alpha = 0;
    c->tile_size = 16;
    c->threads = 0;
    c->weight_floor = 1e-4;
    c->t_near = 0.01;
    c->parallel_eps = 1e-8;
    c->alpha_floor = 0.05;
    c->alpha1 = 5.0;
    c->alpha2 = 1.0;
}

// Host-side view record; ray basis in the exact order of ray_basis()
// (renderer.cpp:32-38): base = rot_wc * ((0.5-cx)/fx, (0.5-cy)/fy, 1) with the
// stored-Matrix3d row order a0 + (a1 + a2); du = col0/fx; dv = col1/fy.
ViewDev make_view(const psg_camera& c, long long pix_off) {
    ViewDev v{};
    v.fx = c.fx;
    v.fy = c.fy;
    v.cx = c.cx;
    v.cy = c.cy;
    for (int i = 0; i < 9; ++i) v.R[i] = c.rot_wc[i];
    for (int i = 0; i < 3; ++i) v.t[i] = c.t_wc[i];
    const double a = (0.5 - c.cx) / c.fx, b = (0.5 - c.cy) / c.fy, d = 1.0;
    for (int r = 0; r < 3; ++r) {
        volatile double p0 = c.rot_wc[3 * r] * a;  // volatile: keep every rounding step
        volatile double p1 = c.rot_wc[3 * r + 1] * b;
        volatile double p2 = c.rot_wc[3 * r + 2] * d;
        volatile double s12 = p1 + p2;
        v.base[r] = p0 + s12;
        v.du[r] = c.rot_wc[3 * r] / c.fx;
        v.dv[r] = c.rot_wc[3 * r + 1] / c.fy;
    }
    v.W = c.width;
    v.H = c.height;
    v.tiles_x = (c.width + kTile - 1) / kTile;
    v.tiles_y = (c.height + kTile - 1) / kTile;
    v.pix_off = pix_off;
    return v;
}

RenderParams make_params(const psg_render_config& c, double lambda, double view_scale) {
    RenderParams rp{};
    rp.lambda = lambda;
    // splat_cut_margin(lambda, floor) * 1.05 (splatting.hpp:48-51, renderer.cpp:122)
    rp.cut = std::log(2.0 / c.weight_floor - 1.0) / (5.0 * lambda) * 1.05;
    rp.arg_cut = std::log(2.0 / c.weight_floor - 1.0);  // renderer.cpp:248
    rp.weight_floor = c.weight_floor;
    rp.t_near = c.t_near;
    rp.parallel_eps = c.parallel_eps;
    rp.alpha_floor = c.alpha_floor;
    rp.alpha1 = c.alpha1;
    rp.alpha2 = c.alpha2;
    rp.view_scale = view_scale;
    rp.max_records = c.max_records;
    rp.normalize_by_alpha = c.normalize_by_alpha;
    return rp;
}

int check_ctx(psg_context* ctx) {
    if (!ctx) return fail(PSG_EINVAL, "null context");
    PSG_CUDA(cudaSetDevice(ctx->device));
    return PSG_OK;
}

int check_cfg(const psg_render_config& c) {
    if (c.max_records > kMaxRecordCap)  // renderer.cpp:234-235
        return fail(PSG_EINVAL, "render_view: max_records above compile-time cap");
    if (c.max_records < 1) return fail(PSG_EINVAL, "render_view: max_records must be >= 1");
    if (c.tile_size != kTile) return fail(PSG_EINVAL, "tile_size must be 16 on the device");
    if (!(c.weight_floor > 0.0 && c.weight_floor < 2.0))
        return fail(PSG_EINVAL, "weight_floor must be in (0, 2)");
    return PSG_OK;
}

// Bin the batch described by (vids, views): rect/count, scan, scatter.
// sync: read the bin-entry total, record units and crowded tiles back and size
// every buffer exactly (the drop-in calls, deterministic mode, replays); returns
// kSplit when the entries exceed the context's pair limit. async: no host sync;
// the buffers keep the capacity earlier steps needed and k_bin_guard aborts the
// step on the device when they do not fit (replayed by settle()).
constexpr int kSplit = -100;
constexpr unsigned long long kNoLimit = ~0ull >> 1;

int bin_batch(psg_context* ctx, const ViewDev* d_views, const std::vector<ViewDev>& hv,
              const std::vector<int>& vids, double cut, Batch& batch, Bins& bins, bool sync,
              int64_t* total) {
    Nvtx nvtx_range("psg.bin");
    const int n = int(vids.size());
    cudaStream_t s = ctx->stream;
    const size_t need = size_t(2 * n + 1);
    // staging slot: reused once its previous upload has completed
    const int ri = ctx->ring_i++ % psg_context::kStage;
    if (ctx->ring_ev[ri]) PSG_CUDA(cudaEventSynchronize(ctx->ring_ev[ri]));
    else PSG_CUDA(cudaEventCreateWithFlags(&ctx->ring_ev[ri], cudaEventDisableTiming));
    if (need > ctx->ring_cap[ri]) {
        if (ctx->h_ring[ri]) cudaFreeHost(ctx->h_ring[ri]);
        ctx->h_ring[ri] = nullptr;
        ctx->ring_cap[ri] = 0;
        PSG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_ring[ri]), need * 2 * sizeof(int),
                               cudaHostAllocDefault));
        ctx->ring_cap[ri] = need * 2;
    }
    int* hvid = ctx->h_ring[ri];
    int* htb = hvid + n;
    int T = 0, max_tiles = 0;
    for (int k = 0; k < n; ++k) {
        const ViewDev& v = hv[size_t(vids[k])];
        hvid[k] = vids[k];
        htb[k] = T;
        T += v.tiles_x * v.tiles_y;
        max_tiles = std::max(max_tiles, v.tiles_x * v.tiles_y);
    }
    htb[n] = T;
    int rc;
    if ((rc = grow(ctx->d_vid, ctx->vid_cap, need))) return rc;
    PSG_CUDA(cudaMemcpyAsync(ctx->d_vid, hvid, need * sizeof(int), cudaMemcpyHostToDevice, s));
    PSG_CUDA(cudaEventRecord(ctx->ring_ev[ri], s));
    if ((rc = grow(ctx->d_counts, ctx->counts_cap, size_t(T) + 1))) return rc;
    if ((rc = grow(ctx->d_offsets, ctx->offsets_cap, size_t(T) + 1))) return rc;
    if ((rc = grow(ctx->d_cursor, ctx->cursor_cap, size_t(T) + 1))) return rc;
    if ((rc = grow(ctx->d_rects, ctx->rects_cap, size_t(n) * size_t(std::max<int64_t>(ctx->P, 1)))))
        return rc;
    batch.views = d_views;
    batch.vid = ctx->d_vid;
    batch.tile_base = ctx->d_vid + n;
    batch.n = n;
    batch.max_tiles = max_tiles;
    bins.counts = ctx->d_counts;
    bins.offsets = ctx->d_offsets;
    bins.cursor = ctx->d_cursor;
    bins.rects = ctx->d_rects;
    if ((rc = grow(ctx->d_big, ctx->big_cap, size_t(T) + 1))) return rc;
    bins.big = ctx->d_big;
    bins.n_big_dev = reinterpret_cast<int*>(ctx->d_misc + 4);
    bins.n_heavy_dev = reinterpret_cast<int*>(ctx->d_misc + 14);
    bins.n_light_dev = reinterpret_cast<int*>(ctx->d_misc + 15);
    bins.halt = ctx->run_halt;
    bins.big_cap = int(ctx->big_cap);
    bins.work_ctr = reinterpret_cast<int*>(ctx->d_misc + 5);
    bins.big_ctr = reinterpret_cast<int*>(ctx->d_misc + 3);
    bins.abort = reinterpret_cast<int*>(ctx->d_misc + 7);
    bins.pairs64 = ctx->d_misc + 8;
    bins.pair_px = &ctx->d_stats->pair_px;
    bins.T = T;
    if ((rc = grow(ctx->d_units, ctx->units_cap, 2 * (size_t(T) + 1)))) return rc;
    bins.units = ctx->d_units;
    bins.unit_off = ctx->d_units + (size_t(T) + 1);
    if ((rc = grow(ctx->d_tile_slot, ctx->tile_slot_cap, size_t(T) + 1))) return rc;
    bins.tile_slot = ctx->d_tile_slot;
    if ((rc = grow(ctx->d_desc, ctx->desc_cap, size_t(n) * size_t(max_tiles) + 1))) return rc;
    bins.desc = ctx->d_desc;
    PSG_CUDA(cudaMemsetAsync(bins.n_big_dev, 0, sizeof(int), s));
    PSG_CUDA(cudaMemsetAsync(ctx->d_misc + 14, 0, 2 * sizeof(unsigned long long), s));  // heavy, light
    PSG_CUDA(cudaMemsetAsync(bins.pairs64, 0, sizeof(unsigned long long), s));
    PSG_CUDA(cudaMemsetAsync(ctx->d_counts, 0, (size_t(T) + 1) * sizeof(int), s));
    // view-independent plane geometry from the resident parameters, every pass:
    // the optimiser moves the planes between steps (make_prim_views, renderer.cpp:40-58)
    launch_plane_setup(ctx->d_center, ctx->d_rot, ctx->d_radii, ctx->P, ctx->d_geo, ctx->d_geof, s);
    launch_rect_count(batch, ctx->d_geo, ctx->P, cut, bins, s);
    launch_big_tiles(batch, bins, kResCapTiles, s);
    size_t tmp = 0, tmp2 = 0;
    PSG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, ctx->d_counts, ctx->d_offsets, T + 1, s));
    PSG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, bins.units, bins.unit_off, T + 1, s));
    tmp = std::max(tmp, tmp2);
    if (tmp > ctx->cub_cap) {
        if (ctx->d_cub) cudaFree(ctx->d_cub);
        ctx->d_cub = nullptr;
        ctx->cub_cap = 0;
        PSG_CUDA(cudaMalloc(&ctx->d_cub, tmp));
        ctx->cub_cap = tmp;
    }
    tmp = ctx->cub_cap;
    PSG_CUDA(cub::DeviceScan::ExclusiveSum(ctx->d_cub, tmp, ctx->d_counts, ctx->d_offsets, T + 1, s));
    tmp = ctx->cub_cap;
    PSG_CUDA(cub::DeviceScan::ExclusiveSum(ctx->d_cub, tmp, bins.units, bins.unit_off, T + 1, s));
    if (sync) {
        // pairs64, units, n_big -> pinned h_total[0..2]
        PSG_CUDA(cudaMemcpyAsync(ctx->h_total, bins.pairs64, 8, cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->h_total + 1, bins.unit_off + T, 8, cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->h_total + 2, bins.n_big_dev, 4, cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaStreamSynchronize(s));
        const int64_t pairs = ctx->h_total[0], units = ctx->h_total[1];
        int32_t h_big = 0;
        std::memcpy(&h_big, ctx->h_total + 2, 4);
        if (pairs > ctx->pair_limit) {
            *total = pairs;
            return kSplit;
        }
        // a quarter of headroom: the next steps' view sets bin a little more or less
        // (each overflow of an asynchronous step costs a host round trip and a
        // reallocation)
        if ((rc = grow(ctx->d_items, ctx->items_cap, size_t(pairs) + size_t(pairs) / 4 + 1))) return rc;
        if ((rc = grow(ctx->d_pair_tile, ctx->pair_tile_cap, size_t(pairs) + size_t(pairs) / 4 + 1))) return rc;
        if ((rc = grow(ctx->d_recs, ctx->recs_cap, 16 * (size_t(units) + size_t(units) / 4) + 16))) return rc;
        bins.n_pairs = int(pairs);
        bins.n_big = h_big;
        *total = pairs;
        // PSG_TRACE_BINS=1: candidate-count histogram of the batch's tiles (synchronous
        // binnings only; a debugging aid, it reads the counts back)
        static const bool trace_bins = [] {
            const char* e = std::getenv("PSG_TRACE_BINS");
            return e && e[0] == '1';
        }();
        if (trace_bins) {
            std::vector<int> hc(static_cast<size_t>(T), 0);
            PSG_CUDA(cudaMemcpy(hc.data(), ctx->d_counts, size_t(T) * sizeof(int), cudaMemcpyDeviceToHost));
            long long h[7] = {0, 0, 0, 0, 0, 0, 0};
            long long work[7] = {0, 0, 0, 0, 0, 0, 0};
            for (int c : hc) {
                const int k = c == 0 ? 0 : c <= 128 ? 1 : c <= 256 ? 2 : c <= 512 ? 3 : c <= 1024 ? 4 : c <= 2048 ? 5 : 6;
                ++h[k];
                work[k] += c;
            }
            std::fprintf(stderr,
                         "psg.bins views %d tiles %d pairs %lld | tiles (pairs) by candidates: 0: %lld, <=128: %lld "
                         "(%lld), <=256: %lld (%lld), <=512: %lld (%lld), <=1024: %lld (%lld), <=2048: %lld "
                         "(%lld), >2048: %lld (%lld)\n",
                         n, T, (long long)pairs, h[0], h[1], work[1], h[2], work[2], h[3], work[3], h[4], work[4], h[5],
                         work[5], h[6], work[6]);
        }
    } else {
        if ((rc = grow(ctx->d_items, ctx->items_cap, 1))) return rc;
        if ((rc = grow(ctx->d_pair_tile, ctx->pair_tile_cap, 1))) return rc;
        if ((rc = grow(ctx->d_recs, ctx->recs_cap, 16))) return rc;
        bins.n_pairs = -1;
        bins.n_big = -1;
        *total = -1;
    }
    bins.items = ctx->d_items;
    bins.pair_tile = ctx->d_pair_tile;
    bins.recs = ctx->d_recs;
    bins.items_cap = (long long)std::min(ctx->items_cap, ctx->pair_tile_cap);
    // capacity guard (async) or statistics only (sync: everything fits)
    launch_bin_guard(bins, (long long)(ctx->recs_cap / 16), sync ? (long long)kNoLimit : ctx->pair_limit,
                     ctx->d_misc + 9, sync ? nullptr : ctx->d_grads + size_t(ctx->P) * 11 + 1, ctx->d_stats, s);
    PSG_CUDA(cudaMemcpyAsync(ctx->d_cursor, ctx->d_offsets, size_t(T) * sizeof(int),
                             cudaMemcpyDeviceToDevice, s));
    launch_scatter(batch, ctx->P, bins, s);
    ctx->stats.tiles += T;
    return PSG_OK;
}

}  // namespace

namespace psg {
int set_error(int status, const std::string& msg) { return fail(status, msg); }
}  // namespace psg

namespace {

int refresh_counts(psg_context* ctx) {
    // valid-target counts per view (renderer.cpp:328-334), computed once: targets are static
    const int nv = int(ctx->h_views.size());
    if (nv == 0 || !ctx->d_td) return PSG_OK;
    unsigned long long* d_cnt = nullptr;
    PSG_CUDA(cudaMalloc(&d_cnt, sizeof(unsigned long long) * 2 * size_t(nv)));
    PSG_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * 2 * size_t(nv), ctx->stream));
    launch_target_counts(ctx->d_views, nv, ctx->d_td, ctx->d_tn, d_cnt, ctx->stream);
    std::vector<unsigned long long> h(2 * size_t(nv));
    PSG_CUDA(cudaMemcpyAsync(h.data(), d_cnt, h.size() * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(d_cnt);
    for (int i = 0; i < nv; ++i) {
        ctx->h_views[size_t(i)].inv_d = h[2 * size_t(i)] ? 1.0 / double(h[2 * size_t(i)]) : 0.0;
        ctx->h_views[size_t(i)].inv_n = h[2 * size_t(i) + 1] ? 1.0 / double(h[2 * size_t(i) + 1]) : 0.0;
    }
    PSG_CUDA(cudaMemcpyAsync(ctx->d_views, ctx->h_views.data(), sizeof(ViewDev) * size_t(nv),
                             cudaMemcpyHostToDevice, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->host_inv_stale = false;
    return PSG_OK;
}

__global__ void k_iota(int* v, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = int(i);
}

__global__ void k_fold_loss(const double* view_loss, const int* vid, const ViewDev* views, int n,
                            double alpha1, double alpha2, double view_scale, double* acc) {
    double s = 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const ViewDev& v = views[vid[k]];
        // lg.loss = a1*sum_n*inv_n + a2*sum_d*inv_d, scaled (renderer.cpp:369, optimizer.cpp:74)
        const double l = alpha1 * view_loss[2 * k + 1] * v.inv_n + alpha2 * view_loss[2 * k] * v.inv_d;
        s += l * view_scale;
    }
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    __shared__ double part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += part[w];
        *acc += t;
    }
}

}  // namespace

extern "C" {

const char* psg_last_error(void) { return g_err.c_str(); }
int psg_abi_version(void) { return PSG_ABI_VERSION; }
void psg_default_config(psg_render_config* cfg) { default_cfg(cfg); }

double psg_lambda_schedule(int64_t ite, double base, double rate, double lmax) {
    const double l = base * std::exp(-(1.0 - rate * double(ite)));  // splatting.cpp:7-10
    return std::min(l, lmax);
}

int psg_create(int device, int precision, psg_context** out) {
    if (!out) return fail(PSG_EINVAL, "null out pointer");
    *out = nullptr;
    if (precision != PSG_FP32 && precision != PSG_FP64 && precision != PSG_MIXED)
        return fail(PSG_EINVAL, "bad precision");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(PSG_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(PSG_EINVAL, "device index out of range");
    PSG_CUDA(cudaSetDevice(device));
    psg_context* ctx = new psg_context();
    ctx->device = device;
    ctx->precision = precision;
    default_cfg(&ctx->cfg);
    int lo_prio = 0, hi_prio = 0;
    if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio) != cudaSuccess ||
        cudaStreamCreateWithPriority(&ctx->aux.stream, cudaStreamNonBlocking, hi_prio) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->aux.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->aux.join, cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&ctx->d_misc, 16 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&ctx->d_stats_snap, sizeof(Stats)) != cudaSuccess ||
        cudaMalloc(&ctx->d_stats, sizeof(Stats)) != cudaSuccess ||
        cudaMalloc(&ctx->d_view1, sizeof(ViewDev)) != cudaSuccess ||
        cudaMalloc(&ctx->d_sums, 2 * sizeof(double)) != cudaSuccess ||
        cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_total), 64, cudaHostAllocDefault) != cudaSuccess) {
        delete ctx;
        return fail(PSG_ECUDA, "context allocation failed");
    }
    ctx->stream = ctx->own_stream;
    cudaMemset(ctx->d_stats, 0, sizeof(Stats));
    cudaMemset(ctx->d_misc, 0, 16 * sizeof(unsigned long long));
    *out = ctx;
    return PSG_OK;
}

int psg_destroy(psg_context* ctx) {
    if (!ctx) return PSG_OK;
    { std::lock_guard<std::recursive_mutex> wait_for_callers(ctx->mu); }
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->comm) nccl_api().comm_destroy(ctx->comm);
    void* ptrs[] = {ctx->d_center, ctx->d_rot, ctx->d_radii, ctx->d_geo, ctx->d_geof, ctx->d_grads, ctx->d_big,
                    ctx->d_views, ctx->d_td, ctx->d_tn, ctx->d_vid, ctx->d_counts,
                    ctx->d_offsets, ctx->d_cursor, ctx->d_items, ctx->d_rects, ctx->d_cub,
                    ctx->d_view_loss, ctx->d_misc, ctx->d_stats, ctx->d_view1, ctx->d_maps,
                    ctx->d_rec_prim, ctx->d_rec_count, ctx->d_t1, ctx->d_sums, ctx->d_g1,
                    ctx->d_smaps, ctx->d_m, ctx->d_v, ctx->d_step, ctx->d_rgs, ctx->d_rgc,
                    ctx->d_pow, ctx->d_split, ctx->d_recs, ctx->d_desc, ctx->d_units,
                    ctx->d_pair_tile, ctx->d_tile_slot, ctx->d_det, ctx->d_det_sort, ctx->d_snap,
                    ctx->d_stats_snap, ctx->d_cnt, ctx->d_runlog, ctx->d_pack, ctx->d_pack_off};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (int i = 0; i < psg_context::kStage; ++i) {
        if (ctx->h_ring[i]) cudaFreeHost(ctx->h_ring[i]);
        if (ctx->ring_ev[i]) cudaEventDestroy(ctx->ring_ev[i]);
    }
    if (ctx->h_total) cudaFreeHost(ctx->h_total);
    if (ctx->h_big) cudaFreeHost(ctx->h_big);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->aux.stream) cudaStreamDestroy(ctx->aux.stream);
    if (ctx->aux.fork) cudaEventDestroy(ctx->aux.fork);
    if (ctx->aux.join) cudaEventDestroy(ctx->aux.join);
    delete ctx;
    return PSG_OK;
}

int psg_set_stream(psg_context* ctx, void* stream) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return PSG_OK;
}

void* psg_get_stream(psg_context* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int psg_set_config(psg_context* ctx, const psg_render_config* cfg) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (!cfg) return fail(PSG_EINVAL, "null config");
    ctx->cfg = *cfg;
    return PSG_OK;
}

int psg_synchronize(psg_context* ctx) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    return PSG_OK;
}

int psg_set_planes(psg_context* ctx, int64_t n, const double* center, const double* rotation,
                   const double* radii, const int64_t* ids) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (n < 0 || (n > 0 && (!center || !rotation || !radii)))
        return fail(PSG_EINVAL, "set_planes: bad arguments");
    if (n >= (int64_t(1) << 26)) return fail(PSG_EINVAL, "set_planes: too many planes (limit 2^26)");
    ctx->P = n;
    ctx->optim_ready = false;  // a new scene starts a fresh optimiser state
    ctx->ids.assign(size_t(n), 0);
    for (int64_t i = 0; i < n; ++i) ctx->ids[size_t(i)] = ids ? ids[i] : i;
    if (n == 0) return PSG_OK;
    const size_t un = size_t(n);
    if ((rc = grow(ctx->d_center, ctx->plane_cap, un * 3))) return rc;
    if ((rc = grow(ctx->d_rot, ctx->plane_cap_q, un * 4))) return rc;
    if ((rc = grow(ctx->d_radii, ctx->plane_cap_r, un * 4))) return rc;
    if ((rc = grow(ctx->d_geo, ctx->geo_cap, un))) return rc;
    if ((rc = grow(ctx->d_geof, ctx->geof_cap, un))) return rc;
    if ((rc = grow(ctx->d_grads, ctx->grads_cap, un * 11 + 2))) return rc;
    cudaStream_t s = ctx->stream;
    PSG_CUDA(cudaMemcpyAsync(ctx->d_center, center, un * 3 * 8, cudaMemcpyHostToDevice, s));
    PSG_CUDA(cudaMemcpyAsync(ctx->d_rot, rotation, un * 4 * 8, cudaMemcpyHostToDevice, s));
    PSG_CUDA(cudaMemcpyAsync(ctx->d_radii, radii, un * 4 * 8, cudaMemcpyHostToDevice, s));
    return PSG_OK;
}

int64_t psg_num_planes(psg_context* ctx) { return ctx ? ctx->P : -1; }

int psg_set_views(psg_context* ctx, int n_views, const psg_camera* cams, const float* td,
                  const float* tn) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (n_views < 0 || (n_views > 0 && !cams)) return fail(PSG_EINVAL, "set_views: bad arguments");
    for (int i = 0; i < n_views; ++i) {
        if (cams[i].width < 1 || cams[i].height < 1)
            return fail(PSG_EINVAL, "set_views: empty view");
        if (cams[i].width > kMaxSide || cams[i].height > kMaxSide)
            return fail(PSG_EINVAL, "set_views: width and height must be <= 32767");
    }
    ctx->h_views.clear();
    long long off = 0;
    for (int i = 0; i < n_views; ++i) {
        ctx->h_views.push_back(make_view(cams[i], off));
        off += (long long)cams[i].width * cams[i].height;
    }
    ctx->total_px = off;
    if ((rc = grow(ctx->d_views, ctx->views_cap, size_t(std::max(n_views, 1))))) return rc;
    // + one tile row of padding: the rasteriser's TMA row copies of a right-edge
    // tile may read up to 15 pixels past the last row
    if ((rc = grow(ctx->d_td, ctx->td_cap, size_t(std::max<long long>(off, 1)) + 16))) return rc;
    if ((rc = grow(ctx->d_tn, ctx->tn_cap, size_t(std::max<long long>(3 * off, 1)) + 48))) return rc;
    ctx->targets_tma = true;
    for (int i = 0; i < n_views; ++i) ctx->targets_tma = ctx->targets_tma && cams[i].width % 4 == 0;
    PSG_CUDA(cudaMemcpyAsync(ctx->d_views, ctx->h_views.data(), sizeof(ViewDev) * size_t(n_views),
                             cudaMemcpyHostToDevice, ctx->stream));
    if (td && tn) {
        PSG_CUDA(cudaMemcpyAsync(ctx->d_td, td, size_t(off) * 4, cudaMemcpyHostToDevice, ctx->stream));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_tn, tn, size_t(off) * 12, cudaMemcpyHostToDevice, ctx->stream));
    } else {
        PSG_CUDA(cudaMemsetAsync(ctx->d_td, 0, size_t(off) * 4, ctx->stream));
        PSG_CUDA(cudaMemsetAsync(ctx->d_tn, 0, size_t(off) * 12, ctx->stream));
    }
    return refresh_counts(ctx);
}

int psg_update_targets(psg_context* ctx, int first, int count, const float* td, const float* tn) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    const int nv = int(ctx->h_views.size());
    if (first < 0 || count < 0 || first + count > nv || !td || !tn)
        return fail(PSG_EINVAL, "update_targets: bad range");
    if (count == 0) return PSG_OK;
    const long long o0 = ctx->h_views[size_t(first)].pix_off;
    const ViewDev& last = ctx->h_views[size_t(first + count - 1)];
    const long long o1 = last.pix_off + (long long)last.W * last.H;
    PSG_CUDA(cudaMemcpyAsync(ctx->d_td + o0, td, size_t(o1 - o0) * 4, cudaMemcpyHostToDevice, ctx->stream));
    PSG_CUDA(cudaMemcpyAsync(ctx->d_tn + 3 * o0, tn, size_t(o1 - o0) * 12, cudaMemcpyHostToDevice, ctx->stream));
    return PSG_OK;
}

int psg_get_targets(psg_context* ctx, int view, float* td, float* tn) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (view < 0 || view >= int(ctx->h_views.size())) return fail(PSG_EINVAL, "bad view");
    const ViewDev& v = ctx->h_views[size_t(view)];
    const size_t np = size_t(v.W) * size_t(v.H);
    PSG_CUDA(cudaMemcpyAsync(td, ctx->d_td + v.pix_off, np * 4, cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaMemcpyAsync(tn, ctx->d_tn + 3 * v.pix_off, np * 12, cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    return PSG_OK;
}

int psg_render_ground_truth(psg_context* ctx, int n_faces, const double* faces) {
    Nvtx nvtx_range("psg.render_ground_truth");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (n_faces < 0 || (n_faces > 0 && !faces)) return fail(PSG_EINVAL, "bad faces");
    const int nv = int(ctx->h_views.size());
    if (nv == 0) return PSG_OK;
    double* d_faces = nullptr;
    PSG_CUDA(cudaMalloc(&d_faces, sizeof(double) * 15 * size_t(std::max(n_faces, 1))));
    PSG_CUDA(cudaMemcpyAsync(d_faces, faces, sizeof(double) * 15 * size_t(n_faces),
                             cudaMemcpyHostToDevice, ctx->stream));
    int max_px = 0;
    for (const ViewDev& v : ctx->h_views) max_px = std::max(max_px, v.W * v.H);
    launch_render_gt(ctx->d_views, nv, d_faces, n_faces, ctx->d_td, ctx->d_tn, max_px, ctx->stream);
    PSG_CUDA(cudaGetLastError());
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(d_faces);
    return refresh_counts(ctx);
}

int psg_zero_grads(psg_context* ctx) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    // the open window's steps are discarded with their gradients, aborted or not
    ctx->pending.clear();
    ctx->window_open = false;
    ctx->window_allreduced = false;
    if (ctx->P > 0)
        PSG_CUDA(cudaMemsetAsync(ctx->d_grads, 0, (size_t(ctx->P) * 11 + 2) * sizeof(double), ctx->stream));
    return PSG_OK;
}

}  // extern "C"

namespace {

// Map buffers and per-view loss sums of a step over n views (all sub-batches of a
// split step write into them at their slot offset).
int step_outputs(psg_context* ctx, const std::vector<int>& vids, int flags) {
    const int n = int(vids.size());
    int rc;
    if ((rc = grow(ctx->d_view_loss, ctx->view_loss_cap, size_t(2 * n)))) return rc;
    PSG_CUDA(cudaMemsetAsync(ctx->d_view_loss, 0, sizeof(double) * 2 * size_t(n), ctx->stream));
    if (flags & PSG_STEP_WRITE_MAPS) {
        long long stride = 0;
        for (int v : vids)
            stride = std::max<long long>(stride, (long long)ctx->h_views[size_t(v)].W * ctx->h_views[size_t(v)].H);
        if ((rc = grow(ctx->d_smaps, ctx->smaps_cap, size_t(stride) * 5 * size_t(n)))) return rc;
        ctx->smaps_stride = stride;
        ctx->smaps_n = n;
    }
    return PSG_OK;
}

// Bin + rasterise views `vids` as slots [slot0, slot0 + |vids|) of the current
// step's outputs. sync: exact sizes (deterministic mode, replays), and a view
// group whose bin entries exceed the pair limit is split in halves.
int step_run(psg_context* ctx, const std::vector<int>& vids, double lambda, double view_scale, int flags,
             int slot0, bool sync) {
    const int n = int(vids.size());
    cudaStream_t s = ctx->stream;
    const RenderParams rp = make_params(ctx->cfg, lambda, view_scale);
    Batch batch{};
    Bins bins{};
    int64_t total = 0;
    int rc = bin_batch(ctx, ctx->d_views, ctx->h_views, vids, rp.cut, batch, bins, sync, &total);
    if (rc == kSplit) {
        if (n == 1)
            return fail(PSG_EINVAL, "step: one view has " + std::to_string(total) +
                                        " tile-plane bin entries, above the 32-bit limit");
        const int h = n / 2;
        std::vector<int> a(vids.begin(), vids.begin() + h), b(vids.begin() + h, vids.end());
        if ((rc = step_run(ctx, a, lambda, view_scale, flags, slot0, true))) return rc;
        return step_run(ctx, b, lambda, view_scale, flags, slot0 + h, true);
    }
    if (rc) return rc;
    RasterIO io{};
    io.td = ctx->d_td;
    io.tn = ctx->d_tn;
    if (flags & PSG_STEP_WRITE_MAPS) {
        const long long st = ctx->smaps_stride, nf = ctx->smaps_n;
        io.out_depth_f = ctx->d_smaps + slot0 * st;
        io.out_alpha_f = ctx->d_smaps + st * nf + slot0 * st;
        io.out_normal_f = ctx->d_smaps + 2 * st * nf + 3 * slot0 * st;
        io.map_stride = st;
    }
    io.grads = ctx->d_grads;
    io.view_loss = ctx->d_view_loss + 2 * size_t(slot0);
    io.do_backward = (flags & PSG_STEP_NO_BACKWARD) ? 0 : 1;
    io.tma_targets = ctx->targets_tma ? 1 : 0;
    size_t det_g = 0, det_l = 0;
    if (ctx->deterministic) {
        int Tt = 0;
        for (int v : vids) Tt += ctx->h_views[size_t(v)].tiles_x * ctx->h_views[size_t(v)].tiles_y;
        det_g = size_t(total) * 8 * 11;
        det_l = size_t(Tt) * 8 * 2;
        const size_t det_m = (size_t(total) + 1) / 2;  // one 32-bit warp mask per bin entry
        if ((rc = grow(ctx->d_det, ctx->det_cap, det_g + det_l + det_m + 1))) return rc;
        // the gradient partials need no clearing: only slots a warp wrote (mask) are read
        PSG_CUDA(cudaMemsetAsync(ctx->d_det + det_g, 0, (det_l + det_m) * sizeof(double), s));
        io.det_grads = ctx->d_det;
        io.det_loss = ctx->d_det + det_g;
        io.det_mask = reinterpret_cast<unsigned*>(ctx->d_det + det_g + det_l);
    }
    io.stats = ctx->d_stats;
    launch_raster(ctx->precision, ctx->deterministic ? kFusedDet : kFused, batch, ctx->d_geo, ctx->d_geof,
                  ctx->P, bins, rp, io, s, ctx->aux);
    PSG_CUDA(cudaGetLastError());
    if (ctx->deterministic && total > 0) {
        // bin entries sorted by plane, entry order kept (stable radix sort)
        if ((rc = grow(ctx->d_det_sort, ctx->det_sort_cap, 3 * size_t(total) + 1))) return rc;
        int* keys_out = ctx->d_det_sort;
        int* vals_in = keys_out + total;
        int* vals_out = vals_in + total;
        k_iota<<<unsigned((total + 255) / 256), 256, 0, s>>>(vals_in, total);
        int bits = 1;
        while ((int64_t(1) << bits) <= ctx->P) ++bits;
        size_t tmp = 0;
        PSG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, bins.items, keys_out, vals_in, vals_out,
                                                 int(total), 0, bits, s));
        if (tmp > ctx->cub_cap) {
            if (ctx->d_cub) cudaFree(ctx->d_cub);
            ctx->d_cub = nullptr;
            ctx->cub_cap = 0;
            PSG_CUDA(cudaMalloc(&ctx->d_cub, tmp));
            ctx->cub_cap = tmp;
        }
        tmp = ctx->cub_cap;
        PSG_CUDA(cub::DeviceRadixSort::SortPairs(ctx->d_cub, tmp, bins.items, keys_out, vals_in, vals_out,
                                                 int(total), 0, bits, s));
        launch_det_reduce(keys_out, vals_out, total, ctx->P, ctx->d_det,
                          reinterpret_cast<const unsigned*>(ctx->d_det + det_g + det_l), ctx->d_grads, batch,
                          ctx->d_det + det_g, io.view_loss, s);
        PSG_CUDA(cudaGetLastError());
    } else if (ctx->deterministic) {
        launch_det_reduce(nullptr, nullptr, 0, 0, nullptr, nullptr, ctx->d_grads, batch, ctx->d_det + det_g,
                          io.view_loss, s);
    }
    k_fold_loss<<<1, 256, 0, s>>>(io.view_loss, ctx->d_vid, ctx->d_views, n, ctx->cfg.alpha1, ctx->cfg.alpha2,
                                  view_scale, ctx->d_grads + size_t(ctx->P) * 11);
    PSG_CUDA(cudaGetLastError());
    return PSG_OK;
}

int open_window(psg_context* ctx) {
    if (ctx->window_open) return PSG_OK;
    int rc;
    const size_t g = size_t(ctx->P) * 11 + 2;
    if ((rc = grow(ctx->d_snap, ctx->snap_cap, g))) return rc;
    PSG_CUDA(cudaMemcpyAsync(ctx->d_snap, ctx->d_grads, g * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    PSG_CUDA(cudaMemcpyAsync(ctx->d_stats_snap, ctx->d_stats, sizeof(Stats), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    ctx->host_stats_snap = ctx->stats;
    ctx->window_open = true;
    ctx->window_allreduced = false;
    return PSG_OK;
}

// The window's steps again, from the gradients and statistics of its start, with
// exact sizes (and the all-reduce again when the window had one: the guard count
// travels in the reduced buffer, so every rank replays together).
int replay_window(psg_context* ctx) {
    cudaStream_t s = ctx->stream;
    const size_t g = size_t(ctx->P) * 11 + 2;
    PSG_CUDA(cudaMemcpyAsync(ctx->d_grads, ctx->d_snap, g * 8, cudaMemcpyDeviceToDevice, s));
    PSG_CUDA(cudaMemsetAsync(ctx->d_grads + g - 1, 0, sizeof(double), s));
    PSG_CUDA(cudaMemcpyAsync(ctx->d_stats, ctx->d_stats_snap, sizeof(Stats), cudaMemcpyDeviceToDevice, s));
    PSG_CUDA(cudaMemsetAsync(ctx->d_misc + 9, 0, 2 * sizeof(unsigned long long), s));
    ctx->stats = ctx->host_stats_snap;
    std::vector<psg_context::Pending> pend;
    pend.swap(ctx->pending);
    ctx->window_open = false;
    int rc;
    for (const auto& p : pend) {
        if (!p.outs.empty() && (rc = step_outputs(ctx, p.outs, p.flags))) return rc;
        if ((rc = step_run(ctx, p.vids, p.lambda, p.view_scale, p.flags, p.slot0, true))) return rc;
        ctx->stats.views += int64_t(p.vids.size());
        for (int v : p.vids) ctx->stats.pixels += (long long)ctx->h_views[size_t(v)].W * ctx->h_views[size_t(v)].H;
    }
    if (ctx->window_allreduced) {
        ctx->window_allreduced = false;
        if ((rc = psg_allreduce_grads(ctx))) return rc;
    }
    ctx->stats.replays += 1;
    return PSG_OK;
}

// Close the step window before anything reads results or changes what its steps
// read: one guard read-back (a synchronisation), and a replay if a step aborted.
int settle(psg_context* ctx) {
    if (!ctx->window_open) return PSG_OK;
    PSG_CUDA(cudaMemcpyAsync(ctx->h_total + 7, ctx->d_grads + size_t(ctx->P) * 11 + 1, 8,
                             cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    double guard = 0.0;
    std::memcpy(&guard, ctx->h_total + 7, 8);
    if (guard == 0.0) {
        ctx->pending.clear();
        ctx->window_open = false;
        ctx->window_allreduced = false;
        return PSG_OK;
    }
    return replay_window(ctx);
}

__global__ void k_set_inv(ViewDev* views, const unsigned long long* counts, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long cd = counts[2 * i], cn = counts[2 * i + 1];
    views[i].inv_d = cd ? 1.0 / double(cd) : 0.0;  // renderer.cpp:328-334
    views[i].inv_n = cn ? 1.0 / double(cn) : 0.0;
}

}  // namespace

extern "C" {

int psg_set_pair_limit(psg_context* ctx, int64_t limit) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (limit < 1 || limit > 2147483647LL) return fail(PSG_EINVAL, "set_pair_limit: limit must be in [1, 2^31-1]");
    ctx->pair_limit = limit;
    return PSG_OK;
}

}  // extern "C"

namespace {

// One step over `all` in passes of `chunk` views (psg_step: one pass; psg_step_host:
// one pass per streamed chunk, after its copy). Outputs (per-view losses, maps) are
// laid out for the whole step; each pass writes its slots.
int step_passes(psg_context* ctx, const std::vector<int>& all, int chunk, double lambda, double view_scale,
                int flags, const std::function<int(int, int)>& before_pass) {
    int rc;
    cudaStream_t s = ctx->stream;
    // deterministic mode sizes its partial buffers from the entry total: synchronous
    const bool sync = ctx->deterministic;
    if (sync) {
        if ((rc = settle(ctx))) return rc;
    } else if ((rc = open_window(ctx))) {
        return rc;
    }
    if ((rc = step_outputs(ctx, all, flags))) return rc;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->timing) {
        PSG_CUDA(cudaEventCreate(&e0));
        PSG_CUDA(cudaEventCreate(&e1));
        PSG_CUDA(cudaEventRecord(e0, s));
    }
    const int n = int(all.size());
    for (int c0 = 0; c0 < n; c0 += chunk) {
        const int c1 = std::min(n, c0 + chunk);
        if (before_pass && (rc = before_pass(c0, c1))) return rc;
        std::vector<int> sub(all.begin() + c0, all.begin() + c1);
        if (!sync)
            ctx->pending.push_back({sub, lambda, view_scale, flags, c0, c0 == 0 ? all : std::vector<int>()});
        if ((rc = step_run(ctx, sub, lambda, view_scale, flags, c0, sync))) return rc;
    }
    if (ctx->timing) {
        PSG_CUDA(cudaEventRecord(e1, s));
        ctx->events.emplace_back(e0, e1);
    }
    ctx->last_vids = all;
    ctx->last_view_scale = view_scale;
    ctx->stats.views += n;
    for (int v : all) ctx->stats.pixels += (long long)ctx->h_views[size_t(v)].W * ctx->h_views[size_t(v)].H;
    return PSG_OK;
}

}  // namespace

extern "C" {

int psg_step(psg_context* ctx, const int32_t* view_ids, int n, double lambda, double view_scale,
             int flags) {
    Nvtx nvtx_range("psg.step");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = check_cfg(ctx->cfg))) return rc;
    if (n < 0 || (n > 0 && !view_ids)) return fail(PSG_EINVAL, "step: bad view list");
    if (!(lambda > 0.0)) return fail(PSG_EINVAL, "step: lambda must be > 0");
    if (ctx->P == 0 || n == 0) {
        ctx->last_vids.clear();
        return PSG_OK;
    }
    std::vector<int> vids(view_ids, view_ids + n);
    for (int v : vids)
        if (v < 0 || v >= int(ctx->h_views.size())) return fail(PSG_EINVAL, "step: view id out of range");
    return step_passes(ctx, vids, n, lambda, view_scale, flags, nullptr);
}

int psg_step_host(psg_context* ctx, int first, int count, double lambda, double view_scale,
                  int flags, const float* td, const float* tn, int chunk_views) {
    Nvtx nvtx_range("psg.step_host");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = check_cfg(ctx->cfg))) return rc;
    const int nv = int(ctx->h_views.size());
    if (first < 0 || count < 0 || first + count > nv || (count > 0 && (!td || !tn)))
        return fail(PSG_EINVAL, "step_host: bad view range");
    if (!(lambda > 0.0)) return fail(PSG_EINVAL, "step: lambda must be > 0");
    if (chunk_views < 1) chunk_views = 128;
    if (count == 0) return PSG_OK;
    const long long base = ctx->h_views[size_t(first)].pix_off;
    // the copies overwrite targets that earlier work on the context stream may still
    // read: the copy stream waits for everything enqueued so far
    std::vector<cudaEvent_t> ev;
    cudaEvent_t ready;
    PSG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    ev.push_back(ready);
    PSG_CUDA(cudaEventRecord(ready, ctx->stream));
    PSG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ready, 0));
    // enqueue every chunk's copy first: the copy engine streams targets while the
    // compute stream works through the chunks already resident
    for (int c0 = 0; c0 < count; c0 += chunk_views) {
        const int c1 = std::min(count, c0 + chunk_views);
        const long long o0 = ctx->h_views[size_t(first + c0)].pix_off;
        const ViewDev& last = ctx->h_views[size_t(first + c1 - 1)];
        const long long o1 = last.pix_off + (long long)last.W * last.H;
        PSG_CUDA(cudaMemcpyAsync(ctx->d_td + o0, td + (o0 - base), size_t(o1 - o0) * 4,
                                 cudaMemcpyHostToDevice, ctx->copy_stream));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_tn + 3 * o0, tn + 3 * (o0 - base), size_t(o1 - o0) * 12,
                                 cudaMemcpyHostToDevice, ctx->copy_stream));
        cudaEvent_t e;
        PSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        PSG_CUDA(cudaEventRecord(e, ctx->copy_stream));
        ev.push_back(e);
    }
    if ((rc = grow(ctx->d_cnt, ctx->cnt_cap, 2 * size_t(count)))) return rc;
    std::vector<int> all;
    for (int i = 0; i < count; ++i) all.push_back(first + i);
    auto before_pass = [&](int c0, int c1) -> int {
        PSG_CUDA(cudaStreamWaitEvent(ctx->stream, ev[size_t(1 + c0 / chunk_views)], 0));
        // render_loss counts the valid pixels of the targets it is given
        // (renderer.cpp:328-334): the streamed chunk's counts, on the device
        PSG_CUDA(cudaMemsetAsync(ctx->d_cnt + 2 * c0, 0, 2 * size_t(c1 - c0) * 8, ctx->stream));
        launch_target_counts(ctx->d_views + first + c0, c1 - c0, ctx->d_td, ctx->d_tn, ctx->d_cnt + 2 * c0,
                             ctx->stream);
        k_set_inv<<<unsigned((c1 - c0 + 127) / 128), 128, 0, ctx->stream>>>(ctx->d_views + first + c0,
                                                                           ctx->d_cnt + 2 * c0, c1 - c0);
        PSG_CUDA(cudaGetLastError());
        return PSG_OK;
    };
    if (ctx->P > 0) rc = step_passes(ctx, all, chunk_views, lambda, view_scale, flags, before_pass);
    ctx->host_inv_stale = true;
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    return rc;
}

int psg_finalize_grads(psg_context* ctx, int64_t* bad_id) {
    Nvtx nvtx_range("psg.finalize_grads");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (ctx->P == 0) return PSG_OK;
    cudaStream_t s = ctx->stream;
    unsigned long long first_bad = 0;
    for (int attempt = 0;; ++attempt) {
        PSG_CUDA(cudaMemsetAsync(ctx->d_misc, 0xff, sizeof(unsigned long long), s));
        launch_finalize_grads(ctx->d_geo, ctx->d_grads, ctx->P, ctx->d_misc, s);
        PSG_CUDA(cudaMemcpyAsync(ctx->h_total, ctx->d_misc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->h_total + 7, ctx->d_grads + size_t(ctx->P) * 11 + 1, 8,
                                 cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaStreamSynchronize(s));
        double guard = 0.0;
        std::memcpy(&guard, ctx->h_total + 7, 8);
        if (ctx->window_open && guard != 0.0 && attempt == 0) {
            if ((rc = replay_window(ctx))) return rc;  // restores the pre-finalize gradients
            continue;
        }
        ctx->pending.clear();
        ctx->window_open = false;
        ctx->window_allreduced = false;
        break;
    }
    std::memcpy(&first_bad, ctx->h_total, sizeof(first_bad));
    if (first_bad != ~0ull) {
        const int64_t id = ctx->ids[size_t(first_bad)];
        if (bad_id) *bad_id = id;
        return fail(PSG_ENONFINITE,
                    "backward: non-finite gradient for primitive id " + std::to_string(id));
    }
    return PSG_OK;
}

int psg_read_grads(psg_context* ctx, double* grads, double* loss) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (ctx->P == 0) {
        if (loss) *loss = 0.0;
        return PSG_OK;
    }
    if (grads)
        PSG_CUDA(cudaMemcpyAsync(grads, ctx->d_grads, size_t(ctx->P) * 11 * 8, cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaMemcpyAsync(ctx->h_total + 6, ctx->d_grads + size_t(ctx->P) * 11, 8, cudaMemcpyDeviceToHost,
                             ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (loss) std::memcpy(loss, ctx->h_total + 6, 8);
    return PSG_OK;
}

int psg_read_view_losses(psg_context* ctx, double* losses, int n) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    const int m = int(ctx->last_vids.size());
    if (n < m || !losses) return fail(PSG_EINVAL, "read_view_losses: buffer too small");
    std::vector<double> raw(2 * size_t(m));
    if (m > 0)
        PSG_CUDA(cudaMemcpyAsync(raw.data(), ctx->d_view_loss, raw.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    // the normalisers of streamed targets are computed on the device (psg_step_host)
    std::vector<ViewDev> dv;
    if (ctx->host_inv_stale && !ctx->h_views.empty()) {
        dv.resize(ctx->h_views.size());
        PSG_CUDA(cudaMemcpyAsync(dv.data(), ctx->d_views, dv.size() * sizeof(ViewDev), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    }
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < m; ++k) {
        const size_t vi = size_t(ctx->last_vids[size_t(k)]);
        const ViewDev& v = dv.empty() ? ctx->h_views[vi] : dv[vi];
        losses[k] = (ctx->cfg.alpha1 * raw[2 * size_t(k) + 1] * v.inv_n +
                     ctx->cfg.alpha2 * raw[2 * size_t(k)] * v.inv_d) * ctx->last_view_scale;
    }
    return PSG_OK;
}

int psg_read_step_maps(psg_context* ctx, int k, float* depth, float* normal, float* alpha) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    const int n = int(ctx->last_vids.size());
    if (k < 0 || k >= n || !ctx->d_smaps || ctx->smaps_n != n)
        return fail(PSG_EINVAL, "read_step_maps: no maps for slot");
    const ViewDev& v = ctx->h_views[size_t(ctx->last_vids[size_t(k)])];
    const size_t np = size_t(v.W) * size_t(v.H);
    const long long st = ctx->smaps_stride;
    cudaStream_t s = ctx->stream;
    if (depth) PSG_CUDA(cudaMemcpyAsync(depth, ctx->d_smaps + k * st, np * 4, cudaMemcpyDeviceToHost, s));
    if (alpha) PSG_CUDA(cudaMemcpyAsync(alpha, ctx->d_smaps + st * n + k * st, np * 4, cudaMemcpyDeviceToHost, s));
    if (normal)
        PSG_CUDA(cudaMemcpyAsync(normal, ctx->d_smaps + 2 * st * n + 3 * k * st, np * 12, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    return PSG_OK;
}

int psg_set_timing(psg_context* ctx, int enable) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    ctx->timing = enable != 0;
    return PSG_OK;
}

int psg_get_kernel_ms(psg_context* ctx, double* raster_ms, int* launches) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    double tot = 0.0;
    for (auto& ev : ctx->events) {
        float ms = 0.0f;
        PSG_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
        tot += ms;
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    if (raster_ms) *raster_ms = tot;
    if (launches) *launches = int(ctx->events.size());
    ctx->events.clear();
    return PSG_OK;
}

int psg_get_stats(psg_context* ctx, psg_stats* out) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    Stats st{};
    PSG_CUDA(cudaMemcpyAsync(&st, ctx->d_stats, sizeof(Stats), cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = ctx->stats;
    out->pairs = int64_t(st.pairs);
    out->big_tiles = int64_t(st.big);
    out->zbound_violations = int64_t(st.zviol);
    out->pixel_pairs = int64_t(st.pair_px);
    out->live_records = int64_t(st.live);
    out->cull_checks = int64_t(st.cull_checks);
    out->cull_misses = int64_t(st.cull_miss);
    return PSG_OK;
}

// -DPSG_PROBE builds: the per-pixel work counters (12 x u64; zeros otherwise):
// considered candidates, exact tests, exact rejections with a full list, insertions,
// mid-list insertions, shifts, pixels done early, pixels with full lists, pixels,
// exact rejections with a free list, appends dropped by a full list, candidates of
// the pixels' tiles.
int psg_debug_probe(psg_context* ctx, uint64_t* out) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    Stats st{};
    PSG_CUDA(cudaMemcpyAsync(&st, ctx->d_stats, sizeof(Stats), cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 12; ++i) out[i] = st.probe[i];
    return PSG_OK;
}

int psg_reset_stats(psg_context* ctx) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    ctx->stats = psg_stats{};
    PSG_CUDA(cudaMemsetAsync(ctx->d_stats, 0, sizeof(Stats), ctx->stream));
    return PSG_OK;
}

// ---- drop-in single-view calls --------------------------------------------

}  // extern "C"

namespace {
int single_view_bins(psg_context* ctx, const psg_camera* cam, double lambda, Batch& batch,
                     Bins& bins, int64_t* total) {
    std::vector<ViewDev> hv{make_view(*cam, 0)};
    PSG_CUDA(cudaMemcpyAsync(ctx->d_view1, hv.data(), sizeof(ViewDev), cudaMemcpyHostToDevice, ctx->stream));
    const RenderParams rp = make_params(ctx->cfg, lambda, 1.0);
    std::vector<int> vids{0};
    const int rc = bin_batch(ctx, ctx->d_view1, hv, vids, rp.cut, batch, bins, true, total);
    if (rc == kSplit)
        return fail(PSG_EINVAL, "render_view: " + std::to_string(*total) +
                                    " tile-plane bin entries, above the 32-bit limit");
    return rc;
}
// ---- host side of the drop-in calls. Their buffers are the reference's pageable
// host vectors; they go through one pinned staging area with multi-threaded host
// copies (a pageable cudaMemcpy is a single-threaded staged copy), and the 30-slot
// record lists cross PCIe as live records only: render_view packs them on the
// device and expands them into the caller's -1 padded layout on the host, backward
// packs them on the host and expands them on the device.
// Persistent host workers for the drop-in calls' copies and record (un)packing:
// spawning threads per call cost more than the copies at 640x480 (measured).
class HostPool {
public:
    static HostPool& get() {
        static HostPool pool;
        return pool;
    }
    size_t size() const { return workers_.size() + 1; }
    // run f(k) for k in [0, n) on the workers and the calling thread; returns when done
    void run(size_t n, const std::function<void(size_t)>& f) {
        if (n <= 1 || workers_.empty()) {
            for (size_t k = 0; k < n; ++k) f(k);
            return;
        }
        std::unique_lock<std::mutex> caller(call_mu_);  // one parallel region at a time
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &f;
            n_ = n;
            next_ = 0;
            pending_ = n;
            ++gen_;
        }
        cv_.notify_all();
        drain();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

private:
    HostPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned nw = std::min(15u, hw > 1 ? hw - 1 : 0u);
        for (unsigned i = 0; i < nw; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    void drain() {
        for (;;) {
            size_t k;
            const std::function<void(size_t)>* f;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (!job_ || next_ >= n_) return;
                k = next_++;
                f = job_;
            }
            (*f)(k);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_ && next_ < n_); });
                if (stop_) return;
                seen = gen_;
            }
            drain();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(size_t)>* job_ = nullptr;
    size_t n_ = 0, next_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

template <typename F>
void host_parallel(size_t n, size_t grain, const F& f) {
    HostPool& pool = HostPool::get();
    const size_t nt = std::min<size_t>(pool.size(), std::max<size_t>(1, n / std::max<size_t>(grain, 1)));
    if (nt <= 1) {
        f(size_t(0), n);
        return;
    }
    pool.run(nt, [&](size_t k) { f(n * k / nt, n * (k + 1) / nt); });
}

// dense arrays (maps, targets, dL/dmaps): through the pinned staging area with the
// pool's parallel copies (1), or straight from / to the caller's pageable buffers
// with the driver's staged copy (0). PSG_DROPIN_STAGING selects; default 0.
bool dense_staging() {
    static const bool on = [] {
        const char* e = std::getenv("PSG_DROPIN_STAGING");
        return e && e[0] == '1';
    }();
    return on;
}

void host_copy(void* dst, const void* src, size_t bytes) {
    host_parallel(bytes, size_t(512) << 10, [&](size_t a, size_t b) {
        std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    });
}

int ensure_staging(psg_context* ctx, size_t bytes) {
    if (bytes <= ctx->h_big_cap) return PSG_OK;
    if (ctx->h_big) {
        PSG_CUDA(cudaStreamSynchronize(ctx->stream));
        cudaFreeHost(ctx->h_big);
    }
    ctx->h_big = nullptr;
    ctx->h_big_cap = 0;
    const size_t cap = std::max(bytes, size_t(16) << 20);
    PSG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_big), cap, cudaHostAllocDefault));
    ctx->h_big_cap = cap;
    return PSG_OK;
}

__global__ void k_pack_records(const int* rec_prim, const unsigned short* rec_count, const long long* off,
                               int M, long long np, int* out) {
    const long long px = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (px >= np) return;
    const int c = min(int(rec_count[px]), M);
    for (int j = 0; j < c; ++j) out[off[px] + j] = rec_prim[px * M + j];
}

__global__ void k_unpack_records(const int* packed, const unsigned short* rec_count, const long long* off,
                                 int M, long long np, int* rec_prim) {
    const long long px = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (px >= np) return;
    const int c = min(int(rec_count[px]), M);
    for (int j = 0; j < M; ++j) rec_prim[px * M + j] = j < c ? packed[off[px] + j] : -1;
}

__global__ void k_count_to_ll(const unsigned short* rec_count, int M, long long np, long long* out) {
    const long long px = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (px < np) out[px] = min(int(rec_count[px]), M);
    if (px == np) out[px] = 0;
}

// exclusive scan of min(rec_count, M) into ctx->d_pack_off [np + 1] (device)
int record_offsets(psg_context* ctx, const unsigned short* d_count, int M, long long np) {
    int rc;
    if ((rc = grow(ctx->d_pack_off, ctx->pack_off_cap, 2 * size_t(np + 1)))) return rc;
    long long* cnt = ctx->d_pack_off + (np + 1);
    k_count_to_ll<<<unsigned((np + 256) / 256), 256, 0, ctx->stream>>>(d_count, M, np, cnt);
    size_t tmp = 0;
    PSG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, ctx->d_pack_off, np + 1, ctx->stream));
    if (tmp > ctx->cub_cap) {
        if (ctx->d_cub) cudaFree(ctx->d_cub);
        ctx->d_cub = nullptr;
        ctx->cub_cap = 0;
        PSG_CUDA(cudaMalloc(&ctx->d_cub, tmp));
        ctx->cub_cap = tmp;
    }
    tmp = ctx->cub_cap;
    PSG_CUDA(cub::DeviceScan::ExclusiveSum(ctx->d_cub, tmp, cnt, ctx->d_pack_off, np + 1, ctx->stream));
    return PSG_OK;
}

}  // namespace

extern "C" {

int psg_render_view(psg_context* ctx, const psg_camera* cam, double lambda, int keep_records,
                    double* depth, double* normal, double* alpha, int32_t* rec_prim,
                    uint16_t* rec_count) {
    Nvtx nvtx_range("psg.render_view");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (!cam || cam->width < 1 || cam->height < 1)  // renderer.cpp:233
        return fail(PSG_EINVAL, "render_view: empty view");
    if (cam->width > kMaxSide || cam->height > kMaxSide)
        return fail(PSG_EINVAL, "render_view: width and height must be <= 32767");
    if ((rc = check_cfg(ctx->cfg))) return rc;
    if (!depth || !normal || !alpha) return fail(PSG_EINVAL, "render_view: null map buffer");
    if (keep_records && (!rec_prim || !rec_count))
        return fail(PSG_EINVAL, "render_view: null record buffer");
    const size_t np = size_t(cam->width) * size_t(cam->height);
    const int M = ctx->cfg.max_records;
    cudaStream_t s = ctx->stream;
    if ((rc = grow(ctx->d_maps, ctx->maps_cap, np * 5))) return rc;
    if (keep_records) {
        if ((rc = grow(ctx->d_rec_prim, ctx->rec_prim_cap, np * size_t(M)))) return rc;
        if ((rc = grow(ctx->d_rec_count, ctx->rec_count_cap, np))) return rc;
    }
    if (ctx->P == 0) {  // no primitives: zero maps, empty records
        std::memset(depth, 0, np * 8);
        std::memset(normal, 0, np * 24);
        std::memset(alpha, 0, np * 8);
        if (keep_records) {
            for (size_t i = 0; i < np * size_t(M); ++i) rec_prim[i] = -1;
            std::memset(rec_count, 0, np * 2);
        }
        return PSG_OK;
    }
    Batch batch{};
    Bins bins{};
    int64_t total = 0;
    if ((rc = single_view_bins(ctx, cam, lambda, batch, bins, &total))) return rc;
    RasterIO io{};
    io.out_depth_d = ctx->d_maps;
    io.out_alpha_d = ctx->d_maps + np;
    io.out_normal_d = ctx->d_maps + 2 * np;
    io.rec_prim = ctx->d_rec_prim;
    io.rec_count = ctx->d_rec_count;
    io.stats = ctx->d_stats;
    const RenderParams rp = make_params(ctx->cfg, lambda, 1.0);
    launch_raster(ctx->precision, keep_records ? kFwdRecords : kFwdMaps, batch, ctx->d_geo,
                  ctx->d_geof, ctx->P, bins, rp, io, s, ctx->aux);
    PSG_CUDA(cudaGetLastError());
    // staging: maps (40 B/px) | counts (2 B/px, padded) | packed live records
    const size_t maps_b = np * 40, cnt_b = (np * 2 + 15) & ~size_t(15);
    long long n_live = 0;
    if (keep_records) {
        if ((rc = record_offsets(ctx, ctx->d_rec_count, M, (long long)np))) return rc;
        PSG_CUDA(cudaMemcpyAsync(&ctx->h_total[4], ctx->d_pack_off + np, 8, cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaStreamSynchronize(s));
        n_live = ctx->h_total[4];
        if ((rc = grow(ctx->d_pack, ctx->pack_cap, size_t(n_live) + 1))) return rc;
        k_pack_records<<<unsigned((np + 255) / 256), 256, 0, s>>>(ctx->d_rec_prim, ctx->d_rec_count,
                                                               ctx->d_pack_off, M, (long long)np, ctx->d_pack);
        PSG_CUDA(cudaGetLastError());
    }
    const size_t rec_b = keep_records ? cnt_b + size_t(n_live) * 4 : 0;
    const bool stage = dense_staging();
    if ((rc = ensure_staging(ctx, (stage ? maps_b : 0) + rec_b))) return rc;
    unsigned char* st = ctx->h_big;
    const size_t rec0 = stage ? maps_b : 0;
    if (stage) {
        PSG_CUDA(cudaMemcpyAsync(st, ctx->d_maps, maps_b, cudaMemcpyDeviceToHost, s));  // depth | alpha | normal
    } else {
        PSG_CUDA(cudaMemcpyAsync(depth, ctx->d_maps, np * 8, cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaMemcpyAsync(alpha, ctx->d_maps + np, np * 8, cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaMemcpyAsync(normal, ctx->d_maps + 2 * np, np * 24, cudaMemcpyDeviceToHost, s));
    }
    if (keep_records) {
        PSG_CUDA(cudaMemcpyAsync(st + rec0, ctx->d_rec_count, np * 2, cudaMemcpyDeviceToHost, s));
        if (n_live)
            PSG_CUDA(cudaMemcpyAsync(st + rec0 + cnt_b, ctx->d_pack, size_t(n_live) * 4, cudaMemcpyDeviceToHost, s));
    }
    PSG_CUDA(cudaStreamSynchronize(s));
    if (stage) {
        host_copy(depth, st, np * 8);
        host_copy(alpha, st + np * 8, np * 8);
        host_copy(normal, st + np * 16, np * 24);
    }
    if (keep_records) {
        const unsigned short* hc = reinterpret_cast<const unsigned short*>(st + rec0);
        const int* hp = reinterpret_cast<const int*>(st + rec0 + cnt_b);
        std::memcpy(rec_count, hc, np * 2);
        // expand into the caller's layout: live records, then -1 up to M per pixel
        const size_t nt = std::max<size_t>(1, std::min<size_t>(16, np / 16384));
        std::vector<long long> base(nt + 1, 0);
        for (size_t k = 0; k < nt; ++k) {
            long long c = 0;
            for (size_t px = np * k / nt; px < np * (k + 1) / nt; ++px) c += std::min<int>(hc[px], M);
            base[k + 1] = base[k] + c;
        }
        host_parallel(nt, 1, [&](size_t a, size_t b) {
            for (size_t k = a; k < b; ++k) {
                long long o = base[k];
                for (size_t px = np * k / nt; px < np * (k + 1) / nt; ++px) {
                    const int c = std::min<int>(hc[px], M);
                    int32_t* dst = rec_prim + px * size_t(M);
                    for (int j = 0; j < c; ++j) dst[j] = hp[o + j];
                    for (int j = c; j < M; ++j) dst[j] = -1;
                    o += c;
                }
            }
        });
    }
    return PSG_OK;
}

int psg_render_loss(psg_context* ctx, const psg_camera* cam, const float* td, const float* tn,
                    const double* depth, const double* normal, const double* alpha, double* loss,
                    double* d_depth, double* d_normal, double* d_alpha) {
    Nvtx nvtx_range("psg.render_loss");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (!cam || cam->width < 1 || cam->height < 1) return fail(PSG_EINVAL, "render_loss: empty view");
    if (cam->width > kMaxSide || cam->height > kMaxSide)
        return fail(PSG_EINVAL, "render_loss: width and height must be <= 32767");
    if (!td || !tn || !depth || !normal || !alpha || !loss || !d_depth || !d_normal)
        return fail(PSG_EINVAL, "render_loss: null buffer");
    const size_t np = size_t(cam->width) * size_t(cam->height);
    cudaStream_t s = ctx->stream;
    if ((rc = grow(ctx->d_maps, ctx->maps_cap, np * 5))) return rc;
    if ((rc = grow(ctx->d_t1, ctx->t1_cap, np * 4))) return rc;
    if ((rc = grow(ctx->d_g1, ctx->g1_cap, np * 5))) return rc;
    // targets (16 B/px) | maps (40 B/px) through the pinned staging area, or direct
    const bool stage = dense_staging();
    if (!stage) {
        PSG_CUDA(cudaMemcpyAsync(ctx->d_t1, td, np * 4, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_t1 + np, tn, np * 12, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_maps, depth, np * 8, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_maps + np, alpha, np * 8, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_maps + 2 * np, normal, np * 24, cudaMemcpyHostToDevice, s));
    } else {
        if ((rc = ensure_staging(ctx, np * 56))) return rc;
        unsigned char* st = ctx->h_big;
        PSG_CUDA(cudaStreamSynchronize(s));  // the staging area is free
        host_copy(st, td, np * 4);
        host_copy(st + np * 4, tn, np * 12);
        host_copy(st + np * 16, depth, np * 8);
        host_copy(st + np * 24, alpha, np * 8);
        host_copy(st + np * 32, normal, np * 24);
        PSG_CUDA(cudaMemcpyAsync(ctx->d_t1, st, np * 16, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_maps, st + np * 16, np * 40, cudaMemcpyHostToDevice, s));
    }
    ViewDev hv = make_view(*cam, 0);
    PSG_CUDA(cudaMemcpyAsync(ctx->d_view1, &hv, sizeof(ViewDev), cudaMemcpyHostToDevice, s));
    PSG_CUDA(cudaMemsetAsync(ctx->d_misc, 0, 4 * sizeof(unsigned long long), s));
    PSG_CUDA(cudaMemsetAsync(ctx->d_sums, 0, 2 * sizeof(double), s));
    const RenderParams rp = make_params(ctx->cfg, 1.0, 1.0);
    double* dA = d_alpha ? ctx->d_g1 + 4 * np : nullptr;
    launch_loss(ctx->d_view1, ctx->d_t1, ctx->d_t1 + np, ctx->d_maps, ctx->d_maps + 2 * np,
                ctx->d_maps + np, rp, cam->width, cam->height, ctx->d_g1, ctx->d_g1 + np, dA,
                ctx->d_sums, ctx->d_misc + 1, s);
    PSG_CUDA(cudaGetLastError());
    double sums[2];
    unsigned long long counts[2];
    // dL/d(depth | normal | alpha) back through the staging area (the H2D above has
    // been consumed once the stream reaches these copies)
    if (stage) {
        PSG_CUDA(cudaMemcpyAsync(ctx->h_big, ctx->d_g1, np * (d_alpha ? 40 : 32), cudaMemcpyDeviceToHost, s));
    } else {
        PSG_CUDA(cudaMemcpyAsync(d_depth, ctx->d_g1, np * 8, cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaMemcpyAsync(d_normal, ctx->d_g1 + np, np * 24, cudaMemcpyDeviceToHost, s));
        if (d_alpha) PSG_CUDA(cudaMemcpyAsync(d_alpha, dA, np * 8, cudaMemcpyDeviceToHost, s));
    }
    PSG_CUDA(cudaMemcpyAsync(sums, ctx->d_sums, 16, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaMemcpyAsync(counts, ctx->d_misc + 1, 16, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (stage) {
        host_copy(d_depth, ctx->h_big, np * 8);
        host_copy(d_normal, ctx->h_big + np * 8, np * 24);
        if (d_alpha) host_copy(d_alpha, ctx->h_big + np * 32, np * 8);
    }
    const double inv_d = counts[0] ? 1.0 / double(counts[0]) : 0.0;
    const double inv_n = counts[1] ? 1.0 / double(counts[1]) : 0.0;
    *loss = ctx->cfg.alpha1 * sums[1] * inv_n + ctx->cfg.alpha2 * sums[0] * inv_d;  // renderer.cpp:369
    return PSG_OK;
}

int psg_backward(psg_context* ctx, const psg_camera* cam, double lambda, int max_records,
                 const int32_t* rec_prim, const uint16_t* rec_count, const double* d_depth,
                 const double* d_normal, const double* d_alpha, double* grads, int64_t* bad_id) {
    Nvtx nvtx_range("psg.backward");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (!rec_count || !rec_prim)  // renderer.cpp:376-377
        return fail(PSG_EINVAL, "backward: forward pass ran without keep_records");
    if (!cam || cam->width < 1 || cam->height < 1) return fail(PSG_EINVAL, "backward: empty view");
    if (cam->width > kMaxSide || cam->height > kMaxSide)
        return fail(PSG_EINVAL, "backward: width and height must be <= 32767");
    if (max_records < 1 || max_records > kMaxRecordCap) return fail(PSG_EINVAL, "backward: bad max_records");
    if (!d_depth || !d_normal || !grads) return fail(PSG_EINVAL, "backward: null buffer");
    if (ctx->P == 0) return PSG_OK;
    const size_t np = size_t(cam->width) * size_t(cam->height);
    const size_t G = size_t(ctx->P) * 11;
    cudaStream_t s = ctx->stream;
    Batch batch{};
    Bins bins{};
    int64_t total = 0;
    if ((rc = single_view_bins(ctx, cam, lambda, batch, bins, &total))) return rc;
    if ((rc = grow(ctx->d_rec_prim, ctx->rec_prim_cap, np * size_t(max_records)))) return rc;
    if ((rc = grow(ctx->d_rec_count, ctx->rec_count_cap, np))) return rc;
    if ((rc = grow(ctx->d_g1, ctx->g1_cap, np * 5 + G))) return rc;
    // staging: dL/dmaps (40 B/px) | grads (88 B/plane) | counts (2 B/px, padded) |
    // live records packed on the host (the entries below min(count, M) of each pixel,
    // the only ones backward reads, renderer.cpp:409-433)
    const int M = max_records;
    const size_t nt = std::max<size_t>(1, std::min<size_t>(16, np / 16384));
    std::vector<long long> base(nt + 1, 0);
    for (size_t k = 0; k < nt; ++k) {
        long long c = 0;
        for (size_t px = np * k / nt; px < np * (k + 1) / nt; ++px) c += std::min<int>(rec_count[px], M);
        base[k + 1] = base[k] + c;
    }
    const long long n_live = base[nt];
    const bool stage = dense_staging();
    // staging: [dL/dmaps (40 B/px) | grads (88 B/plane)] when staged | counts | live records
    const size_t dm_b = stage ? np * 40 : 0, g_b = G * 8, cnt_b = (np * 2 + 15) & ~size_t(15);
    const size_t gs_b = stage ? g_b : 0;
    if ((rc = ensure_staging(ctx, dm_b + gs_b + cnt_b + size_t(n_live) * 4))) return rc;
    unsigned char* st = ctx->h_big;
    PSG_CUDA(cudaStreamSynchronize(s));  // the staging area is free
    double* dg = ctx->d_g1 + 5 * np;
    if (stage) {
        host_copy(st, d_depth, np * 8);
        host_copy(st + np * 8, d_normal, np * 24);
        if (d_alpha) host_copy(st + np * 32, d_alpha, np * 8);
        host_copy(st + dm_b, grads, g_b);
    } else {
        PSG_CUDA(cudaMemcpyAsync(ctx->d_g1, d_depth, np * 8, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_g1 + np, d_normal, np * 24, cudaMemcpyHostToDevice, s));
        if (d_alpha) PSG_CUDA(cudaMemcpyAsync(ctx->d_g1 + 4 * np, d_alpha, np * 8, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(dg, grads, g_b, cudaMemcpyHostToDevice, s));
    }
    std::memcpy(st + dm_b + gs_b, rec_count, np * 2);
    int32_t* hp = reinterpret_cast<int32_t*>(st + dm_b + gs_b + cnt_b);
    host_parallel(nt, 1, [&](size_t a, size_t b) {
        for (size_t k = a; k < b; ++k) {
            long long o = base[k];
            for (size_t px = np * k / nt; px < np * (k + 1) / nt; ++px) {
                const int c = std::min<int>(rec_count[px], M);
                const int32_t* src = rec_prim + px * size_t(M);
                for (int j = 0; j < c; ++j) hp[o + j] = src[j];
                o += c;
            }
        }
    });
    if (stage) {
        PSG_CUDA(cudaMemcpyAsync(ctx->d_g1, st, d_alpha ? dm_b : np * 32, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(dg, st + dm_b, g_b, cudaMemcpyHostToDevice, s));
    }
    PSG_CUDA(cudaMemcpyAsync(ctx->d_rec_count, st + dm_b + gs_b, np * 2, cudaMemcpyHostToDevice, s));
    if ((rc = grow(ctx->d_pack, ctx->pack_cap, size_t(n_live) + 1))) return rc;
    if (n_live)
        PSG_CUDA(cudaMemcpyAsync(ctx->d_pack, hp, size_t(n_live) * 4, cudaMemcpyHostToDevice, s));
    if ((rc = record_offsets(ctx, ctx->d_rec_count, M, (long long)np))) return rc;
    k_unpack_records<<<unsigned((np + 255) / 256), 256, 0, s>>>(ctx->d_pack, ctx->d_rec_count, ctx->d_pack_off, M,
                                                             (long long)np, ctx->d_rec_prim);
    PSG_CUDA(cudaGetLastError());
    BackwardIO io{};
    io.rec_prim = ctx->d_rec_prim;
    io.rec_count = ctx->d_rec_count;
    io.M = max_records;
    io.d_depth = ctx->d_g1;
    io.d_normal = ctx->d_g1 + np;
    io.d_alpha = d_alpha ? ctx->d_g1 + 4 * np : nullptr;
    io.grads = dg;
    const RenderParams rp = make_params(ctx->cfg, lambda, 1.0);
    launch_backward_records(ctx->precision, batch, ctx->d_geo, ctx->P, bins, rp, io, s);
    PSG_CUDA(cudaGetLastError());
    PSG_CUDA(cudaMemsetAsync(ctx->d_misc, 0xff, sizeof(unsigned long long), s));
    launch_finalize_grads(ctx->d_geo, dg, ctx->P, ctx->d_misc, s);
    unsigned long long first_bad = 0;
    if (stage) PSG_CUDA(cudaMemcpyAsync(st + dm_b, dg, g_b, cudaMemcpyDeviceToHost, s));
    else PSG_CUDA(cudaMemcpyAsync(grads, dg, g_b, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaMemcpyAsync(&first_bad, ctx->d_misc, 8, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    if (stage) host_copy(grads, st + dm_b, g_b);
    if (first_bad != ~0ull) {
        const int64_t id = ctx->ids[size_t(first_bad)];
        if (bad_id) *bad_id = id;
        return fail(PSG_ENONFINITE, "backward: non-finite gradient for primitive id " + std::to_string(id));
    }
    return PSG_OK;
}

int64_t psg_debug_bins(psg_context* ctx, const psg_camera* cam, double lambda, int32_t* offsets,
                       int32_t* items, int64_t cap) {
    if (check_ctx(ctx)) return -1;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (!cam || cam->width < 1 || cam->height < 1) return fail(PSG_EINVAL, "debug_bins: empty view"), -1;
    if (cam->width > kMaxSide || cam->height > kMaxSide) return fail(PSG_EINVAL, "debug_bins: view too large"), -1;
    const int T = ((cam->width + kTile - 1) / kTile) * ((cam->height + kTile - 1) / kTile);
    if (ctx->P == 0) {
        if (offsets) std::memset(offsets, 0, size_t(T + 1) * 4);
        return 0;
    }
    Batch batch{};
    Bins bins{};
    int64_t total = 0;
    if (single_view_bins(ctx, cam, lambda, batch, bins, &total)) return -1;
    launch_sort_bins(bins.offsets, bins.items, T, ctx->stream);
    if (offsets) cudaMemcpyAsync(offsets, bins.offsets, size_t(T + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (items && cap >= total)
        cudaMemcpyAsync(items, bins.items, size_t(total) * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return fail(PSG_ECUDA, "debug_bins failed"), -1;
    return total;
}

// ---- NCCL -----------------------------------------------------------------

int psg_nccl_unique_id(char* id_out) {
    if (!id_out) return fail(PSG_EINVAL, "null id buffer");
    const NcclApi& nc = nccl_api();
    if (!nc.ok) return fail(PSG_ENCCL, "libnccl.so.2 not found");
    ncclUniqueId id;
    const ncclResult_t r = nc.get_unique_id(&id);
    if (r != ncclSuccess) return fail(PSG_ENCCL, std::string("ncclGetUniqueId: ") + nc.error_string(r));
    static_assert(sizeof(ncclUniqueId) == PSG_NCCL_ID_BYTES, "nccl id size");
    std::memcpy(id_out, &id, sizeof id);
    return PSG_OK;
}

int psg_comm_init(psg_context* ctx, const char* id, int nranks, int rank) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (!id || nranks < 1 || rank < 0 || rank >= nranks) return fail(PSG_EINVAL, "comm_init: bad arguments");
    const NcclApi& nc = nccl_api();
    if (!nc.ok) return fail(PSG_ENCCL, "libnccl.so.2 not found");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    const ncclResult_t r = nc.comm_init_rank(&ctx->comm, nranks, uid, rank);
    if (r != ncclSuccess) return fail(PSG_ENCCL, std::string("ncclCommInitRank: ") + nc.error_string(r));
    ctx->rank = rank;
    ctx->world = nranks;
    return PSG_OK;
}

int psg_allreduce_grads(psg_context* ctx) {
    Nvtx nvtx_range("psg.allreduce_grads");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (!ctx->comm) return fail(PSG_EINVAL, "allreduce: no communicator");
    if (ctx->P == 0) return PSG_OK;
    const NcclApi& nc = nccl_api();
    // gradients, the step loss and the step-window guard count (every rank learns
    // that some rank must replay, and all replay together)
    const ncclResult_t r = nc.all_reduce(ctx->d_grads, ctx->d_grads, size_t(ctx->P) * 11 + 2,
                                         ncclDouble, ncclSum, ctx->comm, ctx->stream);
    if (r != ncclSuccess) return fail(PSG_ENCCL, std::string("ncclAllReduce: ") + nc.error_string(r));
    if (ctx->window_open) ctx->window_allreduced = true;
    return PSG_OK;
}

int psg_comm_destroy(psg_context* ctx) {
    if (!ctx || !ctx->comm) return PSG_OK;
    nccl_api().comm_destroy(ctx->comm);
    ctx->comm = nullptr;
    ctx->rank = 0;
    ctx->world = 1;
    return PSG_OK;
}

void* psg_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
    return p;
}

void psg_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"

// ---- device optimiser (Optimizer, optimizer.cpp) ---------------------------
namespace {

// order-independent hash of the parameter bits (XOR of per-element mixes)
__global__ void k_checksum(const double* c, const double* q, const double* r, int64_t P,
                           unsigned long long* out) {
    unsigned long long h = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 11 * P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = i < 3 * P ? c[i] : (i < 7 * P ? q[i - 3 * P] : r[i - 7 * P]);
        unsigned long long z = (unsigned long long)__double_as_longlong(x) + 0x9E3779B97F4A7C15ull * (i + 1);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        h ^= z ^ (z >> 31);
    }
    for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0 && h) atomicXor(out, h);
}

uint64_t splitmix64(uint64_t x) {  // optimizer.cpp:13-18
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// seeded_shuffle (optimizer.cpp:22-28) of iota(n) for one epoch
void epoch_order(uint64_t seed, int64_t epoch, int64_t n, std::vector<int64_t>& order) {
    order.resize(size_t(n));
    for (int64_t i = 0; i < n; ++i) order[size_t(i)] = i;
    uint64_t st = splitmix64(seed) ^ splitmix64(uint64_t(epoch));
    for (uint64_t i = uint64_t(n); i > 1; --i) {
        st = splitmix64(st);
        std::swap(order[size_t(i - 1)], order[size_t(st % i)]);
    }
}

int64_t view_for_slot(psg_context* ctx, uint64_t seed, int64_t slot) {  // optimizer.cpp:49-59
    const int64_t n = int64_t(ctx->h_views.size());
    const int64_t epoch = slot / n;
    if (epoch != ctx->epoch_cached || seed != ctx->epoch_seed ||
        int64_t(ctx->epoch_order.size()) != n) {
        epoch_order(seed, epoch, n, ctx->epoch_order);
        ctx->epoch_cached = epoch;
        ctx->epoch_seed = seed;
    }
    return ctx->epoch_order[size_t(slot % n)];
}

template <typename T>
int alloc_exact(T*& p, size_t n) {
    if (p) cudaFree(p);
    p = nullptr;
    PSG_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T)));
    return PSG_OK;
}

int optim_alloc(psg_context* ctx, size_t P) {
    int rc;
    if ((rc = alloc_exact(ctx->d_m, P * 11)) || (rc = alloc_exact(ctx->d_v, P * 11)) ||
        (rc = alloc_exact(ctx->d_step, P)) || (rc = alloc_exact(ctx->d_rgs, P * 4)) ||
        (rc = alloc_exact(ctx->d_rgc, P)))
        return rc;
    return PSG_OK;
}

int optim_zero(psg_context* ctx, bool adam, bool stats) {
    const size_t P = size_t(ctx->P);
    cudaStream_t s = ctx->stream;
    if (adam) {
        PSG_CUDA(cudaMemsetAsync(ctx->d_m, 0, P * 11 * 8, s));
        PSG_CUDA(cudaMemsetAsync(ctx->d_v, 0, P * 11 * 8, s));
        PSG_CUDA(cudaMemsetAsync(ctx->d_step, 0, P * 8, s));
    }
    if (stats) {
        PSG_CUDA(cudaMemsetAsync(ctx->d_rgs, 0, P * 4 * 8, s));
        PSG_CUDA(cudaMemsetAsync(ctx->d_rgc, 0, P * 8, s));
    }
    return PSG_OK;
}

// Optimizer(Scene, ...) (optimizer.cpp:32-40): zero Adam state and statistics
int ensure_optim(psg_context* ctx) {
    if (ctx->optim_ready) return PSG_OK;
    int rc;
    if ((rc = optim_alloc(ctx, size_t(ctx->P)))) return rc;
    if ((rc = optim_zero(ctx, true, true))) return rc;
    ctx->max_step = 0;
    ctx->iteration = 0;
    int64_t nid = 0;
    for (int64_t id : ctx->ids) nid = std::max(nid, id + 1);
    ctx->next_id = nid;
    ctx->optim_ready = true;
    return PSG_OK;
}

// bias-correction table pow(beta, s), s = 0..len-1, from the host libm exactly
// as adam_scalar_update evaluates it (optimizer.hpp:43-44)
constexpr int64_t kMaxAdamStep = int64_t(1) << 26;

int ensure_pow(psg_context* ctx, double b1, double b2, int64_t need) {
    if (ctx->d_pow && ctx->pow_len > need && ctx->pow_b1 == b1 && ctx->pow_b2 == b2) return PSG_OK;
    if (need > kMaxAdamStep + 1) return fail(PSG_EINVAL, "optimizer: Adam step counter above 2^26");
    const int64_t len = std::max<int64_t>(std::min<int64_t>(2 * need + 2, kMaxAdamStep + 2), 4096);
    std::vector<double> h;
    try {
        h.resize(size_t(2 * len));
    } catch (const std::bad_alloc&) {
        return fail(PSG_ENOMEM, "optimizer: bias-correction table allocation failed");
    }
    for (int64_t k = 0; k < len; ++k) {
        h[size_t(k)] = std::pow(b1, double(k));
        h[size_t(len + k)] = std::pow(b2, double(k));
    }
    int rc;
    if ((rc = alloc_exact(ctx->d_pow, size_t(2 * len)))) return rc;
    PSG_CUDA(cudaMemcpyAsync(ctx->d_pow, h.data(), h.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->pow_len = len;
    ctx->pow_b1 = b1;
    ctx->pow_b2 = b2;
    return PSG_OK;
}

OptimIO optim_io(psg_context* ctx) {
    OptimIO io{};
    io.P = ctx->P;
    io.center = ctx->d_center;
    io.rot = ctx->d_rot;
    io.radii = ctx->d_radii;
    io.m = ctx->d_m;
    io.v = ctx->d_v;
    io.step = ctx->d_step;
    io.rgs = ctx->d_rgs;
    io.rgc = ctx->d_rgc;
    io.grads = ctx->d_grads;
    io.pow1 = ctx->d_pow;
    io.pow2 = ctx->d_pow + ctx->pow_len;
    return io;
}

}  // namespace

void psg_default_optim_config(psg_optim_config* c) {  // optimizer.hpp:10-27, splatting.hpp:8-13
    if (!c) return;
    std::memset(c, 0, sizeof *c);
    c->lr_center = 0.001;
    c->lr_radii = 0.001;
    c->lr_rotation = 0.001;
    c->beta1 = 0.9;
    c->beta2 = 0.999;
    c->eps = 1e-8;
    c->split_interval = 1000;
    c->split_grad_threshold = 0.2;
    c->enable_split = 1;
    c->single_radii = 0;
    c->views_per_step = 1;
    c->seed = 0;
    c->radii_floor = 1e-4;
    c->lambda_base = 20.0;
    c->lambda_rate = 0.001;
    c->lambda_max = 300.0;
}

int64_t psg_view_for_slot(uint64_t seed, int64_t n_views, int64_t slot) {
    if (n_views <= 0 || slot < 0) return -1;
    std::vector<int64_t> order;
    epoch_order(seed, slot / n_views, n_views, order);
    return order[size_t(slot % n_views)];
}

int psg_optim_reset(psg_context* ctx, int64_t iteration, int64_t next_id) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    ctx->optim_ready = false;
    if ((rc = ensure_optim(ctx))) return rc;
    ctx->iteration = iteration;
    if (next_id >= 0) ctx->next_id = next_id;
    return PSG_OK;
}

int psg_set_grads(psg_context* ctx, const double* grads, double loss) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (ctx->P > 0 && !grads) return fail(PSG_EINVAL, "set_grads: null grads");
    if (ctx->P > 0)
        PSG_CUDA(cudaMemcpyAsync(ctx->d_grads, grads, size_t(ctx->P) * 11 * 8, cudaMemcpyHostToDevice,
                                 ctx->stream));
    if (ctx->d_grads) {
        PSG_CUDA(cudaMemcpyAsync(ctx->d_grads + size_t(ctx->P) * 11, &loss, 8, cudaMemcpyHostToDevice,
                                 ctx->stream));
        PSG_CUDA(cudaMemsetAsync(ctx->d_grads + size_t(ctx->P) * 11 + 1, 0, 8, ctx->stream));
        PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return PSG_OK;
}

int psg_optim_apply(psg_context* ctx, const psg_optim_config* cfg) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (!cfg) return fail(PSG_EINVAL, "optim_apply: null config");
    if ((rc = ensure_optim(ctx))) return rc;
    if (ctx->P == 0) return PSG_OK;
    if ((rc = ensure_pow(ctx, cfg->beta1, cfg->beta2, ctx->max_step + 1))) return rc;
    OptimParams c{};
    c.lr_center = cfg->lr_center;
    c.lr_radii = cfg->lr_radii;
    c.lr_rotation = cfg->lr_rotation;
    c.beta1 = cfg->beta1;
    c.beta2 = cfg->beta2;
    c.eps = cfg->eps;
    c.radii_floor = cfg->radii_floor;
    c.single_radii = cfg->single_radii != 0;
    launch_optim_apply(optim_io(ctx), c, ctx->stream);
    PSG_CUDA(cudaGetLastError());
    ctx->max_step += 1;
    return PSG_OK;
}

int psg_optim_step_local(psg_context* ctx, const psg_optim_config* cfg, int rank, int world) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (!cfg) return fail(PSG_EINVAL, "optim_step: null config");
    if (ctx->h_views.empty()) return fail(PSG_EINVAL, "optimizer: no views");
    if (cfg->views_per_step < 1) return fail(PSG_EINVAL, "optimizer: views_per_step < 1");
    if (world < 1 || rank < 0 || rank >= world) return fail(PSG_EINVAL, "optim_step: bad rank/world");
    if ((rc = ensure_optim(ctx))) return rc;
    const double lambda =
        psg_lambda_schedule(ctx->iteration, cfg->lambda_base, cfg->lambda_rate, cfg->lambda_max);
    const int V = cfg->views_per_step;
    // slot k of this iteration goes to rank k mod world
    std::vector<int32_t> vids;
    for (int k = 0; k < V; ++k) {
        const int64_t v = view_for_slot(ctx, cfg->seed, ctx->iteration * V + k);
        if (k % world == rank) vids.push_back(int32_t(v));
    }
    if ((rc = psg_zero_grads(ctx))) return rc;
    if (!vids.empty() &&
        (rc = psg_step(ctx, vids.data(), int(vids.size()), lambda, 1.0 / double(V), 0)))
        return rc;
    return PSG_OK;
}

int psg_optim_step_finish(psg_context* ctx, const psg_optim_config* cfg, double* loss_out) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (!cfg) return fail(PSG_EINVAL, "optim_step: null config");
    if ((rc = ensure_optim(ctx))) return rc;
    // tangent projection + finiteness (renderer.cpp:516-527) and the loss read-back
    // with a single synchronisation
    double loss = 0.0;
    if (ctx->P > 0) {
        cudaStream_t s = ctx->stream;
        for (int attempt = 0;; ++attempt) {
            PSG_CUDA(cudaMemsetAsync(ctx->d_misc, 0xff, sizeof(unsigned long long), s));
            launch_finalize_grads(ctx->d_geo, ctx->d_grads, ctx->P, ctx->d_misc, s);
            PSG_CUDA(cudaMemcpyAsync(ctx->h_total, ctx->d_misc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
            PSG_CUDA(cudaMemcpyAsync(ctx->h_total + 3, ctx->d_grads + size_t(ctx->P) * 11, 2 * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
            PSG_CUDA(cudaStreamSynchronize(s));
            double guard = 0.0;
            std::memcpy(&guard, ctx->h_total + 4, 8);
            if (ctx->window_open && guard != 0.0 && attempt == 0) {
                if ((rc = replay_window(ctx))) return rc;
                continue;
            }
            ctx->pending.clear();
            ctx->window_open = false;
            ctx->window_allreduced = false;
            break;
        }
        unsigned long long first_bad = 0;
        std::memcpy(&first_bad, ctx->h_total, sizeof first_bad);
        std::memcpy(&loss, ctx->h_total + 3, sizeof loss);
        if (first_bad != ~0ull) {
            const int64_t id = ctx->ids[size_t(first_bad)];
            return fail(PSG_ENONFINITE, "backward: non-finite gradient for primitive id " + std::to_string(id));
        }
    }
    if (!std::isfinite(loss)) {  // optimizer.cpp:83-89
        const double lambda =
            psg_lambda_schedule(ctx->iteration, cfg->lambda_base, cfg->lambda_rate, cfg->lambda_max);
        char msg[256];
        std::snprintf(msg, sizeof msg, "optimizer: non-finite loss %g at iteration %lld (lambda %g, %lld primitives)",
                      loss, (long long)ctx->iteration, lambda, (long long)ctx->P);
        return fail(PSG_ENONFINITE, msg);
    }
    if ((rc = psg_optim_apply(ctx, cfg))) return rc;
    ctx->iteration += 1;
    if (loss_out) *loss_out = loss;
    return PSG_OK;
}

int psg_optim_step(psg_context* ctx, const psg_optim_config* cfg, double* loss_out) {
    Nvtx nvtx_range("psg.optim_step");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = psg_optim_step_local(ctx, cfg, ctx->rank, ctx->world))) return rc;
    if (ctx->comm && (rc = psg_allreduce_grads(ctx))) return rc;
    if ((rc = psg_optim_step_finish(ctx, cfg, loss_out))) return rc;
    if (ctx->comm && cfg->check_ranks) {
        // SURVEY.md 8e guard: every rank must hold bit-identical parameters
        uint64_t c = 0;
        if ((rc = psg_params_checksum(ctx, &c))) return rc;
        uint64_t* d = nullptr;
        PSG_CUDA(cudaMalloc(&d, 2 * sizeof(uint64_t)));
        const uint64_t h[2] = {c, ~c};
        uint64_t r[2] = {0, 0};
        cudaMemcpyAsync(d, h, sizeof h, cudaMemcpyHostToDevice, ctx->stream);
        const NcclApi& nc = nccl_api();
        const ncclResult_t nr = nc.all_reduce(d, d, 2, ncclUint64, ncclMax, ctx->comm, ctx->stream);
        cudaMemcpyAsync(r, d, sizeof r, cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        cudaFree(d);
        if (nr != ncclSuccess) return fail(PSG_ENCCL, std::string("ncclAllReduce: ") + nc.error_string(nr));
        if (r[0] != c || ~r[1] != c)
            return fail(PSG_ENCCL, "optimizer: parameters diverged across ranks at iteration " +
                                       std::to_string(ctx->iteration - 1));
    }
    return PSG_OK;
}

namespace {

// Optimizer::run (optimizer.cpp:204-214) without a synchronisation per iteration:
// blocks of up to kRunBlock iterations are enqueued back to back (view choice and
// lambda come from the host schedule), each iteration's Adam is gated on the device
// by k_run_gate, and the host reads the block's losses once. An iteration that
// must not apply (capacity abort, non-finite gradient or loss) halts the block:
// every later Adam of the block is skipped, so the parameters are exactly those
// before the halted iteration, which then reruns on the synchronous path (replay
// with exact sizes, or the reference's exception). Split iterations run settled.
constexpr int kRunBlock = 64;

int optim_run_deferred(psg_context* ctx, const psg_optim_config* cfg, int64_t end_iteration, double* losses,
                       double* lambdas, int64_t* primitive_counts, int64_t capacity, int64_t* n_done) {
    int rc;
    int64_t k = 0;
    cudaStream_t s = ctx->stream;
    const int V = cfg->views_per_step;
    if ((rc = grow(ctx->d_runlog, ctx->runlog_cap, kRunBlock))) return rc;
    // PSG_TRACE_RUN=1: host timings of the settled split steps and the queued blocks
    static const bool trace = [] {
        const char* e = std::getenv("PSG_TRACE_RUN");
        return e && e[0] == '1';
    }();
    auto now_ms = [] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
            .count();
    };
    unsigned long long* halt = ctx->d_misc + 11;  // [11] halted iteration, [12] reason
    // steps queued after a halt skip their binning and rendering (k_bin_guard)
    struct HaltScope {
        psg_context* c;
        ~HaltScope() { c->run_halt = nullptr; }
    } halt_scope{ctx};
    int* gate = reinterpret_cast<int*>(ctx->d_misc + 13);
    OptimParams c{};
    c.lr_center = cfg->lr_center;
    c.lr_radii = cfg->lr_radii;
    c.lr_rotation = cfg->lr_rotation;
    c.beta1 = cfg->beta1;
    c.beta2 = cfg->beta2;
    c.eps = cfg->eps;
    c.radii_floor = cfg->radii_floor;
    c.single_radii = cfg->single_radii != 0;
    auto record = [&](int64_t row, double loss, double lambda) {
        if (row < capacity) {
            if (losses) losses[row] = loss;
            if (lambdas) lambdas[row] = lambda;
            if (primitive_counts) primitive_counts[row] = ctx->P;
        }
    };
    while (ctx->iteration < end_iteration) {
        const bool split_now = cfg->enable_split && cfg->split_interval > 0 && ctx->iteration != 0 &&
                               ctx->iteration % cfg->split_interval == 0;
        if (split_now || ctx->P == 0) {  // settled path for this iteration
            int64_t split = 0;
            const double tr0 = trace ? now_ms() : 0.0;
            if ((rc = psg_optim_maybe_split(ctx, cfg, &split))) return rc;
            const double lambda =
                psg_lambda_schedule(ctx->iteration, cfg->lambda_base, cfg->lambda_rate, cfg->lambda_max);
            double loss = 0.0;
            const double tr1 = trace ? now_ms() : 0.0;
            if ((rc = psg_optim_step(ctx, cfg, &loss))) return rc;
            if (trace)
                std::fprintf(stderr, "psg.run it %lld split %lld P %lld: maybe_split %.2f ms, step %.2f ms\n",
                             (long long)ctx->iteration - 1, (long long)split, (long long)ctx->P, tr1 - tr0,
                             now_ms() - tr1);
            record(k++, loss, lambda);
            if (n_done) *n_done = k;
            continue;
        }
        // the block ends before the next split iteration
        int64_t nb = std::min<int64_t>(kRunBlock, end_iteration - ctx->iteration);
        if (cfg->enable_split && cfg->split_interval > 0) {
            const int64_t next = (ctx->iteration / cfg->split_interval + 1) * cfg->split_interval;
            nb = std::min<int64_t>(nb, next - ctx->iteration);
        }
        const int64_t it0 = ctx->iteration;
        const double tb0 = trace ? now_ms() : 0.0;
        PSG_CUDA(cudaMemsetAsync(halt, 0xff, sizeof(unsigned long long), s));
        std::vector<double> lam(size_t(nb), 0.0);
        ctx->run_halt = halt;
        for (int64_t j = 0; j < nb; ++j) {
            const int64_t it = it0 + j;
            lam[size_t(j)] = psg_lambda_schedule(it, cfg->lambda_base, cfg->lambda_rate, cfg->lambda_max);
            std::vector<int> vids;
            for (int q = 0; q < V; ++q) {
                const int64_t v = view_for_slot(ctx, cfg->seed, it * V + q);
                if (q % ctx->world == ctx->rank) vids.push_back(int(v));
            }
            // psg_zero_grads + psg_step (optimizer.cpp:67-81), without host waits
            ctx->pending.clear();
            ctx->window_open = false;
            ctx->window_allreduced = false;
            PSG_CUDA(cudaMemsetAsync(ctx->d_grads, 0, (size_t(ctx->P) * 11 + 2) * sizeof(double), s));
            if (!vids.empty() && (rc = step_passes(ctx, vids, int(vids.size()), lam[size_t(j)], 1.0 / double(V), 0,
                                                   nullptr)))
                return rc;
            if (ctx->comm && (rc = psg_allreduce_grads(ctx))) return rc;
            PSG_CUDA(cudaMemsetAsync(ctx->d_misc, 0xff, sizeof(unsigned long long), s));
            launch_finalize_grads(ctx->d_geo, ctx->d_grads, ctx->P, ctx->d_misc, s);
            launch_run_gate(ctx->d_grads + size_t(ctx->P) * 11, ctx->d_misc, it, ctx->d_runlog + j, gate, halt, s);
            if ((rc = ensure_pow(ctx, cfg->beta1, cfg->beta2, ctx->max_step + 1))) return rc;
            OptimIO io = optim_io(ctx);
            io.gate = gate;
            launch_optim_apply(io, c, s);
            PSG_CUDA(cudaGetLastError());
            ctx->max_step += 1;  // an upper bound of the step counters (pow table size)
        }
        ctx->run_halt = nullptr;
        std::vector<double> blk_loss(static_cast<size_t>(nb));
        PSG_CUDA(cudaMemcpyAsync(ctx->h_total + 5, halt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaMemcpyAsync(blk_loss.data(), ctx->d_runlog, size_t(nb) * 8, cudaMemcpyDeviceToHost, s));
        const double tb1 = trace ? now_ms() : 0.0;
        PSG_CUDA(cudaStreamSynchronize(s));
        if (trace)
            std::fprintf(stderr, "psg.run block it %lld n %lld: enqueue %.2f ms, wait %.2f ms\n", (long long)it0,
                         (long long)nb, tb1 - tb0, now_ms() - tb1);
        ctx->pending.clear();
        ctx->window_open = false;
        ctx->window_allreduced = false;
        const unsigned long long h = uint64_t(ctx->h_total[5]);
        const int64_t good = h == ~0ull ? nb : int64_t(h) - it0;
        for (int64_t j = 0; j < good; ++j) record(k++, blk_loss[size_t(j)], lam[size_t(j)]);
        ctx->iteration = it0 + good;
        if (n_done) *n_done = k;
        if (good < nb) {
            // the halted iteration on the synchronous path: a capacity abort replays
            // with exact sizes; a non-finite gradient or loss raises the reference's error
            const double lambda =
                psg_lambda_schedule(ctx->iteration, cfg->lambda_base, cfg->lambda_rate, cfg->lambda_max);
            double loss = 0.0;
            if ((rc = psg_optim_step(ctx, cfg, &loss))) return rc;
            ctx->stats.replays += 1;
            record(k++, loss, lambda);
            if (n_done) *n_done = k;
        }
    }
    return PSG_OK;
}

}  // namespace

int psg_optim_run(psg_context* ctx, const psg_optim_config* cfg, int64_t end_iteration, double* losses,
                  double* lambdas, int64_t* primitive_counts, int64_t capacity, int64_t* n_done) {
    Nvtx nvtx_range("psg.optim_run");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (n_done) *n_done = 0;
    if (!cfg) return fail(PSG_EINVAL, "optim_run: null config");
    if (ctx->h_views.empty()) return fail(PSG_EINVAL, "optimizer: no views");
    if (cfg->views_per_step < 1) return fail(PSG_EINVAL, "optimizer: views_per_step < 1");
    if ((rc = check_cfg(ctx->cfg))) return rc;
    if ((rc = settle(ctx))) return rc;
    if ((rc = ensure_optim(ctx))) return rc;
    // the rank-consistency check needs a read-back every step: synchronous loop
    // (PSG_RUN_SYNC=1 forces it, for A/B measurements)
    static const bool force_sync = [] {
        const char* e = std::getenv("PSG_RUN_SYNC");
        return e && e[0] == '1';
    }();
    if (!(ctx->comm && cfg->check_ranks) && !force_sync)
        return optim_run_deferred(ctx, cfg, end_iteration, losses, lambdas, primitive_counts, capacity, n_done);
    int64_t k = 0;
    while (ctx->iteration < end_iteration) {  // optimizer.cpp:207-212
        int64_t split = 0;
        if ((rc = psg_optim_maybe_split(ctx, cfg, &split))) return rc;
        const double lambda =
            psg_lambda_schedule(ctx->iteration, cfg->lambda_base, cfg->lambda_rate, cfg->lambda_max);
        double loss = 0.0;
        if ((rc = psg_optim_step(ctx, cfg, &loss))) return rc;
        if (k < capacity) {
            if (losses) losses[k] = loss;
            if (lambdas) lambdas[k] = lambda;
            if (primitive_counts) primitive_counts[k] = ctx->P;
        }
        ++k;
        if (n_done) *n_done = k;
    }
    return PSG_OK;
}

int psg_optim_maybe_split(psg_context* ctx, const psg_optim_config* cfg, int64_t* n_split) {
    Nvtx nvtx_range("psg.maybe_split");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (!cfg) return fail(PSG_EINVAL, "maybe_split: null config");
    if (n_split) *n_split = 0;
    if (!cfg->enable_split || cfg->split_interval <= 0) return PSG_OK;  // optimizer.cpp:143-144
    if ((rc = ensure_optim(ctx))) return rc;
    if (ctx->iteration == 0 || ctx->iteration % cfg->split_interval != 0) return PSG_OK;
    const int64_t P = ctx->P;
    cudaStream_t s = ctx->stream;
    if (P > 0) {
        if ((rc = grow(ctx->d_split, ctx->split_cap, size_t(3 * P)))) return rc;
        int* axis = ctx->d_split;
        int* cnt = axis + P;
        int* pos = cnt + P;
        launch_split_mark(P, ctx->d_rgs, ctx->d_rgc, cfg->split_grad_threshold, axis, cnt, s);
        size_t tmp = 0;
        PSG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, pos, int(P), s));
        if (tmp > ctx->cub_cap) {
            if (ctx->d_cub) cudaFree(ctx->d_cub);
            ctx->d_cub = nullptr;
            ctx->cub_cap = 0;
            PSG_CUDA(cudaMalloc(&ctx->d_cub, tmp));
            ctx->cub_cap = tmp;
        }
        tmp = ctx->cub_cap;
        PSG_CUDA(cub::DeviceScan::ExclusiveSum(ctx->d_cub, tmp, cnt, pos, int(P), s));
        std::vector<int> h_axis(static_cast<size_t>(P));
        PSG_CUDA(cudaMemcpyAsync(h_axis.data(), axis, size_t(P) * sizeof(int), cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaStreamSynchronize(s));
        int64_t k = 0;
        for (int a : h_axis) k += a >= 0;
        if (k > 0) {
            const int64_t Q = P + k;
            if (Q >= (int64_t(1) << 26)) return fail(PSG_EINVAL, "maybe_split: too many planes (limit 2^26)");
            OptimIO src = optim_io(ctx), dst{};
            dst.P = Q;
            double *c = nullptr, *q = nullptr, *r = nullptr, *m = nullptr, *v = nullptr;
            long long* st = nullptr;
            if ((rc = alloc_exact(c, size_t(Q) * 3)) || (rc = alloc_exact(q, size_t(Q) * 4)) ||
                (rc = alloc_exact(r, size_t(Q) * 4)) || (rc = alloc_exact(m, size_t(Q) * 11)) ||
                (rc = alloc_exact(v, size_t(Q) * 11)) || (rc = alloc_exact(st, size_t(Q))))
                return rc;
            dst.center = c;
            dst.rot = q;
            dst.radii = r;
            dst.m = m;
            dst.v = v;
            dst.step = st;
            launch_split_write(src, dst, axis, pos, s);
            PSG_CUDA(cudaGetLastError());
            PSG_CUDA(cudaStreamSynchronize(s));
            cudaFree(ctx->d_center);
            cudaFree(ctx->d_rot);
            cudaFree(ctx->d_radii);
            cudaFree(ctx->d_m);
            cudaFree(ctx->d_v);
            cudaFree(ctx->d_step);
            ctx->d_center = c;
            ctx->d_rot = q;
            ctx->d_radii = r;
            ctx->plane_cap = size_t(Q) * 3;
            ctx->plane_cap_q = size_t(Q) * 4;
            ctx->plane_cap_r = size_t(Q) * 4;
            ctx->d_m = m;
            ctx->d_v = v;
            ctx->d_step = st;
            // ids: children claim next_id in primitive order (optimizer.cpp:190-191)
            std::vector<int64_t> ids;
            ids.reserve(size_t(Q));
            for (int64_t i = 0; i < P; ++i) {
                if (h_axis[size_t(i)] < 0) {
                    ids.push_back(ctx->ids[size_t(i)]);
                } else {
                    ids.push_back(ctx->next_id++);
                    ids.push_back(ctx->next_id++);
                }
            }
            ctx->ids.swap(ids);
            ctx->P = Q;
            if ((rc = alloc_exact(ctx->d_rgs, size_t(Q) * 4)) || (rc = alloc_exact(ctx->d_rgc, size_t(Q))))
                return rc;
            if ((rc = grow(ctx->d_geo, ctx->geo_cap, size_t(Q))) ||
                (rc = grow(ctx->d_geof, ctx->geof_cap, size_t(Q))) ||
                (rc = grow(ctx->d_grads, ctx->grads_cap, size_t(Q) * 11 + 2)))
                return rc;
            if (n_split) *n_split = k;
        }
    }
    // running means restart after every firing (optimizer.cpp:198-199)
    return optim_zero(ctx, false, true);
}

int psg_get_planes(psg_context* ctx, double* center, double* rotation, double* radii, int64_t* ids) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    const size_t P = size_t(ctx->P);
    cudaStream_t s = ctx->stream;
    if (P > 0) {
        if (center) PSG_CUDA(cudaMemcpyAsync(center, ctx->d_center, P * 3 * 8, cudaMemcpyDeviceToHost, s));
        if (rotation) PSG_CUDA(cudaMemcpyAsync(rotation, ctx->d_rot, P * 4 * 8, cudaMemcpyDeviceToHost, s));
        if (radii) PSG_CUDA(cudaMemcpyAsync(radii, ctx->d_radii, P * 4 * 8, cudaMemcpyDeviceToHost, s));
        PSG_CUDA(cudaStreamSynchronize(s));
    }
    if (ids) std::memcpy(ids, ctx->ids.data(), P * sizeof(int64_t));
    return PSG_OK;
}

int psg_optim_get_state(psg_context* ctx, double* m, double* v, int64_t* step, double* rgs,
                        int64_t* rgc, int64_t* iteration, int64_t* next_id) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = ensure_optim(ctx))) return rc;
    const size_t P = size_t(ctx->P);
    cudaStream_t s = ctx->stream;
    if (P > 0) {
        if (m) PSG_CUDA(cudaMemcpyAsync(m, ctx->d_m, P * 11 * 8, cudaMemcpyDeviceToHost, s));
        if (v) PSG_CUDA(cudaMemcpyAsync(v, ctx->d_v, P * 11 * 8, cudaMemcpyDeviceToHost, s));
        if (step) PSG_CUDA(cudaMemcpyAsync(step, ctx->d_step, P * 8, cudaMemcpyDeviceToHost, s));
        if (rgs) PSG_CUDA(cudaMemcpyAsync(rgs, ctx->d_rgs, P * 4 * 8, cudaMemcpyDeviceToHost, s));
        if (rgc) PSG_CUDA(cudaMemcpyAsync(rgc, ctx->d_rgc, P * 8, cudaMemcpyDeviceToHost, s));
    }
    PSG_CUDA(cudaStreamSynchronize(s));
    if (iteration) *iteration = ctx->iteration;
    if (next_id) *next_id = ctx->next_id;
    return PSG_OK;
}

int psg_optim_set_state(psg_context* ctx, const double* m, const double* v, const int64_t* step,
                        const double* rgs, const int64_t* rgc, int64_t iteration, int64_t next_id) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if ((rc = ensure_optim(ctx))) return rc;
    const size_t P = size_t(ctx->P);
    cudaStream_t s = ctx->stream;
    if (P > 0) {
        if (!m || !v || !step || !rgs || !rgc) return fail(PSG_EINVAL, "optim_set_state: null array");
        // the bias corrections read pow(beta, s) from a host table (ensure_pow)
        for (size_t i = 0; i < P; ++i)
            if (step[i] < 0 || step[i] > kMaxAdamStep)
                return fail(PSG_EINVAL, "optim_set_state: Adam step counter out of range [0, 2^26]");
        PSG_CUDA(cudaMemcpyAsync(ctx->d_m, m, P * 11 * 8, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_v, v, P * 11 * 8, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_step, step, P * 8, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_rgs, rgs, P * 4 * 8, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaMemcpyAsync(ctx->d_rgc, rgc, P * 8, cudaMemcpyHostToDevice, s));
        PSG_CUDA(cudaStreamSynchronize(s));
    }
    int64_t mx = 0;
    for (size_t i = 0; i < P; ++i) mx = std::max<int64_t>(mx, step[i]);
    ctx->max_step = mx;
    ctx->iteration = iteration;
    ctx->next_id = next_id;
    return PSG_OK;
}

int psg_merge_planes(psg_context* ctx, const double* scene_center, double normal_deg,
                     double merge_offset, double merge_adjacency, int use_adjacency,
                     int32_t* instance_of, double* inst_normal, double* inst_offset,
                     double* inst_area, int64_t* n_instances) {
    Nvtx nvtx_range("psg.merge_planes");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (!scene_center || !n_instances || (ctx->P > 0 && (!instance_of || !inst_normal ||
                                                          !inst_offset || !inst_area)))
        return fail(PSG_EINVAL, "merge_planes: bad arguments");
    const size_t P = size_t(ctx->P);
    std::vector<double> c(P * 3), q(P * 4), r(P * 4);
    if ((rc = psg_get_planes(ctx, c.data(), q.data(), r.data(), nullptr))) return rc;
    std::string err;
    if (psg::merge_planes_run(ctx->P, c.data(), q.data(), r.data(), ctx->ids.data(), scene_center,
                              normal_deg, merge_offset, merge_adjacency, use_adjacency, ctx->stream,
                              instance_of, inst_normal, inst_offset, inst_area, n_instances, &err))
        return fail(PSG_ECUDA, "merge_planes: " + err);
    return PSG_OK;
}

int psg_refresh_target_counts(psg_context* ctx) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    return refresh_counts(ctx);
}

int psg_init_from_depth(psg_context* ctx, int n_primitives, uint64_t seed, double radius_scale,
                        int64_t* n_out) {
    Nvtx nvtx_range("psg.init_from_depth");
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    if (n_out) *n_out = 0;
    if (n_primitives < 1) return fail(PSG_EINVAL, "init: n_primitives must be >= 1");
    if (ctx->h_views.empty()) return fail(PSG_EIO, "init: no valid depth pixels in any view");
    double *c = nullptr, *q = nullptr, *r = nullptr;
    long long k = 0;
    std::string err;
    const int st = psg::init_from_depth_run(ctx->d_views, int(ctx->h_views.size()), ctx->d_td, ctx->d_tn,
                                            ctx->total_px, n_primitives, seed, radius_scale, ctx->stream,
                                            &c, &q, &r, &k, &err);
    if (st == 3) return fail(PSG_EIO, err);  // std::runtime_error in the reference
    if (st) return fail(PSG_ECUDA, "init_from_depth: " + err);
    cudaFree(ctx->d_center);
    cudaFree(ctx->d_rot);
    cudaFree(ctx->d_radii);
    ctx->d_center = c;
    ctx->d_rot = q;
    ctx->d_radii = r;
    ctx->plane_cap = size_t(k) * 3;
    ctx->plane_cap_q = size_t(k) * 4;
    ctx->plane_cap_r = size_t(k) * 4;
    ctx->P = k;
    ctx->ids.resize(size_t(k));
    for (long long i = 0; i < k; ++i) ctx->ids[size_t(i)] = i;  // scene.claim_id() in order
    ctx->optim_ready = false;
    if ((rc = grow(ctx->d_geo, ctx->geo_cap, size_t(k))) || (rc = grow(ctx->d_geof, ctx->geof_cap, size_t(k))) ||
        (rc = grow(ctx->d_grads, ctx->grads_cap, size_t(k) * 11 + 2)))
        return rc;
    if (n_out) *n_out = k;
    return PSG_OK;
}

int psg_params_checksum(psg_context* ctx, uint64_t* out) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if (!out) return fail(PSG_EINVAL, "params_checksum: null out");
    *out = 0;
    if (ctx->P == 0) return PSG_OK;
    unsigned long long* d = reinterpret_cast<unsigned long long*>(ctx->d_misc + 6);
    PSG_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), ctx->stream));
    k_checksum<<<296, 256, 0, ctx->stream>>>(ctx->d_center, ctx->d_rot, ctx->d_radii, ctx->P, d);
    PSG_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    PSG_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = h;
    return PSG_OK;
}

int psg_set_deterministic(psg_context* ctx, int enable) {
    int rc;
    if ((rc = check_ctx(ctx))) return rc;
    std::lock_guard<std::recursive_mutex> ctx_lock(ctx->mu);
    if ((rc = settle(ctx))) return rc;
    ctx->deterministic = enable != 0;
    return PSG_OK;
}
