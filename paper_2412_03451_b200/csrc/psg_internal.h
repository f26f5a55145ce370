// Internal declarations shared by the CUDA translation units and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <stdint.h>

// Device bounds checks, compiled in only by the checked build (`make checks`,
// -DPSG_CHECKS): a failed check prints its location and traps, so the launch
// fails loudly with cudaErrorLaunchFailure. Free in the product build.
#ifdef PSG_CHECKS
#include <cstdio>
#define PSG_CHECK(cond)                                                                        \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("PSG_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,  \
                   __LINE__, int(blockIdx.x), int(threadIdx.x));                              \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define PSG_CHECK(cond) \
    do {                \
    } while (0)
#endif

namespace psg {

constexpr int kTile = 16;            // renderer.hpp:19 (tile_size), fixed on device
constexpr int kTilePix = kTile * kTile;
constexpr int kMaxRecordCap = 64;    // renderer.cpp:14
constexpr double kZClip = 1e-6;      // renderer.cpp:15

// View-independent plane geometry, fp64 (make_prim_views' frame part,
// renderer.cpp:46-50, geometry.cpp:10-40). 20 doubles = 160 B, AoS so one
// candidate fetch touches two 128 B lines.
struct PlaneGeo {
    double c[3], vx[3], vy[3], n[3], r[4], q[4];
};

// fp32 mirror of the view-independent plane data for fp32 arithmetic
// (avoids per-use fp64->fp32 conversions, which issue on the narrow XU pipe).
struct PlaneF {
    float n[3], vx[3], vy[3], q[4], r[4];
    float pad[3];
};

// One registered view. The ray basis is computed on the host in the exact
// order of ray_basis() (renderer.cpp:32-38).
struct ViewDev {
    double fx, fy, cx, cy;
    double R[9];  // rot_wc, row-major
    double t[3];
    double base[3], du[3], dv[3];
    double inv_d, inv_n;  // 1/count_d, 1/count_n (renderer.cpp:328-334)
    long long pix_off;    // offset of this view's targets, in pixels
    int W, H, tiles_x, tiles_y;
};

struct RenderParams {
    double lambda;
    double cut;      // splat_cut_margin(lambda, floor) * 1.05 (renderer.cpp:122), host glibc log
    double arg_cut;  // log(2/floor - 1) (renderer.cpp:248)
    double weight_floor, t_near, parallel_eps, alpha_floor, alpha1, alpha2;
    double view_scale;
    int max_records;
    int normalize_by_alpha;
};

// Per-batch description handed to the binning and raster kernels.
struct Batch {
    const ViewDev* views;  // all registered views (device)
    const int* vid;        // [n] view index per batch slot
    const int* tile_base;  // [n+1] first global tile of each batch slot
    int n;
    int max_tiles;  // max tiles of one view in the batch
};

// Binning outputs (CSR over the batch's tiles).
struct Bins {
    int* counts;     // [T+1]
    int* offsets;    // [T+1] exclusive scan of counts
    int* cursor;     // [T] scatter cursors
    int* items;      // plane indices
    short4* rects;   // [n*P] pixel rect (u0,u1,v0,v1) per (slot, plane); x>y = empty
    int2* big;       // crowded tiles (> 256 candidates): (batch slot, tile)
    int* n_big_dev;  // device counter of `big`
    int* n_heavy_dev;  // crowded tiles over 4x the resident cap, listed first (the rest from the end)
    int* n_light_dev;  // the others
    const unsigned long long* halt;  // deferred Optimizer::run: halted iteration (~0 = running), else null
    int big_cap;       // entries of `big`
    int n_big;       // host copy (synchronous binning), -1 = device only (async step)
    int* work_ctr;   // tile counter of the persistent resident kernel
    int* big_ctr;    // crowded-tile counter of the k_raster<BIG> CTAs
    unsigned long long* pair_px;  // += sum over tiles of |candidates| * |pixels| (Q_v)
    unsigned char* recs;      // prebuilt record blocks of the resident tiles (psg_raster.cu)
    struct TileDesc* desc;    // [n * max_tiles] work descriptors
    long long* units;         // [T+1] record-block size of each tile, 16-byte units
    long long* unit_off;      // [T+1] exclusive scan of units
    int* pair_tile;           // [pairs] batch tile of each bin entry (k_scatter)
    int* tile_slot;           // [T] batch slot of each batch tile (k_big_tiles)
    int n_pairs;              // host copy of the bin entry total; -1 = device only (async step)
    int T;                    // tiles of the batch
    long long items_cap;      // capacity of items / pair_tile
    unsigned long long* pairs64;  // [1] 64-bit bin-entry total (k_big_tiles)
    int* abort;               // [1] set by k_bin_guard when a capacity is exceeded: every later
                              // kernel of the step returns at once and the host replays it
};
// Work descriptor of one (slot, tile) item of the persistent rasteriser.
struct alignas(16) TileDesc {
    long long off16;  // record block offset in 16-byte units
    int n;            // candidates; 0 empty, -2 crowded (BIG launch), -3 outside the view
    int rows;         // image rows in the tile (target row copies)
    long long tgt;    // first target pixel of the tile (view pix_off + row0 * W + col0)
    int W;            // view width (target row pitch)
    int pad;
};
#ifndef PSG_BIG_LPT
#define PSG_BIG_LPT 1  // crowded tiles claimed longest first (two size classes)
#endif
#ifndef PSG_GEO_REC
#define PSG_GEO_REC 1  // resident records carry the plane geometry the exact test and backward read
#endif
constexpr int kRecUnitsPerPair = PSG_GEO_REC ? 18 : 9;  // = kRecUnits of psg_raster.cu (16-byte units)
#ifndef PSG_RES_CAP
#define PSG_RES_CAP 128  // tiles with up to this many candidates stay resident (<= 256)
#endif
constexpr int kResCapTiles = PSG_RES_CAP;  // = kResCap of psg_raster.cu

struct Stats {
    unsigned long long big_tiles;
    unsigned long long zviol;
    unsigned long long pair_px;  // pixel-candidate pairs (SURVEY.md 8d Q_v)
    unsigned long long live;     // composited records, first opaque one included (L_v)
    unsigned long long cull_checks;  // checked build: fp32-culled candidates re-tested exactly
    unsigned long long cull_miss;    // checked build: of those, accepted by the exact fp64 test
    unsigned long long pairs;        // bin entries (k_bin_guard)
    unsigned long long big;          // crowded tiles (k_bin_guard)
    unsigned long long probe[12];    // -DPSG_PROBE builds only: per-pixel work counters (psg_debug_probe)
};

// ---- psg_optim.cu (compiled with -fmad=false: bit-exact fp64) ----
struct OptimIO {
    int64_t P;
    double* center;   // [P*3]
    double* rot;      // [P*4]
    double* radii;    // [P*4]
    double* m;        // [P*11] Adam first moments
    double* v;        // [P*11] Adam second moments
    long long* step;  // [P]
    double* rgs;      // [P*4] radii_grad_sum
    long long* rgc;   // [P] radii_grad_count
    const double* grads;  // [P*11] finalized gradients
    const double* pow1;   // pow(beta1, s), s = 0..cap (host libm)
    const double* pow2;
    const int* gate;      // deferred Optimizer::run: apply only when *gate != 0 (null: always)
};
struct OptimParams {
    double lr_center, lr_radii, lr_rotation, beta1, beta2, eps, radii_floor;
    int single_radii;
};
void launch_optim_apply(const OptimIO& io, const OptimParams& c, cudaStream_t s);
// Deferred Optimizer::run: after each iteration's finalize, one thread decides
// whether Adam may apply (the reference checks loss finiteness before it,
// optimizer.cpp:83-89; a capacity abort or a non-finite gradient also stop the
// loop) and logs the loss. halt[0] = first halted iteration (~0 = running),
// halt[1] = reason (1 capacity abort, 2 non-finite gradient, 3 non-finite loss).
void launch_run_gate(const double* grads_tail /* loss, guard */, const unsigned long long* first_bad,
                     long long iteration, double* log_slot, int* gate, unsigned long long* halt,
                     cudaStream_t s);
void launch_split_mark(int64_t P, const double* rgs, const long long* rgc, double thr, int* axis,
                       int* cnt, cudaStream_t s);
void launch_split_write(const OptimIO& src, const OptimIO& dst, const int* axis, const int* pos,
                        cudaStream_t s);

// ---- psg_merge.cu (-fmad=false): merge_planes, pair test on the device ----
// Returns 0, or nonzero with *err set. Inputs are host arrays.
int merge_planes_run(int64_t P, const double* c, const double* q, const double* r,
                     const int64_t* ids, const double* scene_center, double normal_deg,
                     double merge_offset, double merge_adjacency, int use_adjacency,
                     cudaStream_t s, int32_t* instance_of, double* inst_normal,
                     double* inst_offset, double* inst_area, int64_t* n_inst, std::string* err);

// ---- psg_init.cu (-fmad=false): init_from_depth over the resident targets ----
// On success *center/*rot/*radii are fresh device arrays of *k_out primitives.
int init_from_depth_run(const ViewDev* d_views, int n_views, const float* td, const float* tn,
                        long long n_px, int k, uint64_t seed, double radius_scale, cudaStream_t s,
                        double** center, double** rot, double** radii, long long* k_out,
                        std::string* err);

// ---- psg_binning.cu (compiled with -fmad=false: bit-exact fp64) ----
void launch_plane_setup(const double* center, const double* rot, const double* radii, int64_t n,
                        PlaneGeo* out, PlaneF* outf, cudaStream_t s);
void launch_rect_count(const Batch& b, const PlaneGeo* planes, int64_t P, double cut, Bins bins,
                       cudaStream_t s);
void launch_scatter(const Batch& b, int64_t P, Bins bins, cudaStream_t s);
// compact the crowded tiles (count > threshold) into bins.big
void launch_big_tiles(const Batch& b, Bins bins, int threshold, cudaStream_t s);
// after the scans: capacity check of an async step (abort flag, needed sizes, overflow
// count in the gradient buffer's guard slot) and the pair / crowded-tile statistics
void launch_bin_guard(const Bins& bins, long long recs_cap16, long long pair_limit,
                      unsigned long long* need, double* overflow, Stats* st, cudaStream_t s);
void launch_sort_bins(const int* offsets, int* items, int T, cudaStream_t s);  // ascending per tile
void launch_render_gt(const ViewDev* views, int n_views, const double* faces, int n_faces,
                      float* td, float* tn, int max_pixels, cudaStream_t s);
void launch_target_counts(const ViewDev* views, int n_views, const float* td, const float* tn,
                          unsigned long long* counts /* 2 per view */, cudaStream_t s);

// ---- psg_raster.cu ----
// kFusedDet = kFused in deterministic mode (its own instantiation, so the default
// kernel carries none of the partial-buffer code)
enum RasterMode { kFused = 0, kFwdMaps = 1, kFwdRecords = 2, kFusedDet = 3 };

struct RasterIO {
    // targets (fused)
    const float* td;
    const float* tn;
    // map outputs: f32 batch maps (fused, optional) or f64 single-view maps
    float* out_depth_f;
    float* out_normal_f;
    float* out_alpha_f;
    double* out_depth_d;
    double* out_normal_d;
    double* out_alpha_d;
    long long map_stride;  // pixels per batch slot in the f32 batch maps
    // records (kFwdRecords)
    int* rec_prim;
    unsigned short* rec_count;
    // gradients / loss (fused)
    double* grads;      // [P*11]
    double* view_loss;  // [n*2]: sum_depth, sum_normal (raw, pre-normalisation)
    int do_backward;
    int tma_targets;  // fused: targets rows are 16-byte aligned (every W % 4 == 0): TMA-staged
    double* det_grads;  // deterministic mode: [pairs * 8 warps * 11] partials (valid where det_mask says), else null
    double* det_loss;   // deterministic mode: [tiles * 8 warps * 2] loss partials, else null
    unsigned* det_mask; // deterministic mode: [pairs] bit w set once warp w wrote its partial
    Stats* stats;
};

// Second stream for the crowded-tile launch (forked from / joined into s).
struct AuxStream {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
void launch_raster(int precision, RasterMode mode, const Batch& b, const PlaneGeo* planes,
                   const PlaneF* planesf, int64_t P, const Bins& bins, const RenderParams& rp,
                   const RasterIO& io, cudaStream_t s, const AuxStream& aux);

struct BackwardIO {
    const int* rec_prim;
    const unsigned short* rec_count;
    int M;
    const double* d_depth;
    const double* d_normal;
    const double* d_alpha;  // may be null
    double* grads;
};
void launch_backward_records(int precision, const Batch& b, const PlaneGeo* planes, int64_t P,
                             const Bins& bins, const RenderParams& rp, const BackwardIO& io,
                             cudaStream_t s);

void launch_loss(const ViewDev* view, const float* td, const float* tn, const double* depth,
                 const double* normal, const double* alpha, const RenderParams& rp, int W, int H,
                 double* d_depth, double* d_normal, double* d_alpha, double* sums /* 2 */,
                 unsigned long long* counts /* 2 */, cudaStream_t s);

// deterministic mode: fixed-order reductions of the partials (bins.items sorted
// by plane with their bin-entry order kept)
void launch_det_reduce(const int* sorted_pid, const int* sorted_pair, int64_t n_pairs, int64_t P,
                       const double* det_grads, const unsigned* det_mask, double* grads, const Batch& b,
                       const double* det_loss,
                       double* view_loss, cudaStream_t s);
void launch_finalize_grads(const PlaneGeo* planes, double* grads, int64_t n,
                           unsigned long long* first_bad, cudaStream_t s);

}  // namespace psg
