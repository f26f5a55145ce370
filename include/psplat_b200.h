/* psplat_b200 — B200-native (sm_100a) plane-splat hot path behind a C ABI.
 *
 * Drop-in boundary for psplat::Renderer (reference: proj/core/include/psplat/
 * renderer.hpp:92-117, proj/core/src/renderer.cpp:231-528). Plain pointers and
 * sizes only; no CUDA, Eigen or torch types cross this boundary.
 *
 * Every entry point returns a status code (PSG_OK on success). The message of
 * the last failure on the calling thread is available from psg_last_error().
 * Status codes mirror the reference's exceptions:
 *   PSG_EINVAL     <- std::invalid_argument   (renderer.cpp:233-235,320-321,376-377)
 *   PSG_ENONFINITE <- std::runtime_error "backward: non-finite gradient for
 *                     primitive id N"          (renderer.cpp:521-526)
 * Host-pointer arguments are ordinary (pageable) or pinned host memory; calls
 * that return host data synchronise the context stream before returning.
 * Threading: the reference's Renderer methods are const and may be called from
 * several threads. Calls on one psg_context from several host
 * threads are serialised by a per-context lock; their device work is ordered on
 * the context stream. Use one context per GPU (or per stream) for concurrency.
 *
 * Layout conventions (all match the reference's in-memory layouts):
 *   planes  : SoA, center[n*3], rotation[n*4] (w,x,y,z; renormalised on device as
 *             geometry.cpp:19-21), radii[n*4] (r_x+, r_x-, r_y+, r_y-), ids[n]
 *   maps    : depth[H*W], normal[H*W*3] (interleaved), alpha[H*W] (renderer.hpp:33-46)
 *   records : rec_prim[H*W*M] (int32, -1 padded), rec_count[H*W] (uint16)
 *   grads   : grads[n*11] = d_center(3), d_rotation(4), d_radii(4) per plane,
 *             the PrimGrad order of renderer.hpp:56-60
 *   targets : depth f32[H*W] (<= 0 invalid), normal f32[H*W*3] (0-vector invalid)
 */
#ifndef PSPLAT_B200_H
#define PSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSG_ABI_VERSION 4

enum psg_status {
    PSG_OK = 0,
    PSG_EINVAL = 1,
    PSG_ECUDA = 2,
    PSG_ENONFINITE = 3,
    PSG_ENCCL = 4,
    PSG_ENOMEM = 5,
    PSG_EIO = 6 /* dataset / map file errors (the reference's std::runtime_error) */
};

/* Arithmetic of the rasteriser / backward. Binning is always fp64 (bit-exact
 * with renderer.cpp:71-147); PSG_FP64 reproduces the reference's fp64 maths,
 * PSG_FP32 is the throughput mode. */
enum psg_precision { PSG_FP32 = 0, PSG_FP64 = 1, PSG_MIXED = 2 };

/* psplat::RenderConfig (renderer.hpp:10-21); `threads` is accepted and ignored. */
typedef struct {
    int32_t max_records;        /* M, <= 64 (renderer.cpp:14,234-235) */
    int32_t normalize_by_alpha; /* bool */
    int32_t tile_size;          /* must be 16 on device */
    int32_t threads;
    double weight_floor;
    double t_near;
    double parallel_eps;
    double alpha_floor;
    double alpha1;
    double alpha2;
} psg_render_config;

/* psplat::CameraView without its targets (geometry.hpp:51-67). rot_wc row-major. */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double rot_wc[9];
    double t_wc[3];
} psg_camera;

typedef struct psg_context psg_context;

/* Counters of the batched psg_step path, summed since psg_create or the last
 * psg_reset_stats (for roofline reporting). */
typedef struct {
    int64_t views;          /* views processed */
    int64_t pixels;         /* sum of W*H */
    int64_t tiles;          /* 16x16 tile slots binned */
    int64_t pairs;          /* (tile, plane) bin entries = sum of candidate-list lengths */
    int64_t big_tiles;      /* crowded tiles rendered by the streaming launch */
    int64_t zbound_violations; /* must be 0: depth-bound early-exit contract check */
    int64_t pixel_pairs;    /* Q_v summed: sum over tiles of |candidates| * |pixels| */
    int64_t live_records;   /* L_v summed: composited records per pixel, first opaque included */
    /* checked build only (libpsplat_b200_checks.so, -DPSG_CHECKS): every candidate the
     * fp32 cull (or the per-pixel footprint rect) rejects in the exact modes is
     * re-tested with the exact fp64 test; misses must be 0. Both 0 in the product build. */
    int64_t cull_checks;
    int64_t cull_misses;
    /* psg_step never synchronises; a step whose bins outgrow the buffers earlier
     * steps sized (or pass pair_limit) aborts on the device and is replayed with
     * exact sizes by the next result-reading call. Replayed step windows: */
    int64_t replays;
} psg_stats;

const char* psg_last_error(void);
int psg_abi_version(void);
void psg_default_config(psg_render_config* cfg);
/* lambda = min(base * exp(-(1 - rate*ite)), max)  (splatting.cpp:7-10) */
double psg_lambda_schedule(int64_t ite, double base, double rate, double lmax);

/* ---- context ------------------------------------------------------------ */
int psg_create(int device, int precision, psg_context** out);
int psg_destroy(psg_context* ctx);
/* Launch on `stream` (a cudaStream_t passed as void*); NULL = the context's own. */
int psg_set_stream(psg_context* ctx, void* stream);
void* psg_get_stream(psg_context* ctx);
int psg_set_config(psg_context* ctx, const psg_render_config* cfg);
int psg_synchronize(psg_context* ctx);

/* Upload the plane set (Scene::primitives). Host pointers; ids may be NULL. */
int psg_set_planes(psg_context* ctx, int64_t n, const double* center, const double* rotation,
                   const double* radii, const int64_t* ids);
int64_t psg_num_planes(psg_context* ctx);

/* ---- drop-in Renderer calls (one view, host buffers) ---------------------- */
/* Renderer::render_view (renderer.cpp:231-317). Maps are written as f64 like
 * RenderedMaps; rec_prim/rec_count are written when keep_records != 0 and then
 * hold the reference's full per-pixel lists (M nearest, (z, prim) ascending). */
int psg_render_view(psg_context* ctx, const psg_camera* cam, double lambda, int keep_records,
                    double* depth, double* normal, double* alpha, int32_t* rec_prim,
                    uint16_t* rec_count);
/* Renderer::render_loss (renderer.cpp:319-371). d_alpha may be NULL. */
int psg_render_loss(psg_context* ctx, const psg_camera* cam, const float* target_depth,
                    const float* target_normal, const double* depth, const double* normal,
                    const double* alpha, double* loss, double* d_depth, double* d_normal,
                    double* d_alpha);
/* Renderer::backward (renderer.cpp:373-528): grads[n*11] is accumulated into
 * (+=), then tangent-projected and finiteness-checked as the reference does.
 * On PSG_ENONFINITE, *bad_id (if non-NULL) receives the primitive id. */
int psg_backward(psg_context* ctx, const psg_camera* cam, double lambda, int max_records,
                 const int32_t* rec_prim, const uint16_t* rec_count, const double* d_depth,
                 const double* d_normal, const double* d_alpha, double* grads,
                 int64_t* bad_id);

/* ---- resident views and the fused batched step (the hot path) ------------- */
/* Register views and copy their targets to HBM (targets may be NULL and filled
 * later by psg_update_targets or psg_render_ground_truth). Replaces any
 * previous view set. Per-view valid-target counts (renderer.cpp:328-332) are
 * computed once here, since targets are static. */
int psg_set_views(psg_context* ctx, int n_views, const psg_camera* cams,
                  const float* target_depth, const float* target_normal);
/* Re-upload targets of views [first, first+count) from host memory, async on
 * the stream (pinned memory gives full PCIe bandwidth). */
int psg_update_targets(psg_context* ctx, int first, int count, const float* target_depth,
                       const float* target_normal);
/* Download the targets of one view (testing). */
int psg_get_targets(psg_context* ctx, int view, float* target_depth, float* target_normal);
/* Render exact synthetic targets for all registered views on the device
 * (synthetic.cpp:144-175 semantics, fp64): faces are 15 doubles each
 * (center 3, u 3, v 3, half_u, half_v, normal 3, instance id). */
int psg_render_ground_truth(psg_context* ctx, int n_faces, const double* faces);

enum psg_step_flags {
    PSG_STEP_WRITE_MAPS = 1, /* keep f32 maps of the batch for psg_read_step_maps */
    PSG_STEP_NO_BACKWARD = 2 /* forward + loss only */
};
/* Optimizer::step's view loop (optimizer.cpp:67-81) fused: for each listed
 * view, forward + L1 loss + backward with loss and dL/dmaps scaled by
 * view_scale; plane gradients accumulate into the context's device buffer.
 * Asynchronous on the context stream. */
int psg_step(psg_context* ctx, const int32_t* view_ids, int n, double lambda, double view_scale,
             int flags);
/* The same step with the views' targets supplied from host memory (the
 * reference-facing form: CameraView carries its targets): views
 * [first, first+count) of the registered set, targets concatenated in that
 * order. Copies run on a separate stream in chunks of chunk_views views and
 * overlap the fused compute of the chunks already resident (pinned memory gives
 * full PCIe bandwidth). Per-view valid-target counts are the ones registered
 * with psg_set_views / psg_render_ground_truth. */
int psg_step_host(psg_context* ctx, int first, int count, double lambda, double view_scale,
                  int flags, const float* target_depth, const float* target_normal,
                  int chunk_views);
int psg_zero_grads(psg_context* ctx);
/* Deterministic mode: psg_step writes per-(bin entry, warp)
 * gradient and per-(tile, warp) loss partials and reduces them in a fixed order,
 * so repeated steps (and resumed runs) are bitwise reproducible; costs one
 * zeroed partial buffer of 704 B per bin entry and a sort. Default off (fp64
 * atomics: run-to-run spread ~1e-15 relative). */
int psg_set_deterministic(psg_context* ctx, int enable);
/* Tangent projection of d_rotation + finiteness check over the accumulated
 * gradients (renderer.cpp:516-527), once per step. Synchronises. */
int psg_finalize_grads(psg_context* ctx, int64_t* bad_id);
/* Copy accumulated grads (n*11 f64) and the summed loss to the host (sync). */
int psg_read_grads(psg_context* ctx, double* grads, double* loss);
/* Per-view loss of the last step (n values, view order of the psg_step call). */
int psg_read_view_losses(psg_context* ctx, double* losses, int n);
int psg_read_step_maps(psg_context* ctx, int k, float* depth, float* normal, float* alpha);
int psg_get_stats(psg_context* ctx, psg_stats* out);
/* Largest number of (tile, plane) bin entries one binning pass may hold (default and
 * maximum 2^31 - 1: the CSR offsets are 32-bit). A step over more is split into view
 * groups that fit; a single view above it fails with PSG_EINVAL. Lowered by tests. */
int psg_set_pair_limit(psg_context* ctx, int64_t limit);
int psg_reset_stats(psg_context* ctx);
/* Debug builds compiled with -DPSG_PROBE: 12 per-pixel work counters (see psg_api.cu). */
int psg_debug_probe(psg_context* ctx, uint64_t* out12);
/* Time the rasteriser launches with CUDA events on the context stream (for the
 * roofline's per-launch duration). psg_get_kernel_ms synchronises, returns the
 * summed milliseconds of the launches recorded since timing was enabled (or
 * since the previous call) and resets the sum. */
int psg_set_timing(psg_context* ctx, int enable);
int psg_get_kernel_ms(psg_context* ctx, double* raster_ms, int* launches);

/* ---- device optimiser (Optimizer, optimizer.cpp) ---- */
/* OptimConfig (optimizer.hpp:10-27) + the SplatParams lambda schedule
 * (splatting.hpp:8-13). The merge settings are not used on this path. */
typedef struct {
    double lr_center, lr_radii, lr_rotation;
    double beta1, beta2, eps;
    int64_t split_interval;
    double split_grad_threshold;
    int32_t enable_split;
    int32_t single_radii;
    int32_t views_per_step;
    int32_t check_ranks; /* with a communicator: verify bit-identical parameters after
                            every step (SURVEY.md 8e guard); PSG_ENCCL on divergence */
    uint64_t seed;
    double radii_floor;
    double lambda_base, lambda_rate, lambda_max;
} psg_optim_config;

void psg_default_optim_config(psg_optim_config* cfg);
/* Optimizer::view_for_slot (optimizer.cpp:49-59): seeded epoch shuffle. */
int64_t psg_view_for_slot(uint64_t seed, int64_t n_views, int64_t slot);
/* The optimiser state (Adam moments and steps, radii gradient sums, iteration,
 * next id) lives on the device next to the planes. psg_set_planes starts a
 * fresh state, as constructing an Optimizer does (optimizer.cpp:32-40);
 * psg_optim_reset does so explicitly (next_id < 0: max(id) + 1). */
int psg_optim_reset(psg_context* ctx, int64_t iteration, int64_t next_id);
/* Optimizer::step (optimizer.cpp:61-98) on the device: lambda from the
 * schedule, views_per_step views from view_for_slot (slot k on rank k mod N
 * when a communicator is set, then psg_allreduce_grads), forward + loss +
 * backward, tangent projection and finiteness check, radii gradient sums, Adam,
 * quaternion renormalisation, radii clamp. Reads only the loss back. */
int psg_optim_step(psg_context* ctx, const psg_optim_config* cfg, double* loss);
/* The same step in two halves around a caller-provided all-reduce (e.g. through
 * torch.distributed): _local renders this rank's slots (k mod world == rank) into
 * the context's gradient buffer (loss in its last slot, see psg_read_grads /
 * psg_set_grads); _finish finalises, checks the loss and applies Adam. */
int psg_optim_step_local(psg_context* ctx, const psg_optim_config* cfg, int rank, int world);
int psg_optim_step_finish(psg_context* ctx, const psg_optim_config* cfg, double* loss);
/* Order-independent 64-bit hash of the parameter bits (rank consistency checks). */
int psg_params_checksum(psg_context* ctx, uint64_t* out);
/* optimizer.cpp:84-95 alone, on the gradients already in the context (from
 * psg_step + psg_finalize_grads, or psg_set_grads). */
int psg_optim_apply(psg_context* ctx, const psg_optim_config* cfg);
/* Optimizer::maybe_split (optimizer.cpp:142-202) as a device compaction; the
 * plane count grows by *n_split. */
int psg_optim_maybe_split(psg_context* ctx, const psg_optim_config* cfg, int64_t* n_split);
/* Optimizer::run (optimizer.cpp:204-214): maybe_split + step until the iteration
 * counter reaches `end_iteration`, in native code. Row k of the log (when the
 * arrays are non-NULL, `capacity` rows at most) is the LossLogRow of the k-th
 * step run: its loss, its lambda and the primitive count after it. `n_done`
 * receives the number of steps run (also on error). */
int psg_optim_run(psg_context* ctx, const psg_optim_config* cfg, int64_t end_iteration, double* losses,
                  double* lambdas, int64_t* primitive_counts, int64_t capacity, int64_t* n_done);
/* Replace the accumulated gradients (n*11 f64) and loss (external gradients). */
int psg_set_grads(psg_context* ctx, const double* grads, double loss);
/* Download the current planes (n from psg_num_planes). Any pointer may be NULL. */
int psg_get_planes(psg_context* ctx, double* center, double* rotation, double* radii, int64_t* ids);
/* Optimiser state: m, v [n*11], step [n], radii_grad_sum [n*4], count [n]. */
int psg_optim_get_state(psg_context* ctx, double* m, double* v, int64_t* step, double* rgs,
                        int64_t* rgc, int64_t* iteration, int64_t* next_id);
int psg_optim_set_state(psg_context* ctx, const double* m, const double* v, const int64_t* step,
                        const double* rgs, const int64_t* rgc, int64_t iteration, int64_t next_id);

/* merge_planes (optimizer.cpp:236-299) on the current planes: the O(P^2) pair
 * test (normal gate, offset gate, adjacency via rect_distance) on the device,
 * components and instance summaries on the host, bit-identical to the
 * reference. instance_of[P] indexes the instances in the reference's order
 * (area descending, then smallest member id); per instance normal[3], offset,
 * area (arrays of capacity P). */
int psg_merge_planes(psg_context* ctx, const double* scene_center, double normal_deg,
                     double merge_offset, double merge_adjacency, int use_adjacency,
                     int32_t* instance_of, double* inst_normal, double* inst_offset,
                     double* inst_area, int64_t* n_instances);

/* ---- PSMP dataset loader (dataio.cpp:19-201) ---------
 * root/cameras.txt + root/depth/<id>.f32 + root/normal/<id>.f32. psg_dataset_open
 * parses the cameras (every stride-th line) and checks every map header;
 * psg_dataset_read reads and validates the targets of views [first, first+count)
 * into caller buffers (concatenated in view order) with `threads` reader threads
 * (0 = all cores); psg_load_dataset registers the views with the context and
 * streams their targets into HBM through two pinned staging buffers, reads
 * overlapping copies. meta.json is left to the host language. */
typedef struct psg_dataset psg_dataset;
int psg_dataset_open(const char* root, int stride, psg_dataset** out);
int psg_dataset_close(psg_dataset* ds);
int psg_dataset_size(const psg_dataset* ds, int* n_views, int64_t* n_pixels);
int psg_dataset_cameras(const psg_dataset* ds, psg_camera* cams, int32_t* ids);
int psg_dataset_read(const psg_dataset* ds, int first, int count, float* target_depth,
                     float* target_normal, int threads);
int psg_load_dataset(psg_context* ctx, const psg_dataset* ds, int chunk_views, int threads);
/* write_map_f32 / read_map_f32 (dataio.cpp:65-97); data may be NULL to read the
 * header only; cap = capacity of data in floats. */
int psg_write_map_f32(const char* path, int width, int height, int channels, const float* data);
int psg_read_map_f32(const char* path, int expected_channels, int* width, int* height, float* data,
                     int64_t cap);
/* Recompute the per-view valid-target counts (renderer.cpp:328-332) after
 * psg_update_targets changed targets (psg_set_views and the loaders do it). */
int psg_refresh_target_counts(psg_context* ctx);

/* init_from_depth (scene_init.cpp:70-104) from the
 * registered views' resident targets: seeded reservoir sample of n_primitives
 * valid pixels, back-projected, radius = max(radius_scale * nearest-neighbour
 * distance, 1e-4), rotation = quat_from_z_to(normal); replaces the context's
 * planes (ids 0..n-1) and starts a fresh optimiser state. Bit-identical to the
 * reference. PSG_EIO when no pixel is valid. */
int psg_init_from_depth(psg_context* ctx, int n_primitives, uint64_t seed, double radius_scale,
                        int64_t* n_out);

/* ---- debug / parity ------------------------------------------------------- */
/* bin_primitives (renderer.cpp:115-147) on the device: CSR per tile with items
 * ascending per tile. Returns the number of items (or < 0 on error); items is
 * written only when cap >= that number. */
int64_t psg_debug_bins(psg_context* ctx, const psg_camera* cam, double lambda, int32_t* offsets,
                       int32_t* items, int64_t cap);

/* ---- multi-GPU: view-sharded data parallel, NCCL all-reduce of gradients -- */
#define PSG_NCCL_ID_BYTES 128
int psg_nccl_unique_id(char* id_out /* PSG_NCCL_ID_BYTES */);
int psg_comm_init(psg_context* ctx, const char* id, int nranks, int rank);
/* Sum the accumulated grads and step loss over all ranks (ncclAllReduce on the
 * context stream). */
int psg_allreduce_grads(psg_context* ctx);
int psg_comm_destroy(psg_context* ctx);

/* Pinned host memory helpers (for end-to-end copies at full PCIe rate). */
void* psg_host_alloc(size_t bytes);
void psg_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
