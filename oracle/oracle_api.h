/* TEST INFRASTRUCTURE ONLY — shared C declarations of the two CPU oracles.
 *
 *  ref_*  : oracle/_ref/libpsplat_ref.so — the reference's own sources
 *           (/root/reference/proj/core/src + tests/support) compiled verbatim
 *           through oracle/eigen_shim, wrapped by oracle/ref_harness.cpp.
 *  orc_*  : oracle/_build/liboracle.so   — oracle/psplat_oracle.c, a plain-C
 *           restatement of the same algorithm, line-cited against the reference.
 *
 * Both expose the same signatures so tests can compare them call for call.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
 * arm may load these libraries; the product path never does.
 */
#ifndef PSPLAT_ORACLE_API_H
#define PSPLAT_ORACLE_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* psplat::CameraView minus its targets (geometry.hpp:51-67). rot_wc row-major. */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double rot_wc[9];
    double t_wc[3];
} orc_camera;

/* psplat::RenderConfig (renderer.hpp:10-21). */
typedef struct {
    int32_t max_records;
    int32_t normalize_by_alpha;
    int32_t tile_size;
    int32_t threads;
    double weight_floor;
    double t_near;
    double parallel_eps;
    double alpha_floor;
    double alpha1;
    double alpha2;
} orc_config;

/* Planes as SoA: center[n*3], rotation[n*4] (w,x,y,z), radii[n*4], ids[n]. */

#define ORC_DECLARE(prefix)                                                                   \
    void prefix##default_config(orc_config* cfg);                                             \
    double prefix##lambda_schedule(int64_t ite, double base, double rate, double lmax);      \
    void prefix##plane_splat_weight(double px, double py, const double* radii, double lambda, \
                                    double* out11);                                           \
    int prefix##render_view(const orc_camera* cam, int64_t n, const double* center,          \
                            const double* rotation, const double* radii, double lambda,      \
                            const orc_config* cfg, int keep_records, double* depth,          \
                            double* normal, double* alpha, int32_t* rec_prim,                \
                            uint16_t* rec_count);                                             \
    int prefix##reference_render(const orc_camera* cam, int64_t n, const double* center,     \
                                 const double* rotation, const double* radii, double lambda, \
                                 const orc_config* cfg, double* depth, double* normal,       \
                                 double* alpha);                                              \
    int prefix##render_loss(const orc_camera* cam, const float* tdepth, const float* tnormal, \
                            const orc_config* cfg, const double* depth, const double* normal, \
                            const double* alpha, double* loss, double* d_depth,              \
                            double* d_normal, double* d_alpha);                              \
    int prefix##backward(const orc_camera* cam, int64_t n, const double* center,             \
                         const double* rotation, const double* radii, const int64_t* ids,    \
                         double lambda, const orc_config* cfg, int max_records,              \
                         const int32_t* rec_prim, const uint16_t* rec_count,                 \
                         const double* d_depth, const double* d_normal,                      \
                         const double* d_alpha, double* grads, char* err, int errlen);       \
    int64_t prefix##bin_primitives(const orc_camera* cam, int64_t n, const double* center,   \
                                   const double* rotation, const double* radii,              \
                                   double lambda, const orc_config* cfg, int32_t* offsets,   \
                                   int32_t* items, int64_t items_cap);                       \
    int prefix##gather_intersections(const orc_camera* cam, int64_t n, const double* center, \
                                     const double* rotation, const double* radii,            \
                                     double lambda, const orc_config* cfg, int u, int v,     \
                                     int32_t* prim, double* z, double* w, int cap);          \
    void prefix##random_scene(uint64_t seed, int n, double* center, double* rotation,        \
                              double* radii, int64_t* ids);                                   \
    void prefix##make_view(int width, int height, double focal, int random_pose,             \
                           uint64_t seed, orc_camera* cam);                                  \
    void prefix##fill_random_targets(const orc_camera* cam, uint64_t seed, float* tdepth,    \
                                     float* tnormal);                                        \
    double prefix##fd_loss_gradient(const orc_camera* cam, const float* tdepth,              \
                                    const float* tnormal, int64_t n, const double* center,   \
                                    const double* rotation, const double* radii,             \
                                    int64_t prim, int param, double lambda, double step,     \
                                    const orc_config* cfg);

ORC_DECLARE(ref_)
ORC_DECLARE(orc_)

/* Synthetic box-room generators (synthetic.cpp, scene_init.cpp). The room is
 * identified by (width, depth, height, n_boxes, seed); faces are returned as
 * 15 doubles each: center 3, u 3, v 3, half_u, half_v, normal 3, instance id. */
int ref_room_faces(double w, double d, double h, int boxes, uint64_t seed, double* faces,
                   int cap);
int ref_room_views(double w, double d, double h, int boxes, uint64_t seed_room, int n_views,
                   uint64_t seed_traj, int width, int height, double hfov_deg, orc_camera* cams,
                   char* err, int errlen);
void ref_render_ground_truth(double w, double d, double h, int boxes, uint64_t seed_room,
                             int n_views, const orc_camera* cams, float* tdepth, float* tnormal,
                             int threads);
int64_t ref_init_from_depth(int n_views, const orc_camera* cams, const float* tdepth,
                            const float* tnormal, int n_prims, uint64_t seed, double* center,
                            double* rotation, double* radii, int64_t* ids);

/* init_from_depth with an explicit radius_scale (scene_init.cpp:70-104); the
 * restatement returns -1 for n_prims < 1 and -2 when no pixel is valid. */
int64_t ref_init_from_depth_cfg(int n_views, const orc_camera* cams, const float* tdepth,
                                const float* tnormal, int n_prims, uint64_t seed,
                                double radius_scale, double* center, double* rotation,
                                double* radii, int64_t* ids);
int64_t orc_init_from_depth(int n_views, const orc_camera* cams, const float* tdepth,
                            const float* tnormal, int n_prims, uint64_t seed, double radius_scale,
                            double* center, double* rotation, double* radii, int64_t* ids);

/* CPU baseline: n_iter view-passes (render_view(keep) + render_loss + backward)
 * of the reference Renderer; returns wall seconds, writes the last loss. */
double ref_time_viewpass(const orc_camera* cam, const float* tdepth, const float* tnormal,
                         int64_t n, const double* center, const double* rotation,
                         const double* radii, double lambda, const orc_config* cfg, int n_iter,
                         double* last_loss);
double ref_time_render(const orc_camera* cam, int64_t n, const double* c, const double* q,
                       const double* r, double lambda, const orc_config* cfg, int n_iter);
int ref_hardware_threads(void);

/* ---- optimiser (optimizer.hpp / optimizer.cpp) ----------------------------- */
/* psplat::OptimConfig (optimizer.hpp:10-27). */
typedef struct {
    double lr_center, lr_radii, lr_rotation;
    double beta1, beta2, eps;
    int64_t split_interval;
    double split_grad_threshold;
    int32_t enable_split, single_radii;
    double merge_normal_deg, merge_offset, merge_adjacency;
    int32_t merge_use_adjacency, views_per_step;
    uint64_t seed;
    double radii_floor;
} orc_optim_config;

/* Restatement (orc_) on flat arrays. Per primitive: grads[11] (center 3,
 * rotation 4, radii 4), Adam m[11], v[11], step, radii_grad_sum[4],
 * radii_grad_count. */
void orc_default_optim_config(orc_optim_config* cfg);
int64_t orc_view_for_slot(uint64_t seed, int64_t n_views, int64_t slot);
void orc_accumulate_radii_grads(int64_t n, const double* grads, double* rgs, int64_t* rgc);
void orc_apply_adam(int64_t n, double* center, double* rotation, double* radii, double* m,
                    double* v, int64_t* step, const double* grads, const orc_optim_config* cfg);
/* Optimizer::maybe_split. Returns -1 when it does not fire (state untouched),
 * else the number of split primitives; outputs (capacity 2n) receive the new
 * scene and Adam state, *n_out its size, *next_id is advanced; the caller then
 * zeroes the radii statistics (size *n_out). */
int64_t orc_maybe_split(int64_t n, int64_t iteration, const orc_optim_config* cfg,
                        const double* center, const double* rotation, const double* radii,
                        const int64_t* ids, const double* m, const double* v, const int64_t* step,
                        const double* rgs, const int64_t* rgc, int64_t* next_id,
                        double* center_out, double* rotation_out, double* radii_out,
                        int64_t* ids_out, double* m_out, double* v_out, int64_t* step_out,
                        int64_t* n_out);

/* merge_planes (optimizer.cpp:236-299) and rect_distance (geometry.cpp:131-149),
 * same signature for ref_ and orc_. instance_of[n] indexes the sorted instance
 * list; per instance normal[3], offset, area (capacity n). Returns the count. */
#define ORC_DECLARE_MERGE(prefix)                                                              \
    int64_t prefix##merge_planes(int64_t n, const double* center, const double* rotation,     \
                                 const double* radii, const int64_t* ids,                     \
                                 const double* scene_center, double normal_deg,               \
                                 double merge_offset, double merge_adjacency,                 \
                                 int use_adjacency, int32_t* instance_of,                     \
                                 double* inst_normal, double* inst_offset, double* inst_area); \
    double prefix##rect_distance(const double* ca, const double* qa, const double* ra,        \
                                 const double* cb, const double* qb, const double* rb);
ORC_DECLARE_MERGE(ref_)
ORC_DECLARE_MERGE(orc_)

/* The reference psplat::Optimizer itself (ref_), driven through its public API. */
void ref_default_optim_config(orc_optim_config* cfg);
void* ref_optimizer_create(int64_t n, const double* center, const double* rotation,
                           const double* radii, const int64_t* ids, int64_t next_id, int n_views,
                           const orc_camera* cams, const float* tdepth, const float* tnormal,
                           const orc_optim_config* ocfg, const orc_config* rcfg,
                           double lambda_base, double lambda_rate, double lambda_max);
void ref_optimizer_destroy(void* opt);
/* 0 = ok, 1 = std::runtime_error, 2 = std::invalid_argument (message in err). */
int ref_optimizer_step(void* opt, double* loss, char* err, int errlen);
int ref_optimizer_maybe_split(void* opt);
int64_t ref_optimizer_size(void* opt);
int64_t ref_optimizer_view_for_slot(void* opt, int64_t slot);
void ref_optimizer_get(void* opt, double* center, double* rotation, double* radii, int64_t* ids,
                       double* m, double* v, int64_t* step, double* rgs, int64_t* rgc,
                       int64_t* iteration, int64_t* next_id);
void ref_optimizer_set_stats(void* opt, int64_t iteration, const double* rgs, const int64_t* rgc);
void ref_optimizer_last_grads(void* opt, double* grads);

#ifdef __cplusplus
}
#endif
#endif
