// TEST INFRASTRUCTURE ONLY — extern "C" wrapper around the reference's own code.
//
// This TU #includes the reference's renderer.cpp (path passed by the Makefile as
// REF_RENDERER_CPP) so that its anonymous-namespace internals (make_prim_views,
// bin_primitives, projected_rect, eval_candidate; renderer.cpp:12-186) are
// reachable for the bit-exact binning check. No reference file is copied or
// modified: the sources are compiled in place from /root/reference by
// oracle/Makefile into oracle/_ref/libpsplat_ref.so.
#include REF_RENDERER_CPP

#include "psplat/optimizer.hpp"
#include "psplat/scene_init.hpp"
#include "psplat/synthetic.hpp"
#include "support/reference_renderer.hpp"
#include "support/test_scenes.hpp"

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>

#include "oracle_api.h"

using namespace psplat;

namespace {

RenderConfig to_cfg(const orc_config* c) {
    RenderConfig r;
    r.max_records = c->max_records;
    r.weight_floor = c->weight_floor;
    r.t_near = c->t_near;
    r.parallel_eps = c->parallel_eps;
    r.alpha_floor = c->alpha_floor;
    r.normalize_by_alpha = c->normalize_by_alpha != 0;
    r.alpha1 = c->alpha1;
    r.alpha2 = c->alpha2;
    r.tile_size = c->tile_size;
    r.threads = c->threads;
    return r;
}

CameraView to_view(const orc_camera* c, const float* td = nullptr, const float* tn = nullptr) {
    CameraView v;
    v.fx = c->fx;
    v.fy = c->fy;
    v.cx = c->cx;
    v.cy = c->cy;
    v.width = c->width;
    v.height = c->height;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v.rot_wc(i, j) = c->rot_wc[3 * i + j];
    for (int i = 0; i < 3; ++i) v.t_wc[i] = c->t_wc[i];
    if (td) v.target_depth.assign(td, td + v.pixel_count());
    if (tn) v.target_normal.assign(tn, tn + 3 * v.pixel_count());
    return v;
}

void from_view(const CameraView& v, orc_camera* c) {
    c->fx = v.fx;
    c->fy = v.fy;
    c->cx = v.cx;
    c->cy = v.cy;
    c->width = v.width;
    c->height = v.height;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c->rot_wc[3 * i + j] = v.rot_wc(i, j);
    for (int i = 0; i < 3; ++i) c->t_wc[i] = v.t_wc[i];
}

Scene to_scene(int64_t n, const double* c, const double* q, const double* r,
               const int64_t* ids = nullptr) {
    Scene s;
    s.primitives.resize(std::size_t(n));
    for (int64_t i = 0; i < n; ++i) {
        PlanePrimitive& p = s.primitives[std::size_t(i)];
        p.center = Vec3(c[3 * i], c[3 * i + 1], c[3 * i + 2]);
        p.rotation = Quat(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]);
        p.radii = Vec4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
        p.id = ids ? ids[i] : i;
    }
    s.next_id = n;
    return s;
}

void from_scene(const Scene& s, double* c, double* q, double* r, int64_t* ids) {
    for (std::size_t i = 0; i < s.primitives.size(); ++i) {
        const PlanePrimitive& p = s.primitives[i];
        for (int k = 0; k < 3; ++k) c[3 * i + k] = p.center[k];
        for (int k = 0; k < 4; ++k) q[4 * i + k] = p.rotation[k];
        for (int k = 0; k < 4; ++k) r[4 * i + k] = p.radii[k];
        if (ids) ids[i] = p.id;
    }
}

void copy_maps(const RenderedMaps& m, double* depth, double* normal, double* alpha) {
    if (depth) std::memcpy(depth, m.depth.data(), m.depth.size() * sizeof(double));
    if (normal) std::memcpy(normal, m.normal.data(), m.normal.size() * sizeof(double));
    if (alpha) std::memcpy(alpha, m.alpha.data(), m.alpha.size() * sizeof(double));
}

}  // namespace

extern "C" {

void ref_default_config(orc_config* c) {
    const RenderConfig r;
    c->max_records = r.max_records;
    c->weight_floor = r.weight_floor;
    c->t_near = r.t_near;
    c->parallel_eps = r.parallel_eps;
    c->alpha_floor = r.alpha_floor;
    c->normalize_by_alpha = r.normalize_by_alpha;
    c->alpha1 = r.alpha1;
    c->alpha2 = r.alpha2;
    c->tile_size = r.tile_size;
    c->threads = r.threads;
}

double ref_lambda_schedule(int64_t ite, double base, double rate, double lmax) {
    SplatParams p;
    p.lambda_base = base;
    p.lambda_rate = rate;
    p.lambda_max = lmax;
    return lambda_schedule(ite, p);
}

void ref_plane_splat_weight(double px, double py, const double* radii, double lambda,
                            double* o) {
    const SplatEval ev =
        plane_splat_weight(px, py, Vec4(radii[0], radii[1], radii[2], radii[3]), lambda);
    o[0] = ev.weight;
    o[1] = ev.w_x;
    o[2] = ev.w_y;
    o[3] = ev.d_px;
    o[4] = ev.d_py;
    for (int k = 0; k < 4; ++k) o[5 + k] = ev.d_radii[k];
    o[9] = ev.x_selected ? 1.0 : 0.0;
    o[10] = 0.0;
}

int ref_render_view(const orc_camera* cam, int64_t n, const double* c, const double* q,
                    const double* r, double lambda, const orc_config* cfg, int keep,
                    double* depth, double* normal, double* alpha, int32_t* rec_prim,
                    uint16_t* rec_count) {
    try {
        const Renderer ren{to_cfg(cfg)};
        const ForwardResult f = ren.render_view(to_view(cam), to_scene(n, c, q, r), lambda, keep);
        copy_maps(f.maps, depth, normal, alpha);
        if (keep && rec_prim)
            std::memcpy(rec_prim, f.rec_prim.data(), f.rec_prim.size() * sizeof(int32_t));
        if (keep && rec_count)
            std::memcpy(rec_count, f.rec_count.data(), f.rec_count.size() * sizeof(uint16_t));
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 2;
    }
}

int ref_reference_render(const orc_camera* cam, int64_t n, const double* c, const double* q,
                         const double* r, double lambda, const orc_config* cfg, double* depth,
                         double* normal, double* alpha) {
    const RenderedMaps m = testing::reference_render(to_view(cam), to_scene(n, c, q, r), lambda,
                                                     to_cfg(cfg));
    copy_maps(m, depth, normal, alpha);
    return 0;
}

int ref_render_loss(const orc_camera* cam, const float* td, const float* tn,
                    const orc_config* cfg, const double* depth, const double* normal,
                    const double* alpha, double* loss, double* d_depth, double* d_normal,
                    double* d_alpha) {
    try {
        const CameraView view = to_view(cam, td, tn);
        RenderedMaps m;
        m.resize(view.width, view.height);
        m.depth.assign(depth, depth + view.pixel_count());
        m.normal.assign(normal, normal + 3 * view.pixel_count());
        m.alpha.assign(alpha, alpha + view.pixel_count());
        const LossGrads lg = Renderer{to_cfg(cfg)}.render_loss(m, view);
        *loss = lg.loss;
        std::memcpy(d_depth, lg.d_depth.data(), lg.d_depth.size() * sizeof(double));
        std::memcpy(d_normal, lg.d_normal.data(), lg.d_normal.size() * sizeof(double));
        if (d_alpha) {
            if (lg.d_alpha.empty())
                std::memset(d_alpha, 0, view.pixel_count() * sizeof(double));
            else
                std::memcpy(d_alpha, lg.d_alpha.data(), lg.d_alpha.size() * sizeof(double));
        }
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

int ref_backward(const orc_camera* cam, int64_t n, const double* c, const double* q,
                 const double* r, const int64_t* ids, double lambda, const orc_config* cfg,
                 int max_records, const int32_t* rec_prim, const uint16_t* rec_count,
                 const double* d_depth, const double* d_normal, const double* d_alpha,
                 double* grads, char* err, int errlen) {
    try {
        const CameraView view = to_view(cam);
        const std::size_t np = view.pixel_count();
        ForwardResult f;
        f.max_records = max_records;
        f.maps.resize(view.width, view.height);
        if (rec_count) {
            f.rec_prim.assign(rec_prim, rec_prim + np * std::size_t(max_records));
            f.rec_count.assign(rec_count, rec_count + np);
        }
        LossGrads lg;
        lg.d_depth.assign(d_depth, d_depth + np);
        lg.d_normal.assign(d_normal, d_normal + 3 * np);
        if (d_alpha) lg.d_alpha.assign(d_alpha, d_alpha + np);
        GradientBuffer gb;
        gb.reset(std::size_t(n));
        for (int64_t i = 0; i < n; ++i) {
            PrimGrad& g = gb.grads[std::size_t(i)];
            for (int k = 0; k < 3; ++k) g.d_center[k] = grads[11 * i + k];
            for (int k = 0; k < 4; ++k) g.d_rotation[k] = grads[11 * i + 3 + k];
            for (int k = 0; k < 4; ++k) g.d_radii[k] = grads[11 * i + 7 + k];
        }
        Renderer{to_cfg(cfg)}.backward(view, to_scene(n, c, q, r, ids), lambda, f, lg, gb);
        for (int64_t i = 0; i < n; ++i) {
            const PrimGrad& g = gb.grads[std::size_t(i)];
            for (int k = 0; k < 3; ++k) grads[11 * i + k] = g.d_center[k];
            for (int k = 0; k < 4; ++k) grads[11 * i + 3 + k] = g.d_rotation[k];
            for (int k = 0; k < 4; ++k) grads[11 * i + 7 + k] = g.d_radii[k];
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        if (err) std::snprintf(err, std::size_t(errlen), "%s", e.what());
        return 1;
    } catch (const std::runtime_error& e) {
        if (err) std::snprintf(err, std::size_t(errlen), "%s", e.what());
        return 3;
    }
}

int64_t ref_bin_primitives(const orc_camera* cam, int64_t n, const double* c, const double* q,
                           const double* r, double lambda, const orc_config* cfg,
                           int32_t* offsets, int32_t* items, int64_t cap) {
    const CameraView view = to_view(cam);
    const Scene scene = to_scene(n, c, q, r);
    const RenderConfig rc = to_cfg(cfg);
    const std::vector<PrimView> pvs = make_prim_views(view, scene);
    const Binning bin = bin_primitives(view, scene, pvs, lambda, rc);
    if (offsets) std::memcpy(offsets, bin.offsets.data(), bin.offsets.size() * sizeof(int32_t));
    const int64_t total = int64_t(bin.items.size());
    if (items && cap >= total) std::memcpy(items, bin.items.data(), std::size_t(total) * 4);
    return total;
}

int ref_gather_intersections(const orc_camera* cam, int64_t n, const double* c,
                             const double* q, const double* r, double lambda,
                             const orc_config* cfg, int u, int v, int32_t* prim, double* z,
                             double* w, int cap) {
    const CameraView view = to_view(cam);
    const Scene scene = to_scene(n, c, q, r);
    const auto frames = testing::build_frames(scene);
    const auto recs = gather_intersections(generate_ray(view, u, v), view, scene.primitives,
                                           frames, lambda, to_cfg(cfg));
    const int cnt = int(recs.size());
    for (int i = 0; i < cnt && i < cap; ++i) {
        prim[i] = recs[std::size_t(i)].prim_index;
        z[i] = recs[std::size_t(i)].z_cam;
        w[i] = recs[std::size_t(i)].weight;
    }
    return cnt;
}

void ref_random_scene(uint64_t seed, int n, double* c, double* q, double* r, int64_t* ids) {
    from_scene(testing::random_scene(seed, n), c, q, r, ids);
}

void ref_make_view(int width, int height, double focal, int random_pose, uint64_t seed,
                   orc_camera* cam) {
    from_view(testing::make_view(width, height, focal, random_pose != 0, seed), cam);
}

void ref_fill_random_targets(const orc_camera* cam, uint64_t seed, float* td, float* tn) {
    CameraView v = to_view(cam);
    testing::fill_random_targets(v, seed);
    std::memcpy(td, v.target_depth.data(), v.target_depth.size() * sizeof(float));
    std::memcpy(tn, v.target_normal.data(), v.target_normal.size() * sizeof(float));
}

double ref_fd_loss_gradient(const orc_camera* cam, const float* td, const float* tn, int64_t n,
                            const double* c, const double* q, const double* r, int64_t prim,
                            int param, double lambda, double step, const orc_config* cfg) {
    const Renderer ren{to_cfg(cfg)};
    return testing::fd_loss_gradient(ren, to_view(cam, td, tn), to_scene(n, c, q, r),
                                     std::size_t(prim), param, lambda, step);
}

int ref_room_faces(double w, double d, double h, int boxes, uint64_t seed, double* out,
                   int cap) {
    const SyntheticScene room = generate_box_room(w, d, h, boxes, seed);
    const int nf = int(room.faces.size());
    for (int i = 0; i < nf && i < cap; ++i) {
        const GtFace& f = room.faces[std::size_t(i)];
        double* o = out + 15 * i;
        for (int k = 0; k < 3; ++k) {
            o[k] = f.center[k];
            o[3 + k] = f.u_axis[k];
            o[6 + k] = f.v_axis[k];
            o[11 + k] = f.normal[k];
        }
        o[9] = f.half_u;
        o[10] = f.half_v;
        o[14] = double(f.instance_id);
    }
    return nf;
}

int ref_room_views(double w, double d, double h, int boxes, uint64_t seed_room, int n_views,
                   uint64_t seed_traj, int width, int height, double hfov_deg, orc_camera* cams,
                   char* err, int errlen) {
    try {
        const SyntheticScene room = generate_box_room(w, d, h, boxes, seed_room);
        const auto poses = sample_trajectory(room, n_views, seed_traj);
        const double fx = (width / 2.0) / std::tan(hfov_deg * M_PI / 360.0);
        for (std::size_t i = 0; i < poses.size(); ++i) {
            CameraView v;
            v.width = width;
            v.height = height;
            v.fx = v.fy = fx;
            v.cx = width / 2.0;
            v.cy = height / 2.0;
            v.rot_wc = poses[i].rot_wc;
            v.t_wc = poses[i].t_wc;
            from_view(v, cams + i);
        }
        return 0;
    } catch (const std::exception& e) {
        if (err) std::snprintf(err, std::size_t(errlen), "%s", e.what());
        return 1;
    }
}

void ref_render_ground_truth(double w, double d, double h, int boxes, uint64_t seed_room,
                             int n_views, const orc_camera* cams, float* td, float* tn,
                             int threads) {
    const SyntheticScene room = generate_box_room(w, d, h, boxes, seed_room);
    if (threads <= 0) threads = default_thread_count();
    parallel_for(std::size_t(n_views), threads, [&](std::size_t i) {
        CameraView v = to_view(cams + i);
        render_ground_truth(room, v);
        const std::size_t np = v.pixel_count();
        std::memcpy(td + i * np, v.target_depth.data(), np * sizeof(float));
        std::memcpy(tn + 3 * i * np, v.target_normal.data(), 3 * np * sizeof(float));
    });
}

int64_t ref_init_from_depth(int n_views, const orc_camera* cams, const float* td,
                            const float* tn, int n_prims, uint64_t seed, double* c, double* q,
                            double* r, int64_t* ids) {
    std::vector<CameraView> views;
    views.reserve(std::size_t(n_views));
    std::size_t off = 0;
    for (int i = 0; i < n_views; ++i) {
        views.push_back(to_view(cams + i, td + off, tn + 3 * off));
        off += views.back().pixel_count();
    }
    InitConfig ic;
    ic.n_primitives = n_prims;
    ic.seed = seed;
    const Scene s = init_from_depth(views, ic);
    from_scene(s, c, q, r, ids);
    return int64_t(s.primitives.size());
}

int64_t ref_init_from_depth_cfg(int n_views, const orc_camera* cams, const float* td,
                                const float* tn, int n_prims, uint64_t seed, double radius_scale,
                                double* c, double* q, double* r, int64_t* ids) {
    std::vector<CameraView> views;
    std::size_t off = 0;
    for (int i = 0; i < n_views; ++i) {
        views.push_back(to_view(cams + i, td + off, tn + 3 * off));
        off += views.back().pixel_count();
    }
    InitConfig ic;
    ic.n_primitives = n_prims;
    ic.seed = seed;
    ic.radius_scale = radius_scale;
    try {
        const Scene s = init_from_depth(views, ic);
        from_scene(s, c, q, r, ids);
        return int64_t(s.primitives.size());
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::runtime_error&) {
        return -2;
    }
}

double ref_time_viewpass(const orc_camera* cam, const float* td, const float* tn, int64_t n,
                         const double* c, const double* q, const double* r, double lambda,
                         const orc_config* cfg, int n_iter, double* last_loss) {
    const CameraView view = to_view(cam, td, tn);
    const Scene scene = to_scene(n, c, q, r);
    const Renderer ren{to_cfg(cfg)};
    double loss = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int it = 0; it < n_iter; ++it) {
        const ForwardResult fwd = ren.render_view(view, scene, lambda, true);
        const LossGrads lg = ren.render_loss(fwd.maps, view);
        GradientBuffer gb;
        ren.backward(view, scene, lambda, fwd, lg, gb);
        loss = lg.loss;
    }
    const double s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (last_loss) *last_loss = loss;
    return s;
}

// BM_RenderView's loop body (benchmarks/render_bench.cpp:42-51): forward only,
// no records kept.
double ref_time_render(const orc_camera* cam, int64_t n, const double* c, const double* q,
                       const double* r, double lambda, const orc_config* cfg, int n_iter) {
    const CameraView view = to_view(cam);
    const Scene scene = to_scene(n, c, q, r);
    const Renderer ren{to_cfg(cfg)};
    const auto t0 = std::chrono::steady_clock::now();
    double sink = 0;
    for (int it = 0; it < n_iter; ++it) {
        const ForwardResult fwd = ren.render_view(view, scene, lambda, false);
        sink += fwd.maps.depth[0];
    }
    const double s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return sink == sink ? s : -s;
}

int ref_hardware_threads(void) { return default_thread_count(); }

int64_t ref_merge_planes(int64_t n, const double* c, const double* q, const double* r,
                         const int64_t* ids, const double* sc, double normal_deg,
                         double merge_offset, double merge_adjacency, int use_adjacency,
                         int32_t* instance_of, double* inst_normal, double* inst_offset,
                         double* inst_area) {
    const Scene scene = to_scene(n, c, q, r, ids);
    OptimConfig cfg;
    cfg.merge_normal_deg = normal_deg;
    cfg.merge_offset = merge_offset;
    cfg.merge_adjacency = merge_adjacency;
    cfg.merge_use_adjacency = use_adjacency != 0;
    const auto inst = merge_planes(scene, Vec3(sc[0], sc[1], sc[2]), cfg);
    for (std::size_t t = 0; t < inst.size(); ++t) {
        for (std::int32_t m : inst[t].member_indices) instance_of[m] = std::int32_t(t);
        for (int k = 0; k < 3; ++k) inst_normal[3 * t + k] = inst[t].normal[k];
        inst_offset[t] = inst[t].offset;
        inst_area[t] = inst[t].area;
    }
    return int64_t(inst.size());
}

double ref_rect_distance(const double* ca, const double* qa, const double* ra, const double* cb,
                         const double* qb, const double* rb) {
    PlanePrimitive a, b;
    a.center = Vec3(ca[0], ca[1], ca[2]);
    a.rotation = Quat(qa[0], qa[1], qa[2], qa[3]);
    a.radii = Vec4(ra[0], ra[1], ra[2], ra[3]);
    b.center = Vec3(cb[0], cb[1], cb[2]);
    b.rotation = Quat(qb[0], qb[1], qb[2], qb[3]);
    b.radii = Vec4(rb[0], rb[1], rb[2], rb[3]);
    return rect_distance(a, plane_frame(quat_normalized(a.rotation)), b,
                         plane_frame(quat_normalized(b.rotation)));
}

// ---- psplat::Optimizer through its public API (optimizer.hpp:76-117)
void ref_default_optim_config(orc_optim_config* c) {
    const OptimConfig o;
    c->lr_center = o.lr_center;
    c->lr_radii = o.lr_radii;
    c->lr_rotation = o.lr_rotation;
    c->beta1 = o.beta1;
    c->beta2 = o.beta2;
    c->eps = o.eps;
    c->split_interval = o.split_interval;
    c->split_grad_threshold = o.split_grad_threshold;
    c->enable_split = o.enable_split;
    c->single_radii = o.single_radii;
    c->merge_normal_deg = o.merge_normal_deg;
    c->merge_offset = o.merge_offset;
    c->merge_adjacency = o.merge_adjacency;
    c->merge_use_adjacency = o.merge_use_adjacency;
    c->views_per_step = o.views_per_step;
    c->seed = o.seed;
    c->radii_floor = o.radii_floor;
}

void* ref_optimizer_create(int64_t n, const double* c, const double* q, const double* r,
                           const int64_t* ids, int64_t next_id, int n_views,
                           const orc_camera* cams, const float* td, const float* tn,
                           const orc_optim_config* oc, const orc_config* rc, double lambda_base,
                           double lambda_rate, double lambda_max) {
    Scene scene = to_scene(n, c, q, r, ids);
    scene.next_id = next_id;
    std::vector<CameraView> views;
    std::size_t off = 0;
    for (int i = 0; i < n_views; ++i) {
        views.push_back(to_view(cams + i, td + off, tn + 3 * off));
        off += views.back().pixel_count();
    }
    OptimConfig o;
    o.lr_center = oc->lr_center;
    o.lr_radii = oc->lr_radii;
    o.lr_rotation = oc->lr_rotation;
    o.beta1 = oc->beta1;
    o.beta2 = oc->beta2;
    o.eps = oc->eps;
    o.split_interval = oc->split_interval;
    o.split_grad_threshold = oc->split_grad_threshold;
    o.enable_split = oc->enable_split != 0;
    o.single_radii = oc->single_radii != 0;
    o.merge_normal_deg = oc->merge_normal_deg;
    o.merge_offset = oc->merge_offset;
    o.merge_adjacency = oc->merge_adjacency;
    o.merge_use_adjacency = oc->merge_use_adjacency != 0;
    o.views_per_step = oc->views_per_step;
    o.seed = oc->seed;
    o.radii_floor = oc->radii_floor;
    SplatParams sp;
    sp.lambda_base = lambda_base;
    sp.lambda_rate = lambda_rate;
    sp.lambda_max = lambda_max;
    sp.weight_floor = rc->weight_floor;
    return new Optimizer(std::move(scene), std::move(views), o, to_cfg(rc), sp);
}

void ref_optimizer_destroy(void* opt) { delete static_cast<Optimizer*>(opt); }

int ref_optimizer_step(void* opt, double* loss, char* err, int errlen) {
    try {
        *loss = static_cast<Optimizer*>(opt)->step();
        return 0;
    } catch (const std::invalid_argument& e) {
        if (err && errlen > 0) std::snprintf(err, std::size_t(errlen), "%s", e.what());
        return 2;
    } catch (const std::exception& e) {
        if (err && errlen > 0) std::snprintf(err, std::size_t(errlen), "%s", e.what());
        return 1;
    }
}

int ref_optimizer_maybe_split(void* opt) { return static_cast<Optimizer*>(opt)->maybe_split(); }

int64_t ref_optimizer_size(void* opt) {
    return int64_t(static_cast<Optimizer*>(opt)->scene().primitives.size());
}

int64_t ref_optimizer_view_for_slot(void* opt, int64_t slot) {
    return int64_t(static_cast<Optimizer*>(opt)->view_for_slot(slot));
}

void ref_optimizer_get(void* opt, double* c, double* q, double* r, int64_t* ids, double* m,
                       double* v, int64_t* step, double* rgs, int64_t* rgc, int64_t* iteration,
                       int64_t* next_id) {
    const OptimState& st = static_cast<Optimizer*>(opt)->state();
    from_scene(st.scene, c, q, r, ids);
    for (std::size_t i = 0; i < st.adam.size(); ++i) {
        for (int k = 0; k < 11; ++k) {
            m[11 * i + k] = st.adam[i].m[std::size_t(k)];
            v[11 * i + k] = st.adam[i].v[std::size_t(k)];
        }
        step[i] = st.adam[i].step;
        for (int k = 0; k < 4; ++k) rgs[4 * i + k] = st.radii_grad_sum[i][k];
        rgc[i] = st.radii_grad_count[i];
    }
    *iteration = st.iteration;
    *next_id = st.scene.next_id;
}

void ref_optimizer_set_stats(void* opt, int64_t iteration, const double* rgs, const int64_t* rgc) {
    OptimState& st = static_cast<Optimizer*>(opt)->state();
    st.iteration = iteration;
    for (std::size_t i = 0; i < st.radii_grad_sum.size(); ++i) {
        for (int k = 0; k < 4; ++k) st.radii_grad_sum[i][k] = rgs[4 * i + k];
        st.radii_grad_count[i] = rgc[i];
    }
}

void ref_optimizer_last_grads(void* opt, double* g) {
    const GradientBuffer& gb = static_cast<Optimizer*>(opt)->last_gradients();
    for (std::size_t i = 0; i < gb.grads.size(); ++i) {
        for (int k = 0; k < 3; ++k) g[11 * i + k] = gb.grads[i].d_center[k];
        for (int k = 0; k < 4; ++k) g[11 * i + 3 + k] = gb.grads[i].d_rotation[k];
        for (int k = 0; k < 4; ++k) g[11 * i + 7 + k] = gb.grads[i].d_radii[k];
    }
}

}  // extern "C"
