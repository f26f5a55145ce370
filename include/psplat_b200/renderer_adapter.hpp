// Drop-in C++ adapter: psplat_b200::Renderer has the exact method signatures of
// psplat::Renderer (reference proj/core/include/psplat/renderer.hpp:92-117) and
// forwards every call to the sm_100a implementation through the C ABI of
// include/psplat_b200.h. Include it after "psplat/renderer.hpp" inside the
// reference build; Optimizer::step (optimizer.cpp:71-80) can then swap
//   psplat::Renderer renderer_{cfg};
// for
//   psplat_b200::Renderer renderer_{cfg};
// unchanged otherwise. Errors are rethrown as the reference's exception types:
// PSG_EINVAL -> std::invalid_argument, PSG_ENONFINITE -> std::runtime_error.
//
// One CUDA context is owned per adapter instance (device 0 unless set with
// set_device before the first call). Maps and gradients stay fp64 at the
// boundary, as RenderedMaps / GradientBuffer require.
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "psplat/renderer.hpp"
#include "psplat_b200.h"

namespace psplat_b200 {

class Renderer {
public:
    explicit Renderer(psplat::RenderConfig cfg, int precision = PSG_FP64, int device = 0)
        : cfg_(cfg), precision_(precision), device_(device) {}
    ~Renderer() {
        if (ctx_) psg_destroy(ctx_);
    }
    Renderer(const Renderer&) = delete;
    Renderer& operator=(const Renderer&) = delete;

    // Renderer::render_view (renderer.cpp:231-317)
    psplat::ForwardResult render_view(const psplat::CameraView& view, const psplat::Scene& scene,
                                      double lambda, bool keep_records = false) const {
        if (view.width < 1 || view.height < 1)
            throw std::invalid_argument("render_view: empty view");
        prepare(scene);
        psplat::ForwardResult r;
        r.maps.resize(view.width, view.height);
        r.max_records = cfg_.max_records;
        if (keep_records) {
            r.rec_prim.assign(view.pixel_count() * std::size_t(cfg_.max_records), -1);
            r.rec_count.assign(view.pixel_count(), 0);
        }
        const psg_camera cam = to_cam(view);
        check(psg_render_view(ctx_, &cam, lambda, keep_records ? 1 : 0, r.maps.depth.data(),
                              r.maps.normal.data(), r.maps.alpha.data(),
                              keep_records ? r.rec_prim.data() : nullptr,
                              keep_records ? r.rec_count.data() : nullptr));
        return r;
    }

    // Renderer::render_loss (renderer.cpp:319-371)
    psplat::LossGrads render_loss(const psplat::RenderedMaps& maps,
                                  const psplat::CameraView& view) const {
        if (maps.width != view.width || maps.height != view.height)
            throw std::invalid_argument("render_loss: resolution mismatch");
        ensure();
        set_cfg();
        psplat::LossGrads lg;
        lg.d_depth.assign(view.pixel_count(), 0.0);
        lg.d_normal.assign(view.pixel_count() * 3, 0.0);
        if (cfg_.normalize_by_alpha) lg.d_alpha.assign(view.pixel_count(), 0.0);
        const psg_camera cam = to_cam(view);
        check(psg_render_loss(ctx_, &cam, view.target_depth.data(), view.target_normal.data(),
                              maps.depth.data(), maps.normal.data(), maps.alpha.data(), &lg.loss,
                              lg.d_depth.data(), lg.d_normal.data(),
                              cfg_.normalize_by_alpha ? lg.d_alpha.data() : nullptr));
        return lg;
    }

    // Renderer::backward (renderer.cpp:373-528); gradbuf is accumulated into.
    void backward(const psplat::CameraView& view, const psplat::Scene& scene, double lambda,
                  const psplat::ForwardResult& fwd, const psplat::LossGrads& loss_grads,
                  psplat::GradientBuffer& gradbuf) const {
        if (fwd.rec_count.empty())
            throw std::invalid_argument("backward: forward pass ran without keep_records");
        prepare(scene);
        const std::size_t n = scene.primitives.size();
        if (gradbuf.grads.size() != n) gradbuf.reset(n);
        std::vector<double> g(n * 11);
        for (std::size_t i = 0; i < n; ++i) {
            const psplat::PrimGrad& pg = gradbuf.grads[i];
            for (int k = 0; k < 3; ++k) g[11 * i + k] = pg.d_center[k];
            for (int k = 0; k < 4; ++k) g[11 * i + 3 + k] = pg.d_rotation[k];
            for (int k = 0; k < 4; ++k) g[11 * i + 7 + k] = pg.d_radii[k];
        }
        const psg_camera cam = to_cam(view);
        int64_t bad = -1;
        const int st = psg_backward(ctx_, &cam, lambda, fwd.max_records, fwd.rec_prim.data(),
                                    fwd.rec_count.data(), loss_grads.d_depth.data(),
                                    loss_grads.d_normal.data(),
                                    loss_grads.d_alpha.empty() ? nullptr : loss_grads.d_alpha.data(),
                                    g.data(), &bad);
        for (std::size_t i = 0; i < n; ++i) {
            psplat::PrimGrad& pg = gradbuf.grads[i];
            for (int k = 0; k < 3; ++k) pg.d_center[k] = g[11 * i + k];
            for (int k = 0; k < 4; ++k) pg.d_rotation[k] = g[11 * i + 3 + k];
            for (int k = 0; k < 4; ++k) pg.d_radii[k] = g[11 * i + 7 + k];
        }
        check(st);
    }

    const psplat::RenderConfig& config() const { return cfg_; }
    psplat::RenderConfig& config() { return cfg_; }

private:
    static void check(int st) {
        if (st == PSG_OK) return;
        const std::string msg = psg_last_error();
        if (st == PSG_EINVAL) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }
    void ensure() const {
        if (!ctx_) check(psg_create(device_, precision_, &ctx_));
    }
    void set_cfg() const {
        psg_render_config c;
        c.max_records = cfg_.max_records;
        c.normalize_by_alpha = cfg_.normalize_by_alpha ? 1 : 0;
        c.tile_size = cfg_.tile_size;
        c.threads = cfg_.threads;
        c.weight_floor = cfg_.weight_floor;
        c.t_near = cfg_.t_near;
        c.parallel_eps = cfg_.parallel_eps;
        c.alpha_floor = cfg_.alpha_floor;
        c.alpha1 = cfg_.alpha1;
        c.alpha2 = cfg_.alpha2;
        check(psg_set_config(ctx_, &c));
    }
    void prepare(const psplat::Scene& scene) const {
        ensure();
        set_cfg();
        const std::size_t n = scene.primitives.size();
        center_.resize(3 * n);
        rot_.resize(4 * n);
        radii_.resize(4 * n);
        ids_.resize(n);
        for (std::size_t i = 0; i < n; ++i) {
            const psplat::PlanePrimitive& p = scene.primitives[i];
            for (int k = 0; k < 3; ++k) center_[3 * i + k] = p.center[k];
            for (int k = 0; k < 4; ++k) rot_[4 * i + k] = p.rotation[k];
            for (int k = 0; k < 4; ++k) radii_[4 * i + k] = p.radii[k];
            ids_[i] = p.id;
        }
        check(psg_set_planes(ctx_, int64_t(n), center_.data(), rot_.data(), radii_.data(),
                             ids_.data()));
    }
    static psg_camera to_cam(const psplat::CameraView& v) {
        psg_camera c;
        c.fx = v.fx;
        c.fy = v.fy;
        c.cx = v.cx;
        c.cy = v.cy;
        c.width = v.width;
        c.height = v.height;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) c.rot_wc[3 * i + j] = v.rot_wc(i, j);
        for (int i = 0; i < 3; ++i) c.t_wc[i] = v.t_wc[i];
        return c;
    }

    psplat::RenderConfig cfg_;
    int precision_;
    int device_;
    mutable psg_context* ctx_ = nullptr;
    mutable std::vector<double> center_, rot_, radii_;
    mutable std::vector<int64_t> ids_;
};

}  // namespace psplat_b200
