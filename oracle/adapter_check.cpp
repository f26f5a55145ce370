// TEST INFRASTRUCTURE ONLY — drop-in check of include/psplat_b200/renderer_adapter.hpp.
//
// Built against the reference's own headers and sources (oracle/Makefile), it
// runs psplat::Renderer (CPU, the reference) and psplat_b200::Renderer (GPU, via
// the C ABI) on the reference's fixture scenes with identical call sequences —
// exactly Optimizer::step's render_view(keep) -> render_loss -> backward
// (optimizer.cpp:71-80) — and reports the largest differences. Exit status 1 if
// a tolerance of the fp64 contract is exceeded.
#include <cmath>
#include <cstdio>

#include "psplat/renderer.hpp"
#include "psplat_b200/renderer_adapter.hpp"
#include "support/test_scenes.hpp"

using namespace psplat;

int main() {
    double worst_map = 0, worst_grad = 0, worst_loss = 0;
    int rec_mismatch = 0;
    for (std::uint64_t seed : {1u, 2u, 3u, 4u, 11u}) {
        const Scene scene = testing::random_scene(seed, 24);
        CameraView view = testing::make_view(48, 40, 30.0, true, seed);
        testing::fill_random_targets(view, seed);
        for (double lambda : {7.4, 40.0, 300.0}) {
            RenderConfig cfg;
            cfg.threads = 4;
            Renderer ref{cfg};
            psplat_b200::Renderer gpu{cfg, PSG_FP64};
            const ForwardResult fr = ref.render_view(view, scene, lambda, true);
            const ForwardResult fg = gpu.render_view(view, scene, lambda, true);
            for (std::size_t i = 0; i < view.pixel_count(); ++i) {
                worst_map = std::max(worst_map, std::abs(fr.maps.depth[i] - fg.maps.depth[i]));
                worst_map = std::max(worst_map, std::abs(fr.maps.alpha[i] - fg.maps.alpha[i]));
            }
            rec_mismatch += fr.rec_prim != fg.rec_prim;
            const LossGrads lr = ref.render_loss(fr.maps, view);
            const LossGrads lgp = gpu.render_loss(fg.maps, view);
            worst_loss = std::max(worst_loss, std::abs(lr.loss - lgp.loss) / std::max(1e-300, std::abs(lr.loss)));
            GradientBuffer gr, gg;
            ref.backward(view, scene, lambda, fr, lr, gr);
            gpu.backward(view, scene, lambda, fg, lgp, gg);
            double gmax = 0;
            for (const PrimGrad& g : gr.grads) gmax = std::max({gmax, g.d_center.cwiseAbs().maxCoeff(),
                                                                g.d_rotation.cwiseAbs().maxCoeff(),
                                                                g.d_radii.cwiseAbs().maxCoeff()});
            for (std::size_t i = 0; i < gr.grads.size(); ++i) {
                const double e = std::max({(gr.grads[i].d_center - gg.grads[i].d_center).cwiseAbs().maxCoeff(),
                                           (gr.grads[i].d_rotation - gg.grads[i].d_rotation).cwiseAbs().maxCoeff(),
                                           (gr.grads[i].d_radii - gg.grads[i].d_radii).cwiseAbs().maxCoeff()});
                worst_grad = std::max(worst_grad, e / std::max(gmax, 1e-300));
            }
        }
    }
    // error contract: the same exception types and messages
    bool errors_ok = false;
    try {
        RenderConfig cfg;
        cfg.max_records = 65;
        psplat_b200::Renderer gpu{cfg};
        gpu.render_view(testing::make_view(8, 8, 8.0), testing::random_scene(1, 2), 10.0);
    } catch (const std::invalid_argument& e) {
        errors_ok = std::string(e.what()).find("max_records") != std::string::npos;
    }
    const bool ok = worst_map <= 1e-12 && worst_grad <= 1e-9 && worst_loss <= 1e-10 &&
                    rec_mismatch == 0 && errors_ok;
    std::printf("{\"adapter_check\": %s, \"max_map_abs\": %.3g, \"max_grad_rel\": %.3g, "
                "\"max_loss_rel\": %.3g, \"record_list_mismatches\": %d, \"errors_ok\": %s}\n",
                ok ? "true" : "false", worst_map, worst_grad, worst_loss, rec_mismatch,
                errors_ok ? "true" : "false");
    return ok ? 0 : 1;
}
