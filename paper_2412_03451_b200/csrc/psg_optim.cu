// Device optimiser: Adam + quaternion renormalisation + radii clamp + the
// radii-gradient running sums (Optimizer::step tail, optimizer.cpp:84-140), and
// Optimizer::maybe_split as a stream compaction (optimizer.cpp:142-202).
// Compiled with -fmad=false and written in the reference's operation order, so
// every update is bit-identical to the reference given the same gradients. The
// bias corrections pow(beta, step) come from a host-built table (std::pow of the
// host libm, as the reference computes them): the device pow is not correctly
// rounded in the same places.
#include "psg_internal.h"

namespace psg {
namespace {

// quat_normalized (geometry.cpp:19-21): q / sqrt((w^2 + y^2) + (x^2 + z^2)),
// the Vector4d squaredNorm reduction order.
__device__ __forceinline__ void quat_normalized(const double* q, double* o) {
    const double n = sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]));
    for (int k = 0; k < 4; ++k) o[k] = q[k] / n;
}

// adam_scalar_update (optimizer.hpp:39-46)
__device__ __forceinline__ double adam_update(double& m, double& v, double g, double lr,
                                              double b1, double b2, double eps, double pow1,
                                              double pow2) {
    m = b1 * m + (1.0 - b1) * g;
    v = b2 * v + (1.0 - b2) * g * g;
    const double m_hat = m / (1.0 - pow1);
    const double v_hat = v / (1.0 - pow2);
    return lr * m_hat / (sqrt(v_hat) + eps);
}

__global__ void k_optim_apply(OptimIO io, OptimParams c) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= io.P || (io.gate && !*io.gate)) return;
    double g[11];
    for (int k = 0; k < 11; ++k) g[k] = io.grads[11 * i + k];
    // raw (pre-Adam) radii gradients feed the split rule (optimizer.cpp:84-87)
    for (int k = 0; k < 4; ++k) io.rgs[4 * i + k] += fabs(g[7 + k]);
    io.rgc[i] += 1;

    double* m = io.m + 11 * i;
    double* v = io.v + 11 * i;
    double mm[11], vv[11];
    for (int k = 0; k < 11; ++k) {
        mm[k] = m[k];
        vv[k] = v[k];
    }
    if (c.single_radii) {  // optimizer.cpp:110-119
        g[7] = g[8] = g[7] + g[8];
        g[9] = g[10] = g[9] + g[10];
        mm[8] = mm[7];
        vv[8] = vv[7];
        mm[10] = mm[9];
        vv[10] = vv[9];
    }
    const long long s = io.step[i] + 1;
    io.step[i] = s;
    const double p1 = io.pow1[s], p2 = io.pow2[s];
    double upd[11];
    for (int k = 0; k < 11; ++k) {
        const double lr = k < 3 ? c.lr_center : (k < 7 ? c.lr_rotation : c.lr_radii);
        upd[k] = adam_update(mm[k], vv[k], g[k], lr, c.beta1, c.beta2, c.eps, p1, p2);
    }
    for (int k = 0; k < 11; ++k) {
        m[k] = mm[k];
        v[k] = vv[k];
    }
    double* ce = io.center + 3 * i;
    double* q = io.rot + 4 * i;
    double* r = io.radii + 4 * i;
    for (int k = 0; k < 3; ++k) ce[k] -= upd[k];
    double qq[4], rr[4];
    for (int k = 0; k < 4; ++k) qq[k] = q[k] - upd[3 + k];
    for (int k = 0; k < 4; ++k) rr[k] = r[k] - upd[7 + k];
    if (c.single_radii) {
        rr[1] = rr[0];
        rr[3] = rr[2];
    }
    double qn[4];
    quat_normalized(qq, qn);
    for (int k = 0; k < 4; ++k) q[k] = qn[k];
    // std::max(r, floor): NaN stays NaN
    for (int k = 0; k < 4; ++k) r[k] = rr[k] < c.radii_floor ? c.radii_floor : rr[k];
}

// optimizer.cpp:150-160: 0 = cut along Y (X gradients), 1 = cut along X, -1 = keep
__global__ void k_split_mark(int64_t P, const double* rgs, const long long* rgc, double thr,
                             int* axis, int* cnt) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= P) return;
    int a = -1;
    if (rgc[i] != 0) {
        const double n = double(rgc[i]);
        double mean[4];
        for (int k = 0; k < 4; ++k) mean[k] = rgs[4 * i + k] / n;
        const double mx = 0.5 * (mean[0] + mean[1]);
        const double my = 0.5 * (mean[2] + mean[3]);
        const bool tx = mx > thr, ty = my > thr;
        if (tx || ty) a = (tx && (!ty || mx >= my)) ? 0 : 1;
    }
    axis[i] = a;
    cnt[i] = a < 0 ? 1 : 2;
}

// optimizer.cpp:169-195: parents keep their state; children tile the parent
// exactly along the cut axis and start with zero Adam state.
__global__ void k_split_write(OptimIO src, OptimIO dst, const int* axis, const int* pos) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= src.P) return;
    const int a = axis[i];
    const int64_t o = pos[i];
    if (a < 0) {
        for (int k = 0; k < 3; ++k) dst.center[3 * o + k] = src.center[3 * i + k];
        for (int k = 0; k < 4; ++k) dst.rot[4 * o + k] = src.rot[4 * i + k];
        for (int k = 0; k < 4; ++k) dst.radii[4 * o + k] = src.radii[4 * i + k];
        for (int k = 0; k < 11; ++k) dst.m[11 * o + k] = src.m[11 * i + k];
        for (int k = 0; k < 11; ++k) dst.v[11 * o + k] = src.v[11 * i + k];
        dst.step[o] = src.step[i];
        return;
    }
    double qn[4];
    quat_normalized(src.rot + 4 * i, qn);
    const double w = qn[0], x = qn[1], y = qn[2], z = qn[3];
    // plane_frame columns (geometry.cpp:10-17,33-40)
    double dir[3];
    if (a == 0) {
        dir[0] = 1 - 2 * (y * y + z * z);
        dir[1] = 2 * (x * y + w * z);
        dir[2] = 2 * (x * z - w * y);
    } else {
        dir[0] = 2 * (x * y - w * z);
        dir[1] = 1 - 2 * (x * x + z * z);
        dir[2] = 2 * (y * z + w * x);
    }
    const int ra = a == 0 ? 0 : 2;
    const double ha = src.radii[4 * i + ra] * 0.5, hb = src.radii[4 * i + ra + 1] * 0.5;
    for (int ch = 0; ch < 2; ++ch) {
        const int64_t oo = o + ch;
        for (int k = 0; k < 3; ++k) {
            const double pc = src.center[3 * i + k];
            dst.center[3 * oo + k] = ch == 0 ? pc + dir[k] * ha : pc - dir[k] * hb;
        }
        for (int k = 0; k < 4; ++k) dst.rot[4 * oo + k] = src.rot[4 * i + k];
        for (int k = 0; k < 4; ++k) dst.radii[4 * oo + k] = src.radii[4 * i + k];
        dst.radii[4 * oo + ra] = dst.radii[4 * oo + ra + 1] = ch == 0 ? ha : hb;
        for (int k = 0; k < 11; ++k) dst.m[11 * oo + k] = 0.0;
        for (int k = 0; k < 11; ++k) dst.v[11 * oo + k] = 0.0;
        dst.step[oo] = 0;
    }
}

__global__ void k_run_gate(const double* tail, const unsigned long long* first_bad, long long it,
                           double* log_slot, int* gate, unsigned long long* halt) {
    const double loss = tail[0], guard = tail[1];
    int ok = 0;
    if (halt[0] == ~0ull) {
        if (guard != 0.0) {
            halt[1] = 1;
        } else if (*first_bad != ~0ull) {
            halt[1] = 2;
        } else if (!isfinite(loss)) {
            halt[1] = 3;
        } else {
            ok = 1;
            *log_slot = loss;
        }
        if (!ok) halt[0] = (unsigned long long)it;
    }
    *gate = ok;
}

}  // namespace

void launch_run_gate(const double* tail, const unsigned long long* first_bad, long long iteration,
                     double* log_slot, int* gate, unsigned long long* halt, cudaStream_t s) {
    k_run_gate<<<1, 1, 0, s>>>(tail, first_bad, iteration, log_slot, gate, halt);
}

void launch_optim_apply(const OptimIO& io, const OptimParams& c, cudaStream_t s) {
    if (io.P <= 0) return;
    k_optim_apply<<<unsigned((io.P + 127) / 128), 128, 0, s>>>(io, c);
}

void launch_split_mark(int64_t P, const double* rgs, const long long* rgc, double thr, int* axis,
                       int* cnt, cudaStream_t s) {
    if (P <= 0) return;
    k_split_mark<<<unsigned((P + 127) / 128), 128, 0, s>>>(P, rgs, rgc, thr, axis, cnt);
}

void launch_split_write(const OptimIO& src, const OptimIO& dst, const int* axis, const int* pos,
                        cudaStream_t s) {
    if (src.P <= 0) return;
    k_split_write<<<unsigned((src.P + 127) / 128), 128, 0, s>>>(src, dst, axis, pos);
}

}  // namespace psg
