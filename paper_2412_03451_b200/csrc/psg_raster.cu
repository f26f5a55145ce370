// Per-tile rasteriser: forward splatting, fused L1 loss and analytic backward.
//
// One CTA of 256 threads owns one 16x16 screen tile of one view; each thread
// owns one pixel. Replaces the two tile_job loops of Renderer::render_view and
// Renderer::backward (renderer.cpp:251-314, 407-500) and the pixel loop of
// render_loss (renderer.cpp:319-371).
//
// Fast path (tile candidate count <= CAP):
//   1. each candidate gets a conservative lower bound z_min of its camera depth
//      over the tile (1/z is affine in pixel coordinates on a plane, so the
//      bound comes from the four corner rays); keys (z_min, plane index) are
//      bitonic-sorted in shared memory;
//   2. the view-dependent plane records (make_prim_views, renderer.cpp:40-58)
//      are built in sorted order in shared memory;
//   3. every pixel keeps the reference's bounded, (z, prim)-ordered top-M list
//      (renderer.cpp:276-290) in local memory, and composites a prefix of it as
//      soon as no later candidate can precede it (z < z_min of the next
//      candidate). A pixel is done when its transmittance is exactly 0 (an
//      interior hit has weight exactly 1, splatting.cpp:22-26) or M records are
//      composited; the tile stops scanning candidates when all pixels are done.
//      Records behind the first opaque one contribute exact zeros to maps and
//      gradients, so this live-prefix evaluation is exact.
//   4. (fused) the pixel-local loss and dL/dmaps; per-view sums are reduced per
//      CTA and added with one atomic per view.
//   5. (fused) reverse sweep over the live records (renderer.cpp:461-495) with
//      per-record gradients pre-reduced across the warp with shuffles when all
//      lanes hit the same plane (else shared-memory atomics), accumulated per
//      candidate slot in shared memory (the reference's per-tile `local`
//      buffers, renderer.cpp:416) and flushed with one global fp64 atomic per
//      (tile, plane, parameter).
// Big tiles (> CAP candidates) take a chunked, unsorted path with the same
// per-pixel list semantics and global atomics.
//
// Precision: Real = float (throughput) or double. In the double build every
// multiply/add that the reference performs is issued as an explicitly rounded
// __dmul_rn/__dadd_rn (no FMA contraction), so maps match the reference to the
// last few ulps (exp() is the only non-correctly-rounded step).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "psg_internal.h"

namespace psg {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ arithmetic
template <typename R>
struct Ar;
template <>
struct Ar<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double ex(double x) { return exp(x); }
    static __device__ __forceinline__ double eps() { return DBL_EPSILON; }
};
template <>
struct Ar<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
    static __device__ __forceinline__ float add(float a, float b) { return a + b; }
    static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
    static __device__ __forceinline__ float ex(float x) { return expf(x); }
    static __device__ __forceinline__ float eps() { return FLT_EPSILON; }
};

template <typename R>
__device__ __forceinline__ R dot3(const R* a, const R* b) {
    using A = Ar<R>;
    return A::add(A::add(A::mul(a[0], b[0]), A::mul(a[1], b[1])), A::mul(a[2], b[2]));
}
__device__ __forceinline__ double dot3_rn(const double* a, const double* b) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])),
                     __dmul_rn(a[2], b[2]));
}

// ------------------------------------------------------------------ records
template <typename R>
struct alignas(16) Cand {
    R n[3], vx[3], vy[3], spo[3];
    R kpn, flip;
    R r[4];
    R mcam[3];
    R q[4];
    int pid;
    short ru0, ru1, rv0, rv1;  // conservative pixel rect from binning (renderer.cpp:71-113)
};

// View-dependent part of make_prim_views (renderer.cpp:51-55) in fp64 with the
// reference's rounding, then narrowed to R.
template <typename R>
__device__ void build_cand(const ViewDev& v, const PlaneGeo& p, int pid, short4 rect,
                           Cand<R>& c) {
    double spo[3];
    for (int k = 0; k < 3; ++k) spo[k] = __dsub_rn(p.c[k], v.t[k]);
    const double kpn = dot3_rn(spo, p.n);
    const double flip = kpn < 0 ? 1.0 : -1.0;
    for (int r = 0; r < 3; ++r) {  // flip * (rot_cw * n), stored-matrix row order a0+(a1+a2)
        const double m = __dadd_rn(__dmul_rn(v.R[r], p.n[0]),
                                   __dadd_rn(__dmul_rn(v.R[3 + r], p.n[1]),
                                             __dmul_rn(v.R[6 + r], p.n[2])));
        c.mcam[r] = R(__dmul_rn(flip, m));
    }
    for (int k = 0; k < 3; ++k) {
        c.n[k] = R(p.n[k]);
        c.vx[k] = R(p.vx[k]);
        c.vy[k] = R(p.vy[k]);
        c.spo[k] = R(spo[k]);
    }
    c.kpn = R(kpn);
    c.flip = R(flip);
    for (int k = 0; k < 4; ++k) {
        c.r[k] = R(p.r[k]);
        c.q[k] = R(p.q[k]);
    }
    c.pid = pid;
    c.ru0 = rect.x;
    c.ru1 = rect.y;
    c.rv0 = rect.z;
    c.rv1 = rect.w;
}

// Lower bound of the camera depth z = k_pn / (dir_un . n) over the tile's pixel
// centres, with slack for rounding in precision R. Returns +inf (as a key) when
// no pixel of the tile can produce t > 0.
template <typename R>
__device__ unsigned zmin_key_bits(const ViewDev& v, const PlaneGeo& p, int u0, int u1, int v0,
                                  int v1) {
    double spo[3];
    for (int k = 0; k < 3; ++k) spo[k] = p.c[k] - v.t[k];
    const double kpn = (spo[0] * p.n[0] + spo[1] * p.n[1]) + spo[2] * p.n[2];
    if (!(fabs(kpn) > 0.0)) return 0x7f800000u;  // camera on the plane: t == 0 everywhere
    double smax = -DBL_MAX, dmax = 0.0;
    const int us[2] = {u0, u1}, vs[2] = {v0, v1};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            double d[3];
            for (int k = 0; k < 3; ++k) d[k] = v.base[k] + us[a] * v.du[k] + vs[b] * v.dv[k];
            const double s = ((d[0] * p.n[0] + d[1] * p.n[1]) + d[2] * p.n[2]) / kpn;
            smax = fmax(smax, s);
            dmax = fmax(dmax, sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]));
        }
    const double eps = double(Ar<R>::eps());
    const double s_hi = smax + fabs(smax) * 64.0 * eps + 64.0 * eps * dmax / fabs(kpn);
    if (!(s_hi > 0.0)) return 0x7f800000u;  // 1/z <= 0 on the whole tile: no hit in front
    const float z = __double2float_rd((1.0 / s_hi) * (1.0 - 64.0 * eps));
    return __float_as_uint(fmaxf(z, 0.0f));
}

// Rectangle kernel (plane_splat_weight, splatting.cpp:12-40) with the per-axis
// weight written as a >= 0 ? 1 : 2*sigmoid(a): identical to the reference after
// its clamp for every a, and keeps interior weights exactly 1 so transmittance
// reaches exactly 0.
template <typename R>
struct Splat {
    R w;      // blended weight in [0,1]
    R dsel;   // d w / d P_sel
    R drsel;  // d w / d r_sel
    int rsel; // index of the radius carrying gradient (0..3)
    bool xsel;
};

template <typename R>
__device__ __forceinline__ R axis_weight(R a) {
    using A = Ar<R>;
    if (a >= R(0)) return R(1);
    return A::mul(R(2), R(1) / A::add(R(1), A::ex(-a)));
}

template <typename R>
__device__ __forceinline__ Splat<R> splat_eval(R px, R py, const R* r, R k) {
    using A = Ar<R>;
    const int bx = px > R(0) ? 0 : 1;
    const int by = py > R(0) ? 2 : 3;
    const R ax = A::mul(k, A::sub(r[bx], fabs(px)));
    const R ay = A::mul(k, A::sub(r[by], fabs(py)));
    const R wx = axis_weight(ax), wy = axis_weight(ay);
    Splat<R> s;
    s.xsel = wx <= wy;
    const R raw = s.xsel ? wx : wy;
    s.w = raw;
    s.rsel = s.xsel ? bx : by;
    s.dsel = R(0);
    s.drsel = R(0);
    if (raw < R(1)) {
        const R sg = A::mul(raw, R(0.5));  // sigmoid value: raw = 2*s exactly
        const R dwdu = A::mul(A::mul(R(2), sg), A::sub(R(1), sg));
        s.drsel = A::mul(dwdu, k);
        const R p = s.xsel ? px : py;
        s.dsel = A::mul(s.drsel, p > R(0) ? R(-1) : R(1));
    }
    return s;
}

struct Ray64 {
    double d[3];
    double mu;
};

template <typename R>
struct PixelRay {
    R d[3];
    R mu;
};

// Pixel ray exactly as render_view forms it (renderer.cpp:265-268).
template <typename R>
__device__ __forceinline__ PixelRay<R> pixel_ray(const ViewDev& v, int u, int w) {
    using A = Ar<R>;
    R dir[3];
    for (int k = 0; k < 3; ++k)
        dir[k] = A::add(A::add(R(v.base[k]), A::mul(R(u), R(v.du[k]))), A::mul(R(w), R(v.dv[k])));
    PixelRay<R> ray;
    const R inv_len = R(1) / sqrt(dot3(dir, dir));
    for (int k = 0; k < 3; ++k) ray.d[k] = A::mul(dir[k], inv_len);
    ray.mu = inv_len;
    return ray;
}

struct EvalParams {
    double k;        // 5 * lambda
    double neg_cut;  // -(arg_cut + 1)
    double floor_, t_near, eps;
};

// eval_candidate (renderer.cpp:159-184).
template <typename R>
__device__ __forceinline__ bool eval_cand(const Cand<R>& c, const PixelRay<R>& ray, R k,
                                          R neg_cut, R floor_, R t_near, R peps, R& z_out,
                                          R& w_out) {
    using A = Ar<R>;
    const R denom = dot3(ray.d, c.n);
    if (fabs(denom) < peps) return false;
    const R t = c.kpn / denom;
    if (t <= t_near) return false;
    R e[3];
    for (int q = 0; q < 3; ++q) e[q] = A::sub(A::mul(t, ray.d[q]), c.spo[q]);
    const R px = dot3(e, c.vx);
    const R ax = A::mul(k, A::sub(px > R(0) ? c.r[0] : c.r[1], fabs(px)));
    if (ax < neg_cut) return false;
    const R py = dot3(e, c.vy);
    const R ay = A::mul(k, A::sub(py > R(0) ? c.r[2] : c.r[3], fabs(py)));
    if (ay < neg_cut) return false;
    const R wx = axis_weight(ax), wy = axis_weight(ay);
    const R w = wx < wy ? wx : wy;
    if (w < floor_) return false;
    z_out = A::mul(t, ray.mu);
    w_out = w;
    return true;
}

// Per-record gradient (renderer.cpp:464-494) for record j of a pixel. The
// rotation terms are regrouped as
//   d_rot[a] = (c*flip*g_Nw - coef_n*e) . J_n[:,a] + (g_w*d_psel*e) . J_sel[:,a],
// which equals the reference's dt_a/dp_a form algebraically.
template <typename R>
__device__ __forceinline__ void record_grad(const Cand<R>& c, const PixelRay<R>& ray, R k, R gD,
                                            const R* gN, R gA, const R* gNw, R Tj, R& S,
                                            R* out) {
    using A = Ar<R>;
    const R denom = dot3(ray.d, c.n);
    const R t = c.kpn / denom;
    const R z = A::mul(t, ray.mu);
    R e[3];
    for (int q = 0; q < 3; ++q) e[q] = A::sub(A::mul(t, ray.d[q]), c.spo[q]);
    const R px = dot3(e, c.vx), py = dot3(e, c.vy);
    const Splat<R> sp = splat_eval(px, py, c.r, k);
    const R phi = A::add(A::add(A::mul(gD, z), dot3(gN, c.mcam)), gA);
    const R g_w = A::mul(Tj, A::sub(phi, S));
    S = A::add(A::mul(sp.w, phi), A::mul(A::sub(R(1), sp.w), S));
    const R cc = A::mul(Tj, sp.w);
    const R g_z = A::mul(cc, gD);
    const R* vsel = sp.xsel ? c.vx : c.vy;
    const R d_dot_vsel = dot3(ray.d, vsel);
    const R gwdp = A::mul(g_w, sp.dsel);
    const R coef_n = A::add(A::mul(gwdp, d_dot_vsel), A::mul(g_z, ray.mu)) / denom;
    for (int q = 0; q < 3; ++q) out[q] = A::sub(A::mul(coef_n, c.n[q]), A::mul(gwdp, vsel[q]));
    R vn[3], vs[3];
    const R cf = A::mul(cc, c.flip);
    for (int q = 0; q < 3; ++q) {
        vn[q] = A::sub(A::mul(cf, gNw[q]), A::mul(coef_n, e[q]));
        vs[q] = A::mul(gwdp, e[q]);
    }
    const R w2 = R(2) * c.q[0], x2 = R(2) * c.q[1], y2 = R(2) * c.q[2], z2 = R(2) * c.q[3];
    // J_n columns (renderer.cpp:399-401)
    const R jn[4][3] = {{y2, -x2, R(0)}, {z2, -w2, -R(2) * x2}, {w2, z2, -R(2) * y2}, {x2, y2, R(0)}};
    R js[4][3];
    if (sp.xsel) {  // J_vx (renderer.cpp:393-395)
        const R t0[4][3] = {{R(0), z2, -y2}, {R(0), y2, z2}, {-R(2) * y2, x2, -w2}, {-R(2) * z2, w2, x2}};
        for (int a = 0; a < 4; ++a)
            for (int q = 0; q < 3; ++q) js[a][q] = t0[a][q];
    } else {  // J_vy (renderer.cpp:396-398)
        const R t1[4][3] = {{-z2, R(0), x2}, {y2, -R(2) * x2, w2}, {x2, R(0), z2}, {-w2, -R(2) * z2, y2}};
        for (int a = 0; a < 4; ++a)
            for (int q = 0; q < 3; ++q) js[a][q] = t1[a][q];
    }
    for (int a = 0; a < 4; ++a) out[3 + a] = A::add(dot3(vn, jn[a]), dot3(vs, js[a]));
    for (int q = 0; q < 4; ++q) out[7 + q] = R(0);
    out[7 + sp.rsel] = A::mul(g_w, sp.drsel);
}

// Warp-cooperative accumulation of 11 gradient values into dst[slot*11 + k].
// All 32 lanes must call this together.
template <typename R, typename D>
__device__ __forceinline__ void warp_accumulate(D* dst, int slot, bool act, const R* g) {
    const unsigned am = __ballot_sync(kFull, act);
    if (am == 0) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(am) - 1;
    const int lslot = __shfl_sync(kFull, slot, leader);
    const bool uniform = __all_sync(kFull, !act || slot == lslot);
    if (uniform) {
#pragma unroll
        for (int q = 0; q < 11; ++q) {
            R v = act ? g[q] : R(0);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
            if (lane == leader && v != R(0)) atomicAdd(dst + size_t(lslot) * 11 + q, D(v));
        }
    } else if (act) {
#pragma unroll
        for (int q = 0; q < 11; ++q)
            if (g[q] != R(0)) atomicAdd(dst + size_t(slot) * 11 + q, D(g[q]));
    }
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

template <typename R>
struct Cap;
template <>
struct Cap<float> {
    static constexpr int value = 256;
};
template <>
struct Cap<double> {
    static constexpr int value = 128;
};

__device__ __forceinline__ double sgn(double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); }

// In-place ascending bitonic sort of n (power of two) 64-bit keys by 256 threads.
__device__ void bitonic_sort(unsigned long long* keys, int n) {
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool asc = (lo & size) == 0;
                const unsigned long long a = keys[lo], b = keys[hi];
                if ((a > b) == asc) {
                    keys[lo] = b;
                    keys[hi] = a;
                }
            }
        }
    }
    __syncthreads();
}

template <typename R>
struct PixelState {
    R lz[kMaxRecordCap];
    R lw[kMaxRecordCap];  // weight while pending, transmittance T_j once composited
    int lref[kMaxRecordCap];
    int cnt, fin;
    R T, D, N[3], Aa;
    bool done;
};

template <typename R, int MODE>
__global__ void __launch_bounds__(kTilePix)
    k_raster(Batch b, const PlaneGeo* __restrict__ planes, int64_t P, Bins bins, RenderParams rp,
             RasterIO io) {
    using A = Ar<R>;
    constexpr int CAP = Cap<R>::value;
    __shared__ unsigned long long s_keys[CAP];
    __shared__ Cand<R> s_cand[CAP];
    __shared__ R s_gacc[MODE == kFused ? CAP * 11 : 1];
    __shared__ double s_red[2][kTilePix / 32];
    __shared__ int s_misc[2];

    const int slot_k = blockIdx.y;
    const ViewDev& v = b.views[b.vid[slot_k]];
    const int tile = blockIdx.x;
    if (tile >= v.tiles_x * v.tiles_y) return;
    const int gt = b.tile_base[slot_k] + tile;
    const int off = bins.offsets[gt];
    const int n = bins.offsets[gt + 1] - off;
    const int* items = bins.items + off;
    const short4* rects = bins.rects + int64_t(slot_k) * P;

    const int tx = tile % v.tiles_x, ty = tile / v.tiles_x;
    const int tu0 = tx * kTile, tv0 = ty * kTile;
    const int tu1 = min(v.W, tu0 + kTile) - 1, tv1 = min(v.H, tv0 + kTile) - 1;
    const int tid = threadIdx.x;
    const int pu = tu0 + (tid & (kTile - 1)), pv = tv0 + (tid >> 4);
    const bool valid = pu < v.W && pv < v.H;

    const R k = R(5.0 * rp.lambda);
    const R neg_cut = R(-(rp.arg_cut + 1.0));
    const R floor_ = R(rp.weight_floor), t_near = R(rp.t_near), peps = R(rp.parallel_eps);
    const int M = rp.max_records;
    const bool fast = n <= CAP;
    const bool allow_finalize = MODE != kFwdRecords && fast;

    PixelState<R> ps;
    ps.cnt = 0;
    ps.fin = 0;
    ps.T = R(1);
    ps.D = R(0);
    ps.N[0] = ps.N[1] = ps.N[2] = R(0);
    ps.Aa = R(0);
    ps.done = !valid;
    const PixelRay<R> ray = pixel_ray<R>(v, pu, pv);

    auto pid_of = [&](int ref) { return fast ? s_cand[ref].pid : ref; };
    auto insert = [&](R z, R w, int ref, int pid) {
        int pos = ps.cnt;
        while (pos > ps.fin &&
               (ps.lz[pos - 1] > z || (ps.lz[pos - 1] == z && pid_of(ps.lref[pos - 1]) > pid)))
            --pos;
        if (pos >= M) return;
        const int last = min(ps.cnt, M - 1);
        for (int s = last; s > pos; --s) {
            ps.lz[s] = ps.lz[s - 1];
            ps.lw[s] = ps.lw[s - 1];
            ps.lref[s] = ps.lref[s - 1];
        }
        ps.lz[pos] = z;
        ps.lw[pos] = w;
        ps.lref[pos] = ref;
        if (ps.cnt < M) ++ps.cnt;
    };
    // front-to-back compositing of list entry fin (renderer.cpp:296-302)
    auto composite_one = [&](const R* mcam) {
        const R w = ps.lw[ps.fin];
        const R cc = A::mul(ps.T, w);
        ps.D = A::add(ps.D, A::mul(cc, ps.lz[ps.fin]));
        for (int q = 0; q < 3; ++q) ps.N[q] = A::add(ps.N[q], A::mul(cc, mcam[q]));
        ps.Aa = A::add(ps.Aa, cc);
        ps.lw[ps.fin] = ps.T;
        ps.T = A::mul(ps.T, A::sub(R(1), w));
        ++ps.fin;
    };

    int n_live = 0;
    if (fast && n > 0) {
        // (1) depth bounds and sort keys
        int npow = 1;
        while (npow < n) npow <<= 1;
        for (int i = tid; i < npow; i += blockDim.x) {
            unsigned long long key = ~0ull;
            if (i < n) {
                const int pid = items[i];
                const unsigned zb = zmin_key_bits<R>(v, planes[pid], tu0, tu1, tv0, tv1);
                key = (static_cast<unsigned long long>(zb) << 32) | unsigned(pid);
            }
            s_keys[i] = key;
        }
        bitonic_sort(s_keys, npow);
        // (2) records in sorted order; culled candidates (key z = +inf) sort last
        for (int i = tid; i < n; i += blockDim.x) {
            const int pid = int(s_keys[i] & 0xffffffffu);
            build_cand<R>(v, planes[pid], pid, rects[pid], s_cand[i]);
        }
        if (tid == 0) {
            int c = n;
            while (c > 0 && unsigned(s_keys[c - 1] >> 32) >= 0x7f800000u) --c;
            s_misc[0] = c;
        }
        if (MODE == kFused)
            for (int i = tid; i < n * 11; i += blockDim.x) s_gacc[i] = R(0);
        __syncthreads();
        n_live = s_misc[0];

        // (3) candidate scan with prefix finalisation and tile early exit
        for (int base = 0; base < n_live; base += 32) {
            if (__syncthreads_and(ps.done)) break;
            if (ps.done) continue;
            const int end = min(base + 32, n_live);
            for (int c = base; c < end; ++c) {
                const Cand<R>& cd = s_cand[c];
                if (allow_finalize) {
                    const R zmin = R(__uint_as_float(unsigned(s_keys[c] >> 32)));
                    while (ps.fin < ps.cnt && ps.lz[ps.fin] < zmin) {
                        composite_one(s_cand[ps.lref[ps.fin]].mcam);
                        if (ps.T == R(0) || ps.fin == M) {
                            ps.done = true;
                            break;
                        }
                    }
                    if (ps.done) break;
                }
                if (unsigned(pu - cd.ru0) > unsigned(cd.ru1 - cd.ru0) ||
                    unsigned(pv - cd.rv0) > unsigned(cd.rv1 - cd.rv0))
                    continue;  // outside the conservative cut-expanded footprint
                R z, w;
                if (!eval_cand(cd, ray, k, neg_cut, floor_, t_near, peps, z, w)) continue;
                if (allow_finalize &&
                    z < R(__uint_as_float(unsigned(s_keys[c] >> 32))) && io.stats)
                    atomicAdd(&io.stats->zviol, 1ull);
                insert(z, w, c, cd.pid);
            }
        }
        // tail: composite what is left (all of it when finalisation is off)
        while (!ps.done && ps.fin < ps.cnt) {
            composite_one(s_cand[ps.lref[ps.fin]].mcam);
            if (MODE != kFwdRecords && (ps.T == R(0) || ps.fin == M)) ps.done = true;
        }
    } else if (n > 0) {
        // big tile: chunks of CAP candidates in bin order, no early exit
        if (tid == 0 && io.stats) atomicAdd(&io.stats->big_tiles, 1ull);
        for (int cb = 0; cb < n; cb += CAP) {
            const int cn = min(CAP, n - cb);
            __syncthreads();
            for (int i = tid; i < cn; i += blockDim.x) {
                const int pid = items[cb + i];
                build_cand<R>(v, planes[pid], pid, rects[pid], s_cand[i]);
            }
            __syncthreads();
            if (!ps.done)
                for (int c = 0; c < cn; ++c) {
                    const Cand<R>& cd = s_cand[c];
                    if (unsigned(pu - cd.ru0) > unsigned(cd.ru1 - cd.ru0) ||
                        unsigned(pv - cd.rv0) > unsigned(cd.rv1 - cd.rv0))
                        continue;
                    R z, w;
                    if (!eval_cand(cd, ray, k, neg_cut, floor_, t_near, peps, z, w)) continue;
                    insert(z, w, cd.pid, cd.pid);
                }
        }
        while (!ps.done && ps.fin < ps.cnt) {
            Cand<R> cd;
            const int pid = ps.lref[ps.fin];
            build_cand<R>(v, planes[pid], pid, rects[pid], cd);
            composite_one(cd.mcam);
            if (MODE != kFwdRecords && (ps.T == R(0) || ps.fin == M)) ps.done = true;
        }
    }

    // ---- outputs: maps and records
    const long long px = (long long)pv * v.W + pu;
    if (valid) {
        if (io.out_depth_f) {
            const long long o = (long long)slot_k * io.map_stride + px;
            io.out_depth_f[o] = float(ps.D);
            io.out_alpha_f[o] = float(ps.Aa);
            io.out_normal_f[3 * o] = float(ps.N[0]);
            io.out_normal_f[3 * o + 1] = float(ps.N[1]);
            io.out_normal_f[3 * o + 2] = float(ps.N[2]);
        }
        if (io.out_depth_d) {
            io.out_depth_d[px] = double(ps.D);
            io.out_alpha_d[px] = double(ps.Aa);
            io.out_normal_d[3 * px] = double(ps.N[0]);
            io.out_normal_d[3 * px + 1] = double(ps.N[1]);
            io.out_normal_d[3 * px + 2] = double(ps.N[2]);
        }
        if (MODE == kFwdRecords) {
            io.rec_count[px] = (unsigned short)ps.cnt;
            for (int j = 0; j < ps.cnt; ++j) io.rec_prim[px * M + j] = pid_of(ps.lref[j]);
            for (int j = ps.cnt; j < M; ++j) io.rec_prim[px * M + j] = -1;
        }
    }
    if (MODE != kFused) return;

    // ---- (4) loss (renderer.cpp:338-369), pixel-local; per-view sums reduced here
    double gD = 0.0, gA = 0.0, gN[3] = {0.0, 0.0, 0.0};
    double sd = 0.0, sn = 0.0;
    if (valid) {
        const double a = double(ps.Aa);
        if (!(a < rp.alpha_floor)) {
            const long long o = v.pix_off + px;
            const bool norm_on = rp.normalize_by_alpha && a > 1e-12;
            const double scale = norm_on ? 1.0 / a : 1.0;
            const float tdv = io.td[o];
            if (tdv > 0.0f) {
                const double dr = double(ps.D) * scale;
                const double diff = dr - double(tdv);
                sd += fabs(diff);
                const double g = rp.alpha2 * sgn(diff) * v.inv_d;
                gD = g * scale;
                if (norm_on) gA -= g * dr * scale;
            }
            const float t0 = io.tn[3 * o], t1 = io.tn[3 * o + 1], t2 = io.tn[3 * o + 2];
            if (t0 != 0.0f || t1 != 0.0f || t2 != 0.0f) {
                const double nr[3] = {double(ps.N[0]) * scale, double(ps.N[1]) * scale,
                                      double(ps.N[2]) * scale};
                const double nt[3] = {double(t0), double(t1), double(t2)};
                const double cos_term = 1.0 - ((nr[0] * nt[0] + nr[1] * nt[1]) + nr[2] * nt[2]);
                sn += fabs(cos_term);
                double g[3];
                for (int q = 0; q < 3; ++q) g[q] = -sgn(cos_term) * nt[q];
                for (int q = 0; q < 3; ++q) {
                    sn += fabs(nr[q] - nt[q]);
                    g[q] += sgn(nr[q] - nt[q]);
                }
                const double gs = rp.alpha1 * v.inv_n;
                for (int q = 0; q < 3; ++q) g[q] *= gs;
                for (int q = 0; q < 3; ++q) gN[q] = g[q] * scale;
                if (norm_on) gA -= ((g[0] * nr[0] + g[1] * nr[1]) + g[2] * nr[2]) * scale;
            }
            // Optimizer::step scales dL/dmaps by 1/views_per_step (optimizer.cpp:73-78)
            gD *= rp.view_scale;
            gA *= rp.view_scale;
            for (int q = 0; q < 3; ++q) gN[q] *= rp.view_scale;
        }
    }
    {
        const double wsd = warp_sum(sd), wsn = warp_sum(sn);
        if ((tid & 31) == 0) {
            s_red[0][tid >> 5] = wsd;
            s_red[1][tid >> 5] = wsn;
        }
        __syncthreads();
        if (tid < 32) {
            double a0 = tid < kTilePix / 32 ? s_red[0][tid] : 0.0;
            double a1 = tid < kTilePix / 32 ? s_red[1][tid] : 0.0;
            a0 = warp_sum(a0);
            a1 = warp_sum(a1);
            if (tid == 0) {
                if (a0 != 0.0) atomicAdd(io.view_loss + 2 * slot_k, a0);
                if (a1 != 0.0) atomicAdd(io.view_loss + 2 * slot_k + 1, a1);
            }
        }
    }
    if (!io.do_backward || n == 0) return;

    // ---- (5) backward: reverse sweep over the live records
    // renderer.cpp:426-433: skip pixels with a zero upstream gradient (Eigen
    // isZero() on g_n means every |component| <= 1e-12).
    const bool active = valid && ps.fin > 0 &&
                        !(gD == 0.0 && gA == 0.0 && fabs(gN[0]) <= 1e-12 &&
                          fabs(gN[1]) <= 1e-12 && fabs(gN[2]) <= 1e-12);
    const int myL = active ? ps.fin : 0;
    const int Lmax = __reduce_max_sync(kFull, myL);
    R rgN[3], rgNw[3];
    for (int q = 0; q < 3; ++q) rgN[q] = R(gN[q]);
    for (int r = 0; r < 3; ++r)  // rot_wc * g_n (renderer.cpp:439), stored-matrix order
        rgNw[r] = R(v.R[3 * r] * gN[0] + (v.R[3 * r + 1] * gN[1] + v.R[3 * r + 2] * gN[2]));
    const R rgD = R(gD), rgA = R(gA);
    R S = R(0);
    for (int r = 0; r < Lmax; ++r) {
        const int j = myL - 1 - r;
        const bool act = j >= 0;
        R g[11];
        int ref = -1;
        if (act) {
            ref = ps.lref[j];
            if (fast) {
                record_grad(s_cand[ref], ray, k, rgD, rgN, rgA, rgNw, ps.lw[j], S, g);
            } else {
                Cand<R> cd;
                build_cand<R>(v, planes[ref], ref, rects[ref], cd);
                record_grad(cd, ray, k, rgD, rgN, rgA, rgNw, ps.lw[j], S, g);
            }
        } else {
            for (int q = 0; q < 11; ++q) g[q] = R(0);
        }
        if (fast)
            warp_accumulate<R, R>(s_gacc, ref, act, g);
        else
            warp_accumulate<R, double>(io.grads, ref, act, g);
    }
    if (!fast) return;
    __syncthreads();
    for (int i = tid; i < n_live * 11; i += blockDim.x) {
        const R val = s_gacc[i];
        if (val != R(0)) atomicAdd(io.grads + size_t(s_cand[i / 11].pid) * 11 + (i % 11), double(val));
    }
}

// Renderer::backward from stored records (renderer.cpp:373-528), one CTA per
// tile; candidate slots are looked up by plane index as slot_of() does
// (renderer.cpp:417-419).
template <typename R>
__global__ void __launch_bounds__(kTilePix)
    k_backward_records(Batch b, const PlaneGeo* __restrict__ planes, int64_t P, Bins bins,
                       RenderParams rp, BackwardIO io) {
    using A = Ar<R>;
    constexpr int CAP = Cap<R>::value;
    __shared__ unsigned long long s_keys[CAP];
    __shared__ Cand<R> s_cand[CAP];
    __shared__ R s_gacc[CAP * 11];

    const ViewDev& v = b.views[b.vid[0]];
    const int tile = blockIdx.x;
    if (tile >= v.tiles_x * v.tiles_y) return;
    const int gt = b.tile_base[0] + tile;
    const int off = bins.offsets[gt];
    const int n = bins.offsets[gt + 1] - off;
    if (n == 0) return;  // renderer.cpp:409-410
    const int* items = bins.items + off;
    const short4* rects = bins.rects;
    const int tx = tile % v.tiles_x, ty = tile / v.tiles_x;
    const int tid = threadIdx.x;
    const int pu = tx * kTile + (tid & (kTile - 1)), pv = ty * kTile + (tid >> 4);
    const bool valid = pu < v.W && pv < v.H;
    const bool fast = n <= CAP;
    const R k = R(5.0 * rp.lambda);
    const int M = io.M;

    int npow = 1;
    if (fast) {
        while (npow < n) npow <<= 1;
        for (int i = tid; i < npow; i += blockDim.x)
            s_keys[i] = i < n ? ((unsigned long long)unsigned(items[i]) << 32) : ~0ull;
        bitonic_sort(s_keys, npow);
        for (int i = tid; i < n; i += blockDim.x) {
            const int pid = int(s_keys[i] >> 32);
            build_cand<R>(v, planes[pid], pid, rects[pid], s_cand[i]);
        }
        for (int i = tid; i < n * 11; i += blockDim.x) s_gacc[i] = R(0);
        __syncthreads();
    }
    auto slot_of = [&](int pid) {
        int lo = 0, hi = n;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s_cand[mid].pid < pid) lo = mid + 1; else hi = mid;
        }
        return (lo < n && s_cand[lo].pid == pid) ? lo : -1;
    };

    const long long px = (long long)pv * v.W + pu;
    int cnt = valid ? min(int(io.rec_count[px]), M) : 0;
    double gD = 0, gA = 0, gN[3] = {0, 0, 0};
    if (cnt > 0) {
        gD = io.d_depth[px];
        gA = io.d_alpha ? io.d_alpha[px] : 0.0;
        for (int q = 0; q < 3; ++q) gN[q] = io.d_normal[3 * px + q];
        if (gD == 0.0 && gA == 0.0 && fabs(gN[0]) <= 1e-12 && fabs(gN[1]) <= 1e-12 &&
            fabs(gN[2]) <= 1e-12)
            cnt = 0;
    }
    const PixelRay<R> ray = pixel_ray<R>(v, pu, pv);
    R lT[kMaxRecordCap];
    int lref[kMaxRecordCap];  // >= 0: shared slot; < 0: -(pid+1), global path
    {
        R T = R(1);
        for (int j = 0; j < cnt; ++j) {
            const int pid = io.rec_prim[px * M + j];
            const int sl = fast ? slot_of(pid) : -1;
            Cand<R> tmp;
            const Cand<R>* cd = &tmp;
            if (sl >= 0) cd = &s_cand[sl]; else build_cand<R>(v, planes[pid], pid, rects[pid], tmp);
            const R denom = dot3(ray.d, cd->n);
            const R t = cd->kpn / denom;
            R e[3];
            for (int q = 0; q < 3; ++q) e[q] = A::sub(A::mul(t, ray.d[q]), cd->spo[q]);
            const Splat<R> sp = splat_eval(dot3(e, cd->vx), dot3(e, cd->vy), cd->r, k);
            lT[j] = T;
            lref[j] = sl >= 0 ? sl : -(pid + 1);
            T = A::mul(T, A::sub(R(1), sp.w));
        }
    }
    R rgN[3], rgNw[3];
    for (int q = 0; q < 3; ++q) rgN[q] = R(gN[q]);
    for (int r = 0; r < 3; ++r)
        rgNw[r] = R(v.R[3 * r] * gN[0] + (v.R[3 * r + 1] * gN[1] + v.R[3 * r + 2] * gN[2]));
    const R rgD = R(gD), rgA = R(gA);
    const int Lmax = __reduce_max_sync(kFull, cnt);
    R S = R(0);
    for (int r = 0; r < Lmax; ++r) {
        const int j = cnt - 1 - r;
        const bool act = j >= 0;
        R g[11];
        int ref = 0;
        bool shared_slot = true;
        if (act) {
            ref = lref[j];
            if (ref >= 0) {
                record_grad(s_cand[ref], ray, k, rgD, rgN, rgA, rgNw, lT[j], S, g);
            } else {
                const int pid = -ref - 1;
                Cand<R> cd;
                build_cand<R>(v, planes[pid], pid, rects[pid], cd);
                record_grad(cd, ray, k, rgD, rgN, rgA, rgNw, lT[j], S, g);
                shared_slot = false;
                ref = pid;
            }
        } else {
            for (int q = 0; q < 11; ++q) g[q] = R(0);
        }
        const bool all_shared = __all_sync(kFull, shared_slot);
        if (all_shared) {
            warp_accumulate<R, R>(s_gacc, ref, act, g);
        } else {
            const int gref = act && shared_slot ? s_cand[ref].pid : ref;
            warp_accumulate<R, double>(io.grads, gref, act, g);
        }
    }
    if (!fast) return;
    __syncthreads();
    for (int i = tid; i < n * 11; i += blockDim.x) {
        const R val = s_gacc[i];
        if (val != R(0)) atomicAdd(io.grads + size_t(s_cand[i / 11].pid) * 11 + (i % 11), double(val));
    }
}

// render_loss (renderer.cpp:319-371) over caller-provided f64 maps.
__global__ void k_loss(const float* __restrict__ td, const float* __restrict__ tn,
                       const double* __restrict__ depth, const double* __restrict__ normal,
                       const double* __restrict__ alpha, RenderParams rp, int np,
                       const unsigned long long* __restrict__ counts, double* d_depth,
                       double* d_normal, double* d_alpha, double* sums) {
    const double inv_d = counts[0] ? 1.0 / double(counts[0]) : 0.0;
    const double inv_n = counts[1] ? 1.0 / double(counts[1]) : 0.0;
    double sd = 0, sn = 0;
    for (int px = blockIdx.x * blockDim.x + threadIdx.x; px < np; px += gridDim.x * blockDim.x) {
        double gD = 0, gA = 0, gN[3] = {0, 0, 0};
        const double a = alpha[px];
        if (!(a < rp.alpha_floor)) {
            const bool norm_on = rp.normalize_by_alpha && a > 1e-12;
            const double scale = norm_on ? 1.0 / a : 1.0;
            if (td[px] > 0.0f) {
                const double dr = depth[px] * scale;
                const double diff = dr - double(td[px]);
                sd += fabs(diff);
                const double g = rp.alpha2 * sgn(diff) * inv_d;
                gD = g * scale;
                if (norm_on) gA -= g * dr * scale;
            }
            const float t0 = tn[3 * px], t1 = tn[3 * px + 1], t2 = tn[3 * px + 2];
            if (t0 != 0.0f || t1 != 0.0f || t2 != 0.0f) {
                const double nr[3] = {normal[3 * px] * scale, normal[3 * px + 1] * scale,
                                      normal[3 * px + 2] * scale};
                const double nt[3] = {double(t0), double(t1), double(t2)};
                const double cos_term = 1.0 - ((nr[0] * nt[0] + nr[1] * nt[1]) + nr[2] * nt[2]);
                sn += fabs(cos_term);
                double g[3];
                for (int q = 0; q < 3; ++q) g[q] = -sgn(cos_term) * nt[q];
                for (int q = 0; q < 3; ++q) {
                    sn += fabs(nr[q] - nt[q]);
                    g[q] += sgn(nr[q] - nt[q]);
                }
                const double gs = rp.alpha1 * inv_n;
                for (int q = 0; q < 3; ++q) g[q] *= gs;
                for (int q = 0; q < 3; ++q) gN[q] = g[q] * scale;
                if (norm_on) gA -= ((g[0] * nr[0] + g[1] * nr[1]) + g[2] * nr[2]) * scale;
            }
        }
        d_depth[px] = gD;
        for (int q = 0; q < 3; ++q) d_normal[3 * px + q] = gN[q];
        if (d_alpha) d_alpha[px] = gA;
    }
    sd = warp_sum(sd);
    sn = warp_sum(sn);
    if ((threadIdx.x & 31) == 0) {
        if (sd != 0.0) atomicAdd(sums, sd);
        if (sn != 0.0) atomicAdd(sums + 1, sn);
    }
}

// Tangent projection and finiteness check (renderer.cpp:516-527).
__global__ void k_finalize(const PlaneGeo* __restrict__ planes, double* grads, int64_t n,
                           unsigned long long* first_bad) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double* g = grads + 11 * i;
    const double* q = planes[i].q;
    const double qd = (q[0] * g[3] + q[2] * g[5]) + (q[1] * g[4] + q[3] * g[6]);
    for (int a = 0; a < 4; ++a) g[3 + a] -= q[a] * qd;
    bool ok = true;
    for (int a = 0; a < 11; ++a) ok = ok && isfinite(g[a]);
    if (!ok) atomicMin(first_bad, (unsigned long long)i);
}

template <typename R, int MODE>
void launch_raster_t(const Batch& b, const PlaneGeo* planes, const Bins& bins,
                     const RenderParams& rp, const RasterIO& io, int64_t P, cudaStream_t s) {
    dim3 grid(unsigned(b.max_tiles), unsigned(b.n));
    k_raster<R, MODE><<<grid, kTilePix, 0, s>>>(b, planes, P, bins, rp, io);
}

}  // namespace

void launch_raster(int precision, RasterMode mode, const Batch& b, const PlaneGeo* planes,
                   int64_t P, const Bins& bins, const RenderParams& rp, const RasterIO& io,
                   cudaStream_t s) {
    if (b.n <= 0 || b.max_tiles <= 0) return;
    if (precision == 0) {
        if (mode == kFused) launch_raster_t<float, kFused>(b, planes, bins, rp, io, P, s);
        else if (mode == kFwdMaps) launch_raster_t<float, kFwdMaps>(b, planes, bins, rp, io, P, s);
        else launch_raster_t<float, kFwdRecords>(b, planes, bins, rp, io, P, s);
    } else {
        if (mode == kFused) launch_raster_t<double, kFused>(b, planes, bins, rp, io, P, s);
        else if (mode == kFwdMaps) launch_raster_t<double, kFwdMaps>(b, planes, bins, rp, io, P, s);
        else launch_raster_t<double, kFwdRecords>(b, planes, bins, rp, io, P, s);
    }
}

void launch_backward_records(int precision, const Batch& b, const PlaneGeo* planes, int64_t P,
                             const Bins& bins, const RenderParams& rp, const BackwardIO& io,
                             cudaStream_t s) {
    if (b.max_tiles <= 0) return;
    if (precision == 0)
        k_backward_records<float><<<b.max_tiles, kTilePix, 0, s>>>(b, planes, P, bins, rp, io);
    else
        k_backward_records<double><<<b.max_tiles, kTilePix, 0, s>>>(b, planes, P, bins, rp, io);
}

void launch_loss(const ViewDev* view, const float* td, const float* tn, const double* depth,
                 const double* normal, const double* alpha, const RenderParams& rp, int W, int H,
                 double* d_depth, double* d_normal, double* d_alpha, double* sums,
                 unsigned long long* counts, cudaStream_t s) {
    launch_target_counts(view, 1, td, tn, counts, s);
    const int np = W * H;
    const int blocks = min(1184, (np + 255) / 256);
    k_loss<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(td, tn, depth, normal, alpha, rp, np, counts,
                                                   d_depth, d_normal, d_alpha, sums);
}

void launch_finalize_grads(const PlaneGeo* planes, double* grads, int64_t n,
                           unsigned long long* first_bad, cudaStream_t s) {
    if (n <= 0) return;
    k_finalize<<<unsigned((n + 255) / 256), 256, 0, s>>>(planes, grads, n, first_bad);
}

}  // namespace psg
