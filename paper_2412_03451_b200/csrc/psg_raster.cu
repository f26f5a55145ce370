// Per-tile rasteriser: forward splatting, fused L1 loss and analytic backward.
//
// One CTA of 256 threads owns one 16x16 screen tile of one view; each thread
// owns one pixel. Replaces the two tile_job loops of Renderer::render_view and
// Renderer::backward (renderer.cpp:251-314, 407-500) and the pixel loop of
// render_loss (renderer.cpp:319-371).
//
// Candidate scan. For every (tile, plane) candidate the CTA stores a 64-byte
// scan record in shared memory: the plane's homography from the tile's pixel
// offsets (a, c) in [0,16)^2 to (D, Nx, Ny), where D = dir_un . n and the
// in-plane offsets are P = N / D and the camera depth is z = k_pn / D (a plane
// maps image coordinates projectively). The coefficients are formed in fp64 per
// (tile, plane) and evaluated per pixel in fp32: two FMAs per quantity and one
// reciprocal, and ~10x less cancellation error than t*d - s_po because every
// term is bounded by the tile's footprint on the plane.
//
// Precision modes (template PREC):
//   0 fp32 : the fp32 homography evaluation decides (throughput mode);
//   1 fp64 : the fp32 evaluation only culls, with margins that can never reject
//            a candidate the exact test accepts; survivors are re-evaluated with
//            the reference's own fp64 expression sequence (explicitly rounded
//            __dmul_rn/__dadd_rn, no FMA contraction), so weights, depths,
//            records and every downstream value follow the reference to the ulp;
//   2 mixed: the fp64 forward of mode 1 (records, maps, loss, and the branch of
//            the rectangle kernel each record took), fp32 backward arithmetic.
//
// Ordering and early exit (fast path, n <= CAP candidates): candidates are
// bitonic-sorted by a conservative lower bound z_min of their depth over the
// tile (1/z is affine in pixel coordinates on a plane, so the four corner rays
// bound it). Each pixel keeps the reference's bounded (z, prim)-ordered top-M
// list (renderer.cpp:276-290) in local memory and composites its prefix as soon
// as no later candidate can precede it (z < z_min of the next candidate). A
// pixel is done when its transmittance is exactly 0 (interior hits weigh exactly
// 1, splatting.cpp:22-26) or M records are composited; the tile stops scanning
// when every pixel is done. Records behind the first opaque one contribute exact
// zeros to maps and gradients, so the live-prefix evaluation is exact.
//
// Backward (fused): pass 1 runs the suffix recursion (renderer.cpp:461-471) per
// pixel over its live records; pass 2 walks the warp's records merged by
// candidate slot (ascending, via __reduce_min_sync), so each (warp, plane) pair
// is reduced once with shuffles and written with 11 native fp64 global
// reductions (REDG.ADD.F64). Shared-memory float atomics are avoided: on sm_100
// they compile to CAS loops (ATOMS.CAST.SPIN).
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdio>
#include <cstdlib>

#include <cfloat>
#include <climits>
#include <cstdint>
#include <algorithm>
#include <mutex>
#include <type_traits>

#include "psg_internal.h"

namespace psg {
namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef PSG_CHUNK
#define PSG_CHUNK 128  // >= the resident cap (one chunk); crowded tiles stream chunks of this size (128: a
                       // smaller shared-memory footprint leaves L1 to their lists; +1 % at lambda 7.36)
#endif
constexpr int kChunk = PSG_CHUNK;  // candidate records staged in shared memory at once
static_assert(kChunk >= kResCapTiles, "resident tiles are one chunk");
constexpr int kResCap = kResCapTiles;  // tiles with up to this many candidates stay resident
constexpr int kKeyCap = 2048;  // crowded tiles with up to this many candidates are depth-sorted

// resident record keys: depth-bound bits << 32 | consumer-warp mask << 8 | record index
// (< kResCap); a warp skips the candidates whose footprint misses its pixel block
constexpr int kKeyMaskShift = 8;
constexpr unsigned kKeyIdxMask = 0xffu;
// build-time switches for A/B variants (scripts/ab_variants.sh); defaults = product
#ifndef PSG_TGT_TMA
#define PSG_TGT_TMA 0  // 1: fp64/mixed fused targets staged by TMA row copies with the records
#endif
// Depth-bound violations (the early-exit contract: no accepted candidate lies in
// front of its own depth-bound key) are counted by the checked build only: the
// compare keeps the key live through the exact test, and that register costs the
// product kernel 7 % at lambda 300 (measured). scripts/cull_audit.py runs whole
// workloads through the checked build.
#ifndef PSG_SLOTS
#define PSG_SLOTS 16
#endif
#ifndef PSG_BIG_PACKED
#define PSG_BIG_PACKED 1  // crowded tiles: 16-byte (z, plane | payload) list entries
#endif
#ifndef PSG_BATCH_EXACT
#define PSG_BATCH_EXACT 1  // exact modes, resident tiles: cull a group of candidates, then run the
                           // exact tests converged (-3 % at lambda 300; +11 % on crowded tiles: off there)
#endif
#ifndef PSG_BATCH_MAX_N
#define PSG_BATCH_MAX_N 128  // ... on tiles with at most this many candidates, in the high-lambda
                             // resident instantiation (the low-lambda one has its own limit, 0:
                             // long lists keep the per-candidate early exit). Measured (C3, fp64,
                             // with the footprint masks): 128 is +0.8 % over 64 at lambda 300 and
                             // +0.4 % at 150; 32 -7 %, none -2 %
#endif
#ifndef PSG_BIG_RECOMPUTE_T
#define PSG_BIG_RECOMPUTE_T 1  // crowded tiles: recompute t in the backward instead of storing it
#endif
#ifndef PSG_RES_MIN_BLOCKS
#define PSG_RES_MIN_BLOCKS 0  // >0: override the resident kernel's CTAs-per-SM register bound
#endif
#ifndef PSG_RING_SLACK
#define PSG_RING_SLACK 8192  // record ring bytes beyond one largest block
#endif
#ifndef PSG_CENTER_ORDER
#define PSG_CENTER_ORDER 1  // crowded tiles: candidates in order of their depth at the tile centre
                            // (closer to each pixel's depth order: fewer list shifts), early exit
                            // on the suffix minima of the depth bounds
#endif
#ifndef PSG_SHIFT_UNROLL
#define PSG_SHIFT_UNROLL 4  // crowded tiles: list entries loaded ahead per shift round trip
#endif
#ifndef PSG_RES_SORT_U
#define PSG_RES_SORT_U 1  // ... and its backward slot sort loads ahead like the crowded tiles'
#endif
#ifndef PSG_BATCH_MAX_N_LOW
#define PSG_BATCH_MAX_N_LOW 0  // ... the group culls' candidate limit in the low-lambda instantiation (off:
                               // +4 % at lambda 54, +1 % at 20; 32 and 128 were slower)
#endif
#ifndef PSG_RES_U_LOW
#define PSG_RES_U_LOW 2  // entries ahead in the low-lambda resident instantiation
#endif
#ifndef PSG_RES_U2_LAMBDA
#define PSG_RES_U2_LAMBDA 100.0  // resident tiles below this lambda: shifts two entries ahead
#endif
#ifndef PSG_SHIFT_UNROLL_RES
#define PSG_SHIFT_UNROLL_RES 1  // resident tiles (short lists; registers are the limit there)
#endif
#ifndef PSG_REF_IN_ENT
#define PSG_REF_IN_ENT 1  // crowded fp64 lists: candidate reference inside the 16-byte entry
#endif
#ifndef PSG_SORT_UNROLL
#define PSG_SORT_UNROLL 4  // crowded tiles: the same for the backward's slot-order insertion sort
#endif
#ifndef PSG_PROBE
#define PSG_PROBE 0  // 1: count per-pixel work (candidates, exact tests, insertions, shifts);
                     // 2: cycles the persistent kernel's warps wait on the record ring
#endif
#ifndef PSG_ZVIOL
#ifdef PSG_CHECKS
#define PSG_ZVIOL 1
#else
#define PSG_ZVIOL 0
#endif
#endif

// ------------------------------------------------------------------ fp64 helpers
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dot3_rn(const double* a, const double* b) {
    return dadd(dadd(dmul(a[0], b[0]), dmul(a[1], b[1])), dmul(a[2], b[2]));
}
__device__ __forceinline__ double dot3d(const double* a, const double* b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

// ------------------------------------------------------------------ records
struct alignas(16) ScanRec {
    float g0, g1, g2, kpn;   // D(a,c) = g2 + a*g0 + c*g1 ; z = kpn / D
    float hx0, hx1, hx2, r0; // Nx(a,c) ; P_x = Nx / D
    float hy0, hy1, hy2, r1; // Ny(a,c) ; P_y = Ny / D
    float r2, r3;
    int ru, rv;              // conservative pixel rect from binning, packed lo | hi << 16
};

// View-dependent plane data (make_prim_views, renderer.cpp:51-55) with the
// reference's rounding: s_po, k_pn, flip, m_cam.
struct PlaneView {
    double spo[3];
    double kpn, flip;
    double mcam[3];
};

__device__ __forceinline__ PlaneView plane_view(const ViewDev& v, const PlaneGeo& p) {
    PlaneView pv;
    for (int k = 0; k < 3; ++k) pv.spo[k] = dsub(p.c[k], v.t[k]);
    pv.kpn = dot3_rn(pv.spo, p.n);
    pv.flip = pv.kpn < 0 ? 1.0 : -1.0;
    for (int r = 0; r < 3; ++r) {  // flip * (rot_cw * n): stored-matrix row order a0 + (a1 + a2)
        const double m = dadd(dmul(v.R[r], p.n[0]), dadd(dmul(v.R[3 + r], p.n[1]), dmul(v.R[6 + r], p.n[2])));
        pv.mcam[r] = dmul(pv.flip, m);
    }
    return pv;
}

// Per-tile constants of the view's ray field: b0 = dir_un at the tile origin and
// an upper bound of |dir_un| over the tile (for the depth-bound slack).
struct TileRays {
    double b0[3];
    double dmax;
    int na, nc;  // pixel extent of the tile minus one (15 except at image borders)
};

__device__ __forceinline__ TileRays tile_rays(const ViewDev& v, int u0, int v0, int u1, int v1) {
    TileRays t;
    for (int k = 0; k < 3; ++k) t.b0[k] = v.base[k] + u0 * v.du[k] + v0 * v.dv[k];
    t.na = u1 - u0;
    t.nc = v1 - v0;
    double dm = 0.0;
    for (int a = 0; a < 2; ++a)
        for (int c = 0; c < 2; ++c) {
            double d[3];
            for (int k = 0; k < 3; ++k) d[k] = t.b0[k] + (a * t.na) * v.du[k] + (c * t.nc) * v.dv[k];
            dm = fmax(dm, dot3d(d, d));
        }
    t.dmax = sqrt(dm);
    return t;
}

__device__ __forceinline__ unsigned zbound_from(double kpn, double g0, double g1, double g2,
                                                const TileRays& tr);

#ifndef PSG_FOOT_MASK
#define PSG_FOOT_MASK 1  // warp masks from the footprint in plane coordinates (0: the pixel rect only)
#endif
#ifndef PSG_FOOT_MASK_BIG
#define PSG_FOOT_MASK_BIG 0  // ... also per staged record of crowded tiles
#endif
// Consumer warps (8x4 pixel blocks of the 16x16 tile) that can hold a pixel whose
// exact test accepts the plane. In plane coordinates the pixel at tile offset
// (a, c) lands on P = N(a, c) / D(a, c) with N, D affine (the scan record's
// homography, here from its fp64 coefficients); every accepted pixel has P inside
// the cut-expanded rectangle [-(r1 + m), r0 + m] x [-(r3 + m), r2 + m], m = (arg_cut
// + 1) / k (eval_candidate's a >= -(arg_cut + 1) on both axes). Where D keeps one
// sign s over a block, "P_x > xhi at every pixel" is "s (N_x - xhi D) > 0", an affine
// function whose minimum over the block is at a corner; likewise for the other
// three sides. A block that such a test puts wholly outside drops out; blocks
// where D comes near zero (grazing rays) stay in.
// footprint margin in plane units for footprint_mask: (arg_cut + 1) / k, widened for
// the rounding of the two evaluations (relative 1e-6, absolute 1e-7)
__host__ __device__ __forceinline__ double foot_cut(const RenderParams& rp) {
    return (rp.arg_cut + 1.0) / (5.0 * rp.lambda) * (1.0 + 1e-6) + 1e-7;
}
__device__ __forceinline__ unsigned footprint_mask(double g0, double g1, double g2, double hx0, double hx1,
                                                   double hx2, double hy0, double hy1, double hy2,
                                                   const PlaneGeo& p, double cut_k) {
    const double sc = fabs(g2) + 15.0 * (fabs(g0) + fabs(g1));
    const double xhi = p.r[0] + cut_k, xlo = -(p.r[1] + cut_k);
    const double yhi = p.r[2] + cut_k, ylo = -(p.r[3] + cut_k);
    // F = N - bound * D, one affine function per side: (f2, f0, f1) = value at the
    // tile origin, per-column and per-row slopes
    const double F[4][3] = {{hx2 - xhi * g2, hx0 - xhi * g0, hx1 - xhi * g1},
                            {hx2 - xlo * g2, hx0 - xlo * g0, hx1 - xlo * g1},
                            {hy2 - yhi * g2, hy0 - yhi * g0, hy1 - yhi * g1},
                            {hy2 - ylo * g2, hy0 - ylo * g0, hy1 - ylo * g1}};
    // the range of an affine f over block w is [lo0, hi0] + a0 f0 + c0 f1, with
    // [lo0, hi0] its range over the block at the origin (7 columns, 3 rows)
    auto range0 = [](double f2, double f0, double f1, double& lo0, double& hi0) {
        lo0 = f2 + fmin(0.0, 7.0 * f0) + fmin(0.0, 3.0 * f1);
        hi0 = f2 + fmax(0.0, 7.0 * f0) + fmax(0.0, 3.0 * f1);
    };
    double dlo0, dhi0;
    range0(g2, g0, g1, dlo0, dhi0);
    double lo0[4], hi0[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) range0(F[q][0], F[q][1], F[q][2], lo0[q], hi0[q]);
    unsigned m = 0;
#pragma unroll 1
    for (int w = 0; w < 8; ++w) {  // not unrolled: registers set the record build's occupancy
        const double a0 = (w & 1) * 8, c0 = (w >> 1) * 4;
        const double od = a0 * g0 + c0 * g1;
        const double dlo = dlo0 + od, dhi = dhi0 + od;
        bool out = false;
        if (dlo > 1e-6 * sc || dhi < -1e-6 * sc) {
            const bool pos = dlo > 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double of = a0 * F[q][1] + c0 * F[q][2];
                const double lo = lo0[q] + of, hi = hi0[q] + of;
                // P beyond an upper bound (q even) at every pixel: F > 0 throughout
                // where D > 0, F < 0 where D < 0; a lower bound (q odd): the reverse
                out |= ((q & 1) == 0) == pos ? lo > 0.0 : hi < 0.0;
            }
        }
        m |= unsigned(!out) << w;
    }
    return m;
}

// Scan record of one (tile, plane) candidate, plus the float bits of a
// conservative lower bound of the plane's camera depth z = k_pn / D over the
// tile's pixel centres (1/z = D / k_pn is affine in (a, c), so its maximum is at
// a corner), with slack for fp32 rounding; +inf when no pixel can hit with t > 0.
// Consumer warps (8x4 blocks of a 16-wide tile or strip with origin (u0, v0)) whose
// block meets the candidate's conservative pixel rect (the scan's per-pixel test).
__device__ __forceinline__ unsigned rect_mask(short4 rect, int u0, int v0) {
    unsigned wm = 0;
    for (int w = 0; w < 8; ++w) {
        const int c0 = u0 + (w & 1) * 8, r0 = v0 + (w >> 1) * 4;
        wm |= unsigned(rect.x <= c0 + 7 && rect.y >= c0 && rect.z <= r0 + 3 && rect.w >= r0) << w;
    }
    return wm;
}

__device__ __forceinline__ unsigned build_scan(const ViewDev& v, const TileRays& tr,
                                               const PlaneGeo& p, short4 rect, ScanRec& s,
                                               unsigned* fmask = nullptr, double cut_k = 0.0) {
    double spo[3];
    for (int k = 0; k < 3; ++k) spo[k] = p.c[k] - v.t[k];
    const double kpn = dot3d(spo, p.n);
    const double g0 = dot3d(v.du, p.n), g1 = dot3d(v.dv, p.n), g2 = dot3d(tr.b0, p.n);
    const double sx = dot3d(spo, p.vx), sy = dot3d(spo, p.vy);
    s.g0 = float(g0);
    s.g1 = float(g1);
    s.g2 = float(g2);
    s.kpn = float(kpn);
    const double hx0 = kpn * dot3d(v.du, p.vx) - sx * g0, hx1 = kpn * dot3d(v.dv, p.vx) - sx * g1,
                 hx2 = kpn * dot3d(tr.b0, p.vx) - sx * g2;
    const double hy0 = kpn * dot3d(v.du, p.vy) - sy * g0, hy1 = kpn * dot3d(v.dv, p.vy) - sy * g1,
                 hy2 = kpn * dot3d(tr.b0, p.vy) - sy * g2;
    s.hx0 = float(hx0);
    s.hx1 = float(hx1);
    s.hx2 = float(hx2);
    s.hy0 = float(hy0);
    s.hy1 = float(hy1);
    s.hy2 = float(hy2);
    if (fmask) *fmask = PSG_FOOT_MASK ? footprint_mask(g0, g1, g2, hx0, hx1, hx2, hy0, hy1, hy2, p, cut_k) : 0xffu;
    s.r0 = float(p.r[0]);
    s.r1 = float(p.r[1]);
    s.r2 = float(p.r[2]);
    s.r3 = float(p.r[3]);
    s.ru = (int(rect.x) & 0xffff) | (int(rect.y) << 16);
    s.rv = (int(rect.z) & 0xffff) | (int(rect.w) << 16);
    return zbound_from(kpn, g0, g1, g2, tr);
}

// Depth-bound key only (streamed tiles sort all candidates before staging records).
__device__ __forceinline__ unsigned zbound_bits(const ViewDev& v, const TileRays& tr, const PlaneGeo& p) {
    double spo[3];
    for (int k = 0; k < 3; ++k) spo[k] = p.c[k] - v.t[k];
    return zbound_from(dot3d(spo, p.n), dot3d(v.du, p.n), dot3d(v.dv, p.n), dot3d(tr.b0, p.n), tr);
}
// The same key plus the plane's depth at the tile centre (the processing order of
// PSG_CENTER_ORDER; +inf where the centre ray misses the plane's front).
__device__ __forceinline__ unsigned zbound_center(const ViewDev& v, const TileRays& tr, const PlaneGeo& p,
                                                  float& zc) {
    double spo[3];
    for (int k = 0; k < 3; ++k) spo[k] = p.c[k] - v.t[k];
    const double kpn = dot3d(spo, p.n), g0 = dot3d(v.du, p.n), g1 = dot3d(v.dv, p.n), g2 = dot3d(tr.b0, p.n);
    const double dc = g2 + 0.5 * (tr.na * g0 + tr.nc * g1);
    const double z = kpn / dc;
    zc = z > 0.0 ? float(z) : CUDART_INF_F;
    return zbound_from(kpn, g0, g1, g2, tr);
}

__device__ __forceinline__ unsigned zbound_from(double kpn, double g0, double g1, double g2,
                                                const TileRays& tr) {
    if (!(fabs(kpn) > 0.0)) return 0x7f800000u;
    const double dhi = g2 + fmax(0.0, tr.na * g0) + fmax(0.0, tr.nc * g1);
    const double dlo = g2 + fmin(0.0, tr.na * g0) + fmin(0.0, tr.nc * g1);
    const double smax = (kpn > 0 ? dhi : dlo) / kpn;  // max over the tile of D / k_pn
    const double eps = double(FLT_EPSILON);
    const double s_hi = smax + fabs(smax) * 64.0 * eps + 64.0 * eps * tr.dmax / fabs(kpn);
    if (!(s_hi > 0.0)) return 0x7f800000u;
    // 1/s_hi rounded down in fp32 (s_hi rounded up first), minus the slack
    const float z = __frcp_rd(__double2float_ru(s_hi)) * (1.0f - 64.0f * FLT_EPSILON);
    return __float_as_uint(fmaxf(z, 0.0f));
}

// ------------------------------------------------------------------ splat kernel
// plane_splat_weight (splatting.cpp:12-40) with the per-axis weight written as
// a >= 0 ? 1 : 2*sigmoid(a): identical to the reference after its clamp for every
// a, and keeps interior weights exactly 1.
__device__ __forceinline__ double axis_w64(double a) {
    if (a >= 0.0) return 1.0;
    return dmul(2.0, 1.0 / dadd(1.0, exp(-a)));
}
__device__ __forceinline__ float axis_w32(float a) {
    if (a >= 0.0f) return 1.0f;
    return 2.0f * __frcp_rn(1.0f + expf(-a));
}

template <typename R>
struct Splat {
    R w, dsel, drsel;
    int rsel;
    bool xsel;
};

template <typename R>
__device__ __forceinline__ Splat<R> splat_eval(R px, R py, const R* r, R k) {
    const int bx = px > R(0) ? 0 : 1;
    const int by = py > R(0) ? 2 : 3;
    R ax, ay;
    if constexpr (sizeof(R) == 8) {
        ax = dmul(k, dsub(r[bx], fabs(px)));
        ay = dmul(k, dsub(r[by], fabs(py)));
    } else {
        ax = k * (r[bx] - fabsf(px));
        ay = k * (r[by] - fabsf(py));
    }
    Splat<R> s;
    s.xsel = ax <= ay;  // = (w_x <= w_y): 2 sigma is monotone
    R raw;
    if constexpr (sizeof(R) == 8) raw = axis_w64(s.xsel ? ax : ay);
    else raw = axis_w32(s.xsel ? ax : ay);
    s.w = raw;
    s.rsel = s.xsel ? bx : by;
    s.dsel = R(0);
    s.drsel = R(0);
    if (raw < R(1)) {
        const R sg = raw * R(0.5);  // sigmoid value: raw = 2*s exactly
        const R dwdu = (R(2) * sg) * (R(1) - sg);
        s.drsel = dwdu * k;
        s.dsel = s.drsel * ((s.xsel ? px : py) > R(0) ? R(-1) : R(1));
    }
    return s;
}

// ------------------------------------------------------------------ pixel state
struct PixelRay {
    double d[3];  // normalised ray (renderer.cpp:265-268), exact reference rounding
    double mu;    // 1/|dir_un|
    float a, c;   // pixel offsets inside the tile
    float L;      // |dir_un|
    float d32[3];
};

__device__ __forceinline__ PixelRay pixel_ray(const ViewDev& v, int u, int w, int u0, int v0) {
    PixelRay r;
    double dir[3];
    for (int k = 0; k < 3; ++k) dir[k] = dadd(dadd(v.base[k], dmul(double(u), v.du[k])), dmul(double(w), v.dv[k]));
    const double len = sqrt(dot3_rn(dir, dir));
    const double inv = 1.0 / len;
    for (int k = 0; k < 3; ++k) {
        r.d[k] = dmul(dir[k], inv);
        r.d32[k] = float(r.d[k]);
    }
    r.mu = inv;
    r.a = float(u - u0);
    r.c = float(w - v0);
    r.L = float(len);
    return r;
}

struct Params32 {
    float k, neg_cut, floor_, t_near, peps;
};

// Branch of the rectangle kernel carrying gradient: the selected axis and the
// side of its radius (r_x+, r_x-, r_y+, r_y-), renderer.cpp / splatting.cpp:25-33.

// fp32 homography test. Returns 0 = reject, 1 = accept with (z, w, rsel),
// 2 = undecided (exact-forward modes: the fp64 test must decide; z = the fp32
// depth, or -1 when the ray is too grazing for it to be trusted).
template <bool kExactFwd>
__device__ __forceinline__ int scan_eval(const ScanRec& s, const PixelRay& ray, const Params32& p,
                                         float& z, float& w, int& rsel) {
    const float D = fmaf(ray.c, s.g1, fmaf(ray.a, s.g0, s.g2));
    if (!kExactFwd) {
        if (fabsf(D) < p.peps * ray.L) return 0;  // |d.n| < parallel_eps
    } else {
        // the sign/size of D is only trusted where fp32 rounding cannot flip it
        z = -1.0f;
        if (!(fabsf(D) > 1e-2f * ray.L)) return 2;  // grazing rays (> 89.4 deg): exact path
    }
    const float rD = __frcp_rn(D);
    const float zz = s.kpn * rD;
    const float t = zz * ray.L;  // t = k_pn / (d . n)
    if (!kExactFwd) {
        if (t <= p.t_near) return 0;
    } else {
        if (t < p.t_near * 0.999f) return 0;
    }
    const float px = fmaf(ray.c, s.hx1, fmaf(ray.a, s.hx0, s.hx2)) * rD;
    const float ax = p.k * ((px > 0.0f ? s.r0 : s.r1) - fabsf(px));
    const float py = fmaf(ray.c, s.hy1, fmaf(ray.a, s.hy0, s.hy2)) * rD;
    const float ay = p.k * ((py > 0.0f ? s.r2 : s.r3) - fabsf(py));
    if (!kExactFwd) {
        if (ax < p.neg_cut || ay < p.neg_cut) return 0;
        // 2 sigma is monotone: min(w_x, w_y) is the weight of min(a_x, a_y), and
        // x_selected (w_x <= w_y) is a_x <= a_y -- one exp instead of two
        const bool xs = ax <= ay;
        const float ww = axis_w32(xs ? ax : ay);
        if (ww < p.floor_) return 0;
        z = zz;
        w = ww;
        rsel = xs ? (px > 0.0f ? 0 : 1) : (py > 0.0f ? 2 : 3);
        return 1;
    } else {
        // w >= floor needs a >= -arg_cut on both axes; margin covers fp32 error
        const float m = 1e-4f * p.k * (fabsf(px) + fabsf(py) + 1.0f) + 1e-3f;
        if (ax < p.neg_cut + 1.0f - m || ay < p.neg_cut + 1.0f - m) return 0;
        z = zz;
        return 2;
    }
}

// View-dependent plane data kept per candidate in shared memory.
struct alignas(16) PV64 {
    double spo[3];
    double kpn, flip;
    double mcam[3];
};
struct alignas(16) PV32 {
    float mcam[3];
    float flip;
};

// The plane geometry the exact test and the fp64 backward read (PlaneGeo without
// the centre), copied into each resident record when PSG_GEO_REC: the producer's
// bulk copy then stages it in shared memory with the record instead of each
// consumer warp loading it through L1.
struct GeoRec {  // PlaneGeo from v_x on (one contiguous 136-byte copy)
    double vx[3], vy[3], n[3], r[4], q[4];
};
static_assert(sizeof(GeoRec) == sizeof(PlaneGeo) - offsetof(PlaneGeo, vx), "GeoRec mirrors PlaneGeo's tail");

__device__ __forceinline__ void store_pv(const PlaneView& pv, PV64& o) {
    for (int k = 0; k < 3; ++k) {
        o.spo[k] = pv.spo[k];
        o.mcam[k] = pv.mcam[k];
    }
    o.kpn = pv.kpn;
    o.flip = pv.flip;
}
__device__ __forceinline__ void store_pv(const PlaneView& pv, PV32& o) {
    for (int k = 0; k < 3; ++k) o.mcam[k] = float(pv.mcam[k]);
    o.flip = float(pv.flip);
}

// eval_candidate (renderer.cpp:159-184) in fp64 with the reference's rounding;
// also returns the gradient-carrying branch of plane_splat_weight.
template <typename G>  // PlaneGeo, or the GeoRec copy staged with a resident record
__device__ __forceinline__ bool exact_eval(const G& p, const PV64& pv, const PixelRay& ray,
                                           double k, double neg_cut, double floor_, double t_near,
                                           double peps, double zcut, double& z, double& w,
                                           double& t_out, int& rsel) {
    const double denom = dot3_rn(ray.d, p.n);
    if (fabs(denom) < peps) return false;
    const double t = pv.kpn / denom;
    if (t <= t_near) return false;
    const double zz = dmul(t, ray.mu);
    if (zz > zcut) return false;  // would not enter the full list (pos == M)
    double e[3];
    for (int q = 0; q < 3; ++q) e[q] = dsub(dmul(t, ray.d[q]), pv.spo[q]);
    const double px = dot3_rn(e, p.vx);
    const double ax = dmul(k, dsub(px > 0 ? p.r[0] : p.r[1], fabs(px)));
    if (ax < neg_cut) return false;
    const double py = dot3_rn(e, p.vy);
    const double ay = dmul(k, dsub(py > 0 ? p.r[2] : p.r[3], fabs(py)));
    if (ay < neg_cut) return false;
    // plane_splat_weight (splatting.cpp:12-40): 2 sigma is monotone, so min(w_x, w_y)
    // is the weight of min(a_x, a_y) and x_selected (w_x <= w_y, ties to X) is
    // a_x <= a_y: one exp instead of two
    const bool xs = ax <= ay;
    const double ww = axis_w64(xs ? ax : ay);
    if (ww < floor_) return false;
    z = zz;
    w = ww;
    t_out = t;
    rsel = xs ? (px > 0 ? 0 : 1) : (py > 0 ? 2 : 3);
    return true;
}

// Jacobians of (v_x, v_y, n) w.r.t. (w,x,y,z) at q (renderer.cpp:393-401), as
// columns; d_rot[a] = vn . J_n[:,a] + vs . J_sel[:,a].
// Every index below is static and the x/y choice selects values, not arrays: a
// dynamic index or pointer select would place `out` (the 11 gradient values)
// and the Jacobians in local memory (measured: ~45 % of the resident kernel's
// local-memory traffic).
template <typename R>
__device__ __forceinline__ void rot_grad(const R* q, const R* vn, const R* vs, bool xsel, R* out) {
    const R w2 = R(2) * q[0], x2 = R(2) * q[1], y2 = R(2) * q[2], z2 = R(2) * q[3];
    const R jn[4][3] = {{y2, -x2, R(0)}, {z2, -w2, -R(2) * x2}, {w2, z2, -R(2) * y2}, {x2, y2, R(0)}};
    const R jx[4][3] = {{R(0), z2, -y2}, {R(0), y2, z2}, {-R(2) * y2, x2, -w2}, {-R(2) * z2, w2, x2}};
    const R jy[4][3] = {{-z2, R(0), x2}, {y2, -R(2) * x2, w2}, {x2, R(0), z2}, {-w2, -R(2) * z2, y2}};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const R js0 = xsel ? jx[a][0] : jy[a][0];
        const R js1 = xsel ? jx[a][1] : jy[a][1];
        const R js2 = xsel ? jx[a][2] : jy[a][2];
        out[3 + a] = (vn[0] * jn[a][0] + vn[1] * jn[a][1] + vn[2] * jn[a][2]) +
                     (vs[0] * js0 + vs[1] * js1 + vs[2] * js2);
    }
}

// plane_splat_weight partials (splatting.cpp:28-38) from the record's weight and
// branch: the selected raw weight is w = 2*s (exact), dw/du = 2 s (1 - s), zero
// once the raw weight reached 1 (clamp).
template <typename R>
__device__ __forceinline__ Splat<R> splat_from(R w, int rsel, R k) {
    Splat<R> sp;
    sp.w = w;
    sp.rsel = rsel;
    sp.xsel = rsel < 2;
    sp.dsel = R(0);
    sp.drsel = R(0);
    if (w < R(1)) {
        const R sg = w * R(0.5);
        const R dwdu = (R(2) * sg) * (R(1) - sg);
        sp.drsel = dwdu * k;
        sp.dsel = (rsel & 1) ? sp.drsel : -sp.drsel;  // -dw/dr for P > 0, + for P <= 0
    }
    return sp;
}

// Per-record gradient (renderer.cpp:464-494) given the suffix-sweep outputs
// g_w = T_j (phi_j - S_j) and T_j. The rotation terms are regrouped as
//   d_rot[a] = (c*flip*g_Nw - coef_n*e) . J_n[:,a] + (g_w*d_psel*e) . J_sel[:,a],
// algebraically equal to the reference's dt_a / dp_a form.
template <typename R>
__device__ __forceinline__ void finish_grad(const R* n, const R* vx, const R* vy, const R* q, R flip,
                                            const R* d, R mu, R denom, const R* e,
                                            const Splat<R>& sp, R gD, const R* gNw, R Tj, R g_w,
                                            R* out) {
    const R cc = Tj * sp.w;
    const R g_z = cc * gD;
    const R cf = cc * flip;
    R vsel[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) vsel[k] = sp.xsel ? vx[k] : vy[k];
    const R d_dot_vsel = (d[0] * vsel[0] + d[1] * vsel[1]) + d[2] * vsel[2];
    const R gwdp = g_w * sp.dsel;
    const R coef_n = (gwdp * d_dot_vsel + g_z * mu) / denom;
    R vn[3], vs[3];
    for (int q3 = 0; q3 < 3; ++q3) {
        out[q3] = coef_n * n[q3] - gwdp * vsel[q3];
        vn[q3] = cf * gNw[q3] - coef_n * e[q3];
        vs[q3] = gwdp * e[q3];
    }
    rot_grad(q, vn, vs, sp.xsel, out);
    const R gr = g_w * sp.drsel;
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) out[7 + q4] = sp.rsel == q4 ? gr : R(0);
}

// Exact-geometry record gradient in precision R (records path, recomputes the splat).
template <typename R>
__device__ __forceinline__ void record_grad_exact(const PlaneGeo& p, const PlaneView& pv,
                                                  const PixelRay& ray, double lambda_k, R gD,
                                                  const R* gNw, R Tj, R g_w, R* out) {
    R d[3], n[3], vx[3], vy[3], q[4], spo[3], r[4];
    for (int k = 0; k < 3; ++k) {
        d[k] = R(ray.d[k]);
        n[k] = R(p.n[k]);
        vx[k] = R(p.vx[k]);
        vy[k] = R(p.vy[k]);
        spo[k] = R(pv.spo[k]);
    }
    for (int k = 0; k < 4; ++k) {
        q[k] = R(p.q[k]);
        r[k] = R(p.r[k]);
    }
    R denom, t, e[3], px, py;
    if constexpr (sizeof(R) == 8) {
        denom = dot3_rn(d, n);
        t = pv.kpn / denom;
        for (int k = 0; k < 3; ++k) e[k] = dsub(dmul(t, d[k]), spo[k]);
        px = dot3_rn(e, vx);
        py = dot3_rn(e, vy);
    } else {
        denom = (d[0] * n[0] + d[1] * n[1]) + d[2] * n[2];
        t = R(pv.kpn) / denom;
        for (int k = 0; k < 3; ++k) e[k] = t * d[k] - spo[k];
        px = (e[0] * vx[0] + e[1] * vx[1]) + e[2] * vx[2];
        py = (e[0] * vy[0] + e[1] * vy[1]) + e[2] * vy[2];
    }
    const Splat<R> sp = splat_eval<R>(px, py, r, R(lambda_k));
    finish_grad<R>(n, vx, vy, q, R(pv.flip), d, R(ray.mu), denom, e, sp, gD, gNw, Tj, g_w, out);
}

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

// 11 gradient values of the lanes in `part` (all 32 lanes call) -> fp64 REDs
// into dst[pid*11 + q]. A single participant writes its values directly;
// otherwise a transposed butterfly (reduce-scatter over lane bits 4..1, then a
// final pair sum) leaves value q on lanes {l : l>>1 == q} after 16 shuffles
// instead of 11*5, and 11 lanes issue the 11 REDs in parallel.
template <typename R>
__device__ __forceinline__ void warp_flush(double* dst, int pid, unsigned part, const R* g,
                                           double* det = nullptr) {
    // det: deterministic mode, the warp's sum goes to its own zeroed slot (plain
    // stores) and a fixed-order reduction follows the launch
    const int lane = threadIdx.x & 31;
    PSG_CHECK(pid >= 0);
    double* base = det ? det : dst + size_t(pid) * 11;
    if (__popc(part) == 1) {  // direct REDs up to 8 participants measured the same
        if ((part >> lane) & 1u)
            for (int q = 0; q < 11; ++q) {
                if (det) base[q] = double(g[q]);  // the slot is not pre-zeroed
                else if (g[q] != R(0)) atomicAdd(base + q, double(g[q]));
            }
        return;
    }
    R v8[8];
    {
        const bool hi = (lane >> 4) & 1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const R lo_v = g[i], hi_v = (i + 8 < 11) ? g[i + 8] : R(0);
            const R send = hi ? lo_v : hi_v;
            const R keep = hi ? hi_v : lo_v;
            v8[i] = keep + __shfl_xor_sync(kFull, send, 16);
        }
    }
    R v4[4];
    {
        const bool hi = (lane >> 3) & 1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const R send = hi ? v8[i] : v8[i + 4];
            const R keep = hi ? v8[i + 4] : v8[i];
            v4[i] = keep + __shfl_xor_sync(kFull, send, 8);
        }
    }
    R v2[2];
    {
        const bool hi = (lane >> 2) & 1;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const R send = hi ? v4[i] : v4[i + 2];
            const R keep = hi ? v4[i + 2] : v4[i];
            v2[i] = keep + __shfl_xor_sync(kFull, send, 4);
        }
    }
    R v1;
    {
        const bool hi = (lane >> 1) & 1;
        const R send = hi ? v2[0] : v2[1];
        const R keep = hi ? v2[1] : v2[0];
        v1 = keep + __shfl_xor_sync(kFull, send, 2);
    }
    v1 += __shfl_xor_sync(kFull, v1, 1);
    const int q = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
    if ((lane & 1) == 0 && q < 11 && (det || v1 != R(0))) {
        if (det) base[q] = double(v1);
        else atomicAdd(base + q, double(v1));
    }
}

__device__ __forceinline__ double sgn(double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); }

// Ascending bitonic sort of n (power of two) 64-bit keys by the whole CTA.
__device__ void bitonic_sort_block(unsigned long long* keys, int n) {
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

// Ascending bitonic sort of 32 keys held one per lane (one warp, no barriers).
__device__ __forceinline__ unsigned long long bitonic_sort_warp(unsigned long long x) {
    const int lane = threadIdx.x & 31;
    for (int size = 2; size <= 32; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const unsigned long long y = __shfl_xor_sync(kFull, x, stride);
            const bool up = (lane & size) == 0;
            const bool low = (lane & stride) == 0;
            const unsigned long long mn = x < y ? x : y, mx = x < y ? y : x;
            x = (up == low) ? mn : mx;
        }
    }
    return x;
}

// ------------------------------------------------------------------ the kernel
// PREC: 0 = fp32 throughout; 1 = exact (fp64 forward decisions, maps and
// backward arithmetic with the reference's rounding); 2 = mixed (exact fp64
// forward decisions, maps and loss; fp32 backward arithmetic).
template <int PREC>
struct Prec {
    static constexpr bool kExactFwd = PREC != 0;
    using FR = typename std::conditional<PREC == 0, float, double>::type;  // forward lists
    using BR = typename std::conditional<PREC == 1, double, float>::type;  // backward math
    using PV = typename std::conditional<PREC == 0, PV32, PV64>::type;
};

constexpr unsigned kRefMask = 0x0fffffffu;  // list entry: candidate index | branch << 28

// Two launches per pass: resident tiles (<= kChunk candidates; all records stay
// in shared memory) on the full (tile, view) grid, and crowded tiles from the
// compacted list built during binning, with room for kKeyCap sorted keys.
template <int PREC, bool BIG>
constexpr size_t raster_smem_bytes() {
    using PV = typename Prec<PREC>::PV;
    return size_t(BIG ? kKeyCap : kChunk) * sizeof(unsigned long long) +
           size_t(kChunk) * (sizeof(ScanRec) + sizeof(PV) + sizeof(int)) + 16 + (BIG ? kChunk : 0) +
           (BIG && PSG_CENTER_ORDER ? size_t(kKeyCap) * sizeof(float) : 0);
}

// Per-pixel top-M list. The (z, prim)-sorted part holds only the depth, the
// plane id and a payload index, packed so one load compares (z, prim) and one
// move shifts an entry; the payload (weight, t, slot|branch, transmittance) stays
// where it was written. A record evicted by the M-truncation hands its payload
// slot to the newcomer. Sorted entries carry g_w after backward pass 1.
template <typename FR>
struct alignas(sizeof(FR) == 8 ? 16 : 8) ListEnt {
    FR z;
    unsigned pl;  // plane id << 6 | payload index
};
// fp64 entries (crowded tiles) carry the candidate reference in the alignment
// padding: it moves with the shifts for free and leaves the payload smaller
template <>
struct alignas(16) ListEnt<double> {
    double z;
    unsigned pl;
    unsigned ref;  // candidate slot | branch << 28
};
template <typename FR>
__device__ __forceinline__ ListEnt<FR> make_ent(FR z, unsigned pl, unsigned ref) {
    if constexpr (sizeof(FR) == 8) return ListEnt<FR>{z, pl, ref};
    else return ListEnt<FR>{z, pl};
}

// fp32 lists pack (z, prim, payload) in 8 bytes; fp64 lists keep the depth
// and a byte payload index in two arrays (a 16-byte entry costs more L1 than the
// rare tie-break's extra loads: measured)
template <typename FR, bool PACKED = sizeof(FR) == 4>
struct PixelSorted;
template <typename FR>
struct PixelSorted<FR, true> {
    ListEnt<FR> e[kMaxRecordCap];  // sorted by (z, prim)
};
template <typename FR>
struct PixelSorted<FR, false> {
    FR lz[kMaxRecordCap];             // sorted: depth
    unsigned char li[kMaxRecordCap];  // sorted: payload index
};

template <typename FR, bool PACKED = sizeof(FR) == 4>
struct PixelList : PixelSorted<FR, PACKED> {
    FR pw[kMaxRecordCap];             // payload: weight
    FR pt[kMaxRecordCap];             // payload: ray parameter t (exact fp64 backward)
    FR pT[kMaxRecordCap];             // payload: transmittance in front (composited)
    unsigned pref[kMaxRecordCap];     // payload: candidate slot | branch << 28
    unsigned kk[kMaxRecordCap];       // backward: slot << 6 | sorted index, slot-ordered
};

template <int PREC, int MODE, bool BIG, bool PRODUCED, int URES = PSG_SHIFT_UNROLL_RES>
__device__ __forceinline__ void raster_tile(const Batch& b, const PlaneGeo* __restrict__ planes,
                                            const PlaneF* __restrict__ planesf, int64_t P,
                                            const Bins& bins, const RenderParams& rp,
                                            const RasterIO& io, int slot_k, int tile,
                                            unsigned long long* s_keys, ScanRec* s_scan,
                                            typename Prec<PREC>::PV* s_pv, int* s_pid,
                                            int* s_nlive, int n_given = 0,
                                            const float* s_tgt = nullptr, const GeoRec* s_geo = nullptr) {
    using FR = typename Prec<PREC>::FR;
    using BR = typename Prec<PREC>::BR;
    using PV = typename Prec<PREC>::PV;
    constexpr bool kExactFwd = Prec<PREC>::kExactFwd;
    constexpr bool kGeoRec = PSG_GEO_REC && PREC != 0;
    const ViewDev& v = b.views[b.vid[slot_k]];
    int tx, ty;
    if constexpr (PRODUCED) {  // the header packs (column, row): tiles_x <= 2048 (W <= 32767)
        tx = tile & 2047;
        ty = tile >> 11;
        tile = ty * v.tiles_x + tx;
    } else {
        if (tile >= v.tiles_x * v.tiles_y) return;
        tx = tile % v.tiles_x;
        ty = tile / v.tiles_x;
    }
    // produced tiles carry their candidate count in the record block header
    const int gt = PRODUCED ? 0 : b.tile_base[slot_k] + tile;
    const int off = PRODUCED ? 0 : bins.offsets[gt];
    const int n = PRODUCED ? n_given : bins.offsets[gt + 1] - off;
    if (!BIG && n > kResCap) return;  // crowded tile: handled by the BIG launch
    const int* items = bins.items + off;
    const short4* rects = bins.rects + int64_t(slot_k) * P;

    const int tu0 = tx * kTile, tv0 = ty * kTile;
    const int tu1 = min(v.W, tu0 + kTile) - 1, tv1 = min(v.H, tv0 + kTile) - 1;
    const int tid = threadIdx.x, lane = tid & 31;
    // a warp covers an 8x4 pixel block (warps 2 across, 4 down the tile): a
    // plane's footprint edge splits fewer warps than with 16x2 rows
    const int wid = tid >> 5;
    const int pcol = (wid & 1) * 8 + (lane & 7), prow = (wid >> 1) * 4 + (lane >> 3);
    const int pix = prow * kTile + pcol;  // row-major pixel index inside the tile
    const int pu = tu0 + pcol, pv = tv0 + prow;
    const bool valid = pu < v.W && pv < v.H;

    Params32 p32;
    p32.k = float(5.0 * rp.lambda);
    p32.neg_cut = float(-(rp.arg_cut + 1.0));
    p32.floor_ = float(rp.weight_floor);
    p32.t_near = float(rp.t_near);
    p32.peps = float(rp.parallel_eps);
    const double k64 = 5.0 * rp.lambda;
    const double negcut64 = -(rp.arg_cut + 1.0);
    const int M = rp.max_records;
    // Tile modes. Resident (n <= kChunk): every record stays in shared memory,
    // list slots index it. Sorted (n <= kKeyCap): depth-sorted keys for all
    // candidates, records streamed in chunks of kChunk, slots are sorted positions.
    // Unsorted (larger): chunks in bin order, no prefix finalisation.
    const int tmode = !BIG ? 0 : (n <= kKeyCap ? 1 : 2);
    const bool resident = !BIG;
    const bool allow_finalize = MODE != kFwdRecords && tmode != 2;

    // crowded tiles (long lists, mostly mid-list insertions at low lambda): packed
    // 16-byte (z, plane | payload) entries, one load and one store per shift
    // (-1.7 % at lambda 20; a cached m_cam per record was +5 %, not kept)
    constexpr bool kPacked = sizeof(FR) == 4 || (BIG && PSG_BIG_PACKED);
    PixelList<FR, kPacked> L;
    // sorted-entry accessors: depth (g_w after pass 1) and payload index
    auto LZ = [&](int j) -> FR& {
        if constexpr (kPacked) return L.e[j].z;
        else return L.lz[j];
    };
    auto LI = [&](int j) -> int {
        if constexpr (kPacked) return int(L.e[j].pl & 63u);
        else return L.li[j];
    };
    // candidate reference of sorted entry j (payload index p = LI(j))
    constexpr bool kRefInEnt = PSG_REF_IN_ENT && kPacked && sizeof(FR) == 8;
    auto LR = [&](int j, int p) -> unsigned {
        if constexpr (kRefInEnt) return L.e[j].ref;
        else return L.pref[p];
    };
    // list length and finalised prefix: registers, outside the local-memory list
    int Lcnt = 0, Lfin = 0;
    FR T = FR(1), Dm = FR(0), Nm[3] = {FR(0), FR(0), FR(0)}, Am = FR(0);
    bool done = !valid;
    static_assert(BIG != PRODUCED, "resident tiles are produced; crowded tiles stream");
    const PixelRay ray = pixel_ray(v, pu, pv, tu0, tv0);
    // tile ray constants, computed only by threads that build candidate records
    TileRays trays_c;
    bool have_trays = false;
    auto trays = [&]() -> const TileRays& {
        if (!have_trays) {
            trays_c = tile_rays(v, tu0, tv0, tu1, tv1);
            have_trays = true;
        }
        return trays_c;
    };
    int cb = 0, cn = 0;  // staged chunk [cb, cb + cn) of slots (streaming modes)
    int total = 0;       // slots to scan

    // bin entry (position in the tile's bin order) of candidate slot sl: sorted
    // crowded tiles key their depth order by entry, so the deterministic partial of
    // a (warp, candidate) lands on the bin entry whose plane the fixed-order
    // reduction attributes it to
    auto entry_of = [&](int sl) -> int { return tmode == 1 ? int(s_keys[sl] & 0xffffffffu) : sl; };
    auto pid_of = [&](unsigned ref) -> int {
        const int sl = int(ref & kRefMask);
        PSG_CHECK(sl < n);
        const int pid = resident ? s_pid[sl] : items[entry_of(sl)];
        PSG_CHECK(pid >= 0 && pid < P);
        return pid;
    };
    auto res_idx = [&](unsigned ref) -> int {
        const int sl = int(ref & kRefMask);
        if (resident) return sl;
        const int r = sl - cb;
        return (r >= 0 && r < cn) ? r : -1;
    };
    auto pv_of = [&](unsigned ref, PV& tmp) -> const PV& {
        const int r = res_idx(ref);
        if (r >= 0) return s_pv[r];
        store_pv(plane_view(v, planes[pid_of(ref)]), tmp);
        return tmp;
    };
    // crowded tiles: per staged record, the consumer warps its footprint can reach
    // (footprint_mask; after s_nlive in the crowded kernel's shared memory)
    unsigned char* s_wm = BIG ? reinterpret_cast<unsigned char*>(s_nlive + 4) : nullptr;
    // PSG_CENTER_ORDER: the depth bounds, by bin entry, then their suffix minima by slot
    float* s_zb = BIG ? reinterpret_cast<float*>(s_wm + kChunk) : nullptr;
    constexpr bool kCenter = BIG && PSG_CENTER_ORDER;
    const double cut_k = foot_cut(rp);
    // stage records of slots [base, base + count) (streaming modes; CTA-wide)
    auto load_chunk = [&](int base, int count) {
        PSG_CHECK(count <= kChunk && base + count <= n);
        __syncthreads();
        for (int i = tid; i < count; i += blockDim.x) {
            const int pid = items[entry_of(base + i)];
            const PlaneGeo& pg = planes[pid];
            if constexpr (BIG && PSG_FOOT_MASK_BIG) {
                unsigned fm = 0xffu;
                build_scan(v, trays(), pg, rects[pid], s_scan[i], &fm, cut_k);
                s_wm[i] = (unsigned char)(fm & rect_mask(rects[pid], tu0, tv0));
            } else {
                build_scan(v, trays(), pg, rects[pid], s_scan[i]);
            }
            store_pv(plane_view(v, pg), s_pv[i]);
            s_pid[i] = pid;  // the scan reads the chunk's plane ids from shared memory
        }
        __syncthreads();
        cb = base;
        cn = count;
    };
    // zlast = depth of the last (farthest) list entry, kept in a register: depth-bound
    // order makes appends the common case, and a full list rejects farther
    // candidates without touching the list
    FR zlast = FR(0);
    unsigned long long pc[12] = {};  // PSG_PROBE counters (dead code otherwise)
    // zfin = depth of the first unfinalised entry (register copy of lz[fin];
    // +inf when every entry is finalised): the per-candidate finalisation test
    // needs no local-memory load. Crowded tiles and the fp32 resident kernel: in
    // the fp64/mixed resident kernels the extra live register costs more than
    // the load (measured: +1 %, fp32 -2.5 %).
    constexpr bool kZfin = BIG || PREC == 0;
    FR zfin = FR(CUDART_INF);
    auto insert = [&](FR z, FR w, FR t, unsigned ref, int pid) {
        // bounded insertion keyed (z, prim) (renderer.cpp:276-291). One pass: the
        // entries after the new one shift up while the position is searched.
        int pos, p;
        if (PSG_PROBE == 1) ++pc[3];
        if (Lcnt == Lfin || z > zlast) {  // append: the common case in depth-bound order
            if (Lcnt == M) {
                if (PSG_PROBE == 1) ++pc[10];
                return;  // farther than the last entry of a full list
            }
            pos = Lcnt;
            p = Lcnt;
            zlast = z;
        } else {
            int s = Lcnt;
            FR znew_last = zlast;
            if (Lcnt == M) {  // full: the last entry drops out if the new one precedes it
                int pid_last;
                if constexpr (kPacked) pid_last = int(L.e[M - 1].pl >> 6);
                else pid_last = z < zlast ? 0 : pid_of(L.pref[L.li[M - 1]]);
                if (!(z < zlast || pid_last > pid)) return;
                s = M - 1;
                p = LI(M - 1);
                znew_last = z;
            } else {
                p = Lcnt;
            }
            const int s0 = s;
            if (PSG_PROBE == 1) ++pc[4];
            // entries after the new one's place move up one. The dependent chain is
            // a local-memory round trip per entry (the lists of a crowded tile's
            // pixels outgrow L1), so the loads of the next U entries are issued
            // together, ahead of the compares and the stores (crowded tiles, U = 4:
            // +13 % at lambda 7.36, +9 % at lambda 20; resident tiles keep U = 1, the
            // registers cost 6 % at lambda 300)
            constexpr int U = BIG ? PSG_SHIFT_UNROLL : URES;
            bool moving = true;
            while (moving && s > Lfin) {
                FR zq[U];
                ListEnt<FR> eq[U];
                unsigned char liq[U];
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const int j = max(s - 1 - k, 0);  // below Lfin: loaded, never used
                    if constexpr (kPacked) {
                        eq[k] = L.e[j];
                        zq[k] = eq[k].z;
                    } else {
                        zq[k] = L.lz[j];
                        liq[k] = L.li[j];
                    }
                }
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    if (s <= Lfin) {
                        moving = false;
                        break;
                    }
                    if (PSG_PROBE == 1) ++pc[5];
                    const FR zp = zq[k];
                    if constexpr (kPacked) {
                        if (!(zp > z || (zp == z && int(eq[k].pl >> 6) > pid))) {
                            moving = false;
                            break;
                        }
                    } else {
                        if (!(zp > z || (zp == z && pid_of(L.pref[liq[k]]) > pid))) {
                            moving = false;
                            break;
                        }
                    }
                    if (s == s0 && Lcnt == M) znew_last = zp;  // moves into the last place
                    if constexpr (kPacked) {
                        L.e[s] = eq[k];
                    } else {
                        L.lz[s] = zp;
                        L.li[s] = liq[k];
                    }
                    --s;
                }
            }
            pos = s;
            if (Lcnt == M) zlast = znew_last;
            else if (pos == Lcnt) zlast = z;
        }
        PSG_CHECK(pos >= Lfin && pos < M && p >= 0 && p < M && M <= kMaxRecordCap);
        if constexpr (kPacked) {
            L.e[pos] = make_ent<FR>(z, (unsigned(pid) << 6) | unsigned(p), ref);
        } else {
            L.lz[pos] = z;
            L.li[pos] = (unsigned char)p;
        }
        if (kZfin && pos == Lfin) zfin = z;
        L.pw[p] = w;
        if (PREC == 1 && !(BIG && PSG_BIG_RECOMPUTE_T)) L.pt[p] = t;
        if constexpr (!kRefInEnt) L.pref[p] = ref;
        if (Lcnt < M) ++Lcnt;
    };
    // front-to-back compositing of entry fin (renderer.cpp:296-302)
    auto composite_one = [&]() {
        const int j = Lfin;
        const int p = LI(j);
        const FR w = L.pw[p];
        if constexpr (kExactFwd) {
            PV tmp;
            const PV& q = pv_of(LR(j, p), tmp);
            const double cc = dmul(T, w);
            Dm = dadd(Dm, dmul(cc, LZ(j)));
            for (int k3 = 0; k3 < 3; ++k3) Nm[k3] = dadd(Nm[k3], dmul(cc, q.mcam[k3]));
            Am = dadd(Am, cc);
        } else {
            PV tmp;
            const PV& q = pv_of(LR(j, p), tmp);
            const float cc = T * w;
            Dm += cc * LZ(j);
            for (int k3 = 0; k3 < 3; ++k3) Nm[k3] += cc * q.mcam[k3];
            Am += cc;
        }
        L.pT[p] = T;
        T = T * (FR(1) - w);
        ++Lfin;
        if (kZfin) zfin = Lfin < Lcnt ? LZ(Lfin) : FR(CUDART_INF);
    };
#ifdef PSG_CHECKS
    // checked build: every candidate the per-pixel footprint rect or the fp32 cull
    // rejects is re-tested with the exact fp64 test; an acceptance is a cull miss
    unsigned long long n_cull_checks = 0, n_cull_miss = 0;
    auto cull_audit = [&](const PV& pvr, int pid, double zcut) {
        if constexpr (kExactFwd) {
            double z, w, t;
            int rs;
            ++n_cull_checks;
            if (exact_eval(planes[pid], pvr, ray, k64, negcut64, rp.weight_floor, rp.t_near,
                           rp.parallel_eps, zcut, z, w, t, rs))
                ++n_cull_miss;
        }
    };
#endif
    // evaluate candidate `slot` (scan record s, view data pvr) for this pixel; zmin =
    // the candidate's depth-bound key (-inf where order is not used): an accepted
    // depth below it would break the prefix finalisation (counted, must stay 0)
    // the exact fp64 test of a candidate the fp32 cull could not reject, and its insertion
    auto exact_insert = [&](const PV& pvr, int slot, int pid, FR zmin) {
        if constexpr (kExactFwd) {
            double z, w, t;
            int rsel = 0;
            // a full list cannot take a candidate farther than its last entry
            const double zcut = (Lcnt == M && Lcnt > Lfin) ? double(zlast) : CUDART_INF;
            if (PSG_PROBE == 1) ++pc[1];
            bool acc;
            if (!BIG && kGeoRec)
                acc = exact_eval(s_geo[slot], pvr, ray, k64, negcut64, rp.weight_floor, rp.t_near, rp.parallel_eps,
                                 zcut, z, w, t, rsel);
            else
                acc = exact_eval(planes[pid], pvr, ray, k64, negcut64, rp.weight_floor, rp.t_near, rp.parallel_eps,
                                 zcut, z, w, t, rsel);
            if (!acc) {
                if (PSG_PROBE == 1) ++pc[zcut < CUDART_INF ? 2 : 9];
                return;
            }
            if (PSG_ZVIOL && z < zmin) atomicAdd(&io.stats->zviol, 1ull);
            insert(z, w, t, unsigned(slot) | (unsigned(rsel) << 28), pid);
        }
    };
    // footprint rect + fp32 cull: 0 reject, 1 accept (fp32 mode, inserted here),
    // 2 undecided (exact modes: exact_insert decides)
    auto cull = [&](const ScanRec& s, const PV& pvr, int slot, int pid, FR zmin) -> int {
        if (PSG_PROBE == 1) ++pc[0];
        const unsigned du = unsigned(pu - (s.ru & 0xffff)), dv = unsigned(pv - (s.rv & 0xffff));
        if (du > unsigned((s.ru >> 16) - (s.ru & 0xffff)) || dv > unsigned((s.rv >> 16) - (s.rv & 0xffff))) {
#ifdef PSG_CHECKS
            cull_audit(pvr, pid, CUDART_INF);
#endif
            return 0;  // outside the conservative cut-expanded footprint
        }
        float z32 = 0.f, w32 = 0.f;
        int rsel = 0;
        const int st = scan_eval<kExactFwd>(s, ray, p32, z32, w32, rsel);
        if (st == 0) {
#ifdef PSG_CHECKS
            cull_audit(pvr, pid, CUDART_INF);
#endif
            return 0;
        }
        if constexpr (!kExactFwd) {
            if (PSG_ZVIOL && z32 < zmin) atomicAdd(&io.stats->zviol, 1ull);
            insert(z32, w32, FR(0), unsigned(slot) | (unsigned(rsel) << 28), pid);
        }
        return st;
    };
    // evaluate candidate `slot` (scan record s, view data pvr) for this pixel
    auto consider = [&](const ScanRec& s, const PV& pvr, int slot, int pid, FR zmin) {
        if (cull(s, pvr, slot, pid, zmin) == 2) exact_insert(pvr, slot, pid, zmin);
    };

    if (n > 0) {
        // (1) depth keys (+ resident records) and the depth-bound sort
        if (PRODUCED) {
            total = *s_nlive;  // the producer warp built, sorted and counted the records
        } else if (tmode != 2) {
            // crowded tiles (BIG): depth keys of the live candidates (compacted: the
            // sort and the streamed chunks skip the rest), records streamed later
            if (tid == 0) *s_nlive = 0;
            __syncthreads();
            for (int i0 = 0; i0 < n; i0 += blockDim.x) {
                const int i = i0 + tid;
                unsigned zb = 0x7f800000u;
                unsigned kz = 0x7f800000u;  // sort key: the bound, or the centre depth
                if (i < n) {
                    if constexpr (kCenter) {
                        float zc;
                        zb = zbound_center(v, trays(), planes[items[i]], zc);
                        s_zb[i] = __uint_as_float(zb);
                        kz = zb < 0x7f800000u ? __float_as_uint(fminf(zc, 3.0e38f)) : 0x7f800000u;
                    } else {
                        zb = zbound_bits(v, trays(), planes[items[i]]);
                        kz = zb;
                    }
                }
                const bool live = zb < 0x7f800000u;
                const unsigned bal = __ballot_sync(kFull, live);
                int base = 0;
                if (lane == 0 && bal) base = atomicAdd(s_nlive, __popc(bal));
                base = __shfl_sync(kFull, base, 0);
                if (live)
                    s_keys[base + __popc(bal & ((1u << lane) - 1u))] =
                        (static_cast<unsigned long long>(kz) << 32) | unsigned(i);
            }
            __syncthreads();
            total = *s_nlive;
            int npow = 2;
            while (npow < total) npow <<= 1;
            for (int i = total + tid; i < npow; i += blockDim.x) s_keys[i] = ~0ull;
            bitonic_sort_block(s_keys, npow);  // keys carry the entry: the order is unique
            if constexpr (kCenter) {
                // suffix minima of the bounds in processing order: the early exit's lower
                // bound for every later candidate. Thread t owns slots [t*E, t*E + E).
                constexpr int E = kKeyCap / kTilePix;
                float loc[E];
                float m = CUDART_INF_F;
#pragma unroll
                for (int j = E - 1; j >= 0; --j) {
                    const int sl = tid * E + j;
                    const float zv = sl < total ? s_zb[int(s_keys[sl] & 0xffffffffu)] : CUDART_INF_F;
                    m = fminf(m, zv);
                    loc[j] = m;
                }
                // exclusive suffix minimum over the later threads' runs
                float cw = __shfl_down_sync(kFull, m, 1);
                if (lane == 31) cw = CUDART_INF_F;
                for (int o = 1; o < 32; o <<= 1) {
                    const float y = __shfl_down_sync(kFull, cw, o);
                    if (lane + o < 32) cw = fminf(cw, y);
                }
                const float wtot = __shfl_sync(kFull, fminf(m, cw), 0);  // this warp's whole run
                __shared__ float s_wmin[kTilePix / 32];
                if (lane == 0) s_wmin[wid] = wtot;
                __syncthreads();  // (also: every s_zb read above is done)
                float later = CUDART_INF_F;
                for (int w2 = wid + 1; w2 < kTilePix / 32; ++w2) later = fminf(later, s_wmin[w2]);
                const float carry = fminf(cw, later);
#pragma unroll
                for (int j = 0; j < E; ++j) s_zb[tid * E + j] = fminf(loc[j], carry);
                __syncthreads();
            }
        } else {
            total = n;
        }
        if (resident) {
            cb = 0;
            cn = n;
        }
        // (2) candidate scan (depth-bound order unless unsorted), prefix
        // finalisation, tile early exit
        for (int chunk = 0; chunk < total; chunk += kChunk) {
            const int ccount = min(kChunk, total - chunk);
            if (chunk > 0 && __syncthreads_and(done)) break;
            if (!resident) load_chunk(chunk, ccount);
            for (int base = chunk; base < chunk + ccount; base += 32) {
                // a warp whose pixels are all finished stops scanning; no CTA barrier
                // here, the streamed path re-synchronises only between chunks
                if (__all_sync(kFull, done)) break;
                if (done) continue;
                const int end = min(base + 32, chunk + ccount);
                if (kExactFwd && PSG_BATCH_EXACT && !BIG && n <= (URES > 1 ? PSG_BATCH_MAX_N_LOW : PSG_BATCH_MAX_N)) {
                    // (a) the group's fp32 culls for this pixel -> survivor mask; (b) the
                    // exact tests of the survivors with the warp converged, each lane on its
                    // own next survivor: lanes whose survivors are different candidates run
                    // their fp64 tests together instead of one candidate at a time. The
                    // prefix is finalised against each survivor's own depth bound (the
                    // culled candidates in between insert nothing), so the early exit stays.
                    auto finalize_to = [&](FR zmin) {
                        while (kZfin ? zfin < zmin : (Lfin < Lcnt && LZ(Lfin) < zmin)) {
                            composite_one();
                            if (T == FR(0) || Lfin == M) {
                                done = true;
                                break;
                            }
                        }
                    };
                    if (allow_finalize) {
                        finalize_to(FR(__uint_as_float(unsigned(s_keys[base] >> 32))));
                        if (done) continue;
                    }
                    unsigned surv = 0;
                    for (int c = base; c < end; ++c) {
                        if (resident) {
                            const unsigned klo = unsigned(s_keys[c]);
                            if (!((klo >> (kKeyMaskShift + (tid >> 5))) & 1u)) {  // block misses it
#ifdef PSG_CHECKS
                                const int ia = int(klo & kKeyIdxMask);
                                cull_audit(s_pv[ia], s_pid[ia], CUDART_INF);
#endif
                                continue;
                            }
                            const int idx = int(klo & kKeyIdxMask);
                            if (cull(s_scan[idx], s_pv[idx], idx, s_pid[idx], FR(-CUDART_INF)) == 2)
                                surv |= 1u << (c - base);
                        } else {
                            const int r = c - chunk;
                            if (cull(s_scan[r], s_pv[r], c, s_pid[r], FR(-CUDART_INF)) == 2)
                                surv |= 1u << (c - base);
                        }
                    }
                    while (surv) {
                        const int c = base + __ffs(surv) - 1;
                        surv &= surv - 1;
                        FR zmin = FR(-CUDART_INF);
                        if (allow_finalize) {
                            zmin = FR(__uint_as_float(unsigned(s_keys[c] >> 32)));
                            finalize_to(zmin);
                            if (done) break;
                        }
                        if (resident) {
                            const int idx = int(unsigned(s_keys[c]) & kKeyIdxMask);
                            exact_insert(s_pv[idx], idx, s_pid[idx], zmin);
                        } else {
                            const int r = c - chunk;
                            exact_insert(s_pv[r], c, s_pid[r], zmin);
                        }
                    }
                    continue;
                }
                for (int c = base; c < end; ++c) {
                    FR zmin = FR(-CUDART_INF);
                    if (allow_finalize) {
                        zmin = kCenter ? FR(s_zb[c]) : FR(__uint_as_float(unsigned(s_keys[c] >> 32)));
                        while (kZfin ? zfin < zmin : (Lfin < Lcnt && LZ(Lfin) < zmin)) {
                            composite_one();
                            if (T == FR(0) || Lfin == M) {
                                done = true;
                                break;
                            }
                        }
                        if (done) break;
                    }
                    if (resident) {
                        const unsigned klo = unsigned(s_keys[c]);
                        if (!((klo >> (kKeyMaskShift + (tid >> 5))) & 1u)) {  // block misses it
#ifdef PSG_CHECKS
                            const int ia = int(klo & kKeyIdxMask);
                            cull_audit(s_pv[ia], s_pid[ia], CUDART_INF);
#endif
                            continue;
                        }
                        const int idx = int(klo & kKeyIdxMask);
                        consider(s_scan[idx], s_pv[idx], idx, s_pid[idx], zmin);
                    } else {
                        const int r = c - chunk;
                        if (PSG_FOOT_MASK_BIG && !((s_wm[r] >> wid) & 1u)) {  // the footprint misses the block
#ifdef PSG_CHECKS
                            cull_audit(s_pv[r], s_pid[r], CUDART_INF);
#endif
                            continue;
                        }
                        consider(s_scan[r], s_pv[r], c, s_pid[r], zmin);
                    }
                }
            }
        }
    }
#ifdef PSG_CHECKS
    {
        const unsigned long long wc = __reduce_add_sync(kFull, unsigned(n_cull_checks)),
                                 wm = __reduce_add_sync(kFull, unsigned(n_cull_miss));
        if (lane == 0 && wc) atomicAdd(&io.stats->cull_checks, wc);
        if (lane == 0 && wm) atomicAdd(&io.stats->cull_miss, wm);
    }
#endif
    if (PSG_PROBE == 1) {
        pc[6] += valid && done;
        pc[7] += valid && Lcnt == M;
        pc[8] += valid;
        pc[11] += valid ? (unsigned long long)n : 0ull;
        for (int q = 0; q < 12; ++q) {
            unsigned long long x = pc[q];
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
            if (lane == 0 && x) atomicAdd(&io.stats->probe[q], x);
        }
    }
    // tail: composite what is left (everything when finalisation is off)
    while (!done && Lfin < Lcnt) {
        composite_one();
        if (MODE != kFwdRecords && (T == FR(0) || Lfin == M)) done = true;
    }

    // ---- outputs: maps and records
    const long long px = (long long)pv * v.W + pu;
    if (valid) {
        if (io.out_depth_f) {
            const long long o = (long long)slot_k * io.map_stride + px;
            io.out_depth_f[o] = float(Dm);
            io.out_alpha_f[o] = float(Am);
            io.out_normal_f[3 * o] = float(Nm[0]);
            io.out_normal_f[3 * o + 1] = float(Nm[1]);
            io.out_normal_f[3 * o + 2] = float(Nm[2]);
        }
        if (io.out_depth_d) {
            io.out_depth_d[px] = double(Dm);
            io.out_alpha_d[px] = double(Am);
            io.out_normal_d[3 * px] = double(Nm[0]);
            io.out_normal_d[3 * px + 1] = double(Nm[1]);
            io.out_normal_d[3 * px + 2] = double(Nm[2]);
        }
        if (MODE == kFwdRecords) {
            io.rec_count[px] = (unsigned short)Lcnt;
            for (int j = 0; j < Lcnt; ++j) io.rec_prim[px * M + j] = pid_of(LR(j, LI(j)));
            for (int j = Lcnt; j < M; ++j) io.rec_prim[px * M + j] = -1;
        }
    }
    if (MODE != kFused && MODE != kFusedDet) return;
    constexpr bool kDet = MODE == kFusedDet;

    // ---- (4) loss (renderer.cpp:338-369), pixel-local; warp sums -> one RED per warp
    double gD = 0.0, gA = 0.0, gN[3] = {0.0, 0.0, 0.0};
    double sd = 0.0, sn = 0.0;
    if (valid) {
        const double a = double(Am);
        if (!(a < rp.alpha_floor)) {
            const long long o = v.pix_off + px;
            const bool norm_on = rp.normalize_by_alpha && a > 1e-12;
            const double scale = norm_on ? 1.0 / a : 1.0;
            // targets: staged in shared memory by the producer's TMA row copies
            // ([16 rows x 16 px] depth, then normals), else from HBM
            const float tdv = s_tgt ? s_tgt[pix] : io.td[o];
            if (tdv > 0.0f) {
                const double dr = double(Dm) * scale;
                const double diff = dr - double(tdv);
                sd += fabs(diff);
                const double g = rp.alpha2 * sgn(diff) * v.inv_d;
                gD = g * scale;
                if (norm_on) gA -= g * dr * scale;
            }
            const float* tnp = s_tgt ? s_tgt + kTilePix + 3 * pix : io.tn + 3 * o;
            const float t0 = tnp[0], t1 = tnp[1], t2 = tnp[2];
            if (t0 != 0.0f || t1 != 0.0f || t2 != 0.0f) {
                const double nr[3] = {double(Nm[0]) * scale, double(Nm[1]) * scale, double(Nm[2]) * scale};
                const double nt[3] = {double(t0), double(t1), double(t2)};
                const double cos_term = 1.0 - dot3d(nr, nt);
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
                if (norm_on) gA -= dot3d(g, nr) * scale;
            }
            // Optimizer::step scales dL/dmaps by 1/views_per_step (optimizer.cpp:73-78)
            gD *= rp.view_scale;
            gA *= rp.view_scale;
            for (int q = 0; q < 3; ++q) gN[q] *= rp.view_scale;
        }
    }
    {
        const double wsd = warp_sum(sd), wsn = warp_sum(sn);
        const unsigned wl = __reduce_add_sync(kFull, valid ? unsigned(Lfin) : 0u);
        if (lane == 0) {
            if (kDet) {  // deterministic mode: per-(tile, warp) partials, reduced in order
                double* dl = io.det_loss + ((long long)(b.tile_base[slot_k] + tile) * 8 + wid) * 2;
                dl[0] = wsd;
                dl[1] = wsn;
            } else {
                if (wsd != 0.0) atomicAdd(io.view_loss + 2 * slot_k, wsd);
                if (wsn != 0.0) atomicAdd(io.view_loss + 2 * slot_k + 1, wsn);
            }
            if (wl) atomicAdd(&io.stats->live, (unsigned long long)wl);
        }
    }
    if (!io.do_backward || n == 0) return;

    // ---- (5) backward. Skip pixels with a zero upstream gradient
    // (renderer.cpp:426-433; Eigen isZero() on g_n: every |component| <= 1e-12).
    const bool active = valid && Lfin > 0 &&
                        !(gD == 0.0 && gA == 0.0 && fabs(gN[0]) <= 1e-12 && fabs(gN[1]) <= 1e-12 &&
                          fabs(gN[2]) <= 1e-12);
    // no CTA barriers follow: crowded tiles rebuild a record the forward's last
    // staged chunk does not hold (pv_of / build_scan) instead of re-streaming
    if (__ballot_sync(kFull, active) == 0) return;
    const int nrec = active ? Lfin : 0;
    const int det_off = kDet ? bins.offsets[b.tile_base[slot_k] + tile] : 0;
    // pass 1: suffix recursion (renderer.cpp:441-471) -> g_w per record into lz
    {
        FR S = FR(0);
        for (int j = nrec - 1; j >= 0; --j) {
            const int p = LI(j);
            PV tmp;
            const PV& q = pv_of(LR(j, p), tmp);
            const FR phi = (FR(gD) * LZ(j) +
                            (FR(gN[0]) * FR(q.mcam[0]) + FR(gN[1]) * FR(q.mcam[1]) + FR(gN[2]) * FR(q.mcam[2]))) +
                           FR(gA);
            const FR w = L.pw[p];
            LZ(j) = L.pT[p] * (phi - S);
            S = w * phi + (FR(1) - w) * S;
        }
    }
    // order this pixel's live records by slot for the warp merge (32-bit keys)
    for (int i = 0; i < nrec; ++i) {
        const unsigned key = ((LR(i, LI(i)) & kRefMask) << 6) | unsigned(i);
        int j = i - 1;
        constexpr int US = (BIG || (URES > 1 && PSG_RES_SORT_U)) ? PSG_SORT_UNROLL : 1;  // loads ahead, as in insert
        if constexpr (US == 1) {
            while (j >= 0 && L.kk[j] > key) {
                L.kk[j + 1] = L.kk[j];
                --j;
            }
        } else {
            bool moving = true;
            while (moving && j >= 0) {
                unsigned kq[US];
#pragma unroll
                for (int k = 0; k < US; ++k) kq[k] = L.kk[max(j - k, 0)];
#pragma unroll
                for (int k = 0; k < US; ++k) {
                    if (j < 0 || kq[k] <= key) {
                        moving = false;
                        break;
                    }
                    L.kk[j + 1] = kq[k];
                    --j;
                }
            }
        }
        L.kk[j + 1] = key;
    }
    BR gNw[3];
    for (int r = 0; r < 3; ++r)  // rot_wc * g_n (renderer.cpp:439), stored-matrix order
        gNw[r] = BR(v.R[3 * r] * gN[0] + (v.R[3 * r + 1] * gN[1] + v.R[3 * r + 2] * gN[2]));
    // pass 2: warp-merged by slot; one reduction + 11 fp64 REDs per (warp, plane).
    // Streaming modes walk the slots chunk by chunk so every record is staged.
    int ptr = 0;
    // the lane's next record, staged in registers one iteration ahead so its
    // local-memory loads overlap the previous iteration's reduction
    // (fp64 keeps only the indices staged: its register budget is spent)
    constexpr bool kStageVals = PREC != 1;
    int c_sl = INT_MAX, c_p = 0, c_jj = 0;
    unsigned c_ref = 0;
    FR c_w = FR(0), c_T = FR(0), c_gw = FR(0);
    auto stage = [&]() {
        if (ptr < nrec) {
            const unsigned kk = L.kk[ptr];
            c_jj = int(kk & 63u);
            c_p = LI(c_jj);
            c_sl = int(kk >> 6);
            if (kStageVals) {
                c_ref = LR(c_jj, c_p);
                c_w = L.pw[c_p];
                c_T = L.pT[c_p];
                c_gw = LZ(c_jj);
            }
        } else {
            c_sl = INT_MAX;
        }
    };
    stage();
    {
        const int lim = INT_MAX;
        for (;;) {
            const int my = c_sl < lim ? c_sl : INT_MAX;
            const int s = __reduce_min_sync(kFull, my);
            if (s == INT_MAX) break;
            const bool part = my == s;
            const unsigned pm = __ballot_sync(kFull, part);
            BR g[11];
            for (int q = 0; q < 11; ++q) g[q] = BR(0);
            const int pid = pid_of(unsigned(s));
            if (part) {
                const unsigned ref = kStageVals ? c_ref : LR(c_jj, c_p);
                const Splat<BR> sp = splat_from<BR>(BR(kStageVals ? c_w : L.pw[c_p]), int(ref >> 28), BR(k64));
                const BR Tj = BR(kStageVals ? c_T : L.pT[c_p]), g_w = BR(kStageVals ? c_gw : LZ(c_jj));
                PV tmp;
                const PV& q = pv_of(ref, tmp);
                if constexpr (PREC == 1) {
                    const double *gn, *gvx, *gvy, *gq;
                    if constexpr (!BIG && kGeoRec) {
                        const GeoRec& pg = s_geo[res_idx(ref)];
                        gn = pg.n;
                        gvx = pg.vx;
                        gvy = pg.vy;
                        gq = pg.q;
                    } else {
                        const PlaneGeo& pg = planes[pid];
                        gn = pg.n;
                        gvx = pg.vx;
                        gvy = pg.vy;
                        gq = pg.q;
                    }
                    const double denom = dot3_rn(ray.d, gn);
                    // = k_pn / denom: stored by the forward, or recomputed (the same IEEE
                    // division of the same operands) where the list's footprint in L1 matters
                    const double t = (BIG && PSG_BIG_RECOMPUTE_T) ? q.kpn / denom : L.pt[c_p];
                    double e[3];
                    for (int k3 = 0; k3 < 3; ++k3) e[k3] = dsub(dmul(t, ray.d[k3]), q.spo[k3]);
                    finish_grad<double>(gn, gvx, gvy, gq, q.flip, ray.d, ray.mu, denom, e, sp,
                                        BR(gD), gNw, Tj, g_w, g);
                } else {
                    ScanRec sr;
                    const ScanRec* srp = &sr;
                    const int r = res_idx(ref);
                    if (r >= 0) srp = &s_scan[r]; else build_scan(v, trays(), planes[pid], rects[pid], sr);
                    const PlaneF& pf = planesf[pid];
                    const float D = fmaf(ray.c, srp->g1, fmaf(ray.a, srp->g0, srp->g2));
                    const float rD = __frcp_rn(D);
                    const float pxx = fmaf(ray.c, srp->hx1, fmaf(ray.a, srp->hx0, srp->hx2)) * rD;
                    const float pyy = fmaf(ray.c, srp->hy1, fmaf(ray.a, srp->hy0, srp->hy2)) * rD;
                    float e[3];
                    for (int k3 = 0; k3 < 3; ++k3) e[k3] = pxx * pf.vx[k3] + pyy * pf.vy[k3];  // on-plane offset
                    finish_grad<float>(pf.n, pf.vx, pf.vy, pf.q, float(q.flip), ray.d32, float(ray.mu),
                                       D / ray.L, e, sp, float(gD), gNw, Tj, g_w, g);
                }
                ++ptr;
                stage();
            }
            if constexpr (kDet) {
                const int ent = det_off + (resident ? s : entry_of(s));
                warp_flush<BR>(io.grads, pid, pm, g, io.det_grads + ((long long)ent * 8 + wid) * 11);
                if (lane == 0) atomicOr(io.det_mask + ent, 1u << wid);
            } else {
                warp_flush<BR>(io.grads, pid, pm, g);
            }
        }
    }
}

template <int PREC, int MODE, bool BIG>
#ifndef PSG_BIG_MIN_BLOCKS
#define PSG_BIG_MIN_BLOCKS 3  // crowded-tile kernel, fp64/mixed: CTAs per SM the registers allow
#endif
__global__ void __launch_bounds__(kTilePix, PREC == 0 ? 4 : PSG_BIG_MIN_BLOCKS)
    k_raster(Batch b, const PlaneGeo* __restrict__ planes, const PlaneF* __restrict__ planesf,
             int64_t P, Bins bins, RenderParams rp, RasterIO io) {
    using PV = typename Prec<PREC>::PV;
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* s_keys = reinterpret_cast<unsigned long long*>(smem);
    ScanRec* s_scan = reinterpret_cast<ScanRec*>(s_keys + kKeyCap);
    PV* s_pv = reinterpret_cast<PV*>(s_scan + kChunk);
    int* s_pid = reinterpret_cast<int*>(s_pv + kChunk);
    int* s_nlive = s_pid + kChunk;
    static_assert(BIG, "resident tiles go through k_raster_resident");
    if (*bins.abort) return;
    // crowded tiles, claimed one at a time from a counter (their costs vary by 100x):
    // async steps know the list length only on the device and launch the resident
    // CTA count of this kernel
    const int nb = bins.n_big >= 0 ? bins.n_big : *bins.n_big_dev;
    __shared__ int s_bi;
    for (;;) {
        __syncthreads();  // the previous tile's shared memory and s_bi are free
        if (threadIdx.x == 0) s_bi = atomicAdd(bins.big_ctr, 1);
        __syncthreads();
        const int bi = s_bi;
        if (bi >= nb) break;
        const int nh = *bins.n_heavy_dev;  // final before this kernel: binning has completed
        const int2 e = bins.big[bi < nh ? bi : bins.big_cap - 1 - (bi - nh)];
        raster_tile<PREC, MODE, BIG, false>(b, planes, planesf, P, bins, rp, io, e.x, e.y, s_keys,
                                            s_scan, s_pv, s_pid, s_nlive);
    }
}

// ------------------------------------------------------------------ persistent kernel
// Resident tiles (<= kResCap candidates) are rendered by persistent CTAs of 8
// consumer warps + 1 producer warp. The producer claims the next (view, tile)
// with an atomic counter, walks its dependent loads (view, CSR offsets, items,
// plane data), builds and depth-sorts the candidate records into one of two
// shared-memory buffers, and publishes it on a named barrier; the consumers
// render the previous buffer meanwhile. Per-tile setup latency and CTA launch
// cost are thereby off the critical path.
// shared-memory mbarriers: each consumer warp waits on the producer alone, so a
// fast warp starts the next tile while a slow one finishes the current tile
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                     smem_u32(b))
                 : "memory");
}
// a waiting warp sleeps (up to the hint) instead of spinning: spinning consumer
// warps otherwise take issue slots from the producer warp on their SMSP
#ifndef PSG_WAIT_HINT_NS
#define PSG_WAIT_HINT_NS 100000
#endif
constexpr unsigned kWaitHintNs = PSG_WAIT_HINT_NS;
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
    unsigned ok;
    do {
        if constexpr (kWaitHintNs > 0) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(smem_u32(b)), "r"(parity), "r"(kWaitHintNs)
                : "memory");
        } else {
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(smem_u32(b)), "r"(parity)
                : "memory");
        }
    } while (!ok);
}

// ---- prebuilt per-tile record blocks (resident tiles, 0 < n <= kResCap)
// One contiguous block per tile in HBM, copied into shared memory by one
// cp.async.bulk (TMA) per tile:
//   [hdr: n, slot_k, tile, n_live][keys: n (padded to 2)][scan: n][pv: n][pid: n (padded to 4)]
// keys are depth-sorted (z-bound bits << 32 | index). Block sizes are at most
// 16 * (kRecUnits * n + 2) bytes; blocks of crowded tiles are not stored, and the
// offsets are the exclusive scan of those sizes (k_big_tiles + CUB, bin_batch).
constexpr int kRecUnits = kRecUnitsPerPair;  // 16-byte units per candidate: >= (8 + 64 + 64 + 4 [+ 136]) / 16

template <int PREC>
struct RecLayout {
    using PV = typename Prec<PREC>::PV;
    __host__ __device__ static constexpr int keys_off() { return 16; }
    __host__ __device__ static constexpr int scan_off(int n) { return 16 + 8 * ((n + 1) & ~1); }
    __host__ __device__ static constexpr int pv_off(int n) { return scan_off(n) + int(sizeof(ScanRec)) * n; }
    __host__ __device__ static constexpr int pid_off(int n) { return pv_off(n) + int(sizeof(PV)) * n; }
    __host__ __device__ static constexpr int geo_off(int n) { return pid_off(n) + 4 * ((n + 3) & ~3); }
    __host__ __device__ static constexpr int bytes(int n) {
        // a multiple of 16 (cp.async.bulk sizes)
        return (geo_off(n) + (PSG_GEO_REC && PREC != 0 ? int(sizeof(GeoRec)) * n : 0) + 15) & ~15;
    }
};
static_assert(RecLayout<1>::bytes(1) <= 16 * (kRecUnits + 2), "record block layout");
static_assert(RecLayout<1>::bytes(kResCap) <= 16 * (kRecUnits * kResCap + 2), "record block layout");
static_assert(RecLayout<1>::bytes(3) % 16 == 0 && RecLayout<0>::bytes(3) % 16 == 0, "bulk-copy sizes");
static_assert(kRecUnits == kRecUnitsPerPair && kResCap == kResCapTiles, "psg_internal.h constants");
constexpr int kResSortW = kResCap <= 128 ? 128 : 256;  // k_build_tiles' bitonic width
static_assert(kResCap <= 256, "resident record indices are 8 bits");

// Record build, flattened over bin entries: one thread per (tile, plane) pair of
// a resident tile writes its scan record, view data, plane id and unsorted depth
// key into the tile's block (full occupancy; a warp per tile left most lanes idle
// on the typical 2-4 candidate tile).
template <int PREC>
__device__ __forceinline__ void build_pair(const Batch& b, const PlaneGeo* __restrict__ planes, int64_t P,
                                           const Bins& bins, int p, double cut_k);
#ifndef PSG_BUILD_MIN_BLOCKS
#define PSG_BUILD_MIN_BLOCKS 2  // record build: 2 CTAs per SM (<= 128 registers, no spills; 1 CTA left it latency-bound)
#endif
template <int PREC>
__global__ void __launch_bounds__(256, PSG_BUILD_MIN_BLOCKS) k_build_pairs(Batch b, const PlaneGeo* __restrict__ planes,
                                                     int64_t P, Bins bins, double cut_k) {
    using PV = typename Prec<PREC>::PV;
    using L = RecLayout<PREC>;
    if (*bins.abort) return;
    // async steps size the grid by the SM count and read the entry total here
    const int np = bins.n_pairs >= 0 ? bins.n_pairs : bins.offsets[bins.T];
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x)
        build_pair<PREC>(b, planes, P, bins, p, cut_k);
}

template <int PREC>
__device__ __forceinline__ void build_pair(const Batch& b, const PlaneGeo* __restrict__ planes, int64_t P,
                                           const Bins& bins, int p, double cut_k) {
    using PV = typename Prec<PREC>::PV;
    using L = RecLayout<PREC>;
    const int gt = bins.pair_tile[p];
    const int off = bins.offsets[gt];
    const int n = bins.offsets[gt + 1] - off;
    if (n > kResCap) return;  // crowded tile: the BIG launch builds its own records
    const int i = p - off;
    const int slot_k = bins.tile_slot[gt];
    const int tile = gt - b.tile_base[slot_k];
    const ViewDev& v = b.views[b.vid[slot_k]];
    const int tx = tile % v.tiles_x, ty = tile / v.tiles_x;
    const int tu0 = tx * kTile, tv0 = ty * kTile;
    const TileRays trays = tile_rays(v, tu0, tv0, min(v.W, tu0 + kTile) - 1, min(v.H, tv0 + kTile) - 1);
    unsigned char* blk = bins.recs + 16 * bins.unit_off[gt];
    const int pid = bins.items[p];
    PSG_CHECK(pid >= 0 && pid < P && i >= 0 && i < n && L::bytes(n) <= 16 * bins.units[gt] &&
              bins.unit_off[gt + 1] - bins.unit_off[gt] == bins.units[gt]);
    const PlaneGeo& pg = planes[pid];
    ScanRec sr;
    const short4 rect = bins.rects[int64_t(slot_k) * P + pid];
    unsigned fm = 0xffu;
    unsigned zb = build_scan(v, trays, pg, rect, sr, &fm, cut_k);
    reinterpret_cast<ScanRec*>(blk + L::scan_off(n))[i] = sr;
    PV o;
    store_pv(plane_view(v, pg), o);
    reinterpret_cast<PV*>(blk + L::pv_off(n))[i] = o;
    reinterpret_cast<int*>(blk + L::pid_off(n))[i] = pid;
    // the consumer warps whose 8x4 pixel block meets the candidate's footprint rect
    // (the per-pixel test of the scan, per block) and its footprint in plane
    // coordinates: the others skip it whole; a candidate no warp can use is dead
    const unsigned wm = rect_mask(rect, tu0, tv0) & fm;
#ifndef PSG_CHECKS
    if (wm == 0) zb = 0x7f800000u;  // (the checked build keeps it for the cull audit)
#endif
    reinterpret_cast<unsigned long long*>(blk + L::keys_off())[i] =
        (static_cast<unsigned long long>(zb) << 32) | (wm << kKeyMaskShift) | unsigned(i);
}

// Per work item t = slot * max_tiles + tile: the descriptor desc[t] = (block
// offset, n) with n = 0 empty, -2 crowded (the BIG launch renders it), -3 outside
// the view; for resident tiles the depth sort of the block's keys, the live count
// and the block header (n, slot, tile, n_live). One warp per item.
template <int PREC>
__global__ void __launch_bounds__(256) k_build_tiles(Batch b, Bins bins, int total_items,
                                                     const PlaneGeo* __restrict__ planes) {
    using L = RecLayout<PREC>;
    __shared__ unsigned long long s_keys[8][kResSortW];  // bitonic sort width: next power of two >= kResCap
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned long long* wk = s_keys[wib];
    const int nwarps = gridDim.x * 8;
    if (*bins.abort) return;
    for (int t = blockIdx.x * 8 + wib; t < total_items; t += nwarps) {
        const int slot_k = t / b.max_tiles, tile = t - slot_k * b.max_tiles;
        const ViewDev& v = b.views[b.vid[slot_k]];
        if (tile >= v.tiles_x * v.tiles_y) {
            if (lane == 0) bins.desc[t] = TileDesc{0, -3, 0, 0, 0, 0};
            continue;
        }
        const int gt = b.tile_base[slot_k] + tile;
        const int n = bins.offsets[gt + 1] - bins.offsets[gt];
        const long long off16 = bins.unit_off[gt];
        if (n == 0 || n > kResCap) {
            // empty tiles carry the packed tile coordinates for the producer's header
            if (lane == 0)
                bins.desc[t] = TileDesc{off16, n == 0 ? 0 : -2, 0, 0, 0,
                                        n == 0 ? (tile % v.tiles_x) | ((tile / v.tiles_x) << 11) : 0};
            continue;
        }
        unsigned char* blk = bins.recs + 16 * off16;
        unsigned long long* keys = reinterpret_cast<unsigned long long*>(blk + L::keys_off());
        int live = 0;
        if (n <= 32) {
            unsigned long long key = lane < n ? keys[lane] : ~0ull;
            key = bitonic_sort_warp(key);
            if (lane < n) keys[lane] = key;
            if (lane == 0 && (n & 1)) keys[n] = ~0ull;
            live = __popc(__ballot_sync(kFull, lane < n && (key >> 32) < 0x7f800000ull));
        } else {
            int npow = 64;
            while (npow < n) npow <<= 1;
            for (int i = lane; i < npow; i += 32) wk[i] = i < n ? keys[i] : ~0ull;
            __syncwarp();
            for (int size = 2; size <= npow; size <<= 1)
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int i = lane; i < npow / 2; i += 32) {
                        const int lo = 2 * i - (i & (stride - 1));
                        const int hi = lo + stride;
                        const bool asc = (lo & size) == 0;
                        const unsigned long long x = wk[lo], y = wk[hi];
                        if ((x > y) == asc) {
                            wk[lo] = y;
                            wk[hi] = x;
                        }
                    }
                    __syncwarp();
                }
            int c = 0;
            for (int i = lane; i < ((n + 1) & ~1); i += 32) {
                const unsigned long long k = i < n ? wk[i] : ~0ull;
                keys[i] = k;
                c += i < n && (k >> 32) < 0x7f800000ull;
            }
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
            live = c;
            __syncwarp();
        }
        if constexpr (PSG_GEO_REC && PREC != 0) {
            // the records' plane geometry: contiguous 136-byte copies, the warp's lanes
            // over (record, double) pairs
            constexpr int kD = int(sizeof(GeoRec) / sizeof(double));
            const int* pids = reinterpret_cast<const int*>(blk + L::pid_off(n));
            double* gd = reinterpret_cast<double*>(blk + L::geo_off(n));
            for (int e = lane; e < n * kD; e += 32) {
                const int r = e / kD;
                gd[e] = reinterpret_cast<const double*>(&planes[pids[r]].vx[0])[e - r * kD];
            }
        }
        if (lane == 0) {
            const int tx = tile % v.tiles_x, ty = tile / v.tiles_x;
            // header: the tile as packed (column, row) so consumers skip the division
            *reinterpret_cast<int4*>(blk) = make_int4(n, slot_k, tx | (ty << 11), live);
            bins.desc[t] = TileDesc{off16, n, min(kTile, v.H - ty * kTile),
                                    v.pix_off + (long long)(ty * kTile) * v.W + tx * kTile, v.W, 0};
        }
    }
}

// Record blocks of the persistent rasteriser go through a byte ring in shared
// memory (one largest block + 8 KB; 2x and 1x + 4/16 KB measured the same) with
// up to kSlots tiles in flight: at
// λ = 300 most blocks are a few hundred bytes, so the producer runs many cheap
// tiles ahead instead of one.
constexpr int kSlots = PSG_SLOTS;  // 8 and 12 measured within noise; a larger ring is slower (L1)
constexpr int kTgtBytes = 16 * kTilePix;  // a tile's targets: depth f32 + normal 3 x f32

template <int PREC>
__host__ __device__ constexpr int res_ring_bytes() {
    return ((RecLayout<PREC>::bytes(kResCap) + 127) & ~127) + (PREC != 0 && PSG_TGT_TMA ? kTgtBytes : 0) +
           PSG_RING_SLACK;  // largest + slack
}

template <int PREC>
constexpr size_t resident_smem_bytes() {
    return size_t(res_ring_bytes<PREC>()) + 2 * kSlots * sizeof(unsigned long long) + kSlots * sizeof(int);
}

constexpr int kResThreads = kTilePix + 32;
// resident CTAs per SM: fp32 fits 4 (56 registers); the fp64 paths keep 3 (72)
template <int PREC>
constexpr int res_min_blocks() { return PSG_RES_MIN_BLOCKS > 0 ? PSG_RES_MIN_BLOCKS : (PREC == 0 ? 4 : 3); }

__device__ __forceinline__ void mb_arrive_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
// TMA bulk copy global -> shared, completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Persistent rasteriser: per CTA one producer lane claims tiles from a global
// counter and streams each tile's prebuilt record block into a shared-memory ring
// with one TMA bulk copy; eight consumer warps render the tiles in claim order
// (one pixel per thread). Per slot: full[s] completes on the copy's bytes (or
// the producer's arrive for tiles without a block), empty[s] on the 256
// consumer threads, slot_off[s] locates the block in the ring.
// URES: list entries loaded ahead per shift (2 for the low-lambda instantiation, whose
// lists are long; 1 at high lambda, where the registers cost more than it saves)
template <int PREC, int MODE, int URES = PSG_SHIFT_UNROLL_RES>
__global__ void __launch_bounds__(kResThreads, res_min_blocks<PREC>())
    k_raster_resident(Batch b, const PlaneGeo* __restrict__ planes, const PlaneF* __restrict__ planesf,
                      int64_t P, Bins bins, RenderParams rp, RasterIO io, int* work_ctr,
                      int total_items) {
    using PV = typename Prec<PREC>::PV;
    using L = RecLayout<PREC>;
    constexpr int kRing = res_ring_bytes<PREC>();
    // targets staged by TMA for the fp64 paths; the fp32 kernel (4 CTAs/SM, faster
    // tiles) keeps more tiles in its ring by reading them from HBM (measured)
    constexpr bool kTgtTma = (MODE == kFused || MODE == kFusedDet) && PREC != 0 && PSG_TGT_TMA;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + kRing);
    unsigned long long* empty = full + kSlots;
    int* slot_off = reinterpret_cast<int*>(empty + kSlots);
    if (*bins.abort) return;  // a capacity was exceeded: the host replays this step
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; ++i) {
            mb_init(&full[i], 1);
            mb_init(&empty[i], kTilePix);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kTilePix / 32) {
        // ---------------- producer (one lane). Ring allocation is FIFO: blocks in
        // flight occupy [tail, head) modulo the ring; a block never wraps (the
        // ring tail is skipped instead). A new block waits for the oldest slots
        // to drain until it fits. Crowded tiles (the BIG launch) take no slot.
        if (lane != 0) return;
        int f_off[kSlots];  // ring offsets of the blocks in flight, FIFO by issue order
        int f_first = 0, f_count = 0, head = 0;
        // claims run two items ahead and the next descriptor load is issued before
        // the current item is processed, so neither latency is on the issue path
        const long long p_start = PSG_PROBE == 2 ? clock64() : 0;
        int t = atomicAdd(work_ctr, 1);
        TileDesc d = t < total_items ? bins.desc[t] : TileDesc{0, -1, 0, 0, 0, 0};
        int t2 = t < total_items ? atomicAdd(work_ctr, 1) : total_items;
        for (int it = 0;; ++it) {
            const TileDesc d2 = t2 < total_items ? bins.desc[t2] : TileDesc{0, -1, 0, 0, 0, 0};
            const int t3 = t2 < total_items ? atomicAdd(work_ctr, 1) : total_items;
            if (d.n == -2 || d.n == -3) {  // no slot
                --it;
            } else {
                const int slot = it % kSlots;
                const bool tgt = kTgtTma && io.tma_targets && d.n > 0;
                const int need = d.n > 0 ? ((L::bytes(d.n) + 127) & ~127) + (tgt ? kTgtBytes : 0) : 128;
                // reclaim: the slot itself, then space, oldest first
                auto pop = [&]() {
                    const int s0 = (it - f_count) % kSlots;  // slot of the oldest in flight
                    const long long tw0 = PSG_PROBE == 2 ? clock64() : 0;
                    mb_wait(&empty[s0], (((it - f_count) / kSlots)) & 1);
                    if (PSG_PROBE == 2) atomicAdd(&io.stats->probe[1], (unsigned long long)(clock64() - tw0));
                    f_first = (f_first + 1) % kSlots;
                    --f_count;
                };
                if (f_count == kSlots) pop();
                int at = -1;
                for (;;) {
                    if (f_count == 0) {
                        head = 0;
                        at = 0;
                        break;
                    }
                    // (head never catches up with tail while blocks are in flight,
                    // so head == tail always means an empty ring)
                    const int tail = f_off[f_first];
                    if (head >= tail) {
                        if (kRing - head >= need) { at = head; break; }
                        if (tail > need) { at = 0; break; }
                    } else if (tail - head > need) {
                        at = head;
                        break;
                    }
                    pop();
                }
                PSG_CHECK(d.n <= kResCap && at >= 0 && at + need <= kRing);
                const int fi = (f_first + f_count) % kSlots;
                f_off[fi] = at;
                ++f_count;
                head = at + need;
                unsigned char* B = smem + at;
                slot_off[slot] = d.n == -1 ? -1 : at;
                if (d.n == -1) {
                    mb_arrive(&full[slot]);
                    if (PSG_PROBE == 2) {  // producer: total cycles, CTAs
                        atomicAdd(&io.stats->probe[5], (unsigned long long)(clock64() - p_start));
                        atomicAdd(&io.stats->probe[6], 1ull);
                    }
                    break;
                }
                if (d.n > 0) {
                    const unsigned bytes = unsigned(L::bytes(d.n));
                    // the tile's target rows (loss inputs), 64 B + 192 B each; their
                    // location comes with the descriptor (no view lookups here)
                    const int rows = tgt ? d.rows : 0;
                    const int W = d.W;
                    const float* td0 = io.td + d.tgt;
                    const float* tn0 = io.tn + 3 * d.tgt;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mb_arrive_expect_tx(&full[slot], bytes + unsigned(rows) * 256u);
                    bulk_g2s(B, bins.recs + 16 * d.off16, bytes, &full[slot]);
                    unsigned char* T = B + ((bytes + 127) & ~127);
                    for (int r = 0; r < rows; ++r) {
                        bulk_g2s(T + 64 * r, td0 + (long long)r * W, 64u, &full[slot]);
                        bulk_g2s(T + 4 * kTilePix + 192 * r, tn0 + 3LL * r * W, 192u, &full[slot]);
                    }
                } else {
                    const int slot_k = t / b.max_tiles;
                    *reinterpret_cast<int4*>(B) = make_int4(0, slot_k, d.pad, 0);  // packed (column, row)
                    mb_arrive(&full[slot]);
                }
            }
            d = d2;
            t = t2;
            t2 = t3;
        }
        return;
    }
    // ---------------- consumers (8 warps, one pixel per thread), slots in order
    const long long t_start = PSG_PROBE == 2 ? clock64() : 0;
    unsigned long long t_wait = 0;
    for (int it = 0;; ++it) {
        const int slot = it % kSlots;
        const long long tw0 = PSG_PROBE == 2 ? clock64() : 0;
        mb_wait(&full[slot], (it / kSlots) & 1);
        if (PSG_PROBE == 2) t_wait += (unsigned long long)(clock64() - tw0);
        const int off = slot_off[slot];
        if (off < 0) {
            if (PSG_PROBE == 2 && lane == 0) {  // per consumer warp: cycles waiting / in the loop
                atomicAdd(&io.stats->probe[2], t_wait);
                atomicAdd(&io.stats->probe[3], (unsigned long long)(clock64() - t_start));
                atomicAdd(&io.stats->probe[4], 1ull);
            }
            break;
        }
        unsigned char* B = smem + off;
        int* hdr = reinterpret_cast<int*>(B);
        const int n = hdr[0];
        PSG_CHECK(n <= kResCap && hdr[1] >= 0 && hdr[1] < b.n && hdr[3] >= 0 && hdr[3] <= max(n, 0));
        if (n >= 0)
            raster_tile<PREC, MODE, false, true, URES>(
                b, planes, planesf, P, bins, rp, io, hdr[1], hdr[2],
                reinterpret_cast<unsigned long long*>(B + L::keys_off()),
                reinterpret_cast<ScanRec*>(B + L::scan_off(n)), reinterpret_cast<PV*>(B + L::pv_off(n)),
                reinterpret_cast<int*>(B + L::pid_off(n)), &hdr[3], n,
                (kTgtTma && io.tma_targets && n > 0)
                    ? reinterpret_cast<const float*>(B + ((L::bytes(n) + 127) & ~127))
                    : nullptr,
                reinterpret_cast<const GeoRec*>(B + L::geo_off(n)));
        mb_arrive(&empty[slot]);
    }
}

// Renderer::backward from stored records (renderer.cpp:373-528), one CTA per
// tile, exact geometry in precision R; records merged per warp by plane index.
template <typename R>
__global__ void __launch_bounds__(kTilePix)
    k_backward_records(Batch b, const PlaneGeo* __restrict__ planes, int64_t P, Bins bins,
                       RenderParams rp, BackwardIO io) {
    const ViewDev& v = b.views[b.vid[0]];
    const int tile = blockIdx.x;
    if (tile >= v.tiles_x * v.tiles_y) return;
    const int gt = b.tile_base[0] + tile;
    if (bins.offsets[gt + 1] - bins.offsets[gt] == 0) return;  // renderer.cpp:409-410
    const int tx = tile % v.tiles_x, ty = tile / v.tiles_x;
    const int tid = threadIdx.x;
    const int tu0 = tx * kTile, tv0 = ty * kTile;
    const int pu = tu0 + (tid & (kTile - 1)), pv = tv0 + (tid >> 4);
    const bool valid = pu < v.W && pv < v.H;
    const int M = io.M;
    const double k64 = 5.0 * rp.lambda;

    const long long px = (long long)pv * v.W + pu;
    int cnt = valid ? min(int(io.rec_count[px]), M) : 0;
    double gD = 0, gA = 0, gN[3] = {0, 0, 0};
    if (cnt > 0) {
        gD = io.d_depth[px];
        gA = io.d_alpha ? io.d_alpha[px] : 0.0;
        for (int q = 0; q < 3; ++q) gN[q] = io.d_normal[3 * px + q];
        if (gD == 0.0 && gA == 0.0 && fabs(gN[0]) <= 1e-12 && fabs(gN[1]) <= 1e-12 && fabs(gN[2]) <= 1e-12)
            cnt = 0;
    }
    if (__ballot_sync(kFull, cnt > 0) == 0) return;
    const PixelRay ray = pixel_ray(v, pu, pv, tu0, tv0);
    R rgN[3], rgNw[3];
    for (int q = 0; q < 3; ++q) rgN[q] = R(gN[q]);
    for (int r = 0; r < 3; ++r)
        rgNw[r] = R(v.R[3 * r] * gN[0] + (v.R[3 * r + 1] * gN[1] + v.R[3 * r + 2] * gN[2]));
    const R rgD = R(gD), rgA = R(gA);
    R lT[kMaxRecordCap], lg[kMaxRecordCap], lw[kMaxRecordCap], lphi[kMaxRecordCap];
    int lp[kMaxRecordCap];
    {
        R T = R(1);
        for (int j = 0; j < cnt; ++j) {  // replay (renderer.cpp:441-459)
            const int pid = io.rec_prim[px * M + j];
            const PlaneGeo& pg = planes[pid];
            const PlaneView pvw = plane_view(v, pg);
            R d[3], n[3], vx[3], vy[3], r[4], e[3], t, z;
            for (int k = 0; k < 3; ++k) {
                d[k] = R(ray.d[k]);
                n[k] = R(pg.n[k]);
                vx[k] = R(pg.vx[k]);
                vy[k] = R(pg.vy[k]);
            }
            for (int k = 0; k < 4; ++k) r[k] = R(pg.r[k]);
            R px_, py_;
            if constexpr (sizeof(R) == 8) {
                const double denom = dot3_rn(d, n);
                t = pvw.kpn / denom;
                for (int k = 0; k < 3; ++k) e[k] = dsub(dmul(t, d[k]), pvw.spo[k]);
                px_ = dot3_rn(e, vx);
                py_ = dot3_rn(e, vy);
                z = dmul(t, ray.mu);
            } else {
                const R denom = (d[0] * n[0] + d[1] * n[1]) + d[2] * n[2];
                t = R(pvw.kpn) / denom;
                for (int k = 0; k < 3; ++k) e[k] = t * d[k] - R(pvw.spo[k]);
                px_ = (e[0] * vx[0] + e[1] * vx[1]) + e[2] * vx[2];
                py_ = (e[0] * vy[0] + e[1] * vy[1]) + e[2] * vy[2];
                z = t * R(ray.mu);
            }
            const Splat<R> sp = splat_eval<R>(px_, py_, r, R(k64));
            lT[j] = T;
            lw[j] = sp.w;
            lp[j] = pid;
            lphi[j] = (rgD * z + (rgN[0] * R(pvw.mcam[0]) + rgN[1] * R(pvw.mcam[1]) + rgN[2] * R(pvw.mcam[2]))) + rgA;
            T = T * (R(1) - sp.w);
        }
        R S = R(0);
        for (int j = cnt - 1; j >= 0; --j) {  // suffix sweep (renderer.cpp:463-471)
            lg[j] = lT[j] * (lphi[j] - S);
            S = lw[j] * lphi[j] + (R(1) - lw[j]) * S;
        }
    }
    for (int i = 1; i < cnt; ++i) {  // order by plane index for the warp merge
        const int p0 = lp[i];
        const R g0 = lg[i], t0 = lT[i];
        int j = i - 1;
        while (j >= 0 && lp[j] > p0) {
            lp[j + 1] = lp[j];
            lg[j + 1] = lg[j];
            lT[j + 1] = lT[j];
            --j;
        }
        lp[j + 1] = p0;
        lg[j + 1] = g0;
        lT[j + 1] = t0;
    }
    int ptr = 0;
    for (;;) {
        const int my = ptr < cnt ? lp[ptr] : INT_MAX;
        const int s = __reduce_min_sync(kFull, my);
        if (s == INT_MAX) break;
        const bool part = my == s;
        const unsigned pm = __ballot_sync(kFull, part);
        R g[11];
        for (int q = 0; q < 11; ++q) g[q] = R(0);
        if (part) {
            const PlaneGeo& pg = planes[s];
            record_grad_exact<R>(pg, plane_view(v, pg), ray, k64, rgD, rgNw, lT[ptr], lg[ptr], g);
            ++ptr;
        }
        warp_flush<R>(io.grads, s, pm, g);
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
                const double nr[3] = {normal[3 * px] * scale, normal[3 * px + 1] * scale, normal[3 * px + 2] * scale};
                const double nt[3] = {double(t0), double(t1), double(t2)};
                const double cos_term = 1.0 - dot3d(nr, nt);
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
                if (norm_on) gA -= dot3d(g, nr) * scale;
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

// PSG_DEBUG_SYNC=1: synchronise after every rasteriser launch and name the
// kernel that faulted (debugging aid; off by default).
bool debug_sync(const char* what, cudaStream_t s) {
    static const int on = [] {
        const char* e = std::getenv("PSG_DEBUG_SYNC");
        return e && e[0] == '1' ? 1 : 0;
    }();
    if (!on) return true;
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        std::fprintf(stderr, "psg: %s failed: %s\n", what, cudaGetErrorString(e));
        return false;
    }
    return true;
}

constexpr int kMaxDevices = 64;

// Per-device launch state (the dynamic shared-memory opt-in and the occupancy-sized
// grids are properties of a device and a kernel): set once per (kernel, device),
// thread-safe, so several contexts on several devices can launch concurrently.
struct RasterGrids {
    int res = 0;    // persistent resident CTAs: SMs x occupancy
    int big = 0;    // crowded-tile CTAs of an async step: SMs x occupancy
    int build = 0;  // grid-stride record build
};

template <int PREC, int MODE>
const RasterGrids& raster_grids() {
    static std::once_flag once[kMaxDevices];
    static RasterGrids grids[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    dev = dev < kMaxDevices ? dev : kMaxDevices - 1;
    std::call_once(once[dev], [dev] {
        constexpr size_t smem_res = resident_smem_bytes<PREC>();
        constexpr size_t smem_big = raster_smem_bytes<PREC, true>();
        RasterGrids& g = grids[dev];
        int sms = 0, occ = 0, occ_big = 0;
        if (cudaFuncSetAttribute(k_raster_resident<PREC, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem_res)) != cudaSuccess ||
            cudaFuncSetAttribute(k_raster_resident<PREC, MODE, PSG_RES_U_LOW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem_res)) != cudaSuccess ||
            cudaFuncSetAttribute(k_raster<PREC, MODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem_big)) != cudaSuccess)
            std::fprintf(stderr, "psplat_b200: cudaFuncSetAttribute failed on device %d\n", dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_raster_resident<PREC, MODE>, kResThreads, smem_res);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_big, k_raster<PREC, MODE, true>, kTilePix, smem_big);
        g.res = sms * (occ > 0 ? occ : 1);
        g.big = sms * (occ_big > 0 ? occ_big : 1);
        g.build = sms * 8;
    });
    return grids[dev];
}

template <int PREC, int MODE>
void launch_raster_t(const Batch& b, const PlaneGeo* planes, const PlaneF* planesf, const Bins& bins,
                     const RenderParams& rp, const RasterIO& io, int64_t P, cudaStream_t s,
                     const AuxStream& aux) {
    constexpr size_t smem_res = resident_smem_bytes<PREC>();
    constexpr size_t smem_big = raster_smem_bytes<PREC, true>();
    const RasterGrids& g = raster_grids<PREC, MODE>();
    const int total = b.n * b.max_tiles;
    // crowded-tile grid: the exact count after a synchronous binning, else the
    // resident CTA count looping over the device-side list (async steps)
    const int big_grid = bins.n_big >= 0 ? bins.n_big : std::min(g.big, std::max(bins.T, 1));
    // crowded tiles first, on the aux stream: their long single-CTA tiles overlap
    // the record build and the persistent kernel instead of forming a tail
    const bool fork = big_grid > 0 && aux.stream;
    if (big_grid > 0) cudaMemsetAsync(bins.big_ctr, 0, sizeof(int), s);
    if (fork) {
        cudaEventRecord(aux.fork, s);
        cudaStreamWaitEvent(aux.stream, aux.fork, 0);
        k_raster<PREC, MODE, true><<<unsigned(big_grid), kTilePix, smem_big, aux.stream>>>(
            b, planes, planesf, P, bins, rp, io);
        cudaEventRecord(aux.join, aux.stream);
        debug_sync("k_raster<big>", aux.stream);
    }
    {
        const int build_grid = bins.n_pairs >= 0 ? (bins.n_pairs + 255) / 256 : g.build;
        if (build_grid > 0)
            k_build_pairs<PREC><<<unsigned(build_grid), 256, 0, s>>>(b, planes, P, bins, foot_cut(rp));
        debug_sync("k_build_pairs", s);
        const int blocks = std::min(g.build * 2, (total + 7) / 8);
        k_build_tiles<PREC><<<unsigned(blocks > 0 ? blocks : 1), 256, 0, s>>>(b, bins, total, planes);
        debug_sync("k_build_tiles", s);
    }
    cudaMemsetAsync(bins.work_ctr, 0, sizeof(int), s);
    // low lambda: long lists, the two-ahead shift instantiation (+1.4 % at lambda 7.36,
    // +2.6 % at 20; -0.5 % at 300, where the single-shift one runs)
    if (PREC != 0 && rp.lambda < PSG_RES_U2_LAMBDA)
        k_raster_resident<PREC, MODE, PSG_RES_U_LOW><<<unsigned(std::min(g.res, total)), kResThreads, smem_res, s>>>(
            b, planes, planesf, P, bins, rp, io, bins.work_ctr, total);
    else
        k_raster_resident<PREC, MODE><<<unsigned(std::min(g.res, total)), kResThreads, smem_res, s>>>(
            b, planes, planesf, P, bins, rp, io, bins.work_ctr, total);
    debug_sync("k_raster_resident", s);
    if (fork)
        cudaStreamWaitEvent(s, aux.join, 0);
    else if (big_grid > 0)
        k_raster<PREC, MODE, true><<<unsigned(big_grid), kTilePix, smem_big, s>>>(b, planes, planesf, P,
                                                                                 bins, rp, io);
}

template <int PREC>
void launch_mode(RasterMode mode, const Batch& b, const PlaneGeo* planes, const PlaneF* planesf,
                 int64_t P, const Bins& bins, const RenderParams& rp, const RasterIO& io, cudaStream_t s,
                 const AuxStream& aux) {
    if (mode == kFused) launch_raster_t<PREC, kFused>(b, planes, planesf, bins, rp, io, P, s, aux);
    else if (mode == kFusedDet) launch_raster_t<PREC, kFusedDet>(b, planes, planesf, bins, rp, io, P, s, aux);
    else if (mode == kFwdMaps) launch_raster_t<PREC, kFwdMaps>(b, planes, planesf, bins, rp, io, P, s, aux);
    else launch_raster_t<PREC, kFwdRecords>(b, planes, planesf, bins, rp, io, P, s, aux);
}

}  // namespace

void launch_raster(int precision, RasterMode mode, const Batch& b, const PlaneGeo* planes,
                   const PlaneF* planesf, int64_t P, const Bins& bins, const RenderParams& rp,
                   const RasterIO& io, cudaStream_t s, const AuxStream& aux) {
    if (b.n <= 0 || b.max_tiles <= 0) return;
    if (precision == 0) launch_mode<0>(mode, b, planes, planesf, P, bins, rp, io, s, aux);
    else if (precision == 1) launch_mode<1>(mode, b, planes, planesf, P, bins, rp, io, s, aux);
    else launch_mode<2>(mode, b, planes, planesf, P, bins, rp, io, s, aux);
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

namespace {

// deterministic mode: plane p's gradient = its bin entries in entry order, each
// summing the 8 warps' partials in warp order (one thread per (plane, param))
__global__ void k_det_grads(const int* __restrict__ spid, const int* __restrict__ spair, int64_t npairs,
                            int64_t P, const double* __restrict__ det, const unsigned* __restrict__ mask,
                            double* grads) {
    // one warp per plane: lane l sums entries a+l, a+l+32, ... (warps in order, only
    // the (entry, warp) partials that were written), then a fixed butterfly: the
    // order depends only on the stable entry order, so results are bitwise stable
    const int64_t p = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= P) return;
    auto lower = [&](int64_t key) {
        int64_t lo = 0, hi = npairs;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (spid[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    const int64_t a = lower(p), e = lower(p + 1);
    double acc[11];
    for (int q = 0; q < 11; ++q) acc[q] = 0.0;
    for (int64_t k = a + lane; k < e; k += 32) {
        const int pair = spair[k];
        unsigned m = mask[pair];
        const double* d = det + int64_t(pair) * 8 * 11;
        while (m) {
            const int w = __ffs(m) - 1;
            m &= m - 1;
            for (int q = 0; q < 11; ++q) acc[q] += d[w * 11 + q];
        }
    }
    for (int q = 0; q < 11; ++q) {
        double v = acc[q];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) grads[p * 11 + q] += v;
    }
}

// deterministic mode: per view, its tiles' (8 warps x 2) loss partials summed by a
// fixed split over 256 threads and a fixed-order tree
__global__ void k_det_loss(Batch b, const double* __restrict__ det_loss, double* view_loss) {
    __shared__ double sd[256], sn[256];
    const int k = blockIdx.x;
    const int64_t t0 = int64_t(b.tile_base[k]) * 8, t1 = int64_t(b.tile_base[k + 1]) * 8;
    const int64_t per = (t1 - t0 + 255) / 256;
    const int64_t a = t0 + threadIdx.x * per, e = min(t1, a + per);
    double d = 0.0, n = 0.0;
    for (int64_t j = a; j < e; ++j) {
        d += det_loss[2 * j];
        n += det_loss[2 * j + 1];
    }
    sd[threadIdx.x] = d;
    sn[threadIdx.x] = n;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sd[threadIdx.x] += sd[threadIdx.x + o];
            sn[threadIdx.x] += sn[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        view_loss[2 * k] += sd[0];
        view_loss[2 * k + 1] += sn[0];
    }
}

}  // namespace

void launch_det_reduce(const int* sorted_pid, const int* sorted_pair, int64_t n_pairs, int64_t P,
                       const double* det_grads, const unsigned* det_mask, double* grads, const Batch& b,
                       const double* det_loss, double* view_loss, cudaStream_t s) {
    if (P > 0 && n_pairs > 0)
        k_det_grads<<<unsigned((P * 32 + 255) / 256), 256, 0, s>>>(sorted_pid, sorted_pair, n_pairs, P,
                                                                  det_grads, det_mask, grads);
    if (b.n > 0) k_det_loss<<<unsigned(b.n), 256, 0, s>>>(b, det_loss, view_loss);
}

void launch_finalize_grads(const PlaneGeo* planes, double* grads, int64_t n,
                           unsigned long long* first_bad, cudaStream_t s) {
    if (n <= 0) return;
    k_finalize<<<unsigned((n + 255) / 256), 256, 0, s>>>(planes, grads, n, first_bad);
}

}  // namespace psg
