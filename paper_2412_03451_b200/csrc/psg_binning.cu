// Plane setup, screen-space bounds and tile binning (fp64, bit-exact), plus the
// synthetic ground-truth target renderer used to build benchmark inputs.
//
// This translation unit is compiled with -fmad=false: every fp64 expression
// below rounds after each multiply and add exactly as the reference's x86-64
// build does (no FMA contraction), so the per-tile candidate sets are identical
// to bin_primitives() (renderer.cpp:115-147) bit for bit. Reduction orders
// follow oracle/eigen_shim/Eigen/Core (3-vector dot: (a0+a1)+a2; 4-vector dot:
// (a0+a2)+(a1+a3); stored Matrix3d*Vector3d row: a0+(a1+a2); transpose()*v row:
// (a0+a1)+a2).
#include <cuda_runtime.h>

#include "psg_internal.h"

namespace psg {
namespace {

__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

// x86-64 cvttsd2si semantics: out-of-range and NaN convert to INT_MIN. The
// reference casts floor/ceil of projected coordinates with int(...)
// (renderer.cpp:108-111); far-clipped projections overflow int and the
// reference then yields an empty rect. Reproduced so bins stay bit-exact.
__device__ __forceinline__ int x86_cvt(double x) {
    if (!(x >= -2147483648.0 && x < 2147483648.0)) return (int)0x80000000;
    return (int)x;
}
__device__ __forceinline__ int wrap_add(int a, int b) {
    return (int)((unsigned)a + (unsigned)b);
}

// quat_normalized + quat_to_matrix + plane_frame (geometry.cpp:10-40) and the
// view-independent part of make_prim_views (renderer.cpp:46-50).
__global__ void k_plane_setup(const double* __restrict__ center, const double* __restrict__ rot,
                              const double* __restrict__ radii, int64_t n, PlaneGeo* out, PlaneF* outf) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double q0 = rot[4 * i], q1 = rot[4 * i + 1], q2 = rot[4 * i + 2], q3 = rot[4 * i + 3];
    const double nq = sqrt((q0 * q0 + q2 * q2) + (q1 * q1 + q3 * q3));
    const double w = q0 / nq, x = q1 / nq, y = q2 / nq, z = q3 / nq;
    PlaneGeo g;
    // columns of quat_to_matrix (row-major fill, geometry.cpp:13-15)
    g.vx[0] = 1 - 2 * (y * y + z * z);
    g.vx[1] = 2 * (x * y + w * z);
    g.vx[2] = 2 * (x * z - w * y);
    g.vy[0] = 2 * (x * y - w * z);
    g.vy[1] = 1 - 2 * (x * x + z * z);
    g.vy[2] = 2 * (y * z + w * x);
    g.n[0] = 2 * (x * z + w * y);
    g.n[1] = 2 * (y * z - w * x);
    g.n[2] = 1 - 2 * (x * x + y * y);
    for (int k = 0; k < 3; ++k) g.c[k] = center[3 * i + k];
    for (int k = 0; k < 4; ++k) g.r[k] = radii[4 * i + k];
    g.q[0] = w;
    g.q[1] = x;
    g.q[2] = y;
    g.q[3] = z;
    out[i] = g;
    PlaneF f;
    for (int k = 0; k < 3; ++k) {
        f.n[k] = float(g.n[k]);
        f.vx[k] = float(g.vx[k]);
        f.vy[k] = float(g.vy[k]);
        f.pad[k] = 0.0f;
    }
    for (int k = 0; k < 4; ++k) {
        f.q[k] = float(g.q[k]);
        f.r[k] = float(g.r[k]);
    }
    outf[i] = f;
}

// projected_rect (renderer.cpp:71-113) followed by the tile range of
// bin_primitives (renderer.cpp:129-130). Returns false for an empty rect.
__device__ bool tile_rect(const ViewDev& v, const PlaneGeo& p, double cut, short4& tr) {
    const double ex_p = p.r[0] + cut, ex_m = p.r[1] + cut;
    const double ey_p = p.r[2] + cut, ey_m = p.r[3] + cut;
    double world[4][3];
    for (int k = 0; k < 3; ++k) {
        world[0][k] = (p.c[k] + ex_p * p.vx[k]) + ey_p * p.vy[k];
        world[1][k] = (p.c[k] - ex_m * p.vx[k]) + ey_p * p.vy[k];
        world[2][k] = (p.c[k] - ex_m * p.vx[k]) - ey_m * p.vy[k];
        world[3][k] = (p.c[k] + ex_p * p.vx[k]) - ey_m * p.vy[k];
    }
    double cam[4][3];
    for (int i = 0; i < 4; ++i) {
        const double d0 = world[i][0] - v.t[0], d1 = world[i][1] - v.t[1],
                     d2 = world[i][2] - v.t[2];
        // rot_cw = rot_wc^T stored; row r of rot_cw is column r of rot_wc
        for (int r = 0; r < 3; ++r) cam[i][r] = v.R[r] * d0 + (v.R[3 + r] * d1 + v.R[6 + r] * d2);
    }
    double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300;
    int n_poly = 0;
    auto add_pt = [&](double x, double y, double z) {
        const double iz = 1.0 / z;
        const double u = v.fx * x * iz + v.cx;
        const double w = v.fy * y * iz + v.cy;
        umin = (u < umin) ? u : umin;  // std::min(umin, u)
        umax = (umax < u) ? u : umax;  // std::max(umax, u)
        vmin = (w < vmin) ? w : vmin;
        vmax = (vmax < w) ? w : vmax;
        ++n_poly;
    };
    for (int i = 0; i < 4; ++i) {
        const double* a = cam[i];
        const double* b = cam[(i + 1) & 3];
        const bool ain = a[2] >= kZClip, bin = b[2] >= kZClip;
        if (ain) add_pt(a[0], a[1], a[2]);
        if (ain != bin) {
            const double s = (kZClip - a[2]) / (b[2] - a[2]);
            add_pt(a[0] + s * (b[0] - a[0]), a[1] + s * (b[1] - a[1]), a[2] + s * (b[2] - a[2]));
        }
    }
    if (n_poly == 0) return false;
    int u0 = wrap_add(x86_cvt(floor(umin - 0.5)), -1);
    int u1 = wrap_add(x86_cvt(ceil(umax - 0.5)), 1);
    int v0 = wrap_add(x86_cvt(floor(vmin - 0.5)), -1);
    int v1 = wrap_add(x86_cvt(ceil(vmax - 0.5)), 1);
    u0 = u0 < 0 ? 0 : u0;
    u1 = u1 > v.W - 1 ? v.W - 1 : u1;
    v0 = v0 < 0 ? 0 : v0;
    v1 = v1 > v.H - 1 ? v.H - 1 : v1;
    if (u0 > u1 || v0 > v1) return false;
    tr = make_short4(short(u0), short(u1), short(v0), short(v1));  // pixel rect
    return true;
}

__global__ void k_rect_count(Batch b, const PlaneGeo* __restrict__ planes, int64_t P, double cut,
                             Bins bins) {
    const int k = blockIdx.y;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const ViewDev& v = b.views[b.vid[k]];
    short4 tr = make_short4(1, 0, 1, 0);
    const bool ok = tile_rect(v, planes[i], cut, tr);
    if (blockIdx.z == 0) bins.rects[int64_t(k) * P + i] = tr;
    if (!ok) return;
    int* cnt = bins.counts + b.tile_base[k];
    // tile rows split over gridDim.z slices as in k_scatter (each slice repeats the
    // projection: small batches have the threads to spare)
    for (int ty = tr.z / kTile + int(blockIdx.z); ty <= tr.w / kTile; ty += int(gridDim.z))
        for (int tx = tr.x / kTile; tx <= tr.y / kTile; ++tx) atomicAdd(cnt + ty * v.tiles_x + tx, 1);
}

__global__ void k_scatter(Batch b, int64_t P, Bins bins) {
    const int k = blockIdx.y;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= P || *bins.abort) return;
    const short4 tr = bins.rects[int64_t(k) * P + i];
    if (tr.x > tr.y) return;
    const int tiles_x = b.views[b.vid[k]].tiles_x;
    int* cur = bins.cursor + b.tile_base[k];
    // tile rows are split over gridDim.z threads: each position comes from an
    // atomic with return, so one thread walking a large footprint alone would
    // set the kernel's length on small batches
    for (int ty = tr.z / kTile + int(blockIdx.z); ty <= tr.w / kTile; ty += int(gridDim.z))
        for (int tx = tr.x / kTile; tx <= tr.y / kTile; ++tx) {
            const int pos = atomicAdd(cur + ty * tiles_x + tx, 1);
            PSG_CHECK(pos < bins.offsets[b.tile_base[k] + ty * tiles_x + tx + 1]);
            bins.items[pos] = int(i);
            bins.pair_tile[pos] = b.tile_base[k] + ty * tiles_x + tx;
        }
}

// Also sums Q_v = sum over tiles of |candidates| * |pixels| (one RED per warp).
__global__ void k_big_tiles(Batch b, Bins bins, int threshold) {
    const int k = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const ViewDev& v = b.views[b.vid[k]];
    unsigned q = 0, cnt = 0;
    if (t < v.tiles_x * v.tiles_y) {
        const int gt = b.tile_base[k] + t;
        const int c = bins.counts[gt];
        bins.tile_slot[gt] = k;
        if (c > threshold) {
            // longest first (their CTAs set the kernel's tail): heavy tiles from the
            // front of the list, the rest from the back
            atomicAdd(bins.n_big_dev, 1);
            if (PSG_BIG_LPT && c > 4 * threshold) {
                bins.big[atomicAdd(bins.n_heavy_dev, 1)] = make_int2(k, t);
            } else {
                bins.big[bins.big_cap - 1 - atomicAdd(bins.n_light_dev, 1)] = make_int2(k, t);
            }
        }
        // record block of a resident tile: header + 9 units per candidate (psg_raster.cu)
        bins.units[gt] = (c > 0 && c <= threshold) ? 2LL + (long long)kRecUnitsPerPair * c : 0LL;
        const int tx = t % v.tiles_x, ty = t / v.tiles_x;
        const int pw = min(16, v.W - tx * 16), ph = min(16, v.H - ty * 16);
        q = unsigned(c) * unsigned(pw * ph);
        cnt = unsigned(c);
    }
    const unsigned wq = __reduce_add_sync(0xffffffffu, q);
    const unsigned wc = __reduce_add_sync(0xffffffffu, cnt);  // <= 32 * 2^26: no wrap
    if ((threadIdx.x & 31) == 0 && wq) atomicAdd(bins.pair_px, (unsigned long long)wq);
    if ((threadIdx.x & 31) == 0 && wc) atomicAdd(bins.pairs64, (unsigned long long)wc);
}

// One thread, after the CUB scans. The 64-bit entry total is exact even when the
// int32 CSR offsets wrapped (more than 2^31 - 1 entries): such a batch, or one
// larger than the buffers sized by earlier steps, aborts and is replayed by the
// host with exact sizes, split into smaller view groups when needed.
__global__ void k_bin_guard(Bins bins, long long recs_cap16, long long pair_limit,
                            unsigned long long* need, double* overflow, Stats* st) {
    if (bins.halt && *bins.halt != ~0ull) {
        // a deferred run halted at an earlier step of this block: the host replays
        // from there, so this step's rendering is skipped (its result is gated off)
        *bins.abort = 1;
        return;
    }
    const unsigned long long pairs = *bins.pairs64;
    const long long units = bins.unit_off[bins.T];
    const long long cap = bins.items_cap < pair_limit ? bins.items_cap : pair_limit;
    const bool bad = pairs > (unsigned long long)cap || units + 1 > recs_cap16;
    *bins.abort = bad ? 1 : 0;
    if (bad) {
        need[0] = pairs > need[0] ? pairs : need[0];
        need[1] = (unsigned long long)units > need[1] ? (unsigned long long)units : need[1];
        if (overflow) *overflow += 1.0;
    } else {
        st->pairs += pairs;
        st->big += (unsigned long long)*bins.n_big_dev;
    }
}

// Debug only: ascending order per tile, as bin_primitives emits it.
__global__ void k_sort_bins(const int* __restrict__ offsets, int* items, int T) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    int* a = items + offsets[t];
    const int n = offsets[t + 1] - offsets[t];
    for (int i = 1; i < n; ++i) {
        const int x = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > x) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = x;
    }
}

// render_ground_truth + cast_gt_ray (synthetic.cpp:57-79,144-175), noise-free.
// faces: 15 doubles each (center, u, v, half_u, half_v, normal, id).
__global__ void k_render_gt(const ViewDev* __restrict__ views, const double* __restrict__ faces,
                            int n_faces, float* __restrict__ td, float* __restrict__ tn) {
    const ViewDev& v = views[blockIdx.y];
    const int px = blockIdx.x * blockDim.x + threadIdx.x;
    if (px >= v.W * v.H) return;
    const int uu = px % v.W, vv = px / v.W;
    const double dc0 = (uu + 0.5 - v.cx) / v.fx, dc1 = (vv + 0.5 - v.cy) / v.fy, dc2 = 1.0;
    double dw[3];
    for (int r = 0; r < 3; ++r) dw[r] = v.R[3 * r] * dc0 + (v.R[3 * r + 1] * dc1 + v.R[3 * r + 2] * dc2);
    double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    int best_face = -1;
    for (int i = 0; i < n_faces; ++i) {
        const double* f = faces + 15 * i;
        const double denom = dot3(dw, f + 11);
        if (fabs(denom) < 1e-12) continue;
        const double co[3] = {f[0] - v.t[0], f[1] - v.t[1], f[2] - v.t[2]};
        const double t = dot3(co, f + 11) / denom;
        if (t <= 1e-9 || t >= best) continue;
        double e[3];
        for (int k = 0; k < 3; ++k) e[k] = (v.t[k] + t * dw[k]) - f[k];
        if (fabs(dot3(e, f + 3)) > f[9] || fabs(dot3(e, f + 6)) > f[10]) continue;
        best = t;
        best_face = i;
    }
    const long long o = v.pix_off + px;
    if (best_face < 0) {
        td[o] = 0.0f;
        tn[3 * o] = tn[3 * o + 1] = tn[3 * o + 2] = 0.0f;
        return;
    }
    td[o] = float(best);
    const double* f = faces + 15 * best_face;
    const double flip = dot3(f + 11, dw) > 0 ? -1.0 : 1.0;
    const double fn0 = flip * f[11], fn1 = flip * f[12], fn2 = flip * f[13];
    for (int i = 0; i < 3; ++i)  // rot_wc.transpose() * n: contiguous rows, (a0+a1)+a2
        tn[3 * o + i] = float((v.R[i] * fn0 + v.R[3 + i] * fn1) + v.R[6 + i] * fn2);
}

__global__ void k_target_counts(const ViewDev* __restrict__ views, const float* __restrict__ td,
                                const float* __restrict__ tn, unsigned long long* counts) {
    const ViewDev& v = views[blockIdx.y];
    const int np = v.W * v.H;
    unsigned cd = 0, cn = 0;
    for (int px = blockIdx.x * blockDim.x + threadIdx.x; px < np; px += gridDim.x * blockDim.x) {
        const long long o = v.pix_off + px;
        cd += td[o] > 0.0f;  // geometry.hpp:61-65
        cn += (tn[3 * o] != 0.0f || tn[3 * o + 1] != 0.0f || tn[3 * o + 2] != 0.0f);
    }
    for (int off = 16; off > 0; off >>= 1) {
        cd += __shfl_xor_sync(0xffffffffu, cd, off);
        cn += __shfl_xor_sync(0xffffffffu, cn, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (cd) atomicAdd(counts + 2 * blockIdx.y, (unsigned long long)cd);
        if (cn) atomicAdd(counts + 2 * blockIdx.y + 1, (unsigned long long)cn);
    }
}

}  // namespace

void launch_plane_setup(const double* center, const double* rot, const double* radii, int64_t n,
                        PlaneGeo* out, PlaneF* outf, cudaStream_t s) {
    if (n <= 0) return;
    k_plane_setup<<<unsigned((n + 255) / 256), 256, 0, s>>>(center, rot, radii, n, out, outf);
}

void launch_rect_count(const Batch& b, const PlaneGeo* planes, int64_t P, double cut, Bins bins,
                       cudaStream_t s) {
    if (P <= 0 || b.n <= 0) return;
    // small batches at low lambda (wide cut margin, large rects): 4 row strides per
    // footprint (C3, 8 views: 124 -> 80 us at lambda 7.36; at lambda 300 the repeated
    // projection costs more than the strides save)
    dim3 grid(unsigned((P + 127) / 128), unsigned(b.n), b.n <= 16 && cut > 0.02 ? 4u : 1u);
    k_rect_count<<<grid, 128, 0, s>>>(b, planes, P, cut, bins);
}

void launch_scatter(const Batch& b, int64_t P, Bins bins, cudaStream_t s) {
    if (P <= 0 || b.n <= 0) return;
    // small batches: 8 row strides per footprint; large ones already fill the GPU
    dim3 grid(unsigned((P + 127) / 128), unsigned(b.n), b.n <= 64 ? 8u : 1u);
    k_scatter<<<grid, 128, 0, s>>>(b, P, bins);
}

void launch_big_tiles(const Batch& b, Bins bins, int threshold, cudaStream_t s) {
    if (b.n <= 0 || b.max_tiles <= 0) return;
    dim3 grid(unsigned((b.max_tiles + 127) / 128), unsigned(b.n));
    k_big_tiles<<<grid, 128, 0, s>>>(b, bins, threshold);
}

void launch_bin_guard(const Bins& bins, long long recs_cap16, long long pair_limit,
                      unsigned long long* need, double* overflow, Stats* st, cudaStream_t s) {
    k_bin_guard<<<1, 1, 0, s>>>(bins, recs_cap16, pair_limit, need, overflow, st);
}

void launch_sort_bins(const int* offsets, int* items, int T, cudaStream_t s) {
    if (T <= 0) return;
    k_sort_bins<<<(T + 127) / 128, 128, 0, s>>>(offsets, items, T);
}

void launch_render_gt(const ViewDev* views, int n_views, const double* faces, int n_faces,
                      float* td, float* tn, int max_pixels, cudaStream_t s) {
    if (n_views <= 0) return;
    dim3 grid(unsigned((max_pixels + 255) / 256), unsigned(n_views));
    k_render_gt<<<grid, 256, 0, s>>>(views, faces, n_faces, td, tn);
}

void launch_target_counts(const ViewDev* views, int n_views, const float* td, const float* tn,
                          unsigned long long* counts, cudaStream_t s) {
    if (n_views <= 0) return;
    dim3 grid(64, unsigned(n_views));
    k_target_counts<<<grid, 256, 0, s>>>(views, td, tn, counts);
}

}  // namespace psg
