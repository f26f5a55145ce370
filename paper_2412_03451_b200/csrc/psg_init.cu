// init_from_depth (scene_init.cpp:41-104) over the views'
// resident targets, bit-identical to the reference:
//   * device: per-pixel validity flags and their inclusive scan (the reference
//     streams every valid back-projected pixel, view-major, row-major);
//   * host: the reservoir's seeded RNG chain (Rng = iterated splitmix64, one draw
//     per valid pixel past the first k). The draws do not depend on pixel values,
//     only on their count, so the chain runs on the host alone: states generated
//     sequentially, the `% (m + 1)` reductions in parallel, hits applied in order;
//   * device: the k sampled pixels back-projected in the reference's operation
//     order (-fmad=false), the O(k^2) nearest-neighbour radii, quat_from_z_to.
#include <cub/device/device_scan.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "psg_internal.h"

namespace psg {
namespace {

__global__ void k_valid_flags(const float* __restrict__ td, const float* __restrict__ tn,
                              long long n, int* flags) {
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n;
         g += (long long)gridDim.x * blockDim.x) {
        const float* t = tn + 3 * g;
        flags[g] = td[g] > 0.0f && (t[0] != 0.0f || t[1] != 0.0f || t[2] != 0.0f);
    }
}

// stored Matrix3d * Vector3d: row i reduces as a0 + (a1 + a2)
__device__ __forceinline__ void mv_stored(const double* R, const double* x, double* o) {
    for (int i = 0; i < 3; ++i) o[i] = R[3 * i] * x[0] + (R[3 * i + 1] * x[1] + R[3 * i + 2] * x[2]);
}
__device__ __forceinline__ double dot3v(const double* a, const double* b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

// world point and normal of global pixel g (scene_init.cpp:50-58)
__device__ void backproject(const ViewDev& v, long long g, const float* td, const float* tn,
                            double* pw, double* nw) {
    const long long px = g - v.pix_off;
    const int u = int(px % v.W), vv = int(px / v.W);
    const double z = td[g];
    const double pc[3] = {(u + 0.5 - v.cx) / v.fx * z, (vv + 0.5 - v.cy) / v.fy * z, z};
    double m[3];
    mv_stored(v.R, pc, m);
    for (int k = 0; k < 3; ++k) pw[k] = m[k] + v.t[k];
    if (nw) {
        const double nc[3] = {double(tn[3 * g]), double(tn[3 * g + 1]), double(tn[3 * g + 2])};
        mv_stored(v.R, nc, m);
        const double n2 = dot3v(m, m);  // Vector3d::normalized
        if (n2 > 0.0) {
            const double s = sqrt(n2);
            for (int k = 0; k < 3; ++k) nw[k] = m[k] / s;
        } else {
            for (int k = 0; k < 3; ++k) nw[k] = m[k];
        }
    }
}

__device__ int view_of(const ViewDev* views, int n_views, long long g) {
    int lo = 0, hi = n_views - 1;  // last view with pix_off <= g
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (views[mid].pix_off <= g) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// sample s = valid pixel of ordinal res[s]: first g with incl[g] > ordinal
__global__ void k_gather(const ViewDev* views, int n_views, const float* td, const float* tn,
                         const int* incl, long long n_px, const long long* res, int k, double* pts,
                         double* nrm) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= k) return;
    const long long m = res[s];
    long long lo = 0, hi = n_px - 1;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if ((long long)incl[mid] > m) hi = mid;
        else lo = mid + 1;
    }
    const ViewDev& v = views[view_of(views, n_views, lo)];
    backproject(v, lo, td, tn, pts + 3 * s, nrm + 3 * s);
}

// order-preserving map of doubles to unsigned 64-bit keys (bounds via integer atomics)
__device__ __forceinline__ unsigned long long dkey(double x) {
    const unsigned long long b = __double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_bounds(const ViewDev* views, int n_views, const float* td, const float* tn,
                         const int* flags, long long n_px, unsigned long long* lohi) {
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n_px;
         g += (long long)gridDim.x * blockDim.x) {
        if (!flags[g]) continue;
        double p[3];
        backproject(views[view_of(views, n_views, g)], g, td, tn, p, nullptr);
        for (int k = 0; k < 3; ++k) {
            atomicMin(&lohi[k], dkey(p[k]));
            atomicMax(&lohi[3 + k], dkey(p[k]));
        }
    }
}

__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    return __longlong_as_double((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k);
}

// nearest neighbour per sample (scene_init.cpp:84-92) and the primitive
__global__ void k_nearest(const double* pts, const double* nrm, int k, double radius_scale,
                          const unsigned long long* lohi, double* center, double* rot,
                          double* radii) {
    __shared__ double sp[256][3];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double pi[3] = {0, 0, 0};
    if (i < k)
        for (int a = 0; a < 3; ++a) pi[a] = pts[3 * i + a];
    double nearest = CUDART_INF;
    for (int j0 = 0; j0 < k; j0 += 256) {
        __syncthreads();
        if (j0 + threadIdx.x < k)
            for (int a = 0; a < 3; ++a) sp[threadIdx.x][a] = pts[3 * (j0 + threadIdx.x) + a];
        __syncthreads();
        const int jn = min(256, k - j0);
        if (i < k)
            for (int jj = 0; jj < jn; ++jj) {
                if (j0 + jj == i) continue;
                const double d[3] = {pi[0] - sp[jj][0], pi[1] - sp[jj][1], pi[2] - sp[jj][2]};
                const double dist = sqrt(dot3v(d, d));
                nearest = dist < nearest ? dist : nearest;  // std::min(nearest, dist)
            }
    }
    if (i >= k) return;
    double radius;
    if (k > 1) {
        const double r = radius_scale * nearest;
        radius = r < 1e-4 ? 1e-4 : r;  // std::max(r, kRadiiFloor)
    } else {
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = dkey_inv(lohi[3 + a]) - dkey_inv(lohi[a]);
        const double f = 0.05 * sqrt(dot3v(d, d));
        radius = f < 10 * 1e-4 ? 10 * 1e-4 : f;
    }
    // quat_from_z_to (geometry.cpp:23-31)
    const double* n = nrm + 3 * i;
    const double e3[3] = {0.0, 0.0, 1.0};
    const double dd = dot3v(e3, n);
    double q[4];
    if (1.0 + dd < 1e-12) {
        q[0] = 0.0;
        q[1] = 1.0;
        q[2] = 0.0;
        q[3] = 0.0;
    } else {
        const double c[3] = {e3[1] * n[2] - e3[2] * n[1], e3[2] * n[0] - e3[0] * n[2],
                             e3[0] * n[1] - e3[1] * n[0]};
        const double qq[4] = {1.0 + dd, c[0], c[1], c[2]};
        const double nn = sqrt((qq[0] * qq[0] + qq[2] * qq[2]) + (qq[1] * qq[1] + qq[3] * qq[3]));
        for (int a = 0; a < 4; ++a) q[a] = qq[a] / nn;
    }
    for (int a = 0; a < 3; ++a) center[3 * i + a] = pi[a];
    for (int a = 0; a < 4; ++a) rot[4 * i + a] = q[a];
    for (int a = 0; a < 4; ++a) radii[4 * i + a] = radius;
}

uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Reservoir (scene_init.cpp:59-66) over `total` valid pixels: res[j] = ordinal of
// the sample in slot j. The state chain is sequential; the reductions of each
// batch of states run on all cores and their hits are applied in ordinal order.
void reservoir(uint64_t seed, long long total, long long k, std::vector<long long>& res) {
    const long long ke = std::min(total, k);
    res.resize(size_t(ke));
    for (long long m = 0; m < ke; ++m) res[size_t(m)] = m;
    if (total <= k) return;
    uint64_t st = splitmix64(seed);
    const int T = std::max(1, std::min(32, int(std::thread::hardware_concurrency()) - 1));
    constexpr long long kChunk = 1 << 19;
    const long long batch = kChunk * T;
    // two state buffers: the workers reduce batch b while this thread generates b + 1
    std::vector<uint64_t> states[2];
    states[0].resize(size_t(batch));
    states[1].resize(size_t(batch));
    std::vector<std::vector<std::pair<long long, long long>>> hits(static_cast<size_t>(T));
    auto gen = [&](std::vector<uint64_t>& buf, long long cnt) {
        for (long long i = 0; i < cnt; ++i) buf[size_t(i)] = st = splitmix64(st);
    };
    long long m0 = k;
    long long cnt = std::min(batch, total - m0);
    gen(states[0], cnt);
    for (int b = 0; cnt > 0; b ^= 1) {
        for (auto& h : hits) h.clear();
        std::vector<std::thread> pool;
        const std::vector<uint64_t>& cur = states[b];
        for (int w = 0; w < T; ++w) {
            const long long a = w * kChunk, e = std::min(cnt, a + kChunk);
            if (a >= e) break;
            pool.emplace_back([&, w, a, e, m0] {
                auto& hw = hits[size_t(w)];
                for (long long i = a; i < e; ++i) {
                    const uint64_t m = uint64_t(m0 + i);
                    const uint64_t j = cur[size_t(i)] % (m + 1);
                    if (j < uint64_t(k)) hw.emplace_back(m0 + i, (long long)j);
                }
            });
        }
        const long long m1 = m0 + cnt;
        const long long cnt1 = std::min(batch, total - m1);
        if (cnt1 > 0) gen(states[b ^ 1], cnt1);  // overlaps the reductions
        for (auto& t : pool) t.join();
        for (int w = 0; w < T; ++w)  // hits in ordinal order: later samples overwrite
            for (const auto& h : hits[size_t(w)]) res[size_t(h.second)] = h.first;
        m0 = m1;
        cnt = cnt1;
    }
}

}  // namespace

int init_from_depth_run(const ViewDev* d_views, int n_views, const float* td, const float* tn,
                        long long n_px, int k, uint64_t seed, double radius_scale, cudaStream_t s,
                        double** center, double** rot, double** radii, long long* k_out,
                        std::string* err) {
    *k_out = 0;
    int* flags = nullptr;
    int* incl = nullptr;
    void* tmp = nullptr;
    long long* d_res = nullptr;
    double* pts = nullptr;
    unsigned long long* lohi = nullptr;
    auto cleanup = [&] {
        cudaFree(flags);
        cudaFree(incl);
        cudaFree(tmp);
        cudaFree(d_res);
        cudaFree(pts);
        cudaFree(lohi);
    };
#define ICHK(x)                               \
    do {                                      \
        cudaError_t e_ = (x);                 \
        if (e_ != cudaSuccess) {              \
            *err = cudaGetErrorString(e_);    \
            cleanup();                        \
            return 1;                         \
        }                                     \
    } while (0)
    if (n_px <= 0 || n_px >= (1LL << 31)) {
        *err = "init_from_depth: pixel count out of range";
        return 2;
    }
    ICHK(cudaMalloc(&flags, sizeof(int) * size_t(n_px)));
    ICHK(cudaMalloc(&incl, sizeof(int) * size_t(n_px)));
    k_valid_flags<<<1184, 256, 0, s>>>(td, tn, n_px, flags);
    size_t tb = 0;
    ICHK(cub::DeviceScan::InclusiveSum(nullptr, tb, flags, incl, int(n_px), s));
    ICHK(cudaMalloc(&tmp, tb));
    ICHK(cub::DeviceScan::InclusiveSum(tmp, tb, flags, incl, int(n_px), s));
    int total = 0;
    ICHK(cudaMemcpyAsync(&total, incl + n_px - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    ICHK(cudaStreamSynchronize(s));
    if (total == 0) {
        *err = "init: no valid depth pixels in any view";
        cleanup();
        return 3;
    }
    std::vector<long long> res;
    reservoir(seed, total, k, res);
    const int ke = int(res.size());
    ICHK(cudaMalloc(&d_res, sizeof(long long) * size_t(ke)));
    ICHK(cudaMalloc(&pts, sizeof(double) * 6 * size_t(ke)));
    ICHK(cudaMalloc(&lohi, sizeof(unsigned long long) * 6));
    ICHK(cudaMemcpyAsync(d_res, res.data(), sizeof(long long) * size_t(ke), cudaMemcpyHostToDevice, s));
    k_gather<<<(ke + 127) / 128, 128, 0, s>>>(d_views, n_views, td, tn, incl, n_px, d_res, ke, pts,
                                              pts + 3 * size_t(ke));
    if (ke == 1) {  // the fallback radius needs the bounds of every valid point
        const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
        ICHK(cudaMemcpyAsync(lohi, init, sizeof init, cudaMemcpyHostToDevice, s));
        k_bounds<<<1184, 256, 0, s>>>(d_views, n_views, td, tn, flags, n_px, lohi);
    }
    ICHK(cudaMalloc(center, sizeof(double) * 3 * size_t(ke)));
    ICHK(cudaMalloc(rot, sizeof(double) * 4 * size_t(ke)));
    ICHK(cudaMalloc(radii, sizeof(double) * 4 * size_t(ke)));
    k_nearest<<<(ke + 255) / 256, 256, 0, s>>>(pts, pts + 3 * size_t(ke), ke, radius_scale, lohi,
                                               *center, *rot, *radii);
    ICHK(cudaGetLastError());
    ICHK(cudaStreamSynchronize(s));
#undef ICHK
    cleanup();
    *k_out = ke;
    return 0;
}

}  // namespace psg
