// merge_planes (optimizer.cpp:236-299) with the O(P^2) pair test on the device.
//
// Host: per-primitive frame / offset / reach in the reference's operation order
// (std::hypot from the host libm, as the reference calls it). Device: every
// pair (i < j) through the normal, offset and adjacency gates, rect_distance
// (geometry.cpp:64-149) included, with -fmad=false so each gate decides exactly
// as the reference does; passing pairs are emitted as edges. Host: connected
// components (the union-find's root is always the component's smallest index)
// and the per-instance summary and ordering of optimizer.cpp:268-298.
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "psg_internal.h"

namespace psg {
namespace {

struct MergePrim {
    double c[3], n[3], vx[3], vy[3], r[4];
    double off, reach;
};

__host__ __device__ __forceinline__ double dot3m(const double* a, const double* b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];  // Vector3d dot order
}
__host__ __device__ __forceinline__ double norm3m(const double* a) { return sqrt(dot3m(a, a)); }
__device__ __forceinline__ double clampd(double v, double lo, double hi) {  // std::clamp
    return v < lo ? lo : (hi < v ? hi : v);
}
__device__ __forceinline__ double mind(double a, double b) { return b < a ? b : a; }  // std::min

// rect_corners (geometry.cpp:64-70)
__device__ void corners(const MergePrim& p, double out[4][3]) {
    for (int k = 0; k < 3; ++k) {
        out[0][k] = (p.c[k] + p.r[0] * p.vx[k]) + p.r[2] * p.vy[k];
        out[1][k] = (p.c[k] - p.r[1] * p.vx[k]) + p.r[2] * p.vy[k];
        out[2][k] = (p.c[k] - p.r[1] * p.vx[k]) - p.r[3] * p.vy[k];
        out[3][k] = (p.c[k] + p.r[0] * p.vx[k]) - p.r[3] * p.vy[k];
    }
}

// point_rect_distance (geometry.cpp:74-80)
__device__ double point_rect(const double* x, const MergePrim& p) {
    double e[3], cl[3], d[3];
    for (int k = 0; k < 3; ++k) e[k] = x[k] - p.c[k];
    const double px = clampd(dot3m(e, p.vx), -p.r[1], p.r[0]);
    const double py = clampd(dot3m(e, p.vy), -p.r[3], p.r[2]);
    for (int k = 0; k < 3; ++k) cl[k] = (p.c[k] + px * p.vx[k]) + py * p.vy[k];
    for (int k = 0; k < 3; ++k) d[k] = x[k] - cl[k];
    return norm3m(d);
}

// segment_segment_distance (geometry.cpp:82-111)
__device__ double seg_seg(const double* p1, const double* q1, const double* p2, const double* q2) {
    double d1[3], d2[3], r[3];
    for (int k = 0; k < 3; ++k) {
        d1[k] = q1[k] - p1[k];
        d2[k] = q2[k] - p2[k];
        r[k] = p1[k] - p2[k];
    }
    const double a = dot3m(d1, d1), e = dot3m(d2, d2), f = dot3m(d2, r);
    double s = 0, t = 0;
    const double eps = 1e-15;
    if (a <= eps && e <= eps) return norm3m(r);
    if (a <= eps) {
        t = clampd(f / e, 0.0, 1.0);
    } else {
        const double c = dot3m(d1, r);
        if (e <= eps) {
            s = clampd(-c / a, 0.0, 1.0);
        } else {
            const double b = dot3m(d1, d2), denom = a * e - b * b;
            if (denom > eps) s = clampd((b * f - c * e) / denom, 0.0, 1.0);
            t = (b * s + f) / e;
            if (t < 0) {
                t = 0;
                s = clampd(-c / a, 0.0, 1.0);
            } else if (t > 1) {
                t = 1;
                s = clampd((b - c) / a, 0.0, 1.0);
            }
        }
    }
    double w[3];
    for (int k = 0; k < 3; ++k) w[k] = (p1[k] + s * d1[k]) - (p2[k] + t * d2[k]);
    return norm3m(w);
}

// segment_crosses_rect (geometry.cpp:114-127)
__device__ bool seg_crosses(const double* a, const double* b, const MergePrim& p) {
    double ea[3], eb[3];
    for (int k = 0; k < 3; ++k) {
        ea[k] = a[k] - p.c[k];
        eb[k] = b[k] - p.c[k];
    }
    const double ha = dot3m(ea, p.n), hb = dot3m(eb, p.n);
    if (ha * hb > 0) return false;
    const double denom = ha - hb;
    if (fabs(denom) < 1e-15) return false;
    const double s = ha / denom;
    double e[3];
    for (int k = 0; k < 3; ++k) e[k] = (a[k] + s * (b[k] - a[k])) - p.c[k];
    const double px = dot3m(e, p.vx), py = dot3m(e, p.vy);
    return px >= -p.r[1] && px <= p.r[0] && py >= -p.r[3] && py <= p.r[2];
}

// rect_distance (geometry.cpp:131-149)
__device__ double rect_dist(const MergePrim& A, const MergePrim& B) {
    double ca[4][3], cb[4][3];
    corners(A, ca);
    corners(B, cb);
    double best = CUDART_INF;
    for (int i = 0; i < 4; ++i) {
        best = mind(best, point_rect(ca[i], B));
        best = mind(best, point_rect(cb[i], A));
    }
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j)
            best = mind(best, seg_seg(ca[i], ca[(i + 1) & 3], cb[j], cb[(j + 1) & 3]));
    for (int i = 0; i < 4; ++i) {
        if (seg_crosses(ca[i], ca[(i + 1) & 3], B)) return 0.0;
        if (seg_crosses(cb[i], cb[(i + 1) & 3], A)) return 0.0;
    }
    return best;
}

struct MergeGates {
    double cos_gate, offset, adjacency;
    int use_adjacency;
};

constexpr int kMergeI = 32;  // primitives i per block (shared memory)

// pairs (i, j), i in this block's chunk, j one per thread; edges i < j that
// pass every gate of optimizer.cpp:256-266
__global__ void __launch_bounds__(256) k_merge_pairs(const MergePrim* __restrict__ prims, int P,
                                                     MergeGates g, int2* edges, int cap,
                                                     unsigned long long* n_edges) {
    __shared__ MergePrim si[kMergeI];
    const int i0 = blockIdx.y * kMergeI;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.x * blockDim.x + blockDim.x - 1 <= i0) return;  // whole block has j <= i
    const int ni = min(kMergeI, P - i0);
    for (int t = threadIdx.x; t < ni * int(sizeof(MergePrim) / 8); t += blockDim.x)
        reinterpret_cast<double*>(si)[t] = reinterpret_cast<const double*>(prims + i0)[t];
    __syncthreads();
    if (j >= P) return;
    const MergePrim pj = prims[j];
    for (int u = 0; u < ni; ++u) {
        const int i = i0 + u;
        if (i >= j) break;
        const MergePrim& pi = si[u];
        if (fabs(dot3m(pi.n, pj.n)) <= g.cos_gate) continue;
        if (fabs(pi.off - pj.off) >= g.offset) continue;
        if (g.use_adjacency) {
            double d[3];
            for (int k = 0; k < 3; ++k) d[k] = pi.c[k] - pj.c[k];
            const double gap = norm3m(d) - pi.reach - pj.reach;
            if (gap >= g.adjacency) continue;
            if (rect_dist(pi, pj) >= g.adjacency) continue;
        }
        const unsigned long long e = atomicAdd(n_edges, 1ull);
        if (e < (unsigned long long)cap) edges[e] = make_int2(i, j);
    }
}

// quat_normalized + plane_frame (geometry.cpp:10-40), host, reference order
void host_frame(const double* q, double* vx, double* vy, double* n) {
    const double nn = std::sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]));
    const double w = q[0] / nn, x = q[1] / nn, y = q[2] / nn, z = q[3] / nn;
    vx[0] = 1 - 2 * (y * y + z * z);
    vx[1] = 2 * (x * y + w * z);
    vx[2] = 2 * (x * z - w * y);
    vy[0] = 2 * (x * y - w * z);
    vy[1] = 1 - 2 * (x * x + z * z);
    vy[2] = 2 * (y * z + w * x);
    n[0] = 2 * (x * z + w * y);
    n[1] = 2 * (y * z - w * x);
    n[2] = 1 - 2 * (x * x + y * y);
}

}  // namespace

int merge_planes_run(int64_t P, const double* c, const double* q, const double* r,
                     const int64_t* ids, const double* sc, double normal_deg, double merge_offset,
                     double merge_adjacency, int use_adjacency, cudaStream_t s,
                     int32_t* instance_of, double* inst_normal, double* inst_offset,
                     double* inst_area, int64_t* n_inst, std::string* err) {
    *n_inst = 0;
    if (P <= 0) return 0;
    std::vector<MergePrim> h(static_cast<size_t>(P));
    for (int64_t i = 0; i < P; ++i) {
        MergePrim& m = h[size_t(i)];
        host_frame(q + 4 * i, m.vx, m.vy, m.n);
        for (int k = 0; k < 3; ++k) m.c[k] = c[3 * i + k];
        for (int k = 0; k < 4; ++k) m.r[k] = r[4 * i + k];
        double e[3];
        for (int k = 0; k < 3; ++k) e[k] = m.c[k] - sc[k];
        m.off = std::fabs(dot3m(e, m.n));
        m.reach = std::hypot(m.r[0] < m.r[1] ? m.r[1] : m.r[0], m.r[2] < m.r[3] ? m.r[3] : m.r[2]);
    }
    MergeGates g{std::cos(normal_deg * M_PI / 180.0), merge_offset, merge_adjacency, use_adjacency};
    MergePrim* d_prims = nullptr;
    int2* d_edges = nullptr;
    unsigned long long* d_n = nullptr;
    std::vector<int2> edges;
    int cap = int(std::min<int64_t>(std::max<int64_t>(4 * P, 1024), int64_t(1) << 28));
    auto cleanup = [&] {
        if (d_prims) cudaFree(d_prims);
        if (d_edges) cudaFree(d_edges);
        if (d_n) cudaFree(d_n);
    };
#define MCHK(x)                                     \
    do {                                            \
        cudaError_t e_ = (x);                       \
        if (e_ != cudaSuccess) {                    \
            *err = cudaGetErrorString(e_);          \
            cleanup();                              \
            return 1;                               \
        }                                           \
    } while (0)
    MCHK(cudaMalloc(&d_prims, sizeof(MergePrim) * size_t(P)));
    MCHK(cudaMalloc(&d_n, sizeof(unsigned long long)));
    MCHK(cudaMemcpyAsync(d_prims, h.data(), sizeof(MergePrim) * size_t(P), cudaMemcpyHostToDevice, s));
    for (;;) {
        MCHK(cudaMalloc(&d_edges, sizeof(int2) * size_t(cap)));
        MCHK(cudaMemsetAsync(d_n, 0, sizeof(unsigned long long), s));
        dim3 grid(unsigned((P + 255) / 256), unsigned((P + kMergeI - 1) / kMergeI));
        k_merge_pairs<<<grid, 256, 0, s>>>(d_prims, int(P), g, d_edges, cap, d_n);
        MCHK(cudaGetLastError());
        unsigned long long ne = 0;
        MCHK(cudaMemcpyAsync(&ne, d_n, sizeof ne, cudaMemcpyDeviceToHost, s));
        MCHK(cudaStreamSynchronize(s));
        if (ne <= (unsigned long long)cap) {
            edges.resize(size_t(ne));
            MCHK(cudaMemcpyAsync(edges.data(), d_edges, sizeof(int2) * size_t(ne), cudaMemcpyDeviceToHost, s));
            MCHK(cudaStreamSynchronize(s));
            break;
        }
        cudaFree(d_edges);
        d_edges = nullptr;
        if (ne >= (1ull << 31)) {
            *err = "merge_planes: too many candidate pairs";
            cleanup();
            return 2;
        }
        cap = int(ne);
    }
    cleanup();
#undef MCHK

    // connected components; root = smallest index (UnionFind, optimizer.cpp:216-232)
    std::vector<int32_t> parent(static_cast<size_t>(P));
    std::iota(parent.begin(), parent.end(), 0);
    auto find = [&](int32_t a) {
        while (parent[size_t(a)] != a) a = parent[size_t(a)] = parent[size_t(parent[size_t(a)])];
        return a;
    };
    for (const int2& e : edges) {
        const int32_t a = find(e.x), b = find(e.y);
        if (a != b) parent[size_t(std::max(a, b))] = std::min(a, b);
    }
    std::vector<std::vector<int32_t>> groups(static_cast<size_t>(P));
    for (int32_t i = 0; i < int32_t(P); ++i) groups[size_t(find(i))].push_back(i);

    struct Inst {
        double area, offset, normal[3];
        int64_t min_id;
        int32_t root;
    };
    std::vector<Inst> inst;
    auto area_of = [&](int32_t m) {
        const double* rm = r + 4 * int64_t(m);
        return (rm[0] + rm[1]) * (rm[2] + rm[3]);  // PlanePrimitive::area, geometry.hpp:31
    };
    for (int32_t gi = 0; gi < int32_t(P); ++gi) {
        const auto& mem = groups[size_t(gi)];
        if (mem.empty()) continue;
        Inst I{};
        I.root = gi;
        int32_t largest = mem[0];
        I.min_id = ids[mem[0]];
        for (int32_t m : mem) {
            I.area += area_of(m);
            I.min_id = std::min(I.min_id, ids[m]);
            if (area_of(m) > area_of(largest)) largest = m;
        }
        double ns[3] = {0, 0, 0};
        double os = 0;
        const double* nl = h[size_t(largest)].n;
        for (int32_t m : mem) {
            const double* nm = h[size_t(m)].n;
            const double sign = dot3m(nm, nl) < 0 ? -1.0 : 1.0;
            const double w = area_of(m) * sign;
            for (int k = 0; k < 3; ++k) ns[k] += w * nm[k];
            os += area_of(m) * h[size_t(m)].off;
        }
        const double n2 = dot3m(ns, ns);
        if (std::sqrt(n2) > 1e-12) {
            const double nn = std::sqrt(n2);
            for (int k = 0; k < 3; ++k) I.normal[k] = ns[k] / nn;
        } else {
            for (int k = 0; k < 3; ++k) I.normal[k] = nl[k];
        }
        I.offset = os / I.area;
        inst.push_back(I);
    }
    std::sort(inst.begin(), inst.end(), [](const Inst& a, const Inst& b) {
        if (a.area != b.area) return a.area > b.area;
        return a.min_id < b.min_id;
    });
    std::vector<int32_t> slot(static_cast<size_t>(P), -1);
    for (size_t t = 0; t < inst.size(); ++t) {
        slot[size_t(inst[t].root)] = int32_t(t);
        for (int k = 0; k < 3; ++k) inst_normal[3 * t + k] = inst[t].normal[k];
        inst_offset[t] = inst[t].offset;
        inst_area[t] = inst[t].area;
    }
    for (int32_t i = 0; i < int32_t(P); ++i) instance_of[i] = slot[size_t(find(i))];
    *n_inst = int64_t(inst.size());
    return 0;
}

}  // namespace psg
