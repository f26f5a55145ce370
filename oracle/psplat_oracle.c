/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 *
 * This file is the CPU oracle the CUDA path is checked against. It restates,
 * in fp64 and in the same operation order, the reference's
 *   geometry.cpp:10-63, splatting.hpp:32-51, splatting.cpp:7-40,
 *   renderer.cpp:18-528 and tests/support/{reference_renderer,test_scenes}.cpp
 * (all paths relative to /root/reference/proj). It is single-threaded; the
 * reference's results are thread-count invariant by construction
 * (renderer.cpp:502-514, test_renderer.cpp:351-381), so this is equivalent.
 *
 * Pinning: tests/test_oracle.py compares every entry point below, call for call
 * and bit for bit, with oracle/_ref/libpsplat_ref.so (the reference sources
 * compiled through oracle/eigen_shim), and checks the reference's own fixtures
 * (test_renderer.cpp, test_splatting.cpp, acceptance_main.cpp:133-292).
 *
 * Reduction order follows oracle/eigen_shim/Eigen/Core: 3-vector dots
 * (a0+a1)+a2, 4-vector dots (a0+a2)+(a1+a3), stored Matrix3d*Vector3d rows
 * a0+(a1+a2), transpose()*Vector3d rows (a0+a1)+a2.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu baseline) load this.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_api.h"

#define K_MAX_RECORD_CAP 64 /* renderer.cpp:14 */
#define K_ZCLIP 1e-6        /* renderer.cpp:15 */

/* ---------------------------------------------------------------- vectors */
typedef struct { double v[3]; } v3;
typedef struct { double v[4]; } v4;
typedef struct { double m[9]; } m3; /* row-major m[3*i+j] */

static v3 V3(double a, double b, double c) { v3 r = {{a, b, c}}; return r; }
static double dot3(v3 a, v3 b) { return (a.v[0] * b.v[0] + a.v[1] * b.v[1]) + a.v[2] * b.v[2]; }
static double dot4(v4 a, v4 b) {
    return (a.v[0] * b.v[0] + a.v[2] * b.v[2]) + (a.v[1] * b.v[1] + a.v[3] * b.v[3]);
}
static v3 add3(v3 a, v3 b) { return V3(a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]); }
static v3 sub3(v3 a, v3 b) { return V3(a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]); }
static v3 scl3(double s, v3 a) { return V3(s * a.v[0], s * a.v[1], s * a.v[2]); }
static v3 mul3s(v3 a, double s) { return V3(a.v[0] * s, a.v[1] * s, a.v[2] * s); }
static v3 div3s(v3 a, double s) { return V3(a.v[0] / s, a.v[1] / s, a.v[2] / s); }
static double norm3(v3 a) { return sqrt(dot3(a, a)); }
static v3 normalized3(v3 a) {
    const double n2 = dot3(a, a);
    return n2 > 0.0 ? div3s(a, sqrt(n2)) : a;
}
/* stored Mat3 * v: row i reduces as a0 + (a1 + a2) */
static v3 mv_stored(const m3* M, v3 x) {
    v3 r;
    for (int i = 0; i < 3; ++i)
        r.v[i] = M->m[3 * i] * x.v[0] + (M->m[3 * i + 1] * x.v[1] + M->m[3 * i + 2] * x.v[2]);
    return r;
}
static v3 col3(const m3* M, int j) { return V3(M->m[j], M->m[3 + j], M->m[6 + j]); }
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static int imin(int a, int b) { return (b < a) ? b : a; }
static int imax(int a, int b) { return (a < b) ? b : a; }
/* int(x) as x86-64 cvttsd2si executes it: out-of-range/NaN -> INT_MIN; the
 * +-1 that follows wraps (renderer.cpp:108-111 as compiled for x86-64). */
static int x86_cvt(double x) {
    if (!(x >= -2147483648.0 && x < 2147483648.0)) return (int)0x80000000u;
    return (int)x;
}
static int wrap_add(int a, int b) { return (int)((unsigned)a + (unsigned)b); }
static int all_finite3(v3 a) { return isfinite(a.v[0]) && isfinite(a.v[1]) && isfinite(a.v[2]); }

/* ---------------------------------------------------------------- geometry.cpp */
/* quat_to_matrix, geometry.cpp:10-17 */
static m3 quat_to_matrix(v4 q) {
    const double w = q.v[0], x = q.v[1], y = q.v[2], z = q.v[3];
    m3 m = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
             2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
             2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    return m;
}
/* quat_normalized, geometry.cpp:19-21: q / q.norm() */
static v4 quat_normalized(v4 q) {
    const double n = sqrt(dot4(q, q));
    v4 r = {{q.v[0] / n, q.v[1] / n, q.v[2] / n, q.v[3] / n}};
    return r;
}
typedef struct { v3 vx, vy, n; } frame_t;
/* plane_frame, geometry.cpp:33-40 */
static frame_t plane_frame(v4 q) {
    const m3 r = quat_to_matrix(q);
    frame_t f = {col3(&r, 0), col3(&r, 1), col3(&r, 2)};
    return f;
}

/* ---------------------------------------------------------------- splatting */
/* lambda_schedule, splatting.cpp:7-10 */
double orc_lambda_schedule(int64_t ite, double base, double rate, double lmax) {
    const double l = base * exp(-(1.0 - rate * (double)ite));
    return dmin(l, lmax);
}
static double sigmoid(double u) { return 1.0 / (1.0 + exp(-u)); } /* splatting.hpp:45 */
/* splat_cut_margin, splatting.hpp:48-51 */
static double splat_cut_margin(double lambda, double floor_) {
    return log(2.0 / floor_ - 1.0) / (5.0 * lambda);
}

typedef struct {
    double weight, w_x, w_y, d_px, d_py, d_radii[4];
    int x_selected;
} splat_eval;

/* plane_splat_weight, splatting.cpp:12-40 */
static splat_eval plane_splat_weight(double p_x, double p_y, const double* radii, double lambda) {
    const double k = 5.0 * lambda;
    const int bx = p_x > 0 ? 0 : 1;
    const int by = p_y > 0 ? 2 : 3;
    const double sx = sigmoid(k * (radii[bx] - fabs(p_x)));
    const double sy = sigmoid(k * (radii[by] - fabs(p_y)));
    splat_eval ev;
    memset(&ev, 0, sizeof ev);
    ev.w_x = 2.0 * sx;
    ev.w_y = 2.0 * sy;
    ev.x_selected = ev.w_x <= ev.w_y;
    const double raw = ev.x_selected ? ev.w_x : ev.w_y;
    ev.weight = dmin(raw, 1.0);
    if (raw < 1.0) {
        if (ev.x_selected) {
            const double dwdu = 2.0 * sx * (1.0 - sx);
            ev.d_radii[bx] = dwdu * k;
            ev.d_px = dwdu * k * (p_x > 0 ? -1.0 : 1.0);
        } else {
            const double dwdu = 2.0 * sy * (1.0 - sy);
            ev.d_radii[by] = dwdu * k;
            ev.d_py = dwdu * k * (p_y > 0 ? -1.0 : 1.0);
        }
    }
    return ev;
}

void orc_plane_splat_weight(double px, double py, const double* radii, double lambda, double* o) {
    const splat_eval ev = plane_splat_weight(px, py, radii, lambda);
    o[0] = ev.weight;
    o[1] = ev.w_x;
    o[2] = ev.w_y;
    o[3] = ev.d_px;
    o[4] = ev.d_py;
    for (int k = 0; k < 4; ++k) o[5 + k] = ev.d_radii[k];
    o[9] = ev.x_selected ? 1.0 : 0.0;
    o[10] = 0.0;
}

void orc_default_config(orc_config* c) { /* renderer.hpp:10-21 */
    c->max_records = 30;
    c->weight_floor = 1e-4;
    c->t_near = 0.01;
    c->parallel_eps = 1e-8;
    c->alpha_floor = 0.05;
    c->normalize_by_alpha = 0;
    c->alpha1 = 5.0;
    c->alpha2 = 1.0;
    c->tile_size = 16;
    c->threads = 0;
}

/* ---------------------------------------------------------------- renderer.cpp */
typedef struct {
    v3 vx, vy, n, s_po, m_cam;
    double k_pn, flip;
    double radii[4];
    v4 q_hat;
} prim_view; /* PrimView, renderer.cpp:18-26 */

typedef struct {
    const orc_camera* cam;
    m3 rot_wc, rot_cw;
    v3 t_wc;
} view_t;

static view_t make_view_t(const orc_camera* c) {
    view_t v;
    v.cam = c;
    memcpy(v.rot_wc.m, c->rot_wc, sizeof v.rot_wc.m);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v.rot_cw.m[3 * i + j] = c->rot_wc[3 * j + i];
    v.t_wc = V3(c->t_wc[0], c->t_wc[1], c->t_wc[2]);
    return v;
}

typedef struct {
    int64_t n;
    const double *c, *q, *r;
} planes_t;

static v3 p_center(const planes_t* P, int64_t i) {
    return V3(P->c[3 * i], P->c[3 * i + 1], P->c[3 * i + 2]);
}
static v4 p_rot(const planes_t* P, int64_t i) {
    v4 q = {{P->q[4 * i], P->q[4 * i + 1], P->q[4 * i + 2], P->q[4 * i + 3]}};
    return q;
}

/* make_prim_views, renderer.cpp:40-58 */
static prim_view* make_prim_views(const view_t* V, const planes_t* P) {
    prim_view* pvs = (prim_view*)calloc((size_t)(P->n ? P->n : 1), sizeof(prim_view));
    for (int64_t i = 0; i < P->n; ++i) {
        prim_view* pv = &pvs[i];
        pv->q_hat = quat_normalized(p_rot(P, i));
        const frame_t f = plane_frame(pv->q_hat);
        pv->vx = f.vx;
        pv->vy = f.vy;
        pv->n = f.n;
        pv->s_po = sub3(p_center(P, i), V->t_wc);
        pv->k_pn = dot3(pv->s_po, f.n);
        pv->flip = pv->k_pn < 0 ? 1.0 : -1.0;
        pv->m_cam = scl3(pv->flip, mv_stored(&V->rot_cw, f.n));
        for (int k = 0; k < 4; ++k) pv->radii[k] = P->r[4 * i + k];
    }
    return pvs;
}

typedef struct { v3 base, du, dv; } ray_basis_t;
/* ray_basis, renderer.cpp:32-38 */
static ray_basis_t ray_basis(const view_t* V) {
    const orc_camera* c = V->cam;
    ray_basis_t rb;
    rb.base = mv_stored(&V->rot_wc, V3((0.5 - c->cx) / c->fx, (0.5 - c->cy) / c->fy, 1.0));
    rb.du = div3s(col3(&V->rot_wc, 0), c->fx);
    rb.dv = div3s(col3(&V->rot_wc, 1), c->fy);
    return rb;
}

typedef struct { int u0, u1, v0, v1; } pixel_rect;

/* projected_rect, renderer.cpp:71-113 */
static pixel_rect projected_rect(const view_t* V, const prim_view* pv, v3 center, double cut) {
    const orc_camera* c = V->cam;
    const double ex_p = pv->radii[0] + cut, ex_m = pv->radii[1] + cut;
    const double ey_p = pv->radii[2] + cut, ey_m = pv->radii[3] + cut;
    v3 world[4];
    world[0] = add3(add3(center, scl3(ex_p, pv->vx)), scl3(ey_p, pv->vy));
    world[1] = add3(sub3(center, scl3(ex_m, pv->vx)), scl3(ey_p, pv->vy));
    world[2] = sub3(sub3(center, scl3(ex_m, pv->vx)), scl3(ey_m, pv->vy));
    world[3] = sub3(add3(center, scl3(ex_p, pv->vx)), scl3(ey_m, pv->vy));
    v3 poly[8];
    int n_poly = 0;
    v3 cam[4];
    for (int i = 0; i < 4; ++i) cam[i] = mv_stored(&V->rot_cw, sub3(world[i], V->t_wc));
    for (int i = 0; i < 4; ++i) {
        const v3 a = cam[i];
        const v3 b = cam[(i + 1) % 4];
        const int ain = a.v[2] >= K_ZCLIP, bin = b.v[2] >= K_ZCLIP;
        if (ain) poly[n_poly++] = a;
        if (ain != bin) {
            const double s = (K_ZCLIP - a.v[2]) / (b.v[2] - a.v[2]);
            poly[n_poly++] = add3(a, scl3(s, sub3(b, a)));
        }
    }
    pixel_rect rect = {0, -1, 0, -1};
    if (n_poly == 0) return rect;
    double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300;
    for (int i = 0; i < n_poly; ++i) {
        const double iz = 1.0 / poly[i].v[2];
        const double u = c->fx * poly[i].v[0] * iz + c->cx;
        const double v = c->fy * poly[i].v[1] * iz + c->cy;
        umin = dmin(umin, u);
        umax = dmax(umax, u);
        vmin = dmin(vmin, v);
        vmax = dmax(vmax, v);
    }
    rect.u0 = imax(0, wrap_add(x86_cvt(floor(umin - 0.5)), -1));
    rect.u1 = imin(c->width - 1, wrap_add(x86_cvt(ceil(umax - 0.5)), 1));
    rect.v0 = imax(0, wrap_add(x86_cvt(floor(vmin - 0.5)), -1));
    rect.v1 = imin(c->height - 1, wrap_add(x86_cvt(ceil(vmax - 0.5)), 1));
    return rect;
}

typedef struct {
    int tiles_x, tiles_y;
    int32_t* offsets; /* n_tiles + 1 */
    int32_t* items;   /* ascending per tile */
} binning_t;

/* bin_primitives, renderer.cpp:115-147 */
static binning_t bin_primitives(const view_t* V, const planes_t* P, const prim_view* pvs,
                                double lambda, const orc_config* cfg) {
    const orc_camera* c = V->cam;
    binning_t bin;
    bin.tiles_x = (c->width + cfg->tile_size - 1) / cfg->tile_size;
    bin.tiles_y = (c->height + cfg->tile_size - 1) / cfg->tile_size;
    const int n_tiles = bin.tiles_x * bin.tiles_y;
    const double cut = splat_cut_margin(lambda, cfg->weight_floor) * 1.05;
    pixel_rect* rects = (pixel_rect*)malloc(sizeof(pixel_rect) * (size_t)(P->n ? P->n : 1));
    int32_t* counts = (int32_t*)calloc((size_t)n_tiles, sizeof(int32_t));
    const int ts = cfg->tile_size;
    for (int64_t i = 0; i < P->n; ++i) {
        rects[i] = projected_rect(V, &pvs[i], p_center(P, i), cut);
        const pixel_rect r = rects[i];
        if (r.u0 > r.u1 || r.v0 > r.v1) continue;
        for (int ty = r.v0 / ts; ty <= r.v1 / ts; ++ty)
            for (int tx = r.u0 / ts; tx <= r.u1 / ts; ++tx) counts[ty * bin.tiles_x + tx]++;
    }
    bin.offsets = (int32_t*)calloc((size_t)n_tiles + 1, sizeof(int32_t));
    for (int t = 0; t < n_tiles; ++t) bin.offsets[t + 1] = bin.offsets[t] + counts[t];
    bin.items = (int32_t*)malloc(sizeof(int32_t) * (size_t)(bin.offsets[n_tiles] + 1));
    for (int t = 0; t < n_tiles; ++t) counts[t] = bin.offsets[t]; /* cursor */
    for (int64_t i = 0; i < P->n; ++i) {
        const pixel_rect r = rects[i];
        if (r.u0 > r.u1 || r.v0 > r.v1) continue;
        for (int ty = r.v0 / ts; ty <= r.v1 / ts; ++ty)
            for (int tx = r.u0 / ts; tx <= r.u1 / ts; ++tx)
                bin.items[counts[ty * bin.tiles_x + tx]++] = (int32_t)i;
    }
    free(rects);
    free(counts);
    return bin;
}
static void free_binning(binning_t* b) {
    free(b->offsets);
    free(b->items);
}

/* eval_candidate, renderer.cpp:159-184 */
static int eval_candidate(v3 d, double mu, const prim_view* pv, double lambda,
                          const orc_config* cfg, double arg_cut, double* z_out, double* w_out) {
    const double denom = dot3(d, pv->n);
    if (fabs(denom) < cfg->parallel_eps) return 0;
    const double t = pv->k_pn / denom;
    if (t <= cfg->t_near) return 0;
    const double k = 5.0 * lambda;
    const v3 e = sub3(scl3(t, d), pv->s_po);
    const double px = dot3(e, pv->vx);
    const double ax = k * ((px > 0 ? pv->radii[0] : pv->radii[1]) - fabs(px));
    if (ax < -(arg_cut + 1.0)) return 0;
    const double py = dot3(e, pv->vy);
    const double ay = k * ((py > 0 ? pv->radii[2] : pv->radii[3]) - fabs(py));
    if (ay < -(arg_cut + 1.0)) return 0;
    const double wx = 2.0 * sigmoid(ax);
    const double wy = 2.0 * sigmoid(ay);
    const double w = dmin(dmin(wx, wy), 1.0);
    if (w < cfg->weight_floor) return 0;
    *z_out = t * mu;
    *w_out = w;
    return 1;
}

static int check_cfg(const orc_camera* cam, const orc_config* cfg) {
    if (cam->width < 1 || cam->height < 1) return 1;          /* renderer.cpp:233 */
    if (cfg->max_records > K_MAX_RECORD_CAP) return 1;        /* renderer.cpp:234-235 */
    return 0;
}

/* Renderer::render_view, renderer.cpp:231-317 (tile loop run serially) */
int orc_render_view(const orc_camera* cam, int64_t n, const double* center,
                    const double* rotation, const double* radii, double lambda,
                    const orc_config* cfg, int keep, double* depth, double* normal,
                    double* alpha, int32_t* rec_prim, uint16_t* rec_count) {
    if (check_cfg(cam, cfg)) return 1;
    const int W = cam->width, H = cam->height, M = cfg->max_records;
    const size_t np = (size_t)W * (size_t)H;
    memset(depth, 0, np * sizeof(double));
    memset(normal, 0, 3 * np * sizeof(double));
    memset(alpha, 0, np * sizeof(double));
    if (keep) {
        for (size_t i = 0; i < np * (size_t)M; ++i) rec_prim[i] = -1;
        memset(rec_count, 0, np * sizeof(uint16_t));
    }
    const view_t V = make_view_t(cam);
    const planes_t P = {n, center, rotation, radii};
    prim_view* pvs = make_prim_views(&V, &P);
    binning_t bin = bin_primitives(&V, &P, pvs, lambda, cfg);
    const ray_basis_t rb = ray_basis(&V);
    const double arg_cut = log(2.0 / cfg->weight_floor - 1.0);
    const int ts = cfg->tile_size;
    double rz[K_MAX_RECORD_CAP], rw[K_MAX_RECORD_CAP];
    int32_t rp[K_MAX_RECORD_CAP];
    for (int job = 0; job < bin.tiles_x * bin.tiles_y; ++job) {
        const int tx = job % bin.tiles_x, ty = job / bin.tiles_x;
        const int32_t* cand = bin.items + bin.offsets[job];
        const int n_cand = bin.offsets[job + 1] - bin.offsets[job];
        if (n_cand == 0) continue;
        const int u0 = tx * ts, u1 = imin(W, u0 + ts);
        const int v0 = ty * ts, v1 = imin(H, v0 + ts);
        for (int v = v0; v < v1; ++v) {
            for (int u = u0; u < u1; ++u) {
                const v3 dir_un = add3(add3(rb.base, scl3((double)u, rb.du)), scl3((double)v, rb.dv));
                const double inv_len = 1.0 / norm3(dir_un);
                const v3 d = mul3s(dir_un, inv_len);
                const double mu = inv_len;
                int cnt = 0;
                for (int ci = 0; ci < n_cand; ++ci) {
                    const int32_t pi = cand[ci];
                    double z, w;
                    if (!eval_candidate(d, mu, &pvs[pi], lambda, cfg, arg_cut, &z, &w)) continue;
                    int pos = cnt;
                    while (pos > 0 && (rz[pos - 1] > z || (rz[pos - 1] == z && rp[pos - 1] > pi)))
                        --pos;
                    if (pos == M) continue;
                    const int last = imin(cnt, M - 1);
                    for (int s = last; s > pos; --s) {
                        rz[s] = rz[s - 1];
                        rw[s] = rw[s - 1];
                        rp[s] = rp[s - 1];
                    }
                    rz[pos] = z;
                    rw[pos] = w;
                    rp[pos] = pi;
                    if (cnt < M) ++cnt;
                }
                const size_t px = (size_t)v * (size_t)W + (size_t)u;
                double dd = 0, aa = 0, tr = 1.0;
                v3 nn = V3(0, 0, 0);
                for (int j = 0; j < cnt; ++j) {
                    const double cc = tr * rw[j];
                    dd += cc * rz[j];
                    nn = add3(nn, scl3(cc, pvs[rp[j]].m_cam));
                    aa += cc;
                    tr *= 1.0 - rw[j];
                }
                depth[px] = dd;
                alpha[px] = aa;
                normal[3 * px] = nn.v[0];
                normal[3 * px + 1] = nn.v[1];
                normal[3 * px + 2] = nn.v[2];
                if (keep) {
                    rec_count[px] = (uint16_t)cnt;
                    for (int j = 0; j < cnt; ++j) rec_prim[px * (size_t)M + (size_t)j] = rp[j];
                }
            }
        }
    }
    free_binning(&bin);
    free(pvs);
    return 0;
}

static double sgn(double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); }

/* Renderer::render_loss, renderer.cpp:319-371 */
int orc_render_loss(const orc_camera* cam, const float* td, const float* tn,
                    const orc_config* cfg, const double* depth, const double* normal,
                    const double* alpha, double* loss, double* d_depth, double* d_normal,
                    double* d_alpha) {
    const size_t np = (size_t)cam->width * (size_t)cam->height;
    memset(d_depth, 0, np * sizeof(double));
    memset(d_normal, 0, 3 * np * sizeof(double));
    if (d_alpha) memset(d_alpha, 0, np * sizeof(double));
    size_t count_d = 0, count_n = 0;
    for (size_t px = 0; px < np; ++px) { /* geometry.hpp:61-65 */
        if (td[px] > 0.0f) ++count_d;
        if (tn[3 * px] != 0.0f || tn[3 * px + 1] != 0.0f || tn[3 * px + 2] != 0.0f) ++count_n;
    }
    const double inv_d = count_d ? 1.0 / (double)count_d : 0.0;
    const double inv_n = count_n ? 1.0 / (double)count_n : 0.0;
    double sum_depth = 0, sum_normal = 0;
    for (size_t px = 0; px < np; ++px) {
        const double a = alpha[px];
        if (a < cfg->alpha_floor) continue;
        const int norm_on = cfg->normalize_by_alpha && a > 1e-12;
        const double scale = norm_on ? 1.0 / a : 1.0;
        if (td[px] > 0.0f) {
            const double dr = depth[px] * scale;
            const double diff = dr - (double)td[px];
            sum_depth += fabs(diff);
            const double g = cfg->alpha2 * sgn(diff) * inv_d;
            d_depth[px] = g * scale;
            if (norm_on && d_alpha) d_alpha[px] -= g * dr * scale;
        }
        if (tn[3 * px] != 0.0f || tn[3 * px + 1] != 0.0f || tn[3 * px + 2] != 0.0f) {
            const v3 nr = V3(normal[3 * px] * scale, normal[3 * px + 1] * scale,
                             normal[3 * px + 2] * scale);
            const v3 nt = V3((double)tn[3 * px], (double)tn[3 * px + 1], (double)tn[3 * px + 2]);
            const double cos_term = 1.0 - dot3(nr, nt);
            sum_normal += fabs(cos_term);
            v3 g = scl3(-sgn(cos_term), nt);
            for (int k = 0; k < 3; ++k) {
                sum_normal += fabs(nr.v[k] - nt.v[k]);
                g.v[k] += sgn(nr.v[k] - nt.v[k]);
            }
            const double gs = cfg->alpha1 * inv_n;
            for (int k = 0; k < 3; ++k) g.v[k] *= gs;
            for (int k = 0; k < 3; ++k) d_normal[3 * px + k] = g.v[k] * scale;
            if (norm_on && d_alpha) d_alpha[px] -= dot3(g, nr) * scale;
        }
    }
    *loss = cfg->alpha1 * sum_normal * inv_n + cfg->alpha2 * sum_depth * inv_d;
    return 0;
}

/* Renderer::backward, renderer.cpp:373-528 */
int orc_backward(const orc_camera* cam, int64_t n, const double* center, const double* rotation,
                 const double* radii, const int64_t* ids, double lambda, const orc_config* cfg,
                 int M, const int32_t* rec_prim, const uint16_t* rec_count, const double* d_depth,
                 const double* d_normal, const double* d_alpha, double* grads, char* err,
                 int errlen) {
    if (!rec_count) { /* renderer.cpp:376-377 */
        if (err) snprintf(err, (size_t)errlen, "backward: forward pass ran without keep_records");
        return 1;
    }
    const int W = cam->width, H = cam->height;
    const view_t V = make_view_t(cam);
    const planes_t P = {n, center, rotation, radii};
    prim_view* pvs = make_prim_views(&V, &P);
    binning_t bin = bin_primitives(&V, &P, pvs, lambda, cfg);
    const ray_basis_t rb = ray_basis(&V);
    const int has_alpha_grad = d_alpha != NULL;
    const int ts = cfg->tile_size;

    /* quaternion jacobians, renderer.cpp:385-402 (row-major 3x4) */
    double(*jvx)[12] = malloc(sizeof(double[12]) * (size_t)(n ? n : 1));
    double(*jvy)[12] = malloc(sizeof(double[12]) * (size_t)(n ? n : 1));
    double(*jn)[12] = malloc(sizeof(double[12]) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        const double qw = pvs[i].q_hat.v[0], qx = pvs[i].q_hat.v[1], qy = pvs[i].q_hat.v[2],
                     qz = pvs[i].q_hat.v[3];
        const double a[12] = {0, 0, -4 * qy, -4 * qz, 2 * qz, 2 * qy, 2 * qx, 2 * qw,
                              -2 * qy, 2 * qz, -2 * qw, 2 * qx};
        const double b[12] = {-2 * qz, 2 * qy, 2 * qx, -2 * qw, 0, -4 * qx, 0, -4 * qz,
                              2 * qx, 2 * qw, 2 * qz, 2 * qy};
        const double c[12] = {2 * qy, 2 * qz, 2 * qw, 2 * qx, -2 * qx, -2 * qw, 2 * qz, 2 * qy,
                              0, -4 * qx, -4 * qy, 0};
        memcpy(jvx[i], a, sizeof a);
        memcpy(jvy[i], b, sizeof b);
        memcpy(jn[i], c, sizeof c);
    }
    const int n_tiles = bin.tiles_x * bin.tiles_y;
    double* local = NULL; /* per-slot PrimGrad: 11 doubles */
    double rz[K_MAX_RECORD_CAP], rw[K_MAX_RECORD_CAP], rt[K_MAX_RECORD_CAP];
    double rpx[K_MAX_RECORD_CAP], rpy[K_MAX_RECORD_CAP], rT[K_MAX_RECORD_CAP], rphi[K_MAX_RECORD_CAP];
    /* tile_grads kept per tile so the reduction below runs in tile order */
    double** tile_grads = (double**)calloc((size_t)n_tiles, sizeof(double*));
    for (int job = 0; job < n_tiles; ++job) {
        const int32_t* cand = bin.items + bin.offsets[job];
        const int n_cand = bin.offsets[job + 1] - bin.offsets[job];
        if (n_cand == 0) continue;
        const int tx = job % bin.tiles_x, ty = job / bin.tiles_x;
        const int u0 = tx * ts, u1 = imin(W, u0 + ts);
        const int v0 = ty * ts, v1 = imin(H, v0 + ts);
        local = (double*)calloc((size_t)n_cand * 11, sizeof(double));
        for (int v = v0; v < v1; ++v) {
            for (int u = u0; u < u1; ++u) {
                const size_t px = (size_t)v * (size_t)W + (size_t)u;
                const int cnt = rec_count[px];
                if (cnt == 0) continue;
                const double g_d = d_depth[px];
                const v3 g_n = V3(d_normal[3 * px], d_normal[3 * px + 1], d_normal[3 * px + 2]);
                const double g_a = has_alpha_grad ? d_alpha[px] : 0.0;
                /* Eigen isZero(): every |coeff| <= 1e-12 */
                const int gn_zero = fabs(g_n.v[0]) <= 1e-12 && fabs(g_n.v[1]) <= 1e-12 &&
                                    fabs(g_n.v[2]) <= 1e-12;
                if (g_d == 0.0 && g_a == 0.0 && gn_zero) continue;
                const v3 dir_un = add3(add3(rb.base, scl3((double)u, rb.du)), scl3((double)v, rb.dv));
                const double inv_len = 1.0 / norm3(dir_un);
                const v3 d = mul3s(dir_un, inv_len);
                const double mu = inv_len;
                const v3 g_n_world = mv_stored(&V.rot_wc, g_n);
                double tr = 1.0;
                for (int j = 0; j < cnt; ++j) {
                    const int32_t pi = rec_prim[px * (size_t)M + (size_t)j];
                    const prim_view* pv = &pvs[pi];
                    const double denom = dot3(d, pv->n);
                    const double t = pv->k_pn / denom;
                    const v3 e = sub3(scl3(t, d), pv->s_po);
                    rt[j] = t;
                    rz[j] = t * mu;
                    rpx[j] = dot3(e, pv->vx);
                    rpy[j] = dot3(e, pv->vy);
                    const splat_eval ev = plane_splat_weight(rpx[j], rpy[j], pv->radii, lambda);
                    rw[j] = ev.weight;
                    rT[j] = tr;
                    tr *= 1.0 - ev.weight;
                    rphi[j] = g_d * rz[j] + dot3(g_n, pv->m_cam) + g_a;
                }
                double suffix = 0.0;
                for (int j = cnt - 1; j >= 0; --j) {
                    const int32_t pi = rec_prim[px * (size_t)M + (size_t)j];
                    const prim_view* pv = &pvs[pi];
                    const double g_w = rT[j] * (rphi[j] - suffix);
                    suffix = rw[j] * rphi[j] + (1.0 - rw[j]) * suffix;
                    const double c = rT[j] * rw[j];
                    const double g_z = c * g_d;
                    const splat_eval ev = plane_splat_weight(rpx[j], rpy[j], pv->radii, lambda);
                    const double denom = dot3(d, pv->n);
                    const double t = rt[j];
                    const v3 e = sub3(scl3(t, d), pv->s_po);
                    const double d_p_sel = ev.x_selected ? ev.d_px : ev.d_py;
                    const v3 v_sel = ev.x_selected ? pv->vx : pv->vy;
                    const double* j_sel = ev.x_selected ? jvx[pi] : jvy[pi];
                    const double d_dot_vsel = dot3(d, v_sel);
                    /* slot_of: lower_bound over the ascending candidate list (:417-419) */
                    int lo = 0, hi = n_cand;
                    while (lo < hi) {
                        const int mid = (lo + hi) / 2;
                        if (cand[mid] < pi) lo = mid + 1; else hi = mid;
                    }
                    double* pg = local + 11 * (size_t)lo;
                    const double coef_n = (g_w * d_p_sel * d_dot_vsel + g_z * mu) / denom;
                    for (int k = 0; k < 3; ++k)
                        pg[k] += coef_n * pv->n.v[k] - (g_w * d_p_sel) * v_sel.v[k];
                    for (int k = 0; k < 4; ++k) pg[7 + k] += g_w * ev.d_radii[k];
                    const v3 s_minus_td = sub3(pv->s_po, scl3(t, d));
                    for (int a = 0; a < 4; ++a) {
                        const v3 dn_a = V3(jn[pi][a], jn[pi][4 + a], jn[pi][8 + a]);
                        const double dt_a = dot3(s_minus_td, dn_a) / denom;
                        const double dp_a =
                            d_dot_vsel * dt_a + dot3(e, V3(j_sel[a], j_sel[4 + a], j_sel[8 + a]));
                        pg[3 + a] += g_w * d_p_sel * dp_a + g_z * mu * dt_a +
                                     c * pv->flip * dot3(g_n_world, dn_a);
                    }
                }
            }
        }
        tile_grads[job] = local;
    }
    /* ordered reduction over tiles, renderer.cpp:502-514 */
    for (int tile = 0; tile < n_tiles; ++tile) {
        if (!tile_grads[tile]) continue;
        const int32_t* cand = bin.items + bin.offsets[tile];
        const int n_cand = bin.offsets[tile + 1] - bin.offsets[tile];
        for (int ci = 0; ci < n_cand; ++ci)
            for (int k = 0; k < 11; ++k) grads[11 * (size_t)cand[ci] + k] += tile_grads[tile][11 * ci + k];
        free(tile_grads[tile]);
    }
    free(tile_grads);
    /* tangent projection + finiteness, renderer.cpp:516-527 */
    int status = 0;
    for (int64_t i = 0; i < n; ++i) {
        double* pg = grads + 11 * i;
        const v4 dr = {{pg[3], pg[4], pg[5], pg[6]}};
        const double qd = dot4(pvs[i].q_hat, dr);
        for (int k = 0; k < 4; ++k) pg[3 + k] -= pvs[i].q_hat.v[k] * qd;
        const v3 dc = V3(pg[0], pg[1], pg[2]);
        const v3 dq3 = V3(pg[3], pg[4], pg[5]);
        if (!all_finite3(dc) || !all_finite3(dq3) || !isfinite(pg[6]) || !isfinite(pg[7]) ||
            !isfinite(pg[8]) || !isfinite(pg[9]) || !isfinite(pg[10])) {
            if (err)
                snprintf(err, (size_t)errlen, "backward: non-finite gradient for primitive id %lld",
                         (long long)(ids ? ids[i] : i));
            status = 3;
            break;
        }
    }
    free(jvx);
    free(jvy);
    free(jn);
    free_binning(&bin);
    free(pvs);
    return status;
}

int64_t orc_bin_primitives(const orc_camera* cam, int64_t n, const double* center,
                           const double* rotation, const double* radii, double lambda,
                           const orc_config* cfg, int32_t* offsets, int32_t* items, int64_t cap) {
    const view_t V = make_view_t(cam);
    const planes_t P = {n, center, rotation, radii};
    prim_view* pvs = make_prim_views(&V, &P);
    binning_t bin = bin_primitives(&V, &P, pvs, lambda, cfg);
    const int n_tiles = bin.tiles_x * bin.tiles_y;
    const int64_t total = bin.offsets[n_tiles];
    if (offsets) memcpy(offsets, bin.offsets, sizeof(int32_t) * ((size_t)n_tiles + 1));
    if (items && cap >= total) memcpy(items, bin.items, sizeof(int32_t) * (size_t)total);
    free_binning(&bin);
    free(pvs);
    return total;
}

/* ---------------------------------------------------------------- naive oracle */
typedef struct { int32_t prim; double z, w; v3 n_cam; } irec;

static int irec_cmp(const void* pa, const void* pb) {
    const irec* a = (const irec*)pa;
    const irec* b = (const irec*)pb;
    if (a->z != b->z) return a->z < b->z ? -1 : 1;
    return (a->prim > b->prim) - (a->prim < b->prim);
}

/* generate_ray (geometry.cpp:42-50) + gather_intersections (renderer.cpp:188-216) */
static int gather(const view_t* V, const planes_t* P, const frame_t* frames, double lambda,
                  const orc_config* cfg, int u, int v, irec* out /* cap n */) {
    const orc_camera* c = V->cam;
    const v3 d_cam = V3((u + 0.5 - c->cx) / c->fx, (v + 0.5 - c->cy) / c->fy, 1.0);
    const v3 dir = normalized3(mv_stored(&V->rot_wc, d_cam));
    const v3 origin = V->t_wc;
    const v3 cam_z = col3(&V->rot_wc, 2);
    int cnt = 0;
    for (int64_t i = 0; i < P->n; ++i) {
        const frame_t* f = &frames[i];
        const double denom = dot3(dir, f->n); /* intersect, geometry.cpp:52-63 */
        if (fabs(denom) < cfg->parallel_eps) continue;
        const double t = dot3(sub3(p_center(P, i), origin), f->n) / denom;
        if (t <= cfg->t_near) continue;
        const v3 point = add3(origin, scl3(t, dir));
        const double z_cam = t * dot3(dir, cam_z);
        const v3 e = sub3(point, p_center(P, i)); /* project_local, splatting.hpp:32-37 */
        const double px = dot3(e, f->vx), py = dot3(e, f->vy);
        const splat_eval ev = plane_splat_weight(px, py, P->r + 4 * i, lambda);
        if (ev.weight < cfg->weight_floor) continue;
        const double flip = dot3(sub3(p_center(P, i), origin), f->n) < 0 ? 1.0 : -1.0;
        out[cnt].prim = (int32_t)i;
        out[cnt].z = z_cam;
        out[cnt].w = ev.weight;
        out[cnt].n_cam = scl3(flip, mv_stored(&V->rot_cw, f->n));
        ++cnt;
    }
    qsort(out, (size_t)cnt, sizeof(irec), irec_cmp); /* strict total order: stable not needed */
    if (cnt > cfg->max_records) cnt = cfg->max_records;
    return cnt;
}

static frame_t* build_frames(const planes_t* P) { /* reference_renderer.cpp:13-20 */
    frame_t* f = (frame_t*)malloc(sizeof(frame_t) * (size_t)(P->n ? P->n : 1));
    for (int64_t i = 0; i < P->n; ++i) f[i] = plane_frame(quat_normalized(p_rot(P, i)));
    return f;
}

int orc_gather_intersections(const orc_camera* cam, int64_t n, const double* center,
                             const double* rotation, const double* radii, double lambda,
                             const orc_config* cfg, int u, int v, int32_t* prim, double* z,
                             double* w, int cap) {
    const view_t V = make_view_t(cam);
    const planes_t P = {n, center, rotation, radii};
    frame_t* frames = build_frames(&P);
    irec* recs = (irec*)malloc(sizeof(irec) * (size_t)(n ? n : 1));
    const int cnt = gather(&V, &P, frames, lambda, cfg, u, v, recs);
    for (int i = 0; i < cnt && i < cap; ++i) {
        prim[i] = recs[i].prim;
        z[i] = recs[i].z;
        w[i] = recs[i].w;
    }
    free(recs);
    free(frames);
    return cnt;
}

/* reference_render, tests/support/reference_renderer.cpp:22-40 + composite (renderer.cpp:218-229) */
int orc_reference_render(const orc_camera* cam, int64_t n, const double* center,
                         const double* rotation, const double* radii, double lambda,
                         const orc_config* cfg, double* depth, double* normal, double* alpha) {
    const view_t V = make_view_t(cam);
    const planes_t P = {n, center, rotation, radii};
    frame_t* frames = build_frames(&P);
    irec* recs = (irec*)malloc(sizeof(irec) * (size_t)(n ? n : 1));
    for (int v = 0; v < cam->height; ++v) {
        for (int u = 0; u < cam->width; ++u) {
            const int cnt = gather(&V, &P, frames, lambda, cfg, u, v, recs);
            double dd = 0, aa = 0, tr = 1.0;
            v3 nn = V3(0, 0, 0);
            for (int j = 0; j < cnt; ++j) {
                const double c = tr * recs[j].w;
                dd += c * recs[j].z;
                nn = add3(nn, scl3(c, recs[j].n_cam));
                aa += c;
                tr *= 1.0 - recs[j].w;
            }
            const size_t i = (size_t)v * (size_t)cam->width + (size_t)u;
            depth[i] = dd;
            alpha[i] = aa;
            for (int k = 0; k < 3; ++k) normal[3 * i + k] = nn.v[k];
        }
    }
    free(recs);
    free(frames);
    return 0;
}

/* ---------------------------------------------------------------- test_scenes.cpp */
static uint64_t splitmix64(uint64_t x) { /* test_scenes.cpp:7-12 */
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
typedef struct { uint64_t state; } test_rng;
static test_rng rng_make(uint64_t seed) { test_rng r = {splitmix64(seed)}; return r; }
static uint64_t rng_next(test_rng* r) { return r->state = splitmix64(r->state); }
static double rng_uniform(test_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform2(test_rng* r, double lo, double hi) { return lo + (hi - lo) * rng_uniform(r); }

/* The reference builds vectors with parenthesised constructors whose argument
 * evaluation order C++ leaves unspecified; GCC on x86-64 evaluates them last to
 * first. ORC_ARGS3/4 draw in that order and return the values positionally. */
static v3 rng_v3(test_rng* r, double lo, double hi) {
    const double c = rng_uniform2(r, lo, hi);
    const double b = rng_uniform2(r, lo, hi);
    const double a = rng_uniform2(r, lo, hi);
    return V3(a, b, c);
}
static v3 unit_vector(test_rng* r) { /* test_scenes.cpp:21-27 */
    for (;;) {
        const v3 v = rng_v3(r, -1, 1);
        const double n = norm3(v);
        if (n > 1e-3 && n < 1.0) return div3s(v, n);
    }
}
static v4 unit_quat(test_rng* r) { /* test_scenes.cpp:29-35 */
    for (;;) {
        const double d = rng_uniform2(r, -1, 1);
        const double c = rng_uniform2(r, -1, 1);
        const double b = rng_uniform2(r, -1, 1);
        const double a = rng_uniform2(r, -1, 1);
        const v4 q = {{a, b, c, d}};
        const double n = sqrt(dot4(q, q));
        if (n > 1e-3 && n < 1.0) {
            v4 o = {{q.v[0] / n, q.v[1] / n, q.v[2] / n, q.v[3] / n}};
            return o;
        }
    }
}

void orc_random_scene(uint64_t seed, int n, double* c, double* q, double* r, int64_t* ids) {
    test_rng rng = rng_make(seed); /* test_scenes.cpp:37-50 */
    for (int i = 0; i < n; ++i) {
        const double z = rng_uniform2(&rng, 1.8, 3.2);
        const double cy = rng_uniform2(&rng, -0.5, 0.5) * z;
        const double cx = rng_uniform2(&rng, -0.5, 0.5) * z;
        c[3 * i] = cx;
        c[3 * i + 1] = cy;
        c[3 * i + 2] = z;
        const v4 qq = unit_quat(&rng);
        for (int k = 0; k < 4; ++k) q[4 * i + k] = qq.v[k];
        for (int k = 0; k < 4; ++k) r[4 * i + k] = rng_uniform2(&rng, 0.2, 0.7);
        if (ids) ids[i] = i;
    }
}

void orc_make_view(int width, int height, double focal, int random_pose, uint64_t seed,
                   orc_camera* cam) { /* test_scenes.cpp:52-69 */
    memset(cam, 0, sizeof *cam);
    cam->width = width;
    cam->height = height;
    cam->fx = cam->fy = focal;
    cam->cx = width / 2.0;
    cam->cy = height / 2.0;
    cam->rot_wc[0] = cam->rot_wc[4] = cam->rot_wc[8] = 1.0;
    if (random_pose) {
        test_rng rng = rng_make(seed ^ 0x7e57ull);
        const v3 axis = unit_vector(&rng);
        const double angle = rng_uniform2(&rng, -0.15, 0.15);
        const v4 q = {{cos(angle / 2), sin(angle / 2) * axis.v[0], sin(angle / 2) * axis.v[1],
                       sin(angle / 2) * axis.v[2]}};
        const m3 R = quat_to_matrix(quat_normalized(q));
        memcpy(cam->rot_wc, R.m, sizeof R.m);
        const v3 t = rng_v3(&rng, -0.1, 0.1);
        for (int k = 0; k < 3; ++k) cam->t_wc[k] = t.v[k];
    }
}

void orc_fill_random_targets(const orc_camera* cam, uint64_t seed, float* td, float* tn) {
    test_rng rng = rng_make(seed ^ 0x7a67ull); /* test_scenes.cpp:71-81 */
    const size_t np = (size_t)cam->width * (size_t)cam->height;
    for (size_t px = 0; px < np; ++px) {
        td[px] = (float)rng_uniform2(&rng, 1.5, 4.0);
        v3 n = unit_vector(&rng);
        if (n.v[2] > 0) n = scl3(-1.0, n);
        for (int k = 0; k < 3; ++k) tn[3 * px + k] = (float)n.v[k];
    }
}

/* pipeline_loss + fd_loss_gradient, test_scenes.cpp:83-107 */
static double pipeline_loss(const orc_camera* cam, const float* td, const float* tn, int64_t n,
                            const double* c, const double* q, const double* r, double lambda,
                            const orc_config* cfg) {
    const size_t np = (size_t)cam->width * (size_t)cam->height;
    double* buf = (double*)malloc(sizeof(double) * np * 10);
    double *depth = buf, *normal = buf + np, *alpha = buf + 4 * np, *dd = buf + 5 * np,
           *dn = buf + 6 * np;
    orc_render_view(cam, n, c, q, r, lambda, cfg, 0, depth, normal, alpha, NULL, NULL);
    double loss = 0;
    double* da = cfg->normalize_by_alpha ? buf + 9 * np : NULL;
    orc_render_loss(cam, td, tn, cfg, depth, normal, alpha, &loss, dd, dn, da);
    free(buf);
    return loss;
}

double orc_fd_loss_gradient(const orc_camera* cam, const float* td, const float* tn, int64_t n,
                            const double* c, const double* q, const double* r, int64_t prim,
                            int param, double lambda, double step, const orc_config* cfg) {
    double* cc = (double*)malloc(sizeof(double) * (size_t)(n * 11 + 1));
    double *c2 = cc, *q2 = cc + 3 * n, *r2 = cc + 7 * n;
    memcpy(c2, c, sizeof(double) * (size_t)(3 * n));
    memcpy(q2, q, sizeof(double) * (size_t)(4 * n));
    memcpy(r2, r, sizeof(double) * (size_t)(4 * n));
    double* slot = param < 3 ? &c2[3 * prim + param]
                   : param < 7 ? &q2[4 * prim + param - 3]
                               : &r2[4 * prim + param - 7];
    *slot += step;
    const double up = pipeline_loss(cam, td, tn, n, c2, q2, r2, lambda, cfg);
    *slot += -2 * step;
    const double down = pipeline_loss(cam, td, tn, n, c2, q2, r2, lambda, cfg);
    *slot += step;
    free(cc);
    return (up - down) / (2 * step);
}

/* ---------------------------------------------------------------- optimizer */
void orc_default_optim_config(orc_optim_config* c) { /* optimizer.hpp:10-27 */
    c->lr_center = 0.001;
    c->lr_radii = 0.001;
    c->lr_rotation = 0.001;
    c->beta1 = 0.9;
    c->beta2 = 0.999;
    c->eps = 1e-8;
    c->split_interval = 1000;
    c->split_grad_threshold = 0.2;
    c->enable_split = 1;
    c->single_radii = 0;
    c->merge_normal_deg = 25.0;
    c->merge_offset = 0.1;
    c->merge_adjacency = 0.05;
    c->merge_use_adjacency = 1;
    c->views_per_step = 1;
    c->seed = 0;
    c->radii_floor = 1e-4; /* kRadiiFloor, geometry.hpp:19 */
}

/* Optimizer::view_for_slot (optimizer.cpp:49-59) with seeded_shuffle
 * (optimizer.cpp:22-28): Fisher-Yates over iota(n), generator splitmix64
 * iterated from splitmix64(seed) ^ splitmix64(epoch). */
int64_t orc_view_for_slot(uint64_t seed, int64_t n_views, int64_t slot) {
    if (n_views <= 0) return -1;
    const int64_t epoch = slot / n_views;
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_views);
    for (int64_t i = 0; i < n_views; ++i) order[i] = i;
    uint64_t s = splitmix64(seed) ^ splitmix64((uint64_t)epoch);
    for (uint64_t i = (uint64_t)n_views; i > 1; --i) {
        s = splitmix64(s);
        const uint64_t j = s % i;
        const int64_t t = order[i - 1];
        order[i - 1] = order[j];
        order[j] = t;
    }
    const int64_t r = order[slot % n_views];
    free(order);
    return r;
}

/* optimizer.cpp:84-87: radii_grad_sum += |d_radii| (raw, pre-Adam), count += 1 */
void orc_accumulate_radii_grads(int64_t n, const double* g, double* rgs, int64_t* rgc) {
    for (int64_t i = 0; i < n; ++i) {
        for (int k = 0; k < 4; ++k) rgs[4 * i + k] += fabs(g[11 * i + 7 + k]);
        rgc[i] += 1;
    }
}

/* adam_scalar_update, optimizer.hpp:39-46 */
static double adam_scalar_update(double* m, double* v, int64_t step_after, double g, double lr,
                                 double beta1, double beta2, double eps) {
    *m = beta1 * *m + (1.0 - beta1) * g;
    *v = beta2 * *v + (1.0 - beta2) * g * g;
    const double m_hat = *m / (1.0 - pow(beta1, (double)step_after));
    const double v_hat = *v / (1.0 - pow(beta2, (double)step_after));
    return lr * m_hat / (sqrt(v_hat) + eps);
}

/* Optimizer::apply_adam, optimizer.cpp:100-140 */
void orc_apply_adam(int64_t n, double* c, double* q, double* r, double* m, double* v,
                    int64_t* step, const double* grads, const orc_optim_config* cfg) {
    for (int64_t i = 0; i < n; ++i) {
        double g[11], lr[11], upd[11];
        double* mi = m + 11 * i;
        double* vi = v + 11 * i;
        for (int k = 0; k < 11; ++k) g[k] = grads[11 * i + k];
        if (cfg->single_radii) { /* :110-119 */
            g[7] = g[8] = g[7] + g[8];
            g[9] = g[10] = g[9] + g[10];
            mi[8] = mi[7];
            vi[8] = vi[7];
            mi[10] = mi[9];
            vi[10] = vi[9];
        }
        step[i] += 1;
        for (int k = 0; k < 3; ++k) lr[k] = cfg->lr_center;
        for (int k = 3; k < 7; ++k) lr[k] = cfg->lr_rotation;
        for (int k = 7; k < 11; ++k) lr[k] = cfg->lr_radii;
        for (int k = 0; k < 11; ++k)
            upd[k] = adam_scalar_update(&mi[k], &vi[k], step[i], g[k], lr[k], cfg->beta1, cfg->beta2,
                                        cfg->eps);
        for (int k = 0; k < 3; ++k) c[3 * i + k] -= upd[k];
        for (int k = 0; k < 4; ++k) q[4 * i + k] -= upd[3 + k];
        for (int k = 0; k < 4; ++k) r[4 * i + k] -= upd[7 + k];
        if (cfg->single_radii) { /* :133-136 */
            r[4 * i + 1] = r[4 * i];
            r[4 * i + 3] = r[4 * i + 2];
        }
        v4 qq = {{q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]}};
        qq = quat_normalized(qq);
        for (int k = 0; k < 4; ++k) q[4 * i + k] = qq.v[k];
        for (int k = 0; k < 4; ++k) r[4 * i + k] = dmax(r[4 * i + k], cfg->radii_floor);
    }
}

/* Optimizer::maybe_split, optimizer.cpp:142-202 */
int64_t orc_maybe_split(int64_t n, int64_t iteration, const orc_optim_config* cfg,
                        const double* c, const double* q, const double* r, const int64_t* ids,
                        const double* m, const double* v, const int64_t* step, const double* rgs,
                        const int64_t* rgc, int64_t* next_id, double* co, double* qo, double* ro,
                        int64_t* io, double* mo, double* vo, int64_t* so, int64_t* n_out) {
    if (!cfg->enable_split || cfg->split_interval <= 0) return -1;
    if (iteration == 0 || iteration % cfg->split_interval != 0) return -1;
    int64_t n_split = 0, o = 0;
    for (int64_t i = 0; i < n; ++i) {
        int axis = -1;
        if (rgc[i] != 0) {
            double mean[4];
            for (int k = 0; k < 4; ++k) mean[k] = rgs[4 * i + k] / (double)rgc[i];
            const double mean_x = 0.5 * (mean[0] + mean[1]);
            const double mean_y = 0.5 * (mean[2] + mean[3]);
            const int tx = mean_x > cfg->split_grad_threshold;
            const int ty = mean_y > cfg->split_grad_threshold;
            if (tx || ty) axis = (tx && (!ty || mean_x >= mean_y)) ? 0 : 1;
        }
        if (axis < 0) {
            memcpy(co + 3 * o, c + 3 * i, 3 * sizeof(double));
            memcpy(qo + 4 * o, q + 4 * i, 4 * sizeof(double));
            memcpy(ro + 4 * o, r + 4 * i, 4 * sizeof(double));
            io[o] = ids[i];
            memcpy(mo + 11 * o, m + 11 * i, 11 * sizeof(double));
            memcpy(vo + 11 * o, v + 11 * i, 11 * sizeof(double));
            so[o] = step[i];
            ++o;
            continue;
        }
        ++n_split;
        v4 qq = {{q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]}};
        const frame_t f = plane_frame(quat_normalized(qq));
        const v3 pc = V3(c[3 * i], c[3 * i + 1], c[3 * i + 2]);
        const v3 dir = axis == 0 ? f.vx : f.vy;
        const int ra = axis == 0 ? 0 : 2; /* radius index of the + side */
        const double ha = r[4 * i + ra] * 0.5, hb = r[4 * i + ra + 1] * 0.5;
        const v3 ca = add3(pc, mul3s(dir, ha)), cb = sub3(pc, mul3s(dir, hb));
        for (int child = 0; child < 2; ++child, ++o) {
            const v3 cc = child == 0 ? ca : cb;
            const double h = child == 0 ? ha : hb;
            memcpy(co + 3 * o, cc.v, 3 * sizeof(double));
            memcpy(qo + 4 * o, q + 4 * i, 4 * sizeof(double));
            memcpy(ro + 4 * o, r + 4 * i, 4 * sizeof(double));
            ro[4 * o + ra] = ro[4 * o + ra + 1] = h;
            io[o] = (*next_id)++;
            memset(mo + 11 * o, 0, 11 * sizeof(double));
            memset(vo + 11 * o, 0, 11 * sizeof(double));
            so[o] = 0;
        }
    }
    *n_out = o;
    return n_split;
}

/* ---------------------------------------------------------------- merge_planes */
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
static double dclamp(double v, double lo, double hi) { /* std::clamp */
    return v < lo ? lo : (hi < v ? hi : v);
}
/* rect_corners, geometry.cpp:64-70 */
static void rect_corners(v3 p, const double* r, frame_t f, v3 out[4]) {
    out[0] = add3(add3(p, scl3(r[0], f.vx)), scl3(r[2], f.vy));
    out[1] = add3(sub3(p, scl3(r[1], f.vx)), scl3(r[2], f.vy));
    out[2] = sub3(sub3(p, scl3(r[1], f.vx)), scl3(r[3], f.vy));
    out[3] = sub3(add3(p, scl3(r[0], f.vx)), scl3(r[3], f.vy));
}
/* point_rect_distance, geometry.cpp:74-80 */
static double point_rect_distance(v3 x, v3 c, const double* r, frame_t f) {
    const v3 e = sub3(x, c);
    const double px = dclamp(dot3(e, f.vx), -r[1], r[0]);
    const double py = dclamp(dot3(e, f.vy), -r[3], r[2]);
    const v3 closest = add3(add3(c, scl3(px, f.vx)), scl3(py, f.vy));
    return norm3(sub3(x, closest));
}
/* segment_segment_distance, geometry.cpp:82-111 (Ericson) */
static double segment_segment_distance(v3 p1, v3 q1, v3 p2, v3 q2) {
    const v3 d1 = sub3(q1, p1), d2 = sub3(q2, p2), r = sub3(p1, p2);
    const double a = dot3(d1, d1), e = dot3(d2, d2), f = dot3(d2, r);
    double s = 0, t = 0;
    const double eps = 1e-15;
    if (a <= eps && e <= eps) return norm3(r);
    if (a <= eps) {
        t = dclamp(f / e, 0.0, 1.0);
    } else {
        const double c = dot3(d1, r);
        if (e <= eps) {
            s = dclamp(-c / a, 0.0, 1.0);
        } else {
            const double b = dot3(d1, d2), denom = a * e - b * b;
            if (denom > eps) s = dclamp((b * f - c * e) / denom, 0.0, 1.0);
            t = (b * s + f) / e;
            if (t < 0) {
                t = 0;
                s = dclamp(-c / a, 0.0, 1.0);
            } else if (t > 1) {
                t = 1;
                s = dclamp((b - c) / a, 0.0, 1.0);
            }
        }
    }
    return norm3(sub3(add3(p1, scl3(s, d1)), add3(p2, scl3(t, d2))));
}
/* segment_crosses_rect, geometry.cpp:114-127 */
static int segment_crosses_rect(v3 a, v3 b, v3 c, const double* r, frame_t f) {
    const double ha = dot3(sub3(a, c), f.n);
    const double hb = dot3(sub3(b, c), f.n);
    if (ha * hb > 0) return 0;
    const double denom = ha - hb;
    if (fabs(denom) < 1e-15) return 0;
    const double s = ha / denom;
    const v3 x = add3(a, scl3(s, sub3(b, a)));
    const v3 e = sub3(x, c);
    const double px = dot3(e, f.vx), py = dot3(e, f.vy);
    return px >= -r[1] && px <= r[0] && py >= -r[3] && py <= r[2];
}
/* rect_distance, geometry.cpp:131-149 */
static double rect_distance(v3 ca_, const double* ra, frame_t fa, v3 cb_, const double* rb,
                            frame_t fb) {
    v3 ca[4], cb[4];
    rect_corners(ca_, ra, fa, ca);
    rect_corners(cb_, rb, fb, cb);
    double best = INFINITY;
    for (int i = 0; i < 4; ++i) {
        best = dmin(best, point_rect_distance(ca[i], cb_, rb, fb));
        best = dmin(best, point_rect_distance(cb[i], ca_, ra, fa));
    }
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j)
            best = dmin(best, segment_segment_distance(ca[i], ca[(i + 1) % 4], cb[j], cb[(j + 1) % 4]));
    for (int i = 0; i < 4; ++i) {
        if (segment_crosses_rect(ca[i], ca[(i + 1) % 4], cb_, rb, fb)) return 0.0;
        if (segment_crosses_rect(cb[i], cb[(i + 1) % 4], ca_, ra, fa)) return 0.0;
    }
    return best;
}

double orc_rect_distance(const double* ca, const double* qa, const double* ra, const double* cb,
                         const double* qb, const double* rb) {
    const v4 a = {{qa[0], qa[1], qa[2], qa[3]}}, b = {{qb[0], qb[1], qb[2], qb[3]}};
    return rect_distance(V3(ca[0], ca[1], ca[2]), ra, plane_frame(quat_normalized(a)),
                         V3(cb[0], cb[1], cb[2]), rb, plane_frame(quat_normalized(b)));
}

static int32_t uf_find(int32_t* parent, int32_t a) {
    while (parent[a] != a) a = parent[a] = parent[parent[a]];
    return a;
}

typedef struct {
    double area, offset, normal[3];
    int64_t min_id;
    int32_t root;
} orc_inst;

static int inst_cmp(const void* pa, const void* pb) { /* optimizer.cpp:292-296 */
    const orc_inst* a = (const orc_inst*)pa;
    const orc_inst* b = (const orc_inst*)pb;
    if (a->area != b->area) return a->area > b->area ? -1 : 1;
    return a->min_id < b->min_id ? -1 : (a->min_id > b->min_id ? 1 : 0);
}

/* merge_planes, optimizer.cpp:236-299. Writes instance_of[n] (index into the
 * sorted instance list) and per instance normal[3], offset, area; returns the
 * instance count. */
int64_t orc_merge_planes(int64_t n, const double* c, const double* q, const double* r,
                         const int64_t* ids, const double* scene_center, double normal_deg,
                         double merge_offset, double merge_adjacency, int use_adjacency,
                         int32_t* instance_of, double* inst_normal, double* inst_offset,
                         double* inst_area) {
    frame_t* fr = (frame_t*)malloc(sizeof(frame_t) * (size_t)(n ? n : 1));
    double* off = (double*)malloc(sizeof(double) * (size_t)(2 * n + 1));
    double* reach = off + n;
    int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    const v3 sc = V3(scene_center[0], scene_center[1], scene_center[2]);
    for (int64_t i = 0; i < n; ++i) {
        const v4 qq = {{q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]}};
        fr[i] = plane_frame(quat_normalized(qq));
        off[i] = fabs(dot3(sub3(V3(c[3 * i], c[3 * i + 1], c[3 * i + 2]), sc), fr[i].n));
        const double* ri = r + 4 * i;
        reach[i] = hypot(dmax(ri[0], ri[1]), dmax(ri[2], ri[3]));
        parent[i] = (int32_t)i;
    }
    const double cos_gate = cos(normal_deg * M_PI / 180.0);
    for (int64_t i = 0; i < n; ++i) {
        const v3 ci = V3(c[3 * i], c[3 * i + 1], c[3 * i + 2]);
        for (int64_t j = i + 1; j < n; ++j) {
            if (fabs(dot3(fr[i].n, fr[j].n)) <= cos_gate) continue;
            if (fabs(off[i] - off[j]) >= merge_offset) continue;
            if (use_adjacency) {
                const v3 cj = V3(c[3 * j], c[3 * j + 1], c[3 * j + 2]);
                const double gap = norm3(sub3(ci, cj)) - reach[i] - reach[j];
                if (gap >= merge_adjacency) continue;
                if (rect_distance(ci, r + 4 * i, fr[i], cj, r + 4 * j, fr[j]) >= merge_adjacency)
                    continue;
            }
            int32_t a = uf_find(parent, (int32_t)i), b = uf_find(parent, (int32_t)j);
            if (a != b) parent[a > b ? a : b] = a < b ? a : b;
        }
    }
    /* groups in root order, members ascending (optimizer.cpp:268-269) */
    orc_inst* inst = (orc_inst*)malloc(sizeof(orc_inst) * (size_t)(n ? n : 1));
    int32_t* root_of = parent; /* reuse after flattening */
    int32_t* slot = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) slot[i] = -1;
    for (int64_t i = 0; i < n; ++i) root_of[i] = uf_find(parent, (int32_t)i);
    int64_t k = 0;
    for (int64_t g = 0; g < n; ++g) {
        /* members of root g, ascending */
        int any = 0;
        int64_t largest = -1;
        double area = 0;
        int64_t min_id = 0;
        for (int64_t m = g; m < n; ++m) {
            if (root_of[m] != g) continue;
            const double* rm = r + 4 * m;
            const double am = (rm[0] + rm[1]) * (rm[2] + rm[3]);
            area += am;
            if (!any || ids[m] < min_id) min_id = ids[m];
            if (!any) largest = m;
            else {
                const double* rl = r + 4 * largest;
                if (am > (rl[0] + rl[1]) * (rl[2] + rl[3])) largest = m;
            }
            any = 1;
        }
        if (!any) continue;
        v3 nsum = V3(0, 0, 0);
        double osum = 0;
        for (int64_t m = g; m < n; ++m) {
            if (root_of[m] != g) continue;
            const double* rm = r + 4 * m;
            const double am = (rm[0] + rm[1]) * (rm[2] + rm[3]);
            const double sign = dot3(fr[m].n, fr[largest].n) < 0 ? -1.0 : 1.0;
            nsum = add3(nsum, scl3(am * sign, fr[m].n));
            osum += am * off[m];
        }
        orc_inst* I = &inst[k++];
        const v3 nn = norm3(nsum) > 1e-12 ? normalized3(nsum) : fr[largest].n;
        for (int t = 0; t < 3; ++t) I->normal[t] = nn.v[t];
        I->offset = osum / area;
        I->area = area;
        I->min_id = min_id;
        I->root = (int32_t)g;
    }
    qsort(inst, (size_t)k, sizeof(orc_inst), inst_cmp);
    for (int64_t t = 0; t < k; ++t) slot[inst[t].root] = (int32_t)t;
    for (int64_t i = 0; i < n; ++i) instance_of[i] = slot[root_of[i]];
    for (int64_t t = 0; t < k; ++t) {
        for (int u = 0; u < 3; ++u) inst_normal[3 * t + u] = inst[t].normal[u];
        inst_offset[t] = inst[t].offset;
        inst_area[t] = inst[t].area;
    }
    free(fr);
    free(off);
    free(parent);
    free(inst);
    free(slot);
    return k;
}

/* ---------------------------------------------------------------- scene_init.cpp */
/* quat_from_z_to, geometry.cpp:23-31: normalize(1 + e3.n, e3 x n) */
static v4 quat_from_z_to(v3 n) {
    const v3 e3 = V3(0.0, 0.0, 1.0);
    const double d = dot3(e3, n);
    if (1.0 + d < 1e-12) {
        v4 r = {{0.0, 1.0, 0.0, 0.0}};
        return r;
    }
    /* Vector3d::cross: (a.y b.z - a.z b.y, a.z b.x - a.x b.z, a.x b.y - a.y b.x) */
    const v3 c = V3(e3.v[1] * n.v[2] - e3.v[2] * n.v[1], e3.v[2] * n.v[0] - e3.v[0] * n.v[2],
                    e3.v[0] * n.v[1] - e3.v[1] * n.v[0]);
    v4 q = {{1.0 + d, c.v[0], c.v[1], c.v[2]}};
    return quat_normalized(q);
}

/* init_from_depth, scene_init.cpp:41-104 (stream_cloud + nearest neighbour).
 * Returns the primitive count, -1 for n_prims < 1, -2 without valid pixels. */
int64_t orc_init_from_depth(int n_views, const orc_camera* cams, const float* td, const float* tn,
                            int n_prims, uint64_t seed, double radius_scale, double* c, double* q,
                            double* r, int64_t* ids) {
    if (n_prims < 1) return -1;
    const size_t k = (size_t)n_prims;
    v3* pts = (v3*)malloc(sizeof(v3) * k);
    v3* nrm = (v3*)malloc(sizeof(v3) * k);
    size_t have = 0, total = 0;
    test_rng rng = rng_make(seed); /* Rng(seed): state = splitmix64(seed) */
    v3 lo = V3(INFINITY, INFINITY, INFINITY), hi = V3(-INFINITY, -INFINITY, -INFINITY);
    size_t off = 0;
    for (int vi = 0; vi < n_views; ++vi) {
        const orc_camera* cam = &cams[vi];
        m3 R;
        memcpy(R.m, cam->rot_wc, sizeof R.m);
        const v3 t = V3(cam->t_wc[0], cam->t_wc[1], cam->t_wc[2]);
        for (int v = 0; v < cam->height; ++v)
            for (int u = 0; u < cam->width; ++u) {
                const size_t px = off + (size_t)v * cam->width + u;
                const float* tnp = tn + 3 * px;
                if (!(td[px] > 0.0f) || (tnp[0] == 0.0f && tnp[1] == 0.0f && tnp[2] == 0.0f)) continue;
                const double z = td[px];
                const v3 pc = V3((u + 0.5 - cam->cx) / cam->fx * z, (v + 0.5 - cam->cy) / cam->fy * z, z);
                const v3 pw = add3(mv_stored(&R, pc), t);
                for (int a = 0; a < 3; ++a) { /* cwiseMin / cwiseMax */
                    lo.v[a] = (pw.v[a] < lo.v[a]) ? pw.v[a] : lo.v[a];
                    hi.v[a] = (hi.v[a] < pw.v[a]) ? pw.v[a] : hi.v[a];
                }
                const v3 nc = V3(tnp[0], tnp[1], tnp[2]);
                const v3 nw = normalized3(mv_stored(&R, nc));
                if (have < k) {
                    pts[have] = pw;
                    nrm[have] = nw;
                    ++have;
                } else {
                    const size_t j = (size_t)(rng_next(&rng) % (uint64_t)(total + 1));
                    if (j < k) {
                        pts[j] = pw;
                        nrm[j] = nw;
                    }
                }
                ++total;
            }
        off += (size_t)cam->width * cam->height;
    }
    if (have == 0) {
        free(pts);
        free(nrm);
        return -2;
    }
    const double diag = norm3(sub3(hi, lo));
    const double fallback = dmax(0.05 * diag, 10 * 1e-4); /* kRadiiFloor */
    for (size_t i = 0; i < have; ++i) {
        double nearest = INFINITY;
        for (size_t j = 0; j < have; ++j) {
            if (j == i) continue;
            nearest = dmin(nearest, norm3(sub3(pts[i], pts[j])));
        }
        const double radius = have > 1 ? dmax(radius_scale * nearest, 1e-4) : fallback;
        const v4 qq = quat_from_z_to(nrm[i]);
        for (int a = 0; a < 3; ++a) c[3 * i + a] = pts[i].v[a];
        for (int a = 0; a < 4; ++a) q[4 * i + a] = qq.v[a];
        for (int a = 0; a < 4; ++a) r[4 * i + a] = radius;
        ids[i] = (int64_t)i;
    }
    free(pts);
    free(nrm);
    return (int64_t)have;
}
