// PSMP dataset loader: the reference's on-disk format
// (dataio.hpp:12-14, dataio.cpp:19-201) read straight into page-locked staging
// buffers by a pool of reader threads and streamed into the context's resident
// targets, overlapping file reads with host-to-device copies.
//
//   cameras.txt            "id fx fy cx cy width height m00 .. m33" per line
//                          (m = [rot_wc | t_wc] row-major 4x4), '#' comments
//   depth/<id>.f32         PSMP map, 1 channel f32, <= 0 invalid
//   normal/<id>.f32        PSMP map, 3 channels f32 (camera frame), 0-vector invalid
//   PSMP map               "PSMP", u32 version 1, u32 W, u32 H (little endian),
//                          then the row-major channel-interleaved payload
//
// Validation and messages follow load_dataset / read_map_f32 / validate_view:
// std::runtime_error cases return PSG_EIO ("<path>: <what>"), the stride check
// PSG_EINVAL. meta.json (scene centre, GT faces) is left to the host language.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/psplat_b200.h"

namespace psg {
int set_error(int status, const std::string& msg);  // psg_api.cu
}

struct psg_dataset {
    std::string root;
    std::vector<psg_camera> cams;
    std::vector<int32_t> ids;
    std::vector<long long> pix_off;  // prefix of W*H
    long long total_px = 0;
};

namespace {

constexpr char kMagic[4] = {'P', 'S', 'M', 'P'};
constexpr uint32_t kVersion = 1;

int io_fail(const std::string& path, const std::string& what) {
    return psg::set_error(PSG_EIO, path + ": " + what);
}

// read_map_header + payload checks (dataio.cpp:49-59, 84-97)
int read_map(const std::string& path, int channels, int* w, int* h, float* out, long long cap) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return io_fail(path, "cannot open");
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    unsigned char hdr[16];
    const size_t got = std::fread(hdr, 1, 16, f);
    if (got < 4 || std::memcmp(hdr, kMagic, 4) != 0) return io_fail(path, "bad map magic");
    if (got < 16) return io_fail(path, "unsupported map version");
    uint32_t ver, W, H;
    std::memcpy(&ver, hdr + 4, 4);
    std::memcpy(&W, hdr + 8, 4);
    std::memcpy(&H, hdr + 12, 4);
    if (ver != kVersion) return io_fail(path, "unsupported map version");
    if (int(W) <= 0 || int(H) <= 0) return io_fail(path, "bad map dimensions");
    const long long count = (long long)W * H * channels;
    if (std::fseek(f, 0, SEEK_END) != 0) return io_fail(path, "cannot seek");
    const long long size = std::ftell(f);
    if (size - 16 != count * 4) return io_fail(path, "payload length does not match header");
    *w = int(W);
    *h = int(H);
    if (!out) return PSG_OK;
    if (count > cap) return psg::set_error(PSG_EINVAL, path + ": buffer too small");
    std::fseek(f, 16, SEEK_SET);
    if (std::fread(out, 4, size_t(count), f) != size_t(count)) return io_fail(path, "truncated payload");
    return PSG_OK;
}

std::string view_path(const std::string& root, const char* dir, int id) {
    return root + "/" + dir + "/" + std::to_string(id) + ".f32";
}

// validate_view (dataio.cpp:107-121): orthonormal pose, unit valid normals
int validate(const psg_dataset* ds, int k, const float* tn, const std::string& root) {
    const psg_camera& c = ds->cams[size_t(k)];
    double worst = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int r = 0; r < 3; ++r) s += c.rot_wc[3 * r + i] * c.rot_wc[3 * r + j];
            worst = std::max(worst, std::fabs(s - (i == j ? 1.0 : 0.0)));
        }
    const std::string vid = "view " + std::to_string(ds->ids[size_t(k)]);
    if (worst > 1e-6) return io_fail(root, vid + ": pose rotation not orthonormal");
    const long long np = (long long)c.width * c.height;
    for (long long px = 0; px < np; ++px) {
        const float x = tn[3 * px], y = tn[3 * px + 1], z = tn[3 * px + 2];
        if (x == 0.0f && y == 0.0f && z == 0.0f) continue;
        const double n = std::sqrt(double(x) * x + double(y) * y + double(z) * z);
        if (n < 1.0 - 1e-4 || n > 1.0 + 1e-4) return io_fail(root, vid + ": non-unit target normal");
    }
    return PSG_OK;
}

int read_view(const psg_dataset* ds, int k, float* td, float* tn) {
    const psg_camera& c = ds->cams[size_t(k)];
    const int id = ds->ids[size_t(k)];
    const long long np = (long long)c.width * c.height;
    int w = 0, h = 0, rc;
    const std::string dp = view_path(ds->root, "depth", id), nptn = view_path(ds->root, "normal", id);
    if ((rc = read_map(dp, 1, &w, &h, td, np))) return rc;
    if (w != c.width || h != c.height) return io_fail(dp, "resolution differs from cameras.txt");
    if ((rc = read_map(nptn, 3, &w, &h, tn, 3 * np))) return rc;
    if (w != c.width || h != c.height) return io_fail(nptn, "resolution differs from cameras.txt");
    return validate(ds, k, tn, ds->root);
}

}  // namespace

namespace {
struct NvtxRange {  // one NVTX range per call, for the tools
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

extern "C" {

int psg_dataset_open(const char* root, int stride, psg_dataset** out) {
    if (!root || !out) return psg::set_error(PSG_EINVAL, "dataset_open: null argument");
    *out = nullptr;
    if (stride < 1) return psg::set_error(PSG_EINVAL, "load_dataset: stride must be >= 1");
    const std::string cams = std::string(root) + "/cameras.txt";
    std::ifstream in(cams);
    if (!in) return io_fail(cams, "cannot open");
    psg_dataset* ds = new psg_dataset();
    ds->root = root;
    std::string line;
    int line_index = 0;
    while (std::getline(in, line)) {  // dataio.cpp:143-170
        if (line.empty() || line[0] == '#') continue;
        const int idx = line_index++;
        if (idx % stride != 0) continue;
        std::istringstream ls(line);
        psg_camera c{};
        int id = 0;
        double m[16];
        ls >> id >> c.fx >> c.fy >> c.cx >> c.cy >> c.width >> c.height;
        for (double& x : m) ls >> x;
        if (!ls) {
            delete ds;
            return io_fail(cams, "malformed camera line: " + line);
        }
        for (int r = 0; r < 3; ++r)
            for (int cc = 0; cc < 3; ++cc) c.rot_wc[3 * r + cc] = m[4 * r + cc];
        c.t_wc[0] = m[3];
        c.t_wc[1] = m[7];
        c.t_wc[2] = m[11];
        if (c.width < 1 || c.height < 1) {
            delete ds;
            return io_fail(cams, "malformed camera line: " + line);
        }
        ds->pix_off.push_back(ds->total_px);
        ds->total_px += (long long)c.width * c.height;
        ds->cams.push_back(c);
        ds->ids.push_back(id);
    }
    if (ds->cams.empty()) {
        delete ds;
        return io_fail(cams, "no cameras loaded");
    }
    // headers of every map up front: a missing or malformed file fails the open
    for (size_t k = 0; k < ds->cams.size(); ++k) {
        int w = 0, h = 0, rc;
        const std::string dp = view_path(ds->root, "depth", ds->ids[k]);
        const std::string np = view_path(ds->root, "normal", ds->ids[k]);
        if ((rc = read_map(dp, 1, &w, &h, nullptr, 0)) ||
            ((w != ds->cams[k].width || h != ds->cams[k].height) &&
             (rc = io_fail(dp, "resolution differs from cameras.txt"))) ||
            (rc = read_map(np, 3, &w, &h, nullptr, 0)) ||
            ((w != ds->cams[k].width || h != ds->cams[k].height) &&
             (rc = io_fail(np, "resolution differs from cameras.txt")))) {
            delete ds;
            return rc;
        }
    }
    *out = ds;
    return PSG_OK;
}

int psg_dataset_close(psg_dataset* ds) {
    delete ds;
    return PSG_OK;
}

int psg_dataset_size(const psg_dataset* ds, int* n_views, int64_t* n_pixels) {
    if (!ds) return psg::set_error(PSG_EINVAL, "dataset: null handle");
    if (n_views) *n_views = int(ds->cams.size());
    if (n_pixels) *n_pixels = ds->total_px;
    return PSG_OK;
}

int psg_dataset_cameras(const psg_dataset* ds, psg_camera* cams, int32_t* ids) {
    if (!ds) return psg::set_error(PSG_EINVAL, "dataset: null handle");
    if (cams) std::memcpy(cams, ds->cams.data(), ds->cams.size() * sizeof(psg_camera));
    if (ids) std::memcpy(ids, ds->ids.data(), ds->ids.size() * sizeof(int32_t));
    return PSG_OK;
}

int psg_dataset_read(const psg_dataset* ds, int first, int count, float* td, float* tn, int threads) {
    if (!ds) return psg::set_error(PSG_EINVAL, "dataset: null handle");
    if (first < 0 || count < 0 || first + count > int(ds->cams.size()) || (count > 0 && (!td || !tn)))
        return psg::set_error(PSG_EINVAL, "dataset_read: bad range");
    if (count == 0) return PSG_OK;
    if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
    threads = std::min(threads, count);
    const long long base = ds->pix_off[size_t(first)];
    std::atomic<int> next{0};
    std::vector<int> rcs(static_cast<size_t>(threads), PSG_OK);
    std::vector<std::string> errs(static_cast<size_t>(threads));
    auto work = [&](int w) {
        for (;;) {
            const int j = next.fetch_add(1);
            if (j >= count) return;
            const int k = first + j;
            const long long o = ds->pix_off[size_t(k)] - base;
            const int rc = read_view(ds, k, td + o, tn + 3 * o);
            if (rc) {
                rcs[size_t(w)] = rc;
                errs[size_t(w)] = psg_last_error();
                next.store(count);
                return;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < threads; ++w) pool.emplace_back(work, w);
    work(0);
    for (auto& t : pool) t.join();
    for (int w = 0; w < threads; ++w)
        if (rcs[size_t(w)]) return psg::set_error(rcs[size_t(w)], errs[size_t(w)]);
    return PSG_OK;
}

int psg_load_dataset(psg_context* ctx, const psg_dataset* ds, int chunk_views, int threads) {
    NvtxRange nvtx_range("psg.load_dataset");
    if (!ctx || !ds) return psg::set_error(PSG_EINVAL, "load_dataset: null argument");
    int rc;
    const int nv = int(ds->cams.size());
    if ((rc = psg_set_views(ctx, nv, ds->cams.data(), nullptr, nullptr))) return rc;
    if (chunk_views <= 0) chunk_views = 64;
    long long max_px = 0;  // pixels of the largest chunk
    for (int c0 = 0; c0 < nv; c0 += chunk_views) {
        const int c1 = std::min(nv, c0 + chunk_views);
        const long long e = c1 < nv ? ds->pix_off[size_t(c1)] : ds->total_px;
        max_px = std::max(max_px, e - ds->pix_off[size_t(c0)]);
    }
    // two page-locked staging buffers: the reader threads fill one while the
    // other's host-to-device copy runs on the context stream
    cudaStream_t s = static_cast<cudaStream_t>(psg_get_stream(ctx));
    float* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; ++b) {
        stage[b] = static_cast<float*>(psg_host_alloc(size_t(max_px) * 16));
        if (!stage[b] || cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming) != cudaSuccess) {
            for (int q = 0; q < 2; ++q) {
                if (stage[q]) psg_host_free(stage[q]);
                if (done[q]) cudaEventDestroy(done[q]);
            }
            return psg::set_error(PSG_ENOMEM, "load_dataset: pinned staging allocation failed");
        }
    }
    rc = PSG_OK;
    for (int c0 = 0, b = 0; c0 < nv && rc == PSG_OK; c0 += chunk_views, b ^= 1) {
        const int cnt = std::min(chunk_views, nv - c0);
        cudaEventSynchronize(done[b]);  // the copy that last used this buffer
        const long long e = c0 + cnt < nv ? ds->pix_off[size_t(c0 + cnt)] : ds->total_px;
        const long long px = e - ds->pix_off[size_t(c0)];
        float* td = stage[b];
        float* tn = stage[b] + px;
        if ((rc = psg_dataset_read(ds, c0, cnt, td, tn, threads))) break;
        if ((rc = psg_update_targets(ctx, c0, cnt, td, tn))) break;
        if (cudaEventRecord(done[b], s) != cudaSuccess) rc = psg::set_error(PSG_ECUDA, "load_dataset: event");
    }
    cudaStreamSynchronize(s);
    for (int b = 0; b < 2; ++b) {
        psg_host_free(stage[b]);
        cudaEventDestroy(done[b]);
    }
    if (rc) return rc;
    return psg_refresh_target_counts(ctx);
}

int psg_write_map_f32(const char* path, int width, int height, int channels, const float* data) {
    if (!path || !data || width <= 0 || height <= 0 || channels <= 0)
        return psg::set_error(PSG_EINVAL, "write_map_f32: bad arguments");
    FILE* f = std::fopen(path, "wb");
    if (!f) return io_fail(path, "cannot open for writing");
    const uint32_t hdr[3] = {kVersion, uint32_t(width), uint32_t(height)};
    const size_t n = size_t(width) * size_t(height) * size_t(channels);
    const bool ok = std::fwrite(kMagic, 1, 4, f) == 4 && std::fwrite(hdr, 4, 3, f) == 3 &&
                    std::fwrite(data, 4, n, f) == n;
    std::fclose(f);
    return ok ? PSG_OK : io_fail(path, "write failed");
}

int psg_read_map_f32(const char* path, int expected_channels, int* width, int* height, float* data,
                     int64_t cap) {
    if (!path || expected_channels <= 0) return psg::set_error(PSG_EINVAL, "read_map_f32: bad arguments");
    int w = 0, h = 0;
    const int rc = read_map(path, expected_channels, &w, &h, data, data ? cap : 0);
    if (width) *width = w;
    if (height) *height = h;
    return rc;
}

}  // extern "C"
