// TEST INFRASTRUCTURE ONLY — extern "C" access to the reference's dataset I/O.
//
// The reference's dataio.cpp (/root/reference/proj/core/src/dataio.cpp) is compiled
// in place into oracle/_ref/libpsplat_ref.so against the test-only json_shim /
// png_shim headers (nlohmann/json and libpng are not installed here). These
// wrappers let tests/test_dataio.py (CPU) and tests/test_gpu_parity.py (GPU) have
// the reference write datasets and maps and read the repo's, so the device loader
// (psg_load_dataset, psg_dataset_*) is pinned on files the reference itself wrote:
//   write_map_f32 / read_map_f32   dataio.cpp:65-97
//   load_dataset (+validate_view)  dataio.cpp:120-201
//   write_dataset                  dataio.cpp:203-254
// Face rows use the 15-double layout of ref_room_faces (ref_harness.cpp):
// center[3], u_axis[3], v_axis[3], half_u, half_v, normal[3], instance_id.
#include "psplat/dataio.hpp"

#include <cstring>
#include <exception>
#include <string>

#include "oracle_api.h"

using namespace psplat;

namespace {

int report(const std::exception& e, char* err, int errlen) {
    if (err && errlen > 0) {
        std::strncpy(err, e.what(), std::size_t(errlen - 1));
        err[errlen - 1] = '\0';
    }
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    return 3;  // std::runtime_error and everything else
}

void pack_face(const GtFace& f, double* o) {
    for (int k = 0; k < 3; ++k) {
        o[k] = f.center[k];
        o[3 + k] = f.u_axis[k];
        o[6 + k] = f.v_axis[k];
        o[11 + k] = f.normal[k];
    }
    o[9] = f.half_u;
    o[10] = f.half_v;
    o[14] = double(f.instance_id);
}

}  // namespace

extern "C" {

int ref_write_map_f32(const char* path, int width, int height, int channels, const float* data, char* err,
                      int errlen) {
    try {
        write_map_f32(path, width, height, channels, data);
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

// Returns 0 and fills w/h (and data when cap is large enough), or the error class.
int ref_read_map_f32(const char* path, int channels, int* width, int* height, float* data, int64_t cap,
                     char* err, int errlen) {
    try {
        const MapF32 m = read_map_f32(path, channels);
        *width = m.width;
        *height = m.height;
        if (data && cap >= int64_t(m.data.size())) std::memcpy(data, m.data.data(), m.data.size() * 4);
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

// write_dataset with CameraView ids ids[i], targets concatenated in view order.
int ref_write_dataset(const char* root, int n, const orc_camera* cams, const int* ids, const float* td,
                      const float* tn, const double* scene_center, const char* units, int n_faces,
                      const double* faces, char* err, int errlen) {
    try {
        std::vector<CameraView> views(static_cast<std::size_t>(n));
        std::size_t off = 0;
        for (int i = 0; i < n; ++i) {
            CameraView& v = views[std::size_t(i)];
            const orc_camera& c = cams[i];
            v.id = ids[i];
            v.fx = c.fx;
            v.fy = c.fy;
            v.cx = c.cx;
            v.cy = c.cy;
            v.width = c.width;
            v.height = c.height;
            for (int r = 0; r < 3; ++r)
                for (int k = 0; k < 3; ++k) v.rot_wc(r, k) = c.rot_wc[3 * r + k];
            for (int k = 0; k < 3; ++k) v.t_wc[k] = c.t_wc[k];
            const std::size_t np = v.pixel_count();
            v.target_depth.assign(td + off, td + off + np);
            v.target_normal.assign(tn + 3 * off, tn + 3 * (off + np));
            off += np;
        }
        SceneMeta meta;
        meta.scene_center = Vec3(scene_center[0], scene_center[1], scene_center[2]);
        meta.units = units;
        for (int f = 0; f < n_faces; ++f) {
            const double* o = faces + 15 * f;
            GtFace g;
            g.center = Vec3(o[0], o[1], o[2]);
            g.u_axis = Vec3(o[3], o[4], o[5]);
            g.v_axis = Vec3(o[6], o[7], o[8]);
            g.half_u = o[9];
            g.half_v = o[10];
            g.normal = Vec3(o[11], o[12], o[13]);
            g.instance_id = std::uint32_t(o[14]);
            meta.gt_faces.push_back(g);
        }
        write_dataset(root, views, meta);
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

// load_dataset(root, stride). Call with null outputs to get the sizes
// (*n_views, *n_pixels, *n_faces); then with buffers of those sizes.
int ref_load_dataset(const char* root, int stride, int* n_views, int64_t* n_pixels, int* n_faces,
                     orc_camera* cams, int* ids, float* td, float* tn, double* scene_center, char* units,
                     int units_len, int* has_meta, double* faces, char* err, int errlen) {
    try {
        const Dataset ds = load_dataset(root, stride);
        *n_views = int(ds.views.size());
        int64_t np = 0;
        for (const CameraView& v : ds.views) np += int64_t(v.pixel_count());
        *n_pixels = np;
        *n_faces = int(ds.meta.gt_faces.size());
        if (!cams) return 0;
        std::size_t off = 0;
        for (std::size_t i = 0; i < ds.views.size(); ++i) {
            const CameraView& v = ds.views[i];
            orc_camera& c = cams[i];
            ids[i] = v.id;
            c.fx = v.fx;
            c.fy = v.fy;
            c.cx = v.cx;
            c.cy = v.cy;
            c.width = v.width;
            c.height = v.height;
            for (int r = 0; r < 3; ++r)
                for (int k = 0; k < 3; ++k) c.rot_wc[3 * r + k] = v.rot_wc(r, k);
            for (int k = 0; k < 3; ++k) c.t_wc[k] = v.t_wc[k];
            std::memcpy(td + off, v.target_depth.data(), v.pixel_count() * 4);
            std::memcpy(tn + 3 * off, v.target_normal.data(), v.pixel_count() * 12);
            off += v.pixel_count();
        }
        for (int k = 0; k < 3; ++k) scene_center[k] = ds.meta.scene_center[k];
        std::strncpy(units, ds.meta.units.c_str(), std::size_t(units_len - 1));
        units[units_len - 1] = '\0';
        *has_meta = ds.has_meta ? 1 : 0;
        for (std::size_t f = 0; f < ds.meta.gt_faces.size(); ++f) pack_face(ds.meta.gt_faces[f], faces + 15 * f);
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

}  // extern "C"
