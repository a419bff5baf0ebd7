// K8 selection pass: cloud -> per-view mask (selection.py:184-235) and the
// recolour of the masked ground truth (recolor.py:30-39).
//
// Point projection is fp64 with the reference's exact arithmetic: the
// world->camera FMA chain numpy/OpenBLAS uses for `points @ R.T + t`,
// u = fx * x / z + cx unfused, round-half-even (np.rint), and the occlusion test
// z <= depth * (1 + tol).  Quad stamping writes 1-bytes (idempotent), so the
// mask is bit-exact and independent of thread order.
#include <math.h>

#include "common.cuh"

namespace rcgs {

__global__ void project_cloud_kernel(const double* __restrict__ pts, int64_t m, rcgs_camera cam,
                                     const double* __restrict__ depth, int quad, double one_plus_tol,
                                     uint8_t* __restrict__ mask) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double p0 = pts[3 * i], p1 = pts[3 * i + 1], p2 = pts[3 * i + 2];
    const double x = cam_coord(cam.R, cam.t, 0, p0, p1, p2);
    const double y = cam_coord(cam.R, cam.t, 1, p0, p1, p2);
    const double z = cam_coord(cam.R, cam.t, 2, p0, p1, p2);
    if (!(z > 0.0)) return;
    const double u = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fx, x), z), cam.cx);
    const double v = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fy, y), z), cam.cy);
    if (!(fabs(u) < 1e15 && fabs(v) < 1e15)) return;
    const int64_t pu = (int64_t)rint(u), pv = (int64_t)rint(v);
    if (pu < 0 || pu >= cam.width || pv < 0 || pv >= cam.height) return;
    if (!(z <= __dmul_rn(depth[pv * cam.width + pu], one_plus_tol))) return;
    const int half = (quad - 1) / 2;
    for (int dv = -half; dv < quad - half; ++dv) {
        const int64_t qv = pv + dv;
        if (qv < 0 || qv >= cam.height) continue;
        for (int du = -half; du < quad - half; ++du) {
            const int64_t qu = pu + du;
            if (qu < 0 || qu >= cam.width) continue;
            mask[qv * cam.width + qu] = 1;
        }
    }
}

template <typename T>
__global__ void recolor_kernel(const T* __restrict__ img, const uint8_t* __restrict__ mask,
                               int64_t npix, T t0, T t1, T t2, T* __restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npix) return;
    T a = img[3 * p], b = img[3 * p + 1], c = img[3 * p + 2];
    if (mask[p]) {  // np.clip(x * t, 0, 1) == min(max(x * t, 0), 1)
        a = fmin(fmax(a * t0, T(0)), T(1));
        b = fmin(fmax(b * t1, T(0)), T(1));
        c = fmin(fmax(c * t2, T(0)), T(1));
    }
    out[3 * p] = a;
    out[3 * p + 1] = b;
    out[3 * p + 2] = c;
}

}  // namespace rcgs

using namespace rcgs;

extern "C" int rcgs_project_cloud(const double* d_points, int64_t m, const rcgs_camera* cam,
                                  const double* d_depth, int32_t quad, double tol, uint8_t* d_mask,
                                  void* stream) {
    RCGS_CHECK_ARG(cam && d_depth && d_mask, "null argument");
    RCGS_CHECK_ARG(quad >= 1, "quad_size must be >= 1");
    RCGS_CHECK_ARG(m >= 0, "negative point count");
    if (m == 0) return RCGS_OK;
    RCGS_CHECK_ARG(d_points != nullptr, "null points");
    const double one_plus_tol = 1.0 + tol;
    project_cloud_kernel<<<div_up(m, 256), 256, 0, as_stream(stream)>>>(d_points, m, *cam, d_depth, quad,
                                                                          one_plus_tol, d_mask);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_apply_recolor(const float* d_image, const uint8_t* d_mask, int64_t npix,
                                  const float* h_tint3, float* d_out, void* stream) {
    RCGS_CHECK_ARG(d_image && d_mask && h_tint3 && d_out, "null argument");
    for (int i = 0; i < 3; ++i)
        RCGS_CHECK_ARG(isfinite(h_tint3[i]) && h_tint3[i] >= 0.f, "tint components must be finite and >= 0");
    if (npix <= 0) return RCGS_OK;
    recolor_kernel<float><<<div_up(npix, 256), 256, 0, as_stream(stream)>>>(d_image, d_mask, npix, h_tint3[0],
                                                                      h_tint3[1], h_tint3[2], d_out);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_apply_recolor_f64(const double* d_image, const uint8_t* d_mask, int64_t npix,
                                      const double* h_tint3, double* d_out, void* stream) {
    RCGS_CHECK_ARG(d_image && d_mask && h_tint3 && d_out, "null argument");
    for (int i = 0; i < 3; ++i)
        RCGS_CHECK_ARG(isfinite(h_tint3[i]) && h_tint3[i] >= 0.0, "tint components must be finite and >= 0");
    if (npix <= 0) return RCGS_OK;
    recolor_kernel<double><<<div_up(npix, 256), 256, 0, as_stream(stream)>>>(d_image, d_mask, npix, h_tint3[0],
                                                                              h_tint3[1], h_tint3[2], d_out);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}
