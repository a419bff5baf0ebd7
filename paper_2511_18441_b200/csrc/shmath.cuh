// Spherical-harmonics helpers shared by the colour and gradient kernels
// (render.py:103-148, 209-214; backward.py:36-40).
#pragma once
#include "common.cuh"

namespace rcgs {

template <typename T>
__device__ __forceinline__ void sh_basis16(T x, T y, T z, int deg, T* b) {
    b[0] = T(0.28209479177387814);
#pragma unroll
    for (int i = 1; i < 16; ++i) b[i] = T(0);
    if (deg < 1) return;
    b[1] = T(-0.4886025119029199) * y;
    b[2] = T(0.4886025119029199) * z;
    b[3] = T(-0.4886025119029199) * x;
    if (deg < 2) return;
    const T xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    b[4] = T(1.0925484305920792) * xy;
    b[5] = T(-1.0925484305920792) * yz;
    b[6] = T(0.31539156525252005) * (T(2) * zz - xx - yy);
    b[7] = T(-1.0925484305920792) * xz;
    b[8] = T(0.5462742152960396) * (xx - yy);
    if (deg < 3) return;
    b[9] = T(-0.5900435899266435) * y * (T(3) * xx - yy);
    b[10] = T(2.890611442640554) * xy * z;
    b[11] = T(-0.4570457994644658) * y * (T(4) * zz - xx - yy);
    b[12] = T(0.3731763325901154) * z * (T(2) * zz - T(3) * xx - T(3) * yy);
    b[13] = T(-0.4570457994644658) * x * (T(4) * zz - xx - yy);
    b[14] = T(1.445305721320277) * z * (xx - yy);
    b[15] = T(-0.5900435899266435) * x * (xx - T(3) * yy);
}

// One SH basis row (0 beyond the degree, or k > 15) without a local array.
__device__ __forceinline__ float sh_row(int k, float x, float y, float z, int deg) {
    if (k > 15 || (k >= 1 && deg < 1) || (k >= 4 && deg < 2) || (k >= 9 && deg < 3)) return 0.f;
    switch (k) {
        case 0: return 0.28209479177387814f;
        case 1: return -0.4886025119029199f * y;
        case 2: return 0.4886025119029199f * z;
        case 3: return -0.4886025119029199f * x;
        case 4: return 1.0925484305920792f * (x * y);
        case 5: return -1.0925484305920792f * (y * z);
        case 6: return 0.31539156525252005f * (2.f * z * z - x * x - y * y);
        case 7: return -1.0925484305920792f * (x * z);
        case 8: return 0.5462742152960396f * (x * x - y * y);
        case 9: return -0.5900435899266435f * y * (3.f * x * x - y * y);
        case 10: return 2.890611442640554f * (x * y) * z;
        case 11: return -0.4570457994644658f * y * (4.f * z * z - x * x - y * y);
        case 12: return 0.3731763325901154f * z * (2.f * z * z - 3.f * x * x - 3.f * y * y);
        case 13: return -0.4570457994644658f * x * (4.f * z * z - x * x - y * y);
        case 14: return 1.445305721320277f * z * (x * x - y * y);
        default: return -0.5900435899266435f * x * (x * x - 3.f * y * y);
    }
}

struct Center {
    double c[3];
};

// -R^T t (scene.py:72-75)
inline Center camera_center(const rcgs_camera& cam) {
    Center c;
    for (int j = 0; j < 3; ++j)
        c.c[j] = -(cam.R[0 * 3 + j] * cam.t[0] + cam.R[1 * 3 + j] * cam.t[1] + cam.R[2 * 3 + j] * cam.t[2]);
    return c;
}

// normalize(mu - camera_center) in fp64 (render.py:209-210)
__device__ __forceinline__ void view_dir(const double* __restrict__ pos, int64_t g, const double* c,
                                         double& x, double& y, double& z) {
    x = pos[3 * g] - c[0];
    y = pos[3 * g + 1] - c[1];
    z = pos[3 * g + 2] - c[2];
    const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
    x = x / nrm;
    y = y / nrm;
    z = z / nrm;
}

// Colour of one channel-triplet quarter: basis rows 4 part .. 4 part + 3 against
// this quarter's 12 coefficients (coefficient 12 part + e is row 4 part + e / 3,
// channel e % 3), an fp64 fma chain per channel from 0.  The full colour is
// ((q0 + q1) + q2) + q3 over the quarters -- the order color_kernel and the Adam
// colour epilogue share, so both produce identical bits.
__device__ __forceinline__ void color_quarter(const double b[16], const float c12[12], int part, double out[3]) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double bq = part == 0 ? b[q] : (part == 1 ? b[4 + q] : (part == 2 ? b[8 + q] : b[12 + q]));
            acc = fma(bq, (double)c12[3 * q + ch], acc);
        }
        out[ch] = acc;
    }
}

__device__ __forceinline__ double color_combine(double q0, double q1, double q2, double q3) {
    return __dadd_rn(__dadd_rn(__dadd_rn(q0, q1), q2), q3);
}

}  // namespace rcgs
