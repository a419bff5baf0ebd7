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

// ---- fp32 colour with an exact fallback (render.py:209-214)
// The per-step colour is evaluated in fp32: direction, basis and the 16-term
// sums, every operation explicitly rounded so color_kernel and the Adam colour
// epilogue produce the same bits.  Only the activation decision raw + 0.5 > 0
// must match the fp64 reference exactly: the fp32 value is within
// kColorTol * sum|c| of the fp64 one (direction components to ~5e-7, basis rows
// to ~6e-6 absolute, 16 fp32 fma roundings), so when |raw + 0.5| is inside that
// band the gaussian is recomputed with the fp64 path (view_dir, sh_basis16,
// color_quarter) and takes its value and decision from there.
constexpr float kColorTol = 3e-5f;

// normalize(mu - camera_center) in fp32 from the fp64 differences
__device__ __forceinline__ void dir_f32(double dx, double dy, double dz, float& x, float& y, float& z) {
    x = (float)dx;
    y = (float)dy;
    z = (float)dz;
    const float inv = rsqrtf(__fadd_rn(__fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y)), __fmul_rn(z, z)));
    x = __fmul_rn(x, inv);
    y = __fmul_rn(y, inv);
    z = __fmul_rn(z, inv);
}

// SH basis rows in fp32 with explicit rounding (rows above deg are 0)
__device__ __forceinline__ void basis16_rn(float x, float y, float z, int deg, float b[16]) {
    b[0] = 0.28209479177387814f;
#pragma unroll
    for (int i = 1; i < 16; ++i) b[i] = 0.f;
    if (deg < 1) return;
    b[1] = __fmul_rn(-0.4886025119029199f, y);
    b[2] = __fmul_rn(0.4886025119029199f, z);
    b[3] = __fmul_rn(-0.4886025119029199f, x);
    if (deg < 2) return;
    const float xx = __fmul_rn(x, x), yy = __fmul_rn(y, y), zz = __fmul_rn(z, z);
    const float xy = __fmul_rn(x, y), yz = __fmul_rn(y, z), xz = __fmul_rn(x, z);
    b[4] = __fmul_rn(1.0925484305920792f, xy);
    b[5] = __fmul_rn(-1.0925484305920792f, yz);
    b[6] = __fmul_rn(0.31539156525252005f, __fsub_rn(__fsub_rn(__fmul_rn(2.f, zz), xx), yy));
    b[7] = __fmul_rn(-1.0925484305920792f, xz);
    b[8] = __fmul_rn(0.5462742152960396f, __fsub_rn(xx, yy));
    if (deg < 3) return;
    b[9] = __fmul_rn(__fmul_rn(-0.5900435899266435f, y), __fsub_rn(__fmul_rn(3.f, xx), yy));
    b[10] = __fmul_rn(__fmul_rn(2.890611442640554f, xy), z);
    const float q4 = __fsub_rn(__fsub_rn(__fmul_rn(4.f, zz), xx), yy);
    b[11] = __fmul_rn(__fmul_rn(-0.4570457994644658f, y), q4);
    b[12] = __fmul_rn(__fmul_rn(0.3731763325901154f, z),
                      __fsub_rn(__fsub_rn(__fmul_rn(2.f, zz), __fmul_rn(3.f, xx)), __fmul_rn(3.f, yy)));
    b[13] = __fmul_rn(__fmul_rn(-0.4570457994644658f, x), q4);
    b[14] = __fmul_rn(__fmul_rn(1.445305721320277f, z), __fsub_rn(xx, yy));
    b[15] = __fmul_rn(__fmul_rn(-0.5900435899266435f, x), __fsub_rn(xx, __fmul_rn(3.f, yy)));
}

// One quarter (rows 4 part .. 4 part + 3) of the fp32 colour sums and of the
// coefficient magnitudes sum|c| that scale the fallback band
__device__ __forceinline__ void color_quarter_f32(const float b[16], const float c12[12], int part, float out[3],
                                                  float mag[3]) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        float acc = 0.f, m = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float bq = part == 0 ? b[q] : (part == 1 ? b[4 + q] : (part == 2 ? b[8 + q] : b[12 + q]));
            acc = __fmaf_rn(bq, c12[3 * q + ch], acc);
            m = __fadd_rn(m, fabsf(c12[3 * q + ch]));
        }
        out[ch] = acc;
        mag[ch] = m;
    }
}

__device__ __forceinline__ float color_combine_f32(float q0, float q1, float q2, float q3) {
    return __fadd_rn(__fadd_rn(__fadd_rn(q0, q1), q2), q3);
}

// Is channel value v = raw + 0.5 too close to 0 for the fp32 decision?
__device__ __forceinline__ bool color_ambiguous(float v, float mag) {
    return !(fabsf(v) > __fmaf_rn(kColorTol, mag, 1e-30f));
}

// fp64 colour of one gaussian (out of line: the rare fallback of color_kernel)
static __device__ __noinline__ float4 color_f64(const double* __restrict__ pos, const float4* __restrict__ sh, int64_t g,
                                         Center cen, int deg) {
    double x, y, z;
    view_dir(pos, g, cen.c, x, y, z);
    double b[16];
    sh_basis16<double>(x, y, z, deg, b);
    const float4* row = sh + g * 12;
    double qv[4][3];
#pragma unroll
    for (int part = 0; part < 4; ++part) {  // 12 coefficients at a time (registers)
        float c12[12];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const float4 f = __ldcg(row + 3 * part + i);
            c12[4 * i] = f.x;
            c12[4 * i + 1] = f.y;
            c12[4 * i + 2] = f.z;
            c12[4 * i + 3] = f.w;
        }
        color_quarter(b, c12, part, qv[part]);
    }
    int act = 0;
    float col[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const double v = color_combine(qv[0][ch], qv[1][ch], qv[2][ch], qv[3][ch]) + 0.5;
        act |= (v > 0.0) << ch;
        col[ch] = (float)fmax(0.0, v);
    }
    return make_float4(col[0], col[1], col[2], __int_as_float(act));
}

}  // namespace rcgs
