// Scene checkpoint decode on the GPU (scene_io.py:108-153):
// the raw float32 vertex rows of a 3DGS PLY, uploaded as they are, become the
// device scene's fp64 positions and normalised rotations and the optimizer's
// (N, 16, 3) fp32 SH -- no host float64 materialisation or channel-major
// transposes.  Values match the reference loader exactly: float32 -> float64 is
// exact, the quaternion norm is numpy's sqrt(((r0^2 + r1^2) + r2^2) + r3^2) with a
// correctly rounded sqrt and division, and the SH are the stored float32 values.
// (exp / sigmoid of scales and opacities stay on the host in numpy so they round
// as the reference's do.)  The first non-finite vertex of each property group
// and the first zero-norm quaternion are reported for the reference's DataErrors.
#include "common.cuh"

namespace rcgs {

// offsets (in floats within a row): 0..2 x y z, 3..6 rot_0..3, 7..9 f_dc_0..2,
// 10..54 f_rest_0..44, 55 opacity, 56..58 scale_0..2
constexpr int kPlyCols = 59;

struct PlyOffsets {
    int32_t o[kPlyCols];
};

__global__ void ply_decode_kernel(const float* __restrict__ rows, int64_t n, int32_t row_floats, PlyOffsets off,
                                  double* __restrict__ pos, double* __restrict__ rot, float* __restrict__ sh,
                                  unsigned long long* __restrict__ first_bad) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const float* r = rows + g * row_floats;
    // non-finite groups in the reference's check order: position, opacity, scale,
    // rotation, f_dc, f_rest; [6] = zero-norm quaternion
    auto bad = [&](int grp, int lo, int hi) {
        bool b = false;
        for (int c = lo; c < hi; ++c) b |= !isfinite(r[off.o[c]]);
        if (b) atomicMin(&first_bad[grp], (unsigned long long)g);
    };
    bad(0, 0, 3);
    bad(1, 55, 56);
    bad(2, 56, 59);
    bad(3, 3, 7);
    bad(4, 7, 10);
    bad(5, 10, 55);
#pragma unroll
    for (int i = 0; i < 3; ++i) pos[3 * g + i] = (double)r[off.o[i]];
    const double q0 = r[off.o[3]], q1 = r[off.o[4]], q2 = r[off.o[5]], q3 = r[off.o[6]];
    const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q0, q0), __dmul_rn(q1, q1)),
                                                      __dmul_rn(q2, q2)),
                                            __dmul_rn(q3, q3)));
    if (nrm < 1e-12) atomicMin(&first_bad[6], (unsigned long long)g);
    rot[4 * g] = __ddiv_rn(q0, nrm);
    rot[4 * g + 1] = __ddiv_rn(q1, nrm);
    rot[4 * g + 2] = __ddiv_rn(q2, nrm);
    rot[4 * g + 3] = __ddiv_rn(q3, nrm);
    float* o = sh + 48 * g;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        o[c] = r[off.o[7 + c]];  // DC
#pragma unroll
        for (int j = 0; j < 15; ++j) o[3 * (j + 1) + c] = r[off.o[10 + 15 * c + j]];  // channel-major f_rest
    }
}

// SH columns of a checkpoint row buffer (scene_io.py:156-166 on the published
// snapshot, optimize.py:226-238): value = float32(base + (new - old)) in fp64 when
// a base is given (the host's fp64 SH plus the device's fp32 delta), else new.
// One thread per (gaussian, coefficient): SH reads are coalesced, the writes of a
// row land inside one 248-byte record.
__global__ void ply_encode_sh_kernel(const double* __restrict__ base, const float* __restrict__ old32,
                                     const float* __restrict__ new32, int64_t n, int32_t row_floats,
                                     PlyOffsets off, float* __restrict__ rows) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * 48) return;
    const int64_t g = i / 48;
    const int k = (int)(i - g * 48), j = k / 3, c = k - 3 * j;
    float v = new32[i];
    if (base) v = __double2float_rn(__dadd_rn(base[i], __dsub_rn((double)v, (double)old32[i])));
    // coefficient j of channel c: f_dc_c for j == 0, else f_rest_{15c + j - 1}
    const int col = j == 0 ? 7 + c : 10 + 15 * c + (j - 1);
    rows[g * row_floats + off.o[col]] = v;
}

}  // namespace rcgs

using namespace rcgs;

extern "C" int rcgs_ply_encode_sh(const double* d_base, const float* d_old, const float* d_new, int64_t n,
                                  int32_t row_floats, const int32_t* h_offsets59, float* d_rows, void* stream) {
    RCGS_CHECK_ARG(d_new && h_offsets59 && d_rows, "null argument");
    RCGS_CHECK_ARG(!d_base || d_old, "base without old SH");
    RCGS_CHECK_ARG(row_floats >= kPlyCols, "row has %d floats, need >= %d", row_floats, kPlyCols);
    PlyOffsets off;
    for (int i = 0; i < kPlyCols; ++i) {
        RCGS_CHECK_ARG(h_offsets59[i] >= 0 && h_offsets59[i] < row_floats, "bad property offset");
        off.o[i] = h_offsets59[i];
    }
    if (n > 0) {
        ply_encode_sh_kernel<<<div_up(n * 48, 256), 256, 0, as_stream(stream)>>>(d_base, d_old, d_new, n,
                                                                                 row_floats, off, d_rows);
        RCGS_LAUNCH_CHECK();
    }
    return RCGS_OK;
}

extern "C" int rcgs_ply_decode(const float* d_rows, int64_t n, int32_t row_floats, const int32_t* h_offsets59,
                               double* d_pos, double* d_rot, float* d_sh, int64_t* h_first_bad7, void* stream) {
    RCGS_CHECK_ARG(d_rows && h_offsets59 && d_pos && d_rot && d_sh && h_first_bad7, "null argument");
    RCGS_CHECK_ARG(row_floats >= kPlyCols, "row has %d floats, need >= %d", row_floats, kPlyCols);
    cudaStream_t s = as_stream(stream);
    PlyOffsets off;
    for (int i = 0; i < kPlyCols; ++i) {
        RCGS_CHECK_ARG(h_offsets59[i] >= 0 && h_offsets59[i] < row_floats, "bad property offset");
        off.o[i] = h_offsets59[i];
    }
    unsigned long long* bad = nullptr;
    RCGS_TRY(dalloc(&bad, 7, s));
    RCGS_CUDA(cudaMemsetAsync(bad, 0xff, 7 * sizeof(unsigned long long), s));
    if (n > 0) {
        ply_decode_kernel<<<div_up(n, 256), 256, 0, s>>>(d_rows, n, row_floats, off, d_pos, d_rot, d_sh, bad);
        RCGS_LAUNCH_CHECK();
    }
    unsigned long long hb[7];
    RCGS_CUDA(cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaStreamSynchronize(s));
    dfree(bad, s);
    for (int i = 0; i < 7; ++i) h_first_bad7[i] = hb[i] == ~0ull ? -1 : (int64_t)hb[i];
    return RCGS_OK;
}
