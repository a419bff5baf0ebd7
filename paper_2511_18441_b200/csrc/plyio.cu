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

// Rows are staged per block in shared memory (a tile of `tile` whole rows is one
// contiguous, coalesced copy each way); per-gaussian and per-coefficient work
// then reads the tile.  Tiles hold <= 48 KB, so any row width works.
__host__ __device__ inline int ply_tile_rows(int row_floats) {
    const int t = 12288 / row_floats;
    return t < 1 ? 1 : (t > 64 ? 64 : t);
}

// SH coefficient k = 3j + c of a gaussian -> column in the 59-entry order:
// f_dc_c for j == 0, else f_rest_{15c + j - 1} (channel-major, scene_io.py:141-146)
__device__ __forceinline__ int sh_col(int k) {
    const int j = k / 3, c = k - 3 * j;
    return j == 0 ? 7 + c : 10 + 15 * c + (j - 1);
}

__global__ void __launch_bounds__(128) ply_decode_kernel(const float* __restrict__ rows, int64_t n,
                                                         int32_t row_floats, PlyOffsets off, double* __restrict__ pos,
                                                         double* __restrict__ rot, float* __restrict__ sh,
                                                         unsigned long long* __restrict__ first_bad) {
    extern __shared__ float tile_rows[];
    __shared__ int so[kPlyCols];
    const int tile = ply_tile_rows(row_floats);
    const int64_t g0 = (int64_t)blockIdx.x * tile;
    const int nt = (int)(n - g0 < tile ? n - g0 : tile);
    if (threadIdx.x < kPlyCols) so[threadIdx.x] = off.o[threadIdx.x];
    const float* src = rows + g0 * row_floats;
    for (int i = threadIdx.x; i < nt * row_floats; i += blockDim.x) tile_rows[i] = src[i];
    __syncthreads();
    // non-finite groups in the reference's check order: position, opacity, scale,
    // rotation, f_dc, f_rest; [6] = zero-norm quaternion
    if (threadIdx.x < nt) {
        const int t = threadIdx.x;
        const int64_t g = g0 + t;
        const float* r = tile_rows + t * row_floats;
        auto bad = [&](int grp, int lo, int hi) {
            bool b = false;
            for (int c = lo; c < hi; ++c) b |= !isfinite(r[so[c]]);
            if (b) atomicMin(&first_bad[grp], (unsigned long long)g);
        };
        bad(0, 0, 3);
        bad(1, 55, 56);
        bad(2, 56, 59);
        bad(3, 3, 7);
#pragma unroll
        for (int i = 0; i < 3; ++i) pos[3 * g + i] = (double)r[so[i]];
        const double q0 = r[so[3]], q1 = r[so[4]], q2 = r[so[5]], q3 = r[so[6]];
        // numpy's norm: sqrt(((q0^2 + q1^2) + q2^2) + q3^2), each op rounded
        const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q0, q0), __dmul_rn(q1, q1)),
                                                          __dmul_rn(q2, q2)),
                                                __dmul_rn(q3, q3)));
        if (nrm < 1e-12) atomicMin(&first_bad[6], (unsigned long long)g);
        rot[4 * g] = __ddiv_rn(q0, nrm);
        rot[4 * g + 1] = __ddiv_rn(q1, nrm);
        rot[4 * g + 2] = __ddiv_rn(q2, nrm);
        rot[4 * g + 3] = __ddiv_rn(q3, nrm);
    }
    // SH, coefficient-parallel: the tile's output is contiguous -> coalesced stores
    float* dst = sh + g0 * 48;
    for (int i = threadIdx.x; i < nt * 48; i += blockDim.x) {
        const int t = i / 48, k = i - 48 * t;
        const float v = tile_rows[t * row_floats + so[sh_col(k)]];
        if (!isfinite(v)) atomicMin(&first_bad[k < 3 ? 4 : 5], (unsigned long long)(g0 + t));
        dst[i] = v;
    }
}

// SH columns of a checkpoint row buffer (scene_io.py:156-166 on the published
// snapshot, optimize.py:226-238): value = float32(base + (new - old)) in fp64 when
// a base is given (the host's fp64 SH plus the device's fp32 delta), else new.
// The block's rows are read into shared memory, their SH columns replaced, and
// written back whole: coalesced both ways.
__global__ void __launch_bounds__(128) ply_encode_sh_kernel(const double* __restrict__ base,
                                                            const float* __restrict__ old32,
                                                            const float* __restrict__ new32, int64_t n,
                                                            int32_t row_floats, PlyOffsets off,
                                                            float* __restrict__ rows) {
    extern __shared__ float tile_rows[];
    __shared__ int so[kPlyCols];
    const int tile = ply_tile_rows(row_floats);
    const int64_t g0 = (int64_t)blockIdx.x * tile;
    const int nt = (int)(n - g0 < tile ? n - g0 : tile);
    if (threadIdx.x < kPlyCols) so[threadIdx.x] = off.o[threadIdx.x];
    float* row0 = rows + g0 * row_floats;
    for (int i = threadIdx.x; i < nt * row_floats; i += blockDim.x) tile_rows[i] = row0[i];
    __syncthreads();
    const int64_t e0 = g0 * 48;
    for (int i = threadIdx.x; i < nt * 48; i += blockDim.x) {
        const int t = i / 48, k = i - 48 * t;
        float v = new32[e0 + i];
        if (base) v = __double2float_rn(__dadd_rn(base[e0 + i], __dsub_rn((double)v, (double)old32[e0 + i])));
        tile_rows[t * row_floats + so[sh_col(k)]] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nt * row_floats; i += blockDim.x) row0[i] = tile_rows[i];
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
        const int tile = ply_tile_rows(row_floats);
        ply_encode_sh_kernel<<<div_up(n, tile), 128, (size_t)tile * row_floats * sizeof(float), as_stream(stream)>>>(
            d_base, d_old, d_new, n, row_floats, off, d_rows);
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
        const int tile = ply_tile_rows(row_floats);
        ply_decode_kernel<<<div_up(n, tile), 128, (size_t)tile * row_floats * sizeof(float), s>>>(
            d_rows, n, row_floats, off, d_pos, d_rot, d_sh, bad);
        RCGS_LAUNCH_CHECK();
    }
    unsigned long long hb[7];
    RCGS_CUDA(cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaStreamSynchronize(s));
    dfree(bad, s);
    for (int i = 0; i < 7; ++i) h_first_bad7[i] = hb[i] == ~0ull ? -1 : (int64_t)hb[i];
    return RCGS_OK;
}
