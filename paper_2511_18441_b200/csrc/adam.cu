// K7: SH gradient expansion fused with Adam (backward.py:36-40, optimize.py:59-83).
//
// The per-view backward (raster.cu) leaves one fp32 3-vector per gaussian,
// acc[i, ch] = active * sum_p g[p, ch] w_ip.  The dense (N, 16, 3) gradient is
// basis_k(dir_i) * acc[i, ch]; it is never materialised: one thread per float4
// of the 48 coefficients runs Adam with fully coalesced 16-byte SH / m / v
// accesses and rebuilds the (at most two) SH basis rows it needs in fp32.
// A device-side reject flag (non-finite gradient, optimize.py:72-74) skips the
// update, and the device step counter feeds the bias corrections, so a
// sequence of steps needs no host synchronisation.
#include <math.h>

#include <mutex>

#include "common.cuh"
#include "shmath.cuh"

namespace rcgs {

constexpr int kMaxViews = 16;

struct AccViews {
    const float* acc[kMaxViews];
    double cen[kMaxViews][3];
    int n;
};

struct AdamHyper {
    float lr_dc, lr_rest, b1, b2, eps;
};

__device__ __forceinline__ void adam4(float4& p, float4& m, float4& v, const float g[4], int f0,
                                      const AdamHyper& h, float inv_bc1, float inv_bc2) {
    float* pp = &p.x;
    float* mm = &m.x;
    float* vv = &v.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int k = (f0 + j) / 3;
        const float lr = k == 0 ? h.lr_dc : h.lr_rest;
        mm[j] = h.b1 * mm[j] + (1.0f - h.b1) * g[j];
        vv[j] = h.b2 * vv[j] + (1.0f - h.b2) * g[j] * g[j];
        const float mh = mm[j] * inv_bc1, vh = vv[j] * inv_bc2;
        pp[j] -= __fdividef(lr * mh, sqrtf(vh) + h.eps);
    }
}

// Bias corrections 1/(1 - beta^t) for t = step + 1, once per launch (fp64 pow).
__global__ void adam_prep_kernel(const int64_t* __restrict__ step, double db1, double db2,
                                 float2* __restrict__ inv) {
    const double t = (double)(*step + 1);
    *inv = make_float2((float)(1.0 / (1.0 - pow(db1, t))), (float)(1.0 / (1.0 - pow(db2, t))));
}

// SH basis rows 0..15 in fp32 along the unit direction (x, y, z) (render.py SH
// constants; rows above `deg` are 0), written out branch-free.
__device__ __forceinline__ void basis16_f32(float x, float y, float z, int deg, float r[16]) {
    const float xx = x * x, yy = y * y, zz = z * z;
    const float d1 = deg >= 1 ? 1.f : 0.f, d2 = deg >= 2 ? 1.f : 0.f, d3 = deg >= 3 ? 1.f : 0.f;
    r[0] = 0.28209479177387814f;
    r[1] = d1 * -0.4886025119029199f * y;
    r[2] = d1 * 0.4886025119029199f * z;
    r[3] = d1 * -0.4886025119029199f * x;
    r[4] = d2 * 1.0925484305920792f * (x * y);
    r[5] = d2 * -1.0925484305920792f * (y * z);
    r[6] = d2 * 0.31539156525252005f * (2.f * zz - xx - yy);
    r[7] = d2 * -1.0925484305920792f * (x * z);
    r[8] = d2 * 0.5462742152960396f * (xx - yy);
    r[9] = d3 * -0.5900435899266435f * y * (3.f * xx - yy);
    r[10] = d3 * 2.890611442640554f * (x * y) * z;
    r[11] = d3 * -0.4570457994644658f * y * (4.f * zz - xx - yy);
    r[12] = d3 * 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
    r[13] = d3 * -0.4570457994644658f * x * (4.f * zz - xx - yy);
    r[14] = d3 * 1.445305721320277f * z * (xx - yy);
    r[15] = d3 * -0.5900435899266435f * x * (xx - 3.f * yy);
}

// ---- bulk-copy (TMA) + mbarrier helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "RCGS_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra RCGS_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}

// The last block to finish (every block has read *step and *reject by then)
// commits the step: advances the counter unless rejected, records the outcome and
// re-arms the flag.  One thread per block.
__device__ __forceinline__ bool commit_step(unsigned* ticket, bool upd, int64_t* step, int32_t* reject,
                                            double* reject_record, int64_t* snapshot_step, int64_t new_step) {
    __threadfence();
    const bool last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    if (last) {
        if (upd) *step += 1;
        if (snapshot_step) *snapshot_step = new_step;
        *ticket = 0;
        if (reject_record) {  // consume the flag: record it, re-arm it for the next step
            *reject_record = upd ? 0.0 : 1.0;
            if (reject) *reject = 0;
        }
    }
    return last;
}

#ifndef RCGS_ADAM_TILE
#define RCGS_ADAM_TILE 56
#endif
// gaussians per tile: 56 keeps a 2-stage ring (with the side arrays) under a third
// of the SM's shared memory, i.e. 3 CTAs per SM at one view per step
constexpr int kAG = RCGS_ADAM_TILE;
static_assert(kAG % 8 == 0 && kAG <= 64, "whole warps of 8 gaussians; 16-byte side-array tiles");
constexpr int kAThreads = 4 * kAG;          // 4 threads per gaussian, 12 coefficients each
constexpr int kStateG = 64;                 // gaussians per tile_state entry (ABI: 64-gaussian blocks)
#ifndef RCGS_ADAM_STAGES
#define RCGS_ADAM_STAGES 2
#endif
constexpr int kAStages = RCGS_ADAM_STAGES;  // tiles in flight per CTA
constexpr uint32_t kARow = 48 * 4;          // bytes of one gaussian's SH (or m, or v)
constexpr uint32_t kATileBytes = kAG * kARow;
// A stage holds, besides the SH / m / v tiles, the tile's positions (fp64 x 3),
// next-view depth ranks and each view's acc (fp32 x 3), so the update and the
// colour epilogue read no global memory on the critical path.
constexpr uint32_t kAPosBytes = kAG * 24;   // 1536
constexpr uint32_t kARankBytes = kAG * 4;   // 256
constexpr uint32_t kAAccBytes = kAG * 12;   // 768 per view
__host__ __device__ constexpr uint32_t adam_stage_bytes(int n_views) {
    return 3 * kATileBytes + kAPosBytes + kARankBytes + (uint32_t)n_views * kAAccBytes;
}
__host__ __device__ constexpr size_t adam_smem_bytes(int n_views) {
    return (size_t)kAStages * adam_stage_bytes(n_views) + kAStages * sizeof(uint64_t);
}

// Fused SH-gradient expansion + Adam over all N x 48 coefficients (optimize.py
// Adam; recolor.py SH-only refit).  The step streams SH, m and v once each way
// (1152 B per gaussian), so it is HBM bound: persistent CTAs pull 64-gaussian
// tiles of all three arrays with bulk async copies (TMA) into a 2-stage shared
// ring completed by mbarrier transaction counts, update them in shared memory
// (4 threads per gaussian: the view direction and SH basis once per thread
// instead of once per float4) and write them back with bulk stores, which read
// the stage before it is refilled.  Element order, products and Adam formulas
// are the per-element ones of adam4, so results are bit-identical to an
// elementwise update.
__global__ void __launch_bounds__(kAThreads, 3) adam_fused_kernel(
    const double* __restrict__ pos, int64_t n, int deg, float* __restrict__ sh, float* __restrict__ m,
    float* __restrict__ v, AccViews views, AdamHyper h, int64_t* __restrict__ step, double db1, double db2,
    unsigned* __restrict__ ticket, int32_t* __restrict__ reject, const int32_t* __restrict__ next_rank_of,
    Center next_cen, float4* __restrict__ next_color, uint32_t* __restrict__ next_fix,
    double* __restrict__ reject_record,
    float* __restrict__ snapshot, int64_t* __restrict__ snapshot_step, int64_t snapshot_every,
    const uint32_t* __restrict__ tile_state) {
    // a rejected step (non-finite gradient) leaves SH/m/v untouched; with a fused
    // colour epilogue the next view is still coloured from the unchanged SH.
    // Every block still takes the last-block ticket, so the step commit (reject
    // record + re-arming the flag) happens exactly once, after every block has
    // read the flag.
    const bool upd = !(reject && *reject);
    if (!upd && next_color == nullptr) {
        if (threadIdx.x == 0) commit_step(ticket, upd, step, reject, reject_record, nullptr, 0);
        return;
    }
    // publish: this step commits step count *step + 1; a multiple of the cadence
    // also writes the updated tiles to the snapshot (optimize.py:221-222)
    const bool snap = upd && snapshot != nullptr && snapshot_every > 0 && (*step + 1) % snapshot_every == 0;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t stage_bytes = adam_stage_bytes(views.n);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kAStages * stage_bytes);
    const int t = threadIdx.x;
    const int64_t ntiles = (n + kAG - 1) / kAG;
    float* const arrays[3] = {sh, m, v};
    auto stage_base = [&](int s) -> unsigned char* { return smem + (size_t)s * stage_bytes; };
    auto stage_buf = [&](int s, int arr) -> float4* {
        return reinterpret_cast<float4*>(stage_base(s) + (size_t)arr * kATileBytes);
    };
    auto stage_pos = [&](int s) -> double* { return reinterpret_cast<double*>(stage_base(s) + 3 * kATileBytes); };
    auto stage_rank = [&](int s) -> int32_t* {
        return reinterpret_cast<int32_t*>(stage_base(s) + 3 * kATileBytes + kAPosBytes);
    };
    auto stage_acc = [&](int s, int vi) -> float* {
        return reinterpret_cast<float*>(stage_base(s) + 3 * kATileBytes + kAPosBytes + kARankBytes +
                                        (size_t)vi * kAAccBytes);
    };
    // per tile: 2 = full update (SH, m, v in and out), 1 = SH in only (an inactive
    // tile whose SH the fused colour epilogue needs), 0 = nothing.  A tile is
    // inactive when its Adam state is exactly 0 and every view's acc is 0 there
    // (tile_state, adam_active_kernel): Adam then leaves all of it bit-identical
    // (m' = v' = 0, theta' = theta - lr * 0 / (0 + eps)), so the skip is exact.
    auto mode_of = [&](int64_t tile) -> int {
        // the 64-gaussian state blocks overlapping this tile
        const int64_t last = tile * kAG + kAG - 1 < n ? tile * kAG + kAG - 1 : n - 1;
        const int64_t a0 = tile * kAG / kStateG, a1 = last / kStateG;
        const bool active = tile_state == nullptr || tile_state[a0] != 0u || tile_state[a1] != 0u;
        return (upd && active) ? 2 : (next_color != nullptr ? 1 : 0);
    };
    // Side arrays (positions, ranks, acc) ride the same barrier for full tiles; the
    // last, partial tile (byte counts not multiples of 16) reads them from global.
    auto issue = [&](int64_t tile, int s) {  // one thread
        const int64_t g0 = tile * kAG;
        const bool full = n - g0 >= kAG;
        const uint32_t bytes = (uint32_t)(full ? kAG : n - g0) * kARow;
        const uint32_t bar = smem_addr(&bars[s]);
        const int md = mode_of(tile);
        const int na = md == 2 ? 3 : md;
        const bool need_pos = full && md != 0;
        const bool need_rank = full && md != 0 && next_color != nullptr;
        const bool need_acc = full && md == 2;
        const uint32_t tx = (uint32_t)na * bytes + (need_pos ? kAPosBytes : 0u) + (need_rank ? kARankBytes : 0u) +
                            (need_acc ? (uint32_t)views.n * kAAccBytes : 0u);
        mbar_expect_tx(bar, tx);  // 0 bytes: the phase completes at once
        for (int arr = 0; arr < na; ++arr)
            bulk_load(smem_addr(stage_buf(s, arr)), arrays[arr] + g0 * 48, bytes, bar);
        if (need_pos) bulk_load(smem_addr(stage_pos(s)), pos + 3 * g0, kAPosBytes, bar);
        if (need_rank) bulk_load(smem_addr(stage_rank(s)), next_rank_of + g0, kARankBytes, bar);
        if (need_acc)
            for (int vi = 0; vi < views.n; ++vi)
                bulk_load(smem_addr(stage_acc(s, vi)), views.acc[vi] + 3 * g0, kAAccBytes, bar);
    };
    __shared__ float2 s_bc;
    if (t == 0) {
        for (int s = 0; s < kAStages; ++s) mbar_init(smem_addr(&bars[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // bias corrections 1 / (1 - beta^t) for t = step + 1 (fp64 pow)
        const double tt = (double)(*step + 1);
        s_bc = make_float2((float)(1.0 / (1.0 - pow(db1, tt))), (float)(1.0 / (1.0 - pow(db2, tt))));
    }
    __syncthreads();
    if (t == 0) {
        for (int s = 0; s < kAStages; ++s)
            if ((int64_t)blockIdx.x + (int64_t)s * gridDim.x < ntiles) issue(blockIdx.x + (int64_t)s * gridDim.x, s);
    }
    const float2 ibc = s_bc;
    const int gi = t >> 2, part = t & 3;  // gaussian in the tile, 12-coefficient quarter
    const int lane = t & 31;
    const float invn = 1.0f / (float)views.n;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it % kAStages;
        const int64_t g0 = tile * kAG;
        const int ng = (int)(n - g0 < kAG ? n - g0 : kAG);
        const bool full = ng == kAG;
        mbar_wait(smem_addr(&bars[s]), (uint32_t)((it / kAStages) & 1));
        const int md = mode_of(tile);
        // this tile's positions: staged (full tiles) or global (the partial one)
        const double* tpos = full ? stage_pos(s) : pos + 3 * g0;
        float c12[12];  // this thread's 12 coefficients after the update (colour epilogue)
        if (md == 2 && gi < ng) {
            const double px = tpos[3 * gi], py = tpos[3 * gi + 1], pz = tpos[3 * gi + 2];
            float gr[12];
#pragma unroll
            for (int e = 0; e < 12; ++e) gr[e] = 0.f;
            for (int vi = 0; vi < views.n; ++vi) {
                float x = (float)(px - views.cen[vi][0]), y = (float)(py - views.cen[vi][1]),
                      z = (float)(pz - views.cen[vi][2]);
                const float inv = rsqrtf(x * x + y * y + z * z);
                x *= inv;
                y *= inv;
                z *= inv;
                float r[16];
                basis16_f32(x, y, z, deg, r);
                // this thread's rows 4 part .. 4 part + 3 (branch-free selects)
                float b[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    b[q] = part == 0 ? r[q] : (part == 1 ? r[4 + q] : (part == 2 ? r[8 + q] : r[12 + q]));
                const float* acc = (full ? stage_acc(s, vi) : views.acc[vi] + 3 * g0) + 3 * gi;
                const float a3[3] = {acc[0], acc[1], acc[2]};
#pragma unroll
                for (int e = 0; e < 12; ++e) gr[e] += b[e / 3] * a3[e % 3];
            }
            if (views.n > 1) {
#pragma unroll
                for (int e = 0; e < 12; ++e) gr[e] *= invn;
            }
            float4* P = stage_buf(s, 0) + gi * 12 + part * 3;
            float4* Mm = stage_buf(s, 1) + gi * 12 + part * 3;
            float4* V = stage_buf(s, 2) + gi * 12 + part * 3;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                float4 p4 = P[q], m4 = Mm[q], v4 = V[q];
                adam4(p4, m4, v4, &gr[4 * q], part * 12 + 4 * q, h, ibc.x, ibc.y);
                P[q] = p4;
                Mm[q] = m4;
                V[q] = v4;
                c12[4 * q] = p4.x;
                c12[4 * q + 1] = p4.y;
                c12[4 * q + 2] = p4.z;
                c12[4 * q + 3] = p4.w;
            }
        } else if (md == 1 && gi < ng) {  // rejected step or inactive tile: the SH as loaded
            const float* P = reinterpret_cast<const float*>(stage_buf(s, 0)) + gi * 48 + part * 12;
#pragma unroll
            for (int e = 0; e < 12; ++e) c12[e] = P[e];
        }
        // the colour epilogue's inputs leave the stage before it is refilled
        const int64_t g = g0 + gi;
        const bool ok = next_color != nullptr && gi < ng;
        const int32_t rs = ok ? (full ? stage_rank(s)[gi] : next_rank_of[g]) : -1;
        double dx = 1.0, dy = 0.0, dz = 0.0;
        if (ok) {
            dx = tpos[3 * gi] - next_cen.c[0];
            dy = tpos[3 * gi + 1] - next_cen.c[1];
            dz = tpos[3 * gi + 2] - next_cen.c[2];
        }
        // shared-memory writes -> visible to the bulk-copy (async) proxy, then store
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (t == 0 && md == 2) {
            const uint32_t bytes = (uint32_t)ng * kARow;
#pragma unroll
            for (int arr = 0; arr < 3; ++arr) bulk_store(arrays[arr] + g0 * 48, smem_addr(stage_buf(s, arr)), bytes);
            if (snap) bulk_store(snapshot + g0 * 48, smem_addr(stage_buf(s, 0)), bytes);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (t == 0) {
            const int64_t next = tile + (int64_t)kAStages * gridDim.x;
            if (next < ntiles) {
                // the stage is refilled only after the store has read it
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                issue(next, s);
            }
        }
        if (next_color != nullptr) {
            // fused colour pass of the next step's view (render.py:209-214) from the
            // updated coefficients in registers, overlapping the stage's refill: each
            // of a gaussian's 4 threads evaluates its basis-row quarter in fp32 (the
            // operations and order of color_kernel, so the same bits) and lane part 0
            // combines and writes the colour.  A gaussian whose activation is too
            // close to call in fp32 takes the fp64 colour (color_kernel's fallback);
            // its direction costs one fp64 division per lane (lane part p divides
            // component p, then the 4 lanes exchange).
            float fx, fy, fz;
            dir_f32(dx, dy, dz, fx, fy, fz);
            float qf[3] = {0.f, 0.f, 0.f}, mf[3] = {0.f, 0.f, 0.f};
            if (rs >= 0) {
                float bf[16];
                basis16_rn(fx, fy, fz, deg, bf);
                color_quarter_f32(bf, c12, part, qf, mf);
            }
            float col[3];
            int act = 0;
            bool amb = false;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                const float q1 = __shfl_down_sync(0xffffffffu, qf[ch], 1), q2 = __shfl_down_sync(0xffffffffu, qf[ch], 2),
                            q3 = __shfl_down_sync(0xffffffffu, qf[ch], 3);
                const float m1 = __shfl_down_sync(0xffffffffu, mf[ch], 1), m2 = __shfl_down_sync(0xffffffffu, mf[ch], 2),
                            m3 = __shfl_down_sync(0xffffffffu, mf[ch], 3);
                const float v = __fadd_rn(color_combine_f32(qf[ch], q1, q2, q3), 0.5f);
                amb = amb || color_ambiguous(v, color_combine_f32(mf[ch], m1, m2, m3));
                act |= (v > 0.f) << ch;
                col[ch] = fmaxf(0.f, v);
            }
            amb = amb && rs >= 0 && part == 0;
            // rare (never at C3): the gaussian is queued for the fp64 colour, which the
            // last block writes once every block has finished (an inline fp64
            // fallback cost the common path ~40% of the kernel through its registers
            // alone; a separate fixup launch cost a kernel boundary per step)
            if (amb) {
                const uint32_t slot = atomicAdd(next_fix, 1u);
                next_fix[1 + slot] = (uint32_t)g;
            }
            if (rs >= 0 && part == 0)  // colours are stored by scene index
                next_color[g] = make_float4(col[0], col[1], col[2], __int_as_float(act));
        }
    }
    // this block's queue entries and colour stores are visible before its ticket
    __threadfence();
    __syncthreads();
    __shared__ unsigned s_last;
    if (t == 0) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");     // SH stores complete
        asm volatile("fence.proxy.async.global;" ::: "memory");         // ... and ordered before the ticket
        s_last = commit_step(ticket, upd, step, reject, reject_record, snap ? snapshot_step : nullptr, *step + 1);
    }
    __syncthreads();
    if (s_last && next_fix != nullptr) {  // the fp64 colours queued by the epilogue (color_f64)
        __threadfence();
        const uint32_t cnt = __ldcg(next_fix);
        for (uint32_t i = t; i < cnt; i += blockDim.x) {
            const int64_t g = __ldcg(next_fix + 1 + i);
            next_color[g] = color_f64(pos, reinterpret_cast<const float4*>(sh), g, next_cen, deg);
        }
        __syncthreads();
        if (t == 0) *next_fix = 0u;
    }
}

// tile_state[t] |= any view's acc != 0 in tile t (NaN counts as nonzero).  Run
// before the fused Adam of the step, on its stream; state only ever grows, so a
// flag set by a step that is then rejected is merely conservative.
__global__ void adam_active_kernel(AccViews views, int64_t n, uint32_t* __restrict__ state) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool nz = false;
    if (g < n) {
        for (int vi = 0; vi < views.n; ++vi) {
            const float* acc = views.acc[vi] + 3 * g;
            nz = nz || !(acc[0] == 0.f && acc[1] == 0.f && acc[2] == 0.f);
        }
    }
    // a warp covers 32 gaussians of one 64-gaussian state block
    if (__ballot_sync(0xffffffffu, nz) && (threadIdx.x & 31) == 0) state[g / kStateG] = 1u;
}

__global__ void adam_dense_kernel(float4* __restrict__ p, float4* __restrict__ m, float4* __restrict__ v,
                                  const float4* __restrict__ grad, int64_t nq, AdamHyper h,
                                  const float2* __restrict__ bc, const int32_t* __restrict__ reject) {
    if (reject && *reject) return;
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const float2 ibc = *bc;
    const float4 g4 = grad[q];
    const float gr[4] = {g4.x, g4.y, g4.z, g4.w};
    float4 pp = p[q], mm = m[q], vv = v[q];
    adam4(pp, mm, vv, gr, 4 * (int)(q % 12), h, ibc.x, ibc.y);
    p[q] = pp;
    m[q] = mm;
    v[q] = vv;
}

__global__ void step_commit_kernel(int32_t* __restrict__ reject, int64_t* __restrict__ step,
                                   double* __restrict__ reject_record, int64_t* __restrict__ snapshot_step = nullptr,
                                   int64_t every = 0) {
    const bool rej = reject && *reject;
    if (!rej) {
        *step += 1;
        if (snapshot_step && every > 0 && *step % every == 0) *snapshot_step = *step;  // empty scene
    }
    if (reject_record) {
        *reject_record = rej ? 1.0 : 0.0;
        if (reject) *reject = 0;
    }
}

__global__ void sh_grad_kernel(const double* __restrict__ pos, int64_t n, int deg,
                               const float* __restrict__ acc, Center cen, float* __restrict__ grad) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    double x, y, z;
    view_dir(pos, g, cen.c, x, y, z);
    double b[16];
    sh_basis16<double>(x, y, z, deg, b);
    const float a0 = acc[3 * g], a1 = acc[3 * g + 1], a2 = acc[3 * g + 2];
    float* o = grad + 48 * g;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        o[3 * k] = (float)(b[k] * a0);
        o[3 * k + 1] = (float)(b[k] * a1);
        o[3 * k + 2] = (float)(b[k] * a2);
    }
}

__global__ void nonfinite_kernel(const float* __restrict__ x, int64_t count, int32_t* __restrict__ flag) {
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

static AdamHyper hyper(const rcgs_adam_config* c) {
    AdamHyper h;
    h.lr_dc = (float)c->lr_dc;
    h.lr_rest = (float)c->lr_rest;
    h.b1 = (float)c->beta1;
    h.b2 = (float)c->beta2;
    h.eps = (float)c->eps;
    return h;
}

}  // namespace rcgs

using namespace rcgs;

static int adam_fused_impl(const rcgs_scene* sc, float* d_sh, float* d_m, float* d_v,
                           const float* const* h_d_accs, const double* h_centers, int32_t n_views,
                           const rcgs_adam_config* cfg, int32_t* d_reject, int64_t* d_step,
                           double* d_reject_record, rcgs_view* next_view, const rcgs_adam_publish* pub,
                           uint32_t* d_tile_state, void* stream) {
    RCGS_CHECK_ARG(sc && d_sh && d_m && d_v && h_d_accs && h_centers && cfg && d_step, "null argument");
    RCGS_CHECK_ARG(pub == nullptr || (pub->d_snapshot != nullptr && pub->every > 0),
                   "snapshot publication needs a buffer and a positive cadence");
    RCGS_CHECK_ARG(next_view == nullptr || next_view->scene == sc, "next view belongs to another scene");
    RCGS_CHECK_ARG(n_views >= 1 && n_views <= kMaxViews, "views per step must be in [1, %d]", kMaxViews);
    RCGS_CHECK_ARG(sc->n < (int64_t)357913941, "scene too large for 32-bit Adam indexing");
    cudaStream_t s = as_stream(stream);
    if (sc->n > 0) {
        AccViews av;
        av.n = n_views;
        for (int i = 0; i < n_views; ++i) {
            av.acc[i] = h_d_accs[i];
            for (int j = 0; j < 3; ++j) av.cen[i][j] = h_centers[3 * i + j];
        }
        // persistent grid per staged-view count (the stage size depends on it)
        static std::mutex grid_mu;
        static int grids[kMaxViews + 1] = {0};
        const size_t smem = adam_smem_bytes(n_views);
        int grid = 0;
        {
            std::lock_guard<std::mutex> lock(grid_mu);
            if (grids[n_views] == 0) {
                int dev = 0, sms = 0, per_sm = 0;
                RCGS_CUDA(cudaGetDevice(&dev));
                RCGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
                RCGS_CUDA(cudaFuncSetAttribute(adam_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)adam_smem_bytes(kMaxViews)));
                RCGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adam_fused_kernel, kAThreads, smem));
                grids[n_views] = sms * persistent_ctas(per_sm > 0 ? per_sm : 1);
            }
            grid = grids[n_views];
        }
        RCGS_CHECK_ARG(grid > 0, "adam launch setup failed");
        // last-block ticket, one per stream: concurrent launches on different streams
        // must not mix their counts (reset by the last block of each launch)
        unsigned* ticket = stream_ticket(s);
        RCGS_CHECK_ARG(ticket != nullptr, "adam ticket allocation failed");
        const int64_t ntiles = (sc->n + kAG - 1) / kAG;
        Center nc = {{0.0, 0.0, 0.0}};
        const int32_t* nrank = nullptr;
        float4* ncolor = nullptr;
        uint32_t* nfix = nullptr;
        if (next_view != nullptr && next_view->k > 0) {
            nc = camera_center(next_view->cam);
            nrank = next_view->rank_of;
            ncolor = next_view->color;
            nfix = next_view->fix;
        }
        if (d_tile_state != nullptr) {
            adam_active_kernel<<<div_up(sc->n, 256), 256, 0, s>>>(av, sc->n, d_tile_state);
            RCGS_LAUNCH_CHECK();
        }
        // bias corrections from and commit of the device step counter happen inside
        adam_fused_kernel<<<(int)(ntiles < grid ? ntiles : grid), kAThreads, smem, s>>>(
            sc->pos, sc->n, sc->sh_degree, d_sh, d_m, d_v, av, hyper(cfg), d_step, cfg->beta1, cfg->beta2, ticket,
            d_reject, nrank, nc, ncolor, nfix, d_reject_record, pub ? pub->d_snapshot : nullptr,
            pub ? pub->d_snapshot_step : nullptr, pub ? pub->every : 0, d_tile_state);
        RCGS_LAUNCH_CHECK();

        return RCGS_OK;
    }
    step_commit_kernel<<<1, 1, 0, s>>>(d_reject, d_step, d_reject_record, pub ? pub->d_snapshot_step : nullptr,
                                       pub ? pub->every : 0);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_adam_fused(const rcgs_scene* sc, float* d_sh, float* d_m, float* d_v,
                               const float* const* h_d_accs, const double* h_centers, int32_t n_views,
                               const rcgs_adam_config* cfg, int32_t* d_reject, int64_t* d_step,
                               double* d_reject_record, void* stream) {
    return adam_fused_impl(sc, d_sh, d_m, d_v, h_d_accs, h_centers, n_views, cfg, d_reject, d_step,
                           d_reject_record, nullptr, nullptr, nullptr, stream);
}

extern "C" int rcgs_adam_fused_ex(const rcgs_scene* sc, float* d_sh, float* d_m, float* d_v,
                                  const float* const* h_d_accs, const double* h_centers, int32_t n_views,
                                  const rcgs_adam_config* cfg, int32_t* d_reject, int64_t* d_step,
                                  double* d_reject_record, rcgs_view* next_view, const rcgs_adam_publish* publish,
                                  uint32_t* d_tile_state, void* stream) {
    return adam_fused_impl(sc, d_sh, d_m, d_v, h_d_accs, h_centers, n_views, cfg, d_reject, d_step,
                           d_reject_record, next_view, publish, d_tile_state, stream);
}

extern "C" int rcgs_adam_fused_next(const rcgs_scene* sc, float* d_sh, float* d_m, float* d_v,
                                    const float* const* h_d_accs, const double* h_centers, int32_t n_views,
                                    const rcgs_adam_config* cfg, int32_t* d_reject, int64_t* d_step,
                                    double* d_reject_record, rcgs_view* next_view, void* stream) {
    RCGS_CHECK_ARG(next_view != nullptr, "null next view");
    RCGS_CHECK_ARG(next_view->scene == sc, "next view belongs to another scene");
    return adam_fused_impl(sc, d_sh, d_m, d_v, h_d_accs, h_centers, n_views, cfg, d_reject, d_step,
                           d_reject_record, next_view, nullptr, nullptr, stream);
}

extern "C" int rcgs_adam_dense(float* d_params, float* d_m, float* d_v, const float* d_grads, int64_t n,
                               const rcgs_adam_config* cfg, const int32_t* d_reject, int64_t* d_step,
                               void* stream) {
    RCGS_CHECK_ARG(d_params && d_m && d_v && d_grads && cfg && d_step, "null argument");
    cudaStream_t s = as_stream(stream);
    const int64_t nq = n * 12;
    if (nq > 0) {
        float2* bc = nullptr;
        RCGS_TRY(dalloc(&bc, 1, s));
        adam_prep_kernel<<<1, 1, 0, s>>>(d_step, cfg->beta1, cfg->beta2, bc);
        adam_dense_kernel<<<div_up(nq, 256), 256, 0, s>>>(
            reinterpret_cast<float4*>(d_params), reinterpret_cast<float4*>(d_m), reinterpret_cast<float4*>(d_v),
            reinterpret_cast<const float4*>(d_grads), nq, hyper(cfg), bc, d_reject);
        RCGS_LAUNCH_CHECK();
        dfree(bc, s);
    }
    step_commit_kernel<<<1, 1, 0, s>>>(const_cast<int32_t*>(d_reject), d_step, nullptr);  // flag only read
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_sh_grad(const rcgs_scene* sc, const float* d_acc, const double* h_center3, float* d_grad,
                            void* stream) {
    RCGS_CHECK_ARG(sc && d_acc && h_center3 && d_grad, "null argument");
    if (sc->n == 0) return RCGS_OK;
    Center c;
    for (int j = 0; j < 3; ++j) c.c[j] = h_center3[j];
    sh_grad_kernel<<<div_up(sc->n, 256), 256, 0, as_stream(stream)>>>(sc->pos, sc->n, sc->sh_degree, d_acc, c,
                                                                       d_grad);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_nonfinite_check(const float* d_x, int64_t count, int32_t* d_flag, void* stream) {
    RCGS_CHECK_ARG(d_flag != nullptr, "null flag");
    if (count <= 0) return RCGS_OK;
    unsigned blocks = div_up(count, 256);
    if (blocks > 4096) blocks = 4096;
    nonfinite_kernel<<<blocks, 256, 0, as_stream(stream)>>>(d_x, count, d_flag);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}
