// Stable LSD radix sort, onesweep style (hand-written; no CUB).
//
// Used for (a) the global front-to-back order of the kept gaussians: a stable
// sort of the fp64 view-space z bit patterns (positive doubles order like their
// uint64 bits), ties by scene index == np.argsort(z, kind="stable")
// (render.py:216); and (b) the stable (tile | depth) pair sort: pairs are
// emitted in depth-rank order, so a stable sort on the tile id alone yields
// (tile, depth) order.
//
// Per sort: one histogram kernel computes the global digit counts of EVERY
// 8-bit pass at once, one single-block kernel scans them, then each pass is ONE
// scatter kernel.  A scatter block takes the next 4096-item tile (dynamic id,
// so predecessors are always resident or done), ranks its items stably
// (each warp owns 512 consecutive items: match_any ranks + per-warp digit
// counters, then a cross-warp prefix), and finds its per-digit global offset by
// decoupled look-back over the preceding tiles' published (flag | count)
// words.  Four block barriers per tile.
#include "common.cuh"

namespace rcgs {

constexpr int kRNT = 256;
constexpr int kRWarps = kRNT / 32;
constexpr int kRIPT = 16;
constexpr int kRTile = kRNT * kRIPT;      // 4096 items per tile
constexpr int kRPerWarp = kRTile / kRWarps; // 512 consecutive items per warp
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPre = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1u;
constexpr int kMaxPasses = 8;

template <typename K>
__global__ void __launch_bounds__(kRNT) radix_hist_all_kernel(const K* __restrict__ keys, int64_t n,
                                                                int npass, int end_bit,
                                                                uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kMaxPasses][256];
    for (int i = threadIdx.x; i < kMaxPasses * 256; i += kRNT) (&h[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * kRNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRNT) {
        const K k = keys[i];
        for (int p = 0; p < npass; ++p) {
            const int bits = min(8, end_bit - 8 * p);
            atomicAdd(&h[p][(uint32_t)(k >> (8 * p)) & ((1u << bits) - 1u)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * 256; i += kRNT) {
        const uint32_t c = (&h[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// Exclusive scan of each pass's 256 global digit counts (one block).
__global__ void radix_hist_scan_kernel(uint32_t* __restrict__ hist, int npass) {
    __shared__ uint32_t ws[kRWarps];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int p = 0; p < npass; ++p) {
        const uint32_t v = hist[p * 256 + t];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        uint32_t off = 0;
        for (int w = 0; w < warp; ++w) off += ws[w];
        hist[p * 256 + t] = off + x - v;
        __syncthreads();
    }
}

template <typename K>
__global__ void __launch_bounds__(kRNT) radix_onesweep_kernel(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, bool vals_are_index, K* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n, int shift, uint32_t mask, const uint32_t* __restrict__ gstart,
    uint32_t* __restrict__ status, uint32_t* __restrict__ tile_counter) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t wcnt[kRWarps][256];
    __shared__ uint32_t s_base[256];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) s_tile = atomicAdd(tile_counter, 1u);
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) wcnt[w][t] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t wbase = (int64_t)tile * kRTile + (int64_t)warp * kRPerWarp;
    const uint32_t lt = (1u << lane) - 1u;

    K key[kRIPT];
    uint32_t val[kRIPT];
    uint32_t rank[kRIPT];
    // all 16 coalesced loads first (independent, in flight together) ...
#pragma unroll
    for (int r = 0; r < kRIPT; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool valid = i < n;
        key[r] = valid ? kin[i] : K(0);
        val[r] = valid ? (vals_are_index ? (uint32_t)i : vin[i]) : 0u;
    }
    // ... then the stable warp-level ranking
#pragma unroll
    for (int r = 0; r < kRIPT; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = valid ? ((uint32_t)(key[r] >> shift) & mask) : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = valid ? wcnt[warp][d] : 0u;
        __syncwarp();
        rank[r] = before + __popc(peers & lt);
        if (valid && (peers & lt) == 0) wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // cross-warp exclusive prefix (digit t) and this tile's total for digit t
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) {
        const uint32_t c = wcnt[w][t];
        wcnt[w][t] = total;
        total += c;
    }
    // decoupled look-back over the preceding tiles for digit t
    volatile uint32_t* st = status;
    uint32_t excl = 0;
    if (tile == 0) {
        st[t] = kFlagPre | total;
    } else {
        st[(int64_t)tile * 256 + t] = kFlagAgg | total;
        // walk back in batches of 16 independent loads (memory-level parallelism
        // instead of one dependent L2 round trip per predecessor)
        constexpr int kLB = 16;
        bool found = false;
        for (int64_t hi = (int64_t)tile - 1; hi >= 0 && !found; hi -= kLB) {
            uint32_t w[kLB];
#pragma unroll
            for (int b = 0; b < kLB; ++b) w[b] = hi - b >= 0 ? st[(hi - b) * 256 + t] : (2u << 30);
#pragma unroll
            for (int b = 0; b < kLB; ++b) {
                if (found || hi - b < 0) continue;
                while ((w[b] >> 30) == 0) w[b] = st[(hi - b) * 256 + t];
                excl += w[b] & kValMask;
                if ((w[b] >> 30) == 2) found = true;
            }
        }
        st[(int64_t)tile * 256 + t] = kFlagPre | (excl + total);
    }
    s_base[t] = gstart[t] + excl;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRIPT; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        if (i < n) {
            const uint32_t d = (uint32_t)(key[r] >> shift) & mask;
            const uint32_t pos = s_base[d] + wcnt[warp][d] + rank[r];
            kout[pos] = key[r];
            vout[pos] = val[r];
        }
    }
}

template <typename K>
static int radix_sort(K** key_cur, K** key_alt, uint32_t** val_cur, uint32_t** val_alt, bool vals_are_index,
                      int64_t n, int end_bit, cudaStream_t s) {
    if (n <= 0 || end_bit <= 0) return RCGS_OK;
    RCGS_CHECK_ARG(n < (int64_t)kValMask, "radix sort: %lld items exceeds 2^30", (long long)n);
    const int npass = (end_bit + 7) / 8;
    RCGS_CHECK_ARG(npass <= kMaxPasses, "radix sort: %d key bits", end_bit);
    const int64_t ntiles = (n + kRTile - 1) / kRTile;
    // one zeroed scratch: global histograms, per-pass tile counters, per-pass status words
    const int64_t words = (int64_t)npass * 256 + npass + (int64_t)npass * ntiles * 256;
    uint32_t* scratch = nullptr;
    RCGS_TRY(dalloc(&scratch, words, s));
    RCGS_CUDA(cudaMemsetAsync(scratch, 0, words * sizeof(uint32_t), s));
    uint32_t* hist = scratch;
    uint32_t* counters = hist + npass * 256;
    uint32_t* status = counters + npass;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n + kRNT - 1) / kRNT;
    const int hblocks = (int)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
    radix_hist_all_kernel<K><<<hblocks, kRNT, 0, s>>>(*key_cur, n, npass, end_bit, hist);
    radix_hist_scan_kernel<<<1, 256, 0, s>>>(hist, npass);
    for (int p = 0; p < npass; ++p) {
        const int bits = min(8, end_bit - 8 * p);
        radix_onesweep_kernel<K><<<(unsigned)ntiles, kRNT, 0, s>>>(
            *key_cur, *val_cur, p == 0 && vals_are_index, *key_alt, *val_alt, n, 8 * p, (1u << bits) - 1u,
            hist + p * 256, status + (int64_t)p * ntiles * 256, counters + p);
        K* tk = *key_cur;
        *key_cur = *key_alt;
        *key_alt = tk;
        uint32_t* tv = *val_cur;
        *val_cur = *val_alt;
        *val_alt = tv;
    }
    RCGS_LAUNCH_CHECK();
    dfree(scratch, s);
    return RCGS_OK;
}

int radix_sort_u64(uint64_t** key_cur, uint64_t** key_alt, uint32_t** val_cur, uint32_t** val_alt,
                   bool vals_are_index, int64_t n, int end_bit, cudaStream_t s) {
    return radix_sort<uint64_t>(key_cur, key_alt, val_cur, val_alt, vals_are_index, n, end_bit, s);
}

int radix_sort_u32(uint32_t** key_cur, uint32_t** key_alt, uint32_t** val_cur, uint32_t** val_alt,
                   bool vals_are_index, int64_t n, int end_bit, cudaStream_t s) {
    return radix_sort<uint32_t>(key_cur, key_alt, val_cur, val_alt, vals_are_index, n, end_bit, s);
}

}  // namespace rcgs
