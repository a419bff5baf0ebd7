// Stable LSD radix sort, reduce-then-scan (hand-written; no CUB).
//
// Used for (a) the global front-to-back order of the kept gaussians: a stable
// sort of the fp64 view-space z bit patterns (positive doubles order like their
// uint64 bits), ties by scene index == np.argsort(z, kind="stable")
// (render.py:216); and (b) the stable (tile | depth) pair sort: pairs are
// emitted in depth-rank order, so a stable sort on the tile id alone yields
// (tile, depth) order.
//
// Each 8-bit pass is three kernels over 2048-item tiles, all tiles independent:
//   upsweep    per-tile digit histogram (warp-aggregated shared atomics), also
//              added into the pass's global digit totals
//   scan       one block per digit: the digit's start (totals of the digits
//              below it) + exclusive scan of its per-tile counts
//              -> per-(digit, tile) offsets
//   downsweep  stable in-tile ranking (each warp owns 128 consecutive items:
//              ballot-built peer masks + per-warp digit counters, a cross-warp
//              prefix), a local sort by digit in shared memory, and a
//              write-out in which each digit's run is contiguous.
// A single-kernel onesweep pass with decoupled look-back was latency bound here:
// with every tile resident at once, inclusive prefixes propagate ~16 tiles per
// L2 round trip, so a pass over 225-650 tiles took 30-70 us; these three
// kernels have no inter-tile waiting.
#include "common.cuh"

namespace rcgs {

constexpr int kRNT = 256;
constexpr int kRWarps = kRNT / 32;
#ifndef RCGS_RADIX_IPT
#define RCGS_RADIX_IPT 8
#endif
constexpr int kRIPT = RCGS_RADIX_IPT;
constexpr int kRTile = kRNT * kRIPT;      // 2048 items per tile
constexpr int kRPerWarp = kRTile / kRWarps; // 256 consecutive items per warp
constexpr uint32_t kValMask = (1u << 30) - 1u;
constexpr int kMaxPasses = 8;

// Lanes holding the same digit as this lane, among the lanes with `valid` set:
// one ballot per digit bit.  match_any computes the same mask but is a slow
// instruction on sm_100a (measured 9.7 us vs 6.2 us for a ranking pass over 909K
// keys, tools/bench_radix.cu).
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, int bits, bool valid) {
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        if (b < bits) {
            const uint32_t bit = (d >> b) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
    }
    return peers;
}

// Per-tile digit histogram of one pass: hist[d * ntiles + tile].
template <typename K>
__global__ void __launch_bounds__(kRNT) radix_upsweep_kernel(const K* __restrict__ keys, int64_t n, int shift,
                                                             uint32_t mask, uint32_t* __restrict__ tile_hist,
                                                             int ntiles) {
    __shared__ uint32_t h[256];
    const int t = threadIdx.x;
    h[t] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRTile;
    K key[kRIPT];
#pragma unroll
    for (int r = 0; r < kRIPT; ++r) {
        const int64_t i = base + r * kRNT + t;
        key[r] = i < n ? keys[i] : K(0);
    }
#pragma unroll
    for (int r = 0; r < kRIPT; ++r) {
        const int64_t i = base + r * kRNT + t;
        // plain shared atomics (same-address lanes are combined by the hardware): as
        // fast as a copy here, unlike match_any aggregation
        if (i < n) atomicAdd(&h[(uint32_t)(key[r] >> shift) & mask], 1u);
    }
    __syncthreads();
    tile_hist[(int64_t)t * ntiles + blockIdx.x] = h[t];
}

// One block per digit d: rewrites d's row of per-tile counts as its exclusive
// prefix (offsets within the digit) and stores the digit total.  The digit
// starts (exclusive scan of the totals) are formed by each downsweep block.
__global__ void __launch_bounds__(kRNT) radix_scan_kernel(uint32_t* __restrict__ tile_hist,
                                                          uint32_t* __restrict__ totals, int ntiles) {
    __shared__ uint32_t ws[kRWarps];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t d = blockIdx.x;
    uint32_t* row = tile_hist + (int64_t)d * ntiles;
    const int per = (ntiles + kRNT - 1) / kRNT;  // consecutive tiles per thread
    const int lo = t * per, hi = min(ntiles, lo + per);
    uint32_t sum = 0;
    for (int i = lo; i < hi; ++i) sum += row[i];
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    uint32_t run = x - sum;
    for (int w = 0; w < warp; ++w) run += ws[w];
    if (t == kRNT - 1) totals[d] = run + sum;
    for (int i = lo; i < hi; ++i) {
        const uint32_t c = row[i];
        row[i] = run;
        run += c;
    }
}

// Stable in-tile ranking, a local sort by digit in shared memory, then the
// write-out: each digit's run of the tile goes to consecutive addresses at its
// scanned offset (coalesced segments instead of one L2 transaction per item).
template <typename K>
__global__ void __launch_bounds__(kRNT) radix_downsweep_kernel(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, bool vals_are_index, K* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n, int shift, uint32_t mask, const uint32_t* __restrict__ offs,
    const uint32_t* __restrict__ totals, uint32_t nbins, int ntiles) {
    const int bits = 31 - __clz(nbins);
    __shared__ uint32_t wcnt[kRWarps][256];
    __shared__ uint32_t s_base[256];   // global offset of digit d for this tile
    __shared__ uint32_t s_start[256];  // first local slot of digit d
    __shared__ uint32_t ws[kRWarps];
    __shared__ K sk[kRTile];
    __shared__ uint32_t sv[kRTile];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t tile = blockIdx.x;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) wcnt[w][t] = 0;
    {
        // digit start = exclusive scan of the digit totals (one digit per thread)
        const uint32_t tot = (uint32_t)t < nbins ? totals[t] : 0u;
        uint32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        uint32_t st = x - tot;
        for (int w = 0; w < warp; ++w) st += ws[w];
        s_base[t] = (uint32_t)t < nbins ? st + offs[(int64_t)t * ntiles + tile] : 0u;
    }
    __syncthreads();
    const int64_t tbase = (int64_t)tile * kRTile;
    const int64_t wbase = tbase + (int64_t)warp * kRPerWarp;
    const int tn = (int)(n - tbase < kRTile ? n - tbase : kRTile);
    const uint32_t lt = (1u << lane) - 1u;

    K key[kRIPT];
    uint32_t val[kRIPT];
    uint32_t rank[kRIPT];
#pragma unroll
    for (int r = 0; r < kRIPT; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool valid = i < n;
        key[r] = valid ? kin[i] : K(0);
        val[r] = valid ? (vals_are_index ? (uint32_t)i : vin[i]) : 0u;
    }
#pragma unroll
    for (int r = 0; r < kRIPT; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = valid ? ((uint32_t)(key[r] >> shift) & mask) : 0u;
        const uint32_t peers = digit_peers(d, bits, valid);
        const uint32_t before = valid ? wcnt[warp][d] : 0u;
        __syncwarp();
        rank[r] = before + __popc(peers & lt);
        if (valid && (peers & lt) == 0) wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // digit t: cross-warp exclusive offsets, tile total, then the tile-level
    // exclusive prefix over digits (block scan, one digit per thread)
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) {
        const uint32_t c = wcnt[w][t];
        wcnt[w][t] = total;
        total += c;
    }
    uint32_t x = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    uint32_t pre = x - total;
    for (int w = 0; w < warp; ++w) pre += ws[w];
    s_start[t] = pre;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRIPT; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        if (i < n) {
            const uint32_t d = (uint32_t)(key[r] >> shift) & mask;
            const uint32_t lp = s_start[d] + wcnt[warp][d] + rank[r];
            sk[lp] = key[r];
            sv[lp] = val[r];
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRIPT; ++r) {
        const int i = r * kRNT + t;
        if (i < tn) {
            const K kk = sk[i];
            const uint32_t d = (uint32_t)(kk >> shift) & mask;
            const uint32_t pos = s_base[d] + (uint32_t)i - s_start[d];
            RCGS_DCHECK(pos < (uint64_t)n);
            kout[pos] = kk;
            vout[pos] = sv[i];
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
    // scratch: per-pass flagged digit totals + counters (zeroed), one (digit, tile) table
    const int64_t words = (int64_t)npass * 256 + 256 * ntiles;
    uint32_t* scratch = nullptr;
    RCGS_TRY(dalloc(&scratch, words, s));
    uint32_t* totals = scratch;
    uint32_t* table = totals + npass * 256;
    // digits split evenly over the passes (e.g. 13 bits -> 7 + 6): fewer, longer
    // runs per tile in the write-out
    const int per_pass = (end_bit + npass - 1) / npass;
    int shift = 0;
    for (int p = 0; p < npass; ++p) {
        const int bits = min(per_pass, end_bit - shift);
        const uint32_t mask = (1u << bits) - 1u;
        radix_upsweep_kernel<K><<<(unsigned)ntiles, kRNT, 0, s>>>(*key_cur, n, shift, mask, table, (int)ntiles);
        radix_scan_kernel<<<1u << bits, kRNT, 0, s>>>(table, totals + p * 256, (int)ntiles);
        radix_downsweep_kernel<K><<<(unsigned)ntiles, kRNT, 0, s>>>(*key_cur, *val_cur, p == 0 && vals_are_index,
                                                                      *key_alt, *val_alt, n, shift, mask, table,
                                                                      totals + p * 256, 1u << bits, (int)ntiles);
        shift += bits;
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
