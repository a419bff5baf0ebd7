// Device scan and stable LSD radix sort (hand-written; no CUB).
//
// Used for (a) the global front-to-back order of the kept gaussians: a stable
// sort of the fp64 view-space z bit patterns (positive doubles order like their
// uint64 bits), ties by scene index -- np.argsort(z, kind="stable") at
// render.py:216 -- and (b) the stable (tile | depth) pair sort: pairs are emitted
// in depth-rank order, so a stable sort on the tile id alone yields
// (tile, depth) order.
//
// One pass = histogram (per 4096-item block, digit-major counts) -> exclusive
// scan of the digit-major count table -> stable scatter.  Within a block the
// items are ranked round by round (256 items per round, warp match_any for
// intra-warp ranks, a per-digit prefix across the 8 warps), preserving input
// order for equal digits.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace rcgs {

static thread_local char g_err[1024];

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

const char* last_error() { return g_err; }

void retain_pool_memory() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}

void* pinned_scratch(size_t bytes) {
    static thread_local void* buf = nullptr;
    static thread_local size_t cap = 0;
    if (bytes > cap) {
        if (buf) cudaFreeHost(buf);
        buf = nullptr;
        cap = 0;
        if (cudaMallocHost(&buf, bytes) != cudaSuccess) return nullptr;
        cap = bytes;
    }
    return buf;
}

// ---------------------------------------------------------------- block scan
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums,
                                                         uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NW ? warp_sums[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NW) warp_sums[lane] = w;
    }
    __syncthreads();
    uint32_t excl = x - v + (warp > 0 ? warp_sums[warp - 1] : 0u);
    *total = warp_sums[NW - 1];
    __syncthreads();
    return excl;
}

constexpr int kScanNT = 1024;
constexpr int kScanIPT = 4;
constexpr int kScanTile = kScanNT * kScanIPT;

__global__ void scan_reduce_kernel(const uint32_t* __restrict__ in, int64_t n,
                                   uint32_t* __restrict__ block_sums) {
    __shared__ uint32_t ws[32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIPT;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i)
        if (base + i < n) s += in[base + i];
    uint32_t total;
    block_exclusive_scan<kScanNT>(s, ws, &total);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

// Single block: exclusive scan of the block sums in place (any length).
__global__ void scan_spine_kernel(uint32_t* __restrict__ sums, int64_t nb) {
    __shared__ uint32_t ws[32];
    uint32_t carry = 0;
    for (int64_t start = 0; start < nb; start += kScanNT) {
        int64_t i = start + threadIdx.x;
        uint32_t v = i < nb ? sums[i] : 0u;
        uint32_t total;
        uint32_t e = block_exclusive_scan<kScanNT>(v, ws, &total);
        if (i < nb) sums[i] = carry + e;
        carry += total;
    }
}

__global__ void scan_apply_kernel(const uint32_t* __restrict__ in, int64_t n,
                                  const uint32_t* __restrict__ block_offs,
                                  uint32_t* __restrict__ out) {
    __shared__ uint32_t ws[32];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIPT;
    uint32_t v[kScanIPT];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i) {
        v[i] = base + i < n ? in[base + i] : 0u;
        s += v[i];
    }
    uint32_t total;
    uint32_t e = block_exclusive_scan<kScanNT>(s, ws, &total) + block_offs[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i) {
        if (base + i < n) out[base + i] = e;
        e += v[i];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanNT - 1) out[n] = e;
}

int exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t s) {
    if (n == 0) {
        RCGS_CUDA(cudaMemsetAsync(out, 0, sizeof(uint32_t), s));
        return RCGS_OK;
    }
    unsigned nb = div_up(n, kScanTile);
    uint32_t* sums = nullptr;
    RCGS_TRY(dalloc(&sums, nb, s));
    scan_reduce_kernel<<<nb, kScanNT, 0, s>>>(in, n, sums);
    scan_spine_kernel<<<1, kScanNT, 0, s>>>(sums, nb);
    scan_apply_kernel<<<nb, kScanNT, 0, s>>>(in, n, sums, out);
    dfree(sums, s);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

// ---------------------------------------------------------------- radix sort
constexpr int kSortNT = 256;
constexpr int kSortRounds = 16;
constexpr int kSortTile = kSortNT * kSortRounds;  // 4096 items per block
constexpr int kRadix = 256;

template <typename K>
__global__ void radix_hist_kernel(const K* __restrict__ keys, int64_t n, int shift, uint32_t mask,
                                  uint32_t* __restrict__ counts, int nblocks) {
    __shared__ uint32_t hist[kRadix];
    hist[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll 4
    for (int r = 0; r < kSortRounds; ++r) {
        int64_t i = base + r * kSortNT + threadIdx.x;
        if (i < n) atomicAdd(&hist[(uint32_t)(keys[i] >> shift) & mask], 1u);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * nblocks + blockIdx.x] = hist[threadIdx.x];
}

template <typename K>
__global__ void __launch_bounds__(kSortNT) radix_scatter_kernel(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, bool vals_are_index,
    K* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int64_t n, int shift, uint32_t mask,
    const uint32_t* __restrict__ offsets, int nblocks) {
    __shared__ uint32_t base_of[kRadix];
    __shared__ uint32_t warp_cnt[kSortNT / 32][kRadix];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    base_of[t] = offsets[(int64_t)t * nblocks + blockIdx.x];
    const uint32_t lt_mask = (1u << lane) - 1u;
    int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
        int64_t i = base + r * kSortNT + t;
        if (base + r * kSortNT >= n) break;  // uniform across the block
        bool valid = i < n;
        K key = valid ? keys_in[i] : K(0);
        uint32_t val = valid ? (vals_are_index ? (uint32_t)i : vals_in[i]) : 0u;
        uint32_t d = valid ? ((uint32_t)(key >> shift) & mask) : 0x100u;
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t rank_in = __popc(peers & lt_mask);
#pragma unroll
        for (int w = 0; w < kSortNT / 32; ++w) warp_cnt[w][t] = 0;
        __syncthreads();
        if (valid && rank_in == 0) warp_cnt[warp][d] = __popc(peers);
        __syncthreads();
        {
            uint32_t run = base_of[t];
#pragma unroll
            for (int w = 0; w < kSortNT / 32; ++w) {
                uint32_t c = warp_cnt[w][t];
                warp_cnt[w][t] = run;
                run += c;
            }
            base_of[t] = run;
        }
        __syncthreads();
        if (valid) {
            uint32_t pos = warp_cnt[warp][d] + rank_in;
            keys_out[pos] = key;
            vals_out[pos] = val;
        }
        __syncthreads();
    }
}

template <typename K>
static int radix_sort(K** key_cur, K** key_alt, uint32_t** val_cur, uint32_t** val_alt,
                      bool vals_are_index, int64_t n, int end_bit, cudaStream_t s) {
    if (n <= 0 || end_bit <= 0) {
        if (vals_are_index && n > 0) {
            // identity permutation still has to materialise the values
            // (handled by the caller via a pass with end_bit >= 1)
        }
        return RCGS_OK;
    }
    RCGS_CHECK_ARG(n < (int64_t)0xffffffffLL, "radix sort: %lld items exceeds uint32 indexing",
                   (long long)n);
    int nblocks = (int)div_up(n, kSortTile);
    uint32_t *counts = nullptr, *offs = nullptr;
    int64_t ncount = (int64_t)kRadix * nblocks;
    RCGS_TRY(dalloc(&counts, ncount, s));
    RCGS_TRY(dalloc(&offs, ncount + 1, s));
    bool first = true;
    for (int shift = 0; shift < end_bit; shift += 8) {
        int bits = end_bit - shift < 8 ? end_bit - shift : 8;
        uint32_t mask = (1u << bits) - 1u;
        radix_hist_kernel<K><<<nblocks, kSortNT, 0, s>>>(*key_cur, n, shift, mask, counts, nblocks);
        RCGS_TRY(exclusive_scan_u32(counts, offs, ncount, s));
        radix_scatter_kernel<K><<<nblocks, kSortNT, 0, s>>>(*key_cur, *val_cur,
                                                            first && vals_are_index, *key_alt,
                                                            *val_alt, n, shift, mask, offs, nblocks);
        RCGS_LAUNCH_CHECK();
        K* tk = *key_cur; *key_cur = *key_alt; *key_alt = tk;
        uint32_t* tv = *val_cur; *val_cur = *val_alt; *val_alt = tv;
        first = false;
    }
    dfree(counts, s);
    dfree(offs, s);
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

extern "C" const char* rcgs_last_error(void) { return rcgs::last_error(); }
extern "C" int rcgs_version(void) { return RCGS_VERSION; }
