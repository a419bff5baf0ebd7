// Micro-benchmark of a segmented (key u64, val u32) sort with C3-like segment
// lengths: warp bitonic sorts of 32-element runs (shuffles) + merge-path rounds in
// shared memory, one CTA per segment.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/bench_segsort.cu -o tools/_bench_segsort && tools/_bench_segsort
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cstring>
#include <functional>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

struct KV { uint64_t k; uint32_t v; };
__device__ __forceinline__ bool kv_less(uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
    return ka < kb || (ka == kb && va < vb);
}

// one warp sorts 32 (key, val) in registers (lane i holds element i), ascending
__device__ __forceinline__ void warp_bitonic32(uint64_t& k, uint32_t& v, int lane) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const uint64_t ok = __shfl_xor_sync(0xffffffffu, k, stride);
            const uint32_t ov = __shfl_xor_sync(0xffffffffu, v, stride);
            const bool up = (lane & size) == 0;
            const bool lower = (lane & stride) == 0;
            // the lower lane keeps the min when ascending
            const bool other_less = kv_less(ok, ov, k, v);
            const bool take = (lower == up) ? other_less : !other_less;
            if (take) { k = ok; v = ov; }
        }
    }
}

// merge path: number of elements taken from a (len na) among the first d outputs of merge(a, b)
__device__ __forceinline__ int merge_split(const uint64_t* ak, const uint32_t* av, int na, const uint64_t* bk,
                                           const uint32_t* bv, int nb, int d) {
    int lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        // take a[m] before b[d - 1 - m]?  stable: a first on ties (a precedes b)
        if (!kv_less(bk[d - 1 - m], bv[d - 1 - m], ak[m], av[m])) lo = m + 1; else hi = m;
    }
    return lo;
}

template <int NT>
__global__ void __launch_bounds__(NT) segsort_kernel(const uint32_t* __restrict__ seg_off, int nseg,
                                                     uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                     uint32_t lo_len, uint32_t hi_len, int cap) {
    extern __shared__ __align__(16) unsigned char smraw[];
    uint64_t* skb = reinterpret_cast<uint64_t*>(smraw);
    uint32_t* svb = reinterpret_cast<uint32_t*>(skb + 2 * cap);
    uint64_t* sk[2] = {skb, skb + cap};
    uint32_t* sv[2] = {svb, svb + cap};
    const int seg = blockIdx.x;
    const uint32_t x0 = seg_off[seg], len = seg_off[seg + 1] - x0;
    if (len <= lo_len || len > hi_len) return;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int np2 = 32;
    while (np2 < (int)len) np2 <<= 1;
    // load + warp-sort 32-element runs
    for (int c = warp * 32; c < np2; c += NT) {
        const int i = c + lane;
        uint64_t k = ~0ull;
        uint32_t v = 0xffffffffu;
        if (i < (int)len) { k = keys[x0 + i]; v = vals[x0 + i]; }
        warp_bitonic32(k, v, lane);
        sk[0][i] = k;
        sv[0][i] = v;
    }
    __syncthreads();
    int src = 0;
    for (int run = 32; run < np2; run <<= 1) {
        // each thread writes E consecutive outputs of one merged pair
        const int E = np2 / NT > 0 ? np2 / NT : 1;
        for (int o0 = t * E; o0 < np2; o0 += NT * E) {
            const int pair = o0 / (2 * run), base = pair * 2 * run, d = o0 - base;
            const uint64_t* ak = sk[src] + base; const uint32_t* av = sv[src] + base;
            const uint64_t* bk = ak + run; const uint32_t* bv = av + run;
            int ia = merge_split(ak, av, run, bk, bv, run, d), ib = d - ia;
            for (int e = 0; e < E && d + e < 2 * run; ++e) {
                bool takeA;
                if (ia >= run) takeA = false;
                else if (ib >= run) takeA = true;
                else takeA = !kv_less(bk[ib], bv[ib], ak[ia], av[ia]);
                if (takeA) { sk[src ^ 1][base + d + e] = ak[ia]; sv[src ^ 1][base + d + e] = av[ia]; ++ia; }
                else { sk[src ^ 1][base + d + e] = bk[ib]; sv[src ^ 1][base + d + e] = bv[ib]; ++ib; }
            }
        }
        src ^= 1;
        __syncthreads();
    }
    for (int i = t; i < (int)len; i += NT) { keys[x0 + i] = sk[src][i]; vals[x0 + i] = sv[src][i]; }
}

int main() {
    std::mt19937_64 rng(1);
    const int nseg = 8160;
    std::vector<uint32_t> off(nseg + 1, 0);
    std::lognormal_distribution<double> ld(5.3, 0.9);
    std::vector<int> lens(nseg);
    for (int i = 0; i < nseg; ++i) {
        int L = (int)ld(rng);
        if (L > 4470) L = 4470;
        lens[i] = L;
    }
    std::sort(lens.begin(), lens.end(), std::greater<int>());  // heaviest first, as the work order
    for (int i = 0; i < nseg; ++i) off[i + 1] = off[i] + lens[i];
    const uint32_t n = off[nseg];
    int maxlen = 0; for (int i = 0; i < nseg; ++i) maxlen = std::max(maxlen, (int)(off[i + 1] - off[i]));
    printf("segments %d, entries %u, mean %.1f, max %d\n", nseg, n, (double)n / nseg, maxlen);
    std::vector<uint64_t> hk(n); std::vector<uint32_t> hv(n);
    std::uniform_real_distribution<double> zd(1.0, 6.0);
    for (uint32_t i = 0; i < n; ++i) { double z = zd(rng); if (i % 7 == 0 && i) z = *(double*)&hk[i - 1]; memcpy(&hk[i], &z, 8); hv[i] = i; }
    uint32_t* doff; uint64_t* dk; uint32_t* dv;
    CK(cudaMalloc(&doff, (nseg + 1) * 4)); CK(cudaMalloc(&dk, n * 8)); CK(cudaMalloc(&dv, n * 4));
    CK(cudaMemcpy(doff, off.data(), (nseg + 1) * 4, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    CK(cudaFuncSetAttribute(segsort_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 24));
    // the large segments first (as in the work order): launch only their CTAs
    int nlarge = 0;
    while (nlarge < nseg && off[nlarge + 1] - off[nlarge] > 1024) ++nlarge;
    printf("segments over 1024: %d\n", nlarge);
    float best = 1e9, bs = 1e9, bl = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
        CK(cudaMemcpy(dk, hk.data(), n * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dv, hv.data(), n * 4, cudaMemcpyHostToDevice));
        cudaEventRecord(e0);
        segsort_kernel<256><<<nseg, 256, 1024 * 24>>>(doff, nseg, dk, dv, 0, 1024, 1024);
        cudaEventRecord(e1); cudaEventSynchronize(e1); float ms1; cudaEventElapsedTime(&ms1, e0, e1);
        cudaEventRecord(e0);
        segsort_kernel<1024><<<nlarge, 1024, 8192 * 24>>>(doff, nseg, dk, dv, 1024, 8192, 8192);
        cudaEventRecord(e1); cudaEventSynchronize(e1); float ms2; cudaEventElapsedTime(&ms2, e0, e1);
        CK(cudaGetLastError());
        bs = std::min(bs, ms1); bl = std::min(bl, ms2); best = std::min(best, ms1 + ms2);
    }
    // verify
    std::vector<uint64_t> rk(n); std::vector<uint32_t> rv(n);
    CK(cudaMemcpy(rk.data(), dk, n * 8, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(rv.data(), dv, n * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int s = 0; s < nseg; ++s) {
        std::vector<std::pair<uint64_t, uint32_t>> ref;
        for (uint32_t i = off[s]; i < off[s + 1]; ++i) ref.push_back({hk[i], hv[i]});
        std::sort(ref.begin(), ref.end());
        for (uint32_t i = off[s]; i < off[s + 1]; ++i) bad += (rk[i] != ref[i - off[s]].first || rv[i] != ref[i - off[s]].second);
    }
    printf("small %.1f us, large %.1f us, total %.1f us, mismatches %ld\n", bs * 1e3, bl * 1e3, best * 1e3, bad);
    return 0;
}
