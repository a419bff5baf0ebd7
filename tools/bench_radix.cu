// Micro-benchmark of radix-pass building blocks on sm_100a (CUDA events, warm
// L2, 200 repetitions): histogram (upsweep) and stable warp ranking variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bench_radix tools/bench_radix.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int NT = 256, IPT = 4, TILE = NT * IPT;

__device__ __forceinline__ uint32_t ballot_match(uint32_t d) {
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const uint32_t bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

template <int V>
__global__ void __launch_bounds__(NT) up_kernel(const uint32_t* keys, int n, int shift, uint32_t* out, int ntiles) {
    __shared__ uint32_t h[256];
    const int t = threadIdx.x, lane = t & 31;
    h[t] = 0;
    __syncthreads();
    const int base = blockIdx.x * TILE;
    uint32_t k[IPT];
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const int i = base + r * NT + t;
        k[r] = i < n ? keys[i] : 0u;
    }
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const int i = base + r * NT + t;
        const uint32_t d = i < n ? (k[r] >> shift) & 255u : 256u;
        if (V == 0) {
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            if (d < 256u && lane == __ffs(peers) - 1) atomicAdd(&h[d], (uint32_t)__popc(peers));
        } else if (V == 1) {
            if (d < 256u) atomicAdd(&h[d], 1u);
        } else {
            const uint32_t peers = ballot_match(d);
            if (d < 256u && lane == __ffs(peers) - 1) atomicAdd(&h[d], (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    out[t * ntiles + blockIdx.x] = h[t];
}

template <int V>
__global__ void __launch_bounds__(NT) rank_kernel(const uint32_t* keys, int n, int shift, uint32_t* out) {
    __shared__ uint32_t wcnt[8][256];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#pragma unroll
    for (int w = 0; w < 8; ++w) wcnt[w][t] = 0;
    __syncthreads();
    const int wbase = blockIdx.x * TILE + warp * (TILE / 8);
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t k[IPT], rank[IPT];
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const int i = wbase + r * 32 + lane;
        k[r] = i < n ? keys[i] : 0u;
    }
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const int i = wbase + r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = valid ? (k[r] >> shift) & 255u : 256u;
        const uint32_t peers = V == 0 ? __match_any_sync(0xffffffffu, d) : ballot_match(d);
        const uint32_t before = valid ? wcnt[warp][d & 255u] : 0u;
        __syncwarp();
        rank[r] = before + __popc(peers & lt);
        if (valid && (peers & lt) == 0) wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
        const int i = wbase + r * 32 + lane;
        if (i < n) out[i] = rank[r];
    }
}

__global__ void copy_kernel(const uint32_t* a, uint32_t* b, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i] + 1;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(e0);
    for (int i = 0; i < 200; ++i) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1000.f / 200.f;
}

int main() {
    const int n = 909004;
    std::vector<uint32_t> h(n);
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < n; ++i) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        h[i] = (uint32_t)x;
    }
    uint32_t *d, *o, *o2;
    const int ntiles = (n + TILE - 1) / TILE;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&o, n * 4);
    cudaMalloc(&o2, 256 * ntiles * 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    printf("n=%d tiles=%d\n", n, ntiles);
    printf("copy            %7.2f us\n", timeit([&] { copy_kernel<<<(n + 255) / 256, 256>>>(d, o, n); }));
    for (int shift : {0, 24}) {
        printf("shift %d\n", shift);
        printf("  up match      %7.2f us\n", timeit([&] { up_kernel<0><<<ntiles, NT>>>(d, n, shift, o2, ntiles); }));
        printf("  up atomics    %7.2f us\n", timeit([&] { up_kernel<1><<<ntiles, NT>>>(d, n, shift, o2, ntiles); }));
        printf("  up ballot     %7.2f us\n", timeit([&] { up_kernel<2><<<ntiles, NT>>>(d, n, shift, o2, ntiles); }));
        printf("  rank match    %7.2f us\n", timeit([&] { rank_kernel<0><<<ntiles, NT>>>(d, n, shift, o); }));
        printf("  rank ballot   %7.2f us\n", timeit([&] { rank_kernel<1><<<ntiles, NT>>>(d, n, shift, o); }));
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
