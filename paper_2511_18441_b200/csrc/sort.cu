// Device scan (reduce-then-scan) and the library's error/allocation helpers.
// The radix sort lives in radix.cu.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include <cstdlib>

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
        // blocks freed on one stream may be reused by another only once the free
        // has completed: with internal dependencies the pool would make the main
        // stream wait on a builder stream's queued work (or vice versa)
        static const bool internal = getenv("RCGS_POOL_INTERNAL_DEPS") != nullptr;
        int allow = internal ? 1 : 0;
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &allow);
    }
    done_dev = dev;
}

int pool_reserve(int64_t bytes, cudaStream_t s) {
    retain_pool_memory();
    // several moderate blocks (the pool sub-allocates from freed blocks)
    const int64_t chunk = (int64_t)256 << 20;
    const int64_t n = (bytes + chunk - 1) / chunk;
    void* ptrs[4096];
    int64_t got = 0;
    for (; got < n && got < 4096; ++got) {
        if (cudaMallocAsync(&ptrs[got], chunk, s) != cudaSuccess) {
            cudaGetLastError();
            break;
        }
    }
    for (int64_t i = 0; i < got; ++i) cudaFreeAsync(ptrs[i], s);
    RCGS_CUDA(cudaStreamSynchronize(s));
    return RCGS_OK;
}

// Per-thread pinned staging for small device->host reads.  Builder threads come
// and go (one pair per prefetcher), so the buffer is released when its thread
// exits instead of leaking one pinned page per thread.
namespace {
struct PinnedScratch {
    void* buf = nullptr;
    size_t cap = 0;
    ~PinnedScratch() {
        if (buf) cudaFreeHost(buf);  // errors at process teardown are irrelevant
    }
};
}  // namespace

void* pinned_scratch(size_t bytes) {
    static thread_local PinnedScratch ps;
    if (bytes > ps.cap) {
        if (ps.buf) cudaFreeHost(ps.buf);
        ps.buf = nullptr;
        ps.cap = 0;
        if (cudaMallocHost(&ps.buf, bytes) != cudaSuccess) return nullptr;
        ps.cap = bytes;
    }
    return ps.buf;
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

}  // namespace rcgs

extern "C" const char* rcgs_last_error(void) { return rcgs::last_error(); }
extern "C" int rcgs_version(void) { return RCGS_VERSION; }

#ifdef RCGS_CHECKED
#include <vector>
namespace rcgs {
static std::vector<unsigned long long (*)(bool)>& violation_readers() {
    static std::vector<unsigned long long (*)(bool)> v;
    return v;
}
void register_violation_reader(unsigned long long (*fn)(bool)) { violation_readers().push_back(fn); }
}  // namespace rcgs
#endif

#ifdef RCGS_CHECKED
namespace rcgs {
__global__ void debug_selftest_kernel(int fail) { RCGS_DCHECK(fail == 0); }
}  // namespace rcgs
#endif

// Checked builds: one deliberate check (fail != 0 counts one violation), to
// prove the counter works before a suite run relies on it reading zero.
extern "C" int rcgs_debug_selftest(int fail) {
#ifdef RCGS_CHECKED
    rcgs::debug_selftest_kernel<<<1, 1>>>(fail);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
#else
    (void)fail;
    RCGS_CHECK_ARG(false, "release build: no device checks");
#endif
}

// Checked builds: device bound-check failures since the last reset (and reset
// them when reset != 0); returns RCGS_EINVAL in release builds, which have no checks.
extern "C" int rcgs_debug_violations(uint64_t* h_count, int reset) {
    RCGS_CHECK_ARG(h_count != nullptr, "null argument");
#ifdef RCGS_CHECKED
    RCGS_CUDA(cudaDeviceSynchronize());
    unsigned long long v = 0;
    for (auto fn : rcgs::violation_readers()) v += fn(reset != 0);
    *h_count = v;
    return RCGS_OK;
#else
    (void)reset;
    *h_count = 0;
    RCGS_CHECK_ARG(false, "release build: no device checks (build with EXTRA=-DRCGS_CHECKED)");
#endif
}

extern "C" int rcgs_pool_reserve(int64_t bytes, void* stream) {
    RCGS_CHECK_ARG(bytes >= 0, "negative size");
    return rcgs::pool_reserve(bytes, rcgs::as_stream(stream));
}
