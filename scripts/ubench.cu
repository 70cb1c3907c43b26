// Microbenchmarks of the pipe and memory rates the roofline of the scoring
// kernels is stated against:
//   brute : the BRUTE scan's compare loop (ISETP + predicated IMAD per (query,
//           set, bin) equality test, 32 query values in registers) -> the
//           measured issue-bound rate of bin-compares
//   lop3  : independent LOP3 chains -> ALU-pipe lane-ops/s
//   imad  : independent IMAD chains -> FMA-pipe lane-ops/s
//   gather: warps reading random 128-B rows of an L2-resident table (lane =
//           word) -> L2 row-gather bandwidth at several table sizes
//   stream: a flat read of 4 GB -> HBM read bandwidth
// Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 1;                                                             \
        }                                                                         \
    } while (0)

__device__ __forceinline__ void acc_eq(uint32_t &c, uint32_t v, uint32_t q, uint32_t one) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, %2;\n\t@p mad.lo.u32 %0, %0, %3, %3;\n}"
                 : "+r"(c)
                 : "r"(v), "r"(q), "r"(one));
}

// 32 query values per thread, one set value per iteration (like scan_bins with B = 32, SPT = 1)
__global__ void __launch_bounds__(128) brute(uint32_t iters, uint32_t one, uint32_t *sink) {
    uint32_t q[32], c[32];
#pragma unroll
    for (int i = 0; i < 32; i++) {
        q[i] = threadIdx.x * 131u + i * 7u;
        c[i] = 0;
    }
    uint32_t v = blockIdx.x;
    for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
#pragma unroll
            for (int i = 0; i < 32; i++) acc_eq(c[i], v + u, q[i], one);
        }
        v += 4 * one;
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 32; i++) s ^= c[i];
    if (s == 0x9E3779B9u) *sink = s;
}

__global__ void __launch_bounds__(256) lop3(uint32_t iters, uint32_t k, uint32_t *sink) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x + i;
    for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 16; u++)
#pragma unroll
            for (int i = 0; i < 8; i++) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(k), "r"(it));
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= a[i];
    if (s == 0x9E3779B9u) *sink = s;
}

__global__ void __launch_bounds__(256) imad(uint32_t iters, uint32_t k, uint32_t *sink) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x + i;
    for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 16; u++)
#pragma unroll
            for (int i = 0; i < 8; i++) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(k), "r"(it));
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s ^= a[i];
    if (s == 0x9E3779B9u) *sink = s;
}

// each warp reads `per_warp` random rows of 128 B (lane = word), U rows in flight; the row
// sequence is a multiplicative walk (one IMAD per row) so the loads, not the index math,
// bound the rate
template <int U>
__global__ void __launch_bounds__(256) gather(const uint32_t *tab, uint32_t nrows_mask, uint32_t per_warp,
                                              uint32_t *sink) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t h = wid * 0x9E3779B1u + 12345u, acc = 0;
    const uint32_t *tl = tab + lane;
    for (uint32_t i = 0; i < per_warp; i += U) {
        uint32_t r[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            h = h * 0x2545F491u + 0x9E3779B9u;
            r[u] = __ldg(tl + (uint64_t)((h >> 7) & nrows_mask) * 32);
        }
#pragma unroll
        for (int u = 0; u < U; u++) acc ^= r[u];
    }
    if (acc == 0x9E3779B9u) *sink = acc;
}

// the same with 256-B rows, one 8-B load per lane (the BITMAP scan's 2,048-query rows)
template <int U>
__global__ void __launch_bounds__(256) gather2(const uint2 *tab, uint32_t nrows_mask, uint32_t per_warp,
                                               uint32_t *sink) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t h = wid * 0x9E3779B1u + 12345u, acc = 0;
    const uint2 *tl = tab + lane;
    for (uint32_t i = 0; i < per_warp; i += U) {
        uint2 r[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            h = h * 0x2545F491u + 0x9E3779B9u;
            r[u] = __ldg(tl + (uint64_t)((h >> 7) & nrows_mask) * 32);
        }
#pragma unroll
        for (int u = 0; u < U; u++) acc ^= r[u].x ^ r[u].y;
    }
    if (acc == 0x9E3779B9u) *sink = acc;
}

__global__ void stream(const uint4 *F, uint64_t n, uint32_t *sink) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 x = __ldcs(F + i);
        acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <class F>
float time_ms(F launch, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; r++) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    uint32_t *sink;
    CK(cudaMalloc(&sink, 4));
    printf("{\"sms\": %d, \"clock_khz_attr\": %d", nsm, clk);

    {   // brute compare loop: 4 CTAs x 128 threads per SM (the scan's occupancy at B = 32)
        const uint32_t iters = 4096;
        const int grid = nsm * 4 * 8;
        float ms = time_ms([&] { brute<<<grid, 128>>>(iters, 1u, sink); }, 5);
        const double cmp = (double)grid * 128 * iters * 4 * 32;
        printf(", \"brute_compares_per_s\": %.6e, \"brute_ms\": %.3f", cmp / (ms / 1e3), ms);
    }
    {
        const uint32_t iters = 8192;
        const int grid = nsm * 8;
        float ms = time_ms([&] { lop3<<<grid, 256>>>(iters, 0x1234567u, sink); }, 5);
        const double ops = (double)grid * 256 * iters * 16 * 8;
        printf(", \"lop3_lane_ops_per_s\": %.6e", ops / (ms / 1e3));
        ms = time_ms([&] { imad<<<grid, 256>>>(iters, 0x1234567u, sink); }, 5);
        printf(", \"imad_lane_ops_per_s\": %.6e", ops / (ms / 1e3));
    }
    {   // L2 / L1 row gathers
        const uint64_t max_bytes = 256ull << 20;
        uint32_t *tab;
        CK(cudaMalloc(&tab, max_bytes));
        CK(cudaMemset(tab, 1, max_bytes));
        const uint32_t per_warp = 2048;
        const int grid = nsm * 8;
        printf(", \"gather_128B_rows_GBps\": {");
        const uint64_t sizes[] = {64ull << 10, 1ull << 20, 16ull << 20, 64ull << 20, 256ull << 20};
        for (int i = 0; i < 5; i++) {
            const uint32_t nrows = (uint32_t)(sizes[i] / 128);
            float ms = time_ms([&] { gather<16><<<grid, 256>>>(tab, nrows - 1, per_warp, sink); }, 5);
            const double bytes = (double)grid * 8 * per_warp * 128;
            printf("%s\"%llu\": %.1f", i ? ", " : "", (unsigned long long)sizes[i], bytes / (ms / 1e3) / 1e9);
        }
        printf("}, \"gather_256B_rows_GBps\": {");
        for (int i = 0; i < 5; i++) {
            const uint32_t nrows = (uint32_t)(sizes[i] / 256);
            float ms = time_ms([&] { gather2<16><<<grid, 256>>>((const uint2 *)tab, nrows - 1, per_warp, sink); }, 5);
            const double bytes = (double)grid * 8 * per_warp * 256;
            printf("%s\"%llu\": %.1f", i ? ", " : "", (unsigned long long)sizes[i], bytes / (ms / 1e3) / 1e9);
        }
        printf("}");
        CK(cudaFree(tab));
    }
    {
        const uint64_t bytes = 4ull << 30;
        uint4 *F;
        CK(cudaMalloc(&F, bytes));
        CK(cudaMemset(F, 0, bytes));
        float ms = time_ms([&] { stream<<<nsm * 8, 512>>>(F, bytes / 16, sink); }, 5);
        printf(", \"hbm_read_GBps\": %.1f", (double)bytes / (ms / 1e3) / 1e9);
        CK(cudaFree(F));
    }
    printf("}\n");
    return 0;
}
