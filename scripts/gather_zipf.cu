// Row gathers (256-B rows, lane = 8 B, 16 loads in flight per warp, 2 CTAs of 8 warps per SM
// as the BITMAP scan) vs the row table's size and the rows' popularity: uniform over 2^p rows
// (8 .. 128 MB), log-uniform (Zipf(1)-like, as the query-value rows on Zipf words), and a
// window of 1/32 of a 64-MB table that moves with the loop (all warps in lockstep, or each at
// its own offset).  Row indices are power-of-two masks (no division in the loop).  Through L1
// (ld.global.nc) or L2 only (ld.global.cg).  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_zipf gather_zipf.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// MODE 0 uniform, 1 log-uniform, 2 window lockstep, 3 window scattered
template <int MODE, bool CG>
__global__ void __launch_bounds__(256) gather(const uint2 *tab, uint32_t log2rows, uint32_t per_warp,
                                              uint32_t *sink) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t h = wid * 0x9E3779B1u + 12345u, acc = 0;
    const uint32_t mask = (1u << log2rows) - 1u, wmask = (1u << (log2rows - 5)) - 1u;
    uint32_t win = MODE == 2 ? 0u : (wid * 7u) & 31u;
    const uint2 *tl = tab + lane;
    for (uint32_t i = 0; i < per_warp; i += 16) {
        uint2 r[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
            h = h * 0x2545F491u + 0x9E3779B9u;
            uint32_t row;
            if (MODE == 0) {
                row = (h >> 7) & mask;
            } else if (MODE == 1) {
                const float x = (float)(h >> 8) * (1.0f / 16777216.0f);
                row = ((uint32_t)exp2f(x * (float)log2rows) - 1u) & mask;
            } else {
                row = (win << (log2rows - 5)) | ((h >> 7) & wmask);
            }
            const uint2 *p = tl + (uint64_t)row * 32;
            if (CG) {
                asm volatile("ld.global.cg.v2.u32 {%0, %1}, [%2];" : "=r"(r[u].x), "=r"(r[u].y) : "l"(p));
            } else {
                r[u] = __ldg(p);
            }
        }
#pragma unroll
        for (int u = 0; u < 16; u++) acc ^= r[u].x ^ r[u].y;
        win = (win + 1) & 31u;
    }
    if (acc == 0x9E3779B9u) *sink = acc;
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
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *sink;
    cudaMalloc(&sink, 4);
    uint2 *tab;
    cudaMalloc(&tab, 128ull << 20);
    cudaMemset(tab, 1, 128ull << 20);
    const uint32_t per_warp = 8192;
    const int grid = nsm * 2;
    printf("{");
    bool first = true;
    auto run = [&](auto kern, const char *name, uint32_t lr) {
        float ms = time_ms([&] { kern<<<grid, 256>>>(tab, lr, per_warp, sink); }, 5);
        const double b = (double)grid * 8 * per_warp * 256;
        printf("%s\"%s_%uMB\": %.1f", first ? "" : ", ", name, (1u << lr) >> 12, b / (ms / 1e3) / 1e9);
        first = false;
    };
    for (uint32_t lr : {15u, 16u, 17u, 18u, 19u}) {  // 8 .. 128 MB
        run(gather<0, false>, "uniform_ldg", lr);
        run(gather<0, true>, "uniform_cg", lr);
    }
    for (uint32_t lr : {16u, 18u}) {
        run(gather<1, false>, "zipf_ldg", lr);
        run(gather<1, true>, "zipf_cg", lr);
        run(gather<2, false>, "window_lockstep_ldg", lr);
        run(gather<3, false>, "window_scattered_ldg", lr);
    }
    printf("}\n");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "%s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
