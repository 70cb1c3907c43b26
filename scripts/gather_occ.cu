// Random 256-B row gathers from a 16-MB L2-resident table (lane = 8 B) at several
// occupancies (CTAs of 8 warps per SM) and loads in flight per warp (U): how many bytes in
// flight the BITMAP scan needs to approach the gather peak.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_occ gather_occ.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

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

// the same through cp.async (16 B per lane, two rows per instruction) into a per-warp smem
// ring of S slots of 16 rows; the warp reads each landed slot back (LDS.64) like the scan
template <int S>
__global__ void __launch_bounds__(256) gather_cp(const uint4 *tab, uint32_t nrows_mask, uint32_t per_warp,
                                                 uint32_t *sink) {
    extern __shared__ __align__(16) uint4 ring[];  // [8 warps][S][16 rows][16 uint4]
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint4 *my = ring + (size_t)warp * S * 256;
    uint32_t h = wid * 0x9E3779B1u + 12345u, acc = 0;
    auto issue = [&](uint32_t slot) {
#pragma unroll
        for (int u = 0; u < 8; u++) {  // rows 2u, 2u+1: lanes 0-15 / 16-31
            h = h * 0x2545F491u + 0x9E3779B9u;
            const uint32_t r0 = (h >> 7) & nrows_mask;
            h = h * 0x2545F491u + 0x9E3779B9u;
            const uint32_t r1 = (h >> 7) & nrows_mask;
            const uint32_t r = lane < 16 ? r0 : r1;
            const uint4 *src = tab + (uint64_t)r * 16 + (lane & 15);
            uint4 *dst = my + slot * 256 + (2 * u + (lane >> 4)) * 16 + (lane & 15);
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const uint32_t nb = per_warp / 16;
    for (uint32_t i = 0; i < S - 1 && i < nb; i++) issue(i);
    for (uint32_t i = 0; i < nb; i++) {
        if (i + S - 1 < nb) issue((i + S - 1) % S);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
        __syncwarp();
        const uint2 *sl = reinterpret_cast<const uint2 *>(my + (i % S) * 256);
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const uint2 y = sl[u * 32 + lane];
            acc ^= y.x ^ y.y;
        }
        __syncwarp();
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
    const uint64_t bytes = 16ull << 20;
    uint32_t *tab;
    cudaMalloc(&tab, bytes);
    cudaMemset(tab, 1, bytes);
    const uint32_t nrows = (uint32_t)(bytes / 256), per_warp = 4096;
    printf("{\"ldg\": {");
    const int ctas[] = {1, 2, 3, 4, 8};
    bool first = true;
    for (int c : ctas) {
        const int grid = nsm * c * 4;
        auto run = [&](auto kern, const char *name) {
            float ms = time_ms([&] { kern<<<grid, 256>>>((const uint2 *)tab, nrows - 1, per_warp, sink); }, 5);
            const double b = (double)grid * 8 * per_warp * 256;
            printf("%s\"%s_ctas%d\": %.1f", first ? "" : ", ", name, c, b / (ms / 1e3) / 1e9);
            first = false;
        };
        run(gather2<8>, "U8");
        run(gather2<16>, "U16");
        run(gather2<32>, "U32");
    }
    printf("}, \"cp_async\": {");
    first = true;
    for (int c : {1, 2, 3}) {
        const int grid = nsm * c * 4;
        auto run = [&](auto kern, int S) {
            const size_t smem = (size_t)8 * S * 4096;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            float ms = time_ms([&] { kern<<<grid, 256, smem>>>((const uint4 *)tab, nrows - 1, per_warp, sink); }, 5);
            const double b = (double)grid * 8 * per_warp * 256;
            printf("%s\"S%d_ctas%d\": %.1f", first ? "" : ", ", S, c, b / (ms / 1e3) / 1e9);
            first = false;
        };
        if (c <= 3) run(gather_cp<2>, 2);
        if (c <= 2) run(gather_cp<3>, 3);
        if (c <= 1) run(gather_cp<4>, 4);
        if (c <= 1) run(gather_cp<6>, 6);
    }
    printf("}}\n");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "%s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
