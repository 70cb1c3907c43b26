// Microbenchmark (not part of the library): streaming a bin-major u32 matrix
// [rows][ld] through shared memory with 2-D TMA boxes of different shapes,
// versus plain coalesced loads.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_bench tma_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
            sa(b)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *m, int x, int y, uint64_t *b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            sa(dst)),
        "l"((uint64_t)m), "r"(x), "r"(y), "r"(sa(b))
        : "memory");
}

// one producer lane, NC consumer warps that just sum one word per lane
__global__ void __launch_bounds__(288, 1) stream_tma(const __grid_constant__ CUtensorMap map, int ld, int rows,
                                                     int boxw, int boxh, int nst, unsigned long long *sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t *full = (uint64_t *)sm, *empty = full + nst;
    uint32_t *ring = (uint32_t *)(sm + 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int stage_words = boxw * boxh;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int xt = ld / boxw, yt = rows / boxh;
    const int items = xt * yt;
    // contiguous range of items per CTA, x fastest within a row band... iterate y inside x (bins inside sets)
    const int per = (items + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * per, i1 = min(items, i0 + per);
    if (warp == 8) {
        if (lane == 0)
            for (int n = 0; n < i1 - i0; n++) {
                const int it = i0 + n, st = n % nst, rnd = n / nst;
                if (rnd) wait(&empty[st], (rnd - 1) & 1);
                expect_tx(&full[st], stage_words * 4);
                const int x = (it / yt) * boxw, y = (it % yt) * boxh;
                tma2d(ring + st * stage_words, &map, x, y, &full[st]);
            }
        return;
    }
    unsigned long long acc = 0;
    for (int n = warp; n < i1 - i0; n += 8) {
        const int st = n % nst;
        wait(&full[st], (n / nst) & 1);
        const uint32_t *t = ring + st * stage_words;
        for (int k = lane; k < stage_words; k += 32 * 8) acc += t[k];
        __syncwarp();
        if (lane == 0) arrive(&empty[st]);
    }
    if (acc == 0x1234567) sink[0] = acc;
}

// plain loads: thread per column group, 4 rows in flight
__global__ void stream_ldg(const uint32_t *F, long ld, int rows, unsigned long long *sink) {
    unsigned long long acc = 0;
    for (long c = (blockIdx.x * (long)blockDim.x + threadIdx.x) * 4; c < ld; c += (long)gridDim.x * blockDim.x * 4)
        for (int r = 0; r < rows; r += 4) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) v[u] = __ldg((const uint4 *)(F + (long)(r + u) * ld + c));
#pragma unroll
            for (int u = 0; u < 4; u++) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
    if (acc == 0x1234567) sink[0] = acc;
}

int main() {
    const long ld = 200000, rows = 256;
    uint32_t *F;
    unsigned long long *sink;
    cudaMalloc(&F, ld * rows * 4);
    cudaMalloc(&sink, 8);
    cudaMemset(F, 1, ld * rows * 4);
    void *fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = (double)ld * rows * 4;
    {
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            stream_ldg<<<148 * 8, 256>>>(F, ld, rows, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 2) printf("ldg: %.1f us  %.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
        }
    }
    const int shapes[][2] = {{32, 32}, {64, 32}, {128, 32}, {256, 32}, {256, 8}, {64, 64}, {128, 64}, {256, 16}};
    for (auto &sh : shapes) {
        const int bw = sh[0], bh = sh[1];
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
        cuuint64_t str[1] = {(cuuint64_t)ld * 4};
        cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, F, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); continue; }
        const int stage = bw * bh * 4;
        for (int nst : {8, 16}) {
            const int smem = 1024 + nst * stage;
            if (smem > 227 * 1024) continue;
            cudaFuncSetAttribute(stream_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            float ms = 0;
            for (int rep = 0; rep < 3; rep++) {
                cudaEventRecord(e0);
                stream_tma<<<148, 288, smem>>>(m, ld, rows, bw, bh, nst, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            cudaError_t err = cudaGetLastError();
            printf("tma box %3d x %2d (%5d B) nst %2d: %.1f us  %.0f GB/s %s\n", bw, bh, stage, nst, ms * 1e3,
                   bytes / ms / 1e6, cudaGetErrorString(err));
        }
    }
    return 0;
}
