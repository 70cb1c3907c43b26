// Bandwidth of the bin-major collection read patterns (no compute): a
// [rows][ld] uint32 matrix read by CTAs that each own a column strip of
// `strip` bytes and walk every row with U row loads in flight per thread.
// Measures how DRAM bandwidth depends on the strip width (the contiguous run
// each CTA reads per row) and on the bytes in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o access_bench access_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int VEC, int U>
__global__ void strips(const uint32_t *F, uint64_t ld, uint32_t rows, uint64_t ncols, uint32_t *sink) {
    // CTA strip = blockDim.x * VEC columns; grid-stride over strips
    const uint64_t strip_cols = (uint64_t)blockDim.x * VEC;
    const uint64_t nstrip = ncols / strip_cols;
    uint32_t acc = 0;
    for (uint64_t st = blockIdx.x; st < nstrip; st += gridDim.x) {
        const uint32_t *p = F + st * strip_cols + threadIdx.x * VEC;
        for (uint32_t r = 0; r < rows; r += U) {
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (VEC == 4) {
                    const uint4 x = __ldcs(reinterpret_cast<const uint4 *>(p + (uint64_t)(r + u) * ld));
                    acc ^= x.x ^ x.y ^ x.z ^ x.w;
                } else if (VEC == 2) {
                    const uint2 x = __ldcs(reinterpret_cast<const uint2 *>(p + (uint64_t)(r + u) * ld));
                    acc ^= x.x ^ x.y;
                } else {
                    acc ^= __ldcs(p + (uint64_t)(r + u) * ld);
                }
            }
        }
    }
    if (acc == 0x12345678u) *sink = acc;
}

__global__ void flat(const uint4 *F, uint64_t n, uint32_t *sink) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 x = __ldcs(F + i);
        acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <int VEC, int U>
void run(const uint32_t *F, uint64_t ld, uint32_t rows, uint32_t *sink, int threads, int ctas_per_sm) {
    const uint64_t strip_cols = (uint64_t)threads * VEC;
    const uint64_t ncols = ld / strip_cols * strip_cols;
    int nsm = 148;
    const int grid = nsm * ctas_per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    strips<VEC, U><<<grid, threads>>>(F, ld, rows, ncols, sink);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int i = 0; i < reps; i++) strips<VEC, U><<<grid, threads>>>(F, ld, rows, ncols, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)ncols * rows * 4;
    printf("{\"vec\": %d, \"U\": %d, \"threads\": %d, \"ctas_per_sm\": %d, \"strip_bytes\": %llu, \"GBps\": %.1f}\n", VEC, U,
           threads, ctas_per_sm, (unsigned long long)(strip_cols * 4), bytes * reps / (ms * 1e-3) / 1e9);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
}

int main() {
    const uint32_t rows = 512;
    const uint64_t ld = 1000064;  // the image-like collection: 10^6 sets x 512 bins (2.05 GB)
    uint32_t *F, *sink;
    cudaMalloc(&F, (size_t)rows * ld * 4);
    cudaMalloc(&sink, 4);
    cudaMemset(F, 1, (size_t)rows * ld * 4);
    {
        const uint64_t n = (uint64_t)rows * ld / 4;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        flat<<<148 * 8, 256>>>(reinterpret_cast<const uint4 *>(F), n, sink);
        cudaEventRecord(e0);
        for (int i = 0; i < 5; i++) flat<<<148 * 8, 256>>>(reinterpret_cast<const uint4 *>(F), n, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"flat\": 1, \"GBps\": %.1f}\n", (double)n * 16 * 5 / (ms * 1e-3) / 1e9);
    }
    // the BRUTE scan's pattern (128 threads x uint2 = 1 KB strips), then wider strips / more in flight
    for (int cps : {3, 6, 8}) {
        run<2, 4>(F, ld, rows, sink, 128, cps);
        run<2, 8>(F, ld, rows, sink, 128, cps);
        run<2, 16>(F, ld, rows, sink, 128, cps);
        run<4, 4>(F, ld, rows, sink, 128, cps);
        run<4, 8>(F, ld, rows, sink, 128, cps);
        run<4, 16>(F, ld, rows, sink, 128, cps);
    }
    for (int cps : {2, 4}) {
        run<4, 4>(F, ld, rows, sink, 256, cps);
        run<4, 8>(F, ld, rows, sink, 256, cps);
        run<4, 8>(F, ld, rows, sink, 512, cps / 2);
        run<4, 4>(F, ld, rows, sink, 1024, 1);
    }
    return 0;
}
