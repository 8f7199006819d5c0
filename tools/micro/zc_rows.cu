// Zero-copy write patterns of the compressed frame transfer: the same bytes
// written into mapped host memory (a) as one short run per CTA at a fixed row
// stride (the encoder's layout), (b) contiguously, one CTA per run, (c)
// contiguously by a grid-stride loop of 148 x 8 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/zc_rows tools/micro/zc_rows.cu
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

__global__ void rows(unsigned *out, int run, long stride) {
    unsigned *d = out + blockIdx.x * stride;
    for (int i = threadIdx.x; i < run; i += blockDim.x) d[i] = i;
}
__global__ void contiguous_runs(unsigned *out, int run) {
    unsigned *d = out + (long)blockIdx.x * run;
    for (int i = threadIdx.x; i < run; i += blockDim.x) d[i] = i;
}
__global__ void grid_stride(unsigned *out, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) out[i] = (unsigned)i;
}

static unsigned *g_dev = nullptr;
unsigned *dsrc_dev() {
    if (!g_dev) cudaMalloc(&g_dev, 64u << 20);
    return g_dev;
}

template <typename F>
float time_us(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> t;
    for (int k = 0; k < 60; k++) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (k >= 10) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    unsigned *h, *d;
    const size_t bytes = 64u << 20;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    cudaHostGetDevicePointer((void **)&d, h, 0);
    const int rows_n[] = {720, 1080, 2160};
    const int runs[] = {116, 168, 256, 1344};
    for (int R : rows_n)
        for (int run : runs) {
            const long stride = 1344;
            const double kb = 4.0 * R * run / 1024;
            float a = time_us([&] { rows<<<R, 256>>>(d, run, stride); });
            float b = time_us([&] { contiguous_runs<<<R, 256>>>(d, run); });
            float c = time_us([&] { grid_stride<<<148 * 8, 256>>>(d, (long)R * run); });
            printf("rows %4d x %4d words (%7.1f KB): strided rows %6.1f us (%5.1f GB/s) | contiguous runs %6.1f us | grid-stride %6.1f us (%5.1f GB/s)\n",
                   R, run, kb, a, kb * 1.024e-3 / a * 1e3, b, c, kb * 1.024e-3 / c * 1e3);
        }
    float e = time_us([] {});
    printf("empty event pair %.1f us\n", e);
    // zero-copy kernel time against size (one CTA of 256 per 32 KB): the intercept is the fixed cost
    for (double kb : {0.0, 4.0, 16.0, 64.0, 128.0, 256.0, 512.0}) {
        const long n = (long)(kb * 256);
        float t = time_us([&] { grid_stride<<<std::max(1L, n / 8192), 256>>>(d, n); });
        float tr = time_us([&] { grid_stride<<<std::max(1L, n / 8192), 256>>>(dsrc_dev(), n); });
        printf("zero-copy %6.1f KB: %6.1f us   (same kernel into device memory %6.1f us)\n", kb, t, tr);
    }
    // the same sizes by the copy engine, device -> pinned host
    unsigned *dsrc;
    cudaMalloc(&dsrc, bytes);
    for (double kb : {64.0, 326.2, 489.4, 720.0, 978.8, 1417.5, 3600.0}) {
        const size_t n = (size_t)(kb * 1024);
        float t = time_us([&] { cudaMemcpyAsync(h, dsrc, n, cudaMemcpyDeviceToHost, 0); });
        printf("DMA D2H %7.1f KB: %6.1f us (%5.1f GB/s)\n", kb, t, kb * 1.024e-3 / t * 1e3);
    }
    return 0;
}
