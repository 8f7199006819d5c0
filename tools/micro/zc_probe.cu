// PCIe write patterns into a mapped, page-locked host frame (zero-copy) against
// a device frame + cudaMemcpyAsync D2H.  Decides how the kernels should deliver
// a frame to the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/zc_probe tools/micro/zc_probe.cu
//   tools/micro/zc_probe [width height]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e = (x);                                                      \
        if (e != cudaSuccess) {                                                   \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));      \
            exit(1);                                                              \
        }                                                                         \
    } while (0)

// (a) a warp per 8x4 pixel patch, 4 B per lane: 4 x 32 B row segments per store
__global__ void patch_store(uint32_t *out, int w, int h) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;  // 128 threads = 16x8 tile
    const int x = blockIdx.x * 16 + (warp & 1) * 8 + (lane & 7);
    const int y = blockIdx.y * 8 + (warp >> 1) * 4 + (lane >> 3);
    if (x < w && y < h) out[(size_t)y * w + x] = 0xff000000u | (x * 7 + y);
}
// (b) a warp per 32 consecutive pixels of a row: 128 B per store
__global__ void row_store(uint32_t *out, int w, int h) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < (size_t)w * h) out[i] = 0xff000000u | (uint32_t)i;
}
// (c) 16 B per lane: 512 B per warp store
__global__ void row_store_v4(uint4 *out, size_t n4) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n4) out[i] = make_uint4(1, 2, 3, (uint32_t)i);
}
// (d) copy a device frame into the host frame with 16 B per lane (a copy kernel)
__global__ void copy_v4(uint4 *dst, const uint4 *src, size_t n4) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = __ldcs(src + i);
}
// (d2) the same with 4 loads in flight per thread
__global__ void copy_v4x4(uint4 *dst, const uint4 *src, size_t n4) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        uint4 a = __ldcg(src + i), b = __ldcg(src + i + stride), c = __ldcg(src + i + 2 * stride),
              d = __ldcg(src + i + 3 * stride);
        dst[i] = a;
        dst[i + stride] = b;
        dst[i + 2 * stride] = c;
        dst[i + 3 * stride] = d;
    }
    for (; i < n4; i += stride) dst[i] = __ldcg(src + i);
}
// (e) scattered 4 B stores (a sampler resolving parked pixels): every 25th pixel
__global__ void scatter_store(uint32_t *out, size_t n, int stride) {
    const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * stride;
    if (i < n) out[i] = 0xff00ff00u;
}

int main(int argc, char **argv) {
    const int w = argc > 2 ? atoi(argv[1]) : 1280, h = argc > 2 ? atoi(argv[2]) : 720;
    const size_t n = (size_t)w * h, bytes = n * 4;
    uint32_t *host, *hdev, *dev;
    CK(cudaHostAlloc(&host, bytes, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void **)&hdev, host, 0));
    CK(cudaMalloc(&dev, bytes));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto time_it = [&](const char *name, auto fn) {
        for (int i = 0; i < 5; i++) fn();
        CK(cudaStreamSynchronize(st));
        float best = 1e9, sum = 0;
        const int reps = 50;
        for (int i = 0; i < reps; i++) {
            CK(cudaEventRecord(e0, st));
            fn();
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
            sum += ms;
        }
        printf("%-44s best %7.1f us  mean %7.1f us  (%5.1f GB/s at best)\n", name, best * 1e3, sum / reps * 1e3,
               bytes / (best * 1e-3) / 1e9);
    };
    printf("frame %dx%d, %.2f MB\n", w, h, bytes / 1e6);
    {
        cudaStream_t s2[4];
        cudaEvent_t f[4];
        for (int i = 0; i < 4; i++) {
            CK(cudaStreamCreateWithFlags(&s2[i], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&f[i], cudaEventDisableTiming));
        }
        for (int k : {2, 3, 4}) {
            char name[64];
            snprintf(name, sizeof name, "cudaMemcpyAsync D2H as %d concurrent parts", k);
            time_it(name, [&] {
                CK(cudaEventRecord(f[0], st));
                for (int i = 0; i < k; i++) {
                    CK(cudaStreamWaitEvent(s2[i], f[0], 0));
                    const size_t a = bytes * i / k / 16 * 16, b = bytes * (i + 1) / k / 16 * 16;
                    CK(cudaMemcpyAsync((char *)host + a, (char *)dev + a, (i == k - 1 ? bytes : b) - a,
                                       cudaMemcpyDeviceToHost, s2[i]));
                    CK(cudaEventRecord(f[i], s2[i]));
                }
                for (int i = 0; i < k; i++) CK(cudaStreamWaitEvent(st, f[i], 0));
            });
        }
    }
    time_it("cudaMemcpyAsync D2H (pinned)", [&] { CK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st)); });
    time_it("zero-copy 8x4 patches (32 B segments)",
            [&] { patch_store<<<dim3((w + 15) / 16, (h + 7) / 8), 128, 0, st>>>(hdev, w, h); });
    time_it("zero-copy rows, 4 B/lane (128 B)", [&] { row_store<<<(n + 255) / 256, 256, 0, st>>>(hdev, w, h); });
    time_it("zero-copy rows, 16 B/lane (512 B)",
            [&] { row_store_v4<<<(n / 4 + 255) / 256, 256, 0, st>>>((uint4 *)hdev, n / 4); });
    for (int g : {148, 296, 592}) {
        char name[64];
        snprintf(name, sizeof name, "copy kernel dev->host 16 B/lane, %d CTAs", g);
        time_it(name, [&] { copy_v4<<<g, 256, 0, st>>>((uint4 *)hdev, (const uint4 *)dev, n / 4); });
    }
    for (int g : {8, 16, 32}) {
        char name[64];
        snprintf(name, sizeof name, "copy kernel dev->host 16 B/lane, %d CTAs x1024", g);
        time_it(name, [&] { copy_v4<<<g, 1024, 0, st>>>((uint4 *)hdev, (const uint4 *)dev, n / 4); });
    }
    for (int g : {1, 2, 4, 8}) {
        for (int t : {256, 512, 1024}) {
            char name[64];
            snprintf(name, sizeof name, "copy kernel x4 in flight, %d CTAs x%d", g, t);
            time_it(name, [&] { copy_v4x4<<<g, t, 0, st>>>((uint4 *)hdev, (const uint4 *)dev, n / 4); });
        }
    }
    {
        const int stride = 25;
        const size_t cnt = (n + stride - 1) / stride;
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        float best = 1e9;
        for (int i = 0; i < 50; i++) {
            CK(cudaEventRecord(a, st));
            scatter_store<<<(cnt + 255) / 256, 256, 0, st>>>(hdev, n, stride);
            CK(cudaEventRecord(b, st));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = ms < best ? ms : best;
        }
        printf("zero-copy scattered 4 B stores, %zu pixels: best %.1f us (%.0f M stores/s)\n", cnt, best * 1e3,
               cnt / (best * 1e-3) / 1e6);
    }
    return 0;
}
