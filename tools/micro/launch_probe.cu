// Host cost of one kernel launch by parameter size, with and without the
// programmatic-stream-serialisation attribute (the culled path's trace and
// sampler launches carry ~0.9 KB of parameters).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/launch_probe tools/micro/launch_probe.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
struct Blob {
    float v[N / 4];
};

template <int N>
__global__ void k_blob(const Blob<N> b, float *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && b.v[0] == 12345.f) out[0] = b.v[N / 4 - 1];
}

template <int N>
void run(cudaStream_t st, float *out, bool pdl) {
    Blob<N> b = {};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    for (int i = 0; i < 200; i++) cudaLaunchKernelEx(&cfg, k_blob<N>, b, out);
    cudaStreamSynchronize(st);
    const int reps = 2000;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; i++) cudaLaunchKernelEx(&cfg, k_blob<N>, b, out);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    printf("params %5d B  pdl %d: %.2f us per launch (host)\n", N, pdl,
           std::chrono::duration<double, std::micro>(t1 - t0).count() / reps);
}

int main() {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    float *out;
    cudaMalloc(&out, 64);
    for (int pdl = 0; pdl < 2; pdl++) {
        run<64>(st, out, pdl);
        run<256>(st, out, pdl);
        run<1024>(st, out, pdl);
        run<2048>(st, out, pdl);
        run<4096>(st, out, pdl);
    }
    return 0;
}
