// Issue-rate probe: 3-register FFMA vs paired FFMA2 (__ffma2_rn) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_rate ffma2_rate.cu   (measured on B200:
// both ~50 TFLOP/s — FFMA2 does two FMAs per issue slot at the same FMA-pipe rate)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float *out, float s, int iters) {
    float a[8], b[8];
    for (int i = 0; i < 8; i++) { a[i] = threadIdx.x * 1e-3f + i; b[i] = s * (i + 1); }
    float2 p[4], q[4], r[4];
    for (int i = 0; i < 4; i++) { p[i] = make_float2(a[2*i], a[2*i+1]); q[i] = make_float2(b[2*i], b[2*i+1]); r[i] = make_float2(s, -s); }
    for (int it = 0; it < iters; it++) {
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 8; i++) a[i] = fmaf(a[i], b[i], a[(i + 1) & 7]);
        } else {
#pragma unroll
            for (int i = 0; i < 4; i++) p[i] = __ffma2_rn(p[i], q[i], r[i]);
        }
    }
    float acc = 0.f;
    for (int i = 0; i < 8; i++) acc += a[i];
    for (int i = 0; i < 4; i++) acc += p[i].x + p[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int mode = 0; mode < 2; mode++) {
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<148 * 8, 256>>>(out, 1.0001f, iters);
            else k<1><<<148 * 8, 256>>>(out, 1.0001f, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            // FMAs executed: threads * iters * 8 (both modes do 8 lane-FMAs per iteration)
            double fmas = 148.0 * 8 * 256 * iters * 8;
            printf("%s: %.3f ms, %.1f TFLOP/s\n", mode == 0 ? "FFMA x8 " : "FFMA2 x4", ms, 2 * fmas / ms / 1e9);
        }
    }
    return 0;
}
