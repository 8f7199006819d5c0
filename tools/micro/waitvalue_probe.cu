// Reaction latency of cuStreamWaitValue32 on a flag written by a running
// kernel, against an event dependency, measured with %globaltimer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/waitvalue_probe tools/micro/waitvalue_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x)                                                                \
    do {                                                                     \
        cudaError_t e = (x);                                                 \
        if (e != cudaSuccess) {                                              \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                         \
        }                                                                    \
    } while (0)

__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// spins `ns`, then (one thread) stamps t[0] and sets *flag = v
__global__ void producer(unsigned *flag, unsigned v, uint64_t ns, uint64_t *t, int mode) {
    const uint64_t t0 = gtime();
    while (gtime() - t0 < ns) {
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        t[0] = gtime();
        if (mode == 0) {
            __threadfence_system();
            atomicExch(flag, v);
        } else {
            __threadfence();
            atomicExch(flag, v);
        }
    }
}
__global__ void consumer(uint64_t *t) {
    if (threadIdx.x == 0 && blockIdx.x == 0) t[1] = gtime();
}
// keeps the SMs busy (a background kernel on the main stream)
__global__ void busy(uint64_t ns) {
    const uint64_t t0 = gtime();
    while (gtime() - t0 < ns) {
    }
}

typedef CUresult (*WaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

int main(int argc, char **argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    const int order = argc > 2 ? atoi(argv[2]) : 0;  // 1: producer enqueued before the wait
    setvbuf(stdout, nullptr, _IONBF, 0);
    printf("start\n");
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q));
    WaitFn wait = (WaitFn)p;
    unsigned *flag;
    uint64_t *t, *th;
    CK(cudaMalloc(&flag, 64));
    CK(cudaMemset(flag, 0, 64));
    CK(cudaMalloc(&t, 64));
    CK(cudaHostAlloc(&th, 64, 0));
    int least, greatest;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    cudaStream_t a, b, c;
    CK(cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, least));
    CK(cudaStreamCreateWithPriority(&b, cudaStreamNonBlocking, greatest));
    CK(cudaStreamCreateWithPriority(&c, cudaStreamNonBlocking, least));
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    unsigned v = 0;
    for (int mode = 0; mode < 4; mode++) {
        if (only >= 0 && mode != only) continue;
        // mode 0: wait-value, system fence; 1: wait-value, gpu fence; 2: event dependency;
        // 3: wait-value with the SMs kept busy by a background kernel
        double sum = 0, worst = 0;
        const int reps = 40;
        for (int r = 0; r < reps + 3; r++) {
            ++v;
            if (mode == 3) busy<<<148 * 4, 128, 0, c>>>(60000);
            if (order) producer<<<1, 32, 0, a>>>(flag, v, 20000, t, mode == 1 ? 1 : 0);
            if (mode < 2 || mode == 3) {
                if (wait(b, (CUdeviceptr)flag, v, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
                    printf("wait failed\n");
                    return 1;
                }
            }
            if (!order) producer<<<1, 32, 0, a>>>(flag, v, 20000, t, mode == 1 ? 1 : 0);
            if (mode == 2) {
                CK(cudaEventRecord(ev, a));
                CK(cudaStreamWaitEvent(b, ev, 0));
            }
            consumer<<<1, 32, 0, b>>>(t);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(th, t, 16, cudaMemcpyDeviceToHost));
            if (r >= 3) {
                const double d = (double)(th[1] - th[0]) / 1e3;
                sum += d;
                worst = d > worst ? d : worst;
            }
        }
        const char *names[] = {"waitValue, system fence", "waitValue, gpu fence", "event dependency",
                               "waitValue, SMs busy"};
        printf("%-28s flag -> dependent kernel start: mean %.2f us, worst %.2f us\n", names[mode], sum / reps, worst);
    }
    return 0;
}
