// Host-side cost of detecting an in-place skybox edit (25 MB of float32
// texels): bitwise compare against a kept copy (reads 2x the bytes) vs a
// 128-bit hash of the caller's array alone, over T OpenMP threads.
//   gcc -O3 -march=native -fopenmp -o tools/micro/host_hash tools/micro/host_hash.c
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + 1e-9 * t.tv_nsec;
}

static inline uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v * 0x9E3779B97F4A7C15ull;
    h = (h << 31) | (h >> 33);
    return h * 0xC2B2AE3D27D4EB4Full;
}

// two 64-bit lanes per 16 bytes, 4 independent accumulator pairs
static void hash_chunk(const uint64_t *p, size_t n, uint64_t out[2]) {
    uint64_t a0 = 1, a1 = 2, a2 = 3, a3 = 4, b0 = 5, b1 = 6, b2 = 7, b3 = 8;
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        a0 = mix(a0, p[i]);
        b0 = mix(b0, p[i + 1] ^ 0x5555);
        a1 = mix(a1, p[i + 2]);
        b1 = mix(b1, p[i + 3] ^ 0x5555);
        a2 = mix(a2, p[i + 4]);
        b2 = mix(b2, p[i + 5] ^ 0x5555);
        a3 = mix(a3, p[i + 6]);
        b3 = mix(b3, p[i + 7] ^ 0x5555);
    }
    for (; i < n; i++) a0 = mix(a0, p[i]);
    out[0] = mix(mix(mix(a0, a1), a2), a3);
    out[1] = mix(mix(mix(b0, b1), b2), b3);
}

int main(void) {
    const size_t bytes = (size_t)2048 * 1024 * 3 * 4;
    uint64_t *a = aligned_alloc(64, bytes), *b = aligned_alloc(64, bytes);
    memset(a, 1, bytes);
    memcpy(b, a, bytes);
    printf("procs %d, %zu MB\n", omp_get_num_procs(), bytes >> 20);
    for (int t = 1; t <= omp_get_num_procs(); t *= 2) {
        double best_c = 1e9, best_h = 1e9;
        for (int rep = 0; rep < 20; rep++) {
            double t0 = now();
            int diff = 0;
#pragma omp parallel for num_threads(t) reduction(| : diff)
            for (int k = 0; k < 4 * t; k++) {
                size_t lo = bytes * k / (4 * t), hi = bytes * (k + 1) / (4 * t);
                diff |= memcmp((char *)a + lo, (char *)b + lo, hi - lo) != 0;
            }
            double t1 = now();
            uint64_t acc0 = 0, acc1 = 0;
#pragma omp parallel for num_threads(t) reduction(^ : acc0, acc1)
            for (int k = 0; k < 4 * t; k++) {
                size_t lo = bytes / 8 * k / (4 * t), hi = bytes / 8 * (k + 1) / (4 * t);
                uint64_t h[2];
                hash_chunk(a + lo, hi - lo, h);
                acc0 ^= mix(h[0], (uint64_t)k);
                acc1 ^= mix(h[1], (uint64_t)k + 77);
            }
            double t2 = now();
            if (diff || acc0 == 42) printf("!");
            if (t1 - t0 < best_c) best_c = t1 - t0;
            if (t2 - t1 < best_h) best_h = t2 - t1;
        }
        printf("threads %2d: compare %7.1f us, hash %7.1f us\n", t, best_c * 1e6, best_h * 1e6);
    }
    return 0;
}
