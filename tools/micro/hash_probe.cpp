// Throughput of the skybox content hash (rt_host.cu: hash_bytes, four
// multiply-rotate lanes per 32 bytes) against an 8-lane AVX-512 variant, on
// the 25 MB texel array of C3/C4, by thread count; and a plain read (sum).
//   g++ -O3 -fopenmp -o tools/micro/hash_probe tools/micro/hash_probe.cpp
#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

constexpr uint64_t kP1 = 0x9E3779B185EBCA87ull, kP2 = 0xC2B2AE3D27D4EB4Full;
inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
inline uint64_t hround(uint64_t acc, uint64_t w) { return rotl64(acc + w * kP2, 31) * kP1; }

uint64_t hash4(const char *p, size_t n) {
    uint64_t v1 = kP1 + kP2, v2 = kP2, v3 = 0, v4 = 0 - kP1;
    for (size_t i = 0; i + 32 <= n; i += 32) {
        uint64_t w[4];
        std::memcpy(w, p + i, 32);
        v1 = hround(v1, w[0]);
        v2 = hround(v2, w[1]);
        v3 = hround(v3, w[2]);
        v4 = hround(v4, w[3]);
    }
    return v1 ^ v2 ^ v3 ^ v4;
}

__attribute__((target("avx512f,avx512dq"))) uint64_t hash8(const char *p, size_t n) {
    __m512i acc = _mm512_set1_epi64((long long)kP1), p2 = _mm512_set1_epi64((long long)kP2),
            p1 = _mm512_set1_epi64((long long)kP1);
    for (size_t i = 0; i + 64 <= n; i += 64) {
        const __m512i w = _mm512_loadu_si512(p + i);
        acc = _mm512_mullo_epi64(_mm512_rol_epi64(_mm512_add_epi64(acc, _mm512_mullo_epi64(w, p2)), 31), p1);
    }
    alignas(64) uint64_t l[8];
    _mm512_store_si512(l, acc);
    uint64_t h = 0;
    for (int k = 0; k < 8; k++) h = hround(h, l[k]);
    return h;
}

// one 64x64 -> 128-bit multiply per 16 bytes (folded: low ^ high), four
// independent lanes; the old state added back so a zero product keeps history
inline uint64_t mix128(uint64_t a, uint64_t b) {
    const unsigned __int128 r = (unsigned __int128)a * b;
    return (uint64_t)r ^ (uint64_t)(r >> 64);
}
uint64_t hash16(const char *p, size_t n) {
    constexpr uint64_t k0 = 0xa0761d6478bd642full, k1 = 0xe7037ed1a0b428dbull, k2 = 0x8ebc6af09c88c6e3ull,
                       k3 = 0x589965cc75374cc3ull;
    uint64_t s0 = k0, s1 = k1, s2 = k2, s3 = k3;
    for (size_t i = 0; i + 64 <= n; i += 64) {
        uint64_t w[8];
        std::memcpy(w, p + i, 64);
        s0 += mix128(w[0] ^ s0, w[1] ^ k0);
        s1 += mix128(w[2] ^ s1, w[3] ^ k1);
        s2 += mix128(w[4] ^ s2, w[5] ^ k2);
        s3 += mix128(w[6] ^ s3, w[7] ^ k3);
    }
    return mix128(s0 ^ s2, s1 ^ s3);
}

__attribute__((target("avx512f"))) uint64_t sum8(const char *p, size_t n) {
    __m512i acc = _mm512_setzero_si512();
    for (size_t i = 0; i + 64 <= n; i += 64) acc = _mm512_xor_si512(acc, _mm512_loadu_si512(p + i));
    alignas(64) uint64_t l[8];
    _mm512_store_si512(l, acc);
    return l[0] ^ l[7];
}

int main() {
    const size_t bytes = 2048ull * 1024 * 3 * 4;
    std::vector<float> a(bytes / 4);
    for (size_t i = 0; i < a.size(); i++) a[i] = (float)(i % 1000) * 1e-3f;
    const char *p = (const char *)a.data();
    for (int which = 0; which < 4; which++) {
        for (int t : {1, 4, 8, 16}) {
            std::vector<double> ts;
            volatile uint64_t sink = 0;
            for (int rep = 0; rep < 30; rep++) {
                const auto t0 = std::chrono::steady_clock::now();
                const int chunks = 64;
                uint64_t h = 0;
#pragma omp parallel for num_threads(t) schedule(static) reduction(^ : h)
                for (int k = 0; k < chunks; k++) {
                    const size_t lo = bytes * k / chunks / 64 * 64, hi = bytes * (k + 1) / chunks / 64 * 64;
                    h ^= which == 0   ? hash4(p + lo, hi - lo)
                         : which == 1 ? hash8(p + lo, hi - lo)
                         : which == 2 ? sum8(p + lo, hi - lo)
                                      : hash16(p + lo, hi - lo);
                }
                sink = sink ^ h;
                ts.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
            }
            std::sort(ts.begin(), ts.end());
            printf("%-12s threads %2d: %7.1f us (%6.1f GB/s)\n",
                   (const char *[]){"hash 4-lane", "hash avx512", "read (xor)", "hash mix128"}[which],
                   t, ts[ts.size() / 2], bytes / ts[ts.size() / 2] / 1e3);
        }
    }
    return 0;
}
