// Host side of a lossless row-run frame codec: how fast can the host expand
// a compressed frame into the caller's framebuffer, by thread count?
// Format per row: tokens {u32 nlit | nrep << 16, nlit pixels}: copy the
// literals, then repeat the last written pixel nrep times.  Baseline: a plain
// multi-threaded memcpy of the whole frame.
//   gcc -O3 -march=native -fopenmp -o tools/micro/frame_codec tools/micro/frame_codec.c
//   tools/micro/frame_codec tools/micro/_data/C2.bin 1280 720
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now_us(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

static int cmp_d(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return x < y ? -1 : x > y;
}

// encode one row; returns words written
static size_t encode_row(const uint32_t *px, int w, uint32_t *out) {
    size_t o = 0;
    int i = 0;
    while (i < w) {
        size_t hdr = o++;
        int nlit = 0;
        // literals: until a run of >= 2 equal-to-left pixels starts
        while (i < w) {
            if (i > 0 && px[i] == px[i - 1] && i + 1 < w && px[i + 1] == px[i]) break;
            if (i > 0 && px[i] == px[i - 1] && i + 1 == w) break;
            out[o++] = px[i++];
            nlit++;
        }
        int nrep = 0;
        while (i < w && px[i] == px[i - 1] && nrep < 65535) {
            i++;
            nrep++;
        }
        out[hdr] = (uint32_t)nlit | ((uint32_t)nrep << 16);
    }
    return o;
}

static inline void fill32(uint32_t *p, uint32_t v, int n) {
    for (int k = 0; k < n; k++) p[k] = v;
}

static void decode_row(const uint32_t *in, int w, uint32_t *px) {
    int i = 0;
    while (i < w) {
        const uint32_t h = *in++;
        const int nlit = h & 0xffff, nrep = h >> 16;
        memcpy(px + i, in, (size_t)nlit * 4);
        in += nlit;
        i += nlit;
        fill32(px + i, px[i - 1], nrep);
        i += nrep;
    }
}

// Format B: per row w/8 mask bytes (bit j of byte g: pixel 8g+j differs from
// its left neighbour; a row's first pixel always does) and the row's literal
// pixels; rows' literal offsets from a prefix sum.  AVX2 decode: each group of
// 8 pixels is one permute of the next 8 literals (index of the last literal at
// or before each position) blended with the previous pixel (= the last
// literal emitted) for positions before the group's first literal.
static __m256i lut_idx[256], lut_pre[256];
__attribute__((target("avx2"))) static void init_lut(void) {
    for (int m = 0; m < 256; m++) {
        int idx[8], pre[8], k = -1;
        for (int j = 0; j < 8; j++) {
            if ((m >> j) & 1) k++;
            idx[j] = k < 0 ? 0 : k;
            pre[j] = k < 0 ? -1 : 0;
        }
        lut_idx[m] = _mm256_loadu_si256((const __m256i *)idx);
        lut_pre[m] = _mm256_loadu_si256((const __m256i *)pre);
    }
}
static size_t encode_b_row(const uint32_t *px, int w, uint8_t *mk, uint32_t *lit) {
    size_t n = 0;
    for (int g = 0; g < w / 8; g++) {
        uint8_t m = 0;
        for (int j = 0; j < 8; j++) {
            const int i = 8 * g + j;
            if (i == 0 || px[i] != px[i - 1]) {
                m |= 1 << j;
                lit[n++] = px[i];
            }
        }
        mk[g] = m;
    }
    return n;
}
__attribute__((target("avx2,popcnt"))) static void decode_b_row(const uint8_t *mk, const uint32_t *lit, int w, uint32_t *out) {
    for (int g = 0; g < w / 8; g++) {
        const unsigned m = mk[g];
        const __m256i L = _mm256_loadu_si256((const __m256i *)lit);
        const __m256i P = _mm256_permutevar8x32_epi32(L, lut_idx[m]);
        const __m256i prev = _mm256_set1_epi32((int)lit[-1]);
        _mm256_storeu_si256((__m256i *)(out + 8 * g), _mm256_blendv_epi8(P, prev, lut_pre[m]));
        lit += __builtin_popcount(m);
    }
}

int main(int argc, char **argv) {
    if (argc < 4) return 2;
    const int w = atoi(argv[2]), h = atoi(argv[3]);
    const size_t npx = (size_t)w * h;
    uint32_t *frame = malloc(npx * 4), *dst = aligned_alloc(64, npx * 4), *enc = malloc(npx * 8 + (size_t)h * 64);
    size_t *off = malloc(sizeof(size_t) * (h + 1));
    FILE *f = fopen(argv[1], "rb");
    if (!f || fread(frame, 4, npx, f) != npx) return 3;
    fclose(f);
    size_t o = 0;
    for (int r = 0; r < h; r++) {
        off[r] = o;
        o += encode_row(frame + (size_t)r * w, w, enc + o);
    }
    off[h] = o;
    printf("%s %dx%d: %zu B -> %zu B (%.3f)\n", argv[1], w, h, npx * 4, o * 4, (double)o / npx);
    init_lut();
    uint8_t *mk = malloc(npx / 8);
    uint32_t *lits = malloc(npx * 4 + 64) + 1;  // lit[-1] readable
    size_t *loff = malloc(sizeof(size_t) * (h + 1)), nl = 0;
    for (int r = 0; r < h; r++) {
        loff[r] = nl;
        nl += encode_b_row(frame + (size_t)r * w, w, mk + (size_t)r * (w / 8), lits + nl);
    }
    loff[h] = nl;
    printf("format B: %zu mask B + %zu literal B = %zu B (%.3f)\n", npx / 8, nl * 4, npx / 8 + nl * 4,
           (npx / 8 + nl * 4) / (double)(npx * 4));
    const int reps = 400;
    double *t = malloc(sizeof(double) * reps);
    int threads[] = {1, 2, 4, 8, 12, 16, 24, 32};
    const int max_threads = omp_get_max_threads();
    for (int ti = 0; ti < 8; ti++) {
        const int nt = threads[ti];
        if (nt > max_threads) break;
        omp_set_num_threads(nt);
        for (int mode = 0; mode < 4; mode++) {
            for (int k = 0; k < reps; k++) {
                const double t0 = now_us();
                if (mode == 0) {
#pragma omp parallel for schedule(static)
                    for (int r = 0; r < h; r++) decode_row(enc + off[r], w, dst + (size_t)r * w);
                } else if (mode == 2) {
#pragma omp parallel for schedule(static)
                    for (int r = 0; r < h; r++) decode_b_row(mk + (size_t)r * (w / 8), lits + loff[r], w, dst + (size_t)r * w);
                } else if (mode == 3) {
#pragma omp parallel for schedule(static, 2)
                    for (int r = 0; r < h; r++) decode_b_row(mk + (size_t)r * (w / 8), lits + loff[r], w, dst + (size_t)r * w);
                } else {
#pragma omp parallel
                    {
                        const int id = omp_get_thread_num(), n = omp_get_num_threads();
                        const size_t a = npx * id / n, b = npx * (id + 1) / n;
                        memcpy(dst + a, frame + a, (b - a) * 4);
                    }
                }
                t[k] = now_us() - t0;
                // a gap like a frame's GPU time between decodes (the pool's threads keep spinning or sleep)
                const double g = now_us();
                while (now_us() - g < 60.0) {
                }
            }
            qsort(t, reps, sizeof(double), cmp_d);
            if (mode >= 2 && memcmp(dst, frame, npx * 4) != 0) printf("SIMD MISMATCH\n");
            printf("threads %2d %-7s median %7.1f us  p10 %7.1f  p90 %7.1f\n", nt, (const char *[]){"decode", "memcpy", "simd", "simd-il"}[mode], t[reps / 2],
                   t[reps / 10], t[reps * 9 / 10]);
        }
        if (memcmp(dst, frame, npx * 4) != 0) printf("MISMATCH\n");
        memset(dst, 0, npx * 4);
#pragma omp parallel for schedule(static)
        for (int r = 0; r < h; r++) decode_row(enc + off[r], w, dst + (size_t)r * w);
        if (memcmp(dst, frame, npx * 4) != 0) printf("DECODE MISMATCH\n");
    }
    return 0;
}
