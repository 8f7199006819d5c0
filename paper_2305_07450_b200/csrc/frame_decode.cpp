// Host side of the compressed frame transfer (frame_codec.h): expand rows
// into the caller's framebuffer.  Packed literals are first widened from 3
// bytes to a pixel with alpha 0xFF (one permute + byte shuffle per 8).  A
// zero mask word is 32 repeats of the pixel to the left (4 stores); any other
// word is 4 groups of 8 pixels, each one AVX2 permute of the next 8 literals
// (for every position the index of the last literal at or before it) blended
// with the previous pixel (= the last literal consumed) for the positions
// before the group's first literal.  Rows are split over an OpenMP team
// (tools/codec_expand_bench.py).  A scalar path serves CPUs without AVX2.
#include "frame_codec.h"

#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <string>
#include <vector>

namespace {

struct Lut {
    alignas(32) int32_t idx[256][8];  // position j -> literal index (0 before the first)
    alignas(32) int32_t pre[256][8];  // -1 where j precedes the group's first literal
    Lut() {
        for (int m = 0; m < 256; m++) {
            int k = -1;
            for (int j = 0; j < 8; j++) {
                if ((m >> j) & 1) k++;
                idx[m][j] = k < 0 ? 0 : k;
                pre[m][j] = k < 0 ? -1 : 0;
            }
        }
    }
};
const Lut g_lut;

// The widest expander the CPU runs; $B200RT_CODEC_ISA (scalar | avx2 |
// avx512) picks a narrower one (the CPU tests run each).
enum Isa { kScalar, kAvx2, kAvx512 };
Isa codec_isa() {
    static const Isa isa = [] {
        const bool a2 = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("popcnt");
        const bool a512 = a2 && __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                          __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512vbmi") &&
                          __builtin_cpu_supports("avx512vpopcntdq");
        Isa best = a512 ? kAvx512 : a2 ? kAvx2 : kScalar;
        if (const char *e = std::getenv("B200RT_CODEC_ISA")) {
            const std::string v(e);
            if (v == "scalar") best = kScalar;
            if (v == "avx2" && a2) best = kAvx2;
        }
        return best;
    }();
    return isa;
}

// A row's header words (frame_codec.h).
struct Row {
    int n;                  // literals
    bool packed;            // 3 bytes each
    const uint32_t *bm;     // bit j: mask word j listed
    const uint32_t *masks;  // the listed mask words
    const uint32_t *lits;   // the literal words
    int64_t words;          // the row's run (what crossed PCIe)
};

Row parse(const uint32_t *base, int width) {
    const int nb = rt::codec_bitmap_words(width);
    Row r;
    r.n = (int)(base[0] & 0x7fffffffu);
    r.packed = base[0] >> 31;
    r.bm = base + 1;
    r.masks = r.bm + nb;
    int nnz = 0;
    for (int b = 0; b < nb; b++) nnz += __builtin_popcount(r.bm[b]);
    r.lits = r.masks + nnz;
    r.words = 1 + nb + nnz + (r.packed ? (3 * (int64_t)r.n + 3) / 4 : r.n);
    return r;
}

inline uint32_t mask_word(const Row &r, int j, const uint32_t *&next) {
    return (r.bm[j >> 5] >> (j & 31)) & 1u ? *next++ : 0u;
}

inline uint32_t widen(const uint8_t *b) { return 0xff000000u | b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16; }

void unpack_scalar(const uint32_t *src, int n, uint32_t *dst) {
    const uint8_t *b = reinterpret_cast<const uint8_t *>(src);
    for (int i = 0; i < n; i++) dst[i] = widen(b + 3 * i);
}

__attribute__((target("avx2"))) void unpack_avx2(const uint32_t *src, int n, uint32_t *dst) {
    const uint8_t *b = reinterpret_cast<const uint8_t *>(src);
    const __m256i lanes = _mm256_setr_epi32(0, 1, 2, 3, 3, 4, 5, 6);  // bytes 0-15 | 12-27
    const __m256i shuf = _mm256_setr_epi8(0, 1, 2, -128, 3, 4, 5, -128, 6, 7, 8, -128, 9, 10, 11, -128,  //
                                          0, 1, 2, -128, 3, 4, 5, -128, 6, 7, 8, -128, 9, 10, 11, -128);
    const __m256i alpha = _mm256_set1_epi32((int)0xff000000u);
    int i = 0;
    for (; i + 8 <= n; i += 8) {  // (reads 8 bytes past the 24 used: inside the row's stride or the pad)
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(b + 3 * i));
        const __m256i w = _mm256_shuffle_epi8(_mm256_permutevar8x32_epi32(v, lanes), shuf);
        _mm256_storeu_si256(reinterpret_cast<__m256i *>(dst + i), _mm256_or_si256(w, alpha));
    }
    for (; i < n; i++) dst[i] = widen(b + 3 * i);
}

void row_scalar(const Row &r, const uint32_t *lit, int w, uint32_t *out) {
    const uint32_t *next = r.masks;
    uint32_t v = 0, wd = 0;
    for (int x = 0; x < w; x++) {
        if ((x & 31) == 0) wd = mask_word(r, x >> 5, next);
        if ((wd >> (x & 31)) & 1u) v = *lit++;
        out[x] = v;
    }
}

__attribute__((target("avx2,popcnt"))) inline void group_avx2(unsigned m, const uint32_t *&lit, uint32_t *out) {
    const __m256i L = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(lit));
    const __m256i P = _mm256_permutevar8x32_epi32(L, _mm256_load_si256(reinterpret_cast<const __m256i *>(g_lut.idx[m])));
    const __m256i prev = _mm256_set1_epi32((int)lit[-1]);  // (row start: pixel 0 is a literal, unused)
    const __m256i pre = _mm256_load_si256(reinterpret_cast<const __m256i *>(g_lut.pre[m]));
    _mm256_storeu_si256(reinterpret_cast<__m256i *>(out), _mm256_blendv_epi8(P, prev, pre));
    lit += __builtin_popcount(m);
}

__attribute__((target("avx2,popcnt"))) void row_avx2(const Row &r, const uint32_t *lit, int w, uint32_t *out) {
    const uint32_t *next = r.masks;
    const int words = w / 32;
    for (int j = 0; j < words; j++) {
        const uint32_t wd = mask_word(r, j, next);
        uint32_t *o = out + 32 * j;
        if (wd == 0) {  // 32 repeats of the pixel to the left (C2: 59% of the words)
            const __m256i prev = _mm256_set1_epi32((int)lit[-1]);
            _mm256_storeu_si256(reinterpret_cast<__m256i *>(o), prev);
            _mm256_storeu_si256(reinterpret_cast<__m256i *>(o + 8), prev);
            _mm256_storeu_si256(reinterpret_cast<__m256i *>(o + 16), prev);
            _mm256_storeu_si256(reinterpret_cast<__m256i *>(o + 24), prev);
            continue;
        }
        group_avx2(wd & 0xff, lit, o);
        group_avx2((wd >> 8) & 0xff, lit, o + 8);
        group_avx2((wd >> 16) & 0xff, lit, o + 16);
        group_avx2(wd >> 24, lit, o + 24);
    }
    if (32 * words < w) {  // the last, partial mask word
        const uint32_t wd = mask_word(r, words, next);
        int x = 32 * words;
        for (int g = 0; x + 8 <= w; g++, x += 8) group_avx2((wd >> (8 * g)) & 0xff, lit, out + x);
        uint32_t v = x > 0 ? out[x - 1] : 0u;
        for (; x < w; x++) {
            if ((wd >> (x & 31)) & 1u) v = *lit++;
            out[x] = v;
        }
    }
}

// AVX-512 (VBMI + VPOPCNTDQ): 16 pixels a step.  Lane j's literal index is
// popcount(m & (2^(j+1) - 1)) - 1 (no table); lanes before the first literal
// keep the previous pixel (a merge-masked permute).
constexpr uint32_t kPrefix[16] = {0x1,   0x3,   0x7,   0xf,   0x1f,   0x3f,   0x7f,   0xff,
                                  0x1ff, 0x3ff, 0x7ff, 0xfff, 0x1fff, 0x3fff, 0x7fff, 0xffff};
#define RT_AVX512 __attribute__((target("avx512f,avx512bw,avx512vl,avx512vbmi,avx512vpopcntdq,popcnt")))

RT_AVX512 inline __m512i half_avx512(unsigned m, const uint32_t *&lit) {
    const __m512i cnt = _mm512_popcnt_epi32(_mm512_and_si512(_mm512_set1_epi32((int)m), _mm512_loadu_si512(kPrefix)));
    const __mmask16 k = _mm512_test_epi32_mask(cnt, cnt);
    const __m512i idx = _mm512_sub_epi32(cnt, _mm512_set1_epi32(1));
    const __m512i v = _mm512_mask_permutexvar_epi32(_mm512_set1_epi32((int)lit[-1]), k, idx, _mm512_loadu_si512(lit));
    lit += __builtin_popcount(m);
    return v;
}

RT_AVX512 void unpack_avx512(const uint32_t *src, int n, uint32_t *dst) {
    const uint8_t *b = reinterpret_cast<const uint8_t *>(src);
    alignas(64) uint8_t sel[64];
    for (int k = 0; k < 16; k++)
        for (int t = 0; t < 4; t++) sel[4 * k + t] = (uint8_t)(t < 3 ? 3 * k + t : 0);
    const __m512i idx = _mm512_load_si512(sel);
    const __m512i alpha = _mm512_set1_epi32((int)0xff000000u);
    int i = 0;
    for (; i + 16 <= n; i += 16) {  // (reads 16 bytes past the 48 used: inside the row's stride or the pad)
        const __m512i v = _mm512_loadu_si512(b + 3 * i);
        _mm512_storeu_si512(dst + i, _mm512_or_si512(_mm512_permutexvar_epi8(idx, v), alpha));
    }
    for (; i < n; i++) dst[i] = widen(b + 3 * i);
}

RT_AVX512 void row_avx512(const Row &r, const uint32_t *lit, int w, uint32_t *out) {
    const uint32_t *next = r.masks;
    const int words = w / 32;
    for (int j = 0; j < words; j++) {
        const uint32_t wd = mask_word(r, j, next);
        uint32_t *o = out + 32 * j;
        if (wd == 0) {  // 32 repeats of the pixel to the left
            const __m512i prev = _mm512_set1_epi32((int)lit[-1]);
            _mm512_storeu_si512(o, prev);
            _mm512_storeu_si512(o + 16, prev);
            continue;
        }
        _mm512_storeu_si512(o, half_avx512(wd & 0xffffu, lit));
        _mm512_storeu_si512(o + 16, half_avx512(wd >> 16, lit));
    }
    const int rest = w - 32 * words;
    if (rest > 0) {  // the last, partial mask word: masked stores
        const uint32_t wd = mask_word(r, words, next);
        uint32_t *o = out + 32 * words;
        const int lo = rest < 16 ? rest : 16;
        _mm512_mask_storeu_epi32(o, (__mmask16)((1u << lo) - 1u), half_avx512(wd & 0xffffu, lit));
        if (rest > 16) _mm512_mask_storeu_epi32(o + 16, (__mmask16)((1u << (rest - 16)) - 1u), half_avx512(wd >> 16, lit));
    }
}

// a row's widened literals: [0] a readable word before them, 40 spare words
thread_local std::vector<uint32_t> t_scratch;

int64_t expand_row(const uint32_t *base, int width, uint32_t *out, Isa isa) {
    const Row r = parse(base, width);
    const uint32_t *lit = r.lits;  // (unpacked: lit[-1] is a header or mask word, readable)
    if (r.packed) {
        if (t_scratch.size() < (size_t)width + 40) t_scratch.assign((size_t)width + 40, 0u);
        uint32_t *s = t_scratch.data() + 1;
        if (isa == kAvx512)
            unpack_avx512(r.lits, r.n, s);
        else if (isa == kAvx2)
            unpack_avx2(r.lits, r.n, s);
        else
            unpack_scalar(r.lits, r.n, s);
        lit = s;
    }
    if (isa == kAvx512)
        row_avx512(r, lit, width, out);
    else if (isa == kAvx2)
        row_avx2(r, lit, width, out);
    else
        row_scalar(r, lit, width, out);
    return r.words;
}

}  // namespace

namespace rt {

int64_t decode_rows_serial(const uint32_t *host, int width, int y0, int y1, uint32_t *dst, int64_t pitch) {
    const int64_t stride = codec_row_stride(width);
    const Isa isa = codec_isa();
    int64_t total = 0;
    for (int y = y0; y < y1; y++)
        total += expand_row(host + kCodecPad + (size_t)y * stride, width, dst + (size_t)y * pitch, isa);
    return total;
}

int64_t decode_rows(const uint32_t *host, int width, int y0, int y1, uint32_t *dst, int64_t pitch, int threads) {
    if (y1 <= y0) return 0;
    threads = std::max(1, std::min(threads, (y1 - y0) / 4));
    int64_t total = 0;
#pragma omp parallel num_threads(threads) reduction(+ : total)
    {
        const int tid = omp_get_thread_num(), nt = omp_get_num_threads();
        const int a = y0 + (int)((int64_t)(y1 - y0) * tid / nt), b = y0 + (int)((int64_t)(y1 - y0) * (tid + 1) / nt);
        total += decode_rows_serial(host, width, a, b, dst, pitch);
    }
    return total;
}

int64_t decode_bands(const uint32_t *host, int width, int bands, const int *y_at, const int *order,
                     int (*query)(void *arg, int band), int (*wait)(void *arg, int band), void *arg, int *rc,
                     uint32_t *dst, int64_t pitch, int threads, const CodecSideJob *side) {
    constexpr int kBlock = 8;  // rows a thread takes at a time
    std::atomic<int> ready{0};  // bands (in order) known to have landed
    std::atomic<int> failed{0};
    std::atomic<int> next_block[64];
    for (int i = 0; i < bands; i++) next_block[i].store(0);
    std::atomic<int> side_next{0};
    const int side_items = side ? side->items : 0;
    int64_t total = 0;
#pragma omp parallel num_threads(std::max(1, threads)) reduction(+ : total)
    {
        const int tid = omp_get_thread_num();
        while (!failed.load(std::memory_order_relaxed)) {
            int r = ready.load(std::memory_order_acquire);
            if (tid == 0 && r < bands) {  // the calling thread: CUDA stays on it
                const int q = query(arg, order[r]);
                if (q < 0) {
                    *rc = q;
                    failed.store(1);
                    break;
                }
                if (q > 0) ready.store(++r, std::memory_order_release);
            }
            // a block of rows of a landed band
            bool did = false;
            for (int i = 0; i < r && !did; i++) {
                const int k = order[i], y0 = y_at[k], y1 = y_at[k + 1];
                const int nblk = (y1 - y0 + kBlock - 1) / kBlock;
                if (next_block[i].load(std::memory_order_relaxed) >= nblk) continue;
                const int b = next_block[i].fetch_add(1);
                if (b >= nblk) continue;
                total += decode_rows_serial(host, width, y0 + b * kBlock, std::min(y1, y0 + (b + 1) * kBlock), dst, pitch);
                did = true;
            }
            if (did) continue;
            // else a side item
            if (side_next.load(std::memory_order_relaxed) < side_items) {
                const int s = side_next.fetch_add(1);
                if (s < side_items) {
                    side->run(side->arg, s);
                    continue;
                }
            }
            if (r == bands) break;  // every band landed and every block taken
            if (tid == 0) {  // nothing else to do: block until the next band is in
                const int w = wait(arg, order[r]);
                if (w < 0) {
                    *rc = w;
                    failed.store(1);
                    break;
                }
                ready.store(r + 1, std::memory_order_release);
            } else {
                _mm_pause();
            }
        }
    }
    return failed.load() ? -1 : total;
}

}  // namespace rt
