// Compressed frame transfer (rt_host.cu): the finished rows of the device
// frame are encoded on the GPU straight into page-locked, mapped host memory
// and expanded on the host into the caller's framebuffer.
//
// A pixel equal to its left neighbour is a repeat; the others (a row's first
// pixel always) are literals.  Row y of a width-w frame, in uint32 words at
// kCodecPad + y * codec_row_stride(w), with mw = ceil(w / 32) mask words
// (bit i of word j: pixel 32 j + i is a literal) and nb = ceil(mw / 32):
//   word 0          the row's literal count n | packed << 31;
//   nb words        bit j set: mask word j is non-zero (listed next);
//   the non-zero mask words, in order;
//   the literals:   packed (every literal's top byte is 0xFF — the frames'
//                   alpha): 3 bytes each, the low 3 bytes of the pixel in
//                   order, ceil(3n / 4) words; else n words.
// Only this run crosses PCIe — from a 128-byte boundary, in whole 128 B
// segments (C2: 0.33 MB of 3.7).  The fixed row stride needs no prefix sum
// over rows, so bands encode independently.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#ifdef __CUDACC__
#define RT_CODEC_HD __host__ __device__
#else
#define RT_CODEC_HD
#endif

namespace rt {

RT_CODEC_HD inline int codec_mask_words(int width) { return (width + 31) / 32; }
RT_CODEC_HD inline int codec_bitmap_words(int width) { return (codec_mask_words(width) + 31) / 32; }
RT_CODEC_HD inline int64_t codec_row_stride(int width) {
    return (1 + (int64_t)codec_bitmap_words(width) + codec_mask_words(width) + width + 31) / 32 * 32;
}
// words before row 0 and after the last row (the expander reads up to 8
// words past a row's literals)
constexpr int kCodecPad = 32;
// widest row the encoder stages in shared memory
constexpr int kCodecMaxWidth = 16384;

inline size_t codec_host_bytes(int width, int height) {
    return sizeof(uint32_t) * (2 * (size_t)kCodecPad + (size_t)height * codec_row_stride(width));
}

// Encode rows [y0, y1) of a height-row frame (row pitch in pixels) into the
// mapped host buffer whose device address is d_host (layout above), launched
// as a programmatic dependent of the stream's previous kernel.  n_parts > 1:
// only partition `part`'s rows — blocks of block_rows rows dealt round-robin
// over n_parts, counted from y0 (the multi-GPU row partition).
cudaError_t launch_encode_rows(const uint32_t *frame, int64_t pitch, int width, int height, int y0, int y1,
                               uint32_t *d_host, cudaStream_t st, int part = 0, int n_parts = 1,
                               int block_rows = 8);

// Expand rows [y0, y1) of the buffer host into dst (row pitch in pixels) on
// this thread; returns the words those rows moved over PCIe.
int64_t decode_rows_serial(const uint32_t *host, int width, int y0, int y1, uint32_t *dst, int64_t pitch);

// The same over an OpenMP team of up to `threads`.
int64_t decode_rows(const uint32_t *host, int width, int y0, int y1, uint32_t *dst, int64_t pitch, int threads);

// Work the expansion team does while no band has landed (the sky hash's
// chunks, rt_host.cu): items 0..items-1, each run once by some thread.
struct CodecSideJob {
    int items = 0;
    void (*run)(void *arg, int item) = nullptr;
    void *arg = nullptr;
};

// A frame's bands as they land: band order[i] (rows [y_at[k], y_at[k + 1]))
// is expanded once it is in — query(arg, k) 1 (0: not yet, < 0: an error
// code); the calling thread blocks in wait(arg, k) (0 or an error code) only
// when nothing else is left to do.  A team of `threads` takes 8-row blocks of
// the landed bands first and the side job's items otherwise.  Returns the
// words moved, or -1 on an error (its code in *rc).
int64_t decode_bands(const uint32_t *host, int width, int bands, const int *y_at, const int *order,
                     int (*query)(void *arg, int band), int (*wait)(void *arg, int band), void *arg, int *rc,
                     uint32_t *dst, int64_t pitch, int threads, const CodecSideJob *side = nullptr);

}  // namespace rt
