// GPU side of the compressed frame transfer (frame_codec.h): one CTA per row.
// The row is read once from L2 (the frame was just written), its literal
// mask formed with one ballot per 32 pixels, the literals compacted in
// shared memory and the row's run written to the mapped host buffer as whole
// 128-byte segments — PCIe carries ~3 bytes per literal and the non-zero
// mask words instead of 4 bytes per pixel (C2: 0.33 MB of 3.7), in few large
// transactions (zero-copy writes cost ~2.7 ns per 128 B segment, ~47 GB/s;
// scattered small stores run at ~0.7 G/s).
#include "frame_codec.h"

#include <algorithm>

namespace {

constexpr int kCodecThreads = 256;  // 8 warps: a row each

__device__ __forceinline__ unsigned lanemask_lt_() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// kRows rows per CTA, staged in shared memory with every load independent,
// their chunks spread over the 8 warps.  (Per-row "landed" flags behind a
// system-scope fence, so the host could expand rows while others still
// cross PCIe, measured slower: the fences and the host's polling cost more
// than the overlap gave.)
constexpr int kRows = 1;

__global__ void __launch_bounds__(kCodecThreads)
    encode_rows(const uint32_t *__restrict__ frame, int64_t pitch, int width, int y0, int y1, int part, int n_parts,
                int block_rows, uint32_t *__restrict__ out) {
    extern __shared__ uint32_t sm[];
    __shared__ int s_n[kRows], s_nz[kRows], s_opaque[kRows];
    const int nc = rt::codec_mask_words(width), nb = rt::codec_bitmap_words(width);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = kCodecThreads / 32;
    // this CTA's row: the blockIdx-th of rows [y0, y1) — or, for a partition of
    // block_rows-row blocks dealt round-robin over n_parts, of its blocks
    const int b = blockIdx.x * kRows;
    const int r0 = n_parts > 1 ? y0 + ((b / block_rows) * n_parts + part) * block_rows + b % block_rows : y0 + b;
    const int rows = min(kRows, y1 - r0);
    uint32_t *spx = sm;                      // [kRows][width] the rows' pixels
    uint32_t *slit = spx + kRows * width;    // [kRows][width] their literals, compacted
    uint32_t *smask = slit + kRows * width;  // [kRows][nc] mask word per chunk of 32 pixels
    uint32_t *soff = smask + kRows * nc;     // [kRows][nc] literals before each chunk
    uint32_t *snz = soff + kRows * nc;       // [kRows][nc] the non-zero mask words, compacted
    uint32_t *sbm = snz + kRows * nc;        // [kRows][nb] bit c: chunk c's mask word is non-zero
    if (threadIdx.x < kRows) s_opaque[threadIdx.x] = 1;
    // launched as a programmatic dependent of the frame's last kernel: the
    // rows are read only once it is done
    cudaGridDependencySynchronize();
    // the rows into shared memory, every load independent (a chunk loop with
    // a load per step measured 2x slower: its latencies add up)
    for (int r = 0; r < rows; r++) {
        const uint4 *src = reinterpret_cast<const uint4 *>(frame + (int64_t)(r0 + r) * pitch);
        if ((width & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {  // (a caller's frame may be offset)
#pragma unroll 4
            for (int i = threadIdx.x; i < width / 4; i += kCodecThreads)
                reinterpret_cast<uint4 *>(spx + r * width)[i] = __ldcg(src + i);
        } else {
#pragma unroll 4
            for (int i = threadIdx.x; i < width; i += kCodecThreads)
                spx[r * width + i] = __ldcg(frame + (int64_t)(r0 + r) * pitch + i);
        }
    }
    __syncthreads();
    // masks: chunk (r, c) by warp (r nc + c) % warps
    for (int idx = warp; idx < rows * nc; idx += warps) {
        const int r = idx / nc, c = idx - r * nc;
        const int x = 32 * c + lane;
        const bool in = x < width;
        const uint32_t p = in ? spx[r * width + x] : 0u;
        const uint32_t left = x == 0 ? ~p : in ? spx[r * width + x - 1] : 0u;
        const bool lit = in && p != left;
        const unsigned bm = __ballot_sync(0xffffffffu, lit);
        // every literal's top byte 0xFF (the frames' alpha): 3 bytes each suffice
        if (!__all_sync(0xffffffffu, !lit || (p >> 24) == 0xffu) && lane == 0) s_opaque[r] = 0;
        if (lane == 0) {
            smask[idx] = bm;
            soff[idx] = __popc(bm);
        }
    }
    __syncthreads();
    // warp r: row r's literal offsets (exclusive scan), non-zero mask words and bitmap
    if (warp < rows) {
        const int r = warp;
        unsigned carry = 0, nz = 0;
        for (int c0 = 0; c0 < nc; c0 += 32) {
            const int c = c0 + lane;
            const unsigned v = c < nc ? soff[r * nc + c] : 0u, wd = c < nc ? smask[r * nc + c] : 0u;
            unsigned s = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned t = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += t;
            }
            const unsigned nzb = __ballot_sync(0xffffffffu, wd != 0u);
            if (c < nc) soff[r * nc + c] = carry + s - v;
            if (wd != 0u) snz[r * nc + nz + __popc(nzb & lanemask_lt_())] = wd;
            if (lane == 0) sbm[r * nb + (c0 >> 5)] = nzb;
            carry += __shfl_sync(0xffffffffu, s, 31);
            nz += __popc(nzb);
        }
        if (lane == 0) {
            s_n[r] = (int)carry;
            s_nz[r] = (int)nz;
        }
    }
    __syncthreads();
    for (int idx = warp; idx < rows * nc; idx += warps) {
        const int r = idx / nc, c = idx - r * nc;
        const unsigned bm = smask[idx];
        if ((bm >> lane) & 1u) slit[r * width + soff[idx] + __popc(bm & lanemask_lt_())] = spx[r * width + 32 * c + lane];
    }
    __syncthreads();
    // each row's run (frame_codec.h) from a 128 B boundary: whole 128 B segments over PCIe
    for (int r = 0; r < rows; r++) {
        const int n = s_n[r], head = 1 + nb + s_nz[r];
        const bool packed = s_opaque[r] != 0;
        const int total = head + (packed ? (3 * n + 3) / 4 : n);
        const uint32_t *lr = slit + r * width;
        uint32_t *dr = out + (int64_t)(r0 + r) * rt::codec_row_stride(width);
        for (int i = threadIdx.x; i < total; i += kCodecThreads) {
            uint32_t v;
            if (i == 0) {
                v = (uint32_t)n | (packed ? 0x80000000u : 0u);
            } else if (i <= nb) {
                v = sbm[r * nb + i - 1];
            } else if (i < head) {
                v = snz[r * nc + i - 1 - nb];
            } else if (!packed) {
                v = lr[i - head];
            } else {  // bytes 4k .. 4k + 3 of the 3-byte literal stream
                const int k = i - head;
                v = 0;
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int byte = 4 * k + b, li = byte / 3, bi = byte - 3 * li;
                    const uint32_t q = li < n ? lr[li] : 0u;
                    v |= ((q >> (8 * bi)) & 0xffu) << (8 * b);
                }
            }
            dr[i] = v;
        }
    }
}

}  // namespace

namespace rt {

cudaError_t launch_encode_rows(const uint32_t *frame, int64_t pitch, int width, int height, int y0, int y1,
                               uint32_t *d_host, cudaStream_t st, int part, int n_parts, int block_rows) {
    if (y1 <= y0) return cudaSuccess;
    // rows of the partition (blocks j = part, part + n_parts, ... of block_rows rows)
    int rows = y1 - y0;
    if (n_parts > 1) {
        rows = 0;
        for (int j = part; j * block_rows < y1 - y0; j += n_parts) rows += std::min(block_rows, y1 - y0 - j * block_rows);
        if (rows == 0) return cudaSuccess;
    }
    const int nc = codec_mask_words(width);
    const size_t smem = sizeof(uint32_t) * kRows * (2 * (size_t)width + 3 * (size_t)nc + codec_bitmap_words(width));
    if (smem > 48 * 1024) {  // rows wider than ~1,400 pixels (up to kCodecMaxWidth: 206 KB)
        cudaError_t e = cudaFuncSetAttribute(encode_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((rows + kRows - 1) / kRows);
    cfg.blockDim = dim3(kCodecThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, encode_rows, frame, pitch, width, y0, y1, part, n_parts, block_rows,
                              d_host + kCodecPad);
}

}  // namespace rt
