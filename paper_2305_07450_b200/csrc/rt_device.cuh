// Device-side shared definitions of the b200rt frame render (sm_100a).
//
// Layout in HBM (per device, per precision R = float | double):
//   geo   R[n][4]   {cx, cy, cz, r^2} for spheres, {0, h, 0, -1} for planes
//                   (a negative 4th lane marks the horizontal plane); read by
//                   every closest-hit and shadow test, staged into shared
//                   memory per CTA so warp-uniform body loops are broadcasts.
//   mat   R[n][8]   {r, g, b, refl / max_refl, refl, 0, 0, 0}; read only at hits.
//   table R[s][2]   sunflower disc offsets r_i (cos th_i, sin th_i)
//                   (shading.py:89-100), computed on the host in float64 with
//                   the same libm as the reference — a closed-form per-sample
//                   table, there is no RNG in the reference.
//   sky   float4[H][W]  texels pre-clamped to [0,1] (renderer.py:74), RGB + pad.
//   out   uint32 framebuffer, pixel (x, y) at out[y * out_pitch + x].
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rt {

constexpr int kMaxBounce = 31;  // renderer.py:36
constexpr int kTileW = 16;      // CTA tile: 16 x 8 pixels, 4 warps of 8 x 4
constexpr int kTileH = 8;
constexpr int kThreads = 128;
constexpr int kSmemGeoBytes = 32 * 1024;  // scenes up to this size are staged in shared memory
constexpr int kCounterRing = 64;          // work counters per device (one per in-flight launch)

// Camera + frame + partition (one launch renders one row-block partition).
struct FrameArgs {
    uint32_t *out;
    int64_t out_pitch;
    void *radiance;  // optional R[height*width*3], full-frame indexing y*width + x
    int width, height;
    int part, n_parts, block_rows;
    int local_rows;  // rows of this partition, rounded up to whole blocks
    double cam[3];
    double cb, sb, ca, sa;  // cos/sin(pitch), cos/sin(yaw) (host libm, vecmath.py:99-110)
    double vdist;           // camera.py:64-67
    double ndc[4];          // FP32 kernels: u = x*ndc[0] + ndc[1], v = y*ndc[2] + ndc[3] (camera.py:46-54)
    int samples, bounces;
    int peer_out;  // out lives on another GPU: fence the stores at system scope
    unsigned int *work_counter;  // zeroed before the launch: persistent warps take 8x4 patches from it
    int sub_part, sub_parts;     // within a band: rows interleaved in 8-row blocks (sub_parts = 1: all)
    int row_end;                 // rows >= row_end are skipped (end of the band / frame)
    int row0;                    // first frame row of a contiguous band (sub_parts > 1 or n_parts == 1)
    int rgba;                    // pixel byte order: 0 B,G,R,A (0xAARRGGBB), 1 R,G,B,A
};

// The FP32 megakernel's per-frame culling data (render_f32.cu), a kernel
// parameter of its own so the other kernels' parameters stay lean.
struct MegaCull {
    // scenes of up to 8 spheres: per sphere (ascending body order) a
    // conservative pixel box {x0, y0, x1, y1} outside which no primary ray can
    // hit it (nbox = 0: none, every primary ray tests every sphere)
    int nbox;
    int box[8][4];
    // the shadow grid (render_fused_f32.cu, shadow_grid_build): per cell the
    // spheres that can block a shadow ray from it; null: none
    const unsigned *grid;
    float grid_lo[3], grid_inv[3];
    int grid_dim[3];
    int4 hot;  // the tile kernel's hot tile rectangle (tile_of_block); x < 0: bottom rows first
    unsigned long long hot_div[3];  // tile_of_block's divisors as multipliers (tile_divisor)
};

// The spheres whose primary-ray box holds pixel (x, y) (all when no boxes).
__host__ __device__ __forceinline__ unsigned primary_sphere_mask(const MegaCull &mc, int x, int y) {
    if (!mc.nbox) return ~0u;
    unsigned m = 0;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        if (b >= mc.nbox) break;
        const bool in = x >= mc.box[b][0] && x <= mc.box[b][2] && y >= mc.box[b][1] && y <= mc.box[b][3];
        m |= (in ? 1u : 0u) << b;
    }
    return m;
}

template <typename R>
struct SceneArgs {
    const R *geo;
    const R *mat;
    const R *table;
    const float4 *sky;
    int sky_w, sky_h, has_sky;
    int n;
    R light[3];
    R light_radius;
    R lc[3];
    R ambient;
    const double *host_geo;  // host copy of geo (float64), for launch-parameter scene packing
    const double *geo64;     // device geo in float64 (the FP32 kernels' ray chain refines its hits with it)
};

// Wavefront queues (render_wave_f32.cu); slot = bounce * n_pix + local pixel.
struct WaveArgs {
    float4 *hit_p;     // {p.xyz, body index bits}
    float4 *hit_n;     // {n.xyz, Lambert factor}
    float *hit_s;      // Blinn factor
    float *hit_sc;     // shadow coefficient
    int *queue;        // slots holding a hit
    unsigned *count;   // queue lengths; culled path: [0], [3] lane queues, [1] warp queue, [4] spare
    unsigned *count_next;  // culled path: the next frame's counters, zeroed by this frame's trace
    int *queue2;          // culled path: undecided hits (slots)
    unsigned *mask2;      // their candidate-body masks, word-major [words][mask2_stride]
    int64_t mask2_stride;
    float4 *pix;       // {tail rgb, records | exhausted << 8}
    float4 *rec;       // culled path: {body, Lambert, Blinn, coefficient} per hit of a pending pixel
    int *pend;         // culled path: per pixel, its hits still sampling (written when 2 or more)
    unsigned long long *pend64;  // the same buffer as packed counts (render_fused_f32.cu, resolve_hit)
    int64_t n_pix;     // pixels of this partition (local_rows * width)
    unsigned long long *work;  // optional executed-work tallies of the culled path (kWork*), or null
    int cull;          // exact per-hit occluder culling (1); 2: every body left undecided (cull_check)
    float4 *conic;     // culled path: silhouette coefficients of queued hits, [2 kConic][conic_cap]
    unsigned conic_cap;  // queue positions below this may take the silhouette form (0: off)
    // culled path: the shadow grid (rt_build_shadow_grid_f32): per cell of a
    // box around the spheres, the occluders (spheres, or clusters) that may
    // meet the shadow cone of a hit anywhere in the cell; null: none
    const unsigned *grid;
    float grid_lo[3], grid_inv[3];
    int grid_dim[3];
    float4 *lane_q;    // culled path: single-candidate hits sampled one lane each: queue q (0: the
                       // sphere wholly in front, 1: not), row r (0: {p, slot}, 1: {n, sphere}) at
                       // [(2q + r) lane_cap]; lengths count[3] and count[0]
    unsigned lane_cap; // (0: off)
    int4 hot;          // the trace's hot tile rectangle (tile_of_block); x < 0: bottom rows first
    unsigned long long hot_div[3];  // tile_of_block's divisors as multipliers (tile_divisor)
    int compact;       // many-sphere trace: pack the CTA's live rays between bounces (render_fused_f32.cu)
};
// FP64 culled wavefront (render_fused_f64.cu): queues in float64
constexpr int kMaxBodies64 = 256;
struct WaveArgs64 {
    double4 *q;        // queued undecided hits: [2e] {p, record slot}, [2e+1] {n, 0}
    unsigned *mask;    // their candidate-body masks (original indices), word-major [8][mask_stride]
    int64_t mask_stride;
    unsigned *count;   // [1] queue length, [2] parked pixels
    double4 *pix;      // parked pixels: {tail rgb, records | exhausted << 8}
    double4 *rec;      // {body, Lambert, Blinn, coefficient} per hit of a parked pixel
    int *parked;       // parked pixels (local indices)
    int64_t n_pix;
    double4 *lane_q;   // single-sphere undecided hits, one sampling lane each: [2e] {p, slot}, [2e+1] {n, body}
    unsigned lane_cap; // (0: off); length count[3]
};

// executed-work tallies of the culled shadow kernel (rt_work_counts)
enum { kWorkHits = 0, kWorkCullTests, kWorkSampledHits, kWorkShadowRays, kWorkSphereTests, kWorkPlaneTests,
       kWorkTraceRays, kWorkTraceTests, kWorkTraceFullWarps, kWorkConicHits, kWorkConicTests, kWorkLaneHits,
       kWorkConicZTests, kWorkN };
constexpr int kParamSpheres = 512;  // scenes up to this many spheres ride in the launch parameters (~15 KB)
constexpr int kParamMid = 256;      // the culled path's middle size (smaller parameter block and masks)
constexpr int kMaskWords = kParamSpheres / 32;
// candidate-mask words per queued hit of the culled path for a scene of ns
// spheres (the ParamScene<MAXS> instantiation it takes), plus the plane word
inline int rt_mask_words(int ns) { return (ns <= 8 ? 1 : ns <= kParamMid ? kParamMid / 32 : kMaskWords) + 1; }
constexpr int kWaveMinSamples = 8;     // soft shadows at or above this take the wavefront path
constexpr int kGridCells = 48 * 24 * 48;  // shadow grid (x, y, z) of the culled FP32 path
constexpr int kConic = 4;             // silhouette-form spheres per queued hit (rt_wave.cuh; more: the ray form)
constexpr int kWaveSmemSamples = 2048;  // disc tables (16 B/sample) up to this size are staged in shared memory

// Row-block interleave: local row ly of partition `part` -> frame row.
// Partition `part` owns the blocks j = part, part + n_parts, ... of
// block_rows rows.  A contiguous band (n_parts = 1) starts at row0; inside
// it, sub-partition `sub_part` owns the 8-row blocks i = sub_part,
// sub_part + sub_parts, ... (a band split among workers, rt_render_v1 on
// one device).
__host__ __device__ __forceinline__ int map_row(int ly, const FrameArgs &a) {
    if (a.sub_parts > 1) {
        int jl = ly / 8, r = ly - jl * 8;
        return a.row0 + (jl * a.sub_parts + a.sub_part) * 8 + r;
    }
    if (a.n_parts == 1) return a.row0 + ly;
    int jl = ly / a.block_rows;
    int r = ly - jl * a.block_rows;
    return (jl * a.n_parts + a.part) * a.block_rows + r;
}

// Rows of sub-partition p of a band of `rows` rows (rounded up to whole
// 8-row blocks; the kernels skip rows outside the band and the frame).
inline int rt_band_local_rows(int rows, int p, int parts) {
    if (rows <= 0) return 0;
    if (parts == 1) return rows;
    int nb = (rows + 7) / 8;
    int mine = nb > p ? (nb - p + parts - 1) / parts : 0;
    return mine * 8;
}

// Thread -> pixel: each warp shades an 8 x 4 pixel patch (coherent rays),
// the CTA a 16 x 8 tile.
__device__ __forceinline__ void thread_pixel(int &x, int &ly) {
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    x = blockIdx.x * kTileW + (warp & 1) * 8 + (lane & 7);
    ly = blockIdx.y * kTileH + (warp >> 1) * 4 + (lane >> 3);
}

// The same with the tile rows taken bottom first: blocks are dispatched in
// index order, and the scene sits below the horizon, so the costly tiles
// start first and cheap sky tiles fill the last wave.
__device__ __forceinline__ void thread_pixel_bottom_first(int &x, int &ly) {
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    x = blockIdx.x * kTileW + (warp & 1) * 8 + (lane & 7);
    ly = (gridDim.y - 1 - blockIdx.y) * kTileH + (warp >> 1) * 4 + (lane >> 3);
}

// Tile dispatch order with a hot rectangle (tiles [h.x, h.z] x [h.y, h.w],
// local tile rows): the hot tiles first, then the rest; each part bottom row
// first.  h.x < 0: bottom first over the whole grid.  A bijection of the
// linear block index onto the tiles (the hardware dispatches CTAs in
// index order): the costliest tiles start early and the cheap ones fill the
// last wave.
// The divisors of tile_of_block (the grid width W, the rectangle's width rw
// and W - rw) as multipliers formed on the host: q = (j m) >> 32 with
// m = floor(2^32 / d) + 1 is j / d exactly while j d < 2^32 (j < 2^20 tiles,
// d < 2^12) — one wide multiply instead of the generic division sequence,
// which every thread of the trace ran (~4% of its instructions).
inline unsigned long long tile_divisor(int d) { return d > 0 ? (1ull << 32) / (unsigned)d + 1ull : 0ull; }
__device__ __forceinline__ int tdiv(int j, unsigned long long m) { return (int)(((unsigned long long)j * m) >> 32); }

__device__ __forceinline__ void tile_of_block(int4 h, const unsigned long long *dv, int &tx, int &ty) {
    const int W = gridDim.x, H = gridDim.y, b = blockIdx.y * W + blockIdx.x;
    if (h.x < 0) {
        tx = blockIdx.x;
        ty = H - 1 - blockIdx.y;
        return;
    }
    const int rw = h.z - h.x + 1, rh = h.w - h.y + 1, area = rw * rh;
    if (b < area) {
        const int q = tdiv(b, dv[1]);
        tx = h.x + (b - q * rw);
        ty = h.w - q;
        return;
    }
    int j = b - area;
    const int below = (H - 1 - h.w) * W;  // full rows under the rectangle
    if (j < below) {
        const int q = tdiv(j, dv[0]);
        ty = H - 1 - q;
        tx = j - q * W;
        return;
    }
    j -= below;
    const int side = W - rw, beside = side * rh;  // the rectangle's rows, left and right of it
    if (j < beside) {
        const int q = tdiv(j, dv[2]);
        ty = h.w - q;
        const int k = j - q * side;
        tx = k < h.x ? k : k + rw;
        return;
    }
    j -= beside;
    const int q = tdiv(j, dv[0]);
    ty = h.y - 1 - q;  // full rows above it
    tx = j - q * W;
}
__device__ __forceinline__ void thread_pixel_hot_first(int4 h, const unsigned long long *dv, int &x, int &ly) {
    int tx, ty;
    tile_of_block(h, dv, tx, ty);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    x = tx * kTileW + (warp & 1) * 8 + (lane & 7);
    ly = ty * kTileH + (warp >> 1) * 4 + (lane >> 3);
}

// renderer.py:45-50.  rgba = 0: 0xAARRGGBB (the reference's Framebuffer,
// bytes B,G,R,A); rgba = 1: bytes R,G,B,A — the frame server's wire format
// (server.py:56-64), so a frame can be streamed without a host-side repack.
template <typename R>
__device__ __forceinline__ uint32_t pack_color(R r, R g, R b, int rgba) {
    uint32_t ri = (uint32_t)(int)(r * R(255.0) + R(0.5));
    uint32_t gi = (uint32_t)(int)(g * R(255.0) + R(0.5));
    uint32_t bi = (uint32_t)(int)(b * R(255.0) + R(0.5));
    return rgba ? 0xFF000000u | (bi << 16) | (gi << 8) | ri : 0xFF000000u | (ri << 16) | (gi << 8) | bi;
}

}  // namespace rt

// Launchers (one translation unit per precision; the FP64 one is compiled
// with -fmad=false so no a*b+c is contracted, as numba compiles the reference).
// tiles: one CTA per 16 x 8 tile (scenes that fit the launch parameters);
// otherwise persistent warps on a work counter (fa.work_counter, zeroed)
cudaError_t rt_launch_render_f32(const rt::FrameArgs &fa, const rt::SceneArgs<float> &sa, cudaStream_t st,
                                 bool tiles, const rt::MegaCull &mc);
cudaError_t rt_launch_render_f64(const rt::FrameArgs &fa, const rt::SceneArgs<double> &sa, cudaStream_t st);
cudaError_t rt_launch_wave_f32(const rt::FrameArgs &fa, const rt::SceneArgs<float> &sa, const rt::WaveArgs &wa,
                               cudaStream_t st, int *n_kernels, cudaEvent_t *phase_events /* 5 or null */);
int rt_wave_lanes(int samples);
bool rt_fused_fits(const rt::SceneArgs<float> &sa);
// Build the shadow grid of the scene in sa (light included) into `mask`
// (capacity cells), filling wa's grid fields; a scene without spheres or that
// does not fit leaves wa.grid null.
cudaError_t rt_build_shadow_grid_f32(const rt::SceneArgs<float> &sa, unsigned *mask, int capacity, rt::WaveArgs &wa,
                                     cudaStream_t st);
// unclustered FP32 scenes: a bound over every sphere lets a ray skip the
// sphere loop (rt_f32.cuh, pack_params); process-wide switch for A/B runs
void rt_set_sphere_bound(bool on);
cudaError_t rt_launch_fused_f32(const rt::FrameArgs &fa, const rt::SceneArgs<float> &sa, const rt::WaveArgs &wa,
                                cudaStream_t st, int *n_kernels, cudaEvent_t *phase_events /* 5 or null */);
cudaError_t rt_launch_fused_f64(const rt::FrameArgs &fa, const rt::SceneArgs<double> &sa, const rt::WaveArgs64 &wa,
                                cudaStream_t st, int *n_kernels);
cudaError_t rt_launch_trace_f32(const double *d_orig, const double *d_dir, int64_t n, float *d_out,
                                const rt::SceneArgs<float> &sa, int samples, int bounces, cudaStream_t st);
cudaError_t rt_launch_trace_f64(const double *d_orig, const double *d_dir, int64_t n, double *d_out,
                                const rt::SceneArgs<double> &sa, int samples, int bounces, cudaStream_t st);
cudaError_t rt_launch_sky_f64(const double *d_dir, int64_t n, double *d_out, const float4 *sky, int w, int h,
                              cudaStream_t st);
