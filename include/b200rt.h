/*
 * b200rt — C ABI of the B200-native frame render (libb200rt.so).
 *
 * Drop-in boundary for the reference's native render operator: the numba
 * kernel `_render_kernel(pixels, width, height, cam_pos, yaw, pitch, vdist,
 * kinds, positions, sizes, colors, refls, light_pos, light_radius,
 * light_color, ambient, max_refl, sky, sky_w, sky_h, has_sky,
 * shadow_samples, bounce_limit)` (/root/reference/pkg/src/raytracer/
 * renderer.py:227-252), dispatched by `render_frame` (renderer.py:316-349),
 * itself the paper's `Renderer::render(pixels, dimensions, camera, ...)`
 * (/root/reference/PAPER.md:1008-1020).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Scene arrays are the reference's packed
 *    structure-of-arrays (geometry.py:162-176): kinds int32[n] (0 sphere,
 *    1 horizontal plane), positions f64[n][3], sizes f64[n], colors f64[n][3],
 *    refls f64[n]; the skybox is f32[sky_h][sky_w][3] (scene.py:21-35).
 *  - Pixels are uint32 0xAARRGGBB, index x + y*width (renderer.py:45-50,
 *    scene.py:75-94); little-endian bytes are B,G,R,A.
 *  - Every function returns RT_OK (0) or a negative RT_ERR_* code; the
 *    message is in rt_last_error() (thread-local).  Nothing is ever computed
 *    on the CPU: without a CUDA device every compute call fails with
 *    RT_ERR_NO_DEVICE.
 *  - Calls on one rt_ctx are serialised by an internal mutex; the library
 *    never holds the Python GIL (ctypes.CDLL drops it), like the reference's
 *    nogil=True kernel (renderer.py:227).
 */
#ifndef B200RT_H
#define B200RT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RT_ABI_VERSION 1

enum {
    RT_OK = 0,
    RT_ERR_INVALID = -1,   /* bad argument: the reference raises ValueError (renderer.py:322-328) */
    RT_ERR_CUDA = -2,      /* CUDA runtime/kernel failure */
    RT_ERR_NO_DEVICE = -3, /* no usable CUDA device */
    RT_ERR_NOMEM = -4,     /* device or pinned allocation failed */
    RT_ERR_LIMIT = -5      /* beyond a compiled limit (e.g. bounce_limit > 31, renderer.py:36) */
};

/* Arithmetic of the render.
 *  RT_PREC_FP32: the product path — FP32 CUDA cores, cancellation-free sphere
 *                discriminant; within ±1 per 8-bit channel of the reference.
 *  RT_PREC_FP64: validation path — float64 in the reference's literal
 *                operation order, no FMA contraction; bit-identical frames
 *                (golden sha256, pkg/tests/test_acceptance.py:31). */
enum { RT_PREC_FP32 = 0, RT_PREC_FP64 = 1 };

#define RT_MAX_BOUNCE_LIMIT 31   /* renderer.py:36 */
#define RT_DEFAULT_BLOCK_ROWS 8  /* row-block height of the multi-GPU interleave */

typedef struct rt_ctx rt_ctx;

int rt_version(void);
const char *rt_last_error(void);

/* Number of visible CUDA devices (0 on a GPU-less host; never an error). */
int rt_device_count(int32_t *count);

/* Create a context over `n_devices` CUDA devices (NULL `devices` = 0..n-1).
 * Each device gets one stream, scene buffers and a staging framebuffer. */
int rt_ctx_create(rt_ctx **out, const int32_t *devices, int32_t n_devices);
int rt_ctx_destroy(rt_ctx *ctx);

/* Upload (or keep, when unchanged) the scene on every device of ctx.
 * Mirrors renderer._scene_args (renderer.py:282-300). */
int rt_set_scene_v1(rt_ctx *ctx, int32_t n_bodies, const int32_t *kinds, const double *positions,
                    const double *sizes, const double *colors, const double *refls, const double light_pos[3],
                    double light_radius, const double light_color[3], double ambient, double max_refl,
                    const float *sky, int32_t sky_w, int32_t sky_h, int32_t has_sky);

/* The drop-in frame render: replaces `_render_kernel(...)` (renderer.py:227-279).
 * Same argument list and meaning, plus
 *   radiance   NULL, or host float[w*h*3] (RT_PREC_FP32) / double[w*h*3]
 *              (RT_PREC_FP64): pre-quantisation colour per pixel;
 *   n_parts    row-block partitions (the reference's `workers`,
 *              renderer.py:344-349), spread round-robin over ctx's devices;
 *              the frame does not depend on it;
 *   precision  RT_PREC_FP32 or RT_PREC_FP64.
 * Synchronous: the frame is complete in `pixels` on return. */
int rt_render_v1(rt_ctx *ctx, uint32_t *pixels, void *radiance, int32_t width, int32_t height,
                 const double cam_pos[3], double yaw, double pitch, double vdist, int32_t n_bodies,
                 const int32_t *kinds, const double *positions, const double *sizes, const double *colors,
                 const double *refls, const double light_pos[3], double light_radius, const double light_color[3],
                 double ambient, double max_refl, const float *sky, int32_t sky_w, int32_t sky_h, int32_t has_sky,
                 int32_t shadow_samples, int32_t bounce_limit, int32_t n_parts, int32_t precision);

/* Pipelined frames (the frame server's loop, server.py:276-289): enqueue a
 * frame exactly as rt_render_v1 renders it on the context's first device
 * (no radiance, one partition) into frame slot `slot` (0-3) and return at
 * once; the pixels land in the caller's `pixels` (page-locked for PCIe
 * speed: rt_host_register) once rt_frame_wait_v1(slot) returns.  Frames run
 * in submission order and each frame's device-to-host copy overlaps the next
 * frame's kernels.  The scene arguments are consumed before the call returns;
 * `pixels` must stay valid until the wait.  Submitting into a slot whose
 * frame was not waited for waits for it first. */
int rt_render_async_v1(rt_ctx *ctx, int32_t slot, uint32_t *pixels, int32_t width, int32_t height,
                       const double cam_pos[3], double yaw, double pitch, double vdist, int32_t n_bodies,
                       const int32_t *kinds, const double *positions, const double *sizes, const double *colors,
                       const double *refls, const double light_pos[3], double light_radius,
                       const double light_color[3], double ambient, double max_refl, const float *sky, int32_t sky_w,
                       int32_t sky_h, int32_t has_sky, int32_t shadow_samples, int32_t bounce_limit,
                       int32_t precision);
int rt_frame_wait_v1(rt_ctx *ctx, int32_t slot);

/* Device-resident render of one row-block partition with the scene last set
 * by rt_set_scene_v1 on device slot `slot`.  Row y is rendered iff
 * (y / block_rows) % n_parts == part; pixel (x, y) is stored at
 * d_out[y * out_pitch + x] — d_out may be a peer GPU's framebuffer mapped
 * through rt_ipc_open (the render then writes over NVLink, no gather pass).
 * Asynchronous on `stream` (a cudaStream_t; NULL = the slot's own stream). */
int rt_render_device_v1(rt_ctx *ctx, int32_t slot, uint32_t *d_out, int64_t out_pitch, void *d_radiance,
                        int32_t width, int32_t height, const double cam_pos[3], double yaw, double pitch,
                        double vdist, int32_t shadow_samples, int32_t bounce_limit, int32_t part, int32_t n_parts,
                        int32_t block_rows, int32_t precision, void *stream);

/* Batched `ray_trace_iterative` (renderer.py:303-313): out_rgb[i] is the
 * pre-quantisation colour of ray (origins[i], dirs[i]); host buffers,
 * float[n*3] (FP32) or double[n*3] (FP64).  Synchronous. */
int rt_trace_rays_v1(rt_ctx *ctx, const double *origins, const double *dirs, int64_t n_rays, void *out_rgb,
                     int32_t n_bodies, const int32_t *kinds, const double *positions, const double *sizes,
                     const double *colors, const double *refls, const double light_pos[3], double light_radius,
                     const double light_color[3], double ambient, double max_refl, const float *sky,
                     int32_t sky_w, int32_t sky_h, int32_t has_sky, int32_t shadow_samples, int32_t bounce_limit,
                     int32_t precision);

/* `skybox_sample` (renderer.py:60-79) for a batch of unit directions, in
 * float64 (bit-identical to the reference). Synchronous, host buffers. */
int rt_sky_sample_v1(rt_ctx *ctx, const double *dirs, int64_t n, double *out_rgb, const float *sky, int32_t sky_w,
                     int32_t sky_h);

/* Page-lock and map a host framebuffer: rt_render_v1 then writes it directly
 * from the kernels (option "zero_copy") or copies into it at PCIe speed.
 * The caller keeps the memory alive until unregistered.  Returns
 * RT_ALREADY_REGISTERED (> 0, not an error) when the range is already
 * page-locked by someone else — the caller then must not unregister it.  A
 * failed registration leaves no CUDA error pending.  ctx may be NULL (the
 * registration is process-wide: portable + mapped). */
#define RT_ALREADY_REGISTERED 1
int rt_host_register(rt_ctx *ctx, void *ptr, size_t bytes);
int rt_host_unregister(rt_ctx *ctx, void *ptr);

/* Execution options of ctx (default on: wave, cull, conic; the rest off):
 *   "wave"        FP32 soft shadows (samples >= 8) run as trace / shadow /
 *                 shade kernels over HBM queues instead of one megakernel;
 *   "cull"        the wavefront shadow pass skips, per hit, the bodies that
 *                 provably cannot block any of its shadow rays (exact);
 *   "conic"       the culled pass tests a penumbra sphere against the disc
 *                 samples in its silhouette form (six coefficients per hit
 *                 and sphere, a quadratic per sample) instead of one ray per
 *                 sample — the reference's predicate, FP32 rounding near the
 *                 silhouette (off: the ray form, bit-identical to "cull" 0);
 *   "cull_check"  (off) the culled pass leaves every body undecided, so each
 *                 hit is sampled against all of them by the same kernels: with
 *                 "conic" off, frames must equal the culled ones bit for bit;
 *   "count_work"  tally the executed work of the culled pass (rt_work_counts);
 *   "bands"       rt_render_v1 on one device renders this many contiguous row
 *                 bands (1-8), each on its own stream (band 0 at the highest
 *                 priority), and moves each to the host as soon as it is
 *                 done; 0 (default) = by frame size: with option "codec" 1
 *                 below 6 MB, 2 below 24 MB, else 6; raw, 1 below 1 MB, 2
 *                 below 24 MB, else 6;
 *   "band_first"  permille of the frame's rows in band 0 (0, default: equal
 *                 bands; the others always share the rest equally);
 *   "boxes"       (default on, with "cull") FP32 megakernel frames (under 8
 *                 samples) of up to 8 spheres: primary rays test only the
 *                 spheres whose conservative pixel box holds them (exact);
 *   "mega_tiles"  FP32 megakernel (frames under 8 shadow samples, or option
 *                 "wave" off): 1 one CTA per 16x8 tile, 0 persistent warps
 *                 taking 8x4 patches from a counter, -1 (default) tiles below
 *                 8 samples (15-20% faster at s1: no shared counter);
 *   "band_times"  record timed events at each band's kernel end and copy end
 *                 (rt_band_times_ms);
 *   "phases"      record CUDA events between the wavefront kernels so
 *                 rt_phase_ms can report per-phase device times (off by
 *                 default: each event record costs the GPU ~2-3 us);
 *   "rgba"        write pixels as bytes R,G,B,A (the frame server's wire
 *                 format, server.py:56-64) instead of 0xAARRGGBB;
 *   "sphere_bound" (default on; process-wide) FP32 scenes of 3-8 spheres: a
 *                 ray that misses a bound over every sphere skips the sphere
 *                 loop (exact: the clustered walk's bound test and margins;
 *                 trace kernel -3% at C2/C3);
 *   "hot_tiles"   (default on) the culled trace dispatches the tiles of the
 *                 spheres' primary-ray boxes first, frames of up to 8 waves;
 *   "zero_copy"   (default off) when the framebuffer passed to rt_render_v1
 *                 on one device is registered (rt_host_register), the
 *                 kernels store pixels straight into it over PCIe while they
 *                 compute — no copy after the frame, but measured 1.3-2.4x
 *                 slower end to end on B200 (PCIe writes of 32-byte rows
 *                 stall the kernels), so the staged copy is the default;
 *   "codec"       (default on) rt_render_v1 on one device and the pipelined
 *                 frames (rt_render_async_v1) move the finished pixels over
 *                 PCIe compressed, losslessly: each row's mask of pixels that
 *                 differ from their left neighbour and those pixels, written
 *                 by an encode kernel into mapped host memory, then expanded
 *                 into the caller's framebuffer by host threads (AVX2) — band
 *                 by band as each lands.  The frame is the same bit for bit;
 *                 C2 moves 0.33 MB instead of 3.7 (rt_last_d2h_bytes).  Off:
 *                 the raw copy.  Rows wider than 6,144 pixels always copy raw;
 *   "codec_threads" host threads expanding a compressed frame (0, default:
 *                 up to 16 of the OpenMP pool);
 *   "codec_parts" a one-band frame's encode in this many launches, each
 *                 expanded as it lands (0, default: 2 from 2 MB, else 1). */
int rt_set_option(rt_ctx *ctx, const char *name, int32_t value);
/* Executed-work tallies since the last reset (option "count_work"), in this
 * order: hits, per-hit cull tests, hits that sampled, shadow rays, sphere
 * tests, plane tests, bundle-traced rays, their sphere tests, warps whose
 * bundle did not cull, hits sampled in the silhouette form, their sphere
 * tests, hits sampled by the lane sampler (one lane per hit), silhouette
 * tests with the terminator (z) test. */
int rt_work_counts(rt_ctx *ctx, uint64_t *out, int32_t n, int32_t reset);

/* Bytes the last rt_render_v1 / rt_frame_wait_v1 frame moved from the device
 * to the host: the frame (and radiance) raw, or with option "codec" the
 * mask words and literals that crossed PCIe. */
int rt_last_d2h_bytes(rt_ctx *ctx, int64_t *bytes);

/* The host half of option "codec", on its own (no GPU needed): expand a
 * compressed frame host_buf into pixels (row pitch in pixels).  A pixel equal
 * to its left neighbour is a repeat, the others (a row's first pixel always)
 * literals.  In uint32 words, mw = ceil(width / 32), nb = ceil(mw / 32),
 * stride = 32 * ceil((1 + nb + mw + width) / 32), row y at 32 + y * stride:
 *   the literal count n | packed << 31;
 *   nb bitmap words, bit j: mask word j is non-zero and listed next;
 *   the listed mask words in order (bit i of mask word j: pixel 32 j + i is a
 *   literal; unlisted words are 0);
 *   the literals: packed, 3 bytes each (a pixel's low 3 bytes; its top byte
 *   is 0xFF), ceil(3 n / 4) words; else n words.
 * 32 words follow the last row (read, never used).  *words (may be NULL)
 * receives the words the rows' runs occupy — what crossed PCIe. */
int rt_frame_expand_v1(const uint32_t *host_buf, int32_t width, int32_t height, uint32_t *pixels, int64_t pitch,
                       int32_t threads, int64_t *words);

/* Device time (CUDA events) of the render kernels of the last rt_render_v1 /
 * rt_trace_rays_v1 call on ctx's first device, in milliseconds. */
int rt_last_kernel_ms(rt_ctx *ctx, float *ms);
/* Device time of the last wavefront frame's phases on ctx's first device, ms
 * (needs option "phases"):
 * out[0] trace, out[1] classify (culled path), out[2] shadow / sample,
 * out[3] shade.  Zeros when no wavefront frame ran. */
int rt_phase_ms(rt_ctx *ctx, float *out, int32_t n);
/* With option "band_times": for each row band of the last single-device
 * rt_render_v1, out[2k] = ms from the frame's start to the end of band k's
 * kernels and out[2k+1] = to the end of its device-to-host copy (n >= 2 *
 * bands).  Returns the number of bands (0: none timed), or a negative code. */
int rt_band_times_ms(rt_ctx *ctx, float *out, int32_t n);
/* Number of kernels this ctx has launched so far. */
int rt_launch_count(rt_ctx *ctx, int64_t *count);

/* CUDA IPC for the one-process-per-GPU row-band gather: export a device
 * allocation (64-byte handle), map a peer's allocation into this process. */
int rt_ipc_get_handle(void *d_ptr, uint8_t handle_out[64]);
int rt_ipc_open(const uint8_t handle[64], void **d_ptr_out);
int rt_ipc_close(void *d_ptr);

/* Synchronous device->host copy of `bytes` from d_src on `stream` (NULL = the
 * slot's stream): rank 0 reads the gathered frame back. */
int rt_copy_to_host(rt_ctx *ctx, int32_t slot, void *host_dst, const void *d_src, size_t bytes, void *stream);
/* Copy partition `part`'s rows (8-row blocks round-robin, as
 * rt_render_device_v1 renders them) of the device frame d_frame into the
 * host frame host_frame (same layout: pixel (x, y) at y * width + x), on
 * `stream` (null: the context's stream), and wait for it.  With one process
 * per GPU and host_frame a page-locked buffer shared by them, every GPU
 * copies its own rows over its own PCIe link.  With option
 * "codec" (default) the rows cross compressed and this process's threads
 * expand them (rt_last_d2h_bytes: what crossed). */
int rt_copy_partition_to_host(rt_ctx *ctx, int32_t slot, uint32_t *host_frame, const uint32_t *d_frame, int32_t width,
                              int32_t height, int32_t part, int32_t n_parts, int32_t block_rows, void *stream);

/* Plain device allocations (cudaMalloc) — IPC-exportable framebuffers. */
int rt_device_malloc(int32_t device, size_t bytes, void **d_ptr_out);
int rt_device_free(void *d_ptr);

/* Measured FP32 roofline denominator: dependent-free FFMA throughput of
 * `device` in TFLOP/s (2 FLOP per FFMA). */
int rt_fp32_peak_tflops(int32_t device, double *tflops);

#ifdef __cplusplus
}
#endif
#endif /* B200RT_H */
