// Host side of libb200rt: the C ABI of include/b200rt.h.
//
// Per-device context (stream, events, scene buffers, staging framebuffer),
// scene upload with change detection (the paper streams only per-frame state,
// PAPER.md:562-564), row-block partitioning over devices, and the copy of the
// finished frame into the caller's host framebuffer.  No pixel is ever
// computed here: every compute entry point launches a CUDA kernel or fails.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <omp.h>

#include "b200rt.h"
#include "frame_codec.h"
#include "rt_device.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define RT_CK(call)                                                                                        \
    do {                                                                                                   \
        cudaError_t e_ = (call);                                                                           \
        if (e_ != cudaSuccess) return fail(RT_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DBuf {
    void *p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap && p) return RT_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (bytes == 0) bytes = 16;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            p = nullptr;
            return fail(RT_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        }
        cap = bytes;
        return RT_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// Page-locked, mapped host memory: the compressed frame transfer's target
// (frame_codec.h), written by the encode kernel through its device address.
struct HBuf {
    void *p = nullptr, *dp = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap && p) return RT_OK;
        release();
        cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
        if (e == cudaSuccess) e = cudaHostGetDevicePointer(&dp, p, 0);
        if (e != cudaSuccess) {
            release();
            cudaGetLastError();
            return fail(RT_ERR_NOMEM, std::string("cudaHostAlloc (mapped): ") + cudaGetErrorString(e));
        }
        cap = bytes;
        return RT_OK;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = dp = nullptr;
        cap = 0;
    }
};

// Host-side canonical scene (float64, the reference's packed layout).
struct HostScene {
    int n = 0;
    std::vector<double> geo;  // [n][4] {cx, cy, cz, r^2} / {0, h, 0, -1}
    std::vector<double> mat;  // [n][8] {r, g, b, refl/max_refl, refl, 0, 0, 0}
    double light[3] = {0, 0, 0}, light_radius = 1, lc[3] = {1, 1, 1}, ambient = 0.15, max_refl = 128;
    std::vector<char> key;  // bytes compared to detect a changed scene
    uint64_t version = 0;
    // skybox: the caller's array and the hash of the texels last uploaded
    const float *sky_ptr = nullptr;
    int sky_w = 1, sky_h = 1, has_sky = 0;
    uint64_t sky_hash = 0;
    uint64_t sky_version = 0;
};

template <typename R>
struct DevScene {
    DBuf geo, mat, table;
    DBuf geo64;  // FP32 scenes: the geometry in float64 too (the kernels' ray chain, refine_hit)
    uint64_t version = ~0ull;
    int table_n = -1;
    double table_radius = NAN;
};

// Queues of one wavefront frame (or row band): FP32 wavefront / culled path
// (w_*) and FP64 culled path (d_*).
struct WaveBufs {
    DBuf w_p, w_n, w_s, w_sc, w_queue, w_queue2, w_mask2, w_count, w_pix, w_rec, w_pending, w_conic, w_lane;
    int count_parity = 0;  // culled FP32 path: which of its two counter sets this frame uses
    DBuf d_q, d_mask, d_pix, d_rec, d_parked, d_lane;
    void release() {
        for (DBuf *b : {&w_p, &w_n, &w_s, &w_sc, &w_queue, &w_queue2, &w_mask2, &w_count, &w_pix, &w_rec, &w_pending,
                        &w_conic, &w_lane, &d_q, &d_mask, &d_pix, &d_rec, &d_parked, &d_lane})
            b->release();
    }
};

constexpr int kMaxBands = 8;

struct Dev {
    int id = 0;
    int sm_count = 148;
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEvent_t pe0 = nullptr, pe1 = nullptr;  // the previous frame's pair while its time is still unread
    cudaEvent_t ph[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // wavefront phase boundaries
    cudaStream_t copy_st = nullptr;           // device->host copies of finished row bands
    cudaEvent_t band_ev[kMaxBands] = {};
    cudaEvent_t copy_ev[kMaxBands] = {};  // a band's copy done (on its own stream)
    // row bands run on their own streams, band 0 at the highest priority: the
    // next band's CTAs fill the SMs a band's tail leaves idle, yet the bands
    // finish in order, so each copy starts as early as it can
    cudaStream_t band_st[kMaxBands] = {};
    cudaEvent_t fork_ev = nullptr;
    cudaEvent_t tl_ev[2 * kMaxBands] = {};  // band_times: band k's kernels end, then its copy ends
    bool ph_valid = false;
    DBuf frame, rad, rays_in, rays_out, sky_raw, sky, counters, w_work;
    // pipelined frames (rt_render_async_v1): per slot a device frame, the
    // event its kernels end with and the event its host copy ends with
    static constexpr int kSlots = 4;
    DBuf slot_frame[kSlots];
    cudaEvent_t slot_comp[kSlots] = {}, slot_done[kSlots] = {};
    bool slot_busy[kSlots] = {};
    // compressed transfer (option codec): the mapped host buffer of
    // rt_render_v1's frames and of each slot, and what a slot's wait expands
    HBuf codec_host;
    HBuf part_codec;  // rt_copy_partition_to_host's
    HBuf slot_codec[kSlots];
    struct SlotOut {
        uint32_t *pixels = nullptr;
        int width = 0, height = 0;
        bool codec = false;
    } slot_out[kSlots];
    // rt_render_device_v1 on caller streams: the end of the last call's
    // kernels, and the end of this call's uploads
    cudaEvent_t dev_call_ev = nullptr, dev_prep_ev = nullptr;
    bool dev_call_pending = false;
    DBuf grid;                        // the culled FP32 path's shadow grid (scene + light)
    uint64_t grid_version = ~0ull;
    rt::WaveArgs grid_wa = {};        // its box and dims (grid null: none)
    WaveBufs wb[kMaxBands];
    unsigned counter_slot = 0;
    uint64_t sky_version = ~0ull;
    DevScene<float> s32;
    DevScene<double> s64;
};

// renderer.py:60-74 clamp, applied once per texel at upload: RGB -> float4.
__global__ void sky_to_float4(const float *raw, float4 *out, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float r = raw[3 * i], g = raw[3 * i + 1], b = raw[3 * i + 2];
    // min(max(c, 0), 1) keeps NaN out of the [0,1] range test like Python's min/max
    r = (0.f > r) ? 0.f : r;
    g = (0.f > g) ? 0.f : g;
    b = (0.f > b) ? 0.f : b;
    r = (1.f < r) ? 1.f : r;
    g = (1.f < g) ? 1.f : g;
    b = (1.f < b) ? 1.f : b;
    out[i] = make_float4(r, g, b, 0.f);
}

// Dependent-free FFMA stream: the measured FP32 roofline denominator.
__global__ void ffma_peak_kernel(float *sink, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
          x7 = x0 + 7;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) {
            x0 = fmaf(x0, a, b);
            x1 = fmaf(x1, a, b);
            x2 = fmaf(x2, a, b);
            x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b);
            x5 = fmaf(x5, a, b);
            x6 = fmaf(x6, a, b);
            x7 = fmaf(x7, a, b);
        }
    }
    float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5f) sink[threadIdx.x] = s;
}

}  // namespace

struct rt_ctx {
    std::vector<Dev> devs;
    bool wave = true;   // FP32 soft shadows take the wavefront path ($B200RT_WAVE=0: megakernel)
    bool cull = true;   // exact per-hit occluder culling in the wavefront shadow pass ($B200RT_CULL=0: off)
    bool count_work = false;  // tally the culled path's executed work (rt_work_counts)
    int bands = 0;            // single-device row bands for copy overlap (0: by frame size)
    int band_first = 0;       // permille of the rows in band 0 (0: equal bands)
    bool band_times = false;  // time each band's kernels and copy (rt_band_times_ms)
    float band_ms[2 * kMaxBands] = {};
    int band_count = 0;
    int band_pending = 0;     // bands of the frame enqueued by enqueue_frame (0: one stream)
    bool phases = false;      // record per-phase events in wavefront frames (rt_phase_ms)
    int rgba = 0;             // pixel byte order of the frames written (0 B,G,R,A / 1 R,G,B,A)
    bool conic = true;        // culled FP32 path: silhouette form of the soft-shadow sphere test
    bool cull_check = false;  // culled FP32 path: classify every body as undecided (an exactness check)
    bool zero_copy = false;   // kernels store straight into a registered (mapped) host framebuffer
    bool boxes = true;        // FP32 scenes of <= 8 spheres: primary-ray sphere boxes (with cull)
    int mega_tiles = -1;      // FP32 megakernel: 1 one CTA per tile, 0 persistent warps, -1 by sample count
    bool hot_tiles = true;    // culled FP32 trace: the spheres' tiles dispatched first
    int compact = 1;          // culled FP32 many-sphere trace: live rays packed between deep bounces
    int band_order = 0;       // copy-overlap bands enqueued 0: top first, 1: bottom first (measured slower)
    int codec = 1;            // host frames cross PCIe compressed (frame_codec.h) and are expanded here
    int codec_threads = 0;    // host threads expanding a frame (0: up to 16 of the OpenMP pool)
    int codec_parts = 0;      // one render band: its encode cut into this many launches (0: 2 from 2 MB)
    // the frame enqueue_frame left for finish_frame to expand (one device)
    struct CodecFrame {
        bool on = false;
        uint32_t *pixels = nullptr;
        int width = 0, height = 0, bands = 0;
        int y_at[kMaxBands + 1] = {};
        int order[kMaxBands] = {};
        bool radiance = false;  // copied raw alongside (finish_frame waits for it)
    } codec_frame;
    int64_t last_d2h_bytes = 0;  // bytes the last frame moved device -> host
    // a compressed frame returns once its last band is expanded: its device
    // time (events ms_e0 -> ms_e1) is read later, off the caller's path
    bool ms_pending = false;
    cudaEvent_t ms_e0 = nullptr, ms_e1 = nullptr;
    std::mutex mu;
    HostScene scene;
    float last_ms = 0.f;
    int64_t launches = 0;
};

namespace {

double golden_angle() { return M_PI * (3.0 - std::sqrt(5.0)); }  // shading.py:29

// shading.py:89-100: (r_i cos th_i, r_i sin th_i) in float64 with the host libm.
std::vector<double> disc_table(int n, double radius) {
    std::vector<double> t(2 * (size_t)n);
    double ga = golden_angle();
    for (int i = 0; i < n; i++) {
        double r = 2.0 * radius * std::sqrt((double)i / (double)n);
        double theta = (double)i * ga;
        t[2 * i] = r * std::cos(theta);
        t[2 * i + 1] = r * std::sin(theta);
    }
    return t;
}

// The skybox is read by the reference on every frame (renderer.py:282-300),
// so an in-place edit of its texels must show in the next frame.  The
// library hashes the caller's texels in full on every frame that reuses the
// same array and compares the hash with that of the texels it uploaded: a
// 64-bit xxh64-style hash (four multiply-rotate lanes per chunk, chunks
// chained in order, so content and position both count), computed over all
// host cores — it reads the array once, where comparing against a kept copy
// read twice the bytes (C3 end to end: the 25 MB compare was the bottleneck,
// 310-470 us by thread count, tools/micro/host_hash.c).  rt_render_v1 runs the
// hash while the frame's kernels execute (the frame is rendered with the
// device copy); a different hash re-uploads the sky and renders the frame
// again before the call returns.
int sky_threads() {
    static int t = [] {
        if (const char *e = std::getenv("B200RT_SKY_THREADS")) return std::max(1, std::atoi(e));
        return std::max(1, std::min(32, omp_get_num_procs()));
    }();
    return t;
}

constexpr uint64_t kP1 = 0x9E3779B185EBCA87ull, kP2 = 0xC2B2AE3D27D4EB4Full, kP3 = 0x165667B19E3779F9ull,
                   kP4 = 0x85EBCA77C2B2AE63ull;
inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
inline uint64_t hround(uint64_t acc, uint64_t w) { return rotl64(acc + w * kP2, 31) * kP1; }
inline uint64_t hmerge(uint64_t h, uint64_t v) { return (h ^ hround(0, v)) * kP1 + kP4; }

// xxh64-style hash of n bytes (n a multiple of 4) at p with a seed
uint64_t hash_bytes(const char *p, size_t n, uint64_t seed) {
    uint64_t v1 = seed + kP1 + kP2, v2 = seed + kP2, v3 = seed, v4 = seed - kP1;
    size_t i = 0;
    for (; i + 32 <= n; i += 32) {
        uint64_t w[4];
        std::memcpy(w, p + i, 32);
        v1 = hround(v1, w[0]);
        v2 = hround(v2, w[1]);
        v3 = hround(v3, w[2]);
        v4 = hround(v4, w[3]);
    }
    uint64_t h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
    h = hmerge(hmerge(hmerge(hmerge(h, v1), v2), v3), v4) + n;
    for (; i + 8 <= n; i += 8) {
        uint64_t w;
        std::memcpy(&w, p + i, 8);
        h = rotl64(h ^ hround(0, w), 27) * kP1 + kP4;
    }
    for (; i + 4 <= n; i += 4) {
        uint32_t w;
        std::memcpy(&w, p + i, 4);
        h = rotl64(h ^ (uint64_t)w * kP1, 23) * kP2 + kP3;
    }
    h ^= h >> 33;
    h *= kP2;
    h ^= h >> 29;
    h *= kP3;
    return h ^ (h >> 32);
}

// the texels' hash: chunks hashed independently (on all host threads, or by
// the compressed frame's expansion team while it waits), chained in order
struct TexelHash {
    const float *a;
    size_t bytes;
    int chunks;
    std::vector<uint64_t> part;
    TexelHash(const float *a_, size_t n) : a(a_), bytes(sizeof(float) * n), chunks(4 * sky_threads()), part(chunks) {}
    void chunk(int k) {
        const size_t lo = bytes * k / chunks / 4 * 4, hi = bytes * (k + 1) / chunks / 4 * 4;
        part[k] = hash_bytes((const char *)a + lo, (k == chunks - 1 ? bytes : hi) - lo, (uint64_t)k);
    }
    static void run(void *self, int k) { static_cast<TexelHash *>(self)->chunk(k); }
    uint64_t value() const {
        uint64_t h = 0x27D4EB2F165667C5ull;
        for (int k = 0; k < chunks; k++) h = hround(h, part[k] ^ (uint64_t)k);
        return h ^ bytes;
    }
};

uint64_t texel_hash(const float *a, size_t n) {
    TexelHash t(a, n);
#pragma omp parallel for num_threads(sky_threads()) schedule(static)
    for (int k = 0; k < t.chunks; k++) t.chunk(k);
    return t.value();
}

// The caller's texels (same array as the last frame's) against the uploaded
// ones; on a difference the sky version is bumped (upload_sky re-uploads).
bool sky_hash_differs(HostScene &s, uint64_t h) {
    if (h == s.sky_hash) return false;
    s.sky_hash = h;
    s.sky_version++;
    return true;
}

bool sky_content_changed(HostScene &s) {
    if (!s.has_sky || !s.sky_ptr) return false;
    return sky_hash_differs(s, texel_hash(s.sky_ptr, (size_t)s.sky_w * s.sky_h * 3));
}

int validate_scene(int32_t n_bodies, const int32_t *kinds, const double *positions, const double *sizes,
                   const double *colors, const double *refls, const double *light_pos, const double *light_color,
                   double max_refl, const float *sky, int32_t sky_w, int32_t sky_h, int32_t has_sky) {
    if (n_bodies < 0) return fail(RT_ERR_INVALID, "n_bodies must be >= 0");
    if (n_bodies > 0 && (!kinds || !positions || !sizes || !colors || !refls))
        return fail(RT_ERR_INVALID, "null scene array");
    if (!light_pos || !light_color) return fail(RT_ERR_INVALID, "null light array");
    if (!(max_refl > 0)) return fail(RT_ERR_INVALID, "max reflectivity must be positive");
    for (int i = 0; i < n_bodies; i++) {
        if (kinds[i] != 0 && kinds[i] != 1) return fail(RT_ERR_INVALID, "body kind must be 0 (sphere) or 1 (plane)");
        if (kinds[i] == 0 && !(sizes[i] > 0)) return fail(RT_ERR_INVALID, "sphere radius must be positive");
    }
    if (has_sky && (!sky || sky_w < 1 || sky_h < 1)) return fail(RT_ERR_INVALID, "bad skybox");
    return RT_OK;
}

// Returns true when the frame reuses the last frame's sky array, whose
// content the caller must still compare (sky_content_changed).
bool set_host_scene(HostScene &s, int32_t n, const int32_t *kinds, const double *positions, const double *sizes,
                    const double *colors, const double *refls, const double *light_pos, double light_radius,
                    const double *light_color, double ambient, double max_refl, const float *sky, int32_t sky_w,
                    int32_t sky_h, int32_t has_sky) {
    std::vector<char> key;
    auto put = [&key](const void *p, size_t b) {
        const char *c = (const char *)p;
        key.insert(key.end(), c, c + b);
    };
    put(&n, sizeof n);
    if (n > 0) {
        put(kinds, sizeof(int32_t) * n);
        put(positions, sizeof(double) * 3 * n);
        put(sizes, sizeof(double) * n);
        put(colors, sizeof(double) * 3 * n);
        put(refls, sizeof(double) * n);
    }
    put(light_pos, sizeof(double) * 3);
    put(&light_radius, sizeof light_radius);
    put(light_color, sizeof(double) * 3);
    put(&ambient, sizeof ambient);
    put(&max_refl, sizeof max_refl);
    if (key != s.key) {
        s.key.swap(key);
        s.n = n;
        s.geo.assign(4 * (size_t)n, 0.0);
        s.mat.assign(8 * (size_t)n, 0.0);
        for (int i = 0; i < n; i++) {
            if (kinds[i] == 0) {
                s.geo[4 * i] = positions[3 * i];
                s.geo[4 * i + 1] = positions[3 * i + 1];
                s.geo[4 * i + 2] = positions[3 * i + 2];
                s.geo[4 * i + 3] = sizes[i] * sizes[i];  // geometry.py:97 radius * radius
            } else {
                s.geo[4 * i + 1] = positions[3 * i + 1];  // plane height = position.y (geometry.py:58-60)
                s.geo[4 * i + 3] = -1.0;
            }
            s.mat[8 * i] = colors[3 * i];
            s.mat[8 * i + 1] = colors[3 * i + 1];
            s.mat[8 * i + 2] = colors[3 * i + 2];
            s.mat[8 * i + 3] = refls[i] / max_refl;  // renderer.py:161
            s.mat[8 * i + 4] = refls[i];
        }
        for (int c = 0; c < 3; c++) {
            s.light[c] = light_pos[c];
            s.lc[c] = light_color[c];
        }
        s.light_radius = light_radius;
        s.ambient = ambient;
        s.max_refl = max_refl;
        s.version++;
    }
    // a different array (or none): a new sky, hashed and uploaded; the same
    // array: its content is hashed in full again (sky_content_changed)
    if (has_sky != s.has_sky || (has_sky && (sky != s.sky_ptr || sky_w != s.sky_w || sky_h != s.sky_h))) {
        s.has_sky = has_sky;
        s.sky_ptr = has_sky ? sky : nullptr;
        s.sky_w = has_sky ? sky_w : 1;
        s.sky_h = has_sky ? sky_h : 1;
        s.sky_hash = has_sky ? texel_hash(sky, (size_t)sky_w * sky_h * 3) : 0;
        s.sky_version++;
        return false;
    }
    return has_sky != 0;
}

template <typename R>
int upload_prec(Dev &d, DevScene<R> &ds, const HostScene &s, int samples) {
    if (ds.version != s.version) {
        std::vector<R> geo(s.geo.begin(), s.geo.end()), mat(s.mat.begin(), s.mat.end());
        int rc;
        if ((rc = ds.geo.ensure(sizeof(R) * geo.size())) || (rc = ds.mat.ensure(sizeof(R) * mat.size()))) return rc;
        // FP32 kernels: the float64 geometry (refine_hit) — {c, r^2} / {0, h, 0, -1}, then 1/r per body
        std::vector<double> geo64(s.geo);
        for (int b = 0; b < s.n; b++) geo64.push_back(s.geo[4 * b + 3] > 0.0 ? 1.0 / std::sqrt(s.geo[4 * b + 3]) : 0.0);
        if (sizeof(R) != sizeof(double) && (rc = ds.geo64.ensure(sizeof(double) * std::max<size_t>(geo64.size(), 1))))
            return rc;
        if (!geo.empty()) {
            RT_CK(cudaMemcpyAsync(ds.geo.p, geo.data(), sizeof(R) * geo.size(), cudaMemcpyHostToDevice, d.st));
            RT_CK(cudaMemcpyAsync(ds.mat.p, mat.data(), sizeof(R) * mat.size(), cudaMemcpyHostToDevice, d.st));
            if (sizeof(R) != sizeof(double))
                RT_CK(cudaMemcpyAsync(ds.geo64.p, geo64.data(), sizeof(double) * geo64.size(), cudaMemcpyHostToDevice,
                                      d.st));
        }
        RT_CK(cudaStreamSynchronize(d.st));  // host vectors die at scope exit
        ds.version = s.version;
    }
    if (samples > 1 && (ds.table_n != samples || !(ds.table_radius == s.light_radius))) {
        std::vector<double> t64 = disc_table(samples, s.light_radius);
        // FP64 kernel: {a_i, b_i}; FP32 kernels: {a_i, b_i, a_i^2 + b_i^2, 0} (float4 loads)
        const int comp = sizeof(R) == sizeof(double) ? 2 : 4;
        std::vector<R> t((size_t)comp * samples, R(0));
        for (int i = 0; i < samples; i++) {
            double a = t64[2 * i], b = t64[2 * i + 1];
            t[comp * i] = (R)a;
            t[comp * i + 1] = (R)b;
            if (comp == 4) t[comp * i + 2] = (R)(a * a + b * b);
        }
        int rc = ds.table.ensure(sizeof(R) * t.size());
        if (rc) return rc;
        RT_CK(cudaMemcpyAsync(ds.table.p, t.data(), sizeof(R) * t.size(), cudaMemcpyHostToDevice, d.st));
        RT_CK(cudaStreamSynchronize(d.st));
        ds.table_n = samples;
        ds.table_radius = s.light_radius;
    }
    return RT_OK;
}

int upload_sky(rt_ctx *ctx, Dev &d) {
    const HostScene &s = ctx->scene;
    if (d.sky_version == s.sky_version) return RT_OK;
    int rc;
    if (s.has_sky) {
        int64_t n = (int64_t)s.sky_w * s.sky_h;
        if ((rc = d.sky_raw.ensure(sizeof(float) * 3 * n)) || (rc = d.sky.ensure(sizeof(float4) * n))) return rc;
        // from the caller's array, whose hash is s.sky_hash (the call is synchronous: it does not change meanwhile)
        RT_CK(cudaMemcpyAsync(d.sky_raw.p, s.sky_ptr, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, d.st));
        sky_to_float4<<<(unsigned)((n + 255) / 256), 256, 0, d.st>>>((const float *)d.sky_raw.p, (float4 *)d.sky.p,
                                                                   n);
        RT_CK(cudaGetLastError());
        ctx->launches++;
        RT_CK(cudaStreamSynchronize(d.st));
        d.sky_raw.release();
    } else {
        if ((rc = d.sky.ensure(sizeof(float4)))) return rc;
        RT_CK(cudaMemsetAsync(d.sky.p, 0, sizeof(float4), d.st));
    }
    d.sky_version = s.sky_version;
    return RT_OK;
}

// Every device's sky up to date before a call returns: the library keeps no
// host copy of the texels (only their hash), so a device that did not take
// part in this call's frame must not be left to upload later from an array
// the caller may since have freed.
int upload_sky_all(rt_ctx *ctx) {
    int rc;
    for (Dev &d : ctx->devs) {
        if (d.sky_version == ctx->scene.sky_version) continue;
        RT_CK(cudaSetDevice(d.id));
        if ((rc = upload_sky(ctx, d))) return rc;
    }
    return RT_OK;
}

template <typename R>
rt::SceneArgs<R> scene_args(const Dev &d, const DevScene<R> &ds, const HostScene &s) {
    rt::SceneArgs<R> a;
    a.geo = (const R *)ds.geo.p;
    a.mat = (const R *)ds.mat.p;
    a.table = (const R *)ds.table.p;
    a.sky = (const float4 *)d.sky.p;
    a.sky_w = s.sky_w;
    a.sky_h = s.sky_h;
    a.has_sky = s.has_sky;
    a.n = s.n;
    for (int c = 0; c < 3; c++) {
        a.light[c] = (R)s.light[c];
        a.lc[c] = (R)s.lc[c];
    }
    a.light_radius = (R)s.light_radius;
    a.ambient = (R)s.ambient;
    a.host_geo = s.geo.data();
    a.geo64 = sizeof(R) == sizeof(double) ? (const double *)ds.geo.p : (const double *)ds.geo64.p;
    return a;
}

int count_spheres(const HostScene &s) {
    int ns = 0;
    for (int b = 0; b < s.n; b++) ns += s.geo[4 * b + 3] >= 0.0 ? 1 : 0;
    return ns;
}

int prepare(rt_ctx *ctx, Dev &d, int precision, int samples) {
    int rc;
    RT_CK(cudaSetDevice(d.id));
    if ((rc = upload_sky(ctx, d))) return rc;
    if (precision == RT_PREC_FP64) return upload_prec(d, d.s64, ctx->scene, samples);
    if ((rc = upload_prec(d, d.s32, ctx->scene, samples))) return rc;
    // the culled path's shadow grid, rebuilt on d.st when the scene or the
    // light changed (before any row band forks off d.st)
    if (ctx->cull && d.grid_version != ctx->scene.version) {
        if ((rc = d.grid.ensure(sizeof(unsigned) * rt::kGridCells))) return rc;
        d.grid_wa = {};
        cudaError_t e = rt_build_shadow_grid_f32(scene_args(d, d.s32, ctx->scene), (unsigned *)d.grid.p,
                                                 rt::kGridCells, d.grid_wa, d.st);
        if (e != cudaSuccess) return fail(RT_ERR_CUDA, std::string("shadow grid: ") + cudaGetErrorString(e));
        d.grid_version = ctx->scene.version;
    }
    return RT_OK;
}

// Rows of partition `part`, rounded up to whole blocks (the kernel skips rows
// past the frame).
int local_rows(int height, int part, int n_parts, int block_rows) {
    if (n_parts == 1) return height;
    int n_blocks = (height + block_rows - 1) / block_rows;
    int mine = n_blocks > part ? (n_blocks - part + n_parts - 1) / n_parts : 0;
    return mine * block_rows;
}

rt::FrameArgs frame_args(uint32_t *out, int64_t pitch, void *rad, int w, int h, const double *cam, double yaw,
                         double pitch_angle, double vdist, int samples, int bounces, int part, int n_parts,
                         int block_rows) {
    rt::FrameArgs fa;
    fa.out = out;
    fa.out_pitch = pitch;
    fa.radiance = rad;
    fa.width = w;
    fa.height = h;
    fa.part = part;
    fa.n_parts = n_parts;
    fa.block_rows = block_rows;
    fa.local_rows = local_rows(h, part, n_parts, block_rows);
    for (int c = 0; c < 3; c++) fa.cam[c] = cam[c];
    fa.cb = std::cos(pitch_angle);  // vecmath.py:101-106, host libm
    fa.sb = std::sin(pitch_angle);
    fa.ca = std::cos(yaw);
    fa.sa = std::sin(yaw);
    fa.vdist = vdist;
    // camera.py:46-54 as one FMA per coordinate (the FP32 kernels round the
    // direction to float anyway; the FP64 kernel keeps the literal formula)
    {
        double W = w, Hh = h;
        if (W > Hh) {
            fa.ndc[0] = 2.0 / Hh;
            fa.ndc[1] = (Hh / 2 - W / 2) / Hh * 2 - 1;
            fa.ndc[2] = -2.0 / Hh;
            fa.ndc[3] = 1.0;
        } else {
            fa.ndc[0] = 2.0 / W;
            fa.ndc[1] = -1.0;
            fa.ndc[2] = -2.0 / W;
            fa.ndc[3] = -((W / 2 - Hh / 2) / W * 2 - 1);
        }
    }
    fa.samples = samples;
    fa.bounces = bounces;
    fa.peer_out = 0;
    fa.work_counter = nullptr;
    fa.sub_part = 0;
    fa.sub_parts = 1;
    fa.row_end = h;
    fa.row0 = 0;
    fa.rgba = 0;
    return fa;
}

// Queue counters: [0, 8) the FP64 and unculled paths (zeroed per frame),
// [8, 16) and [16, 24) the culled FP32 path's two sets (each frame's trace
// zeroes the other set once the previous frame is done: no memset per frame).
int ensure_counts(WaveBufs &b, cudaStream_t st) {
    if (b.w_count.p && b.w_count.cap >= 32 * sizeof(unsigned)) return RT_OK;
    int rc = b.w_count.ensure(32 * sizeof(unsigned));
    if (rc) return rc;
    RT_CK(cudaMemsetAsync(b.w_count.p, 0, 32 * sizeof(unsigned), st));
    b.count_parity = 0;
    return RT_OK;
}

// Per sphere of a scene of up to 8, the pixels whose primary ray can hit it
// (FrameArgs::box): the rays within angle asin(r'/D) of the direction to the
// centre (D away, r' = r inflated well past the FP32 test's rounding and the
// graze tolerance), bounded in camera space by the planes through the eye
// holding an image axis (A s^2 - 2 a.z a s + a^2 - sin^2 = 0 for the slope s
// of each bounding plane), mapped to pixels and padded by two.  A sphere
// behind the eye gets an empty box; one the eye is in or near, or whose cone
// reaches the image plane's horizon, the whole frame.  Exact: a ray outside
// the box misses the sphere in the kernels' own test.
void primary_boxes(rt::MegaCull &mc, const rt::FrameArgs &fa, const HostScene &s) {
    mc.nbox = 0;
    int nb = 0;
    for (int b = 0; b < s.n; b++) nb += s.geo[4 * b + 3] >= 0.0 ? 1 : 0;
    if (nb == 0 || nb > 8) return;
    const double W = fa.width, H = fa.height;
    int k = 0;
    for (int b = 0; b < s.n; b++) {
        const double *g = &s.geo[4 * b];
        if (g[3] < 0.0) continue;
        int *bx = mc.box[k++];
        bx[0] = bx[1] = -1;  // the whole frame
        bx[2] = fa.width;
        bx[3] = fa.height;
        const double r = std::sqrt(g[3]);
        const double wx = g[0] - fa.cam[0], wy = g[1] - fa.cam[1], wz = g[2] - fa.cam[2];
        // world -> camera: undo the yaw, then the pitch (camera.py:70-77 inverted)
        const double cx = wx * fa.ca - wz * fa.sa, z2 = wx * fa.sa + wz * fa.ca;
        const double cy = wy * fa.cb + z2 * fa.sb, cz = -wy * fa.sb + z2 * fa.cb;
        const double D = std::sqrt(cx * cx + cy * cy + cz * cz);
        const double re = r * (1.0 + 1e-3) + 1e-3 + 1e-5 * D;
        if (!(D > 1.001 * re)) continue;
        const double sn = re / D, ax = cx / D, ay = cy / D, az = cz / D;
        if (az < -sn) {  // wholly behind the eye: primary rays point forward
            bx[0] = bx[1] = 1;
            bx[2] = bx[3] = 0;
            continue;
        }
        if (!(az - sn > 1e-3)) continue;
        const double A = az * az - sn * sn;
        auto slopes = [&](double a, double &lo, double &hi) {
            const double B = a * az, sq = std::sqrt(std::max(B * B - A * (a * a - sn * sn), 0.0));
            lo = (B - sq) / A;
            hi = (B + sq) / A;
        };
        double s0, s1, t0, t1;
        slopes(ax, s0, s1);
        slopes(ay, t0, t1);
        // u = vdist * s = x * ndc0 + ndc1, v = vdist * t = y * ndc2 + ndc3 (camera.py:46-54)
        const double xa = (fa.vdist * s0 - fa.ndc[1]) / fa.ndc[0], xb = (fa.vdist * s1 - fa.ndc[1]) / fa.ndc[0];
        const double ya = (fa.vdist * t0 - fa.ndc[3]) / fa.ndc[2], yb = (fa.vdist * t1 - fa.ndc[3]) / fa.ndc[2];
        if (!std::isfinite(xa) || !std::isfinite(xb) || !std::isfinite(ya) || !std::isfinite(yb)) continue;
        auto clampd = [](double v, double lo, double hi) { return std::min(std::max(v, lo), hi); };
        bx[0] = (int)clampd(std::floor(std::min(xa, xb)) - 2.0, -1.0, W);
        bx[2] = (int)clampd(std::ceil(std::max(xa, xb)) + 2.0, -1.0, W);
        bx[1] = (int)clampd(std::floor(std::min(ya, yb)) - 2.0, -1.0, H);
        bx[3] = (int)clampd(std::ceil(std::max(ya, yb)) + 2.0, -1.0, H);
    }
    mc.nbox = nb;
}

// A frame's tile dispatch order (rt_device.cuh tile_of_block): the tiles of
// the spheres' primary-ray boxes (their union's bounding rectangle) first —
// where the bounce chains, penumbrae and shadow rays are — then the rest, so
// the cheap tiles fill the last wave.  It pays where the last wave is a
// large part of the kernel (C2, ~6 waves of 8 resident CTAs per SM: trace
// -4 to -9%); over more waves the other order's locality wins (C3 +3%, C4
// +4%): hot first up to 8 waves, one contiguous partition, scenes of up to 8
// spheres (option hot_tiles).  {-1, ...}: bottom rows first.  The culled
// trace only: the hard-shadow tile megakernel measured slower with it.
int4 hot_rect(rt_ctx *ctx, const Dev &d, const rt::FrameArgs &fa) {
    const int tw = (fa.width + rt::kTileW - 1) / rt::kTileW, th = (fa.local_rows + rt::kTileH - 1) / rt::kTileH;
    if (!ctx->hot_tiles || fa.n_parts != 1 || fa.sub_parts > 1 || count_spheres(ctx->scene) > 8 ||
        (int64_t)tw * th > (int64_t)8 * 8 * d.sm_count)
        return make_int4(-1, -1, -1, -1);
    rt::MegaCull mc = {};
    primary_boxes(mc, fa, ctx->scene);
    int x0 = 1 << 30, y0 = 1 << 30, x1 = -1, y1 = -1;
    for (int b = 0; b < mc.nbox; b++) {
        if (mc.box[b][0] > mc.box[b][2] || mc.box[b][1] > mc.box[b][3]) continue;  // behind the eye
        x0 = std::min(x0, mc.box[b][0]);
        y0 = std::min(y0, mc.box[b][1]);
        x1 = std::max(x1, mc.box[b][2]);
        y1 = std::max(y1, mc.box[b][3]);
    }
    if (x1 < 0) return make_int4(-1, -1, -1, -1);
    const int tx0 = std::max(0, x0 / rt::kTileW), tx1 = std::min(tw - 1, x1 / rt::kTileW);
    const int ty0 = std::max(0, (y0 - fa.row0) / rt::kTileH), ty1 = std::min(th - 1, (y1 - fa.row0) / rt::kTileH);
    return tx0 <= tx1 && ty0 <= ty1 ? make_int4(tx0, ty0, tx1, ty1) : make_int4(-1, -1, -1, -1);
}

// $B200RT_HOST_TIMING: where a synchronous call's host time goes (rt_render_v1 prints it)
bool host_timing_on() {
    static const bool on = std::getenv("B200RT_HOST_TIMING") != nullptr;
    return on;
}
std::chrono::steady_clock::time_point g_t_first_launch, g_t_team_start, g_t_team_end, g_t_sync1, g_t_sync2,
    g_t_elapsed;
bool g_first_launch_pending = false;
inline void stamp(std::chrono::steady_clock::time_point &t) {
    if (host_timing_on()) t = std::chrono::steady_clock::now();
}

int launch_frame(rt_ctx *ctx, Dev &d, rt::FrameArgs fa, int precision, cudaStream_t st, int buf = 0) {
    if (g_first_launch_pending) {
        stamp(g_t_first_launch);
        g_first_launch_pending = false;
    }
    WaveBufs &b = d.wb[buf];
    cudaError_t e;
    fa.rgba = ctx->rgba;
    if (fa.local_rows == 0) return RT_OK;
    int rc = RT_OK;
    d.ph_valid = false;
    // queued hits carry their record slot (bounce * pixels + pixel) in 31 bits:
    // larger frame x bounce products take the megakernels, which queue nothing
    const bool slots_fit = (int64_t)fa.local_rows * fa.width * (fa.bounces + 1) < ((int64_t)1 << 31);
    if (precision == RT_PREC_FP64 && fa.samples >= rt::kWaveMinSamples && ctx->wave && ctx->cull && slots_fit &&
        ctx->scene.n <= rt::kMaxBodies64) {
        rt::WaveArgs64 wa = {};
        wa.n_pix = (int64_t)fa.local_rows * fa.width;
        size_t slots = (size_t)wa.n_pix * (fa.bounces + 1);
        if ((rc = b.d_q.ensure(2 * sizeof(double4) * slots)) ||
            (rc = b.d_mask.ensure(sizeof(unsigned) * slots * (rt::kMaxBodies64 / 32))) ||
            (rc = b.d_pix.ensure(sizeof(double4) * (size_t)wa.n_pix)) || (rc = b.d_rec.ensure(sizeof(double4) * slots)) ||
            (rc = b.d_parked.ensure(sizeof(int) * (size_t)wa.n_pix)) || (rc = ensure_counts(b, st)))
            return rc;
        wa.q = (double4 *)b.d_q.p;
        wa.mask = (unsigned *)b.d_mask.p;
        wa.mask_stride = (int64_t)slots;
        wa.count = (unsigned *)b.w_count.p;
        wa.pix = (double4 *)b.d_pix.p;
        wa.rec = (double4 *)b.d_rec.p;
        wa.parked = (int *)b.d_parked.p;
        if (ctx->conic) {  // single-sphere hits sampled one lane each (render_fused_f64.cu)
            if ((rc = b.d_lane.ensure(2 * sizeof(double4) * (size_t)wa.n_pix))) return rc;
            wa.lane_q = (double4 *)b.d_lane.p;
            wa.lane_cap = (unsigned)wa.n_pix;
        }
        int nk = 0;
        e = rt_launch_fused_f64(fa, scene_args(d, d.s64, ctx->scene), wa, st, &nk);
        ctx->launches += nk - 1;
    } else if (precision == RT_PREC_FP64) {
        e = rt_launch_render_f64(fa, scene_args(d, d.s64, ctx->scene), st);
    } else if (fa.samples >= rt::kWaveMinSamples && ctx->wave && slots_fit) {
        const rt::SceneArgs<float> sa = scene_args(d, d.s32, ctx->scene);
        const bool fused = ctx->cull && rt_fused_fits(sa);
        rt::WaveArgs wa = {};
        wa.n_pix = (int64_t)fa.local_rows * fa.width;
        size_t slots = (size_t)wa.n_pix * (fa.bounces + 1);
        if ((rc = b.w_p.ensure(sizeof(float4) * slots)) || (rc = b.w_n.ensure(sizeof(float4) * slots)) ||
            (rc = ensure_counts(b, st)) || (rc = b.w_pix.ensure(sizeof(float4) * (size_t)wa.n_pix)))
            return rc;
        if (fused) {
            if ((rc = b.w_queue2.ensure(sizeof(int) * slots)) ||
                (rc = b.w_mask2.ensure(sizeof(unsigned) * slots * rt::rt_mask_words(count_spheres(ctx->scene)))) ||
                (rc = b.w_rec.ensure(sizeof(float4) * slots)) ||
                (rc = b.w_pending.ensure(sizeof(unsigned long long) * (size_t)wa.n_pix)))  // pend / pend64
                return rc;
            if (ctx->conic) {  // silhouette coefficients for the first n_pix queued hits
                if ((rc = b.w_conic.ensure(sizeof(float4) * 2 * rt::kConic * (size_t)wa.n_pix))) return rc;
                wa.conic = (float4 *)b.w_conic.p;
                wa.conic_cap = (unsigned)wa.n_pix;
                if ((rc = b.w_lane.ensure(sizeof(float4) * 4 * (size_t)wa.n_pix))) return rc;
                wa.lane_q = (float4 *)b.w_lane.p;
                wa.lane_cap = (unsigned)wa.n_pix;
            }
        } else {
            if ((rc = b.w_s.ensure(sizeof(float) * slots)) || (rc = b.w_sc.ensure(sizeof(float) * slots)) ||
                (rc = b.w_queue.ensure(sizeof(int) * slots)))
                return rc;
        }
        wa.hit_p = (float4 *)b.w_p.p;
        wa.hit_n = (float4 *)b.w_n.p;
        wa.hit_s = (float *)b.w_s.p;
        wa.hit_sc = (float *)b.w_sc.p;
        wa.queue = (int *)b.w_queue.p;
        wa.count = (unsigned *)b.w_count.p;
        wa.queue2 = (int *)b.w_queue2.p;
        wa.mask2 = (unsigned *)b.w_mask2.p;
        wa.mask2_stride = (int64_t)slots;
        wa.pix = (float4 *)b.w_pix.p;
        wa.rec = (float4 *)b.w_rec.p;
        wa.pend = (int *)b.w_pending.p;
        wa.pend64 = (unsigned long long *)b.w_pending.p;
        wa.cull = fused ? (ctx->cull_check ? 2 : 1) : 0;
        if (fused) {
            wa.count = (unsigned *)b.w_count.p + 8 + 8 * b.count_parity;
            wa.count_next = (unsigned *)b.w_count.p + 8 + 8 * (1 - b.count_parity);
            b.count_parity ^= 1;
        }
        if (fused && d.grid_version == ctx->scene.version && d.grid_wa.grid) {
            wa.grid = d.grid_wa.grid;
            for (int a = 0; a < 3; a++) {
                wa.grid_lo[a] = d.grid_wa.grid_lo[a];
                wa.grid_inv[a] = d.grid_wa.grid_inv[a];
                wa.grid_dim[a] = d.grid_wa.grid_dim[a];
            }
        }
        wa.hot = fused ? hot_rect(ctx, d, fa) : make_int4(-1, -1, -1, -1);
        if (wa.hot.x >= 0) {
            const int tw = (fa.width + rt::kTileW - 1) / rt::kTileW, rw = wa.hot.z - wa.hot.x + 1;
            wa.hot_div[0] = rt::tile_divisor(tw);
            wa.hot_div[1] = rt::tile_divisor(rw);
            wa.hot_div[2] = rt::tile_divisor(tw - rw);
        }
        wa.compact = ctx->compact;
        wa.work = nullptr;
        if (ctx->count_work) {
            bool fresh = d.w_work.p == nullptr;
            if ((rc = d.w_work.ensure(sizeof(unsigned long long) * rt::kWorkN))) return rc;
            if (fresh) RT_CK(cudaMemsetAsync(d.w_work.p, 0, sizeof(unsigned long long) * rt::kWorkN, st));
            wa.work = (unsigned long long *)d.w_work.p;
        }
        int nk = 0;
        if (!d.ph[0])
            for (auto &ev : d.ph) RT_CK(cudaEventCreate(&ev));
        cudaEvent_t *ph = ctx->phases ? d.ph : nullptr;  // event records cost ~2-3 us of GPU time each
        e = fused ? rt_launch_fused_f32(fa, sa, wa, st, &nk, ph) : rt_launch_wave_f32(fa, sa, wa, st, &nk, ph);
        d.ph_valid = ctx->phases;
        ctx->launches += nk - 1;  // the common increment below counts one
    } else {
        // few samples: one CTA per tile; many (the megakernel fallback of soft
        // shadows): persistent warps taking patches from a counter, a fresh
        // ring slot per launch (concurrent bands never share one)
        const int ns = count_spheres(ctx->scene), np = ctx->scene.n - ns;
        const bool tiles = (ctx->mega_tiles > 0 || (ctx->mega_tiles < 0 && fa.samples < rt::kWaveMinSamples)) &&
                           ns <= rt::kParamSpheres && np <= 8;
        if (!tiles) {
            if ((rc = d.counters.ensure(sizeof(unsigned) * rt::kCounterRing))) return rc;
            fa.work_counter = (unsigned *)d.counters.p + (d.counter_slot++ % rt::kCounterRing);
            RT_CK(cudaMemsetAsync(fa.work_counter, 0, sizeof(unsigned), st));
        }
        rt::MegaCull mc = {};
        if (ctx->cull && ctx->boxes) primary_boxes(mc, fa, ctx->scene);
        // (hot tiles first measured slower here: P720 s1 b1 +7%)
        mc.hot = make_int4(-1, -1, -1, -1);
        // the shadow grid filters the any-hit tests of scenes up to 8 spheres
        // (it is built over their spheres; larger scenes' bits name clusters)
        if (ctx->cull && ns <= 8 && d.grid_version == ctx->scene.version && d.grid_wa.grid) {
            mc.grid = d.grid_wa.grid;
            for (int c = 0; c < 3; c++) {
                mc.grid_lo[c] = d.grid_wa.grid_lo[c];
                mc.grid_inv[c] = d.grid_wa.grid_inv[c];
                mc.grid_dim[c] = d.grid_wa.grid_dim[c];
            }
        }
        e = rt_launch_render_f32(fa, scene_args(d, d.s32, ctx->scene), st, tiles, mc);
    }
    if (e != cudaSuccess) return fail(RT_ERR_CUDA, std::string("render kernel launch: ") + cudaGetErrorString(e));
    ctx->launches++;
    return RT_OK;
}

// Device-to-host copy of the rows of partition `part` (8-row blocks
// round-robin, map_row): one strided 2D copy of its whole blocks, one copy of
// a trailing partial block.  elem = bytes per pixel (4 for the frame, 12 or 24
// for radiance); host and device frames share the layout.
int copy_partition(void *host, const void *dev, size_t elem, int width, int height, int part, int n_parts,
                   int block_rows, cudaStream_t st) {
    const int n_blocks = (height + block_rows - 1) / block_rows;
    int full = 0;  // owned blocks that are complete
    for (int j = part; j < n_blocks; j += n_parts)
        if ((j + 1) * block_rows <= height) full++;
    const size_t row_b = elem * (size_t)width;
    const size_t off = (size_t)part * block_rows * row_b;
    char *h = (char *)host;
    const char *dv = (const char *)dev;
    if (full > 0)
        RT_CK(cudaMemcpy2DAsync(h + off, row_b * block_rows * n_parts, dv + off, row_b * block_rows * n_parts,
                                row_b * block_rows, full, cudaMemcpyDeviceToHost, st));
    const int last = part + full * n_parts;  // a trailing partial block, if this part owns it
    if (last < n_blocks) {
        const size_t o2 = (size_t)last * block_rows * row_b;
        RT_CK(cudaMemcpyAsync(h + o2, dv + o2, row_b * (height - last * block_rows), cudaMemcpyDeviceToHost, st));
    }
    return RT_OK;
}

int check_frame_args(int32_t w, int32_t h, int32_t samples, int32_t bounces, int32_t precision) {
    if (w < 1 || h < 1) return fail(RT_ERR_INVALID, "frame dimensions must be positive");
    if ((int64_t)w * h > (int64_t)1 << 31) return fail(RT_ERR_LIMIT, "frame too large");
    if (samples < 1) return fail(RT_ERR_INVALID, "shadow sample count must be >= 1");
    if (bounces < 0) return fail(RT_ERR_INVALID, "bounce limit must be >= 0");
    if (bounces > RT_MAX_BOUNCE_LIMIT) return fail(RT_ERR_LIMIT, "bounce limit capped at 31");
    if (precision != RT_PREC_FP32 && precision != RT_PREC_FP64) return fail(RT_ERR_INVALID, "bad precision");
    return RT_OK;
}

}  // namespace

extern "C" {

int rt_version(void) { return RT_ABI_VERSION; }

const char *rt_last_error(void) { return g_err.c_str(); }

int rt_device_count(int32_t *count) {
    if (!count) return fail(RT_ERR_INVALID, "null count");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    *count = n;
    return RT_OK;
}

int rt_ctx_create(rt_ctx **out, const int32_t *devices, int32_t n_devices) {
    if (!out) return fail(RT_ERR_INVALID, "null ctx pointer");
    *out = nullptr;
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail == 0) {
        cudaGetLastError();
        return fail(RT_ERR_NO_DEVICE, "no CUDA device visible: libb200rt has no CPU path");
    }
    if (n_devices < 1) n_devices = 1;
    rt_ctx *ctx = new rt_ctx();
    if (const char *w = std::getenv("B200RT_WAVE")) ctx->wave = std::atoi(w) != 0;
    if (const char *c = std::getenv("B200RT_CULL")) ctx->cull = std::atoi(c) != 0;
    for (int i = 0; i < n_devices; i++) {
        int id = devices ? devices[i] : i;
        if (id < 0 || id >= avail) {
            rt_ctx_destroy(ctx);
            return fail(RT_ERR_NO_DEVICE, "device index out of range");
        }
        Dev d;
        d.id = id;
        bool ok = cudaSetDevice(id) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&d.copy_st, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaEventCreate(&d.e0) == cudaSuccess && cudaEventCreate(&d.e1) == cudaSuccess &&
                  cudaEventCreate(&d.pe0) == cudaSuccess && cudaEventCreate(&d.pe1) == cudaSuccess;
        for (auto &ev : d.band_ev) ok = ok && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
        for (auto &ev : d.copy_ev) ok = ok && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&d.fork_ev, cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&d.dev_call_ev, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&d.dev_prep_ev, cudaEventDisableTiming) == cudaSuccess;
        for (auto &ev : d.tl_ev) ok = ok && cudaEventCreate(&ev) == cudaSuccess;
        for (int k = 0; ok && k < Dev::kSlots; k++)
            ok = cudaEventCreateWithFlags(&d.slot_comp[k], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&d.slot_done[k], cudaEventDisableTiming) ==
                     cudaSuccess;
        int least = 0, greatest = 0;
        if (ok) cudaDeviceGetStreamPriorityRange(&least, &greatest);
        if (ok) cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, id);
        for (int k = 0; ok && k < kMaxBands; k++)
            ok = cudaStreamCreateWithPriority(&d.band_st[k], cudaStreamNonBlocking, std::min(least, greatest + k)) ==
                 cudaSuccess;
        if (!ok) {
            std::string m = cudaGetErrorString(cudaGetLastError());
            ctx->devs.push_back(d);
            rt_ctx_destroy(ctx);
            return fail(RT_ERR_CUDA, "device init: " + m);
        }
        ctx->devs.push_back(d);
    }
    *out = ctx;
    return RT_OK;
}

int rt_ctx_destroy(rt_ctx *ctx) {
    if (!ctx) return RT_OK;
    for (Dev &d : ctx->devs) {
        cudaSetDevice(d.id);
        if (d.st) cudaStreamSynchronize(d.st);
        for (WaveBufs &wb : d.wb) wb.release();
        d.w_work.release();
        d.grid.release();
        for (DBuf *b : {&d.frame, &d.rad, &d.rays_in, &d.rays_out, &d.sky_raw, &d.sky, &d.counters, &d.s32.geo, &d.s32.mat,
                        &d.s32.table, &d.s32.geo64, &d.s64.geo, &d.s64.mat, &d.s64.table})
            b->release();
        for (auto ev : d.ph)
            if (ev) cudaEventDestroy(ev);
        for (auto ev : d.band_ev)
            if (ev) cudaEventDestroy(ev);
        for (auto ev : d.copy_ev)
            if (ev) cudaEventDestroy(ev);
        for (auto bs : d.band_st)
            if (bs) cudaStreamDestroy(bs);
        if (d.fork_ev) cudaEventDestroy(d.fork_ev);
        if (d.dev_call_ev) cudaEventDestroy(d.dev_call_ev);
        if (d.dev_prep_ev) cudaEventDestroy(d.dev_prep_ev);
        for (auto ev : d.tl_ev)
            if (ev) cudaEventDestroy(ev);
        for (int k = 0; k < Dev::kSlots; k++) {
            if (d.slot_comp[k]) cudaEventDestroy(d.slot_comp[k]);
            if (d.slot_done[k]) cudaEventDestroy(d.slot_done[k]);
            d.slot_frame[k].release();
            d.slot_codec[k].release();
        }
        d.codec_host.release();
        d.part_codec.release();
        if (d.copy_st) cudaStreamDestroy(d.copy_st);
        if (d.e0) cudaEventDestroy(d.e0);
        if (d.e1) cudaEventDestroy(d.e1);
        if (d.pe0) cudaEventDestroy(d.pe0);
        if (d.pe1) cudaEventDestroy(d.pe1);
        if (d.st) cudaStreamDestroy(d.st);
    }
    delete ctx;
    return RT_OK;
}

int rt_set_scene_v1(rt_ctx *ctx, int32_t n_bodies, const int32_t *kinds, const double *positions,
                    const double *sizes, const double *colors, const double *refls, const double light_pos[3],
                    double light_radius, const double light_color[3], double ambient, double max_refl,
                    const float *sky, int32_t sky_w, int32_t sky_h, int32_t has_sky) {
    if (!ctx) return fail(RT_ERR_INVALID, "null ctx");
    int rc = validate_scene(n_bodies, kinds, positions, sizes, colors, refls, light_pos, light_color, max_refl, sky,
                            sky_w, sky_h, has_sky);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (set_host_scene(ctx->scene, n_bodies, kinds, positions, sizes, colors, refls, light_pos, light_radius,
                       light_color, ambient, max_refl, sky, sky_w, sky_h, has_sky))
        sky_content_changed(ctx->scene);
    for (Dev &d : ctx->devs) {
        RT_CK(cudaSetDevice(d.id));
        if ((rc = upload_sky(ctx, d))) return rc;
    }
    return RT_OK;
}

}  // extern "C"

namespace {

// The last compressed frame's device time, once its events are done (rt_ctx::ms_pending).
int settle_last_ms(rt_ctx *ctx) {
    if (!ctx->ms_pending) return RT_OK;
    ctx->ms_pending = false;
    RT_CK(cudaEventSynchronize(ctx->ms_e1));
    RT_CK(cudaEventElapsedTime(&ctx->last_ms, ctx->ms_e0, ctx->ms_e1));
    return RT_OK;
}

// Enqueue one frame of rt_render_v1 on n_dev devices (no wait).
int enqueue_frame(rt_ctx *ctx, int n_dev, uint32_t *pixels, void *radiance, int32_t width, int32_t height,
                  const double cam_pos[3], double yaw, double pitch, double vdist, int32_t shadow_samples,
                  int32_t bounce_limit, int32_t n_parts, int32_t precision) {
    int rc;
    const int block_rows = RT_DEFAULT_BLOCK_ROWS;
    const size_t px_bytes = sizeof(uint32_t) * (size_t)width * height;
    const size_t rad_elem = precision == RT_PREC_FP64 ? sizeof(double) : sizeof(float);
    const size_t rad_bytes = rad_elem * 3 * (size_t)width * height;
    for (int g = 0; g < n_dev; g++) {
        Dev &d = ctx->devs[g];
        if ((rc = prepare(ctx, d, precision, shadow_samples))) return rc;
        if ((rc = d.frame.ensure(px_bytes))) return rc;
        if (radiance && (rc = d.rad.ensure(rad_bytes))) return rc;
    }
    // One device: render the frame as contiguous row bands and copy each band
    // to the host on a second stream while the next band renders, so the
    // PCIe transfer (~45-55 GB/s; 3.7 MB at 720p, 33 MB at 4K) hides behind
    // the kernels.  Bands are a partition of the pixels: the frame is the same.
    if (n_dev == 1) {
        Dev &d = ctx->devs[0];
        RT_CK(cudaSetDevice(d.id));
        // A page-locked, mapped framebuffer (rt_host_register) is written by the
        // kernels themselves: pixel stores travel over PCIe while the frame is
        // still being computed, so no copy follows the last kernel.
        uint32_t *host_px = nullptr;
        void *host_rad = nullptr;
        if (ctx->zero_copy && cudaHostGetDevicePointer((void **)&host_px, pixels, 0) == cudaSuccess &&
            (!radiance || cudaHostGetDevicePointer(&host_rad, radiance, 0) == cudaSuccess)) {
            if ((rc = settle_last_ms(ctx))) return rc;
            RT_CK(cudaEventRecord(d.e0, d.st));
            for (int p = 0; p < n_parts; p++) {
                rt::FrameArgs fa = frame_args(host_px, width, host_rad, width, height, cam_pos, yaw, pitch, vdist,
                                              shadow_samples, bounce_limit, p, n_parts, block_rows);
                fa.peer_out = 0;  // kernel completion + stream sync order the stores for the host
                if ((rc = launch_frame(ctx, d, fa, precision, d.st))) return rc;
            }
            RT_CK(cudaEventRecord(d.e1, d.st));
            ctx->band_pending = 0;
            ctx->codec_frame.on = false;
            ctx->last_d2h_bytes = 0;  // (the kernels' own stores)
            return RT_OK;
        }
        cudaGetLastError();  // not registered: a cudaHostGetDevicePointer miss is not an error
        // Bands run on their own prioritised streams (Dev::band_st), so their
        // kernels overlap; what a band costs is its first-band latency and
        // copy setup, against a copy at 45-56 GB/s (70 us for 720p, 585 us at
        // 4K) that also slows the kernels beside it.  Measured
        // best (tools/e2e_ab.py, round 2): 2 bands at 3.7 and 8.3 MB (C3: 258
        // us against 280 with 4), 6 at 33 MB.
        const size_t MB = (size_t)1 << 20;
        // compressed (option codec), the transfer is ~10% of the frame: 1
        // band below 6 MB (C2 104 us against 108 with 2), 2 below 24 MB (C3
        // 207 / 213 with 3), 6 above (C4 531 / 543 with 4); raw, as above
        const bool codec = ctx->codec && width <= rt::kCodecMaxWidth;
        int bands = ctx->bands > 0 ? ctx->bands
                    : codec        ? (px_bytes < 6 * MB ? 1 : px_bytes < 24 * MB ? 2 : 6)
                                   : (px_bytes < MB ? 1 : px_bytes < 24 * MB ? 2 : 6);
        if (ctx->phases) bands = 1;  // phase events describe one frame on one stream
        bands = std::max(1, std::min(bands, height / 8));
        // band boundaries in whole 8-row blocks: band 0 takes band_first
        // permille of the rows (when set), the others share the rest equally
        int y_at[kMaxBands + 1];
        {
            const int blocks = (height + 7) / 8;
            int first = ctx->band_first > 0 && bands > 1 ? (int)((int64_t)blocks * ctx->band_first / 1000)
                                                          : (blocks + bands - 1) / bands;
            first = std::max(1, std::min(first, blocks - (bands - 1)));
            y_at[0] = 0;
            y_at[1] = first;
            const int rest = blocks - first, others = bands - 1;
            for (int k = 1; k < bands; k++) y_at[k + 1] = first + (int)((int64_t)rest * k / others);
            for (int k = 0; k <= bands; k++) y_at[k] = std::min(height, y_at[k] * 8);
        }
        // compressed transfer: each band's rows encoded into the mapped host
        // buffer after its kernels; finish_frame expands them band by band
        // (band k while the later bands still render)
        auto &cf = ctx->codec_frame;
        cf.on = codec;
        if (cf.on) {
            if ((rc = d.codec_host.ensure(rt::codec_host_bytes(width, height)))) return rc;
            cf.pixels = pixels;
            cf.radiance = radiance != nullptr;
            cf.width = width;
            cf.height = height;
            cf.bands = bands;
            for (int k = 0; k <= bands; k++) cf.y_at[k] = y_at[k];
            // one render band: its encode may still be cut into parts (in
            // stream order, an event after each), so the host expands the
            // first rows while the rest cross PCIe
            // (2 parts: C2 99.4 -> 97.8 us, P720 72.1 -> 70.2; 3-4 slower, and C1 +4 us:
            // each launch's flush costs the GPU ~6 us)
            const int want = ctx->codec_parts > 0 ? ctx->codec_parts : px_bytes >= 2 * MB ? 2 : 1;
            if (bands == 1 && want > 1) {
                const int parts = std::max(1, std::min(want, std::min(kMaxBands, height / 8)));
                const int blocks = (height + 7) / 8;
                cf.bands = parts;
                for (int e = 0; e <= parts; e++) cf.y_at[e] = std::min(height, 8 * (int)((int64_t)blocks * e / parts));
                for (int e = 0; e < parts; e++) cf.order[e] = e;
            }
        }
        // the previous compressed frame's events, unread: kept aside and read
        // once this frame is launched
        const bool settle_after = ctx->ms_pending;
        if (settle_after) {
            std::swap(d.e0, d.pe0);
            std::swap(d.e1, d.pe1);
            ctx->ms_e0 = d.pe0;
            ctx->ms_e1 = d.pe1;
        }
        RT_CK(cudaEventRecord(d.e0, d.st));
        if (bands > 1) RT_CK(cudaEventRecord(d.fork_ev, d.st));
        // each band's copy follows its kernels on its own stream, so the
        // copies start in the order the bands finish (P720 end to end 115 ->
        // 106 us, C4 692 -> 681 us against one copy stream).  Bands are
        // enqueued top first; bottom first (option band_order: the costly
        // rows reach the GPU sooner) measured 10-18% slower end to end
        for (int i = 0; i < bands; i++) {
            const int k = ctx->band_order && bands > 1 ? bands - 1 - i : i;
            if (bands > 1) cf.order[i] = k;
            else if (cf.bands == 1) cf.order[0] = 0;
            cudaStream_t bs = bands > 1 ? d.band_st[k] : d.st;
            if (bands > 1) RT_CK(cudaStreamWaitEvent(bs, d.fork_ev, 0));
            const int y0 = y_at[k], y1 = y_at[k + 1];
            for (int p = 0; p < n_parts; p++) {  // the caller's partitions inside the band, same device
                rt::FrameArgs fa = frame_args((uint32_t *)d.frame.p, width, radiance ? d.rad.p : nullptr, width,
                                              height, cam_pos, yaw, pitch, vdist, shadow_samples, bounce_limit, 0, 1,
                                              height);
                // rows [y0, y1) of the frame, partition p of the band (8-row blocks interleaved)
                fa.row0 = y0;
                fa.sub_part = p;
                fa.sub_parts = n_parts;
                fa.local_rows = rt::rt_band_local_rows(y1 - y0, p, n_parts);
                fa.row_end = y1;
                if ((rc = launch_frame(ctx, d, fa, precision, bs, k))) return rc;
            }
            if (ctx->band_times) RT_CK(cudaEventRecord(d.tl_ev[k], bs));
            if (cf.on) {
                // the band's encode right behind its last kernel on the same
                // stream (a programmatic dependent: no launch gap); the host
                // expands the band once copy_ev[k] fires
                if (bands == 1 && cf.bands > 1) {  // encode parts (see above)
                    for (int e = 0; e < cf.bands; e++) {
                        RT_CK(rt::launch_encode_rows((const uint32_t *)d.frame.p, width, width, height, cf.y_at[e],
                                                     cf.y_at[e + 1], (uint32_t *)d.codec_host.dp, bs));
                        RT_CK(cudaEventRecord(d.copy_ev[e], bs));
                    }
                } else {
                    RT_CK(rt::launch_encode_rows((const uint32_t *)d.frame.p, width, width, height, y0, y1,
                                                 (uint32_t *)d.codec_host.dp, bs));
                    RT_CK(cudaEventRecord(d.copy_ev[k], bs));
                }
            }
            RT_CK(cudaEventRecord(d.band_ev[k], bs));
            if (bands > 1) RT_CK(cudaStreamWaitEvent(d.st, d.band_ev[k], 0));  // the join (kernels)
            cudaStream_t cs = bands > 1 ? bs : d.copy_st;
            if (bands == 1) RT_CK(cudaStreamWaitEvent(d.copy_st, d.band_ev[k], 0));
            if (y1 > y0) {
                size_t off = (size_t)y0 * width, cnt = (size_t)(y1 - y0) * width;
                if (!cf.on)
                    RT_CK(cudaMemcpyAsync(pixels + off, (uint32_t *)d.frame.p + off, sizeof(uint32_t) * cnt,
                                          cudaMemcpyDeviceToHost, cs));
                if (radiance)
                    RT_CK(cudaMemcpyAsync((char *)radiance + rad_elem * 3 * off, (char *)d.rad.p + rad_elem * 3 * off,
                                          rad_elem * 3 * cnt, cudaMemcpyDeviceToHost, cs));
            }
            if (ctx->band_times) RT_CK(cudaEventRecord(d.tl_ev[kMaxBands + k], cs));
            if (bands > 1) {  // the band's end, joined into the copy stream that finish_frame waits for
                // (compressed, copy_ev[k] already marks the encode's end for the
                // expansion: band_ev[k], its join done, is recorded again here)
                cudaEvent_t end_ev = cf.on ? d.band_ev[k] : d.copy_ev[k];
                RT_CK(cudaEventRecord(end_ev, bs));
                RT_CK(cudaStreamWaitEvent(d.copy_st, end_ev, 0));
            }
        }
        RT_CK(cudaEventRecord(d.e1, d.st));
        if (settle_after && (rc = settle_last_ms(ctx))) return rc;
        ctx->band_pending = bands;
        ctx->last_d2h_bytes = (cf.on ? 0 : (int64_t)px_bytes) + (radiance ? (int64_t)rad_bytes : 0);
        return RT_OK;
    }
    // several devices: partition p runs on device p % n_dev, each device
    // returns only its rows
    ctx->codec_frame.on = false;
    ctx->last_d2h_bytes = (int64_t)px_bytes + (radiance ? (int64_t)rad_bytes : 0);
    if ((rc = settle_last_ms(ctx))) return rc;
    for (int g = 0; g < n_dev; g++) {
        Dev &d = ctx->devs[g];
        RT_CK(cudaSetDevice(d.id));
        RT_CK(cudaEventRecord(d.e0, d.st));
        for (int p = g; p < n_parts; p += n_dev) {
            rt::FrameArgs fa = frame_args((uint32_t *)d.frame.p, width, radiance ? d.rad.p : nullptr, width, height,
                                          cam_pos, yaw, pitch, vdist, shadow_samples, bounce_limit, p, n_parts,
                                          block_rows);
            if ((rc = launch_frame(ctx, d, fa, precision, d.st))) return rc;
        }
        RT_CK(cudaEventRecord(d.e1, d.st));
    }
    for (int g = 0; g < n_dev; g++) {
        Dev &d = ctx->devs[g];
        RT_CK(cudaSetDevice(d.id));
        for (int p = g; p < n_parts; p += n_dev) {
            if ((rc = copy_partition(pixels, (const uint32_t *)d.frame.p, sizeof(uint32_t), width, height, p, n_parts,
                                     block_rows, d.st)))
                return rc;
            if (radiance &&
                (rc = copy_partition(radiance, d.rad.p, rad_elem * 3, width, height, p, n_parts, block_rows, d.st)))
                return rc;
        }
    }
    ctx->band_pending = 0;
    return RT_OK;
}


int codec_threads(const rt_ctx *ctx) {
    return ctx->codec_threads > 0 ? ctx->codec_threads : std::min(16, omp_get_max_threads());
}

// Wait for the frame enqueued by enqueue_frame (compressed: expanding its
// bands as they land); its device time and band times.
// side: work for the expansion team's waits (only with a compressed frame)
int finish_frame(rt_ctx *ctx, int n_dev, const rt::CodecSideJob *side = nullptr) {
    auto &cf = ctx->codec_frame;
    if (side && !(n_dev == 1 && cf.on)) {  // no expansion team: the side job on its own
#pragma omp parallel for num_threads(sky_threads()) schedule(dynamic)
        for (int i = 0; i < side->items; i++) side->run(side->arg, i);
    }
    if (n_dev == 1 && cf.on) {
        // expand the bands in the order they finish, each as soon as its rows land
        Dev &d = ctx->devs[0];
        RT_CK(cudaSetDevice(d.id));
        // the bands expanded in the order they finish, each the moment its rows
        // are in (the side job — the sky hash — fills the wait)
        struct W {
            Dev *d;
            static int query(void *arg, int k) {
                const cudaError_t e = cudaEventQuery(static_cast<W *>(arg)->d->copy_ev[k]);
                if (e == cudaErrorNotReady) return 0;
                if (e == cudaSuccess) return 1;
                return fail(RT_ERR_CUDA, std::string("compressed frame: ") + cudaGetErrorString(e));
            }
            static int wait(void *arg, int k) {
                const cudaError_t e = cudaEventSynchronize(static_cast<W *>(arg)->d->copy_ev[k]);
                return e == cudaSuccess ? 0 : fail(RT_ERR_CUDA, std::string("compressed frame: ") + cudaGetErrorString(e));
            }
        } w{&d};
        int wrc = RT_OK;
        stamp(g_t_team_start);
        const int64_t words = rt::decode_bands((const uint32_t *)d.codec_host.p, cf.width, cf.bands, cf.y_at,
                                               cf.order, &W::query, &W::wait, &w, &wrc, cf.pixels, cf.width,
                                               std::max(codec_threads(ctx), side ? sky_threads() : 1), side);
        stamp(g_t_team_end);
        cf.on = false;
        if (words < 0) return wrc;
        ctx->last_d2h_bytes += (int64_t)sizeof(uint32_t) * words;
        // the frame is in the caller's buffer and the encode was the streams'
        // last work: return now (stream syncs and the events' elapsed time
        // cost ~8 us here); the device time is read later (settle_last_ms)
        if (!cf.radiance && !ctx->phases && !ctx->band_times) {
            ctx->ms_pending = true;
            ctx->ms_e0 = d.e0;
            ctx->ms_e1 = d.e1;
            ctx->band_count = 0;
            return RT_OK;
        }
    }
    for (int g = 0; g < n_dev; g++) {
        Dev &d = ctx->devs[g];
        RT_CK(cudaSetDevice(d.id));
        if (n_dev == 1) RT_CK(cudaStreamSynchronize(d.copy_st));
        stamp(g_t_sync1);
        RT_CK(cudaStreamSynchronize(d.st));
    }
    stamp(g_t_sync2);
    Dev &d = ctx->devs[0];
    RT_CK(cudaSetDevice(d.id));
    RT_CK(cudaEventElapsedTime(&ctx->last_ms, d.e0, d.e1));
    stamp(g_t_elapsed);
    ctx->band_count = (n_dev == 1 && ctx->band_times) ? ctx->band_pending : 0;
    for (int k = 0; k < ctx->band_count; k++) {
        RT_CK(cudaEventElapsedTime(&ctx->band_ms[k], d.e0, d.tl_ev[k]));
        RT_CK(cudaEventElapsedTime(&ctx->band_ms[kMaxBands + k], d.e0, d.tl_ev[kMaxBands + k]));
    }
    return RT_OK;
}

}  // namespace

extern "C" {


int rt_render_v1(rt_ctx *ctx, uint32_t *pixels, void *radiance, int32_t width, int32_t height,
                 const double cam_pos[3], double yaw, double pitch, double vdist, int32_t n_bodies,
                 const int32_t *kinds, const double *positions, const double *sizes, const double *colors,
                 const double *refls, const double light_pos[3], double light_radius, const double light_color[3],
                 double ambient, double max_refl, const float *sky, int32_t sky_w, int32_t sky_h, int32_t has_sky,
                 int32_t shadow_samples, int32_t bounce_limit, int32_t n_parts, int32_t precision) {
    const auto t_call = std::chrono::steady_clock::now();
    g_first_launch_pending = host_timing_on();
    if (!ctx || !pixels || !cam_pos) return fail(RT_ERR_INVALID, "null argument");
    int rc = check_frame_args(width, height, shadow_samples, bounce_limit, precision);
    if (rc) return rc;
    if ((rc = validate_scene(n_bodies, kinds, positions, sizes, colors, refls, light_pos, light_color, max_refl, sky,
                             sky_w, sky_h, has_sky)))
        return rc;
    if (n_parts < 1) n_parts = 1;
    std::lock_guard<std::mutex> lk(ctx->mu);
    const bool verify_sky = set_host_scene(ctx->scene, n_bodies, kinds, positions, sizes, colors, refls, light_pos,
                                           light_radius, light_color, ambient, max_refl, sky, sky_w, sky_h, has_sky);
    const int n_dev = std::min<int>((int)ctx->devs.size(), n_parts);
    const auto t_enq = std::chrono::steady_clock::now();
    // The frame is enqueued with the device's copy of the sky; when the
    // caller passed the same sky array as before, its texels are hashed in
    // full while the kernels run, and on a different hash the sky is uploaded
    // again and the frame rendered again.
    bool finished = false;
    for (int attempt = 0;; attempt++) {
        if ((rc = enqueue_frame(ctx, n_dev, pixels, radiance, width, height, cam_pos, yaw, pitch, vdist,
                                shadow_samples, bounce_limit, n_parts, precision)))
            return rc;
        if (attempt > 0 || !verify_sky || !ctx->scene.has_sky || !ctx->scene.sky_ptr) break;
        if (ctx->codec_frame.on) {
            // compressed: the host threads hash the sky while they wait for the
            // bands, and expand each band as it lands
            HostScene &sc = ctx->scene;
            TexelHash th(sc.sky_ptr, (size_t)sc.sky_w * sc.sky_h * 3);
            rt::CodecSideJob side{th.chunks, &TexelHash::run, &th};
            if ((rc = finish_frame(ctx, n_dev, &side))) return rc;
            finished = true;
            if (!sky_hash_differs(sc, th.value())) break;
            finished = false;  // stale: rendered again with the new sky
            continue;
        }
        if (!sky_content_changed(ctx->scene)) break;
        if ((rc = finish_frame(ctx, n_dev))) return rc;  // the stale frame ends before the sky is replaced
    }
    const auto t_wait = std::chrono::steady_clock::now();
    if (!finished && (rc = finish_frame(ctx, n_dev))) return rc;
    if (host_timing_on()) {  // $B200RT_HOST_TIMING: where a synchronous call's host time goes
        const auto t_end = std::chrono::steady_clock::now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        fprintf(stderr,
                "rt_render_v1: setup %.1f us, first launch at %.1f, enqueue %.1f us, wait %.1f us (expansion team "
                "%.1f .. %.1f), syncs %.1f %.1f, elapsed %.1f, end %.1f; device e0->e1 %.1f us\n",
                us(t_call, t_enq), us(t_call, g_t_first_launch), us(t_enq, t_wait), us(t_wait, t_end),
                us(t_call, g_t_team_start), us(t_call, g_t_team_end), us(t_call, g_t_sync1), us(t_call, g_t_sync2),
                us(t_call, g_t_elapsed), us(t_call, t_end), 1e3 * ctx->last_ms);
    }
    return upload_sky_all(ctx);
}

int rt_render_device_v1(rt_ctx *ctx, int32_t slot, uint32_t *d_out, int64_t out_pitch, void *d_radiance,
                        int32_t width, int32_t height, const double cam_pos[3], double yaw, double pitch,
                        double vdist, int32_t shadow_samples, int32_t bounce_limit, int32_t part, int32_t n_parts,
                        int32_t block_rows, int32_t precision, void *stream) {
    if (!ctx || !d_out || !cam_pos) return fail(RT_ERR_INVALID, "null argument");
    int rc = check_frame_args(width, height, shadow_samples, bounce_limit, precision);
    if (rc) return rc;
    if (slot < 0 || slot >= (int)ctx->devs.size()) return fail(RT_ERR_INVALID, "bad device slot");
    if (n_parts < 1 || part < 0 || part >= n_parts || block_rows < 1)
        return fail(RT_ERR_INVALID, "bad partition (part, n_parts, block_rows)");
    if (out_pitch < width) return fail(RT_ERR_INVALID, "out_pitch < width");
    std::lock_guard<std::mutex> lk(ctx->mu);
    Dev &d = ctx->devs[slot];
    RT_CK(cudaSetDevice(d.id));
    cudaStream_t st = stream ? (cudaStream_t)stream : d.st;
    // Order this call after the previous one on the device whatever stream
    // either used: the scene / grid uploads of prepare() (on d.st) must not
    // overwrite buffers a previous frame's kernels still read, this frame's
    // kernels must see them complete, and two frames never share the queues
    // of wb[0] at the same time.
    if (d.dev_call_pending) RT_CK(cudaStreamWaitEvent(d.st, d.dev_call_ev, 0));
    if ((rc = prepare(ctx, d, precision, shadow_samples))) return rc;
    if (st != d.st) {
        RT_CK(cudaEventRecord(d.dev_prep_ev, d.st));
        RT_CK(cudaStreamWaitEvent(st, d.dev_prep_ev, 0));
    }
    rt::FrameArgs fa = frame_args(d_out, out_pitch, d_radiance, width, height, cam_pos, yaw, pitch, vdist,
                                  shadow_samples, bounce_limit, part, n_parts, block_rows);
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, d_out) != cudaSuccess) {
        cudaGetLastError();
        fa.peer_out = 1;
    } else {
        fa.peer_out = (attr.type != cudaMemoryTypeDevice || attr.device != d.id) ? 1 : 0;
    }
    if ((rc = launch_frame(ctx, d, fa, precision, st))) return rc;
    RT_CK(cudaEventRecord(d.dev_call_ev, st));
    d.dev_call_pending = true;
    return RT_OK;
}

int rt_trace_rays_v1(rt_ctx *ctx, const double *origins, const double *dirs, int64_t n_rays, void *out_rgb,
                     int32_t n_bodies, const int32_t *kinds, const double *positions, const double *sizes,
                     const double *colors, const double *refls, const double light_pos[3], double light_radius,
                     const double light_color[3], double ambient, double max_refl, const float *sky,
                     int32_t sky_w, int32_t sky_h, int32_t has_sky, int32_t shadow_samples, int32_t bounce_limit,
                     int32_t precision) {
    if (!ctx || (n_rays > 0 && (!origins || !dirs || !out_rgb))) return fail(RT_ERR_INVALID, "null argument");
    if (n_rays < 0) return fail(RT_ERR_INVALID, "n_rays < 0");
    int rc = check_frame_args(1, 1, shadow_samples, bounce_limit, precision);
    if (rc) return rc;
    if ((rc = validate_scene(n_bodies, kinds, positions, sizes, colors, refls, light_pos, light_color, max_refl, sky,
                             sky_w, sky_h, has_sky)))
        return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (set_host_scene(ctx->scene, n_bodies, kinds, positions, sizes, colors, refls, light_pos, light_radius,
                       light_color, ambient, max_refl, sky, sky_w, sky_h, has_sky))
        sky_content_changed(ctx->scene);
    if (n_rays == 0) return upload_sky_all(ctx);
    Dev &d = ctx->devs[0];
    if ((rc = prepare(ctx, d, precision, shadow_samples))) return rc;
    size_t in_b = sizeof(double) * 3 * (size_t)n_rays;
    size_t out_b = (precision == RT_PREC_FP64 ? sizeof(double) : sizeof(float)) * 3 * (size_t)n_rays;
    if ((rc = d.rays_in.ensure(2 * in_b)) || (rc = d.rays_out.ensure(out_b))) return rc;
    double *d_o = (double *)d.rays_in.p, *d_d = d_o + 3 * n_rays;
    RT_CK(cudaMemcpyAsync(d_o, origins, in_b, cudaMemcpyHostToDevice, d.st));
    RT_CK(cudaMemcpyAsync(d_d, dirs, in_b, cudaMemcpyHostToDevice, d.st));
    if ((rc = settle_last_ms(ctx))) return rc;
    RT_CK(cudaEventRecord(d.e0, d.st));
    cudaError_t e;
    if (precision == RT_PREC_FP64)
        e = rt_launch_trace_f64(d_o, d_d, n_rays, (double *)d.rays_out.p, scene_args(d, d.s64, ctx->scene),
                                shadow_samples, bounce_limit, d.st);
    else
        e = rt_launch_trace_f32(d_o, d_d, n_rays, (float *)d.rays_out.p, scene_args(d, d.s32, ctx->scene),
                                shadow_samples, bounce_limit, d.st);
    if (e != cudaSuccess) return fail(RT_ERR_CUDA, std::string("trace kernel launch: ") + cudaGetErrorString(e));
    ctx->launches++;
    RT_CK(cudaEventRecord(d.e1, d.st));
    RT_CK(cudaMemcpyAsync(out_rgb, d.rays_out.p, out_b, cudaMemcpyDeviceToHost, d.st));
    RT_CK(cudaStreamSynchronize(d.st));
    RT_CK(cudaEventElapsedTime(&ctx->last_ms, d.e0, d.e1));
    return upload_sky_all(ctx);
}

int rt_sky_sample_v1(rt_ctx *ctx, const double *dirs, int64_t n, double *out_rgb, const float *sky, int32_t sky_w,
                     int32_t sky_h) {
    if (!ctx || !sky || (n > 0 && (!dirs || !out_rgb))) return fail(RT_ERR_INVALID, "null argument");
    if (sky_w < 1 || sky_h < 1 || n < 0) return fail(RT_ERR_INVALID, "bad skybox / count");
    std::lock_guard<std::mutex> lk(ctx->mu);
    Dev &d = ctx->devs[0];
    RT_CK(cudaSetDevice(d.id));
    int64_t nt = (int64_t)sky_w * sky_h;
    DBuf raw, tex, io;
    int rc;
    if ((rc = raw.ensure(sizeof(float) * 3 * nt)) || (rc = tex.ensure(sizeof(float4) * nt)) ||
        (rc = io.ensure(sizeof(double) * 6 * (size_t)std::max<int64_t>(n, 1)))) {
        raw.release();
        tex.release();
        io.release();
        return rc;
    }
    double *d_in = (double *)io.p, *d_out = d_in + 3 * n;
    cudaError_t e = cudaMemcpyAsync(raw.p, sky, sizeof(float) * 3 * nt, cudaMemcpyHostToDevice, d.st);
    if (e == cudaSuccess && n > 0) e = cudaMemcpyAsync(d_in, dirs, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, d.st);
    if (e == cudaSuccess) {
        sky_to_float4<<<(unsigned)((nt + 255) / 256), 256, 0, d.st>>>((const float *)raw.p, (float4 *)tex.p, nt);
        e = cudaGetLastError();
        ctx->launches++;
    }
    if (e == cudaSuccess && n > 0) {
        e = rt_launch_sky_f64(d_in, n, d_out, (const float4 *)tex.p, sky_w, sky_h, d.st);
        ctx->launches++;
    }
    if (e == cudaSuccess && n > 0)
        e = cudaMemcpyAsync(out_rgb, d_out, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, d.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(d.st);
    raw.release();
    tex.release();
    io.release();
    if (e != cudaSuccess) return fail(RT_ERR_CUDA, std::string("sky sample: ") + cudaGetErrorString(e));
    return RT_OK;
}

int rt_host_register(rt_ctx *ctx, void *ptr, size_t bytes) {
    if (!ptr || bytes == 0) return fail(RT_ERR_INVALID, "bad host range");
    if (ctx) RT_CK(cudaSetDevice(ctx->devs[0].id));
    cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
    if (e == cudaSuccess) return RT_OK;
    cudaGetLastError();  // leave no sticky error for the next launch check to report
    if (e == cudaErrorHostMemoryAlreadyRegistered) return RT_ALREADY_REGISTERED;
    return fail(RT_ERR_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
}

int rt_host_unregister(rt_ctx *ctx, void *ptr) {
    if (!ptr) return fail(RT_ERR_INVALID, "bad host pointer");
    if (ctx) RT_CK(cudaSetDevice(ctx->devs[0].id));
    cudaError_t e = cudaHostUnregister(ptr);
    if (e == cudaSuccess) return RT_OK;
    cudaGetLastError();
    return fail(RT_ERR_CUDA, std::string("cudaHostUnregister: ") + cudaGetErrorString(e));
}

int rt_set_option(rt_ctx *ctx, const char *name, int32_t value) {
    if (!ctx || !name) return fail(RT_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    std::string n(name);
    if (n == "wave") ctx->wave = value != 0;
    else if (n == "cull") ctx->cull = value != 0;
    else if (n == "count_work") ctx->count_work = value != 0;
    else if (n == "bands") ctx->bands = std::max(0, std::min((int)value, kMaxBands));
    else if (n == "phases") ctx->phases = value != 0;
    else if (n == "rgba") ctx->rgba = value != 0;
    else if (n == "zero_copy") ctx->zero_copy = value != 0;
    else if (n == "codec") ctx->codec = value != 0;
    else if (n == "codec_parts") ctx->codec_parts = std::max(0, std::min((int)value, kMaxBands));
    else if (n == "codec_threads") ctx->codec_threads = std::max(0, (int)value);
    else if (n == "conic") ctx->conic = value != 0;
    else if (n == "cull_check") ctx->cull_check = value != 0;
    else if (n == "band_first") ctx->band_first = std::max(0, std::min((int)value, 1000));
    else if (n == "band_times") ctx->band_times = value != 0;
    else if (n == "hot_tiles") ctx->hot_tiles = value != 0;
    else if (n == "compact") ctx->compact = value != 0;
    else if (n == "sphere_bound") rt_set_sphere_bound(value != 0);
    else if (n == "band_order") ctx->band_order = value != 0;
    else if (n == "boxes") ctx->boxes = value != 0;
    else if (n == "mega_tiles") ctx->mega_tiles = value < 0 ? -1 : value != 0;
    else return fail(RT_ERR_INVALID, "unknown option " + n);
    return RT_OK;
}

int rt_work_counts(rt_ctx *ctx, uint64_t *out, int32_t n, int32_t reset) {
    if (!ctx || !out || n < 1) return fail(RT_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    Dev &d = ctx->devs[0];
    RT_CK(cudaSetDevice(d.id));
    unsigned long long h[rt::kWorkN] = {0};
    if (d.w_work.p) {
        RT_CK(cudaStreamSynchronize(d.st));
        RT_CK(cudaMemcpy(h, d.w_work.p, sizeof h, cudaMemcpyDeviceToHost));
        if (reset) RT_CK(cudaMemset(d.w_work.p, 0, sizeof h));
    }
    for (int i = 0; i < n && i < rt::kWorkN; i++) out[i] = h[i];
    return RT_OK;
}

int rt_frame_expand_v1(const uint32_t *host_buf, int32_t width, int32_t height, uint32_t *pixels, int64_t pitch,
                       int32_t threads, int64_t *words) {
    if (!host_buf || !pixels) return fail(RT_ERR_INVALID, "null argument");
    if (width < 1 || height < 1 || pitch < width) return fail(RT_ERR_INVALID, "bad frame size");
    const int64_t n = rt::decode_rows(host_buf, width, 0, height, pixels, pitch, threads > 0 ? threads : 1);
    if (words) *words = n;
    return RT_OK;
}

int rt_last_d2h_bytes(rt_ctx *ctx, int64_t *bytes) {
    if (!ctx || !bytes) return fail(RT_ERR_INVALID, "null argument");
    *bytes = ctx->last_d2h_bytes;
    return RT_OK;
}

int rt_last_kernel_ms(rt_ctx *ctx, float *ms) {
    if (!ctx || !ms) return fail(RT_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    int rc;
    if ((rc = settle_last_ms(ctx))) return rc;
    *ms = ctx->last_ms;
    return RT_OK;
}

int rt_phase_ms(rt_ctx *ctx, float *out, int32_t n) {
    if (!ctx || !out || n < 4) return fail(RT_ERR_INVALID, "need 4 outputs");
    std::lock_guard<std::mutex> lk(ctx->mu);
    Dev &d = ctx->devs[0];
    for (int i = 0; i < 4; i++) out[i] = 0.f;
    if (!d.ph_valid) return RT_OK;
    RT_CK(cudaSetDevice(d.id));
    RT_CK(cudaEventSynchronize(d.ph[4]));
    for (int i = 0; i < 4; i++) RT_CK(cudaEventElapsedTime(&out[i], d.ph[i], d.ph[i + 1]));
    return RT_OK;
}

int rt_band_times_ms(rt_ctx *ctx, float *out, int32_t n) {
    if (!ctx || (!out && n > 0)) return fail(RT_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    const int b = ctx->band_count;
    for (int k = 0; k < b && 2 * k + 1 < n; k++) {
        out[2 * k] = ctx->band_ms[k];
        out[2 * k + 1] = ctx->band_ms[kMaxBands + k];
    }
    return b;
}

int rt_launch_count(rt_ctx *ctx, int64_t *count) {
    if (!ctx || !count) return fail(RT_ERR_INVALID, "null argument");
    *count = ctx->launches;
    return RT_OK;
}

int rt_ipc_get_handle(void *d_ptr, uint8_t handle_out[64]) {
    if (!d_ptr || !handle_out) return fail(RT_ERR_INVALID, "null argument");
    cudaIpcMemHandle_t h;
    RT_CK(cudaIpcGetMemHandle(&h, d_ptr));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle_out, &h, 64);
    return RT_OK;
}

int rt_ipc_open(const uint8_t handle[64], void **d_ptr_out) {
    if (!handle || !d_ptr_out) return fail(RT_ERR_INVALID, "null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    RT_CK(cudaIpcOpenMemHandle(d_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    return RT_OK;
}

int rt_ipc_close(void *d_ptr) {
    if (!d_ptr) return fail(RT_ERR_INVALID, "null argument");
    RT_CK(cudaIpcCloseMemHandle(d_ptr));
    return RT_OK;
}

int rt_copy_to_host(rt_ctx *ctx, int32_t slot, void *host_dst, const void *d_src, size_t bytes, void *stream) {
    if (!ctx || !host_dst || !d_src) return fail(RT_ERR_INVALID, "null argument");
    if (slot < 0 || slot >= (int)ctx->devs.size()) return fail(RT_ERR_INVALID, "bad device slot");
    Dev &d = ctx->devs[slot];
    RT_CK(cudaSetDevice(d.id));
    cudaStream_t st = stream ? (cudaStream_t)stream : d.st;
    RT_CK(cudaMemcpyAsync(host_dst, d_src, bytes, cudaMemcpyDeviceToHost, st));
    RT_CK(cudaStreamSynchronize(st));
    return RT_OK;
}

}  // extern "C"

namespace {
// A pipelined frame's end: its copy (or encode) done, then, compressed, its
// expansion into the caller's framebuffer.
int slot_finish(rt_ctx *ctx, Dev &d, int slot) {
    RT_CK(cudaEventSynchronize(d.slot_done[slot]));
    auto &so = d.slot_out[slot];
    if (so.codec) {
        const int64_t words = rt::decode_rows((const uint32_t *)d.slot_codec[slot].p, so.width, 0, so.height,
                                              so.pixels, so.width, codec_threads(ctx));
        ctx->last_d2h_bytes = (int64_t)sizeof(uint32_t) * words;
    } else {
        ctx->last_d2h_bytes = (int64_t)sizeof(uint32_t) * so.width * so.height;
    }
    d.slot_busy[slot] = false;
    return RT_OK;
}
}  // namespace

extern "C" {

int rt_render_async_v1(rt_ctx *ctx, int32_t slot, uint32_t *pixels, int32_t width, int32_t height,
                       const double cam_pos[3], double yaw, double pitch, double vdist, int32_t n_bodies,
                       const int32_t *kinds, const double *positions, const double *sizes, const double *colors,
                       const double *refls, const double light_pos[3], double light_radius,
                       const double light_color[3], double ambient, double max_refl, const float *sky, int32_t sky_w,
                       int32_t sky_h, int32_t has_sky, int32_t shadow_samples, int32_t bounce_limit,
                       int32_t precision) {
    if (!ctx || !pixels || !cam_pos) return fail(RT_ERR_INVALID, "null argument");
    if (slot < 0 || slot >= Dev::kSlots) return fail(RT_ERR_INVALID, "frame slot out of range");
    int rc = check_frame_args(width, height, shadow_samples, bounce_limit, precision);
    if (rc) return rc;
    if ((rc = validate_scene(n_bodies, kinds, positions, sizes, colors, refls, light_pos, light_color, max_refl, sky,
                             sky_w, sky_h, has_sky)))
        return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    Dev &d = ctx->devs[0];
    RT_CK(cudaSetDevice(d.id));
    if (d.slot_busy[slot]) {  // the slot's previous frame was never waited for: completed now
        if ((rc = slot_finish(ctx, d, slot))) return rc;
    }
    const bool verify_sky = set_host_scene(ctx->scene, n_bodies, kinds, positions, sizes, colors, refls, light_pos,
                                           light_radius, light_color, ambient, max_refl, sky, sky_w, sky_h, has_sky);
    const size_t px_bytes = sizeof(uint32_t) * (size_t)width * height;
    // the kernels on the frame stream (frames in order), the copy on the copy
    // stream: the next frame's kernels overlap this frame's PCIe transfer.
    // The sky is verified while the frame runs (as in rt_render_v1): on a
    // difference the frame is enqueued again after the upload.
    for (int attempt = 0;; attempt++) {
        if ((rc = prepare(ctx, d, precision, shadow_samples))) return rc;
        if ((rc = d.slot_frame[slot].ensure(px_bytes))) return rc;
        rt::FrameArgs fa = frame_args((uint32_t *)d.slot_frame[slot].p, width, nullptr, width, height, cam_pos, yaw,
                                      pitch, vdist, shadow_samples, bounce_limit, 0, 1, RT_DEFAULT_BLOCK_ROWS);
        if ((rc = settle_last_ms(ctx))) return rc;
        RT_CK(cudaEventRecord(d.e0, d.st));
        if ((rc = launch_frame(ctx, d, fa, precision, d.st))) return rc;
        RT_CK(cudaEventRecord(d.e1, d.st));
        RT_CK(cudaEventRecord(d.slot_comp[slot], d.st));
        RT_CK(cudaStreamWaitEvent(d.copy_st, d.slot_comp[slot], 0));
        auto &so = d.slot_out[slot];
        so.codec = ctx->codec && width <= rt::kCodecMaxWidth;
        so.pixels = pixels;
        so.width = width;
        so.height = height;
        if (so.codec) {  // encoded into the slot's mapped buffer; rt_frame_wait_v1 expands it
            if ((rc = d.slot_codec[slot].ensure(rt::codec_host_bytes(width, height)))) return rc;
            RT_CK(rt::launch_encode_rows((const uint32_t *)d.slot_frame[slot].p, width, width, height, 0, height,
                                         (uint32_t *)d.slot_codec[slot].dp, d.copy_st));
        } else {
            RT_CK(cudaMemcpyAsync(pixels, d.slot_frame[slot].p, px_bytes, cudaMemcpyDeviceToHost, d.copy_st));
        }
        RT_CK(cudaEventRecord(d.slot_done[slot], d.copy_st));
        if (attempt > 0 || !verify_sky || !sky_content_changed(ctx->scene)) break;
        RT_CK(cudaEventSynchronize(d.slot_done[slot]));  // the stale frame ends before the sky is replaced
    }
    d.slot_busy[slot] = true;
    return upload_sky_all(ctx);
}

int rt_frame_wait_v1(rt_ctx *ctx, int32_t slot) {
    if (!ctx) return fail(RT_ERR_INVALID, "null argument");
    if (slot < 0 || slot >= Dev::kSlots) return fail(RT_ERR_INVALID, "frame slot out of range");
    Dev &d = ctx->devs[0];
    RT_CK(cudaSetDevice(d.id));
    if (!d.slot_busy[slot]) return RT_OK;
    return slot_finish(ctx, d, slot);
}

int rt_copy_partition_to_host(rt_ctx *ctx, int32_t slot, uint32_t *host_frame, const uint32_t *d_frame, int32_t width,
                              int32_t height, int32_t part, int32_t n_parts, int32_t block_rows, void *stream) {
    if (!ctx || !host_frame || !d_frame) return fail(RT_ERR_INVALID, "null argument");
    if (slot < 0 || slot >= (int)ctx->devs.size()) return fail(RT_ERR_INVALID, "bad device slot");
    if (width < 1 || height < 1 || n_parts < 1 || part < 0 || part >= n_parts || block_rows < 1)
        return fail(RT_ERR_INVALID, "bad partition");
    Dev &d = ctx->devs[slot];
    RT_CK(cudaSetDevice(d.id));
    cudaStream_t st = stream ? (cudaStream_t)stream : d.st;
    int rc;
    if (ctx->codec && width <= rt::kCodecMaxWidth) {
        // compressed (option codec, frame_codec.h): the partition's rows encoded
        // into mapped host memory, then expanded block by block by host threads
        if ((rc = d.part_codec.ensure(rt::codec_host_bytes(width, height)))) return rc;
        RT_CK(rt::launch_encode_rows(d_frame, width, width, height, 0, height, (uint32_t *)d.part_codec.dp, st, part,
                                     n_parts, block_rows));
        RT_CK(cudaStreamSynchronize(st));
        const int n_blocks = (height + block_rows - 1) / block_rows;
        const int mine = n_blocks > part ? (n_blocks - part + n_parts - 1) / n_parts : 0;
        int64_t words = 0;
#pragma omp parallel for num_threads(std::max(1, std::min(codec_threads(ctx), mine))) schedule(dynamic) reduction(+ : words)
        for (int i = 0; i < mine; i++) {
            const int y0 = (part + i * n_parts) * block_rows;
            words += rt::decode_rows_serial((const uint32_t *)d.part_codec.p, width, y0, std::min(height, y0 + block_rows),
                                            host_frame, width);
        }
        ctx->last_d2h_bytes = (int64_t)sizeof(uint32_t) * words;
        return RT_OK;
    }
    rc = copy_partition(host_frame, d_frame, sizeof(uint32_t), width, height, part, n_parts, block_rows, st);
    if (rc) return rc;
    RT_CK(cudaStreamSynchronize(st));
    return RT_OK;
}

int rt_device_malloc(int32_t device, size_t bytes, void **d_ptr_out) {
    if (!d_ptr_out || bytes == 0) return fail(RT_ERR_INVALID, "bad allocation request");
    *d_ptr_out = nullptr;
    RT_CK(cudaSetDevice(device));
    cudaError_t e = cudaMalloc(d_ptr_out, bytes);
    if (e != cudaSuccess) return fail(RT_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return RT_OK;
}

int rt_device_free(void *d_ptr) {
    if (!d_ptr) return RT_OK;
    RT_CK(cudaFree(d_ptr));
    return RT_OK;
}

int rt_fp32_peak_tflops(int32_t device, double *tflops) {
    if (!tflops) return fail(RT_ERR_INVALID, "null argument");
    RT_CK(cudaSetDevice(device));
    int sms = 0;
    RT_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    float *sink = nullptr;
    RT_CK(cudaMalloc(&sink, 1024 * sizeof(float)));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int threads = 256, blocks = sms * 8, iters = 2048;
    ffma_peak_kernel<<<blocks, threads>>>(sink, 64, 1.0001f, 0.5f);  // warm-up / clock ramp
    ffma_peak_kernel<<<blocks, threads>>>(sink, iters, 1.0001f, 0.5f);
    cudaEventRecord(a);
    ffma_peak_kernel<<<blocks, threads>>>(sink, iters, 1.0001f, 0.5f);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (e != cudaSuccess) return fail(RT_ERR_CUDA, std::string("ffma peak: ") + cudaGetErrorString(e));
    double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return RT_OK;
}

}  // extern "C"
