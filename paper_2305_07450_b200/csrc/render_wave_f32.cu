// FP32 wavefront render for soft shadows (shadow_samples >= kWaveMinSamples).
//
// The reference computes each pixel start to finish (renderer.py:227-279):
// ~99% of its work is the soft-shadow loop (`_shadow_coeff`, renderer.py:
// 82-105), 200 shadow rays per hit at the benchmark's s=200, and the number
// of hits per pixel ranges from 0 (sky) to bounce_limit+1.  One thread per
// pixel therefore leaves SMs and lanes idle on the uneven tail.  Here a frame
// is three kernels over HBM/L2-resident queues:
//
//   A  trace   one thread per pixel: the bounce chain (closest hit,
//              geometry.py:191-201), per hit the shading inputs that do not
//              depend on the shadow (Lambert and Blinn factors,
//              shading.py:53-73); hits are appended to a compact queue with
//              one warp-aggregated atomic per warp and bounce;
//   B  shadow  LANES lanes per queued hit, each a slice of the disc samples
//              (a lane takes samples sub, sub+LANES, ...), counts reduced with
//              warp shuffles: every warp does identical work, the any-hit
//              test is branch-free, so lanes and SMs stay busy to the end;
//   C  shade   one thread per pixel: the unwind (renderer.py:185-224) and the
//              pack (renderer.py:45-50).
//
// Per-hit state in HBM, slot = k * n_pix + local pixel (k = bounce):
//   hit_p  float4 {p.x, p.y, p.z, body index (int bits)}   16 B
//   hit_n  float4 {n.x, n.y, n.z, Lambert factor}           16 B
//   hit_s  float  Blinn factor max(n.h,0)^refl               4 B
//   hit_sc float  shadow coefficient                          4 B
//   queue  int    slots with a hit                            4 B
//   pix    float4 {tail rgb, records | exhausted << 8}      16 B per pixel
// At C2 (1280x720, 640 k hits) that is ~40 MB, L2-resident.
//
// Arithmetic is the megakernel's (render_f32.cu) operation for operation, so
// both paths give the same frames.
#include "rt_f32.cuh"

namespace {
using namespace rt;
using namespace rt32;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// --- A: bounce chains --------------------------------------------------------
template <class Geo>
__device__ __forceinline__ void trace_chain(const Geo &geo, const FrameArgs &fa, const SceneArgs<float> &sa,
                                            const WaveArgs &wa, int x, int ly) {
    if (x >= fa.width || ly >= fa.local_rows) return;
    int y = map_row(ly, fa);
    if (y >= fa.height) return;
    const int64_t lp = (int64_t)ly * fa.width + x;
    float3 origin = f3((float)fa.cam[0], (float)fa.cam[1], (float)fa.cam[2]);
    float3 dir = primary_direction(x, y, fa);
    const float3 light = f3(sa.light[0], sa.light[1], sa.light[2]);
    float3 tail = f3(0.f, 0.f, 0.f);
    int m = 0, exhausted = 0;
    for (int k = 0; k <= fa.bounces; k++) {
        Hit h = geo.closest(origin, dir);
        if (h.idx < 0) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            break;
        }
        float3 hit = origin + dir * h.t;
        float3 normal = h.g.w >= 0.f ? normalize3(hit - f3(h.g.x, h.g.y, h.g.z)) : f3(0.f, 1.f, 0.f);
        float3 l = normalize3(light - hit);
        float dfs = fmaxf(dot3(normal, l), 0.f);
        float3 hv = l - dir;
        float hm2 = dot3(hv, hv);
        float s = 0.f;
        if (hm2 > 0.f) {
            float dd = fmaxf(dot3(normal, hv) * rsqrtf(hm2), 0.f);
            s = powf(dd, __ldg(sa.mat + 8 * h.idx + 4));
        }
        const int64_t slot = (int64_t)k * wa.n_pix + lp;
        wa.hit_p[slot] = make_float4(hit.x, hit.y, hit.z, __int_as_float(h.idx));
        wa.hit_n[slot] = make_float4(normal.x, normal.y, normal.z, dfs);
        wa.hit_s[slot] = s;
        // enqueue: one atomic per warp (lanes still in the chain at bounce k)
        unsigned act = __activemask();
        int leader = __ffs(act) - 1;
        unsigned base = 0;
        if ((threadIdx.x & 31) == leader) base = atomicAdd(wa.count, (unsigned)__popc(act));
        base = __shfl_sync(act, base, leader);
        wa.queue[base + __popc(act & lanemask_lt())] = (int)slot;
        m = k + 1;
        if (k == fa.bounces) {
            exhausted = 1;
            break;
        }
        origin = hit + normal * 1e-3f;
        dir = dir - normal * (2.f * dot3(normal, dir));
    }
    wa.pix[lp] = make_float4(tail.x, tail.y, tail.z, __int_as_float(m | (exhausted << 8)));
}

template <int MAXS>
__global__ void __launch_bounds__(kThreads)
    wave_trace_param(const FrameArgs fa, const SceneArgs<float> sa, const WaveArgs wa, const ParamScene<MAXS> ps) {
    int x, ly;
    thread_pixel(x, ly);
    trace_chain(ps, fa, sa, wa, x, ly);
}

template <bool SMEM>
__global__ void __launch_bounds__(kThreads)
    wave_trace_mem(const FrameArgs fa, const SceneArgs<float> sa, const WaveArgs wa) {
    extern __shared__ float4 smem_geo[];
    MemScene geo{reinterpret_cast<const float4 *>(sa.geo), sa.n};
    if constexpr (SMEM) {
        for (int i = threadIdx.x; i < sa.n; i += blockDim.x) smem_geo[i] = geo.geo[i];
        __syncthreads();
        geo.geo = smem_geo;
    }
    int x, ly;
    thread_pixel(x, ly);
    trace_chain(geo, fa, sa, wa, x, ly);
}

// --- B: shadow coefficients (renderer.py:82-105) ------------------------------
// LANES lanes per hit; a warp holds 32/LANES hits and walks the queue in
// lockstep so the shuffles see the whole warp.
template <int LANES, class Geo>
__device__ __forceinline__ void shadow_queue(const Geo &geo, const SceneArgs<float> &sa, const WaveArgs &wa,
                                             int n) {
    extern __shared__ float2 smem_tab[];
    const float2 *__restrict__ tab = reinterpret_cast<const float2 *>(sa.table);
    if (n > 1 && n <= kWaveSmemSamples) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) smem_tab[i] = tab[i];
        __syncthreads();
        tab = smem_tab;
    }
    const unsigned count = *wa.count;
    const int lane = threadIdx.x & 31;
    const int sub = lane % LANES;
    constexpr int kHitsPerWarp = 32 / LANES;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned n_warps = (gridDim.x * blockDim.x) >> 5;
    const float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
    for (unsigned base = warp * kHitsPerWarp; base < count; base += n_warps * kHitsPerWarp) {
        const unsigned q = base + lane / LANES;
        const bool live = q < count;
        int unblocked = 0;
        int slot = 0;
        if (live) {
            slot = __ldg(wa.queue + q);
            float4 P = __ldg(wa.hit_p + slot);
            float4 N = __ldg(wa.hit_n + slot);
            float3 surface = f3(P.x, P.y, P.z), normal = f3(N.x, N.y, N.z);
            float3 origin = surface + normal * 1e-3f;
            const auto lc = geo.localize(origin);
            if (n == 1) {
                if (sub == 0) {
                    float3 dir = normalize3(lp - origin);
                    float3 e = surface - lp;
                    float l2 = dot3(e, e);
                    float limit = l2 > 0.f ? l2 * rsqrtf(l2) : 0.f;
                    unblocked = geo.occluded(lc, dir, limit) ? 0 : 1;
                }
            } else {
                DiscBasis db = disc_basis(surface, lp);
                float3 lo = lp - origin, ls = surface - lp;
#pragma unroll 2
                for (int i = sub; i < n; i += LANES) {
                    float2 ab = tab[i];
                    float3 off = db.bu * ab.x + db.bv * ab.y;
                    float3 dv = lo + off;
                    float r2 = dot3(dv, dv);
                    float3 dir = dv * (r2 > 0.f ? rsqrtf(r2) : 0.f);
                    float3 e = ls - off;
                    float l2 = dot3(e, e);
                    float limit = l2 > 0.f ? l2 * rsqrtf(l2) : 0.f;
                    unblocked += geo.occluded(lc, dir, limit) ? 0 : 1;
                }
            }
        }
#pragma unroll
        for (int o = LANES / 2; o > 0; o >>= 1) unblocked += __shfl_xor_sync(0xffffffffu, unblocked, o);
        if (live && sub == 0) wa.hit_sc[slot] = (float)unblocked / (float)n;
    }
}

#ifndef RT_WAVE_MIN_BLOCKS
#define RT_WAVE_MIN_BLOCKS 1
#endif

template <int LANES, int MAXS>
__global__ void __launch_bounds__(kThreads, RT_WAVE_MIN_BLOCKS)
    wave_shadow_param(const SceneArgs<float> sa, const WaveArgs wa, int n, const ParamScene<MAXS> ps) {
    shadow_queue<LANES>(ps, sa, wa, n);
}

template <int LANES>
__global__ void __launch_bounds__(kThreads) wave_shadow_mem(const SceneArgs<float> sa, const WaveArgs wa, int n) {
    MemScene geo{reinterpret_cast<const float4 *>(sa.geo), sa.n};
    shadow_queue<LANES>(geo, sa, wa, n);
}

// --- C: unwind + pack (renderer.py:185-224, 45-50) ----------------------------
__global__ void __launch_bounds__(kThreads) wave_shade(const FrameArgs fa, const SceneArgs<float> sa,
                                                       const WaveArgs wa) {
    int x, ly;
    thread_pixel(x, ly);
    if (x >= fa.width || ly >= fa.local_rows) return;
    int y = map_row(ly, fa);
    if (y >= fa.height) return;
    const int64_t lp = (int64_t)ly * fa.width + x;
    float4 px = wa.pix[lp];
    int info = __float_as_int(px.w);
    int m = info & 0xff;
    bool exhausted = (info >> 8) & 1;
    float3 col = f3(px.x, px.y, px.z);
    for (int k = m - 1; k >= 0; k--) {
        const int64_t slot = (int64_t)k * wa.n_pix + lp;
        int idx = __float_as_int(wa.hit_p[slot].w);
        float dfs = wa.hit_n[slot].w;
        float s = wa.hit_s[slot];
        float sc = wa.hit_sc[slot];
        float lum = fminf(sa.ambient + sc * dfs * (1.f - sa.ambient), 1.f);
        float sp = sc * s;
        const float4 mt = __ldg(reinterpret_cast<const float4 *>(sa.mat + 8 * idx));
        float br = mt.x, bg = mt.y, bb = mt.z;
        if (!(exhausted && k == m - 1)) {
            float rr = mt.w;
            br = br * (1.f - rr) + col.x * rr;
            bg = bg * (1.f - rr) + col.y * rr;
            bb = bb * (1.f - rr) + col.z * rr;
        }
        col = f3(clamp01(br * lum + sa.lc[0] * sp), clamp01(bg * lum + sa.lc[1] * sp),
                 clamp01(bb * lum + sa.lc[2] * sp));
    }
    fa.out[(int64_t)y * fa.out_pitch + x] = pack_color(col.x, col.y, col.z);
    if (fa.radiance) {
        float *r = (float *)fa.radiance + 3 * ((int64_t)y * fa.width + x);
        r[0] = col.x;
        r[1] = col.y;
        r[2] = col.z;
    }
    if (fa.peer_out) __threadfence_system();
}

template <int LANES>
cudaError_t launch_shadow(const SceneArgs<float> &sa, const WaveArgs &wa, int n, cudaStream_t st, bool param8,
                          const ParamScene<8> &p8, bool param256, const ParamScene<kParamSpheres> &p256) {
    size_t smem = (n > 1 && n <= kWaveSmemSamples) ? sizeof(float2) * (size_t)n : 0;
    if (param8) {
        int ctas = resident_ctas(wave_shadow_param<LANES, 8>, smem);
        wave_shadow_param<LANES, 8><<<ctas, kThreads, smem, st>>>(sa, wa, n, p8);
    } else if (param256) {
        int ctas = resident_ctas(wave_shadow_param<LANES, kParamSpheres>, smem);
        wave_shadow_param<LANES, kParamSpheres><<<ctas, kThreads, smem, st>>>(sa, wa, n, p256);
    } else {
        int ctas = resident_ctas(wave_shadow_mem<LANES>, smem);
        wave_shadow_mem<LANES><<<ctas, kThreads, smem, st>>>(sa, wa, n);
    }
    return cudaGetLastError();
}

}  // namespace

// Lanes per hit: enough samples per lane (>= 16) to amortise the per-hit
// setup, as many lanes as that allows (up to a warp).
int rt_wave_lanes(int samples) {
    int lanes = 1;
    while (lanes < 32 && samples / (lanes * 2) >= 16) lanes *= 2;
    return lanes;
}

cudaError_t rt_launch_wave_f32(const rt::FrameArgs &fa, const rt::SceneArgs<float> &sa, const rt::WaveArgs &wa,
                               cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(wa.count, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    dim3 grid((fa.width + kTileW - 1) / kTileW, (fa.local_rows + kTileH - 1) / kTileH);
    ParamScene<8> p8;
    thread_local ParamScene<kParamSpheres> p256;
    bool param8 = pack_params(sa, p8);
    bool param256 = !param8 && pack_params(sa, p256);
    if (param8)
        wave_trace_param<8><<<grid, kThreads, 0, st>>>(fa, sa, wa, p8);
    else if (param256)
        wave_trace_param<kParamSpheres><<<grid, kThreads, 0, st>>>(fa, sa, wa, p256);
    else if (sizeof(float4) * (size_t)sa.n <= (size_t)kSmemGeoBytes)
        wave_trace_mem<true><<<grid, kThreads, sizeof(float4) * sa.n, st>>>(fa, sa, wa);
    else
        wave_trace_mem<false><<<grid, kThreads, 0, st>>>(fa, sa, wa);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    switch (rt_wave_lanes(fa.samples)) {
        case 1: e = launch_shadow<1>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        case 2: e = launch_shadow<2>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        case 4: e = launch_shadow<4>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        case 8: e = launch_shadow<8>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        case 16: e = launch_shadow<16>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        default: e = launch_shadow<32>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
    }
    if (e != cudaSuccess) return e;
    wave_shade<<<grid, kThreads, 0, st>>>(fa, sa, wa);
    return cudaGetLastError();
}
