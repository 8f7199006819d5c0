// FP32 frame render — the product path on the B200 CUDA cores.
//
// One thread per pixel, a warp per 8x4 pixel patch.  Same control flow as the
// reference (/root/reference/pkg/src/raytracer/renderer.py:108-279): closest
// hit, sunflower soft-shadow coefficient, bounded reflections with a
// register-resident record stack, skybox on miss, Blinn-Phong unwind, pack to
// 0xAARRGGBB.
//
// Scene residency: scenes of up to kParamSpheres spheres and kMaxPlanes
// planes travel inside the kernel's launch parameters (constant bank 0), so
// every warp-uniform body loop reads its operands straight from the constant
// cache with no load instructions and no shared/global traffic; larger scenes
// are staged in shared memory (or read through L1 when they do not fit).
//
// FP32-specific numerics (measured in SURVEY.md §8c):
//  - the sphere test forms the squared ray-to-centre distance as
//    |L - tca*d|^2 instead of L.L - tca^2 (geometry.py:96): algebraically
//    identical, free of the cancellation that makes FP32 misjudge long shadow
//    rays from far plane points and rays near silhouettes;
//  - the any-hit shadow test decides `tca - sqrt(rad) in [0, limit)`
//    (geometry.py:94-104, 204-210) without the square root:
//    t >= 0  <=>  tca^2 >= rad,   t < limit  <=>  tca - limit < 0 or (tca - limit)^2 < rad;
//    the plane test `0 < (h - o.y)/d.y < limit` without the division;
//  - the ray chain (primary direction, hit points, normals, reflections) runs
//    in float64 (rt_f32.cuh: refine_hit) — the search, shadows and shading in FP32;
//  - the disc-sample table is built in float64 on the host and rounded.
#include "rt_f32.cuh"

namespace {
using namespace rt;
using namespace rt32;

// renderer.py:82-105 (+ shading.py:76-86 disc basis, 89-100 disc points)
template <class Geo>
__device__ float shadow_coeff(const Geo &geo, float3 surface, float3 normal, const SceneArgs<float> &sa, int n,
                             const MegaCull &mc) {
    const float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
    const ShadowFrame f = shadow_frame(surface, normal, lp, n > 1);
    const auto lc = geo.localize(f.origin, scene_grid_mask(mc, f.origin));
    const float4 *__restrict__ tab = reinterpret_cast<const float4 *>(sa.table);
    if (n == 1) {  // hard shadows: one ray, the ruled-out spheres skipped
        float3 dir;
        float limit;
        shadow_ray(f, make_float4(0.f, 0.f, 0.f, 0.f), dir, limit);
        return geo.template occluded<true>(lc, dir, limit) ? 0.f : 1.f;
    }
    int unblocked = 0;
#pragma unroll 2
    for (int i = 0; i < n; i++) {
        float3 dir;
        float limit;
        shadow_ray(f, __ldg(tab + i), dir, limit);
        unblocked += geo.occluded(lc, dir, limit) ? 0 : 1;
    }
    return (float)unblocked / (float)n;
}

// renderer.py:108-224.  A record keeps (body, lum, spec): shade_color's
// luminance and specular terms (shading.py:159-165) depend only on the hit,
// so the unwind only mixes, scales and clamps.  The bounce loop is not
// unrolled (it would copy the shadow loop per bounce); the 12-byte records
// live in L1-resident local memory.
// The ray chain runs in float64 (rt_f32.cuh: refine_hit): the FP32 body
// search, shadow rays and shading work on its rounded values.
template <int BMAX, class Geo>
__device__ float3 trace(const Geo &geo, D3 o64, D3 d64, const SceneArgs<float> &sa, int samples,
                        int bounces, const MegaCull &mc, unsigned smask = ~0u) {
    int ridx[BMAX + 1];
    float rlum[BMAX + 1], rspec[BMAX + 1];
    int m = 0;
    bool exhausted = false;
    float3 tail = f3(0.f, 0.f, 0.f);
    float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
#pragma unroll(BMAX <= 1 ? BMAX + 1 : 1)
    for (int k = 0; k <= BMAX; k++) {
        if (k > bounces) break;
        const float3 origin = rnd(o64), dir = rnd(d64);
        Hit h = k == 0 ? geo.template closest<true>(origin, dir, smask) : geo.closest(origin, dir);
        if (h.idx < 0) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            break;
        }
        D3 p64, n64;
        refine_hit(o64, d64, sa.geo64, sa.n, h.idx, p64, n64);
        const float3 hit = rnd(p64), normal = rnd(n64);
        float3 l = normalize3(lp - hit);
        float sc = shadow_coeff(geo, hit, normal, sa, samples, mc);
        // shading.py:53-73, 159-162 (view = -dir)
        float dfs = fmaxf(dot3(normal, l), 0.f);
        float3 hv = l - dir;
        float hm2 = dot3(hv, hv);
        float s = 0.f;
        if (hm2 > 0.f) {
            float dd = fmaxf(dot3(normal, hv) * rsqrtf(hm2), 0.f);
            s = blinn_pow(dd, __ldg(sa.mat + 8 * h.idx + 4));
        }
        float lum = fminf(sa.ambient + sc * dfs * (1.f - sa.ambient), 1.f);
        ridx[k] = h.idx;
        rlum[k] = lum;
        rspec[k] = sc * s;
        m = k + 1;
        if (k == bounces) {
            exhausted = true;
            break;
        }
        reflect64(p64, n64, o64, d64);
    }
    float3 col = tail;
#pragma unroll(BMAX <= 1 ? BMAX + 1 : 1)
    for (int k = BMAX <= 1 ? BMAX : m - 1; k >= 0; k--) {
        if (k >= m) continue;  // (BMAX <= 1: unrolled, the records stay in registers)
        const float4 mt = __ldg(reinterpret_cast<const float4 *>(sa.mat + 8 * ridx[k]));
        float br = mt.x, bg = mt.y, bb = mt.z;
        if (!(exhausted && k == m - 1)) {
            float rr = mt.w;
            br = br * (1.f - rr) + col.x * rr;
            bg = bg * (1.f - rr) + col.y * rr;
            bb = bb * (1.f - rr) + col.z * rr;
        }
        float lum = rlum[k], sp = rspec[k];
        col = f3(clamp01(br * lum + sa.lc[0] * sp), clamp01(bg * lum + sa.lc[1] * sp),
                 clamp01(bb * lum + sa.lc[2] * sp));
    }
    return col;
}

template <int BMAX, class Geo>
__device__ __forceinline__ void shade_pixel(const Geo &geo, const FrameArgs &fa, const SceneArgs<float> &sa,
                                            const MegaCull &mc, int x,
                                            int ly) {
    if (x >= fa.width || ly >= fa.local_rows) return;
    int y = map_row(ly, fa);
    if (y >= fa.row_end) return;
    float3 c = trace<BMAX>(geo, D3{fa.cam[0], fa.cam[1], fa.cam[2]}, primary_direction64(x, y, fa), sa, fa.samples,
                           fa.bounces, mc, primary_sphere_mask(mc, x, y));
    fa.out[(int64_t)y * fa.out_pitch + x] = pack_color(c.x, c.y, c.z, fa.rgba);
    if (fa.radiance) {
        float *r = (float *)fa.radiance + 3 * ((int64_t)y * fa.width + x);
        r[0] = c.x;
        r[1] = c.y;
        r[2] = c.z;
    }
}

// Persistent warps: every warp takes 8x4-pixel patches from a frame-wide
// counter until the frame is done.  A patch's cost ranges from a handful of
// instructions (sky) to ~10^5 per lane (four soft-shadowed hits), so
// scheduling per warp instead of per CTA keeps every SM busy to the end;
// patches are handed out bottom rows first (the scene, below the horizon)
// so the cheap sky patches fill the tail.
template <int BMAX, class Geo>
__device__ __forceinline__ void render_patches(const Geo &geo, const FrameArgs &fa, const SceneArgs<float> &sa,
                                               const MegaCull &mc) {
    const int lane = threadIdx.x & 31;
    const int pw = (fa.width + 7) >> 3;
    const int ph = (fa.local_rows + 3) >> 2;
    const unsigned n_patches = (unsigned)pw * (unsigned)ph;
    for (;;) {
        unsigned p = 0;
        if (lane == 0) p = atomicAdd(fa.work_counter, 1u);
        p = __shfl_sync(0xffffffffu, p, 0);
        if (p >= n_patches) break;
        int prow = ph - 1 - (int)(p / (unsigned)pw);
        int pcol = (int)(p % (unsigned)pw);
        shade_pixel<BMAX>(geo, fa, sa, mc, pcol * 8 + (lane & 7), prow * 4 + (lane >> 3));
        __syncwarp();
    }
    if (fa.peer_out) __threadfence_system();  // frame stores over NVLink land before the kernel retires
}

template <int BMAX, int MAXS>
__global__ void __launch_bounds__(kThreads, RT_F32_MIN_BLOCKS)
    render_f32_param_kernel(const FrameArgs fa, const SceneArgs<float> sa, const ParamScene<MAXS> ps,
                            const MegaCull mc) {
    render_patches<BMAX>(ps, fa, sa, mc);
}

// One CTA per 16 x 8 tile, tile rows bottom first, no work counter: for
// frames whose pixels cost about the same (hard shadows, few samples), where
// one shared counter would serialise ~10^5 atomics per 4K frame.
#ifndef RT_F32_TILE_MIN_BLOCKS
#define RT_F32_TILE_MIN_BLOCKS 7  // 7 CTAs (<= 72 registers): 15-18% faster at s1 b1 than the uncapped 103
#endif
template <int BMAX, int MAXS>
__global__ void __launch_bounds__(kThreads, RT_F32_TILE_MIN_BLOCKS)
    render_f32_tile_kernel(const FrameArgs fa, const SceneArgs<float> sa, const ParamScene<MAXS> ps,
                           const MegaCull mc) {
    int x, ly;
    thread_pixel_hot_first(mc.hot, mc.hot_div, x, ly);
    shade_pixel<BMAX>(ps, fa, sa, mc, x, ly);
    if (fa.peer_out) __threadfence_system();
}

template <int BMAX, bool SMEM>
__global__ void __launch_bounds__(kThreads)
    render_f32_kernel(const FrameArgs fa, const SceneArgs<float> sa, const MegaCull mc) {
    extern __shared__ float4 smem_geo[];
    MemScene geo{reinterpret_cast<const float4 *>(sa.geo), sa.n};
    if constexpr (SMEM) {
        for (int i = threadIdx.x; i < sa.n; i += blockDim.x) smem_geo[i] = geo.geo[i];
        __syncthreads();
        geo.geo = smem_geo;
    }
    render_patches<BMAX>(geo, fa, sa, mc);
}

template <int BMAX, int MAXS>
__global__ void __launch_bounds__(kThreads)
    trace_f32_param_kernel(const double *orig, const double *dirs, int64_t n_rays, float *out,
                           const SceneArgs<float> sa, int samples, int bounces, const ParamScene<MAXS> ps) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rays) return;
    float3 c = trace<BMAX>(ps, D3{orig[3 * i], orig[3 * i + 1], orig[3 * i + 2]},
                           D3{dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]}, sa, samples, bounces, MegaCull{});
    out[3 * i] = c.x;
    out[3 * i + 1] = c.y;
    out[3 * i + 2] = c.z;
}

template <int BMAX>
__global__ void __launch_bounds__(kThreads)
    trace_f32_kernel(const double *orig, const double *dirs, int64_t n_rays, float *out, const SceneArgs<float> sa,
                     int samples, int bounces) {
    MemScene geo{reinterpret_cast<const float4 *>(sa.geo), sa.n};
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rays) return;
    float3 c = trace<BMAX>(geo, D3{orig[3 * i], orig[3 * i + 1], orig[3 * i + 2]},
                           D3{dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]}, sa, samples, bounces, MegaCull{});
    out[3 * i] = c.x;
    out[3 * i + 1] = c.y;
    out[3 * i + 2] = c.z;
}

template <int BMAX>
cudaError_t launch_render(const FrameArgs &fa, const SceneArgs<float> &sa, cudaStream_t st, bool tiles,
                          const MegaCull &mc) {
    if (tiles) {
        const dim3 grid((fa.width + kTileW - 1) / kTileW, (fa.local_rows + kTileH - 1) / kTileH);
        ParamScene<8> ps;
        if (pack_params(sa, ps)) {
            render_f32_tile_kernel<BMAX, 8><<<grid, kThreads, 0, st>>>(fa, sa, ps, mc);
            return cudaGetLastError();
        }
        thread_local ParamScene<kParamSpheres> pl;
        if (pack_params(sa, pl)) {
            render_f32_tile_kernel<BMAX, kParamSpheres><<<grid, kThreads, 0, st>>>(fa, sa, pl, mc);
            return cudaGetLastError();
        }
        return cudaErrorNotSupported;  // larger scenes take the persistent kernels
    }
    {
        ParamScene<8> ps;
        if (pack_params(sa, ps)) {
            static thread_local int ctas = 0;
            if (!ctas) ctas = resident_ctas(render_f32_param_kernel<BMAX, 8>, 0);
            render_f32_param_kernel<BMAX, 8><<<ctas, kThreads, 0, st>>>(fa, sa, ps, mc);
            return cudaGetLastError();
        }
    }
    {
        thread_local ParamScene<kParamSpheres> ps;  // 5 KB: keep it off the stack
        if (pack_params(sa, ps)) {
            static thread_local int ctas = 0;
            if (!ctas) ctas = resident_ctas(render_f32_param_kernel<BMAX, kParamSpheres>, 0);
            render_f32_param_kernel<BMAX, kParamSpheres><<<ctas, kThreads, 0, st>>>(fa, sa, ps, mc);
            return cudaGetLastError();
        }
    }
    size_t geo_bytes = sizeof(float4) * (size_t)sa.n;
    if (geo_bytes <= (size_t)kSmemGeoBytes) {
        int ctas = resident_ctas(render_f32_kernel<BMAX, true>, geo_bytes);
        render_f32_kernel<BMAX, true><<<ctas, kThreads, geo_bytes, st>>>(fa, sa, mc);
    } else {
        static thread_local int ctas = 0;
        if (!ctas) ctas = resident_ctas(render_f32_kernel<BMAX, false>, 0);
        render_f32_kernel<BMAX, false><<<ctas, kThreads, 0, st>>>(fa, sa, mc);
    }
    return cudaGetLastError();
}

template <int BMAX>
cudaError_t launch_trace(const double *o, const double *d, int64_t n, float *out, const SceneArgs<float> &sa,
                         int samples, int bounces, cudaStream_t st) {
    unsigned blocks = (unsigned)((n + kThreads - 1) / kThreads);
    {
        ParamScene<8> ps;
        if (pack_params(sa, ps)) {
            trace_f32_param_kernel<BMAX, 8><<<blocks, kThreads, 0, st>>>(o, d, n, out, sa, samples, bounces, ps);
            return cudaGetLastError();
        }
    }
    trace_f32_kernel<BMAX><<<blocks, kThreads, 0, st>>>(o, d, n, out, sa, samples, bounces);
    return cudaGetLastError();
}

}  // namespace

cudaError_t rt_launch_render_f32(const rt::FrameArgs &fa, const rt::SceneArgs<float> &sa, cudaStream_t st,
                                 bool tiles, const rt::MegaCull &mc) {
    if (fa.bounces <= 1) return launch_render<1>(fa, sa, st, tiles, mc);
    return launch_render<rt::kMaxBounce>(fa, sa, st, tiles, mc);
}

cudaError_t rt_launch_trace_f32(const double *o, const double *d, int64_t n, float *out,
                                const rt::SceneArgs<float> &sa, int samples, int bounces, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    return launch_trace<rt::kMaxBounce>(o, d, n, out, sa, samples, bounces, st);
}
