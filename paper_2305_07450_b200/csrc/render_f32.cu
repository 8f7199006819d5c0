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
//  - primary directions are formed in float64 (camera.py:70-77) and rounded;
//  - the disc-sample table is built in float64 on the host and rounded.
#include "rt_device.cuh"

namespace {
using namespace rt;

#ifndef RT_F32_MIN_BLOCKS
#define RT_F32_MIN_BLOCKS 1  // __launch_bounds__ minimum resident CTAs per SM (register cap)
#endif

constexpr int kMaxPlanes = 8;
constexpr int kParamSpheres = 256;

__device__ __forceinline__ float3 f3(float x, float y, float z) { return make_float3(x, y, z); }
__device__ __forceinline__ float3 operator+(float3 a, float3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ float3 operator-(float3 a, float3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ float3 operator*(float3 a, float s) { return f3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float3 cross3(float3 a, float3 b) {
    return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
// vecmath.py:68-78: zero vector normalises to zero
__device__ __forceinline__ float3 normalize3(float3 a) {
    float m2 = dot3(a, a);
    float inv = m2 > 0.f ? rsqrtf(m2) : 0.f;
    return a * inv;
}

// camera.py:46-77 in float64 (exactly the reference's direction), then rounded
__device__ __forceinline__ float3 primary_direction(int xi, int yi, const FrameArgs &fa) {
    double x = (double)xi, y = (double)yi, w = (double)fa.width, h = (double)fa.height;
    double u, v;
    if (w > h) {
        u = (x - w / 2 + h / 2) / h * 2 - 1;
        v = -(y / h * 2 - 1);
    } else {
        u = x / w * 2 - 1;
        v = -((y - h / 2 + w / 2) / w * 2 - 1);
    }
    double m = sqrt(u * u + v * v + fa.vdist * fa.vdist);
    double dx = u / m, dy = v / m, dz = fa.vdist / m;
    double y2 = dy * fa.cb - dz * fa.sb;
    double z2 = dy * fa.sb + dz * fa.cb;
    double x2 = dx * fa.ca + z2 * fa.sa;
    double z3 = -dx * fa.sa + z2 * fa.ca;
    return f3((float)x2, (float)y2, (float)z3);
}

// geometry.py:83-105 — distance to the sphere, +inf on a miss.
__device__ __forceinline__ float sphere_t(float3 o, float3 d, float4 g) {
    float3 L = f3(g.x - o.x, g.y - o.y, g.z - o.z);
    float tca = dot3(L, d);
    float3 p = L - d * tca;
    float rad = g.w - dot3(p, p);
    float t = tca - sqrtf(fmaxf(rad, 0.f));
    bool hit = (tca >= 0.f) & (rad >= -1e-7f) & (t >= 0.f);
    return hit ? t : INFINITY;
}

// geometry.py:108-117
__device__ __forceinline__ float plane_t(float3 o, float3 d, float h) {
    float t = (h - o.y) / d.y;
    return (d.y != 0.f && t > 0.f) ? t : INFINITY;
}

// occluded_packed's per-body predicate `intersect(...) < limit`
// (geometry.py:94-117, 204-210) as a signed margin: the body blocks the
// shadow ray iff the returned value is > 0.  Written with FMA-pipe arithmetic
// and min/max so a test costs ~13 FMA-pipe and ~4 ALU-pipe instructions and
// no branch:
//   sphere: tca >= 0, rad >= -GRAZE, origin outside (tca^2 >= rad), and
//           t = tca - sqrt(max(rad, 0)) < limit  <=>  min(q, q^2 - rad) < 0, q = tca - limit;
//   plane:  0 < (h - o.y)/d.y < limit  <=>  min(num*dy, limit*|dy| - |num|) > 0.
constexpr float kGraze = 1e-7f;  // geometry.py:24

// L = centre - origin; r2g = r^2 + GRAZE, or -inf when the origin is inside
// the sphere (t < 0 for every direction: it never blocks).
__device__ __forceinline__ float sphere_margin_L(float3 L, float3 d, float r2g, float limit) {
    float tca = fmaf(L.z, d.z, fmaf(L.y, d.y, L.x * d.x));
    float px = fmaf(-tca, d.x, L.x), py = fmaf(-tca, d.y, L.y), pz = fmaf(-tca, d.z, L.z);
    float radg = fmaf(-pz, pz, fmaf(-py, py, fmaf(-px, px, r2g)));  // rad + GRAZE
    float q = tca - limit;
    float e = fmaf(q, q, kGraze) - radg;  // q^2 - rad
    return fminf(fminf(tca, radg), -fminf(q, e));
}

__device__ __forceinline__ float sphere_r2g(float3 L, float r2) {
    return dot3(L, L) >= r2 ? r2 + kGraze : -INFINITY;
}

__device__ __forceinline__ float sphere_margin(float3 o, float3 d, float4 g, float limit) {
    float3 L = f3(g.x - o.x, g.y - o.y, g.z - o.z);
    return sphere_margin_L(L, d, sphere_r2g(L, g.w), limit);
}

__device__ __forceinline__ float plane_margin(float num, float dy, float limit) {
    return fminf(num * dy, fmaf(limit, fabsf(dy), -fabsf(num)));
}

// A closest hit: original body index (tie-break and materials), distance,
// and the sphere centre (planes: w < 0).
struct Hit {
    int idx;
    float t;
    float4 g;
};

// --- scene accessors ---------------------------------------------------------------

// Scene in the launch parameters: spheres in original relative order, planes
// likewise, with their original indices for the lowest-index tie-break.
template <int MAXS>
struct ParamScene {
    float4 sph[MAXS];
    int sph_idx[MAXS];
    float pl_h[kMaxPlanes];
    int pl_idx[kMaxPlanes];
    int ns, np;

    __device__ __forceinline__ Hit closest(float3 o, float3 d) const {
        Hit h{-1, INFINITY, make_float4(0.f, 0.f, 0.f, -1.f)};
        int slot = -1;
#pragma unroll(MAXS <= 8 ? MAXS : 4)
        for (int b = 0; b < MAXS; b++) {
            if (b >= ns) break;
            float t = sphere_t(o, d, sph[b]);
            if (t < h.t) {  // spheres ascend in original index: strict '<' keeps the lowest
                h.t = t;
                slot = b;
            }
        }
        if (slot >= 0) {
            h.idx = sph_idx[slot];
            h.g = sph[slot];
        }
#pragma unroll
        for (int j = 0; j < kMaxPlanes; j++) {
            if (j >= np) break;
            float t = plane_t(o, d, pl_h[j]);
            if (t < h.t || (t == h.t && pl_idx[j] < h.idx)) {  // geometry.py:198 across kinds
                h.t = t;
                h.idx = pl_idx[j];
                h.g = make_float4(0.f, pl_h[j], 0.f, -1.f);
            }
        }
        return h;
    }

    // Per-hit constants of the any-hit loop: the shadow origin is shared by
    // all samples of a hit, so L = c - o, the inside/outside decision and
    // h - o.y are formed once per hit.
    struct Local {
        float3 o;
        float4 L[MAXS <= 8 ? MAXS : 1];  // xyz = centre - origin, w = r2g
        float num[kMaxPlanes];
    };

    __device__ __forceinline__ Local localize(float3 o) const {
        Local lc;
        lc.o = o;
        if constexpr (MAXS <= 8) {
#pragma unroll
            for (int b = 0; b < MAXS; b++) {
                float3 L = f3(sph[b].x - o.x, sph[b].y - o.y, sph[b].z - o.z);
                lc.L[b] = make_float4(L.x, L.y, L.z, sphere_r2g(L, sph[b].w));
            }
        }
#pragma unroll
        for (int j = 0; j < kMaxPlanes; j++) lc.num[j] = pl_h[j] - o.y;
        return lc;
    }

    __device__ __forceinline__ bool occluded(const Local &lc, float3 d, float limit) const {
        float m = -INFINITY;
#pragma unroll
        for (int j = 0; j < kMaxPlanes; j++) {
            if (j >= np) break;
            m = fmaxf(m, plane_margin(lc.num[j], d.y, limit));
        }
        if constexpr (MAXS <= 8) {
#pragma unroll
            for (int b = 0; b < MAXS; b++) {
                if (b >= ns) break;
                float4 L = lc.L[b];
                m = fmaxf(m, sphere_margin_L(f3(L.x, L.y, L.z), d, L.w, limit));
            }
        } else {
#pragma unroll 4
            for (int b = 0; b < MAXS; b++) {
                if (b >= ns) break;
                m = fmaxf(m, sphere_margin(lc.o, d, sph[b], limit));
                if ((b & 3) == 3 && m > 0.f) break;
            }
        }
        return m > 0.f;
    }
};

// Scene in shared memory / global memory in the reference's order:
// {cx, cy, cz, r^2} spheres, {0, h, 0, -1} planes.
struct MemScene {
    const float4 *__restrict__ geo;
    int n;

    __device__ __forceinline__ Hit closest(float3 o, float3 d) const {
        Hit h{-1, INFINITY, make_float4(0.f, 0.f, 0.f, -1.f)};
        for (int b = 0; b < n; b++) {
            float4 g = geo[b];
            float t = g.w >= 0.f ? sphere_t(o, d, g) : plane_t(o, d, g.y);
            if (t < h.t) {
                h.t = t;
                h.idx = b;
                h.g = g;
            }
        }
        return h;
    }

    struct Local {
        float3 o;
    };
    __device__ __forceinline__ Local localize(float3 o) const { return Local{o}; }

    __device__ __forceinline__ bool occluded(const Local &lc, float3 d, float limit) const {
        for (int b = 0; b < n; b++) {
            float4 g = geo[b];
            float m = g.w >= 0.f ? sphere_margin(lc.o, d, g, limit) : plane_margin(g.y - lc.o.y, d.y, limit);
            if (m > 0.f) return true;
        }
        return false;
    }
};

// renderer.py:82-105 (+ shading.py:76-86 disc basis, 89-100 disc points)
template <class Geo>
__device__ float shadow_coeff(const Geo &geo, float3 surface, float3 normal, const SceneArgs<float> &sa, int n) {
    float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
    float3 origin = surface + normal * 1e-3f;
    if (n == 1) {
        float3 dir = normalize3(lp - origin);
        float3 e = surface - lp;
        float l2 = dot3(e, e);
        float limit = l2 > 0.f ? l2 * rsqrtf(l2) : 0.f;
        return geo.occluded(geo.localize(origin), dir, limit) ? 0.f : 1.f;
    }
    float3 axis = normalize3(surface - lp);
    float3 c = cross3(axis, f3(0.f, 1.f, 0.f));
    float m2 = dot3(c, c);
    float3 bu = m2 >= 1e-18f ? c * rsqrtf(m2) : f3(1.f, 0.f, 0.f);
    float3 bv = cross3(axis, bu);
    // shadow ray i: dir = normalize(s_i - origin), limit = |surface - s_i|,
    // with s_i = lp + a_i bu + b_i bv; both share lp - origin / surface - lp.
    float3 lo = lp - origin;
    float3 ls = surface - lp;
    const float2 *__restrict__ tab = reinterpret_cast<const float2 *>(sa.table);
    const auto lc = geo.localize(origin);
    int unblocked = 0;
#pragma unroll 2
    for (int i = 0; i < n; i++) {
        float2 ab = __ldg(tab + i);
        float3 off = bu * ab.x + bv * ab.y;
        float3 dv = lo + off;
        float r2 = dot3(dv, dv);
        float3 dir = dv * (r2 > 0.f ? rsqrtf(r2) : 0.f);
        float3 e = ls - off;
        float l2 = dot3(e, e);
        float limit = l2 > 0.f ? l2 * rsqrtf(l2) : 0.f;
        unblocked += geo.occluded(lc, dir, limit) ? 0 : 1;
    }
    return (float)unblocked / (float)n;
}

// renderer.py:60-74
__device__ float3 sky_sample(float3 d, const float4 *__restrict__ sky, int W, int H) {
    float u = 0.5f + atan2f(d.x, d.z) * 0.15915494309189535f;
    float dy = fminf(fmaxf(d.y, -1.f), 1.f);
    float v = 0.5f - asinf(dy) * 0.3183098861837907f;
    int tx = (int)floorf(u * (float)W);
    tx = ((tx % W) + W) % W;
    int ty = (int)floorf(v * (float)H);
    ty = min(max(ty, 0), H - 1);
    float4 t = __ldg(sky + (int64_t)ty * W + tx);
    return f3(t.x, t.y, t.z);
}

__device__ __forceinline__ float clamp01(float x) { return fminf(fmaxf(x, 0.f), 1.f); }

// renderer.py:108-224.  A record keeps (body, lum, spec): shade_color's
// luminance and specular terms (shading.py:159-165) depend only on the hit,
// so the unwind only mixes, scales and clamps.  The bounce loop is not
// unrolled (it would copy the shadow loop per bounce); the 12-byte records
// live in L1-resident local memory.
template <int BMAX, class Geo>
__device__ float3 trace(const Geo &geo, float3 origin, float3 dir, const SceneArgs<float> &sa, int samples,
                        int bounces) {
    int ridx[BMAX + 1];
    float rlum[BMAX + 1], rspec[BMAX + 1];
    int m = 0;
    bool exhausted = false;
    float3 tail = f3(0.f, 0.f, 0.f);
    float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
#pragma unroll 1
    for (int k = 0; k <= BMAX; k++) {
        if (k > bounces) break;
        Hit h = geo.closest(origin, dir);
        if (h.idx < 0) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            break;
        }
        float3 hit = origin + dir * h.t;
        float3 normal = h.g.w >= 0.f ? normalize3(hit - f3(h.g.x, h.g.y, h.g.z)) : f3(0.f, 1.f, 0.f);
        float3 l = normalize3(lp - hit);
        float sc = shadow_coeff(geo, hit, normal, sa, samples);
        // shading.py:53-73, 159-162 (view = -dir)
        float dfs = fmaxf(dot3(normal, l), 0.f);
        float3 hv = l - dir;
        float hm2 = dot3(hv, hv);
        float s = 0.f;
        if (hm2 > 0.f) {
            float dd = fmaxf(dot3(normal, hv) * rsqrtf(hm2), 0.f);
            s = powf(dd, __ldg(sa.mat + 8 * h.idx + 4));
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
        origin = hit + normal * 1e-3f;
        dir = dir - normal * (2.f * dot3(normal, dir));
    }
    float3 col = tail;
#pragma unroll 1
    for (int k = m - 1; k >= 0; k--) {
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
__device__ __forceinline__ void shade_pixel(const Geo &geo, const FrameArgs &fa, const SceneArgs<float> &sa, int x,
                                            int ly) {
    if (x >= fa.width || ly >= fa.local_rows) return;
    int y = map_row(ly, fa);
    if (y >= fa.height) return;
    float3 dir = primary_direction(x, y, fa);
    float3 c = trace<BMAX>(geo, f3((float)fa.cam[0], (float)fa.cam[1], (float)fa.cam[2]), dir, sa, fa.samples,
                           fa.bounces);
    fa.out[(int64_t)y * fa.out_pitch + x] = pack_color(c.x, c.y, c.z);
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
__device__ __forceinline__ void render_patches(const Geo &geo, const FrameArgs &fa, const SceneArgs<float> &sa) {
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
        shade_pixel<BMAX>(geo, fa, sa, pcol * 8 + (lane & 7), prow * 4 + (lane >> 3));
        __syncwarp();
    }
    if (fa.peer_out) __threadfence_system();  // frame stores over NVLink land before the kernel retires
}

template <int BMAX, int MAXS>
__global__ void __launch_bounds__(kThreads, RT_F32_MIN_BLOCKS)
    render_f32_param_kernel(const FrameArgs fa, const SceneArgs<float> sa, const ParamScene<MAXS> ps) {
    render_patches<BMAX>(ps, fa, sa);
}

template <int BMAX, bool SMEM>
__global__ void __launch_bounds__(kThreads) render_f32_kernel(const FrameArgs fa, const SceneArgs<float> sa) {
    extern __shared__ float4 smem_geo[];
    MemScene geo{reinterpret_cast<const float4 *>(sa.geo), sa.n};
    if constexpr (SMEM) {
        for (int i = threadIdx.x; i < sa.n; i += blockDim.x) smem_geo[i] = geo.geo[i];
        __syncthreads();
        geo.geo = smem_geo;
    }
    render_patches<BMAX>(geo, fa, sa);
}

template <int BMAX, int MAXS>
__global__ void __launch_bounds__(kThreads)
    trace_f32_param_kernel(const double *orig, const double *dirs, int64_t n_rays, float *out,
                           const SceneArgs<float> sa, int samples, int bounces, const ParamScene<MAXS> ps) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rays) return;
    float3 c = trace<BMAX>(ps, f3((float)orig[3 * i], (float)orig[3 * i + 1], (float)orig[3 * i + 2]),
                           f3((float)dirs[3 * i], (float)dirs[3 * i + 1], (float)dirs[3 * i + 2]), sa, samples,
                           bounces);
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
    float3 c = trace<BMAX>(geo, f3((float)orig[3 * i], (float)orig[3 * i + 1], (float)orig[3 * i + 2]),
                           f3((float)dirs[3 * i], (float)dirs[3 * i + 1], (float)dirs[3 * i + 2]), sa, samples,
                           bounces);
    out[3 * i] = c.x;
    out[3 * i + 1] = c.y;
    out[3 * i + 2] = c.z;
}

// Pack the host scene (float64 geo) into the launch-parameter layout; false
// if it does not fit.
template <int MAXS>
bool pack_params(const SceneArgs<float> &sa, ParamScene<MAXS> &ps) {
    ps.ns = ps.np = 0;
    for (int b = 0; b < sa.n; b++) {
        const double *g = sa.host_geo + 4 * b;
        if (g[3] >= 0.0) {
            if (ps.ns == MAXS) return false;
            ps.sph[ps.ns] = make_float4((float)g[0], (float)g[1], (float)g[2], (float)g[3]);
            ps.sph_idx[ps.ns++] = b;
        } else {
            if (ps.np == kMaxPlanes) return false;
            ps.pl_h[ps.np] = (float)g[1];
            ps.pl_idx[ps.np++] = b;
        }
    }
    for (int b = ps.ns; b < MAXS; b++) {
        ps.sph[b] = make_float4(0.f, 0.f, 0.f, 0.f);
        ps.sph_idx[b] = 0;
    }
    for (int j = ps.np; j < kMaxPlanes; j++) {
        ps.pl_h[j] = 0.f;
        ps.pl_idx[j] = 0;
    }
    return true;
}

// Persistent grid: as many CTAs as fit on the device at once.
template <typename K>
int resident_ctas(K kernel, size_t smem) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
    return sms * (per_sm > 0 ? per_sm : 1);
}

template <int BMAX>
cudaError_t launch_render(const FrameArgs &fa, const SceneArgs<float> &sa, cudaStream_t st) {
    {
        ParamScene<8> ps;
        if (pack_params(sa, ps)) {
            static thread_local int ctas = 0;
            if (!ctas) ctas = resident_ctas(render_f32_param_kernel<BMAX, 8>, 0);
            render_f32_param_kernel<BMAX, 8><<<ctas, kThreads, 0, st>>>(fa, sa, ps);
            return cudaGetLastError();
        }
    }
    {
        thread_local ParamScene<kParamSpheres> ps;  // 5 KB: keep it off the stack
        if (pack_params(sa, ps)) {
            static thread_local int ctas = 0;
            if (!ctas) ctas = resident_ctas(render_f32_param_kernel<BMAX, kParamSpheres>, 0);
            render_f32_param_kernel<BMAX, kParamSpheres><<<ctas, kThreads, 0, st>>>(fa, sa, ps);
            return cudaGetLastError();
        }
    }
    size_t geo_bytes = sizeof(float4) * (size_t)sa.n;
    if (geo_bytes <= (size_t)kSmemGeoBytes) {
        int ctas = resident_ctas(render_f32_kernel<BMAX, true>, geo_bytes);
        render_f32_kernel<BMAX, true><<<ctas, kThreads, geo_bytes, st>>>(fa, sa);
    } else {
        static thread_local int ctas = 0;
        if (!ctas) ctas = resident_ctas(render_f32_kernel<BMAX, false>, 0);
        render_f32_kernel<BMAX, false><<<ctas, kThreads, 0, st>>>(fa, sa);
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

cudaError_t rt_launch_render_f32(const rt::FrameArgs &fa, const rt::SceneArgs<float> &sa, cudaStream_t st) {
    return launch_render<rt::kMaxBounce>(fa, sa, st);
}

cudaError_t rt_launch_trace_f32(const double *o, const double *d, int64_t n, float *out,
                                const rt::SceneArgs<float> &sa, int samples, int bounces, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    return launch_trace<rt::kMaxBounce>(o, d, n, out, sa, samples, bounces, st);
}
