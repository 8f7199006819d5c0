// FP32 frame render — the product path on the B200 CUDA cores.
//
// One thread per pixel, a warp per 8x4 pixel patch, the scene's geometry
// staged in shared memory so each warp-uniform body loop is a broadcast.
// Same control flow as the reference (/root/reference/pkg/src/raytracer/
// renderer.py:108-279): closest hit, sunflower soft-shadow coefficient,
// bounded reflections with a register-resident record stack, skybox on miss,
// Blinn-Phong unwind, pack to 0xAARRGGBB.
//
// FP32-specific numerics (the reasons are measured in SURVEY.md §8c):
//  - the sphere test forms the squared ray-to-centre distance as
//    |L - tca*d|^2 instead of L.L - tca^2 (geometry.py:96): algebraically
//    identical, free of the cancellation that makes FP32 misjudge long shadow
//    rays from far plane points and rays near silhouettes;
//  - primary directions are formed in float64 (camera.py:70-77) and rounded;
//  - the disc-sample table is built in float64 on the host and rounded.
#include "rt_device.cuh"

namespace {
using namespace rt;

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

// geometry.py:83-105 with the cancellation-free perpendicular distance.
__device__ __forceinline__ float ray_sphere(float3 o, float3 d, float4 g) {
    float3 L = f3(g.x - o.x, g.y - o.y, g.z - o.z);
    float tca = dot3(L, d);
    if (tca < 0.f) return INFINITY;
    float3 p = L - d * tca;
    float rad = g.w - dot3(p, p);
    if (rad < -1e-7f) return INFINITY;
    rad = fmaxf(rad, 0.f);
    float t = tca - sqrtf(rad);
    if (t < 0.f) return INFINITY;
    return t;
}

// geometry.py:108-117
__device__ __forceinline__ float ray_plane(float3 o, float3 d, float h) {
    if (d.y == 0.f) return INFINITY;
    float t = (h - o.y) / d.y;
    if (t <= 0.f) return INFINITY;
    return t;
}

__device__ __forceinline__ float intersect(float3 o, float3 d, float4 g) {
    return g.w >= 0.f ? ray_sphere(o, d, g) : ray_plane(o, d, g.y);
}

// renderer.py:82-105; occluded_packed (geometry.py:204-210) is an any-hit
// loop whose result does not depend on body order.
__device__ float shadow_coeff(float3 surface, float3 normal, const float4 *__restrict__ geo,
                              const SceneArgs<float> &sa, int n) {
    float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
    float3 origin = surface + normal * 1e-3f;
    float3 bu = f3(1.f, 0.f, 0.f), bv = f3(0.f, 0.f, 1.f);
    if (n > 1) {  // shading.py:76-86
        float3 axis = normalize3(surface - lp);
        float3 c = cross3(axis, f3(0.f, 1.f, 0.f));
        float m2 = dot3(c, c);
        if (m2 >= 1e-18f) bu = c * rsqrtf(m2);
        bv = cross3(axis, bu);
    }
    const float2 *__restrict__ tab = reinterpret_cast<const float2 *>(sa.table);
    int unblocked = 0;
    for (int i = 0; i < n; i++) {
        float3 s = lp;
        if (n > 1) {
            float2 ab = __ldg(tab + i);
            s = lp + bu * ab.x + bv * ab.y;
        }
        float3 dir = normalize3(s - origin);
        float3 e = surface - s;
        float limit = sqrtf(dot3(e, e));
        bool blocked = false;
        for (int b = 0; b < sa.n; b++) {
            if (intersect(origin, dir, geo[b]) < limit) {
                blocked = true;
                break;
            }
        }
        unblocked += blocked ? 0 : 1;
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

// renderer.py:108-224 with records (body, lum, spec) — see render_f64.cu.
template <int BMAX>
__device__ float3 trace(float3 origin, float3 dir, const float4 *__restrict__ geo, const SceneArgs<float> &sa,
                        int samples, int bounces) {
    int ridx[BMAX + 1];
    float rlum[BMAX + 1], rspec[BMAX + 1];
    int m = 0;
    bool exhausted = false;
    float3 tail = f3(0.f, 0.f, 0.f);
    float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
#pragma unroll(BMAX <= 8 ? BMAX + 1 : 1)
    for (int k = 0; k <= BMAX; k++) {
        if (k > bounces) break;
        float best_t = INFINITY;
        int idx = -1;
        for (int b = 0; b < sa.n; b++) {
            float t = intersect(origin, dir, geo[b]);
            if (t < best_t) {
                best_t = t;
                idx = b;
            }
        }
        if (idx < 0) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            break;
        }
        float4 g = geo[idx];
        float3 hit = origin + dir * best_t;
        float3 normal = g.w >= 0.f ? normalize3(hit - f3(g.x, g.y, g.z)) : f3(0.f, 1.f, 0.f);
        float3 l = normalize3(lp - hit);
        float sc = shadow_coeff(hit, normal, geo, sa, samples);
        // shading.py:53-73, 159-162 (view = -dir)
        float dfs = fmaxf(dot3(normal, l), 0.f);
        float3 h = l - dir;
        float hm2 = dot3(h, h);
        float s = 0.f;
        if (hm2 > 0.f) {
            float dd = fmaxf(dot3(normal, h) * rsqrtf(hm2), 0.f);
            s = powf(dd, __ldg(sa.mat + 8 * idx + 4));
        }
        float lum = fminf(sa.ambient + sc * dfs * (1.f - sa.ambient), 1.f);
        ridx[k] = idx;
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
#pragma unroll(BMAX <= 8 ? BMAX + 1 : 1)
    for (int k = BMAX; k >= 0; k--) {
        if (k >= m) continue;
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

template <bool SMEM>
__device__ __forceinline__ const float4 *stage_geo(const SceneArgs<float> &sa, float4 *smem) {
    const float4 *g = reinterpret_cast<const float4 *>(sa.geo);
    if constexpr (!SMEM) return g;
    else {
    for (int i = threadIdx.x; i < sa.n; i += blockDim.x) smem[i] = g[i];
    __syncthreads();
    return smem;
    }
}

template <int BMAX, bool SMEM>
__global__ void __launch_bounds__(kThreads) render_f32_kernel(const FrameArgs fa, const SceneArgs<float> sa) {
    extern __shared__ float4 smem_geo[];
    const float4 *__restrict__ geo = stage_geo<SMEM>(sa, smem_geo);
    int x, ly;
    thread_pixel(x, ly);
    if (x >= fa.width || ly >= fa.local_rows) return;
    int y = map_row(ly, fa);
    if (y >= fa.height) return;
    float3 dir = primary_direction(x, y, fa);
    float3 c = trace<BMAX>(f3((float)fa.cam[0], (float)fa.cam[1], (float)fa.cam[2]), dir, geo, sa, fa.samples,
                           fa.bounces);
    fa.out[(int64_t)y * fa.out_pitch + x] = pack_color(c.x, c.y, c.z);
    if (fa.radiance) {
        float *r = (float *)fa.radiance + 3 * ((int64_t)y * fa.width + x);
        r[0] = c.x;
        r[1] = c.y;
        r[2] = c.z;
    }
    if (fa.peer_out) __threadfence_system();  // frame stores over NVLink land before the kernel retires
}

template <int BMAX, bool SMEM>
__global__ void __launch_bounds__(kThreads)
    trace_f32_kernel(const double *orig, const double *dirs, int64_t n_rays, float *out, const SceneArgs<float> sa,
                     int samples, int bounces) {
    extern __shared__ float4 smem_geo[];
    const float4 *__restrict__ geo = stage_geo<SMEM>(sa, smem_geo);
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rays) return;
    float3 c = trace<BMAX>(f3((float)orig[3 * i], (float)orig[3 * i + 1], (float)orig[3 * i + 2]),
                           f3((float)dirs[3 * i], (float)dirs[3 * i + 1], (float)dirs[3 * i + 2]), geo, sa, samples,
                           bounces);
    out[3 * i] = c.x;
    out[3 * i + 1] = c.y;
    out[3 * i + 2] = c.z;
}

template <int BMAX>
cudaError_t launch_render(const FrameArgs &fa, const SceneArgs<float> &sa, cudaStream_t st) {
    dim3 grid((fa.width + kTileW - 1) / kTileW, (fa.local_rows + kTileH - 1) / kTileH);
    size_t geo_bytes = sizeof(float4) * (size_t)sa.n;
    if (geo_bytes <= (size_t)kSmemGeoBytes)
        render_f32_kernel<BMAX, true><<<grid, kThreads, geo_bytes, st>>>(fa, sa);
    else
        render_f32_kernel<BMAX, false><<<grid, kThreads, 0, st>>>(fa, sa);
    return cudaGetLastError();
}

template <int BMAX>
cudaError_t launch_trace(const double *o, const double *d, int64_t n, float *out, const SceneArgs<float> &sa,
                         int samples, int bounces, cudaStream_t st) {
    unsigned blocks = (unsigned)((n + kThreads - 1) / kThreads);
    size_t geo_bytes = sizeof(float4) * (size_t)sa.n;
    if (geo_bytes <= (size_t)kSmemGeoBytes)
        trace_f32_kernel<BMAX, true><<<blocks, kThreads, geo_bytes, st>>>(o, d, n, out, sa, samples, bounces);
    else
        trace_f32_kernel<BMAX, false><<<blocks, kThreads, 0, st>>>(o, d, n, out, sa, samples, bounces);
    return cudaGetLastError();
}

}  // namespace

cudaError_t rt_launch_render_f32(const rt::FrameArgs &fa, const rt::SceneArgs<float> &sa, cudaStream_t st) {
    if (fa.bounces <= 1) return launch_render<1>(fa, sa, st);
    if (fa.bounces <= 3) return launch_render<3>(fa, sa, st);
    if (fa.bounces <= 8) return launch_render<8>(fa, sa, st);
    return launch_render<rt::kMaxBounce>(fa, sa, st);
}

cudaError_t rt_launch_trace_f32(const double *o, const double *d, int64_t n, float *out,
                                const rt::SceneArgs<float> &sa, int samples, int bounces, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (bounces <= 3) return launch_trace<3>(o, d, n, out, sa, samples, bounces, st);
    return launch_trace<rt::kMaxBounce>(o, d, n, out, sa, samples, bounces, st);
}
