// FP64 validation render: the reference's float64 arithmetic in its literal
// operation order, one thread per pixel.  Compiled with -fmad=false so no
// a*b+c is fused (numba compiles the reference without fast-math, hence
// without FMA contraction); double sqrt and division are IEEE round-to-nearest
// on the device, cos/sin/tan only ever run on the host (camera constants and
// the disc table) with the reference's libm.  Frames reproduce the golden
// sha256 of pkg/tests/test_acceptance.py:31.
//
// Every function cites the reference line it restates
// (/root/reference/pkg/src/raytracer/...).
#include "rt_device.cuh"

namespace {
using namespace rt;

struct d3 {
    double x, y, z;
};
__device__ __forceinline__ d3 mk(double x, double y, double z) { return d3{x, y, z}; }
__device__ __forceinline__ d3 vsub(d3 a, d3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }  // vecmath.py:33
__device__ __forceinline__ double vdot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }  // vecmath.py:49
__device__ __forceinline__ d3 vcross(d3 a, d3 b) {  // vecmath.py:54-60
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double vmag(d3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }  // vecmath.py:63
__device__ __forceinline__ d3 vnormalize(d3 a) {  // vecmath.py:68-78 (zero-safe)
    double m = vmag(a);
    if (m == 0.0) return mk(0.0, 0.0, 0.0);
    return mk(a.x / m, a.y / m, a.z / m);
}
__device__ __forceinline__ double vdistance(d3 a, d3 b) {  // vecmath.py:81-86
    double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
    return sqrt(dx * dx + dy * dy + dz * dz);
}
__device__ __forceinline__ d3 vreflect(d3 i, d3 n) {  // vecmath.py:89-96
    double k = 2.0 * (n.x * i.x + n.y * i.y + n.z * i.z);
    return mk(i.x - k * n.x, i.y - k * n.y, i.z - k * n.z);
}

// camera.py:46-54 + 70-77, vecmath.py:99-110
__device__ __forceinline__ d3 primary_direction(int xi, int yi, const FrameArgs &fa) {
    double x = (double)xi, y = (double)yi, w = (double)fa.width, h = (double)fa.height;
    double u, v;
    if (w > h) {
        u = (x - w / 2 + h / 2) / h * 2 - 1;
        v = -(y / h * 2 - 1);
    } else {
        u = x / w * 2 - 1;
        v = -((y - h / 2 + w / 2) / w * 2 - 1);
    }
    d3 d = vnormalize(mk(u, v, fa.vdist));
    double y2 = d.y * fa.cb - d.z * fa.sb;
    double z2 = d.y * fa.sb + d.z * fa.cb;
    double x2 = d.x * fa.ca + z2 * fa.sa;
    double z3 = -d.x * fa.sa + z2 * fa.ca;
    return mk(x2, y2, z3);
}

// geometry.py:83-105 — literal d2 = L.L - tca^2 (the golden hash encodes it)
__device__ __forceinline__ double ray_sphere(d3 o, d3 d, const double *g) {
    double lx = g[0] - o.x, ly = g[1] - o.y, lz = g[2] - o.z;
    double tca = lx * d.x + ly * d.y + lz * d.z;
    if (tca < 0.0) return INFINITY;
    double d2 = lx * lx + ly * ly + lz * lz - tca * tca;
    double rad = g[3] - d2;  // g[3] = radius * radius, formed on the host in float64
    if (rad < -1e-7) return INFINITY;
    if (rad < 0.0) rad = 0.0;
    double t = tca - sqrt(rad);
    if (t < 0.0) return INFINITY;
    return t;
}

// geometry.py:108-117
__device__ __forceinline__ double ray_plane(d3 o, d3 d, double h) {
    double dy = d.y;
    if (dy == 0.0) return INFINITY;
    double t = (h - o.y) / dy;
    if (t <= 0.0) return INFINITY;
    return t;
}

// geometry.py:179-188
__device__ __forceinline__ double intersect(d3 o, d3 d, const double *g) {
    if (g[3] >= 0.0) return ray_sphere(o, d, g);
    return ray_plane(o, d, g[1]);
}

// shading.py:89-100 with the (r cos, r sin) pair from the host table
__device__ __forceinline__ d3 disc_point(int i, d3 c, d3 u, d3 v, const double *table) {
    double a = table[2 * i];
    double b = table[2 * i + 1];
    return mk(c.x + a * u.x + b * v.x, c.y + a * u.y + b * v.y, c.z + a * u.z + b * v.z);
}

// renderer.py:82-105 (+ shading.py:76-86 disc_basis, geometry.py:204-210)
__device__ double shadow_coeff(d3 surface, d3 normal, const double *__restrict__ geo, const SceneArgs<double> &sa,
                               int n) {
    d3 lp = mk(sa.light[0], sa.light[1], sa.light[2]);
    d3 origin = mk(surface.x + 1e-3 * normal.x, surface.y + 1e-3 * normal.y, surface.z + 1e-3 * normal.z);
    d3 bu, bv;
    if (n > 1) {
        d3 axis = vnormalize(vsub(surface, lp));
        d3 c = vcross(axis, mk(0.0, 1.0, 0.0));
        double m = vmag(c);
        if (m < 1e-9)
            bu = mk(1.0, 0.0, 0.0);
        else
            bu = mk(c.x / m, c.y / m, c.z / m);
        bv = vcross(axis, bu);
    } else {
        bu = mk(1.0, 0.0, 0.0);
        bv = mk(0.0, 0.0, 1.0);
    }
    int unblocked = 0;
    for (int i = 0; i < n; i++) {
        d3 s = (n == 1) ? lp : disc_point(i, lp, bu, bv, sa.table);
        d3 dir = vnormalize(vsub(s, origin));
        double limit = vdistance(surface, s);
        bool blocked = false;
        for (int b = 0; b < sa.n; b++) {
            if (intersect(origin, dir, geo + 4 * b) < limit) {
                blocked = true;
                break;
            }
        }
        if (!blocked) unblocked += 1;
    }
    return (double)unblocked / (double)n;
}

__device__ __forceinline__ double clamp01(double x) {  // min(max(x, 0.0), 1.0)
    double m = (0.0 > x) ? 0.0 : x;
    return (1.0 < m) ? 1.0 : m;
}

// renderer.py:60-74
__device__ d3 sky_sample(d3 d, const float4 *__restrict__ sky, int W, int H) {
    double u = 0.5 + atan2(d.x, d.z) / (2.0 * 3.141592653589793);
    double dy = d.y < -1.0 ? -1.0 : d.y;
    dy = dy > 1.0 ? 1.0 : dy;
    double v = 0.5 - asin(dy) / 3.141592653589793;
    long long tx = (long long)floor(u * (double)W);
    tx = ((tx % W) + W) % W;
    long long ty = (long long)floor(v * (double)H);
    if (ty < 0)
        ty = 0;
    else if (ty > H - 1)
        ty = H - 1;
    float4 t = __ldg(sky + ty * (long long)W + tx);  // texels pre-clamped on upload
    return mk((double)t.x, (double)t.y, (double)t.z);
}

// renderer.py:108-224.  A record keeps (body, lum, spec): shade_color's
// luminance and specular terms (shading.py:159-165) depend only on the hit,
// not on the colour folded in, so they are formed in the forward pass with
// the same operations and the unwind only mixes, scales and clamps.
template <int BMAX>
__device__ d3 trace(d3 origin, d3 dir, const double *__restrict__ geo, const SceneArgs<double> &sa, int samples,
                    int bounces) {
    int ridx[BMAX + 1];
    double rlum[BMAX + 1], rspec[BMAX + 1];
    int m = 0;
    bool exhausted = false;
    d3 tail = mk(0.0, 0.0, 0.0);
    d3 lp = mk(sa.light[0], sa.light[1], sa.light[2]);
#pragma unroll(BMAX <= 8 ? BMAX + 1 : 1)
    for (int k = 0; k <= BMAX; k++) {
        if (k > bounces) break;
        // geometry.py:191-201 closest hit, strict '<' (lowest index wins ties)
        double best_t = INFINITY;
        int idx = -1;
        for (int b = 0; b < sa.n; b++) {
            double t = intersect(origin, dir, geo + 4 * b);
            if (t < best_t) {
                best_t = t;
                idx = b;
            }
        }
        if (idx < 0) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            break;
        }
        const double *g = geo + 4 * idx;
        d3 hit = mk(origin.x + dir.x * best_t, origin.y + dir.y * best_t, origin.z + dir.z * best_t);
        d3 normal = (g[3] >= 0.0) ? vnormalize(vsub(hit, mk(g[0], g[1], g[2]))) : mk(0.0, 1.0, 0.0);
        d3 view = mk(-dir.x, -dir.y, -dir.z);
        d3 l = vnormalize(vsub(lp, hit));
        double sc = shadow_coeff(hit, normal, geo, sa, samples);
        // shading.py:53-73, 159-162
        double dfs = vdot(normal, l);
        dfs = dfs > 0.0 ? dfs : 0.0;
        double hx = l.x + view.x, hy = l.y + view.y, hz = l.z + view.z;
        double hm = sqrt(hx * hx + hy * hy + hz * hz);
        double s;
        if (hm == 0.0) {
            s = 0.0;
        } else {
            double dd = (normal.x * hx + normal.y * hy + normal.z * hz) / hm;
            if (dd < 0.0) dd = 0.0;
            s = pow(dd, __ldg(sa.mat + 8 * idx + 4));
        }
        double lum = sa.ambient + sc * dfs * (1.0 - sa.ambient);
        if (lum > 1.0) lum = 1.0;
        ridx[k] = idx;
        rlum[k] = lum;
        rspec[k] = sc * s;
        m = k + 1;
        if (k == bounces) {
            exhausted = true;
            break;
        }
        origin = mk(hit.x + 1e-3 * normal.x, hit.y + 1e-3 * normal.y, hit.z + 1e-3 * normal.z);
        dir = vreflect(dir, normal);
    }
    if (m == 0) return tail;
    // Unwind (renderer.py:185-224), indices kept compile-time so the records
    // stay in registers: a depth-cut chain shades its last base colour as-is,
    // every other record mixes base*(1-rr) + col*rr first.
    d3 col = tail;
#pragma unroll(BMAX <= 8 ? BMAX + 1 : 1)
    for (int k = BMAX; k >= 0; k--) {
        if (k >= m) continue;
        const double *mt = sa.mat + 8 * ridx[k];
        double br = __ldg(mt), bg = __ldg(mt + 1), bb = __ldg(mt + 2);
        if (!(exhausted && k == m - 1)) {
            double rr = __ldg(mt + 3);
            br = br * (1.0 - rr) + col.x * rr;
            bg = bg * (1.0 - rr) + col.y * rr;
            bb = bb * (1.0 - rr) + col.z * rr;
        }
        double lum = rlum[k], sp = rspec[k];
        col = mk(clamp01(br * lum + sa.lc[0] * sp), clamp01(bg * lum + sa.lc[1] * sp),
                 clamp01(bb * lum + sa.lc[2] * sp));
    }
    return col;
}

template <bool SMEM>
__device__ __forceinline__ const double *stage_geo(const SceneArgs<double> &sa, double *smem) {
    if constexpr (!SMEM) return sa.geo;
    else {
    for (int i = threadIdx.x; i < 4 * sa.n; i += blockDim.x) smem[i] = sa.geo[i];
    __syncthreads();
    return smem;
    }
}

template <int BMAX, bool SMEM>
__global__ void __launch_bounds__(kThreads) render_f64_kernel(const FrameArgs fa, const SceneArgs<double> sa) {
    extern __shared__ double smem_geo[];
    const double *__restrict__ geo = stage_geo<SMEM>(sa, smem_geo);
    int x, ly;
    thread_pixel(x, ly);
    if (x >= fa.width || ly >= fa.local_rows) return;
    int y = map_row(ly, fa);
    if (y >= fa.row_end) return;
    d3 dir = primary_direction(x, y, fa);
    d3 c = trace<BMAX>(mk(fa.cam[0], fa.cam[1], fa.cam[2]), dir, geo, sa, fa.samples, fa.bounces);
    fa.out[(int64_t)y * fa.out_pitch + x] = pack_color(c.x, c.y, c.z, fa.rgba);
    if (fa.radiance) {
        double *r = (double *)fa.radiance + 3 * ((int64_t)y * fa.width + x);
        r[0] = c.x;
        r[1] = c.y;
        r[2] = c.z;
    }
    if (fa.peer_out) __threadfence_system();  // frame stores over NVLink land before the kernel retires
}

template <int BMAX, bool SMEM>
__global__ void __launch_bounds__(kThreads)
    trace_f64_kernel(const double *orig, const double *dirs, int64_t n_rays, double *out, const SceneArgs<double> sa,
                     int samples, int bounces) {
    extern __shared__ double smem_geo[];
    const double *__restrict__ geo = stage_geo<SMEM>(sa, smem_geo);
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rays) return;
    d3 c = trace<BMAX>(mk(orig[3 * i], orig[3 * i + 1], orig[3 * i + 2]),
                       mk(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]), geo, sa, samples, bounces);
    out[3 * i] = c.x;
    out[3 * i + 1] = c.y;
    out[3 * i + 2] = c.z;
}

__global__ void sky_f64_kernel(const double *dirs, int64_t n, double *out, const float4 *sky, int w, int h) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    d3 c = sky_sample(mk(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]), sky, w, h);
    out[3 * i] = c.x;
    out[3 * i + 1] = c.y;
    out[3 * i + 2] = c.z;
}

template <int BMAX>
cudaError_t launch_render(const FrameArgs &fa, const SceneArgs<double> &sa, cudaStream_t st) {
    dim3 grid((fa.width + kTileW - 1) / kTileW, (fa.local_rows + kTileH - 1) / kTileH);
    size_t geo_bytes = sizeof(double) * 4 * (size_t)sa.n;
    if (geo_bytes <= (size_t)kSmemGeoBytes)
        render_f64_kernel<BMAX, true><<<grid, kThreads, geo_bytes, st>>>(fa, sa);
    else
        render_f64_kernel<BMAX, false><<<grid, kThreads, 0, st>>>(fa, sa);
    return cudaGetLastError();
}

template <int BMAX>
cudaError_t launch_trace(const double *o, const double *d, int64_t n, double *out, const SceneArgs<double> &sa,
                         int samples, int bounces, cudaStream_t st) {
    unsigned blocks = (unsigned)((n + kThreads - 1) / kThreads);
    size_t geo_bytes = sizeof(double) * 4 * (size_t)sa.n;
    if (geo_bytes <= (size_t)kSmemGeoBytes)
        trace_f64_kernel<BMAX, true><<<blocks, kThreads, geo_bytes, st>>>(o, d, n, out, sa, samples, bounces);
    else
        trace_f64_kernel<BMAX, false><<<blocks, kThreads, 0, st>>>(o, d, n, out, sa, samples, bounces);
    return cudaGetLastError();
}

}  // namespace

cudaError_t rt_launch_render_f64(const rt::FrameArgs &fa, const rt::SceneArgs<double> &sa, cudaStream_t st) {
    if (fa.bounces <= 1) return launch_render<1>(fa, sa, st);
    if (fa.bounces <= 3) return launch_render<3>(fa, sa, st);
    if (fa.bounces <= 8) return launch_render<8>(fa, sa, st);
    return launch_render<rt::kMaxBounce>(fa, sa, st);
}

cudaError_t rt_launch_trace_f64(const double *o, const double *d, int64_t n, double *out,
                                const rt::SceneArgs<double> &sa, int samples, int bounces, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (bounces <= 3) return launch_trace<3>(o, d, n, out, sa, samples, bounces, st);
    return launch_trace<rt::kMaxBounce>(o, d, n, out, sa, samples, bounces, st);
}

cudaError_t rt_launch_sky_f64(const double *d, int64_t n, double *out, const float4 *sky, int w, int h,
                              cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    sky_f64_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(d, n, out, sky, w, h);
    return cudaGetLastError();
}
