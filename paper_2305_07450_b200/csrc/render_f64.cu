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
#include "rt_f64.cuh"

namespace {
using namespace rt;
using namespace rt64;

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
            s = rtpow::pow_cr(dd, __ldg(sa.mat + 8 * idx + 4));  // rounded like libm (rt_pow.cuh)
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
    thread_pixel_bottom_first(x, ly);
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
