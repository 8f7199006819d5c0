// Float64 device math in the reference's literal operation order, shared by
// the FP64 validation megakernel (render_f64.cu) and the FP64 culled
// wavefront (render_fused_f64.cu).  Both translation units are compiled with
// -fmad=false: numba compiles the reference without FMA contraction.
#pragma once
#include "rt_device.cuh"
#include "rt_pow.cuh"

namespace rt64 {
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

__device__ __forceinline__ double clamp01(double x) {  // min(max(x, 0.0), 1.0)
    double m = (0.0 > x) ? 0.0 : x;
    return (1.0 < m) ? 1.0 : m;
}

// renderer.py:60-74
static __device__ d3 sky_sample(d3 d, const float4 *__restrict__ sky, int W, int H) {
    double u = 0.5 + atan2(d.x, d.z) / (2.0 * 3.141592653589793);
    double dy = d.y < -1.0 ? -1.0 : d.y;
    dy = dy > 1.0 ? 1.0 : dy;
    double v = 0.5 - asin(dy) / 3.141592653589793;
    long long tx = (long long)floor(u * (double)W);
    // ((tx % W) + W) % W for the only reachable tx, -1..W (u is within
    // rounding of [0, 1]): no 64-bit integer divisions
    tx = tx < 0 ? tx + W : (tx >= W ? tx - W : tx);
    long long ty = (long long)floor(v * (double)H);
    if (ty < 0)
        ty = 0;
    else if (ty > H - 1)
        ty = H - 1;
    float4 t = __ldg(sky + ty * (long long)W + tx);  // texels pre-clamped on upload
    return mk((double)t.x, (double)t.y, (double)t.z);
}

// shading.py:76-86 — the disc basis for a surface point
__device__ __forceinline__ void disc_basis(d3 surface, d3 lp, d3 &bu, d3 &bv) {
    d3 axis = vnormalize(vsub(surface, lp));
    d3 c = vcross(axis, mk(0.0, 1.0, 0.0));
    double m = vmag(c);
    if (m < 1e-9)
        bu = mk(1.0, 0.0, 0.0);
    else
        bu = mk(c.x / m, c.y / m, c.z / m);
    bv = vcross(axis, bu);
}

// shading.py:53-73 — Lambert and Blinn factors of a hit (view = -dir)
__device__ __forceinline__ void hit_terms(d3 normal, d3 l, d3 dir, double refl, double &dfs, double &s) {
    d3 view = mk(-dir.x, -dir.y, -dir.z);
    dfs = vdot(normal, l);
    dfs = dfs > 0.0 ? dfs : 0.0;
    double hx = l.x + view.x, hy = l.y + view.y, hz = l.z + view.z;
    double hm = sqrt(hx * hx + hy * hy + hz * hz);
    if (hm == 0.0) {
        s = 0.0;
    } else {
        double dd = (normal.x * hx + normal.y * hy + normal.z * hz) / hm;
        if (dd < 0.0) dd = 0.0;
        s = rtpow::pow_cr(dd, refl);  // shading.py:73 `d**reflectivity`, rounded like libm (rt_pow.cuh)
    }
}

// geometry.py:191-201 closest hit over geo[n][4], strict '<' (lowest index wins ties)
__device__ __forceinline__ int closest(d3 o, d3 d, const double *__restrict__ geo, int n, double &best_t) {
    best_t = INFINITY;
    int idx = -1;
    for (int b = 0; b < n; b++) {
        double t = intersect(o, d, geo + 4 * b);
        if (t < best_t) {
            best_t = t;
            idx = b;
        }
    }
    return idx;
}

// renderer.py:185-224 over records (body, Lambert, Blinn, coefficient):
// shade_color (shading.py:144-168) in the reference's order
template <class Get>
__device__ __forceinline__ d3 unwind(int m, bool exhausted, d3 tail, const SceneArgs<double> &sa, Get get) {
    d3 col = tail;
    for (int k = m - 1; k >= 0; k--) {
        int idx;
        double dfs, s, sc;
        get(k, idx, dfs, s, sc);
        double lum = sa.ambient + sc * dfs * (1.0 - sa.ambient);
        if (lum > 1.0) lum = 1.0;
        double sp = sc * s;
        const double *mt = sa.mat + 8 * idx;
        double br = __ldg(mt), bg = __ldg(mt + 1), bb = __ldg(mt + 2);
        if (!(exhausted && k == m - 1)) {
            double rr = __ldg(mt + 3);
            br = br * (1.0 - rr) + col.x * rr;
            bg = bg * (1.0 - rr) + col.y * rr;
            bb = bb * (1.0 - rr) + col.z * rr;
        }
        col = mk(clamp01(br * lum + sa.lc[0] * sp), clamp01(bg * lum + sa.lc[1] * sp),
                 clamp01(bb * lum + sa.lc[2] * sp));
    }
    return col;
}

}  // namespace rt64
