// Shared device code of the wavefront kernels (render_wave_f32.cu, the
// unculled trace / shadow / shade path, and render_fused_f32.cu, the culled
// path): warp helpers, the warp ray-bundle bound used for closest hits in
// many-sphere scenes, the per-hit shadow cone and its exact body classifier,
// and the unwind.
#pragma once
#include "rt_f32.cuh"

namespace rt32 {

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Many-sphere scenes (> 8 spheres): closest hits against a warp-uniform
// candidate list.  Per bounce the warp bounds its live rays — origins within
// rho of their mean Co, directions within theta of their mean A — so every
// point a ray can reach lies in the cone (Co, A, theta) dilated by rho; a
// sphere farther than its (grazing-padded) radius from that set cannot be
// hit by any of the warp's rays and is skipped.  The 32 lanes classify 32
// spheres at a time; the survivors (a uniform bit mask) are tested by every
// lane in lockstep, ties broken by the lowest original index.
template <int MAXS>
__device__ __forceinline__ bool sphere_meets_bundle(float4 g, float3 co, float3 A, float cos_t, float sin_t,
                                                    float rho) {
    float3 u = f3(g.x - co.x, g.y - co.y, g.z - co.z);
    float u2 = dot3(u, u);
    float h = dot3(u, A);
    float3 w = u - A * h;
    float q = sqrtf(dot3(w, w));
    float un = sqrtf(u2);
    float R = (sqrtf(g.w + 1e-7f) + rho) * (1.f + kBoundRel) + kBoundRel * (1.f + un);
    if (h < -R) return false;
    float dist = (h * cos_t + q * sin_t >= 0.f) ? q * cos_t - h * sin_t : un;
    return dist < R;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// --- B': shadow coefficients with exact occluder culling ---------------------
//
// The shadow rays of one hit all leave the same origin o towards points of
// the light disc (centre L, radius r_i <= 2R, shading.py:89-100) and stop at
// limit = |p - s_i| <= |o - s_i| + 1e-3 (renderer.py:100-101).  Every such
// segment lies in the union of balls B(o + t(L - o), 2R t), t in [0, T],
// T = 1 + 1e-3/(H - 2R) — a solid cone with apex o, axis L - o (length H)
// and half-angle phi, sin phi = 2R / H.  A body that stays outside that cone
// (with a relative margin far above FP32 rounding) fails every one of the
// hit's shadow tests, so skipping it leaves the coefficient unchanged; a
// sphere that swallows the cone's whole cross-section between o and the disc
// blocks every sample, so the coefficient is exactly 0.  Only hits with a
// body in the penumbra test rays, and only against those bodies
// (render_fused_f32.cu: the trace kernel classifies, the sample kernel tests
// the undecided hits' rays).
constexpr float kCullRel = 1e-4f;  // relative margin of the cull / full-block decisions
constexpr float kCullAbs = 1e-5f;  // absolute margin (scene units)

struct Cone {
    float3 o, axis;   // apex, unit axis towards L
    float H, rho;     // axis length, base radius (2R with margin)
    float sin_phi, cos_phi, reach;  // reach = T (H + rho): farthest axial extent of a segment
    float inv_H;
    bool ok;          // a proper cone (the light ball does not swallow the origin)
};

__device__ __forceinline__ Cone make_cone(float3 o, float3 lp, float light_radius) {
    Cone c;
    c.o = o;
    float3 A = lp - o;
    c.H = sqrtf(dot3(A, A));
    c.rho = 2.f * light_radius * (1.f + kCullRel) + kCullAbs;
    c.ok = c.H > 0.f && c.rho < 0.999f * c.H;
    c.axis = A * (c.H > 0.f ? 1.f / c.H : 0.f);
    c.inv_H = c.H > 0.f ? 1.f / c.H : 0.f;
    c.sin_phi = c.ok ? c.rho * c.inv_H : 1.f;
    c.cos_phi = sqrtf(fmaxf(1.f - c.sin_phi * c.sin_phi, 0.f));
    float T = 1.f + (1e-3f + kCullAbs) / fmaxf(c.H - c.rho, 1e-6f);
    c.reach = T * (c.H + c.rho) * (1.f + kCullRel) + kCullAbs;
    return c;
}

// 0: the sphere can block none of the hit's shadow rays; 1: some; 2: all.
// rr = {r, sqrt(r^2 + 1e-7)} (formed on the host): one square root per test.
__device__ __forceinline__ int sphere_class(const Cone &k, float4 g, float2 rr) {
    if (!k.ok) return 1;
    float3 u = f3(g.x - k.o.x, g.y - k.o.y, g.z - k.o.z);
    float u2 = dot3(u, u);
    // the origin inside the sphere: t = tca - sqrt(rad) < 0 for every ray (geometry.py:102-103)
    if (u2 < g.w * (1.f - 4.f * kCullRel) - kCullAbs) return 0;
    float h = dot3(u, k.axis);
    float3 w = u - k.axis * h;
    float q = sqrtf(dot3(w, w));
    float un = fabsf(h) + q;  // >= |u|
    // grazing rays (rad >= -1e-7, geometry.py:98) count as hits: pad the radius
    float rp = rr.y * (1.f + kCullRel) + kCullAbs + 1e-6f * (un + k.H);
    if (h < -rp || h - rp > k.reach) return 0;
    if (h * k.cos_phi + q * k.sin_phi >= 0.f) {
        if (q * k.cos_phi - h * k.sin_phi >= rp) return 0;
    } else if (u2 >= rp * rp) {
        return 0;  // nearest point of the cone is its apex
    }
    // full block: origin clearly outside, sphere wholly before the disc, and
    // the cone's cross-section at the centre's depth inside the great circle
    float rm = rr.x * (1.f - 10.f * kCullRel) - kCullAbs - 1e-6f * (un + k.H);
    if (u2 > g.w * (1.f + 4.f * kCullRel) + kCullAbs && h > 0.f &&
        h + rr.x < (k.H - k.rho) * (1.f - kCullRel) - 2e-3f && q + h * k.inv_H * k.rho * (1.f + kCullRel) < rm)
        return 2;
    return 1;
}

// A cluster bound the cone cannot reach: no member can block (the members'
// own tests would all return 0).
__device__ __forceinline__ bool bound_meets_cone(const Cone &k, float4 B) {
    if (!k.ok) return true;
    float3 u = f3(B.x - k.o.x, B.y - k.o.y, B.z - k.o.z);
    float u2 = dot3(u, u);
    float h = dot3(u, k.axis);
    float3 w = u - k.axis * h;
    float q = sqrtf(dot3(w, w));
    float rp = B.w * (1.f + kCullRel) + kCullAbs + 1e-6f * (fabsf(h) + q + k.H);
    if (h < -rp || h - rp > k.reach) return false;
    if (h * k.cos_phi + q * k.sin_phi >= 0.f) return q * k.cos_phi - h * k.sin_phi < rp;
    return u2 < rp * rp;
}

// --- the silhouette form of the soft-shadow sphere test ----------------------
//
// For one hit the shadow rays run from o along w_i = lo + a_i bu + b_i bv
// (lo = L - o, disc basis bu, bv: shading.py:76-100) and a sphere (centre c,
// u = c - o) blocks sample i iff tca > 0, d2 < r^2 + GRAZE and its entry
// distance is below the limit (geometry.py:94-106, renderer.py:100-103).
// With the origin clearly outside the sphere and |u| < |p - L| (checked once
// per hit and sphere), entry <= tca <= |u| < limit for every sample, so
// only tca > 0 and d2 decide, and
//   d2 = |u x w|^2 / |w|^2 = |u|^2 ((e1.w)^2 + (e2.w)^2) / |w|^2,
//   tca > 0  <=>  n.w > 0      (n = u / |u|, e1, e2 orthonormal, perpendicular to n).
// Every dot product is affine in the disc coordinates (a, b) and |w|^2 =
// |lo|^2 + 2a lo.bu + 2b lo.bv + a^2 + b^2, so with s = |u| / sqrt(r^2 + GRAZE)
//   blocked_i  <=>  x_i^2 + y_i^2 < |w_i|^2  and  z_i > 0,
//   x_i = s e1.lo + a_i s e1.bu + b_i s e1.bv   (y likewise with e2),
//   z_i = sign(n.lo) + a_i n.bu / |n.lo| + b_i n.bv / |n.lo|:
// coefficients formed once per (hit, sphere), then a few FMAs per sample
// instead of a normalised ray and a sphere test.  The z test is dropped when
// every sample direction lies within 90 degrees of u (the cone bound below),
// which leaves it to the self-shadowing terminator hits.  The predicate is the
// reference's on the same real numbers; only FP32 rounding near the
// silhouette differs, of the same order as the ray form's (which also forms
// d2 as a squared perpendicular).  Near z = 0 the rounding of z cannot
// matter: there d2 ~ |u|^2 > r^2 + GRAZE, so the sample is open either way.
//
// Returns 0 (a precondition fails: the hit takes the ray form), 1 (no z test
// needed), 2 (z test, z0 = +1) or 3 (z test, z0 = -1); c = {x0, x1, x2, y0},
// {y1, y2, z1, z2}.
// Every sample direction lies within phi of the cone axis, so tca >= h cos(phi)
// - q sin(phi) for u = c - o split into h along the axis and q across it:
// true when that bound is clearly positive (no z test needed).
__device__ __forceinline__ bool conic_front(const Cone &k, float4 g) {
    const float3 u = f3(g.x - k.o.x, g.y - k.o.y, g.z - k.o.z);
    const float h = dot3(u, k.axis);
    const float3 wp = u - k.axis * h;
    const float q = sqrtf(dot3(wp, wp));
    return h * k.cos_phi - q * k.sin_phi > kCullRel * (fabsf(h) + q) + kCullAbs;
}

__device__ __forceinline__ int conic_coeffs(const Cone &k, float4 g, float3 lo, float3 bu, float3 bv, float ls2,
                                            float4 &ca, float4 &cb) {
    if (!k.ok) return 0;
    const float3 u = f3(g.x - k.o.x, g.y - k.o.y, g.z - k.o.z);
    const float u2 = dot3(u, u);
    const float r2g = g.w + kGraze;
    if (!(u2 > r2g * (1.f + 4.f * kCullRel) + kCullAbs)) return 0;  // origin clearly outside
    const float un = sqrtf(u2);
    if (!(un * (1.f + kCullRel) + kCullAbs < sqrtf(ls2))) return 0;  // entry <= tca <= |u| < |p - L| <= limit
    const bool front = conic_front(k, g);
    const float3 n = u * (1.f / un);
    // orthonormal pair perpendicular to n (branch-free, Duff et al. 2017)
    const float sg = copysignf(1.f, n.z);
    const float ia = -1.f / (sg + n.z);
    const float bb = n.x * n.y * ia;
    const float3 e1 = f3(1.f + sg * n.x * n.x * ia, sg * bb, -sg * n.x);
    const float3 e2 = f3(bb, sg + n.y * n.y * ia, -n.y);
    const float s = un * rsqrtf(r2g);
    ca = make_float4(s * dot3(e1, lo), s * dot3(e1, bu), s * dot3(e1, bv), s * dot3(e2, lo));
    cb = make_float4(s * dot3(e2, bu), s * dot3(e2, bv), 0.f, 0.f);
    if (front) return 1;
    const float z0 = dot3(n, lo);
    if (!(fabsf(z0) > 1e-6f * (sqrtf(dot3(lo, lo)) + 1.f))) return 0;
    const float iz = 1.f / fabsf(z0);
    cb.z = dot3(n, bu) * iz;
    cb.w = dot3(n, bv) * iz;
    return z0 > 0.f ? 2 : 3;
}

// Planes: a shadow segment crosses y = hp iff o.y and its far end (within
// 1e-3 of a disc point, whose height is within rho of L.y) straddle it.
__device__ __forceinline__ int plane_class(const Cone &k, float oy, float ly, float hp) {
    float m = kCullAbs * (1.f + fabsf(hp) + fabsf(ly));
    float lo = ly - k.rho - 1e-3f - m, hi = ly + k.rho + 1e-3f + m;
    float a = oy - hp;
    if ((a > m && lo > hp + m) || (a < -m && hi < hp - m)) return 0;
    if ((a > m && hi < hp - m) || (a < -m && lo > hp + m)) return 2;
    return 1;
}

// renderer.py:185-224: the unwind of one pixel's records (body, Lambert,
// Blinn, shadow coefficient), deepest first; a depth-cut chain shades its
// last base colour as-is, every other record mixes base*(1-rr) + col*rr.
struct Record {
    int idx;
    float dfs, s, sc;
};

// mat4: the bodies' {r, g, b, refl/max_refl} staged in shared memory, or
// null (read from sa.mat)
template <class Get>
__device__ __forceinline__ float3 unwind(int m, bool exhausted, float3 tail, const SceneArgs<float> &sa, Get get,
                                         const float4 *mat4 = nullptr) {
    float3 col = tail;
    for (int k = m - 1; k >= 0; k--) {
        const Record r = get(k);
        float lum = fminf(sa.ambient + r.sc * r.dfs * (1.f - sa.ambient), 1.f);
        float sp = r.sc * r.s;
        const float4 mt = mat4 ? mat4[r.idx] : __ldg(reinterpret_cast<const float4 *>(sa.mat + 8 * r.idx));
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
    return col;
}

// The same for m <= N records, fully unrolled: get(k) sees compile-time k,
// so records held in a register array stay in registers.
template <int N, class Get>
__device__ __forceinline__ float3 unwind_upto(int m, bool exhausted, float3 tail, const SceneArgs<float> &sa, Get get,
                                              const float4 *mat4 = nullptr) {
    float3 col = tail;
#pragma unroll
    for (int k = N - 1; k >= 0; k--) {
        if (k >= m) continue;
        const Record r = get(k);
        float lum = fminf(sa.ambient + r.sc * r.dfs * (1.f - sa.ambient), 1.f);
        float sp = r.sc * r.s;
        const float4 mt = mat4 ? mat4[r.idx] : __ldg(reinterpret_cast<const float4 *>(sa.mat + 8 * r.idx));
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
    return col;
}

__device__ __forceinline__ void store_pixel(const FrameArgs &fa, int x, int y, float3 c) {
    fa.out[(int64_t)y * fa.out_pitch + x] = pack_color(c.x, c.y, c.z, fa.rgba);
    if (fa.radiance) {
        float *r = (float *)fa.radiance + 3 * ((int64_t)y * fa.width + x);
        r[0] = c.x;
        r[1] = c.y;
        r[2] = c.z;
    }
}

}  // namespace rt32
