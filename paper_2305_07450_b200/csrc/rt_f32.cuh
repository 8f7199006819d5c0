// FP32 device math shared by the megakernel (render_f32.cu) and the
// wavefront kernels (render_wave_f32.cu): vector helpers, the reference's
// intersection tests in FP32 form, the launch-parameter / memory scene
// accessors, the skybox lookup.  Both translation units are compiled with
// the same flags (--ftz=true --prec-div=false --prec-sqrt=false).
#pragma once
#include <algorithm>
#include <cmath>
#include <map>
#include <tuple>
#include <utility>
#include <vector>

#include "rt_device.cuh"

#ifndef RT_F32_MIN_BLOCKS
#define RT_F32_MIN_BLOCKS 1  // __launch_bounds__ minimum resident CTAs per SM (register cap)
#endif

namespace rt32 {
using namespace rt;

constexpr int kMaxPlanes = 8;
// plane loops (a scene has one plane or a few): not unrolled, which keeps the
// hot kernels' code — and their instruction-cache misses — smaller
#ifndef RT_PLANE_UNROLL
#define RT_PLANE_UNROLL 1
#endif
constexpr int kPlaneUnroll = RT_PLANE_UNROLL;

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

// --- the ray chain in float64 -------------------------------------------------------
// A bounce chain is sensitive to its rays' rounding: a primary direction
// merely rounded to float32 moves 0.07% of C5's pixels (and 0.2% of C2's)
// more than 1e-4 relative away from the reference (tools/precision_probe.py).
// So the FP32 kernels carry each ray's origin and direction in float64 —
// the primary direction, the hit point and normal of every closest hit, the
// reflected ray — exactly as the reference forms them; the body search, the
// shadow tests and the shading run in FP32 on the rounded values (their
// rounding measured harmless: < 0.004% of pixels).
struct D3 {
    double x, y, z;
};
// cvt.rn.f32.f64 as PTX: one F2F.  Under --ftz=true a C cast becomes
// cvt.rn.ftz, which ptxas emulates with a range test and a predicated
// multiply per component to flush float denormals; the FTZ arithmetic
// downstream flushes any denormal it meets anyway.
__device__ __forceinline__ float d2f(double x) {
    float r;
    asm("cvt.rn.f32.f64 %0, %1;" : "=f"(r) : "d"(x));
    return r;
}
__device__ __forceinline__ float3 rnd(D3 a) { return make_float3(d2f(a.x), d2f(a.y), d2f(a.z)); }

// float64 square root, reciprocal and reciprocal square root from an FP32
// estimate and one Newton step (relative error ~1e-14, far below the float32
// rounding the chain exists to avoid; a handful of DFMAs instead of the
// IEEE sequences).  Arguments are finite, positive and within FP32 range.
__device__ __forceinline__ double sqrt64(double x) {
    const float sf = sqrtf(d2f(x));
    if (!(sf > 0.f)) return 0.0;
    const double s0 = (double)sf;
    return fma(fma(-s0, s0, x), (double)(0.5f / sf), s0);
}
__device__ __forceinline__ double rsqrt64(double x) {
    const double y = (double)rsqrtf(d2f(x));
    return y * fma(-0.5 * x * y, y, 1.5);
}
__device__ __forceinline__ double div64(double a, double b) {
    const double r = (double)(1.f / d2f(b));
    const double q = a * r;
    return fma(fma(-q, b, a), r, q);
}

// camera.py:46-77 in float64: one FMA per NDC coordinate and a reciprocal
// square root instead of the reference's five divisions and a square root
__device__ __forceinline__ D3 primary_direction64(int xi, int yi, const FrameArgs &fa) {
    const double u = fma((double)xi, fa.ndc[0], fa.ndc[1]);
    const double v = fma((double)yi, fa.ndc[2], fa.ndc[3]);
    const double inv = rsqrt64(fma(u, u, fma(v, v, fa.vdist * fa.vdist)));
    const double dx = u * inv, dy = v * inv, dz = fa.vdist * inv;
    const double y2 = dy * fa.cb - dz * fa.sb;
    const double z2 = dy * fa.sb + dz * fa.cb;
    const double x2 = dx * fa.ca + z2 * fa.sa;
    const double z3 = -dx * fa.sa + z2 * fa.ca;
    return D3{x2, y2, z3};
}

// camera.py:46-77 in float64, then rounded
__device__ __forceinline__ float3 primary_direction(int xi, int yi, const FrameArgs &fa) {
    return rnd(primary_direction64(xi, yi, fa));
}

// A closest hit found by the FP32 search, redone in float64 on the body's
// float64 geometry (geo64: the reference's packed {c, r^2} / {0, h, 0, -1}
// per body, then 1/r per body): the distance (geometry.py:83-117, the
// perpendicular formed cancellation-free; a graze the float64 test would call
// a miss counts as the FP32 search's hit), the hit point o + t d and the
// normal (renderer.py:141-151).  reflect64 then forms the reflected ray
// (renderer.py:178-183: origin p + 1e-3 n, direction d - 2 (n.d) n).
__device__ __forceinline__ void refine_hit(D3 o, D3 d, const double *__restrict__ geo64, int n_bodies, int idx, D3 &p,
                                           D3 &n) {
    const double2 g01 = __ldg(reinterpret_cast<const double2 *>(geo64) + 2 * idx);
    const double2 g23 = __ldg(reinterpret_cast<const double2 *>(geo64) + 2 * idx + 1);
    if (g23.y >= 0.0) {
        const double lx = g01.x - o.x, ly = g01.y - o.y, lz = g23.x - o.z;
        const double tca = fma(lz, d.z, fma(ly, d.y, lx * d.x));
        const double px = fma(-tca, d.x, lx), py = fma(-tca, d.y, ly), pz = fma(-tca, d.z, lz);
        const double rad = fma(-pz, pz, fma(-py, py, fma(-px, px, g23.y)));
        const double t = fmax(tca - sqrt64(fmax(rad, 0.0)), 0.0);
        p = D3{fma(d.x, t, o.x), fma(d.y, t, o.y), fma(d.z, t, o.z)};
        const double inv_r = __ldg(geo64 + 4 * n_bodies + idx);
        n = D3{(p.x - g01.x) * inv_r, (p.y - g01.y) * inv_r, (p.z - g23.x) * inv_r};
    } else {
        const double t = div64(g01.y - o.y, d.y);
        p = D3{fma(d.x, t, o.x), fma(d.y, t, o.y), fma(d.z, t, o.z)};
        n = D3{0.0, 1.0, 0.0};
    }
}

__device__ __forceinline__ void reflect64(D3 p, D3 n, D3 &o, D3 &d) {
    o = D3{fma(n.x, 1e-3, p.x), fma(n.y, 1e-3, p.y), fma(n.z, 1e-3, p.z)};
    const double k = 2.0 * fma(n.z, d.z, fma(n.y, d.y, n.x * d.x));
    d = D3{fma(-k, n.x, d.x), fma(-k, n.y, d.y), fma(-k, n.z, d.z)};
}

// geometry.py:83-105 — distance to the sphere, +inf on a miss.
__device__ __forceinline__ float sphere_t(float3 o, float3 d, float4 g) {
    float3 L = f3(g.x - o.x, g.y - o.y, g.z - o.z);
    float tca = dot3(L, d);
    float3 p = L - d * tca;
    float rad = g.w - dot3(p, p);
    float t = tca - sqrtf(fmaxf(rad, 0.f));
    // the reference's tca < 0 miss is implied: t <= tca, so t >= 0 needs tca >= 0
    return (rad >= -1e-7f && t >= 0.f) ? t : INFINITY;
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
// d ** e of the Blinn highlight (shading.py:73) for d in [0, 1] and the
// validated reflectivities e >= 0 (geometry.py:42-48): exp2(e log2 d) with
// pow's special cases (d ** 0 = 1, 0 ** e = 0); log2f / exp2f keep ~1e-7
// relative error, the FP32 budget.  No powf: its ~150 instructions of
// special-case code sat in every hit's path (instruction-cache pressure).
__device__ __forceinline__ float blinn_pow(float d, float e) {
    if (e == 0.f) return 1.f;
    return d > 0.f ? exp2f(e * log2f(d)) : 0.f;
}

constexpr float kGraze = 1e-7f;  // geometry.py:24

// The shadow grid's mask for a shadow origin o (MegaCull::grid): ~0 when
// there is no grid or o lies outside it.
__device__ __forceinline__ unsigned scene_grid_mask(const MegaCull &mc, float3 o) {
    if (!mc.grid) return ~0u;
    const int ix = __float2int_rd((o.x - mc.grid_lo[0]) * mc.grid_inv[0]);
    const int iy = __float2int_rd((o.y - mc.grid_lo[1]) * mc.grid_inv[1]);
    const int iz = __float2int_rd((o.z - mc.grid_lo[2]) * mc.grid_inv[2]);
    if ((unsigned)ix >= (unsigned)mc.grid_dim[0] || (unsigned)iy >= (unsigned)mc.grid_dim[1] ||
        (unsigned)iz >= (unsigned)mc.grid_dim[2])
        return ~0u;
    return __ldg(mc.grid + ((size_t)iz * mc.grid_dim[1] + iy) * mc.grid_dim[0] + ix);
}

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
// Spheres of scenes with more than 8 spheres are grouped into clusters of
// up to kClusterSize (median splits on the host) with a conservative bounding
// sphere, stored cluster-major: closest-hit and any-hit loops skip every
// member of a cluster whose bound the ray cannot reach in time, and the
// shadow-cone classifier skips clusters outside the cone.  Skipping only
// bodies that provably cannot win (or block) leaves every result unchanged.
constexpr int kClusterSize = 16;
constexpr int kMaxClusters = 32;
constexpr float kBoundRel = 1e-4f;  // slack on cluster-skip decisions (FP32 rounding is ~1e-6)

// Entry distance of the ray into the bound (a lower bound of every member's
// hit distance), +inf if the ray misses it, <= 0 if it starts inside.
__device__ __forceinline__ float bound_entry(float3 o, float3 d, float4 B) {
    float3 L = f3(B.x - o.x, B.y - o.y, B.z - o.z);
    float tca = dot3(L, d);
    float3 p = L - d * tca;
    float rad = B.w * B.w - dot3(p, p);
    if (rad < 0.f) return INFINITY;
    float s = sqrtf(rad);
    if (tca + s < 0.f) return INFINITY;  // wholly behind the origin
    return tca - s - kBoundRel * (fabsf(tca) + B.w);
}

template <int MAXS>
struct ParamScene {
    static constexpr bool kClustered = MAXS > 8;
    static constexpr int kNC = kClustered ? kMaxClusters : 1;
    float4 sph[MAXS];
    int sph_idx[MAXS];
    float2 sph_rad[MAXS];    // {r, sqrt(r^2 + 1e-7)} for the shadow-cone classifier
    float pl_h[kMaxPlanes];
    int pl_idx[kMaxPlanes];
    float4 cl[kNC];          // cluster bounds {centre, radius}
    int cl_begin[kNC + 1];   // members of cluster c: slots [cl_begin[c], cl_begin[c+1])
    int ns, np, nc;

    // SPARSE (unclustered scenes): only the spheres in smask are tested — a
    // primary ray's primary_sphere_mask; the others cannot be hit
    template <bool SPARSE = false>
    __device__ __forceinline__ Hit closest(float3 o, float3 d, unsigned smask = ~0u) const {
        Hit h{-1, INFINITY, make_float4(0.f, 0.f, 0.f, -1.f)};
        int slot = -1;
        if constexpr (!kClustered) {
            // nc = 1: cl[0] bounds every sphere (pack_params); a ray missing
            // it cannot hit one (the clustered walk's test, with its margins)
            const bool skip = nc > 0 && bound_entry(o, d, cl[0]) == INFINITY;
#pragma unroll
            for (int b = 0; b < MAXS; b++) {
                if (b >= ns || skip) break;
                if (SPARSE && !((smask >> b) & 1u)) continue;
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
#pragma unroll(kPlaneUnroll)
            for (int j = 0; j < np; j++) {
                float t = plane_t(o, d, pl_h[j]);
                if (t < h.t || (t == h.t && pl_idx[j] < h.idx)) {  // geometry.py:198 across kinds
                    h.t = t;
                    h.idx = pl_idx[j];
                    h.g = make_float4(0.f, pl_h[j], 0.f, -1.f);
                }
            }
        } else {
            // planes first: a floor hit bounds the cluster walk
#pragma unroll(kPlaneUnroll)
            for (int j = 0; j < np; j++) {
                float t = plane_t(o, d, pl_h[j]);
                if (t < h.t || (t == h.t && pl_idx[j] < h.idx)) {
                    h.t = t;
                    h.idx = pl_idx[j];
                    h.g = make_float4(0.f, pl_h[j], 0.f, -1.f);
                }
            }
            for (int c = 0; c < nc; c++) {
                if (bound_entry(o, d, cl[c]) > h.t) continue;
                const int b1 = cl_begin[c + 1];
#pragma unroll 4
                for (int b = cl_begin[c]; b < b1; b++) {
                    float t = sphere_t(o, d, sph[b]);
                    if (t <= h.t) {
                        int id = sph_idx[b];
                        if (t < h.t || id < h.idx) {  // (t, index) order: lowest original index wins ties
                            h.t = t;
                            h.idx = id;
                            slot = b;
                        }
                    }
                }
            }
            if (slot >= 0 && h.idx == sph_idx[slot]) h.g = sph[slot];
        }
        return h;
    }

    // Per-hit constants of the any-hit loop: the shadow origin is shared by
    // all samples of a hit, so L = c - o, the inside/outside decision and
    // h - o.y are formed once per hit.
    // wm (unclustered scenes): the spheres that can block a ray from o, from
    // the shadow grid's cell of o (all when there is none); the others are
    // skipped, which leaves the any-hit answer unchanged.
    struct Local {
        float3 o;
        float4 L[kClustered ? 1 : MAXS];  // xyz = centre - origin, w = r2g
        unsigned wm;
    };

    __device__ __forceinline__ Local localize(float3 o, unsigned wm = ~0u) const {
        Local lc;
        lc.o = o;
        lc.wm = wm;
        if constexpr (!kClustered) {
#pragma unroll
            for (int b = 0; b < MAXS; b++) {
                float3 L = f3(sph[b].x - o.x, sph[b].y - o.y, sph[b].z - o.z);
                // a sphere the grid rules out never blocks: r2g = -inf, as for an origin inside
                lc.L[b] = make_float4(L.x, L.y, L.z, (wm >> b) & 1u ? sphere_r2g(L, sph[b].w) : -INFINITY);
            }
        }
        return lc;
    }

    // SPARSE (one ray per hit): the spheres the grid rules out are skipped;
    // otherwise tested branch-free (their r2g = -inf never blocks)
    template <bool SPARSE = false>
    __device__ __forceinline__ bool occluded(const Local &lc, float3 d, float limit) const {
        float m = -INFINITY;
#pragma unroll(kPlaneUnroll)
        for (int j = 0; j < np; j++) {
            m = fmaxf(m, plane_margin(pl_h[j] - lc.o.y, d.y, limit));
        }
        if constexpr (!kClustered) {
#pragma unroll
            for (int b = 0; b < MAXS; b++) {
                if (b >= ns) break;
                if (SPARSE && !((lc.wm >> b) & 1u)) continue;
                float4 L = lc.L[b];
                m = fmaxf(m, sphere_margin_L(f3(L.x, L.y, L.z), d, L.w, limit));
            }
        } else {
            for (int c = 0; c < nc && !(m > 0.f); c++) {
                if (bound_entry(lc.o, d, cl[c]) >= limit) continue;  // no member within [0, limit)
                for (int b = cl_begin[c]; b < cl_begin[c + 1]; b++) m = fmaxf(m, sphere_margin(lc.o, d, sph[b], limit));
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

    template <bool SPARSE = false>
    __device__ __forceinline__ Hit closest(float3 o, float3 d, unsigned = ~0u) const {
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
    __device__ __forceinline__ Local localize(float3 o, unsigned = ~0u) const { return Local{o}; }

    template <bool SPARSE = false>
    __device__ __forceinline__ bool occluded(const Local &lc, float3 d, float limit) const {
        for (int b = 0; b < n; b++) {
            float4 g = geo[b];
            float m = g.w >= 0.f ? sphere_margin(lc.o, d, g, limit) : plane_margin(g.y - lc.o.y, d.y, limit);
            if (m > 0.f) return true;
        }
        return false;
    }
};

// renderer.py:60-74
static __device__ float3 sky_sample(float3 d, const float4 *__restrict__ sky, int W, int H) {
    float u = 0.5f + atan2f(d.x, d.z) * 0.15915494309189535f;
    float dy = fminf(fmaxf(d.y, -1.f), 1.f);
    float v = 0.5f - asinf(dy) * 0.3183098861837907f;
    int tx = (int)floorf(u * (float)W);
    // ((tx % W) + W) % W of renderer.py:67 for the only reachable tx, -1..W
    // (u is within rounding of [0, 1]): no integer divisions
    tx = tx < 0 ? tx + W : (tx >= W ? tx - W : tx);
    int ty = (int)floorf(v * (float)H);
    ty = min(max(ty, 0), H - 1);
    float4 t = __ldg(sky + (int64_t)ty * W + tx);
    return f3(t.x, t.y, t.z);
}

__device__ __forceinline__ float clamp01(float x) { return fminf(fmaxf(x, 0.f), 1.f); }

// Disc-sample table (shading.py:89-100) and its sunflower basis for a hit.
struct DiscBasis {
    float3 bu, bv;
};

// shading.py:76-86 in FP32
__device__ __forceinline__ DiscBasis disc_basis(float3 surface, float3 lp) {
    float3 axis = normalize3(surface - lp);
    float3 c = cross3(axis, f3(0.f, 1.f, 0.f));
    float m2 = dot3(c, c);
    DiscBasis b;
    b.bu = m2 >= 1e-18f ? c * rsqrtf(m2) : f3(1.f, 0.f, 0.f);
    b.bv = cross3(axis, b.bu);
    return b;
}

// Pack the host scene (float64 geo) into the launch-parameter layout; false
// if it does not fit.
// Median-split clustering of spheres (host): slots [b0, b1) of `order`
// become clusters of at most kClusterSize, split on the longest axis.
inline void split_clusters(const std::vector<float4> &c, std::vector<int> &order, int b0, int b1,
                           std::vector<std::pair<int, int>> &out) {
    if (b1 - b0 <= kClusterSize) {
        out.emplace_back(b0, b1);
        return;
    }
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = b0; i < b1; i++) {
        const float4 &p = c[order[i]];
        const float v[3] = {p.x, p.y, p.z};
        for (int a = 0; a < 3; a++) {
            lo[a] = std::min(lo[a], v[a]);
            hi[a] = std::max(hi[a], v[a]);
        }
    }
    int ax = 0;
    for (int a = 1; a < 3; a++)
        if (hi[a] - lo[a] > hi[ax] - lo[ax]) ax = a;
    int mid = (b0 + b1) / 2;
    auto key = [&](int i) { return ax == 0 ? c[i].x : ax == 1 ? c[i].y : c[i].z; };
    std::nth_element(order.begin() + b0, order.begin() + mid, order.begin() + b1,
                     [&](int a, int b) { return key(a) < key(b) || (key(a) == key(b) && a < b); });
    split_clusters(c, order, b0, mid, out);
    split_clusters(c, order, mid, b1, out);
}

// Pack the host scene (float64 geo) into the launch-parameter layout; false
// if it does not fit.
constexpr int kBoundMinSpheres = 3;  // unclustered scenes of at least this many spheres get a sphere bound
inline bool g_sphere_bound = true;   // (option sphere_bound; a host-side switch for A/B runs)

template <int MAXS>
inline bool pack_params(const SceneArgs<float> &sa, ParamScene<MAXS> &ps) {
    ps.ns = ps.np = 0;
    std::vector<float4> sph;
    std::vector<int> idx;
    for (int b = 0; b < sa.n; b++) {
        const double *g = sa.host_geo + 4 * b;
        if (g[3] >= 0.0) {
            if ((int)sph.size() == MAXS) return false;
            sph.push_back(make_float4((float)g[0], (float)g[1], (float)g[2], (float)g[3]));
            idx.push_back(b);
        } else {
            if (ps.np == kMaxPlanes) return false;
            ps.pl_h[ps.np] = (float)g[1];
            ps.pl_idx[ps.np++] = b;
        }
    }
    ps.ns = (int)sph.size();
    std::vector<int> order(ps.ns);
    for (int i = 0; i < ps.ns; i++) order[i] = i;
    ps.nc = 0;
    if constexpr (ParamScene<MAXS>::kClustered) {
        std::vector<std::pair<int, int>> ranges;
        if (ps.ns > 0) split_clusters(sph, order, 0, ps.ns, ranges);
        if ((int)ranges.size() > kMaxClusters) return false;
        for (auto &r : ranges) {
            // each cluster keeps its members in ascending original order
            std::sort(order.begin() + r.first, order.begin() + r.second);
            double cx = 0, cy = 0, cz = 0;
            for (int i = r.first; i < r.second; i++) {
                cx += sph[order[i]].x;
                cy += sph[order[i]].y;
                cz += sph[order[i]].z;
            }
            double k = 1.0 / (r.second - r.first);
            cx *= k;
            cy *= k;
            cz *= k;
            double R = 0;
            for (int i = r.first; i < r.second; i++) {
                const float4 &p = sph[order[i]];
                double dx = p.x - cx, dy = p.y - cy, dz = p.z - cz;
                R = std::max(R, std::sqrt(dx * dx + dy * dy + dz * dz) + std::sqrt((double)p.w + 1e-7));
            }
            ps.cl[ps.nc] = make_float4((float)cx, (float)cy, (float)cz, (float)(R * (1.0 + 1e-4) + 1e-4));
            ps.cl_begin[ps.nc] = r.first;
            ps.nc++;
        }
        ps.cl_begin[ps.nc] = ps.ns;
    } else if (ps.ns >= kBoundMinSpheres) {
        // one bound over every sphere: a ray that misses it skips the sphere
        // loop (sky rays, rays off into the distance)
        double cx = 0, cy = 0, cz = 0;
        for (const float4 &p : sph) {
            cx += p.x;
            cy += p.y;
            cz += p.z;
        }
        cx /= ps.ns;
        cy /= ps.ns;
        cz /= ps.ns;
        double R = 0;
        for (const float4 &p : sph) {
            double dx = p.x - cx, dy = p.y - cy, dz = p.z - cz;
            R = std::max(R, std::sqrt(dx * dx + dy * dy + dz * dz) + std::sqrt((double)p.w + 1e-7));
        }
        ps.cl[0] = make_float4((float)cx, (float)cy, (float)cz, (float)(R * (1.0 + 1e-4) + 1e-4));
        ps.cl_begin[0] = 0;
        ps.cl_begin[1] = ps.ns;
        ps.nc = g_sphere_bound ? 1 : 0;
    }
    for (int i = 0; i < ps.ns; i++) {
        ps.sph[i] = sph[order[i]];
        ps.sph_idx[i] = idx[order[i]];
        const double r2 = sa.host_geo[4 * idx[order[i]] + 3];
        ps.sph_rad[i] = make_float2((float)std::sqrt(r2), (float)std::sqrt(r2 + 1e-7));
    }
    for (int b = ps.ns; b < MAXS; b++) {
        ps.sph[b] = make_float4(0.f, 0.f, 0.f, 0.f);
        ps.sph_idx[b] = 0;
        ps.sph_rad[b] = make_float2(0.f, 0.f);
    }
    for (int j = ps.np; j < kMaxPlanes; j++) {
        ps.pl_h[j] = 0.f;
        ps.pl_idx[j] = 0;
    }
    for (int c = ps.nc; c < ParamScene<MAXS>::kNC; c++) {
        ps.cl[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        ps.cl_begin[c + 1] = ps.ns;
    }
    return true;
}

// The shadow rays of one hit (renderer.py:82-105): origin o = p + 1e-3 n,
// sample s_i = L + a_i u + b_i v on the disc.  Per ray the kernels need
// dir = normalize(s_i - o) and limit = |p - s_i|; with p - L parallel to the
// disc axis and u, v orthogonal to it, |p - s_i|^2 = |p - L|^2 + a_i^2 + b_i^2,
// so a table entry {a_i, b_i, a_i^2 + b_i^2} (float64 on the host, rounded)
// gives the limit with one FMA and a reciprocal square root.
struct ShadowFrame {
    float3 origin;  // o
    float3 lo;      // L - o
    float3 bu, bv;  // disc basis (zero for hard shadows: s = L)
    float ls2;      // |p - L|^2
};

__device__ __forceinline__ ShadowFrame shadow_frame(float3 surface, float3 normal, float3 lp, bool soft) {
    ShadowFrame f;
    f.origin = surface + normal * 1e-3f;
    f.lo = lp - f.origin;
    float3 ls = surface - lp;
    f.ls2 = dot3(ls, ls);
    if (soft) {
        DiscBasis db = disc_basis(surface, lp);
        f.bu = db.bu;
        f.bv = db.bv;
    } else {
        f.bu = f.bv = f3(0.f, 0.f, 0.f);
    }
    return f;
}

// t = {a_i, b_i, a_i^2 + b_i^2, 0}; all zero for hard shadows
__device__ __forceinline__ void shadow_ray(const ShadowFrame &f, float4 t, float3 &dir, float &limit) {
    float3 dv = f3(fmaf(f.bv.x, t.y, fmaf(f.bu.x, t.x, f.lo.x)), fmaf(f.bv.y, t.y, fmaf(f.bu.y, t.x, f.lo.y)),
                   fmaf(f.bv.z, t.y, fmaf(f.bu.z, t.x, f.lo.z)));
    float r2 = dot3(dv, dv);
    dir = dv * (r2 > 0.f ? rsqrtf(r2) : 0.f);
    float l2 = f.ls2 + t.z;
    limit = l2 > 0.f ? l2 * rsqrtf(l2) : 0.f;
}

// The same without the zero-length guards, for the soft-shadow loops: a
// zero-length vector needs the surface point on the light disc itself, where
// the NaN it produces makes every margin comparison false — unblocked, as the
// reference's zero direction / zero limit give.
__device__ __forceinline__ void shadow_ray_unguarded(const ShadowFrame &f, float4 t, float3 &dir, float &limit) {
    float3 dv = f3(fmaf(f.bv.x, t.y, fmaf(f.bu.x, t.x, f.lo.x)), fmaf(f.bv.y, t.y, fmaf(f.bu.y, t.x, f.lo.y)),
                   fmaf(f.bv.z, t.y, fmaf(f.bu.z, t.x, f.lo.z)));
    dir = dv * rsqrtf(dot3(dv, dv));
    float l2 = f.ls2 + t.z;
    limit = l2 * rsqrtf(l2);
}

// Persistent grid: as many CTAs as fit on the device at once (memoised per
// kernel, shared-memory size and device: the occupancy query costs
// microseconds of host time per launch otherwise).
template <typename K>
inline int resident_ctas(K kernel, size_t smem, int threads = kThreads) {
    int dev = 0;
    cudaGetDevice(&dev);
    static thread_local std::map<std::tuple<const void *, size_t, int, int>, int> memo;
    auto key = std::make_tuple((const void *)kernel, smem, threads, dev);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    int ctas = sms * (per_sm > 0 ? per_sm : 1);
    memo[key] = ctas;
    return ctas;
}

}  // namespace rt32
