// FP64 soft shadows with exact occluder culling: the bit-identical mode at
// wavefront speed.  Three kernels, as the FP32 culled path
// (render_fused_f32.cu) had them: trace + per-hit cone classification,
// sampling of the undecided hits, unwind of the parked pixels.  Every value
// the reference computes is computed here in its literal float64 order
// (rt_f64.cuh, compiled with -fmad=false).  The cone classifier (float32 on
// rounded inputs, margins of 1e-4 relative) only decides which bodies cannot
// block any of a hit's shadow rays, or block all of them; the lane sampler
// decides a sample by a float64 silhouette test only when the decision is
// certain, else by the literal test.  Every decision is the reference's.
//
// Scenes of up to kMaxBodies64 bodies (geometry staged in shared memory per
// CTA, candidate masks over original body indices); larger scenes keep the
// megakernel.
#include <map>
#include <utility>

#include "rt_f64.cuh"

namespace {
using namespace rt;
using namespace rt64;

constexpr int kWords64 = kMaxBodies64 / 32;
constexpr double kCullRel64 = 1e-4;
constexpr double kCullAbs64 = 1e-5;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// The hit's shadow cone and the classification of a body against it (see
// rt_wave.cuh for the geometry: nothing can block / some samples / all).
// In float32 on the float64 inputs rounded once:
// the margins (1e-4 relative, 1e-5 absolute) stand far above both that
// rounding (6e-8 relative) and float32 arithmetic, so the decisions stay
// conservative — exactly the skips the float64 classifier would make, or
// fewer — at a fraction of the float64 pipe's cost.
struct Cone32 {
    float ox, oy, oz, ax, ay, az, H, rho, inv_H, sin_phi, cos_phi, reach;
    bool ok;
};

__device__ __forceinline__ Cone32 make_cone32(d3 o64, d3 lp64, double light_radius) {
    constexpr float rel = (float)kCullRel64, abs_ = (float)kCullAbs64;
    Cone32 c;
    c.ox = (float)o64.x;
    c.oy = (float)o64.y;
    c.oz = (float)o64.z;
    const float Ax = (float)lp64.x - c.ox, Ay = (float)lp64.y - c.oy, Az = (float)lp64.z - c.oz;
    c.H = sqrtf(Ax * Ax + Ay * Ay + Az * Az);
    c.rho = 2.f * (float)light_radius * (1.f + rel) + abs_;
    c.ok = c.H > 0.f && c.rho < 0.999f * c.H;
    c.inv_H = c.H > 0.f ? 1.f / c.H : 0.f;
    c.ax = Ax * c.inv_H;
    c.ay = Ay * c.inv_H;
    c.az = Az * c.inv_H;
    c.sin_phi = c.ok ? c.rho * c.inv_H : 1.f;
    c.cos_phi = sqrtf(fmaxf(1.f - c.sin_phi * c.sin_phi, 0.f));
    const float T = 1.f + (1e-3f + abs_) / fmaxf(c.H - c.rho, 1e-6f);
    c.reach = T * (c.H + c.rho) * (1.f + rel) + abs_;
    return c;
}

__device__ __forceinline__ int body_class32(const Cone32 &k, const double *g, float oy, float ly) {
    constexpr float rel = (float)kCullRel64, abs_ = (float)kCullAbs64;
    if (!k.ok) return 1;
    if (g[3] < 0.0) {  // horizontal plane at g[1]
        const float hp = (float)g[1], m = abs_ * (1.f + fabsf(hp) + fabsf(ly));
        const float lo = ly - k.rho - 1e-3f - m, hi = ly + k.rho + 1e-3f + m;
        const float a = oy - hp;
        if ((a > m && lo > hp + m) || (a < -m && hi < hp - m)) return 0;
        if ((a > m && hi < hp - m) || (a < -m && lo > hp + m)) return 2;
        return 1;
    }
    const float r2 = (float)g[3];
    const float ux = (float)g[0] - k.ox, uy = (float)g[1] - k.oy, uz = (float)g[2] - k.oz;
    const float u2 = ux * ux + uy * uy + uz * uz;
    if (u2 < r2 * (1.f - 4.f * rel) - abs_) return 0;  // origin inside: t < 0 always
    const float h = ux * k.ax + uy * k.ay + uz * k.az;
    const float wx = ux - k.ax * h, wy = uy - k.ay * h, wz = uz - k.az * h;
    const float q = sqrtf(wx * wx + wy * wy + wz * wz);
    const float un = fabsf(h) + q;
    const float r = sqrtf(r2);
    const float rp = sqrtf(r2 + 1e-7f) * (1.f + rel) + abs_ + 1e-6f * (un + k.H);
    if (h < -rp || h - rp > k.reach) return 0;
    if (h * k.cos_phi + q * k.sin_phi >= 0.f) {
        if (q * k.cos_phi - h * k.sin_phi >= rp) return 0;
    } else if (u2 >= rp * rp) {
        return 0;
    }
    const float rm = r * (1.f - 10.f * rel) - abs_ - 1e-6f * (un + k.H);
    if (u2 > r2 * (1.f + 4.f * rel) + abs_ && h > 0.f && h + r < (k.H - k.rho) * (1.f - rel) - 2e-3f &&
        q + h * k.inv_H * k.rho * (1.f + rel) < rm)
        return 2;
    return 1;
}

__device__ __forceinline__ const double *stage(const SceneArgs<double> &sa, double *smem) {
    for (int i = threadIdx.x; i < 4 * sa.n; i += blockDim.x) smem[i] = sa.geo[i];
    __syncthreads();
    return smem;
}

// --- A: trace, classify, unwind the decided pixels ---------------------------------
__global__ void __launch_bounds__(kThreads)
    fused64_trace(const FrameArgs fa, const SceneArgs<double> sa, const WaveArgs64 wa) {
    extern __shared__ double smem_geo[];
    const double *__restrict__ geo = stage(sa, smem_geo);
    const int lane = threadIdx.x & 31;
    int x, ly;
    thread_pixel_bottom_first(x, ly);
    int y = 0;
    bool alive = x < fa.width && ly < fa.local_rows;
    if (alive) {
        y = map_row(ly, fa);
        alive = y < fa.row_end;
    }
    const bool valid = alive;
    const int64_t lp = (int64_t)ly * fa.width + x;
    const d3 light = mk(sa.light[0], sa.light[1], sa.light[2]);
    d3 origin = mk(fa.cam[0], fa.cam[1], fa.cam[2]);
    d3 dir = valid ? primary_direction(x, y, fa) : mk(0.0, 0.0, 1.0);
    d3 tail = mk(0.0, 0.0, 0.0);
    int m = 0, exhausted = 0, npend = 0;
    int ridx[kMaxBounce + 1];
    double rdfs[kMaxBounce + 1], rs[kMaxBounce + 1], rsc[kMaxBounce + 1];
    for (int k = 0; k <= fa.bounces; k++) {
        if (!__any_sync(0xffffffffu, alive)) break;
        double t = INFINITY;
        int idx = -1;
        if (alive) idx = closest(origin, dir, geo, sa.n, t);
        const bool hit_now = alive && idx >= 0;
        if (alive && !hit_now) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            alive = false;
        }
        int cls = 0;
        int64_t slot = 0;
        unsigned mask[kWords64];
        d3 hit = mk(0.0, 0.0, 0.0), normal = mk(0.0, 1.0, 0.0);
        if (hit_now) {
            const double *g = geo + 4 * idx;
            hit = mk(origin.x + dir.x * t, origin.y + dir.y * t, origin.z + dir.z * t);
            normal = (g[3] >= 0.0) ? vnormalize(vsub(hit, mk(g[0], g[1], g[2]))) : mk(0.0, 1.0, 0.0);
            d3 l = vnormalize(vsub(light, hit));
            double dfs, s;
            hit_terms(normal, l, dir, __ldg(sa.mat + 8 * idx + 4), dfs, s);
            // renderer.py:87-89: the shadow rays' origin
            const d3 so = mk(hit.x + 1e-3 * normal.x, hit.y + 1e-3 * normal.y, hit.z + 1e-3 * normal.z);
            const Cone32 cone = make_cone32(so, light, sa.light_radius);
#pragma unroll
            for (int w = 0; w < kWords64; w++) mask[w] = 0;
            bool full = false, any = false;
            for (int b = 0; b < sa.n; b++) {
                int c = body_class32(cone, geo + 4 * b, (float)so.y, (float)light.y);
                mask[b >> 5] |= (c == 1 ? 1u : 0u) << (b & 31);
                full |= c == 2;
                any |= c == 1;
            }
            cls = full ? 2 : (any ? 1 : 0);
            slot = (int64_t)k * wa.n_pix + lp;
            ridx[k] = idx;
            rdfs[k] = dfs;
            rs[k] = s;
            rsc[k] = cls == 2 ? 0.0 : 1.0;  // (double)n / n and 0 / n of renderer.py:105
            if (cls == 1) npend++;
            m = k + 1;
            if (k == fa.bounces) {
                exhausted = 1;
                alive = false;
            } else {
                origin = so;  // renderer.py:178-183: the same offset
                dir = vreflect(dir, normal);
            }
        }
        // a single candidate sphere: a lane of the lane sampler
        int one = -1;
        if (hit_now && cls == 1 && wa.lane_cap) {
            int nc = 0;
#pragma unroll
            for (int w = 0; w < kWords64; w++) {
                if (mask[w]) one = w * 32 + __ffs(mask[w]) - 1;
                nc += __popc(mask[w]);
            }
            if (nc != 1 || geo[4 * one + 3] < 0.0) one = -1;
        }
        bool laned = false;
        {
            const bool want = one >= 0;
            const unsigned lb = __ballot_sync(0xffffffffu, want);
            if (lb) {
                unsigned base = 0;
                if (lane == 0) base = atomicAdd(wa.count + 3, (unsigned)__popc(lb));
                base = __shfl_sync(0xffffffffu, base, 0);
                const unsigned e = base + __popc(lb & lanemask_lt());
                if (want && e < wa.lane_cap) {
                    wa.lane_q[2 * e] = make_double4(hit.x, hit.y, hit.z, (double)slot);
                    wa.lane_q[2 * e + 1] = make_double4(normal.x, normal.y, normal.z, (double)one);
                    laned = true;
                }
            }
        }
        const bool need = hit_now && cls == 1 && !laned;
        const unsigned nb = __ballot_sync(0xffffffffu, need);
        if (nb) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(wa.count + 1, (unsigned)__popc(nb));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (need) {
                const unsigned e = base + __popc(nb & lanemask_lt());
                wa.q[2 * e] = make_double4(hit.x, hit.y, hit.z, (double)slot);
                wa.q[2 * e + 1] = make_double4(normal.x, normal.y, normal.z, 0.0);
#pragma unroll
                for (int w = 0; w < kWords64; w++) wa.mask[(size_t)w * wa.mask_stride + e] = mask[w];
            }
        }
    }
    const bool park = valid && npend > 0;
    const unsigned pb = __ballot_sync(0xffffffffu, park);
    if (pb) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(wa.count + 2, (unsigned)__popc(pb));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (park) wa.parked[base + __popc(pb & lanemask_lt())] = (int)lp;
    }
    if (!valid) return;
    if (!park) {
        const d3 c = unwind(m, exhausted, tail, sa, [&](int k, int &i, double &d, double &s, double &sc) {
            i = ridx[k];
            d = rdfs[k];
            s = rs[k];
            sc = rsc[k];
        });
        fa.out[(int64_t)y * fa.out_pitch + x] = pack_color(c.x, c.y, c.z, fa.rgba);
        if (fa.radiance) {
            double *r = (double *)fa.radiance + 3 * ((int64_t)y * fa.width + x);
            r[0] = c.x;
            r[1] = c.y;
            r[2] = c.z;
        }
        if (fa.peer_out) __threadfence_system();
    } else {
        wa.pix[lp] = make_double4(tail.x, tail.y, tail.z, (double)(m | (exhausted << 8)));
        for (int k = 0; k < m; k++)
            wa.rec[(int64_t)k * wa.n_pix + lp] = make_double4((double)ridx[k], rdfs[k], rs[k], rsc[k]);
    }
}

// --- B1: single-sphere hits, one lane each, decisions exact ---------------------
//
// The reference's test of sample i against sphere g (renderer.py:90-103,
// geometry.py:83-105) is, when the shadow origin o is clearly outside g and
// |g - o| < |p - L| (so the entry point always precedes the limit),
//   blocked  <=>  tca > 0  and  d2 <= r^2 + 1e-7,
// a predicate on the real numbers that the silhouette form (rt_wave.cuh,
// conic_coeffs, here in float64 with explicit FMAs) evaluates as the sign of
// dd = x^2 + y^2 - |w|^2 (and z > 0 for tca).  Both the reference's literal
// float64 arithmetic and this one approximate that predicate; their errors
// are below c eps (s^2 + s (1 + 4R/H) + 1) |w|^2 with s = |u| / r (the literal
// d2 = L.L - tca^2 cancels by s^2).  With tau = 1024 eps (...) |w|^2 far
// above both, a sample with |dd| > tau is decided the way the reference
// decides it; the rare sample inside the band takes the literal test.  Near
// z = 0, d2 ~ |u|^2 > r^2 (1 + 1e-6): the z sign never decides there.  The
// coefficient, unblocked / n, is thus the reference's bit for bit.
__device__ void sample_lanes64(const FrameArgs &fa, const SceneArgs<double> &sa, const WaveArgs64 &wa,
                               const double *geo) {
    const int n = fa.samples;
    const d3 lp = mk(sa.light[0], sa.light[1], sa.light[2]);
    const double *tab = sa.table;
    const double2 *tab2 = reinterpret_cast<const double2 *>(tab);  // {r cos, r sin} per sample (host libm)
    const unsigned count = min(wa.count[3], wa.lane_cap);
    // kSplit adjacent lanes share a hit, each taking every kSplit-th sample:
    // more warps to hide the float64 latency with, for one more setup per hit
    constexpr unsigned kSplit = 2, kPer = 32 / kSplit;
    const unsigned units = (count + kPer - 1) / kPer;
    const unsigned first = (unsigned)(((unsigned long long)units * blockIdx.x) / gridDim.x);
    const unsigned last = (unsigned)(((unsigned long long)units * (blockIdx.x + 1)) / gridDim.x);
    const unsigned lane = threadIdx.x & 31, part = lane % kSplit;
    for (unsigned u = first + (threadIdx.x >> 5); u < last; u += blockDim.x >> 5) {
        const unsigned h = kPer * u + lane / kSplit;
        if (h >= count) continue;  // both lanes of a hit alike
        const double4 P = wa.lane_q[2 * h], N = wa.lane_q[2 * h + 1];
        const double *g = geo + 4 * (int)N.w;
        const d3 surface = mk(P.x, P.y, P.z), normal = mk(N.x, N.y, N.z);
        const d3 origin = mk(surface.x + 1e-3 * normal.x, surface.y + 1e-3 * normal.y, surface.z + 1e-3 * normal.z);
        d3 bu, bv;
        disc_basis(surface, lp, bu, bv);
        // the silhouette coefficients and their preconditions
        const d3 uc = mk(g[0] - origin.x, g[1] - origin.y, g[2] - origin.z);
        const d3 lo = mk(lp.x - origin.x, lp.y - origin.y, lp.z - origin.z);
        const d3 ls = mk(surface.x - lp.x, surface.y - lp.y, surface.z - lp.z);
        const double u2 = fma(uc.z, uc.z, fma(uc.y, uc.y, uc.x * uc.x));
        const double r2g = g[3] + 1e-7;
        const double un = sqrt(u2), H = sqrt(fma(lo.z, lo.z, fma(lo.y, lo.y, lo.x * lo.x)));
        const double rho = 2.0 * sa.light_radius * (1.0 + 1e-6) + 1e-9;
        bool conic = u2 > r2g * (1.0 + 1e-6) + 1e-12 && un * (1.0 + 1e-8) + 1e-12 <
                     sqrt(fma(ls.z, ls.z, fma(ls.y, ls.y, ls.x * ls.x))) && H > 1.001 * rho;
        double x0 = 0, x1 = 0, x2 = 0, y0 = 0, y1 = 0, y2 = 0, z0 = 1, z1 = 0, z2 = 0, b0 = 0, b1 = 0, b2 = 0,
               tau = 0;
        bool front = false;
        if (conic) {
            const d3 nu = mk(uc.x / un, uc.y / un, uc.z / un);
            const d3 ax = mk(lo.x / H, lo.y / H, lo.z / H);
            const double hh = fma(uc.z, ax.z, fma(uc.y, ax.y, uc.x * ax.x));
            const d3 wp = mk(fma(-ax.x, hh, uc.x), fma(-ax.y, hh, uc.y), fma(-ax.z, hh, uc.z));
            const double q = sqrt(fma(wp.z, wp.z, fma(wp.y, wp.y, wp.x * wp.x)));
            const double sin_phi = rho / H, cos_phi = sqrt(1.0 - sin_phi * sin_phi);
            front = hh * cos_phi - q * sin_phi > 1e-8 * (fabs(hh) + q) + 1e-12;
            const double sg = nu.z >= 0.0 ? 1.0 : -1.0;
            const double ia = -1.0 / (sg + nu.z);
            const double bb = nu.x * nu.y * ia;
            const d3 e1 = mk(fma(sg * nu.x * nu.x, ia, 1.0), sg * bb, -sg * nu.x);
            const d3 e2 = mk(bb, fma(nu.y * nu.y, ia, sg), -nu.y);
            const double sc = un / sqrt(r2g);
            auto dot = [](d3 a, d3 b) { return fma(a.z, b.z, fma(a.y, b.y, a.x * b.x)); };
            x0 = sc * dot(e1, lo), x1 = sc * dot(e1, bu), x2 = sc * dot(e1, bv);
            y0 = sc * dot(e2, lo), y1 = sc * dot(e2, bu), y2 = sc * dot(e2, bv);
            z0 = dot(nu, lo), z1 = dot(nu, bu), z2 = dot(nu, bv);
            b0 = dot(lo, lo), b1 = 2.0 * dot(lo, bu), b2 = 2.0 * dot(lo, bv);
            const double s = un / sqrt(g[3] > 0.0 ? g[3] : 1e-300);
            tau = 1024.0 * 2.220446049250313e-16 * (s * s + s * (1.0 + 4.0 * sa.light_radius / H) + 1.0);
            if (!(tau < 1e-3)) conic = false;  // ill-conditioned: every sample literal
        }
        // pass 1: the silhouette decisions (the band's samples counted, not decided)
        int unblocked = 0, amb = n;
        auto sil = [&](int i, double &dd, double &band, double &a, double &b) {
            const double2 t = tab2[i];
            a = t.x;
            b = t.y;
            const double w2 = fma(b1, a, fma(b2, b, b0)) + fma(a, a, b * b);
            const double x = fma(x1, a, fma(x2, b, x0)), y = fma(y1, a, fma(y2, b, y0));
            dd = fma(x, x, fma(y, y, -w2));
            band = tau * w2;
        };
        if (conic) {
            amb = 0;
#pragma unroll 4
            for (int i = part; i < n; i += kSplit) {
                double dd, band, a, b;
                sil(i, dd, band, a, b);
                const bool open = dd > band || (dd < -band && !(front || fma(z1, a, fma(z2, b, z0)) > 0.0));
                unblocked += open ? 1 : 0;
                amb += fabs(dd) <= band ? 1 : 0;
            }
        }
        // pass 2 (rare): the band's samples by the reference's literal test (renderer.py:90-103)
        if (amb) {
            for (int i = part; i < n; i += kSplit) {
                if (conic) {
                    double dd, band, a, b;
                    sil(i, dd, band, a, b);
                    if (!(fabs(dd) <= band)) continue;
                }
                const d3 s = disc_point(i, lp, bu, bv, tab);
                const d3 d = vnormalize(vsub(s, origin));
                unblocked += intersect(origin, d, g) < vdistance(surface, s) ? 0 : 1;
            }
        }
        const unsigned act = __activemask();
#pragma unroll
        for (unsigned o = 1; o < kSplit; o <<= 1) unblocked += __shfl_xor_sync(act, unblocked, o);
        if (part == 0) wa.rec[(int64_t)P.w].w = (double)unblocked / (double)n;
    }
}

// --- B2: one warp per undecided hit, the reference's shadow loop (renderer.py:82-105) ---
__global__ void __launch_bounds__(kThreads)
    fused64_sample(const FrameArgs fa, const SceneArgs<double> sa, const WaveArgs64 wa) {
    extern __shared__ double smem_geo[];
    const double *__restrict__ geo = stage(sa, smem_geo);
    if (wa.lane_cap) sample_lanes64(fa, sa, wa, geo);
    const unsigned count = wa.count[1];
    const int lane = threadIdx.x & 31;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned n_warps = (gridDim.x * blockDim.x) >> 5;
    const int n = fa.samples;
    const d3 lp = mk(sa.light[0], sa.light[1], sa.light[2]);
    for (unsigned h = warp; h < count; h += n_warps) {
        const double4 P = wa.q[2 * h], N = wa.q[2 * h + 1];
        unsigned hm[kWords64];
#pragma unroll
        for (int w = 0; w < kWords64; w++) hm[w] = wa.mask[(size_t)w * wa.mask_stride + h];
        const d3 surface = mk(P.x, P.y, P.z), normal = mk(N.x, N.y, N.z);
        const d3 origin = mk(surface.x + 1e-3 * normal.x, surface.y + 1e-3 * normal.y, surface.z + 1e-3 * normal.z);
        d3 bu, bv;
        disc_basis(surface, lp, bu, bv);
        int unblocked = 0;
        for (int i = lane; i < n; i += 32) {
            const d3 s = disc_point(i, lp, bu, bv, sa.table);
            const d3 d = vnormalize(vsub(s, origin));
            const double limit = vdistance(surface, s);
            bool blocked = false;
#pragma unroll
            for (int w = 0; w < kWords64; w++)
                for (unsigned bm = hm[w]; bm && !blocked; bm &= bm - 1)
                    blocked = intersect(origin, d, geo + 4 * (w * 32 + __ffs(bm) - 1)) < limit;
            unblocked += blocked ? 0 : 1;
        }
        unblocked = __reduce_add_sync(0xffffffffu, unblocked);
        if (lane == 0) {
            const int64_t slot = (int64_t)P.w;
            wa.rec[slot].w = (double)unblocked / (double)n;
        }
    }
}

// --- C: unwind the parked pixels -------------------------------------------------
__global__ void __launch_bounds__(kThreads)
    fused64_finish(const FrameArgs fa, const SceneArgs<double> sa, const WaveArgs64 wa) {
    const unsigned count = wa.count[2];
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const int lpix = wa.parked[i];
        const double4 px = wa.pix[lpix];
        const int info = (int)px.w;
        const d3 c = unwind(info & 0xff, (info >> 8) & 1, mk(px.x, px.y, px.z), sa,
                            [&](int k, int &idx, double &d, double &s, double &sc) {
                                const double4 r = wa.rec[(int64_t)k * wa.n_pix + lpix];
                                idx = (int)r.x;
                                d = r.y;
                                s = r.z;
                                sc = r.w;
                            });
        const int ly = lpix / fa.width, x = lpix - ly * fa.width;
        const int y = map_row(ly, fa);
        fa.out[(int64_t)y * fa.out_pitch + x] = pack_color(c.x, c.y, c.z, fa.rgba);
        if (fa.radiance) {
            double *r = (double *)fa.radiance + 3 * ((int64_t)y * fa.width + x);
            r[0] = c.x;
            r[1] = c.y;
            r[2] = c.z;
        }
        if (fa.peer_out) __threadfence_system();
    }
}

int ctas_for(const void *kernel, size_t smem) {
    static thread_local std::map<std::pair<const void *, size_t>, int> memo;
    auto key = std::make_pair(kernel, smem);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
    return memo[key] = sms * (per_sm > 0 ? per_sm : 1);
}

}  // namespace

cudaError_t rt_launch_fused_f64(const rt::FrameArgs &fa, const rt::SceneArgs<double> &sa, const rt::WaveArgs64 &wa,
                                cudaStream_t st, int *n_kernels) {
    *n_kernels = 0;
    if (sa.n > kMaxBodies64 || fa.samples < 2) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(wa.count, 0, 4 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(double) * 4 * (size_t)(sa.n > 0 ? sa.n : 1);
    dim3 grid((fa.width + kTileW - 1) / kTileW, (fa.local_rows + kTileH - 1) / kTileH);
    fused64_trace<<<grid, kThreads, smem, st>>>(fa, sa, wa);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    fused64_sample<<<ctas_for((const void *)fused64_sample, smem), kThreads, smem, st>>>(fa, sa, wa);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    fused64_finish<<<ctas_for((const void *)fused64_finish, 0), kThreads, 0, st>>>(fa, sa, wa);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *n_kernels = 3;
    return cudaSuccess;
}
