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
    if (y >= fa.row_end) return;
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

template <int MAXS>
__device__ __forceinline__ void trace_chain_bundle(const ParamScene<MAXS> &ps, const FrameArgs &fa,
                                                   const SceneArgs<float> &sa, const WaveArgs &wa, int x, int ly) {
    constexpr int kWords = (MAXS + 31) / 32;
    const int lane = threadIdx.x & 31;
    __shared__ float4 s_cand_sph[kThreads / 32][MAXS];
    __shared__ int s_cand_idx[kThreads / 32][MAXS];
    float4 *cand_sph = s_cand_sph[threadIdx.x >> 5];
    int *cand_idx = s_cand_idx[threadIdx.x >> 5];
    // the lane-parallel bundle test reads 32 different spheres at once: from
    // shared memory (constant-bank reads with divergent addresses serialise)
    __shared__ float4 s_sph[MAXS];
    __shared__ int s_idx[MAXS];
    for (int i = threadIdx.x; i < ps.ns; i += blockDim.x) {
        s_sph[i] = ps.sph[i];
        s_idx[i] = ps.sph_idx[i];
    }
    __syncthreads();
    int y = 0;
    bool alive = x < fa.width && ly < fa.local_rows;
    if (alive) {
        y = map_row(ly, fa);
        alive = y < fa.row_end;
    }
    const bool valid = alive;
    const int64_t lp = (int64_t)ly * fa.width + x;
    float3 origin = f3((float)fa.cam[0], (float)fa.cam[1], (float)fa.cam[2]);
    float3 dir = valid ? primary_direction(x, y, fa) : f3(0.f, 0.f, 1.f);
    const float3 light = f3(sa.light[0], sa.light[1], sa.light[2]);
    float3 tail = f3(0.f, 0.f, 0.f);
    int m = 0, exhausted = 0;
    for (int k = 0; k <= fa.bounces; k++) {
        const unsigned live = __ballot_sync(0xffffffffu, alive);
        if (!live) break;
        // bundle of the live rays
        float3 sd = f3(warp_sum(alive ? dir.x : 0.f), warp_sum(alive ? dir.y : 0.f), warp_sum(alive ? dir.z : 0.f));
        float sn = dot3(sd, sd);
        float3 A = sd * (sn > 0.f ? rsqrtf(sn) : 0.f);
        float cos_t = warp_min(alive ? dot3(dir, A) : 1.f);
        const float inv_n = 1.f / (float)__popc(live);
        float3 co = f3(warp_sum(alive ? origin.x : 0.f) * inv_n, warp_sum(alive ? origin.y : 0.f) * inv_n,
                       warp_sum(alive ? origin.z : 0.f) * inv_n);
        float3 dco = origin - co;
        float rho = warp_max(alive ? sqrtf(dot3(dco, dco)) : 0.f);
        const bool cull = cos_t > 0.25f && sn > 0.f;
        cos_t = fminf(cos_t * (1.f - kBoundRel), 1.f);  // widen the cone for rounding
        const float sin_t = sqrtf(fmaxf(1.f - cos_t * cos_t, 0.f));
        // compact the candidates into this warp's shared-memory list: every
        // lane then walks the same entries (broadcast LDS, unrolled)
        int ncand = 0;
#pragma unroll
        for (int w = 0; w < kWords; w++) {
            const int b = w * 32 + lane;
            const float4 g = s_sph[b < ps.ns ? b : 0];
            bool cand = b < ps.ns && (!cull || sphere_meets_bundle<MAXS>(g, co, A, cos_t, sin_t, rho));
            const unsigned bm = __ballot_sync(0xffffffffu, cand);
            if (cand) {
                const int at = ncand + __popc(bm & lanemask_lt());
                cand_sph[at] = g;
                cand_idx[at] = s_idx[b];
            }
            ncand += __popc(bm);
        }
        __syncwarp();
        if (wa.work && lane == 0) {
            atomicAdd(wa.work + kWorkTraceRays, (unsigned long long)__popc(live));
            atomicAdd(wa.work + kWorkTraceTests, (unsigned long long)__popc(live) * ncand);
            if (!cull) atomicAdd(wa.work + kWorkTraceFullWarps, 1ull);
        }
        Hit h{-1, INFINITY, make_float4(0.f, 0.f, 0.f, -1.f)};
        if (alive) {
#pragma unroll
            for (int j = 0; j < kMaxPlanes; j++) {
                if (j >= ps.np) break;
                float t = plane_t(origin, dir, ps.pl_h[j]);
                if (t < h.t || (t == h.t && ps.pl_idx[j] < h.idx)) {
                    h.t = t;
                    h.idx = ps.pl_idx[j];
                    h.g = make_float4(0.f, ps.pl_h[j], 0.f, -1.f);
                }
            }
            int best = -1;
#pragma unroll 4
            for (int c = 0; c < ncand; c++) {
                float t = sphere_t(origin, dir, cand_sph[c]);
                if (t <= h.t) {
                    int id = cand_idx[c];
                    if (t < h.t || id < h.idx) {  // (t, index) order: lowest original index wins ties
                        h.t = t;
                        h.idx = id;
                        best = c;
                    }
                }
            }
            if (best >= 0 && h.idx == cand_idx[best]) h.g = cand_sph[best];
        }
        __syncwarp();
        const bool hit_now = alive && h.idx >= 0;
        if (alive && !hit_now) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            alive = false;
        }
        int64_t slot_id = 0;
        if (hit_now) {
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
            slot_id = (int64_t)k * wa.n_pix + lp;
            wa.hit_p[slot_id] = make_float4(hit.x, hit.y, hit.z, __int_as_float(h.idx));
            wa.hit_n[slot_id] = make_float4(normal.x, normal.y, normal.z, dfs);
            wa.hit_s[slot_id] = s;
            m = k + 1;
            if (k == fa.bounces) {
                exhausted = 1;
                alive = false;
            } else {
                origin = hit + normal * 1e-3f;
                dir = dir - normal * (2.f * dot3(normal, dir));
            }
        }
        const unsigned hb = __ballot_sync(0xffffffffu, hit_now);
        unsigned base = 0;
        if (lane == 0 && hb) base = atomicAdd(wa.count, (unsigned)__popc(hb));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (hit_now) wa.queue[base + __popc(hb & lanemask_lt())] = (int)slot_id;
    }
    if (valid) wa.pix[lp] = make_float4(tail.x, tail.y, tail.z, __int_as_float(m | (exhausted << 8)));
}

template <int MAXS>
__global__ void __launch_bounds__(kThreads)
    wave_trace_param(const FrameArgs fa, const SceneArgs<float> sa, const WaveArgs wa, const ParamScene<MAXS> ps) {
    int x, ly;
    thread_pixel(x, ly);
    if constexpr (ParamScene<MAXS>::kClustered)
        trace_chain_bundle(ps, fa, sa, wa, x, ly);
    else
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
    // Control flow stays warp-uniform end to end (dead lanes of the last
    // round compute a duplicate and drop it), so the body loops inside the
    // any-hit test branch on uniform predicates only.
    extern __shared__ float4 smem_tab[];
    const float4 *__restrict__ gtab = reinterpret_cast<const float4 *>(sa.table);
    const bool tab_in_smem = n > 1 && n <= kWaveSmemSamples;
    if (tab_in_smem) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) smem_tab[i] = gtab[i];
        __syncthreads();
    }
    const unsigned count = *wa.count;
    const int lane = threadIdx.x & 31;
    const int sub = lane % LANES;
    constexpr int kHitsPerWarp = 32 / LANES;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned n_warps = (gridDim.x * blockDim.x) >> 5;
    const float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
    const int rounds = (n + LANES - 1) / LANES;
    for (unsigned base = warp * kHitsPerWarp; base < count; base += n_warps * kHitsPerWarp) {
        const unsigned q = base + lane / LANES;
        const bool live = q < count;
        const int slot = __ldg(wa.queue + (live ? q : count - 1));
        const float4 P = __ldg(wa.hit_p + slot);
        const float4 N = __ldg(wa.hit_n + slot);
        const ShadowFrame f = shadow_frame(f3(P.x, P.y, P.z), f3(N.x, N.y, N.z), lp, n > 1);
        const auto lc = geo.localize(f.origin);
        int unblocked = 0;
#pragma unroll 2
        for (int j = 0; j < rounds; j++) {
            const int i = sub + j * LANES;
            const bool valid = i < n;
            const int ic = valid ? i : 0;
            const float4 t = n == 1 ? make_float4(0.f, 0.f, 0.f, 0.f) : (tab_in_smem ? smem_tab[ic] : __ldg(gtab + ic));
            float3 dir;
            float limit;
            shadow_ray(f, t, dir, limit);
            unblocked += (valid && !geo.occluded(lc, dir, limit)) ? 1 : 0;
        }
#pragma unroll
        for (int o = LANES / 2; o > 0; o >>= 1) unblocked += __shfl_xor_sync(0xffffffffu, unblocked, o);
        if (live && sub == 0) wa.hit_sc[slot] = (float)unblocked / (float)n;
    }
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
// body in the penumbra test rays, and only against those bodies.
//
// One warp per hit (hits taken from an atomic counter — their costs now
// differ): lanes test one body each for the cull, then take the samples
// lane, lane + 32, ... against the surviving bodies (a warp-uniform mask).
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

// Two kernels:
//  B1  one lane per hit classifies every body (a few instructions per hit);
//      decided hits (nothing can block: 1, something blocks all: 0) are
//      written at once, undecided ones go to a second queue with their
//      body mask (warp-aggregated append);
//  B2  one warp per undecided hit, 32 samples abreast, against that hit's
//      surviving bodies only — every queued hit costs the same, so a static
//      stride keeps the SMs evenly loaded.
template <int MAXS>
__global__ void __launch_bounds__(kThreads)
    wave_cull_classify(const SceneArgs<float> sa, const WaveArgs wa, const ParamScene<MAXS> ps) {
    constexpr int kWords = (MAXS + 31) / 32;  // sphere mask words; one more word for planes
    const unsigned count = *wa.count;
    const int lane = threadIdx.x & 31;
    const float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < count; base += stride) {
        const unsigned q = base + lane;
        const bool live = q < count;
        int slot = 0;
        unsigned mask[kWords + 1];
#pragma unroll
        for (int w = 0; w <= kWords; w++) mask[w] = 0;
        bool full = false, any = false;
        if (live) {
            slot = __ldg(wa.queue + q);
            const float4 P = __ldg(wa.hit_p + slot);
            const float4 N = __ldg(wa.hit_n + slot);
            const float3 origin = f3(P.x, P.y, P.z) + f3(N.x, N.y, N.z) * 1e-3f;
            const Cone k = make_cone(origin, lp, sa.light_radius);
            auto classify = [&](int b) {
                int cls = sphere_class(k, ps.sph[b], ps.sph_rad[b]);  // b warp-uniform: constant-cache broadcast
                mask[b >> 5] |= (cls == 1 ? 1u : 0u) << (b & 31);
                full |= cls == 2;
            };
            if constexpr (!ParamScene<MAXS>::kClustered) {
#pragma unroll
                for (int b = 0; b < MAXS; b++) {
                    if (b >= ps.ns) break;
                    classify(b);
                }
            } else {
                for (int c = 0; c < ps.nc; c++) {
                    if (!bound_meets_cone(k, ps.cl[c])) continue;
                    for (int b = ps.cl_begin[c]; b < ps.cl_begin[c + 1]; b++) classify(b);
                }
            }
#pragma unroll
            for (int j = 0; j < kMaxPlanes; j++) {
                if (j >= ps.np) break;
                int cls = plane_class(k, origin.y, lp.y, ps.pl_h[j]);
                mask[kWords] |= (cls == 1 ? 1u : 0u) << j;
                full |= cls == 2;
            }
#pragma unroll
            for (int w = 0; w <= kWords; w++) any |= mask[w] != 0;
            if (full || !any) wa.hit_sc[slot] = full ? 0.f : 1.f;
        }
        const bool need = live && !full && any;
        const unsigned nb = __ballot_sync(0xffffffffu, need);
        unsigned base2 = 0;
        if (lane == 0 && nb) base2 = atomicAdd(wa.count + 1, (unsigned)__popc(nb));
        base2 = __shfl_sync(0xffffffffu, base2, 0);
        if (need) {
            const unsigned e = base2 + __popc(nb & lanemask_lt());
            wa.queue2[e] = slot;
#pragma unroll
            for (int w = 0; w <= kWords; w++) wa.mask2[(size_t)w * wa.mask2_stride + e] = mask[w];
        }
        if (wa.work) {
            unsigned nl = __popc(__ballot_sync(0xffffffffu, live));
            if (lane == 0) {
                atomicAdd(wa.work + kWorkHits, (unsigned long long)nl);
                atomicAdd(wa.work + kWorkCullTests, (unsigned long long)nl * (ps.ns + ps.np));
            }
        }
    }
}

// The sampling loop of an undecided hit: up to kRegCand candidate spheres
// (and the candidate planes) are held in registers as L = c - o and r^2
// (+graze, or -inf if o is inside), uniform across the warp; a hit with more
// candidates walks them kRegCand at a time, OR-ing each sample's verdict
// into a per-lane bit set (one bit per round).
constexpr int kRegCand = 4;

template <int MAXS, bool SMEM_TAB>
__device__ __forceinline__ void cull_sample_hit(const ParamScene<MAXS> &ps, const SceneArgs<float> &sa,
                                                const WaveArgs &wa, int n, unsigned h, const float4 *tab) {
    constexpr int kWords = (MAXS + 31) / 32;
    const int lane = threadIdx.x & 31;
    const float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
    const int rounds = (n + 31) / 32;
    const int hslot = __ldg(wa.queue2 + h);
    unsigned hm[kWords + 1];
    int nsph = 0;
#pragma unroll
    for (int w = 0; w <= kWords; w++) {
        hm[w] = __ldg(wa.mask2 + (size_t)w * wa.mask2_stride + h);
        if (w < kWords) nsph += __popc(hm[w]);
    }
    const float4 P = __ldg(wa.hit_p + hslot);
    const float4 N = __ldg(wa.hit_n + hslot);
    const ShadowFrame f = shadow_frame(f3(P.x, P.y, P.z), f3(N.x, N.y, N.z), lp, n > 1);
    int unblocked = 0;
    if (nsph == 1 && hm[kWords] == 0) {
        // the common penumbra case: one sphere against every sample; full
        // rounds of 32 samples without bounds checks, then the remainder
        static_assert(kWaveMinSamples > 1, "the wavefront path assumes soft shadows");
        int w = 0;
        while (hm[w] == 0) w++;
        const float4 g = ps.sph[w * 32 + __ffs(hm[w]) - 1];
        const float3 L = f3(g.x - f.origin.x, g.y - f.origin.y, g.z - f.origin.z);
        const float r2g = sphere_r2g(L, g.w);
        auto sample = [&](int i) -> int {
            float4 t;
            if constexpr (SMEM_TAB) {
                extern __shared__ float4 smem_tab_s[];
                t = smem_tab_s[i];
            } else {
                t = __ldg(tab + i);
            }
            float3 dir;
            float limit;
            shadow_ray_unguarded(f, t, dir, limit);
            return sphere_margin_L(L, dir, r2g, limit) > 0.f ? 0 : 1;
        };
        const int full = n >> 5;
#pragma unroll 2
        for (int j = 0; j < full; j++) unblocked += sample(lane + 32 * j);
        if (lane + 32 * full < n) unblocked += sample(lane + 32 * full);
    } else if (nsph <= kRegCand) {
        // up to kRegCand spheres (+ planes): one pass, counted directly
        float4 c[kRegCand];
        int k = 0, w = 0;
        unsigned mw = hm[0];
#pragma unroll
        for (int r = 0; r < kRegCand; r++) {
            c[r] = make_float4(0.f, 0.f, 0.f, -INFINITY);
            while (mw == 0 && w + 1 < kWords) mw = hm[++w];
            if (mw != 0) {
                const float4 g = ps.sph[w * 32 + __ffs(mw) - 1];
                mw &= mw - 1;
                const float3 L = f3(g.x - f.origin.x, g.y - f.origin.y, g.z - f.origin.z);
                c[r] = make_float4(L.x, L.y, L.z, sphere_r2g(L, g.w));
                k++;
            }
        }
        const unsigned pm = hm[kWords];
        for (int j = 0; j < rounds; j++) {
            const int i = lane + 32 * j;
            const int ic = i < n ? i : 0;
            const float4 t = n == 1 ? make_float4(0.f, 0.f, 0.f, 0.f) : (SMEM_TAB ? tab[ic] : __ldg(tab + ic));
            float3 dir;
            float limit;
            shadow_ray(f, t, dir, limit);
            float m = -INFINITY;
#pragma unroll
            for (int r = 0; r < kRegCand; r++)
                if (r < k) m = fmaxf(m, sphere_margin_L(f3(c[r].x, c[r].y, c[r].z), dir, c[r].w, limit));
            for (unsigned b = pm; b; b &= b - 1)
                m = fmaxf(m, plane_margin(ps.pl_h[__ffs(b) - 1] - f.origin.y, dir.y, limit));
            unblocked += (i < n && !(m > 0.f)) ? 1 : 0;
        }
    } else
    // rounds in groups of 64 (a bit per round); candidates kRegCand at a time
    for (int g0 = 0; g0 < rounds; g0 += 64) {
        const int g1 = min(rounds, g0 + 64);
        unsigned long long blocked = 0;  // bit j - g0: sample lane + 32 j is blocked
        int w_cur = 0;
        unsigned m_cur = hm[0];
        for (int done = 0; done < nsph || done == 0; done += kRegCand) {
            float4 c[kRegCand];
            int k = 0;
#pragma unroll
            for (int r = 0; r < kRegCand; r++) {
                c[r] = make_float4(0.f, 0.f, 0.f, -INFINITY);
                while (m_cur == 0 && w_cur + 1 < kWords) m_cur = hm[++w_cur];
                if (m_cur != 0) {
                    const float4 g = ps.sph[w_cur * 32 + __ffs(m_cur) - 1];
                    m_cur &= m_cur - 1;
                    const float3 L = f3(g.x - f.origin.x, g.y - f.origin.y, g.z - f.origin.z);
                    c[r] = make_float4(L.x, L.y, L.z, sphere_r2g(L, g.w));
                    k++;
                }
            }
            const unsigned pm = done == 0 ? hm[kWords] : 0u;  // planes ride with the first chunk
            for (int j = g0; j < g1; j++) {
                const int i = lane + 32 * j;
                const int ic = i < n ? i : 0;
                const float4 t = n == 1 ? make_float4(0.f, 0.f, 0.f, 0.f) : (SMEM_TAB ? tab[ic] : __ldg(tab + ic));
                float3 dir;
                float limit;
                shadow_ray(f, t, dir, limit);
                float m = -INFINITY;
#pragma unroll
                for (int r = 0; r < kRegCand; r++)
                    if (r < k) m = fmaxf(m, sphere_margin_L(f3(c[r].x, c[r].y, c[r].z), dir, c[r].w, limit));
                for (unsigned b = pm; b; b &= b - 1)
                    m = fmaxf(m, plane_margin(ps.pl_h[__ffs(b) - 1] - f.origin.y, dir.y, limit));
                if (m > 0.f) blocked |= 1ull << (j - g0);
            }
            if (nsph <= kRegCand) break;
        }
        for (int j = g0; j < g1; j++) unblocked += (lane + 32 * j < n && !((blocked >> (j - g0)) & 1ull)) ? 1 : 0;
    }
    unblocked = __reduce_add_sync(0xffffffffu, unblocked);
    if (lane == 0) {
        wa.hit_sc[hslot] = (float)unblocked / (float)n;
        if (wa.work) {
            atomicAdd(wa.work + kWorkSampledHits, 1ull);
            atomicAdd(wa.work + kWorkShadowRays, (unsigned long long)n);
            atomicAdd(wa.work + kWorkSphereTests, (unsigned long long)n * nsph);
            atomicAdd(wa.work + kWorkPlaneTests, (unsigned long long)n * __popc(hm[kWords]));
        }
    }
}

template <int MAXS, bool SMEM_TAB>
__global__ void __launch_bounds__(kThreads)
    wave_cull_sample(const SceneArgs<float> sa, const WaveArgs wa, int n, const ParamScene<MAXS> ps) {
    extern __shared__ float4 smem_tab[];
    const float4 *tab = reinterpret_cast<const float4 *>(sa.table);
    if constexpr (SMEM_TAB) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) smem_tab[i] = tab[i];
        __syncthreads();
        tab = smem_tab;
    }
    const unsigned count = wa.count[1];
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned n_warps = (gridDim.x * blockDim.x) >> 5;
    for (unsigned h = warp; h < count; h += n_warps) cull_sample_hit<MAXS, SMEM_TAB>(ps, sa, wa, n, h, tab);
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
    if (y >= fa.row_end) return;
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

template <int MAXS>
cudaError_t launch_cull(const SceneArgs<float> &sa, const WaveArgs &wa, int n, cudaStream_t st,
                        const ParamScene<MAXS> &ps, cudaEvent_t *ev) {
    size_t smem = n <= kWaveSmemSamples ? sizeof(float4) * (size_t)n : 0;
    static thread_local int ctas_c = 0;
    if (!ctas_c) ctas_c = resident_ctas(wave_cull_classify<MAXS>, 0);
    wave_cull_classify<MAXS><<<ctas_c, kThreads, 0, st>>>(sa, wa, ps);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[2], st);
    if (n > 1 && n <= kWaveSmemSamples) {
        int ctas = resident_ctas(wave_cull_sample<MAXS, true>, smem);  // depends on the table size
        wave_cull_sample<MAXS, true><<<ctas, kThreads, smem, st>>>(sa, wa, n, ps);
    } else {
        static thread_local int ctas = 0;
        if (!ctas) ctas = resident_ctas(wave_cull_sample<MAXS, false>, 0);
        wave_cull_sample<MAXS, false><<<ctas, kThreads, 0, st>>>(sa, wa, n, ps);
    }
    e = cudaGetLastError();
    if (ev) cudaEventRecord(ev[3], st);
    return e;
}

template <int LANES>
cudaError_t launch_shadow(const SceneArgs<float> &sa, const WaveArgs &wa, int n, cudaStream_t st, bool param8,
                          const ParamScene<8> &p8, bool param256, const ParamScene<kParamSpheres> &p256) {
    size_t smem = (n > 1 && n <= kWaveSmemSamples) ? sizeof(float4) * (size_t)n : 0;
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
                               cudaStream_t st, int *n_kernels, cudaEvent_t *ev) {
    *n_kernels = 0;
    cudaError_t e = cudaMemsetAsync(wa.count, 0, 4 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    auto mark = [&](int i) {
        if (ev) cudaEventRecord(ev[i], st);
    };
    mark(0);
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
    *n_kernels = 1;
    mark(1);
    if (wa.cull && (param8 || param256)) {
        e = param8 ? launch_cull(sa, wa, fa.samples, st, p8, ev) : launch_cull(sa, wa, fa.samples, st, p256, ev);
        if (e != cudaSuccess) return e;
        *n_kernels += 2;
        wave_shade<<<grid, kThreads, 0, st>>>(fa, sa, wa);
        *n_kernels += 1;
        mark(4);
        return cudaGetLastError();
    }
    mark(2);
    switch (rt_wave_lanes(fa.samples)) {
        case 1: e = launch_shadow<1>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        case 2: e = launch_shadow<2>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        case 4: e = launch_shadow<4>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        case 8: e = launch_shadow<8>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        case 16: e = launch_shadow<16>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
        default: e = launch_shadow<32>(sa, wa, fa.samples, st, param8, p8, param256, p256); break;
    }
    if (e != cudaSuccess) return e;
    mark(3);
    wave_shade<<<grid, kThreads, 0, st>>>(fa, sa, wa);
    *n_kernels = 3;
    mark(4);
    return cudaGetLastError();
}
