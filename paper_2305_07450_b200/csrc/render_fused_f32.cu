// FP32 soft shadows with exact occluder culling — the default product path
// for shadow_samples >= kWaveMinSamples.  Two kernels per frame:
//
//   A  trace   one thread per pixel: the bounce chain (closest hit,
//              geometry.py:191-201; a warp ray-bundle candidate list in scenes
//              of more than 8 spheres), per hit the Lambert and Blinn factors
//              (shading.py:53-73) and the exact classification of every body
//              against the hit's shadow cone (rt_wave.cuh): nothing can block
//              -> coefficient 1, something blocks every sample -> 0, else the
//              hit is queued.  A pixel whose hits are all decided is unwound
//              (renderer.py:185-224) and packed (renderer.py:45-50) right
//              here; otherwise its records are parked in HBM.
//   B  sample  B1: hits with a single candidate sphere, one lane each (two
//              lane queues: sphere wholly in front of the hit / not), every
//              lane on the same disc sample at once; B2: the rest, one warp
//              per hit, 32 samples abreast against its candidates.  The
//              sampler of a pixel's last pending hit unwinds and packs it.
//
// A penumbra sphere is tested in its silhouette form (rt_wave.cuh,
// conic_coeffs: six coefficients per hit and sphere, a quadratic per sample)
// when its preconditions hold, else — and everywhere with option "conic" off
// — in the ray form, operation for operation the unculled kernels'
// (render_wave_f32.cu), whose frames the culled ones then equal bit for bit.
//
// HBM, slot = bounce * n_pix + local pixel:
//   lane_q  {p, record slot}, {n, candidate sphere}       the two lane queues
//   hit_p   {p, slot} or {|lo|^2, 2 lo.bu, 2 lo.bv, slot}  the warp queue (ray / silhouette form)
//   hit_n   {n, silhouette code}, masks word-major, conic coefficients [2j][e]
//   rec     float4 {body, Lambert, Blinn, coefficient}   every hit of a parked pixel
//   pix     float4 {tail rgb, records | exhausted << 8 | several pending << 9}
//   pend    per parked pixel with several pending hits: the countdown
#include "rt_wave.cuh"
#include <cuda/atomic>

namespace {
using namespace rt;
using namespace rt32;

constexpr int kRegCand = 4;  // candidate spheres a sampling warp keeps in registers

// --- the shadow grid ------------------------------------------------------------
// A box around the spheres is cut into kGridCells cells.  A hit's shadow
// segments leave o toward the disc (within 2R of L) and stop at most 1e-3
// beyond it; for every o in a cell (within rb of its centre cc) they lie within
// rb of the cone from cc (half-angle asin(rho / (H - rb)), axial reach
// T (H + rb + rho) with T formed with H - rb - rho): o + t (s - o) =
// cc + t (s - cc) + (1 - t)(o - cc).  An occluder bound clear of that dilated
// cone (sphere_class's outside tests, margins included) cannot meet the cone of
// any hit in the cell, so its bit is clear in the cell's mask.  Hits outside
// the box, or in a cell whose cone degenerates, classify every body.  The
// grid depends on the scene and the light only (rt_host.cu rebuilds it when
// either changes).
__device__ __forceinline__ unsigned grid_mask(const WaveArgs &wa, float3 o) {
    if (!wa.grid) return ~0u;
    const int ix = __float2int_rd((o.x - wa.grid_lo[0]) * wa.grid_inv[0]);
    const int iy = __float2int_rd((o.y - wa.grid_lo[1]) * wa.grid_inv[1]);
    const int iz = __float2int_rd((o.z - wa.grid_lo[2]) * wa.grid_inv[2]);
    if ((unsigned)ix >= (unsigned)wa.grid_dim[0] || (unsigned)iy >= (unsigned)wa.grid_dim[1] ||
        (unsigned)iz >= (unsigned)wa.grid_dim[2])
        return ~0u;
    return __ldg(wa.grid + ((size_t)iz * wa.grid_dim[1] + iy) * wa.grid_dim[0] + ix);
}

template <int MAXS>
__global__ void __launch_bounds__(kThreads)
    shadow_grid_build(const ParamScene<MAXS> ps, const SceneArgs<float> sa, const WaveArgs wa, unsigned *out) {
    const int n_cells = wa.grid_dim[0] * wa.grid_dim[1] * wa.grid_dim[2];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_cells) return;
    const int ix = i % wa.grid_dim[0], iy = (i / wa.grid_dim[0]) % wa.grid_dim[1];
    const int iz = i / (wa.grid_dim[0] * wa.grid_dim[1]);
    const float3 cell = f3(1.f / wa.grid_inv[0], 1.f / wa.grid_inv[1], 1.f / wa.grid_inv[2]);
    const float3 cc = f3(wa.grid_lo[0] + (ix + 0.5f) * cell.x, wa.grid_lo[1] + (iy + 0.5f) * cell.y,
                         wa.grid_lo[2] + (iz + 0.5f) * cell.z);
    // the cell's points lie within rb of cc (the float cell edges add ~1e-6 relative)
    const float rb = 0.5f * sqrtf(dot3(cell, cell)) * (1.f + kCullRel) + kCullAbs +
                     1e-6f * (fabsf(cc.x) + fabsf(cc.y) + fabsf(cc.z));
    const float3 light = f3(sa.light[0], sa.light[1], sa.light[2]);
    const float rho = 2.f * sa.light_radius * (1.f + kCullRel) + kCullAbs;
    const float3 A = light - cc;
    const float H = sqrtf(dot3(A, A));
    if (!(H - rb > rho / 0.999f)) {
        out[i] = ~0u;
        return;
    }
    const float3 axis = A * (1.f / H);
    const float sin_phi = fminf(rho / (H - rb), 1.f);
    const float cos_phi = sqrtf(fmaxf(1.f - sin_phi * sin_phi, 0.f));
    const float T = 1.f + (1e-3f + kCullAbs) / fmaxf(H - rb - rho, 1e-6f);
    const float reach = T * (H + rb + rho) * (1.f + kCullRel) + kCullAbs;
    constexpr bool kClustered = ParamScene<MAXS>::kClustered;
    const int n_occ = kClustered ? ps.nc : ps.ns;
    unsigned m = 0;
    for (int b = 0; b < n_occ && b < 32; b++) {
        float4 g;
        if constexpr (kClustered) {
            g = ps.cl[b];
        } else {
            g = make_float4(ps.sph[b].x, ps.sph[b].y, ps.sph[b].z, ps.sph_rad[b].y);
        }
        const float3 u = f3(g.x - cc.x, g.y - cc.y, g.z - cc.z);
        const float h = dot3(u, axis);
        const float3 w = u - axis * h;
        const float q = sqrtf(dot3(w, w));
        const float rp = (g.w + rb) * (1.f + kCullRel) + kCullAbs + 1e-6f * (fabsf(h) + q + H);
        bool cand;
        if (h < -rp || h - rp > reach) {
            cand = false;
        } else if (h * cos_phi + q * sin_phi >= 0.f) {
            cand = q * cos_phi - h * sin_phi < rp;
        } else {
            cand = dot3(u, u) < rp * rp;
        }
        m |= (cand ? 1u : 0u) << b;
    }
    out[i] = m;
}

// Classify every body against one hit's shadow cone (a single lane); spheres
// (clusters, in clustered scenes) outside the shadow grid's mask wm for the
// hit's cell are skipped: they cannot meet the cone.
// Returns 0 (nothing can block), 2 (a body blocks every sample) or 1
// (undecided; mask[] holds the candidates: sphere slots in words
// 0..kWords-1, planes in word kWords).
template <int MAXS>
__device__ __forceinline__ int classify_hit(const ParamScene<MAXS> &ps, const Cone &k, float oy, float ly,
                                            unsigned *mask, bool check, unsigned wm) {
    constexpr int kWords = (MAXS + 31) / 32;
#pragma unroll
    for (int w = 0; w <= kWords; w++) mask[w] = 0;
    if (__builtin_expect(check, 0)) {  // option cull_check: every body undecided
#pragma unroll 1
        for (int b = 0; b < ps.ns; b++) mask[b >> 5] |= 1u << (b & 31);
        mask[kWords] = (1u << ps.np) - 1u;
        return ps.ns + ps.np > 0 ? 1 : 0;
    }
    bool full = false;
    auto classify = [&](int b) {
        int cls = sphere_class(k, ps.sph[b], ps.sph_rad[b]);
        mask[b >> 5] |= (cls == 1 ? 1u : 0u) << (b & 31);
        full |= cls == 2;
    };
    if constexpr (!ParamScene<MAXS>::kClustered) {
#pragma unroll
        for (int b = 0; b < MAXS; b++) {
            if (b >= ps.ns) break;
            if ((wm >> b) & 1u) classify(b);  // wm: the shadow grid's cell mask
        }
    } else {
        for (int c = 0; c < ps.nc; c++) {
            if (!((wm >> c) & 1u) || !bound_meets_cone(k, ps.cl[c])) continue;
            for (int b = ps.cl_begin[c]; b < ps.cl_begin[c + 1]; b++) classify(b);
        }
    }
#pragma unroll(kPlaneUnroll)
    for (int j = 0; j < ps.np; j++) {
        int cls = plane_class(k, oy, ly, ps.pl_h[j]);
        mask[kWords] |= (cls == 1 ? 1u : 0u) << j;
        full |= cls == 2;
    }
    if (full) return 2;
    bool any = false;
#pragma unroll
    for (int w = 0; w <= kWords; w++) any |= mask[w] != 0;
    return any ? 1 : 0;
}

// The silhouette form for queue entry e (rt_wave.cuh, conic_coeffs): when
// every candidate is a sphere (at most kConic) whose preconditions hold, sphere
// j's coefficients go to wa.conic[2j][e], [2j+1][e] and qp becomes
// {|lo|^2, 2 lo.bu, 2 lo.bv, record slot}.  Returns the entry code
//   spheres | z-tested spheres << 3 | spheres with z0 = -1 << 7
// or 0 (qp untouched: the sampler takes the ray form).
template <int MAXS>
__device__ __forceinline__ int conic_entry(const ParamScene<MAXS> &ps, const WaveArgs &wa, unsigned e,
                                           const unsigned *mask, float4 &qp, float4 qn, float3 light,
                                           float light_radius) {
    constexpr int kWords = (MAXS + 31) / 32;
    if (mask[kWords] != 0) return 0;  // a plane candidate
    int nc = 0;
#pragma unroll
    for (int w = 0; w < kWords; w++) nc += __popc(mask[w]);
    if (nc > kConic) return 0;
    // the hit's shadow frame exactly as the sampler forms it (shadow_frame)
    const ShadowFrame f = shadow_frame(f3(qp.x, qp.y, qp.z), f3(qn.x, qn.y, qn.z), light, true);
    const Cone k = make_cone(f.origin, light, light_radius);
    int j = 0, code = nc;
    for (int w = 0; w < kWords; w++) {
        for (unsigned m = mask[w]; m; m &= m - 1, j++) {
            float4 ca, cb;
            const int r = conic_coeffs(k, ps.sph[w * 32 + __ffs(m) - 1], f.lo, f.bu, f.bv, f.ls2, ca, cb);
            if (r == 0) return 0;
            if (r >= 2) code |= 1 << (3 + j);
            if (r == 3) code |= 1 << (7 + j);
            wa.conic[(size_t)(2 * j) * wa.conic_cap + e] = ca;
            wa.conic[(size_t)(2 * j + 1) * wa.conic_cap + e] = cb;
        }
    }
    qp = make_float4(dot3(f.lo, f.lo), 2.f * dot3(f.lo, f.bu), 2.f * dot3(f.lo, f.bv), qp.w);
    return code;
}

// A pixel's pending counts in one 64-bit word (resolve_hit): four 16-bit
// fields, one per bounce, each holding an unblocked count + 1
__device__ __forceinline__ bool packed_counts(const FrameArgs &fa) { return fa.bounces <= 3 && fa.samples <= 65534; }

// CTA-level compaction of the many-sphere trace's live rays: frames of at
// least kCompactMinBounces bounces, from bounce kCompactFrom on
constexpr int kCompactMinBounces = 4;
constexpr int kCompactFrom = 2;

// --- A ----------------------------------------------------------------------------
// 8 resident CTAs (64 registers) for unclustered scenes: 1.5-3.5% faster at
// C2-C4; the clustered variant needs its registers (6 CTAs; 8 costs C5 10%)
#ifndef RT_TRACE_MIN_BLOCKS
#define RT_TRACE_MIN_BLOCKS 8  // 7 (72 registers): 2-3% slower; 9 (56, spills): equal
#endif
template <int MAXS>
__global__ void __launch_bounds__(kThreads, MAXS <= 8 ? RT_TRACE_MIN_BLOCKS : 6)
    fused_trace(const FrameArgs fa, const SceneArgs<float> sa, const WaveArgs wa, const ParamScene<MAXS> ps) {
    constexpr int kWords = (MAXS + 31) / 32;
    constexpr bool kBundle = ParamScene<MAXS>::kClustered;
    // per-warp candidate lists hold at most 256 spheres: larger scenes build and
    // test them in chunks of 8 mask words (the (t, index) order survives it)
    constexpr int kCandCap = kBundle ? (MAXS < 256 ? MAXS : 256) : 1;
    constexpr int kChunkWords = kCandCap / 32 > 0 ? kCandCap / 32 : 1;
    const int lane = threadIdx.x & 31;
    // many-sphere scenes: spheres staged in shared memory for the lane-parallel
    // bundle test, and a per-warp candidate list (see trace_chain_bundle)
    __shared__ float4 s_sph[kBundle ? MAXS : 1];
    __shared__ int s_idx[kBundle ? MAXS : 1];
    __shared__ float4 s_cand_sph[kThreads / 32][kCandCap];
    __shared__ int s_cand_idx[kThreads / 32][kCandCap];
    if constexpr (kBundle) {
        for (int i = threadIdx.x; i < ps.ns; i += blockDim.x) {
            s_sph[i] = ps.sph[i];
            s_idx[i] = ps.sph_idx[i];
        }
        __syncthreads();
    }
    float4 *cand_sph = s_cand_sph[threadIdx.x >> 5];
    int *cand_idx = s_cand_idx[threadIdx.x >> 5];
    // launched with programmatic dependent launch: the previous frame's
    // sampler may still be draining; nothing global is touched before it is done
    cudaGridDependencySynchronize();
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < 8) wa.count_next[threadIdx.x] = 0;

    int x, ly;
    thread_pixel_hot_first(wa.hot, wa.hot_div, x, ly);
    int y = 0;
    bool alive = x < fa.width && ly < fa.local_rows;
    if (alive) {
        y = map_row(ly, fa);
        alive = y < fa.row_end;
    }
    // many-sphere scenes with deep bounces: the CTA's live rays are packed
    // into its first warps between bounces (ray state through shared memory,
    // bounce records in HBM, a pixel finished the moment its ray ends), so a
    // bounce of a few surviving rays costs one warp, not four (C5 at b8:
    // 6 live lanes per warp from bounce 4 on)
    constexpr bool kCompact = kBundle;
    const bool compact = kCompact && fa.bounces >= kCompactMinBounces && wa.compact;
    bool valid = alive;
    int64_t lp = (int64_t)ly * fa.width + x;
    const float3 light = f3(sa.light[0], sa.light[1], sa.light[2]);
    // the ray chain in float64 (rt_f32.cuh: refine_hit), searched in FP32
    D3 o64{fa.cam[0], fa.cam[1], fa.cam[2]};
    D3 d64 = valid ? primary_direction64(x, y, fa) : D3{0.0, 0.0, 1.0};
    float3 tail = f3(0.f, 0.f, 0.f);
    int m = 0, exhausted = 0, pmask = 0;  // pmask bit k: bounce k's hit is queued
    int ridx[kCompact ? 1 : kMaxBounce + 1];
    float rdfs[kCompact ? 1 : kMaxBounce + 1], rs[kCompact ? 1 : kMaxBounce + 1], rsc[kCompact ? 1 : kMaxBounce + 1];
    // a pixel whose ray has ended: unwound and packed, or parked for the sampler
    auto finish = [&]() {
        if (pmask == 0) {
            const float3 c = kCompact ? unwind(m, exhausted, tail, sa, [&](int k) {
                const float4 r = __ldcg(wa.rec + (int64_t)k * wa.n_pix + lp);
                return Record{__float_as_int(r.x), r.y, r.z, r.w};
            })
                                      : unwind(m, exhausted, tail, sa,
                                               [&](int k) { return Record{ridx[k], rdfs[k], rs[k], rsc[k]}; });
            store_pixel(fa, x, y, c);
            if (fa.peer_out) __threadfence_system();
        } else {
            // parked: the sampler of its last pending hit unwinds it (resolve_hit)
            const bool several = (pmask & (pmask - 1)) != 0;
            const bool packed = packed_counts(fa);
            wa.pix[lp] = make_float4(tail.x, tail.y, tail.z,
                                     __int_as_float(m | (exhausted << 8) | (several << 9) | (packed ? pmask << 10 : 0)));
            if (several) {
                if (packed) {
                    wa.pend64[lp] = 0ull;
                } else {
                    wa.pend[lp] = __popc(pmask);
                }
            }
            if constexpr (!kCompact) {
#pragma unroll 2
                for (int k = 0; k < m; k++)
                    wa.rec[(int64_t)k * wa.n_pix + lp] = make_float4(__int_as_float(ridx[k]), rdfs[k], rs[k], rsc[k]);
            }
        }
    };
    __shared__ int s_wlive[kCompact ? kThreads / 32 : 1];
    for (int k = 0; k <= fa.bounces; k++) {
        if constexpr (kCompact) {
            if (compact) {
                // the CTA loops in step (its barriers); done when no ray lives
                const unsigned wl = __ballot_sync(0xffffffffu, alive);
                if (lane == 0) s_wlive[threadIdx.x >> 5] = __popc(wl);
                const int n_live = __syncthreads_count(alive);
                if (n_live == 0) break;
                int busy = 0, base = 0;
#pragma unroll
                for (int w = 0; w < kThreads / 32; w++) {
                    busy += s_wlive[w] > 0;
                    base += w < (int)(threadIdx.x >> 5) ? s_wlive[w] : 0;
                }
                if (k >= kCompactFrom && busy > (n_live + 31) / 32) {
                    // pack: live ray i -> thread i (the candidate lists' shared memory as scratch)
                    double *st = reinterpret_cast<double *>(&s_cand_sph[0][0]);
                    int *sti = reinterpret_cast<int *>(st + 6 * kThreads);
                    if (alive) {
                        const int i = base + __popc(wl & lanemask_lt());
                        st[6 * i] = o64.x;
                        st[6 * i + 1] = o64.y;
                        st[6 * i + 2] = o64.z;
                        st[6 * i + 3] = d64.x;
                        st[6 * i + 4] = d64.y;
                        st[6 * i + 5] = d64.z;
                        sti[4 * i] = (int)lp;  // < 2^31 (slots_fit); x and y follow from it
                        sti[4 * i + 2] = m;
                        sti[4 * i + 3] = pmask;
                    }
                    __syncthreads();
                    alive = (int)threadIdx.x < n_live;
                    if (alive) {
                        const int i = threadIdx.x;
                        o64 = D3{st[6 * i], st[6 * i + 1], st[6 * i + 2]};
                        d64 = D3{st[6 * i + 3], st[6 * i + 4], st[6 * i + 5]};
                        lp = sti[4 * i];
                        const int ly_i = (int)(lp / fa.width);
                        x = (int)(lp - (int64_t)ly_i * fa.width);
                        y = map_row(ly_i, fa);
                        m = sti[4 * i + 2];
                        pmask = sti[4 * i + 3];
                        exhausted = 0;
                        tail = f3(0.f, 0.f, 0.f);
                    }
                    valid = alive;  // a thread without a ray has no pixel left to finish
                    __syncthreads();  // the scratch is the candidate lists again
                }
            }
        }
        const unsigned live = __ballot_sync(0xffffffffu, alive);
        if (!compact && !live) break;
        const bool was_alive = alive;
        const float3 origin = rnd(o64), dir = rnd(d64);
        Hit h{-1, INFINITY, make_float4(0.f, 0.f, 0.f, -1.f)};
        if constexpr (!kBundle) {
            // (the primary-ray sphere boxes cost this kernel ~4%: its unrolled,
            // branch-free sphere loop keeps more rays in flight)
            if (alive) h = ps.closest(origin, dir);
        } else if (live) {  // (compacting: a warp with no ray left idles through the bounce)
            // warp bundle of the live rays -> uniform candidate list
            float3 sd = f3(warp_sum(alive ? dir.x : 0.f), warp_sum(alive ? dir.y : 0.f),
                           warp_sum(alive ? dir.z : 0.f));
            float sn = dot3(sd, sd);
            float3 A = sd * (sn > 0.f ? rsqrtf(sn) : 0.f);
            float cos_t = warp_min(alive ? dot3(dir, A) : 1.f);
            const float inv_n = 1.f / (float)__popc(live);
            float3 co = f3(warp_sum(alive ? origin.x : 0.f) * inv_n, warp_sum(alive ? origin.y : 0.f) * inv_n,
                           warp_sum(alive ? origin.z : 0.f) * inv_n);
            float3 dco = origin - co;
            float rho = warp_max(alive ? sqrtf(dot3(dco, dco)) : 0.f);
            const bool cull = cos_t > 0.25f && sn > 0.f;
            cos_t = fminf(cos_t * (1.f - kBoundRel), 1.f);
            const float sin_t = sqrtf(fmaxf(1.f - cos_t * cos_t, 0.f));
            if (alive) {
#pragma unroll(kPlaneUnroll)
                for (int j = 0; j < ps.np; j++) {
                    float t = plane_t(origin, dir, ps.pl_h[j]);
                    if (t < h.t || (t == h.t && ps.pl_idx[j] < h.idx)) {
                        h.t = t;
                        h.idx = ps.pl_idx[j];
                        h.g = make_float4(0.f, ps.pl_h[j], 0.f, -1.f);
                    }
                }
            }
            for (int w0 = 0; w0 < kWords; w0 += kChunkWords) {
                int ncand = 0;
#pragma unroll
                for (int w = w0; w < w0 + kChunkWords; w++) {
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
                    if (w0 == 0) atomicAdd(wa.work + kWorkTraceRays, (unsigned long long)__popc(live));
                    atomicAdd(wa.work + kWorkTraceTests, (unsigned long long)__popc(live) * ncand);
                    if (!cull && w0 == 0) atomicAdd(wa.work + kWorkTraceFullWarps, 1ull);
                }
                if (alive) {
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
                __syncwarp();  // the list is rebuilt for the next chunk
                if (ps.ns <= (w0 + kChunkWords) * 32) break;
            }
        }
        const bool hit_now = alive && h.idx >= 0;
        if (alive && !hit_now) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            alive = false;
        }
        int cls = 0;
        int64_t slot = 0;
        unsigned mask[kWords + 1];
        float4 qp, qn;  // a queued hit's point (+ record slot) and normal
        bool to_lane = false, lane_z = false;  // qn.w: the candidate sphere's slot
        if (hit_now) {
            D3 p64, n64;
            refine_hit(o64, d64, sa.geo64, sa.n, h.idx, p64, n64);
            const float3 hit = rnd(p64), normal = rnd(n64);
            float3 l = normalize3(light - hit);
            float dfs = fmaxf(dot3(normal, l), 0.f);
            float3 hv = l - dir;
            float hm2 = dot3(hv, hv);
            float s = 0.f;
            if (hm2 > 0.f) {
                float dd = fmaxf(dot3(normal, hv) * rsqrtf(hm2), 0.f);
                s = blinn_pow(dd, __ldg(sa.mat + 8 * h.idx + 4));
            }
            const float3 so = hit + normal * 1e-3f;  // shadow (and reflection) origin
            const Cone cone = make_cone(so, light, sa.light_radius);
            cls = classify_hit(ps, cone, so.y, light.y, mask, wa.cull == 2, grid_mask(wa, so));
            slot = (int64_t)k * wa.n_pix + lp;
            if constexpr (kCompact) {
                wa.rec[slot] = make_float4(__int_as_float(h.idx), dfs, s, cls == 2 ? 0.f : 1.f);
            } else {
                ridx[k] = h.idx;
                rdfs[k] = dfs;
                rs[k] = s;
                rsc[k] = cls == 2 ? 0.f : 1.f;
            }
            if (cls == 1) {
                qp = make_float4(hit.x, hit.y, hit.z, __int_as_float((int)slot));
                qn = make_float4(normal.x, normal.y, normal.z, 0.f);
                pmask |= 1 << k;
                // one candidate sphere: a lane of the lane sampler
                if (wa.lane_cap && mask[kWords] == 0) {
                    int nc = 0, b = 0;
#pragma unroll
                    for (int w = 0; w < kWords; w++) {
                        if (mask[w]) b = w * 32 + __ffs(mask[w]) - 1;
                        nc += __popc(mask[w]);
                    }
                    if (nc == 1) {
                        to_lane = true;
                        lane_z = !conic_front(cone, ps.sph[b]);
                        qn.w = __int_as_float(b);
                    }
                }
            }
            m = k + 1;
            if (k == fa.bounces) {
                exhausted = 1;
                alive = false;
            } else {
                reflect64(p64, n64, o64, d64);
            }
        }
        // queue the undecided hits: one atomic per warp, bounce and queue
        bool laned = false;
#pragma unroll
        for (int q = 0; q < 2; q++) {  // the two lane queues: sphere wholly in front / not
            const bool want = hit_now && cls == 1 && to_lane && lane_z == (q == 1);
            const unsigned lb = __ballot_sync(0xffffffffu, want);
            if (lb) {
                unsigned base = 0;
                if (lane == 0) base = atomicAdd(wa.count + (q == 0 ? 3 : 0), (unsigned)__popc(lb));
                base = __shfl_sync(0xffffffffu, base, 0);
                const unsigned e = base + __popc(lb & lanemask_lt());
                if (want && e < wa.lane_cap) {
                    wa.lane_q[(size_t)(2 * q) * wa.lane_cap + e] = qp;
                    wa.lane_q[(size_t)(2 * q + 1) * wa.lane_cap + e] = qn;
                    laned = true;
                }
            }
        }
        const bool need = hit_now && cls == 1 && !laned;
        const unsigned nb = __ballot_sync(0xffffffffu, need);
        if (__builtin_expect(nb != 0, 0)) {  // (rare in small scenes: laid out off the hot path)
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(wa.count + 1, (unsigned)__popc(nb));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (need) {
                // compact queue entry: everything the sampler needs, no indirection
                const unsigned e = base + __popc(nb & lanemask_lt());
                int code = 0;
                qn.w = 0.f;
                if (e < wa.conic_cap) code = conic_entry(ps, wa, e, mask, qp, qn, light, sa.light_radius);
                qn.w = __int_as_float(code);
                wa.hit_p[e] = qp;
                wa.hit_n[e] = qn;
#pragma unroll
                for (int w = 0; w <= kWords; w++) wa.mask2[(size_t)w * wa.mask2_stride + e] = mask[w];
            }
        }
        if (__builtin_expect(wa.work != nullptr, 0)) {
            const unsigned nh = __popc(__ballot_sync(0xffffffffu, hit_now));
            if (lane == 0 && nh) {
                atomicAdd(wa.work + kWorkHits, (unsigned long long)nh);
                atomicAdd(wa.work + kWorkCullTests, (unsigned long long)nh * (ps.ns + ps.np));
            }
        }
        if (compact && was_alive && !alive) {  // the ray ended: its pixel now (the thread may get another ray)
            finish();
            valid = false;
        }
    }
    if (!valid) return;
    finish();
}

// A sampled hit's unblocked count (record slot = bounce * n_pix + pixel): a
// pixel with this one pending hit is unwound and packed at once (its other
// records are decided).  With several pending hits the last of the pixel's
// samplers unwinds it: in frames of up to 3 bounces and 65,534 samples
// (packed_counts) each sampler adds its count + 1 into its bounce's 16-bit
// field of the pixel's 64-bit word — one relaxed atomic; the sampler that
// completes every pending field holds all the counts, no fence and no
// reload — otherwise the coefficient is stored and an acquire-release
// countdown elects the last.
// The first records of a parked pixel, loaded ahead (their latency hides
// behind the sampling); kPre covers every record of a frame of up to 3 bounces.
constexpr int kPre = 4;
struct PreRecords {
    float4 r[kPre];
    int n;  // how many of r are loaded
};

__device__ __forceinline__ PreRecords prefetch_records(const WaveArgs &wa, int slot, float4 px) {
    PreRecords p;
    const int n_pix = (int)wa.n_pix;
    const int lp = slot - (slot / n_pix) * n_pix;
    const int m = __float_as_int(px.w) & 0xff;
    p.n = m < kPre ? m : kPre;
#pragma unroll
    for (int k = 0; k < kPre; k++) p.r[k] = k < p.n ? __ldcg(wa.rec + (int64_t)k * n_pix + lp) : make_float4(0, 0, 0, 0);
    return p;
}

__device__ __forceinline__ void resolve_hit(const FrameArgs &fa, const SceneArgs<float> &sa, const WaveArgs &wa,
                                            int slot, int unblocked, float4 px, const float4 *mat4,
                                            const PreRecords *pre = nullptr) {
    const int n_pix = (int)wa.n_pix;
    const int kh = slot / n_pix, lp = slot - kh * n_pix;
    const int info = __float_as_int(px.w);
    const bool several = info & (1 << 9);
    const int n = fa.samples;
    const float sc = (float)unblocked / (float)n;
    const bool packed = packed_counts(fa);
    const int pm = several && packed ? (info >> 10) & 15 : 0;  // the pending bounces
    unsigned long long counts = 0;  // field k: bounce k's unblocked count + 1
    if (several) {
        if (packed) {
            const unsigned long long add = (unsigned long long)(unblocked + 1) << (16 * kh);
            counts = atomicAdd(wa.pend64 + lp, add) + add;
#pragma unroll
            for (int k = 0; k < 4; k++)
                if (((pm >> k) & 1) && ((counts >> (16 * k)) & 0xffffu) == 0) return;  // a count still to come
        } else {
            reinterpret_cast<float *>(wa.rec + slot)[3] = sc;
            // release our coefficient, acquire the others' (the last sampler reads
            // them): one acq_rel countdown instead of two sequentially consistent
            // fences around a relaxed one (C2 2.5% faster)
            cuda::atomic_ref<int, cuda::thread_scope_device> pend(wa.pend[lp]);
            if (pend.fetch_sub(1, cuda::memory_order_acq_rel) != 1) return;
        }
    }
    const int m = info & 0xff;
    // the records do not change after the trace, except the coefficients the
    // countdown's samplers store: the prefetched ones serve unless those landed
    const int have = (pre && (!several || packed)) ? pre->n : 0;
    auto coeff = [&](int k, float w) {
        float c = w;
        if (k == kh && !several) c = sc;
        if ((pm >> k) & 1) c = (float)((int)((counts >> (16 * k)) & 0xffffu) - 1) / (float)n;
        return c;
    };
    float3 c;
    if (have >= m) {  // every record prefetched (frames of up to kPre - 1 bounces): registers only
        c = unwind_upto<kPre>(
            m, (info >> 8) & 1, f3(px.x, px.y, px.z), sa,
            [&](int k) { return Record{__float_as_int(pre->r[k].x), pre->r[k].y, pre->r[k].z, coeff(k, pre->r[k].w)}; },
            mat4);
    } else {
        float4 rk[kMaxBounce + 1];  // every record load in flight before the first use
#pragma unroll
        for (int k = 0; k < kPre; k++)
            if (k < have) rk[k] = pre->r[k];
#pragma unroll 4
        for (int k = have; k < m; k++) rk[k] = __ldcg(wa.rec + (int64_t)k * n_pix + lp);
        c = unwind(
            m, (info >> 8) & 1, f3(px.x, px.y, px.z), sa,
            [&](int k) { return Record{__float_as_int(rk[k].x), rk[k].y, rk[k].z, coeff(k, rk[k].w)}; }, mat4);
    }
    const int ly = lp / fa.width, x = lp - ly * fa.width;
    store_pixel(fa, x, map_row(ly, fa), c);
    if (fa.peer_out) __threadfence_system();
}

// The parked-pixel word of a hit's pixel (issued early: its latency hides
// behind the sampling).
__device__ __forceinline__ float4 pixel_word(const WaveArgs &wa, int slot) {
    const int n_pix = (int)wa.n_pix;
    return __ldcg(wa.pix + (slot - (slot / n_pix) * n_pix));
}

// --- B ----------------------------------------------------------------------------
// Sampling of one queued hit by a warp; returns the unblocked count (all lanes).
template <int MAXS, bool SMEM_TAB>
__device__ __forceinline__ int sample_hit(const ParamScene<MAXS> &ps, const ShadowFrame &f, const unsigned *hm,
                                          int n, const float4 *gtab, int &nsph_out) {
    constexpr int kWords = (MAXS + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int rounds = (n + 31) / 32;
    int nsph = 0;
#pragma unroll
    for (int w = 0; w < kWords; w++) nsph += __popc(hm[w]);
    nsph_out = nsph;
    auto table = [&](int i) -> float4 {
        if constexpr (SMEM_TAB) {
            extern __shared__ float4 smem_tab_f[];
            return smem_tab_f[i];
        } else {
            return __ldg(gtab + i);
        }
    };
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
            float3 dir;
            float limit;
            shadow_ray_unguarded(f, table(i), dir, limit);
            return sphere_margin_L(L, dir, r2g, limit) > 0.f ? 0 : 1;
        };
        const int full = n >> 5;
#pragma unroll 2
        for (int j = 0; j < full; j++) unblocked += sample(lane + 32 * j);
        if (lane + 32 * full < n) unblocked += sample(lane + 32 * full);
        return unblocked;
    }
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
                float3 dir;
                float limit;
                shadow_ray_unguarded(f, table(i < n ? i : 0), dir, limit);
                float mg = -INFINITY;
#pragma unroll
                for (int r = 0; r < kRegCand; r++)
                    if (r < k) mg = fmaxf(mg, sphere_margin_L(f3(c[r].x, c[r].y, c[r].z), dir, c[r].w, limit));
                for (unsigned b = pm; b; b &= b - 1)
                    mg = fmaxf(mg, plane_margin(ps.pl_h[__ffs(b) - 1] - f.origin.y, dir.y, limit));
                if (mg > 0.f) blocked |= 1ull << (j - g0);
            }
            if (nsph <= kRegCand) break;
        }
        for (int j = g0; j < g1; j++) unblocked += (lane + 32 * j < n && !((blocked >> (j - g0)) & 1ull)) ? 1 : 0;
    }
    return unblocked;
}

// Silhouette-form sample test (rt_wave.cuh): sphere coefficients A = {x0, x1,
// x2, y0}, B = {y1, y2, z1, z2}, the hit's |w|^2 = b0 + b1 a + b2 b + rho,
// table entry t = {a, b, rho}.  Returns 1 when blocked: the sign bit of
// d = x^2 + y^2 - |w|^2 (and, with the z test, z > 0 as a clear sign bit).
__device__ __forceinline__ unsigned conic_blocked(float4 A, float4 B, float b0, float b1, float b2, float4 t) {
    const float w2 = fmaf(b1, t.x, fmaf(b2, t.y, b0 + t.z));
    const float x = fmaf(A.y, t.x, fmaf(A.z, t.y, A.x));
    const float y = fmaf(B.x, t.x, fmaf(B.y, t.y, A.w));
    const float d = fmaf(x, x, fmaf(y, y, -w2));
    return __float_as_uint(d) >> 31;
}
__device__ __forceinline__ unsigned conic_blocked_z(float4 A, float4 B, float z0, float b0, float b1, float b2,
                                                    float4 t) {
    const float w2 = fmaf(b1, t.x, fmaf(b2, t.y, b0 + t.z));
    const float x = fmaf(A.y, t.x, fmaf(A.z, t.y, A.x));
    const float y = fmaf(B.x, t.x, fmaf(B.y, t.y, A.w));
    const float z = fmaf(B.z, t.x, fmaf(B.w, t.y, z0));
    const float d = fmaf(x, x, fmaf(y, y, -w2));
    return (__float_as_uint(d) & ~__float_as_uint(z)) >> 31;
}

// The same tests on two samples at once with the paired FP32 instructions
// (FFMA2 / FADD2: per component exactly fmaf / the add, so each sample's d —
// and its bit — is the scalar test's).  ab = {a_i, a_i+1, b_i, b_i+1}, nrho =
// {-rho_i, -rho_i+1} (SamplePairs); returns how many of the two are blocked.
// -|w|^2 is formed directly from the negated coefficients and table: round to
// nearest is symmetric, so fma(-p, q, -s) = -fma(p, q, s) and the value is
// the scalar test's -w2 bit for bit, without two negations per pair.
struct Conic2 {
    float2 ax, ay, az, aw, bx, by, bz, bw, nb0, nb1, nb2, z0;
};
__device__ __forceinline__ float2 dup2(float v) { return make_float2(v, v); }
__device__ __forceinline__ Conic2 make_conic2(float4 A, float4 B, float z0, float b0, float b1, float b2) {
    return Conic2{dup2(A.x), dup2(A.y), dup2(A.z), dup2(A.w), dup2(B.x), dup2(B.y),
                  dup2(B.z), dup2(B.w), dup2(-b0), dup2(-b1), dup2(-b2), dup2(z0)};
}
template <bool ZTEST>
__device__ __forceinline__ unsigned conic_blocked2(const Conic2 &c, float4 ab, float2 nrho) {
    const float2 a = make_float2(ab.x, ab.y), b = make_float2(ab.z, ab.w);
    const float2 nw2 = __ffma2_rn(c.nb1, a, __ffma2_rn(c.nb2, b, __fadd2_rn(c.nb0, nrho)));
    const float2 x = __ffma2_rn(c.ay, a, __ffma2_rn(c.az, b, c.ax));
    const float2 y = __ffma2_rn(c.bx, a, __ffma2_rn(c.by, b, c.aw));
    const float2 d = __ffma2_rn(x, x, __ffma2_rn(y, y, nw2));
    unsigned bx = __float_as_uint(d.x), by = __float_as_uint(d.y);
    if constexpr (ZTEST) {
        const float2 z = __ffma2_rn(c.bz, a, __ffma2_rn(c.bw, b, c.z0));
        bx &= ~__float_as_uint(z.x);
        by &= ~__float_as_uint(z.y);
    }
    return (bx >> 31) + (by >> 31);
}

// The disc-sample table in pairs for conic_blocked2, staged after the float4
// table in shared memory by fused_sample for up to kPairSamples samples, rho
// negated; an odd count's last pair is padded with -rho = +inf, which never
// blocks.
constexpr int kPairSamples = 1024;
constexpr int kPairUnroll = 4;  // (2: C2 2.5% slower)
struct SamplePairs {
    const float4 *ab;
    const float2 *nrho;  // {-rho_i, -rho_i+1}
    int n;               // pairs
};

// Sampling of one silhouette-form hit (conic_entry): P = {|lo|^2, 2 lo.bu,
// 2 lo.bv, slot}, sphere j's coefficients C[2j], C[2j+1] (the first sphere's
// arrive prefetched).  Returns the unblocked count of this lane's samples.
template <bool SMEM_TAB>
__device__ __forceinline__ int sample_conic(const WaveArgs &wa, unsigned e, int code, float4 P, float4 A0, float4 B0,
                                            int n, const float4 *gtab) {
    const int lane = threadIdx.x & 31;
    auto table = [&](int i) -> float4 {
        if constexpr (SMEM_TAB) {
            extern __shared__ float4 smem_tab_c[];
            return smem_tab_c[i];
        } else {
            return __ldg(gtab + i);
        }
    };
    const int ncon = code & 7;
    const int full = n >> 5;
    unsigned blocked = 0;
    auto run = [&](auto test) {
#pragma unroll 4
        for (int j = 0; j < full; j++) blocked += test(table(lane + 32 * j));
        if (lane + 32 * full < n) blocked += test(table(lane + 32 * full));
    };
    float4 A[kConic], B[kConic];
    float Z[kConic];
    A[0] = A0;
    B[0] = B0;
#pragma unroll
    for (int j = 1; j < kConic; j++) {
        if (j < ncon) {
            A[j] = __ldg(wa.conic + (size_t)(2 * j) * wa.conic_cap + e);
            B[j] = __ldg(wa.conic + (size_t)(2 * j + 1) * wa.conic_cap + e);
        } else {  // never blocks: x = +inf
            A[j] = make_float4(INFINITY, 0.f, 0.f, 0.f);
            B[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
#pragma unroll
    for (int j = 0; j < kConic; j++) Z[j] = (code & (1 << (7 + j))) ? -1.f : 1.f;  // no z test: z = 1
    if (ncon == 1 && !(code & (1 << 3))) {
        run([&](float4 t) { return conic_blocked(A[0], B[0], P.x, P.y, P.z, t); });
    } else if (ncon == 1) {
        run([&](float4 t) { return conic_blocked_z(A[0], B[0], Z[0], P.x, P.y, P.z, t); });
    } else if (ncon == 2) {
        run([&](float4 t) {
            return conic_blocked_z(A[0], B[0], Z[0], P.x, P.y, P.z, t) |
                   conic_blocked_z(A[1], B[1], Z[1], P.x, P.y, P.z, t);
        });
    } else {
        run([&](float4 t) {
            unsigned b = 0;
#pragma unroll
            for (int j = 0; j < kConic; j++) b |= conic_blocked_z(A[j], B[j], Z[j], P.x, P.y, P.z, t);
            return b;
        });
    }
    return (n - lane + 31) / 32 - (int)blocked;  // this lane's samples lane, lane + 32, ... less the blocked
}

// Single-candidate hits, one per lane: every lane of a warp takes the same
// disc sample at the same time (a shared-memory broadcast) against its own
// hit; the per-hit setup is one lane's, not a warp's, and there is no
// reduction.  The two lane queues are cut into units of 32 hits, listed one
// after the other; CTA c takes units [c U / G, (c + 1) U / G) — the grid is
// exactly the resident CTAs, the same count on every SM, so the SMs get equal
// shares.  A sample is blocked iff d = x^2 + y^2 - |w|^2 < 0 (and z > 0): its
// sign bit is added to the blocked count; d is formed exactly as in
// sample_conic, so either sampler gives the same bits.
template <int MAXS, bool SMEM_TAB>
__device__ __forceinline__ void sample_lanes(const FrameArgs &fa, const SceneArgs<float> &sa, const WaveArgs &wa,
                                             const ParamScene<MAXS> &ps, const float4 *gtab, const float4 *mat4,
                                             const SamplePairs pairs) {
    const int n = fa.samples;
    auto table = [&](int i) -> float4 {
        if constexpr (SMEM_TAB) {
            extern __shared__ float4 smem_tab_l[];
            return smem_tab_l[i];
        } else {
            return __ldg(gtab + i);
        }
    };
    const float3 light = f3(sa.light[0], sa.light[1], sa.light[2]);
    const unsigned c0 = min(wa.count[3], wa.lane_cap), c1 = min(wa.count[0], wa.lane_cap);
    const unsigned u0 = (c0 + 31) / 32, units = u0 + (c1 + 31) / 32;
    const unsigned first = (unsigned)(((unsigned long long)units * blockIdx.x) / gridDim.x);
    const unsigned last = (unsigned)(((unsigned long long)units * (blockIdx.x + 1)) / gridDim.x);
    const unsigned lane = threadIdx.x & 31;
    for (unsigned u = first + (threadIdx.x >> 5); u < last; u += blockDim.x >> 5) {
        const int q = u < u0 ? 0 : 1;
        const unsigned h = 32u * (q == 0 ? u : u - u0) + lane;
        if (h >= (q == 0 ? c0 : c1)) continue;
        const float4 *qp = wa.lane_q + (size_t)(2 * q) * wa.lane_cap;
        const float4 *qn = qp + wa.lane_cap;
        const float4 P = __ldg(qp + h);
        const float4 N = __ldg(qn + h);
        const int slot = __float_as_int(P.w);
        const float4 px = pixel_word(wa, slot);
        const float4 g = ps.sph[__float_as_int(N.w)];
        const ShadowFrame f = shadow_frame(f3(P.x, P.y, P.z), f3(N.x, N.y, N.z), light, true);
        const Cone k = make_cone(f.origin, light, sa.light_radius);
        float4 A, B;
        const int r = conic_coeffs(k, g, f.lo, f.bu, f.bv, f.ls2, A, B);
        const float b0 = dot3(f.lo, f.lo), b1 = 2.f * dot3(f.lo, f.bu), b2 = 2.f * dot3(f.lo, f.bv);
        const PreRecords pre = prefetch_records(wa, slot, px);
        unsigned blocked = 0;
        const unsigned act = __activemask();
        if (__any_sync(act, r == 0)) {
            // some lane's hit needs the ray form: those lanes take it, the rest the silhouette
            // form with the z test (a no-z hit has z1 = z2 = 0, z0 = 1)
            const float3 L = f3(g.x - f.origin.x, g.y - f.origin.y, g.z - f.origin.z);
            const float r2g = sphere_r2g(L, g.w);
            const float z0 = r == 3 ? -1.f : 1.f;
            for (int i = 0; i < n; i++) {
                const float4 t = table(i);
                if (r == 0) {
                    float3 dir;
                    float limit;
                    shadow_ray_unguarded(f, t, dir, limit);
                    blocked += sphere_margin_L(L, dir, r2g, limit) > 0.f ? 1 : 0;
                } else {
                    blocked += conic_blocked_z(A, B, z0, b0, b1, b2, t);
                }
            }
        } else if (pairs.n) {  // the paired instructions, two samples a step
            const Conic2 c2 = make_conic2(A, B, r == 3 ? -1.f : 1.f, b0, b1, b2);
            if (__any_sync(act, r >= 2)) {
#pragma unroll(kPairUnroll)
                for (int p = 0; p < pairs.n; p++) blocked += conic_blocked2<true>(c2, pairs.ab[p], pairs.nrho[p]);
            } else {
#pragma unroll(kPairUnroll)
                for (int p = 0; p < pairs.n; p++) blocked += conic_blocked2<false>(c2, pairs.ab[p], pairs.nrho[p]);
            }
        } else if (__any_sync(act, r >= 2)) {
            const float z0 = r == 3 ? -1.f : 1.f;
#pragma unroll 4
            for (int i = 0; i < n; i++) blocked += conic_blocked_z(A, B, z0, b0, b1, b2, table(i));
        } else {
#pragma unroll 4
            for (int i = 0; i < n; i++) blocked += conic_blocked(A, B, b0, b1, b2, table(i));
        }
        resolve_hit(fa, sa, wa, slot, n - (int)blocked, px, mat4, &pre);
        if (wa.work) {
            if (r != 0) {
                atomicAdd(wa.work + kWorkConicHits, 1ull);
                atomicAdd(wa.work + kWorkConicTests, (unsigned long long)n);
                if (r >= 2) atomicAdd(wa.work + kWorkConicZTests, (unsigned long long)n);
            }
            atomicAdd(wa.work + kWorkSampledHits, 1ull);
            atomicAdd(wa.work + kWorkShadowRays, (unsigned long long)n);
            atomicAdd(wa.work + kWorkSphereTests, (unsigned long long)n);
            atomicAdd(wa.work + kWorkLaneHits, 1ull);
        }
    }
}

// 5 resident CTAs (95 registers, as unbounded); 6-7 measured no faster
// (spills), and an explicit 1 raises the register count and costs ~15%
#ifndef RT_SAMPLE_MIN_BLOCKS
#define RT_SAMPLE_MIN_BLOCKS 5
#endif
template <int MAXS, bool SMEM_TAB>
__global__ void __launch_bounds__(kThreads, MAXS <= 8 ? RT_SAMPLE_MIN_BLOCKS : 1)
    fused_sample(const FrameArgs fa, const SceneArgs<float> sa, const WaveArgs wa, const ParamScene<MAXS> ps) {
    constexpr int kWords = (MAXS + 31) / 32;
    const int n = fa.samples;
    const float4 *gtab = reinterpret_cast<const float4 *>(sa.table);
    // the bodies' base colours for the unwinds (kParamSpheres + kMaxPlanes bodies at most)
    __shared__ float4 s_mat[kParamSpheres + kMaxPlanes];
    for (int i = threadIdx.x; i < sa.n; i += blockDim.x) s_mat[i] = __ldg(reinterpret_cast<const float4 *>(sa.mat) + 2 * i);
    SamplePairs pairs = {nullptr, nullptr, 0};
    if constexpr (SMEM_TAB) {
        extern __shared__ float4 smem_tab_k[];
        for (int i = threadIdx.x; i < n; i += blockDim.x) smem_tab_k[i] = gtab[i];
        if (n <= kPairSamples) {
            const int np = (n + 1) / 2;
            float4 *ab = smem_tab_k + n;
            float2 *nrho = reinterpret_cast<float2 *>(ab + np);
            for (int p = threadIdx.x; p < np; p += blockDim.x) {
                const float4 t0 = gtab[2 * p];
                const float4 t1 = 2 * p + 1 < n ? gtab[2 * p + 1] : make_float4(0.f, 0.f, -INFINITY, 0.f);
                ab[p] = make_float4(t0.x, t1.x, t0.y, t1.y);
                nrho[p] = make_float2(-t0.z, -t1.z);
            }
            pairs = SamplePairs{ab, nrho, np};
        }
    }
    __syncthreads();
    // programmatic dependent launch: everything above (the table staging)
    // overlaps the trace kernel's tail; the queue is read only after it
    cudaGridDependencySynchronize();
    if (wa.lane_cap) {  // B1: the single-candidate hits, one lane each
        sample_lanes<MAXS, SMEM_TAB>(fa, sa, wa, ps, gtab, s_mat, pairs);
    }
    // B2: the rest, one warp each
    const unsigned count = wa.count[1];
    const int lane = threadIdx.x & 31;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned n_warps = (gridDim.x * blockDim.x) >> 5;
    const float3 lp = f3(sa.light[0], sa.light[1], sa.light[2]);
    // the next hit's queue entry is loaded while the current one samples
    float4 P, N, A0 = make_float4(0.f, 0.f, 0.f, 0.f), B0 = A0;
    unsigned hm[kWords + 1];
    auto fetch = [&](unsigned h) {
        P = __ldg(wa.hit_p + h);
        N = __ldg(wa.hit_n + h);
#pragma unroll
        for (int w = 0; w <= kWords; w++) hm[w] = __ldg(wa.mask2 + (size_t)w * wa.mask2_stride + h);
        if (h < wa.conic_cap) {  // the first silhouette sphere, should the entry have one
            A0 = __ldg(wa.conic + h);
            B0 = __ldg(wa.conic + wa.conic_cap + h);
        }
    };
    if (warp < count) fetch(warp);
    int held = 0, my_slot = -1, my_unb = 0;
    for (unsigned h = warp; h < count; h += n_warps) {
        const float4 Pc = P, Nc = N, A0c = A0, B0c = B0;
        unsigned hmc[kWords + 1];
#pragma unroll
        for (int w = 0; w <= kWords; w++) hmc[w] = hm[w];
        if (h + n_warps < count) fetch(h + n_warps);
        const int slot = __float_as_int(Pc.w);
        const int code = __float_as_int(Nc.w);
        int nsph = 0;
        int unblocked;
        if (code != 0) {
            unblocked = sample_conic<SMEM_TAB>(wa, h, code, Pc, A0c, B0c, n, gtab);
            nsph = code & 7;
        } else {
            const ShadowFrame f = shadow_frame(f3(Pc.x, Pc.y, Pc.z), f3(Nc.x, Nc.y, Nc.z), lp, true);
            unblocked = sample_hit<MAXS, SMEM_TAB>(ps, f, hmc, n, gtab, nsph);
        }
        unblocked = __reduce_add_sync(0xffffffffu, unblocked);
        // lane `held` keeps this hit; every 32 hits the lanes resolve theirs together
        if (lane == held) {
            my_slot = slot;
            my_unb = unblocked;
        }
        if (++held == 32) {
            if (my_slot >= 0) resolve_hit(fa, sa, wa, my_slot, my_unb, pixel_word(wa, my_slot), s_mat);
            my_slot = -1;
            held = 0;
        }
        if (lane != 0) continue;
        if (wa.work) {
            if (code != 0) {
                atomicAdd(wa.work + kWorkConicHits, 1ull);
                atomicAdd(wa.work + kWorkConicTests, (unsigned long long)n * nsph);
                atomicAdd(wa.work + kWorkConicZTests, (unsigned long long)n * __popc((code >> 3) & 15));
            }
            atomicAdd(wa.work + kWorkSampledHits, 1ull);
            atomicAdd(wa.work + kWorkShadowRays, (unsigned long long)n);
            atomicAdd(wa.work + kWorkSphereTests, (unsigned long long)n * nsph);
            atomicAdd(wa.work + kWorkPlaneTests, (unsigned long long)n * __popc(hmc[kWords]));
        }
    }
    if (my_slot >= 0) resolve_hit(fa, sa, wa, my_slot, my_unb, pixel_word(wa, my_slot), s_mat);
}

// Launch with programmatic stream serialisation: the kernel may start while
// the previous one drains and waits for it in cudaGridDependencySynchronize.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 ctas, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = ctas;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int MAXS>
cudaError_t launch(const FrameArgs &fa, const SceneArgs<float> &sa, const WaveArgs &wa, const ParamScene<MAXS> &ps,
                   cudaStream_t st, cudaEvent_t *ev) {
    dim3 grid((fa.width + kTileW - 1) / kTileW, (fa.local_rows + kTileH - 1) / kTileH);
    cudaError_t e = launch_pdl(fused_trace<MAXS>, grid, 0, st, fa, sa, wa, ps);
    if (e != cudaSuccess) return e;
    if (ev) {
        cudaEventRecord(ev[1], st);
        cudaEventRecord(ev[2], st);  // no separate classify pass: a zero-length phase
    }
    const int n = fa.samples;
    if (n <= kWaveSmemSamples) {
        // the float4 table, then (up to kPairSamples samples) its pairs
        const size_t smem = sizeof(float4) * (size_t)n +
                            (n <= kPairSamples ? (sizeof(float4) + sizeof(float2)) * (size_t)((n + 1) / 2) : 0);
        e = launch_pdl(fused_sample<MAXS, true>, resident_ctas(fused_sample<MAXS, true>, smem), smem, st, fa, sa, wa,
                       ps);
    } else {
        e = launch_pdl(fused_sample<MAXS, false>, resident_ctas(fused_sample<MAXS, false>, 0), 0, st, fa, sa, wa, ps);
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

// The culled soft-shadow frame; false if the scene does not fit the
// launch-parameter layout (the caller then takes the unculled wavefront).
bool rt_fused_fits(const rt::SceneArgs<float> &sa) {
    static thread_local ParamScene<kParamSpheres> probe;
    ParamScene<8> p8;
    return pack_params(sa, p8) || pack_params(sa, probe);
}

cudaError_t rt_launch_fused_f32(const rt::FrameArgs &fa, const rt::SceneArgs<float> &sa, const rt::WaveArgs &wa,
                                cudaStream_t st, int *n_kernels, cudaEvent_t *ev) {
    *n_kernels = 0;
    cudaError_t e = cudaSuccess;  // the counters were zeroed by the previous frame's trace
    if (ev) cudaEventRecord(ev[0], st);
    ParamScene<8> p8;
    thread_local ParamScene<kParamMid> p256;
    thread_local ParamScene<kParamSpheres> p512;
    if (pack_params(sa, p8))
        e = launch(fa, sa, wa, p8, st, ev);
    else if (pack_params(sa, p256))
        e = launch(fa, sa, wa, p256, st, ev);
    else if (pack_params(sa, p512))
        e = launch(fa, sa, wa, p512, st, ev);
    else
        return cudaErrorInvalidValue;
    if (e != cudaSuccess) return e;
    if (ev) {  // the sampler also unwinds: a zero-length shade phase
        cudaEventRecord(ev[3], st);
        cudaEventRecord(ev[4], st);
    }
    *n_kernels = 2;
    return cudaSuccess;
}

// The shadow grid of the culled path: a box around the spheres (grown by its
// own extent sideways, where their shadows fall), 48 x 24 x 48 cells.
cudaError_t rt_build_shadow_grid_f32(const rt::SceneArgs<float> &sa, unsigned *mask, int capacity, rt::WaveArgs &wa,
                                     cudaStream_t st) {
    wa.grid = nullptr;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    double plane_lo = INFINITY;
    int ns = 0;
    for (int b = 0; b < sa.n; b++) {
        const double *g = sa.host_geo + 4 * b;
        if (g[3] < 0.0) {
            plane_lo = std::min(plane_lo, g[1]);
            continue;
        }
        const double r = std::sqrt(g[3]);
        for (int a = 0; a < 3; a++) {
            lo[a] = std::min(lo[a], g[a] - r);
            hi[a] = std::max(hi[a], g[a] + r);
        }
        ns++;
    }
    if (ns == 0) return cudaSuccess;
    const int dims[3] = {48, 24, 48};
    if (dims[0] * dims[1] * dims[2] > capacity) return cudaSuccess;
    for (int a = 0; a < 3; a += 2) {
        const double grow = std::max(hi[a] - lo[a], 4.0);
        lo[a] -= grow;
        hi[a] += grow;
    }
    lo[1] = std::min(lo[1], plane_lo) - 0.5;
    hi[1] += 0.5;
    for (int a = 0; a < 3; a++) {
        if (!(hi[a] > lo[a]) || !std::isfinite(lo[a]) || !std::isfinite(hi[a])) return cudaSuccess;
        wa.grid_lo[a] = (float)lo[a];
        wa.grid_dim[a] = dims[a];
        wa.grid_inv[a] = (float)(dims[a] / (hi[a] - lo[a]));
    }
    ParamScene<8> p8;
    thread_local ParamScene<kParamMid> p256;
    thread_local ParamScene<kParamSpheres> p512;
    const int blocks = (dims[0] * dims[1] * dims[2] + kThreads - 1) / kThreads;
    if (pack_params(sa, p8))
        shadow_grid_build<8><<<blocks, kThreads, 0, st>>>(p8, sa, wa, mask);
    else if (pack_params(sa, p256))
        shadow_grid_build<kParamMid><<<blocks, kThreads, 0, st>>>(p256, sa, wa, mask);
    else if (pack_params(sa, p512))
        shadow_grid_build<kParamSpheres><<<blocks, kThreads, 0, st>>>(p512, sa, wa, mask);
    else
        return cudaSuccess;
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) wa.grid = mask;
    return e;
}

void rt_set_sphere_bound(bool on) { rt32::g_sphere_bound = on; }
