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
#include "rt_wave.cuh"

namespace {
using namespace rt;
using namespace rt32;

// --- A: bounce chains --------------------------------------------------------
template <class Geo>
__device__ __forceinline__ void trace_chain(const Geo &geo, const FrameArgs &fa, const SceneArgs<float> &sa,
                                            const WaveArgs &wa, int x, int ly) {
    if (x >= fa.width || ly >= fa.local_rows) return;
    int y = map_row(ly, fa);
    if (y >= fa.row_end) return;
    const int64_t lp = (int64_t)ly * fa.width + x;
    D3 o64{fa.cam[0], fa.cam[1], fa.cam[2]};  // the ray chain in float64 (rt_f32.cuh: refine_hit)
    D3 d64 = primary_direction64(x, y, fa);
    const float3 light = f3(sa.light[0], sa.light[1], sa.light[2]);
    float3 tail = f3(0.f, 0.f, 0.f);
    int m = 0, exhausted = 0;
    for (int k = 0; k <= fa.bounces; k++) {
        const float3 origin = rnd(o64), dir = rnd(d64);
        Hit h = geo.closest(origin, dir);
        if (h.idx < 0) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            break;
        }
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
        reflect64(p64, n64, o64, d64);
    }
    wa.pix[lp] = make_float4(tail.x, tail.y, tail.z, __int_as_float(m | (exhausted << 8)));
}

template <int MAXS>
__device__ __forceinline__ void trace_chain_bundle(const ParamScene<MAXS> &ps, const FrameArgs &fa,
                                                   const SceneArgs<float> &sa, const WaveArgs &wa, int x, int ly) {
    constexpr int kWords = (MAXS + 31) / 32;
    const int lane = threadIdx.x & 31;
    // candidate lists of at most 256 spheres: larger scenes build and test them
    // in chunks of 8 mask words (the (t, index) order survives it)
    constexpr int kCandCap = MAXS < 256 ? MAXS : 256;
    constexpr int kChunkWords = kCandCap / 32 > 0 ? kCandCap / 32 : 1;
    __shared__ float4 s_cand_sph[kThreads / 32][kCandCap];
    __shared__ int s_cand_idx[kThreads / 32][kCandCap];
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
    D3 o64{fa.cam[0], fa.cam[1], fa.cam[2]};  // the ray chain in float64 (rt_f32.cuh: refine_hit)
    D3 d64 = valid ? primary_direction64(x, y, fa) : D3{0.0, 0.0, 1.0};
    const float3 light = f3(sa.light[0], sa.light[1], sa.light[2]);
    float3 tail = f3(0.f, 0.f, 0.f);
    int m = 0, exhausted = 0;
    for (int k = 0; k <= fa.bounces; k++) {
        const unsigned live = __ballot_sync(0xffffffffu, alive);
        if (!live) break;
        const float3 origin = rnd(o64), dir = rnd(d64);
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
        }
        // compact the candidates into this warp's shared-memory list: every
        // lane then walks the same entries (broadcast LDS, unrolled)
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
        const bool hit_now = alive && h.idx >= 0;
        if (alive && !hit_now) {
            if (sa.has_sky) tail = sky_sample(dir, sa.sky, sa.sky_w, sa.sky_h);
            alive = false;
        }
        int64_t slot_id = 0;
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
            slot_id = (int64_t)k * wa.n_pix + lp;
            wa.hit_p[slot_id] = make_float4(hit.x, hit.y, hit.z, __int_as_float(h.idx));
            wa.hit_n[slot_id] = make_float4(normal.x, normal.y, normal.z, dfs);
            wa.hit_s[slot_id] = s;
            m = k + 1;
            if (k == fa.bounces) {
                exhausted = 1;
                alive = false;
            } else {
                reflect64(p64, n64, o64, d64);
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
    fa.out[(int64_t)y * fa.out_pitch + x] = pack_color(col.x, col.y, col.z, fa.rgba);
    if (fa.radiance) {
        float *r = (float *)fa.radiance + 3 * ((int64_t)y * fa.width + x);
        r[0] = col.x;
        r[1] = col.y;
        r[2] = col.z;
    }
    if (fa.peer_out) __threadfence_system();
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
