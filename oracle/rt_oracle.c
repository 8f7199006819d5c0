/*
 * TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * CPU float64 restatement of the reference frame render
 * (/root/reference/pkg/src/raytracer/renderer.py `_render_kernel` / `_trace`
 * and every @njit helper they inline).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * Bit-exactness contract: the reference is numba-compiled float64 without
 * fast-math, so LLVM neither contracts a*b+c into FMA nor reassociates.  This
 * file is compiled with -ffp-contract=off -fno-fast-math and spells every
 * expression in the reference's left-to-right evaluation order; the
 * transcendentals (sqrt, cos, sin, atan2, asin, pow, floor) resolve to the
 * same glibc libm numba calls.  The result is pinned by the reference's golden
 * sha256 (pkg/tests/test_acceptance.py:31) and by fixtures generated from the
 * reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { double x, y, z; } v3;

/* Work counting build (-DRTO_COUNT, librt_oracle_count.so): tallies the
 * reference's control flow for the roofline numerators. */
enum { C_PIX, C_CH_RAYS, C_SH_RAYS, C_HITS, C_REFL, C_SHADE, C_CH_TCA, C_CH_DISC, C_CH_FULL, C_CH_PLANE,
       C_SH_TCA, C_SH_DISC, C_SH_FULL, C_SH_PLANE, C_MISS, C_NCOUNT };
#ifdef RTO_COUNT
static _Thread_local long long *g_cnt;
#define CNT(k) (g_cnt[k]++)
#else
#define CNT(k) ((void)0)
#endif

/* constants: renderer.py:33,36; shading.py:23-29; geometry.py:24 */
#define REFLECT_EPS 1e-3
#define SHADOW_EPS 1e-3
#define GRAZE_EPS 1e-7
#define MAX_BOUNCE_LIMIT 31

/* Precision probe build (-DRTO_ROUND=mask, tools/precision_probe.py only; the
 * pinned oracle never defines it): round chosen intermediates to float32 to
 * measure how sensitive the frame is to each — 1 primary direction, 2 hit
 * point and normal, 4 shadow origin and sample directions, 8 reflected
 * direction and origin, 16 shadow origin only, 32 the shading vectors, 64 the
 * scene geometry of the shadow tests. */
#ifdef RTO_ROUND
static inline double rf(double x) { return (double)(float)x; }
#define RND(bit, v) ((RTO_ROUND & (bit)) ? (v3){rf((v).x), rf((v).y), rf((v).z)} : (v))
#else
#define RND(bit, v) (v)
#endif

static double golden_angle(void) { return M_PI * (3.0 - sqrt(5.0)); } /* shading.py:29 */

static inline v3 mk(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static inline v3 vsub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); } /* vecmath.py:33-36 */
static inline double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; } /* vecmath.py:49-51 */
static inline v3 vcross(v3 a, v3 b) {                                               /* vecmath.py:54-60 */
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline double vmag(v3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); } /* vecmath.py:63-65 */
static inline v3 vnormalize(v3 a) {                                                   /* vecmath.py:68-78 */
    double m = vmag(a);
    if (m == 0.0) return mk(0.0, 0.0, 0.0);
    return mk(a.x / m, a.y / m, a.z / m);
}
static inline double vdistance(v3 a, v3 b) {                                          /* vecmath.py:81-86 */
    double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
    return sqrt(dx * dx + dy * dy + dz * dz);
}
static inline v3 vreflect(v3 i, v3 n) {                                               /* vecmath.py:89-96 */
    double k = 2.0 * (n.x * i.x + n.y * i.y + n.z * i.z);
    return mk(i.x - k * n.x, i.y - k * n.y, i.z - k * n.z);
}
static inline v3 rotate_yaw_pitch(v3 d, double cb, double sb, double ca, double sa) { /* vecmath.py:99-110 */
    double y2 = d.y * cb - d.z * sb;
    double z2 = d.y * sb + d.z * cb;
    double x2 = d.x * ca + z2 * sa;
    double z3 = -d.x * sa + z2 * ca;
    return mk(x2, y2, z3);
}

/* camera.py:46-54 */
static inline void norm_screen_coords(double x, double y, double w, double h, double *u, double *v) {
    if (w > h) {
        *u = (x - w / 2 + h / 2) / h * 2 - 1;
        *v = -(y / h * 2 - 1);
    } else {
        *u = x / w * 2 - 1;
        *v = -((y - h / 2 + w / 2) / w * 2 - 1);
    }
}

/* camera.py:70-77 (cos/sin of yaw and pitch hoisted: same libm values) */
static inline v3 primary_direction(double x, double y, double w, double h, double cb, double sb, double ca,
                                   double sa, double vdist) {
    double u, v;
    norm_screen_coords(x, y, w, h, &u, &v);
    v3 d = vnormalize(mk(u, v, vdist));
    return rotate_yaw_pitch(d, cb, sb, ca, sa);
}

typedef struct {
    int n;
    const int32_t *kinds;
    const double *pos; /* [n,3] */
    const double *size;
    const double *col; /* [n,3] */
    const double *refl;
    v3 light_pos;
    double light_radius;
    v3 light_color;
    double ambient, max_refl;
    const float *sky;
    int sky_w, sky_h, has_sky;
    int samples, bounces;
    double ga;
} scene_t;

/* geometry.py:83-105 — geometric test, literal d2 = L.L - tca^2 */
static inline double ray_sphere(v3 o, v3 d, v3 c, double r, int sh) {
    double lx = c.x - o.x, ly = c.y - o.y, lz = c.z - o.z;
    double tca = lx * d.x + ly * d.y + lz * d.z;
    if (tca < 0.0) { CNT(sh ? C_SH_TCA : C_CH_TCA); return INFINITY; }
    double d2 = lx * lx + ly * ly + lz * lz - tca * tca;
    double rad = r * r - d2;
    if (rad < -GRAZE_EPS) { CNT(sh ? C_SH_DISC : C_CH_DISC); return INFINITY; }
    CNT(sh ? C_SH_FULL : C_CH_FULL);
    if (rad < 0.0) rad = 0.0;
    double t = tca - sqrt(rad);
    if (t < 0.0) return INFINITY;
    return t;
}

/* geometry.py:108-117 */
static inline double ray_plane(v3 o, v3 d, double h, int sh) {
    CNT(sh ? C_SH_PLANE : C_CH_PLANE);
    double dy = d.y;
    if (dy == 0.0) return INFINITY;
    double t = (h - o.y) / dy;
    if (t <= 0.0) return INFINITY;
    return t;
}

/* geometry.py:179-188 */
static inline double intersect(const scene_t *s, v3 o, v3 d, int i, int sh) {
    if (s->kinds[i] == 0)
        return ray_sphere(o, d, mk(s->pos[3 * i], s->pos[3 * i + 1], s->pos[3 * i + 2]), s->size[i], sh);
    return ray_plane(o, d, s->pos[3 * i + 1], sh);
}

/* geometry.py:191-201 — strict '<': lowest index wins ties */
static inline int closest_hit(const scene_t *s, v3 o, v3 d, double *t_out) {
    double best_t = INFINITY;
    int best_i = -1;
    for (int i = 0; i < s->n; i++) {
        double t = intersect(s, o, d, i, 0);
        if (t < best_t) { best_t = t; best_i = i; }
    }
    *t_out = best_t;
    return best_i;
}

/* geometry.py:204-210 */
static inline int occluded(const scene_t *s, v3 o, v3 d, double limit) {
#if defined(RTO_ROUND) && (RTO_ROUND & 64)
    for (int i = 0; i < s->n; i++) { /* probe: float32 scene geometry in the shadow tests */
        double t = s->kinds[i] == 0 ? ray_sphere(o, d, mk(rf(s->pos[3 * i]), rf(s->pos[3 * i + 1]), rf(s->pos[3 * i + 2])),
                                                 rf(s->size[i]), 1)
                                    : ray_plane(o, d, rf(s->pos[3 * i + 1]), 1);
        if (t < limit) return 1;
    }
    return 0;
#endif
    for (int i = 0; i < s->n; i++)
        if (intersect(s, o, d, i, 1) < limit) return 1;
    return 0;
}

/* shading.py:76-86 */
static inline void disc_basis(v3 axis, v3 *u, v3 *v) {
    v3 c = vcross(axis, mk(0.0, 1.0, 0.0));
    double m = vmag(c);
    if (m < 1e-9) *u = mk(1.0, 0.0, 0.0);
    else *u = mk(c.x / m, c.y / m, c.z / m);
    *v = vcross(axis, *u);
}

/* shading.py:89-100 */
static inline v3 disc_point(int i, int n, v3 c, double radius, v3 u, v3 v, double ga) {
    double r = 2.0 * radius * sqrt((double)i / (double)n);
    double theta = (double)i * ga;
    double a = r * cos(theta);
    double b = r * sin(theta);
    return mk(c.x + a * u.x + b * v.x, c.y + a * u.y + b * v.y, c.z + a * u.z + b * v.z);
}

/* renderer.py:82-105 */
static double shadow_coeff(const scene_t *s, v3 surface, v3 normal) {
    int n = s->samples;
    v3 origin = mk(surface.x + SHADOW_EPS * normal.x, surface.y + SHADOW_EPS * normal.y,
                   surface.z + SHADOW_EPS * normal.z);
    origin = RND(4 | 16, origin);
    v3 bu, bv;
    if (n > 1) {
        v3 axis = vnormalize(vsub(surface, s->light_pos));
        disc_basis(axis, &bu, &bv);
    } else {
        bu = mk(1.0, 0.0, 0.0);
        bv = mk(0.0, 0.0, 1.0);
    }
    int unblocked = 0;
    for (int i = 0; i < n; i++) {
        v3 sp = (n == 1) ? s->light_pos : disc_point(i, n, s->light_pos, s->light_radius, bu, bv, s->ga);
        v3 dir = RND(4, vnormalize(vsub(sp, origin)));
        double limit = vdistance(surface, sp);
        CNT(C_SH_RAYS);
        if (!occluded(s, origin, dir, limit)) unblocked += 1;
    }
    return (double)unblocked / (double)n;
}

/* shading.py:53-73 */
static inline double diffuse_factor(v3 n, v3 l) {
    double d = vdot(n, l);
    return d > 0.0 ? d : 0.0;
}
static inline double specular_blinn(v3 n, v3 l, v3 v, double refl) {
    double hx = l.x + v.x, hy = l.y + v.y, hz = l.z + v.z;
    double m = sqrt(hx * hx + hy * hy + hz * hz);
    if (m == 0.0) return 0.0;
    double d = (n.x * hx + n.y * hy + n.z * hz) / m;
    if (d < 0.0) d = 0.0;
    return pow(d, refl);
}
static inline double clamp01(double x) {
    /* min(max(x, 0.0), 1.0) with Python's first-wins tie rule */
    double m = (0.0 > x) ? 0.0 : x;
    return (1.0 < m) ? 1.0 : m;
}

/* shading.py:144-168 */
static inline v3 shade_color(v3 base, v3 n, v3 view, double sc, v3 l, double refl, v3 lc, double ambient) {
    CNT(C_SHADE);
    double d = diffuse_factor(n, l);
    double sp = specular_blinn(n, l, view, refl);
    double lum = ambient + sc * d * (1.0 - ambient);
    if (lum > 1.0) lum = 1.0;
    double spec = sc * sp;
    double r = base.x * lum + lc.x * spec;
    double g = base.y * lum + lc.y * spec;
    double b = base.z * lum + lc.z * spec;
    return mk(clamp01(r), clamp01(g), clamp01(b));
}

/* renderer.py:60-74 */
static inline v3 sky_sample(const scene_t *s, v3 d) {
    double u = 0.5 + atan2(d.x, d.z) / (2.0 * M_PI);
    double dy = d.y < -1.0 ? -1.0 : d.y;
    dy = dy > 1.0 ? 1.0 : dy;
    double v = 0.5 - asin(dy) / M_PI;
    long W = s->sky_w, H = s->sky_h;
    long tx = (long)floor(u * (double)W);
    tx = ((tx % W) + W) % W; /* Python modulo */
    long ty = (long)floor(v * (double)H);
    if (ty < 0) ty = 0;
    else if (ty > H - 1) ty = H - 1;
    const float *t = s->sky + (ty * W + tx) * 3;
    return mk(clamp01((double)t[0]), clamp01((double)t[1]), clamp01((double)t[2]));
}

typedef struct { v3 base, n, view, l; double rr, sc, refl; } rec_t; /* renderer.py:39-42 */

/* renderer.py:108-224 */
static v3 trace(const scene_t *s, v3 origin, v3 dir) {
    rec_t stack[MAX_BOUNCE_LIMIT + 1];
    int m = 0, exhausted = 0;
    v3 tail = mk(0.0, 0.0, 0.0);
    for (int k = 0; k < s->bounces + 1; k++) {
        double t;
        CNT(C_CH_RAYS);
        int idx = closest_hit(s, origin, dir, &t);
        if (idx < 0) {
            CNT(C_MISS);
            if (s->has_sky) tail = sky_sample(s, dir);
            break;
        }
        CNT(C_HITS);
        v3 hit = mk(origin.x + dir.x * t, origin.y + dir.y * t, origin.z + dir.z * t);
        v3 normal;
        if (s->kinds[idx] == 0)
            normal = vnormalize(vsub(hit, mk(s->pos[3 * idx], s->pos[3 * idx + 1], s->pos[3 * idx + 2])));
        else
            normal = mk(0.0, 1.0, 0.0);
        hit = RND(2, hit);
        normal = RND(2, normal);
        v3 view = mk(-dir.x, -dir.y, -dir.z);
        v3 to_light = vnormalize(vsub(s->light_pos, hit));
        double sc = shadow_coeff(s, hit, normal);
        rec_t *r = &stack[m++];
        r->base = mk(s->col[3 * idx], s->col[3 * idx + 1], s->col[3 * idx + 2]);
        r->rr = s->refl[idx] / s->max_refl;
        r->n = RND(32, normal);
        r->view = RND(32, view);
        r->l = RND(32, to_light);
        r->sc = sc;
        r->refl = s->refl[idx];
        if (k == s->bounces) { exhausted = 1; break; }
        CNT(C_REFL);
        origin = mk(hit.x + REFLECT_EPS * normal.x, hit.y + REFLECT_EPS * normal.y, hit.z + REFLECT_EPS * normal.z);
        dir = vreflect(dir, normal);
        origin = RND(8, origin);
        dir = RND(8, dir);
    }
    if (m == 0) return tail;
    v3 col;
    int start;
    if (exhausted) {
        rec_t *r = &stack[m - 1];
        col = shade_color(r->base, r->n, r->view, r->sc, r->l, r->refl, s->light_color, s->ambient);
        start = m - 2;
    } else {
        col = tail;
        start = m - 1;
    }
    for (int k = start; k >= 0; k--) {
        rec_t *r = &stack[k];
        double rr = r->rr;
        v3 mixed = mk(r->base.x * (1.0 - rr) + col.x * rr, r->base.y * (1.0 - rr) + col.y * rr,
                      r->base.z * (1.0 - rr) + col.z * rr);
        col = shade_color(mixed, r->n, r->view, r->sc, r->l, r->refl, s->light_color, s->ambient);
    }
    return col;
}

/* renderer.py:45-50 */
static inline uint32_t pack_color(v3 c) {
    uint32_t r = (uint32_t)(int)(c.x * 255.0 + 0.5);
    uint32_t g = (uint32_t)(int)(c.y * 255.0 + 0.5);
    uint32_t b = (uint32_t)(int)(c.z * 255.0 + 0.5);
    return 0xFF000000u | (r << 16) | (g << 8) | b;
}

static void fill_scene(scene_t *s, int n_bodies, const int32_t *kinds, const double *positions, const double *sizes,
                       const double *colors, const double *refls, const double *light_pos, double light_radius,
                       const double *light_color, double ambient, double max_refl, const float *sky, int sky_w,
                       int sky_h, int has_sky, int samples, int bounces) {
    s->n = n_bodies;
    s->kinds = kinds;
    s->pos = positions;
    s->size = sizes;
    s->col = colors;
    s->refl = refls;
    s->light_pos = mk(light_pos[0], light_pos[1], light_pos[2]);
    s->light_radius = light_radius;
    s->light_color = mk(light_color[0], light_color[1], light_color[2]);
    s->ambient = ambient;
    s->max_refl = max_refl;
    s->sky = sky;
    s->sky_w = sky_w;
    s->sky_h = sky_h;
    s->has_sky = has_sky;
    s->samples = samples;
    s->bounces = bounces;
    s->ga = golden_angle();
}

int rto_version(void) { return 1; }

/*
 * renderer.py:227-279 (`_render_kernel`) + 316-349 (`render_frame`).
 * Renders rows y = row0, row0 + row_step, ... (row_step = 1: the whole frame)
 * into pixels[x + y*w]; radiance (nullable) gets the pre-quantisation RGB.
 * Dynamic scheduling over rows (the reference's static prange chunks leave
 * most workers idle on the sky rows; the results do not depend on it).
 */
int rto_render(uint32_t *pixels, double *radiance, int w, int h, const double *cam_pos, double yaw, double pitch,
               double vdist, int n_bodies, const int32_t *kinds, const double *positions, const double *sizes,
               const double *colors, const double *refls, const double *light_pos, double light_radius,
               const double *light_color, double ambient, double max_refl, const float *sky, int sky_w, int sky_h,
               int has_sky, int samples, int bounces, int row0, int row_step, int nthreads) {
    if (bounces > MAX_BOUNCE_LIMIT || bounces < 0 || samples < 1 || w < 1 || h < 1 || row_step < 1) return -1;
    scene_t s;
    fill_scene(&s, n_bodies, kinds, positions, sizes, colors, refls, light_pos, light_radius, light_color, ambient,
               max_refl, sky, sky_w, sky_h, has_sky, samples, bounces);
    double cb = cos(pitch), sb = sin(pitch), ca = cos(yaw), sa = sin(yaw);
    v3 cam = mk(cam_pos[0], cam_pos[1], cam_pos[2]);
    int nrows = row0 < h ? (h - 1 - row0) / row_step + 1 : 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int ri = 0; ri < nrows; ri++) {
        int y = row0 + ri * row_step;
        for (int x = 0; x < w; x++) {
            v3 d = RND(1, primary_direction((double)x, (double)y, (double)w, (double)h, cb, sb, ca, sa, vdist));
            CNT(C_PIX);
            v3 c = trace(&s, cam, d);
            size_t idx = (size_t)x + (size_t)y * (size_t)w;
            pixels[idx] = pack_color(c);
            if (radiance) {
                radiance[3 * idx] = c.x;
                radiance[3 * idx + 1] = c.y;
                radiance[3 * idx + 2] = c.z;
            }
        }
    }
    return 0;
}

/* renderer.py:303-313 (`ray_trace_iterative`), batched over n rays */
int rto_trace_rays(const double *origins, const double *dirs, long n_rays, double *out_rgb, int n_bodies,
                   const int32_t *kinds, const double *positions, const double *sizes, const double *colors,
                   const double *refls, const double *light_pos, double light_radius, const double *light_color,
                   double ambient, double max_refl, const float *sky, int sky_w, int sky_h, int has_sky, int samples,
                   int bounces, int nthreads) {
    if (bounces > MAX_BOUNCE_LIMIT || bounces < 0 || samples < 1) return -1;
    scene_t s;
    fill_scene(&s, n_bodies, kinds, positions, sizes, colors, refls, light_pos, light_radius, light_color, ambient,
               max_refl, sky, sky_w, sky_h, has_sky, samples, bounces);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
    for (long i = 0; i < n_rays; i++) {
        v3 c = trace(&s, mk(origins[3 * i], origins[3 * i + 1], origins[3 * i + 2]),
                     mk(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]));
        out_rgb[3 * i] = c.x;
        out_rgb[3 * i + 1] = c.y;
        out_rgb[3 * i + 2] = c.z;
    }
    return 0;
}

/* camera.py:70-77 for a batch of pixels (KATs) */
void rto_primary_directions(const int32_t *xs, const int32_t *ys, long n, int w, int h, double yaw, double pitch,
                            double vdist, double *out) {
    double cb = cos(pitch), sb = sin(pitch), ca = cos(yaw), sa = sin(yaw);
    for (long i = 0; i < n; i++) {
        v3 d = primary_direction((double)xs[i], (double)ys[i], (double)w, (double)h, cb, sb, ca, sa, vdist);
        out[3 * i] = d.x;
        out[3 * i + 1] = d.y;
        out[3 * i + 2] = d.z;
    }
}

/* renderer.py:60-74 for a batch of directions */
void rto_sky_samples(const double *dirs, long n, const float *sky, int sky_w, int sky_h, double *out) {
    scene_t s;
    memset(&s, 0, sizeof s);
    s.sky = sky;
    s.sky_w = sky_w;
    s.sky_h = sky_h;
    for (long i = 0; i < n; i++) {
        v3 c = sky_sample(&s, mk(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]));
        out[3 * i] = c.x;
        out[3 * i + 1] = c.y;
        out[3 * i + 2] = c.z;
    }
}

/* shading.py:89-100 sample table: out[2*i] = r_i cos(theta_i), out[2*i+1] = r_i sin(theta_i) */
void rto_disc_table(int n, double radius, double *out) {
    double ga = golden_angle();
    for (int i = 0; i < n; i++) {
        double r = 2.0 * radius * sqrt((double)i / (double)n);
        double theta = (double)i * ga;
        out[2 * i] = r * cos(theta);
        out[2 * i + 1] = r * sin(theta);
    }
}

int rto_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

#ifdef RTO_COUNT
/* Work tallies of rto_render over rows row0, row0+row_step, ... (single
 * thread per row, summed): out[C_NCOUNT] in the enum order above. */
int rto_count_work(long long *out, int w, int h, const double *cam_pos, double yaw, double pitch, double vdist,
                   int n_bodies, const int32_t *kinds, const double *positions, const double *sizes,
                   const double *colors, const double *refls, const double *light_pos, double light_radius,
                   const double *light_color, double ambient, double max_refl, const float *sky, int sky_w,
                   int sky_h, int has_sky, int samples, int bounces, int row0, int row_step, int nthreads) {
    scene_t s;
    fill_scene(&s, n_bodies, kinds, positions, sizes, colors, refls, light_pos, light_radius, light_color, ambient,
               max_refl, sky, sky_w, sky_h, has_sky, samples, bounces);
    double cb = cos(pitch), sb = sin(pitch), ca = cos(yaw), sa = sin(yaw);
    v3 cam = mk(cam_pos[0], cam_pos[1], cam_pos[2]);
    int nrows = row0 < h ? (h - 1 - row0) / row_step + 1 : 0;
    memset(out, 0, sizeof(long long) * C_NCOUNT);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        long long local[C_NCOUNT];
        memset(local, 0, sizeof local);
        g_cnt = local;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int ri = 0; ri < nrows; ri++) {
            int y = row0 + ri * row_step;
            for (int x = 0; x < w; x++) {
                CNT(C_PIX);
                v3 d = primary_direction((double)x, (double)y, (double)w, (double)h, cb, sb, ca, sa, vdist);
                (void)trace(&s, cam, d);
            }
        }
#ifdef _OPENMP
#pragma omp critical
#endif
        for (int k = 0; k < C_NCOUNT; k++) out[k] += local[k];
    }
    return 0;
}
#endif
