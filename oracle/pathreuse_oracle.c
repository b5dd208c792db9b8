/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference hot path.
 * See pathreuse_oracle.h.  Every function cites the reference file:line it follows
 * (paths relative to /root/reference/proj).  Built by oracle/Makefile with -O2 and no
 * -march (no FMA contraction), like the reference, so float results are bit-identical.
 */
#define _GNU_SOURCE
#include "pathreuse_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */
static __thread char g_err[512];
const char* po_last_error(void) { return g_err; }
static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* ------------------------------------------------------------------ vec3.hpp */
typedef struct { float x, y, z; } V;
static V v3(float x, float y, float z) { V r = {x, y, z}; return r; }
static V vadd(V a, V b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
static V vsub(V a, V b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
static V vmul(V a, float s) { return v3(a.x * s, a.y * s, a.z * s); }
static V vmulv(V a, V b) { return v3(a.x * b.x, a.y * b.y, a.z * b.z); }
static V vdiv(V a, float s) { return v3(a.x / s, a.y / s, a.z / s); }
static V vneg(V a) { return v3(-a.x, -a.y, -a.z); }
static float vget(V v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }
static int veq(V a, V b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
static float dot3(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }                 /* :45 */
static V cross3(V a, V b) {                                                                /* :47 */
    return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static float len3(V v) { return sqrtf(dot3(v, v)); }                                      /* :52 */
static V norm3(V v) { return vdiv(v, len3(v)); }                                          /* :54 */
static float fminr(float a, float b) { return (b < a) ? b : a; }  /* std::min */
static float fmaxr(float a, float b) { return (a < b) ? b : a; }  /* std::max */
static double dminr(double a, double b) { return (b < a) ? b : a; }
static double dmaxr(double a, double b) { return (a < b) ? b : a; }
static V vmin3(V a, V b) { return v3(fminr(a.x, b.x), fminr(a.y, b.y), fminr(a.z, b.z)); }
static V vmax3(V a, V b) { return v3(fmaxr(a.x, b.x), fmaxr(a.y, b.y), fmaxr(a.z, b.z)); }
static void basis(V n, V* t, V* b) {                                                      /* :74-80 */
    const float sign = copysignf(1.0f, n.z);
    const float a = -1.0f / (sign + n.z);
    const float c = n.x * n.y * a;
    *t = v3(1.0f + sign * n.x * n.x * a, sign * c, -sign * n.x);
    *b = v3(c, sign + n.y * n.y * a, -n.y);
}

/* ------------------------------------------------------------------ geometry.hpp */
typedef struct { V lo, hi; } Box;
static Box box_empty(void) {
    Box b = {{FLT_MAX, FLT_MAX, FLT_MAX}, {-FLT_MAX, -FLT_MAX, -FLT_MAX}};
    return b;
}
static void box_pt(Box* b, V p) { b->lo = vmin3(b->lo, p); b->hi = vmax3(b->hi, p); }     /* :28-31 */
static void box_box(Box* b, Box o) { b->lo = vmin3(b->lo, o.lo); b->hi = vmax3(b->hi, o.hi); }
typedef struct { V a, b, c; } Tri;
static Box tri_box(Tri t) { Box b = box_empty(); box_pt(&b, t.a); box_pt(&b, t.b); box_pt(&b, t.c); return b; }

/* intersect_triangle, geometry.hpp:86-103 */
static int isect_tri(V o, V d, float tmin, float tmax, Tri tri, float* t_out) {
    const float eps = 1e-7f;
    const V e1 = vsub(tri.b, tri.a), e2 = vsub(tri.c, tri.a);
    const V p = cross3(d, e2);
    const float det = dot3(e1, p);
    if (fabsf(det) < 1e-12f) return 0;
    const float inv = 1.0f / det;
    const V tv = vsub(o, tri.a);
    const float u = dot3(tv, p) * inv;
    if (u < -eps || u > 1.0f + eps) return 0;
    const V q = cross3(tv, e1);
    const float v = dot3(d, q) * inv;
    if (v < -eps || u + v > 1.0f + eps) return 0;
    const float t = dot3(e2, q) * inv;
    if (t <= tmin || t >= tmax) return 0;
    *t_out = t;
    return 1;
}

/* segment_intersects_aabb, geometry.hpp:107-134 */
static int seg_box(V a, V b, Box box) {
    int sw;
    if (b.x != a.x) sw = b.x < a.x;
    else if (b.y != a.y) sw = b.y < a.y;
    else sw = b.z < a.z;
    if (sw) { V t = a; a = b; b = t; }
    double t0 = 0.0, t1 = 1.0;
    for (int ax = 0; ax < 3; ++ax) {
        const double o = vget(a, ax);
        const double d = (double)vget(b, ax) - o;
        const double lo = vget(box.lo, ax), hi = vget(box.hi, ax);
        if (d == 0.0) { if (o < lo || o > hi) return 0; continue; }
        double tn = (lo - o) / d, tf = (hi - o) / d;
        if (tn > tf) { double s = tn; tn = tf; tf = s; }
        t0 = dmaxr(t0, tn);
        t1 = dminr(t1, tf);
        if (t0 > t1) return 0;
    }
    return 1;
}

/* ray_intersects_aabb, geometry.hpp:136-154 */
static int ray_box(V o3, V d3, float tmin, float tmax, Box box) {
    double t0 = tmin, t1 = tmax;
    for (int ax = 0; ax < 3; ++ax) {
        const double o = vget(o3, ax), d = vget(d3, ax);
        const double lo = vget(box.lo, ax), hi = vget(box.hi, ax);
        if (d == 0.0) { if (o < lo || o > hi) return 0; continue; }
        double tn = (lo - o) / d, tf = (hi - o) / d;
        if (tn > tf) { double s = tn; tn = tf; tf = s; }
        t0 = dmaxr(t0, tn);
        t1 = dminr(t1, tf);
        if (t0 > t1) return 0;
    }
    return 1;
}

/* ------------------------------------------------------------------ rng.hpp:27-53 */
static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t rng_bits(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t purpose, uint32_t lane) {
    uint64_t h = mix64(seed);
    h = mix64(h ^ ((uint64_t)a | ((uint64_t)b << 32)));
    h = mix64(h ^ ((uint64_t)c | ((uint64_t)purpose << 32)));
    return mix64(h ^ lane);
}
static float rng_f(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t p, uint32_t l) {
    return (float)(rng_bits(seed, a, b, c, p, l) >> 40) * 0x1.0p-24f;
}
static double rng_d(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, uint32_t p, uint32_t l) {
    return (double)(rng_bits(seed, a, b, c, p, l) >> 11) * 0x1.0p-53;
}
enum { P_DMT = 1, P_EMIT = 2, P_BOUNCE = 3, P_PRUNE = 4 };

/* ------------------------------------------------------------------ transform.hpp / animation.hpp */
typedef struct { float x, y, z, w; } Q;
typedef struct { Q r; V t; float s; } X;
typedef struct { int frame; X xf; } KF;
static int q_eq(Q a, Q b) { return a.x == b.x && a.y == b.y && a.z == b.z && a.w == b.w; }
static int x_eq(X a, X b) { return q_eq(a.r, b.r) && veq(a.t, b.t) && a.s == b.s; }
static float q_norm(Q q) { return sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w); }  /* :17 */
static V rot(Q q, V v) {                                                                   /* :33-37 */
    const V u = v3(q.x, q.y, q.z);
    const V t = vmul(cross3(u, v), 2.0f);
    return vadd(vadd(v, vmul(t, q.w)), cross3(u, t));
}
static Q slerp(Q a, Q b, float t) {                                                        /* :43-61 */
    float c = a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
    if (c < 0.0f) { b.x = -b.x; b.y = -b.y; b.z = -b.z; b.w = -b.w; c = -c; }
    float ka, kb;
    if (c > 0.9995f) { ka = 1.0f - t; kb = t; }
    else {
        const float om = acosf(fminr(c, 1.0f));
        const float is = 1.0f / sinf(om);
        ka = sinf((1.0f - t) * om) * is;
        kb = sinf(t * om) * is;
    }
    Q r = {ka * a.x + kb * b.x, ka * a.y + kb * b.y, ka * a.z + kb * b.z, ka * a.w + kb * b.w};
    const float n = q_norm(r);
    Q o = {r.x / n, r.y / n, r.z / n, r.w / n};
    return o;
}
static V apply(X xf, V p) { return vadd(rot(xf.r, vmul(p, xf.s)), xf.t); }               /* :72 */
static X lerp_x(X a, X b, float t) {                                                       /* :79-85 */
    X r;
    r.r = slerp(a.r, b.r, t);
    r.t = vadd(a.t, vmul(vsub(b.t, a.t), t));
    r.s = a.s + (b.s - a.s) * t;
    return r;
}
static Box xform_box(Box b, X xf) {                                                        /* :88-96 */
    Box o = box_empty();
    for (int i = 0; i < 8; ++i) {
        V c = v3((i & 1) ? b.hi.x : b.lo.x, (i & 2) ? b.hi.y : b.lo.y, (i & 4) ? b.hi.z : b.lo.z);
        box_pt(&o, apply(xf, c));
    }
    return o;
}
static X x_identity(void) { X x = {{0, 0, 0, 1}, {0, 0, 0}, 1.0f}; return x; }
static X xform_at(const KF* k, uint32_t n, int frame) {                                     /* animation.hpp:13-28 */
    if (n == 0) return x_identity();
    if (frame <= k[0].frame) return k[0].xf;
    if (frame >= k[n - 1].frame) return k[n - 1].xf;
    for (uint32_t i = 1; i < n; ++i) {
        if (frame <= k[i].frame) {
            if (frame == k[i].frame) return k[i].xf;
            const float t = (float)(frame - k[i - 1].frame) / (float)(k[i].frame - k[i - 1].frame);
            return lerp_x(k[i - 1].xf, k[i].xf, t);
        }
    }
    return k[n - 1].xf;
}

/* ------------------------------------------------------------------ lights (light.cpp) */
typedef struct { V pos, n, t, b; float s; } Pose;
static int pose_eq(Pose a, Pose b) {
    return veq(a.pos, b.pos) && veq(a.n, b.n) && veq(a.t, b.t) && veq(a.b, b.b) && a.s == b.s;
}
typedef struct {
    int kind;
    V flux;
    float cone, radius, hx, hy;
    KF* kf;
    uint32_t nkf;
} Light;
static Pose pose_at(const Light* L, int frame) {                                          /* :58-68 */
    const X xf = xform_at(L->kf, L->nkf, frame);
    Pose p;
    p.pos = xf.t;
    p.n = rot(xf.r, v3(0, 0, 1));
    p.t = rot(xf.r, v3(1, 0, 0));
    p.b = rot(xf.r, v3(0, 1, 0));
    p.s = xf.s;
    return p;
}
static int is_area(int k) { return k == PRX_LIGHT_DISC_AREA || k == PRX_LIGHT_RECT_AREA; }
static const double kTwoPi = 2.0 * 3.14159265358979323846;
static double cos_half(const Light* L) { return cos((double)L->cone * 3.14159265358979323846 / 360.0); } /* :36 */

static V dir_angles(Pose p, double ct, double phi) {                                       /* :40-47 */
    const double st = sqrt(dmaxr(0.0, 1.0 - ct * ct));
    double sp, cp;
    sincos(phi, &sp, &cp);
    const double cx = cp * st, cy = sp * st;
    return norm3(vadd(vadd(vmul(p.t, (float)cx), vmul(p.b, (float)cy)), vmul(p.n, (float)ct)));
}
static double wrap_unit(double v) { v -= floor(v); if (v >= 1.0) v = 0.0; return v; }       /* :49-53 */
static double clampd(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }

static void warp(const Light* L, Pose p, const float c[4], V* o, V* d) {                  /* :70-117 */
    switch (L->kind) {
        case PRX_LIGHT_POINT:
            *o = p.pos;
            *d = dir_angles(p, 1.0 - 2.0 * c[0], kTwoPi * c[1]);
            break;
        case PRX_LIGHT_SPOT:
            *o = p.pos;
            *d = dir_angles(p, 1.0 - (double)c[0] * (1.0 - cos_half(L)), kTwoPi * c[1]);
            break;
        case PRX_LIGHT_DISC_AREA: {
            const double rmax = (double)L->radius * p.s;
            const double r = rmax * sqrt((double)c[0]);
            double sp, cp;
            sincos(kTwoPi * c[1], &sp, &cp);
            *o = vadd(vadd(p.pos, vmul(p.t, (float)(r * cp))), vmul(p.b, (float)(r * sp)));
            *d = dir_angles(p, sqrt(dmaxr(0.0, 1.0 - c[2])), kTwoPi * c[3]);
            break;
        }
        default: {
            const float hx = L->hx * p.s, hy = L->hy * p.s;
            *o = vadd(vadd(p.pos, vmul(p.t, (2.0f * c[0] - 1.0f) * hx)), vmul(p.b, (2.0f * c[1] - 1.0f) * hy));
            *d = dir_angles(p, sqrt(dmaxr(0.0, 1.0 - c[2])), kTwoPi * c[3]);
            break;
        }
    }
}

static int canon(const Light* L, Pose p, V o, V d, float c[4]) {                          /* :119-175 */
    c[0] = c[1] = c[2] = c[3] = 0.0f;
    const double dn = dot3(d, p.n), dt = dot3(d, p.t), db = dot3(d, p.b);
    const double phi = wrap_unit(atan2(db, dt) / kTwoPi);
    const double tol = 1e-4;
    if (L->kind == PRX_LIGHT_POINT) {
        c[0] = (float)clampd((1.0 - dn) / 2.0, 0.0, 1.0);
        c[1] = (float)phi;
        return 1;
    }
    if (L->kind == PRX_LIGHT_SPOT) {
        const double q = (1.0 - dn) / (1.0 - cos_half(L));
        if (q < 0.0 || q > 1.0) return 0;
        c[0] = (float)dminr(q, 1.0);
        c[1] = (float)phi;
        return 1;
    }
    const V rel = vsub(o, p.pos);
    const double lz = dot3(rel, p.n), lx = dot3(rel, p.t), ly = dot3(rel, p.b);
    if (L->kind == PRX_LIGHT_DISC_AREA) {
        const double rmax = (double)L->radius * p.s;
        if (fabs(lz) > tol * rmax) return 0;
        const double q = (lx * lx + ly * ly) / (rmax * rmax);
        if (q > 1.0 + tol) return 0;
        c[0] = (float)dminr(q, 1.0);
        c[1] = (float)wrap_unit(atan2(ly, lx) / kTwoPi);
    } else {
        const double hx = (double)L->hx * p.s, hy = (double)L->hy * p.s;
        if (fabs(lz) > tol * dmaxr(hx, hy)) return 0;
        const double u = (lx / hx + 1.0) / 2.0, v = (ly / hy + 1.0) / 2.0;
        if (u < -tol || u > 1.0 + tol || v < -tol || v > 1.0 + tol) return 0;
        c[0] = (float)clampd(u, 0.0, 1.0);
        c[1] = (float)clampd(v, 0.0, 1.0);
    }
    if (dn <= 0.0) return 0;
    c[2] = (float)clampd(1.0 - dn * dn, 0.0, 1.0);
    c[3] = (float)phi;
    return 1;
}

static uint32_t cell_of(const uint32_t* dims, uint32_t nd, const float c[4]) {              /* :177-186 */
    uint32_t cell = 0;
    for (uint32_t a = 0; a < nd; ++a) {
        uint32_t idx = (uint32_t)(c[a] * (float)dims[a]);
        if (idx >= dims[a]) idx = dims[a] - 1;
        cell = cell * dims[a] + idx;
    }
    return cell;
}

static void sample_cell(const Light* L, Pose p, const uint32_t* dims, uint32_t nd, uint32_t cell, uint64_t seed,
                        uint32_t path, uint32_t epoch, float c[4], V* o, V* d) {           /* :196-228 */
    float lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
    uint32_t rest = cell;
    for (int a = (int)nd - 1; a >= 0; --a) {
        const uint32_t idx = rest % dims[a];
        rest /= dims[a];
        lo[a] = (float)idx / (float)dims[a];
        hi[a] = (float)(idx + 1) / (float)dims[a];
    }
    c[0] = c[1] = c[2] = c[3] = 0.0f;
    for (uint32_t a = 0; a < nd; ++a) {
        const double u = rng_d(seed, path, epoch, 0, P_EMIT, a);
        const double w = (double)hi[a] - lo[a];
        const double m = dminr(0.4, 2e-5 / w);
        const double t = m + u * (1.0 - 2.0 * m);
        c[a] = (float)(lo[a] + t * w);
    }
    warp(L, p, c, o, d);
}

/* ------------------------------------------------------------------ pure functions */
double po_prune_probability(uint32_t c, uint32_t t) {                                      /* light.hpp:132 */
    if (c == 0 || c <= t) return 0.0;
    return (double)(c - t) / (double)c;
}
int po_energies_close(const float a[3], const float b[3], float th) {                      /* engine.hpp:34 */
    for (int ch = 0; ch < 3; ++ch) {
        const float delta = b[ch] - a[ch], bound = th * a[ch];
        if (delta < -bound || delta > bound) return 0;
    }
    return 1;
}
int po_encode_path_info(uint32_t cell, uint32_t seg, uint32_t start, int rep, int reuse, uint32_t* w) { /* photon_store.cpp:9 */
    if (cell >= (1u << 22)) return fail(PRX_E_OUT_OF_RANGE, "path info: cell id needs 22 bits");
    if (seg < 1 || seg > 16) return fail(PRX_E_OUT_OF_RANGE, "path info: segment count must be in 1..16");
    if (start > 15) return fail(PRX_E_OUT_OF_RANGE, "path info: retrace start must be in 0..15");
    uint32_t x = cell | ((seg - 1) << 22) | (start << 26);
    if (rep) x |= 1u << 30;
    if (reuse) x |= 1u << 31;
    *w = x;
    return 0;
}
void po_decode_path_info(uint32_t w, uint32_t out[5]) {                                    /* photon_store.cpp:22 */
    out[0] = w & ((1u << 22) - 1);
    out[1] = ((w >> 22) & 0xF) + 1;
    out[2] = (w >> 26) & 0xF;
    out[3] = (w >> 30) & 1;
    out[4] = (w >> 31) & 1;
}
void po_memory_footprint(uint64_t n, uint32_t bounces, const uint32_t* dims, uint32_t nd, int area,
                         double out[7]) {                                                   /* photon_store.cpp:38 */
    const double MiB = 1024.0 * 1024.0;
    uint64_t cells = 1;
    for (uint32_t i = 0; i < nd; ++i) cells *= dims[i];
    out[0] = 4.0 * (double)n / MiB;
    out[1] = area ? 12.0 * (double)n / MiB : 0.0;
    out[2] = 2.0 * 4.0 * (double)cells / MiB;
    out[3] = 4.0 * (double)n / MiB;
    out[4] = 32.0 * (double)n * bounces / MiB;
    out[5] = out[0] + out[1] + out[2] + out[3];
    out[6] = out[5] + out[4];
}

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}
/* select_paths_to_prune, engine.cpp:443-471 */
int po_select_paths_to_prune(const uint32_t* paths, size_t n, uint32_t dm_c, uint32_t dm_t, uint64_t seed,
                             uint32_t frame, uint32_t* out, size_t* count) {
    uint32_t* s = (uint32_t*)malloc((n ? n : 1) * 4);
    uint8_t* mark = (uint8_t*)calloc(n ? n : 1, 1);
    memcpy(s, paths, n * 4);
    qsort(s, n, 4, cmp_u32);
    const double prob = po_prune_probability(dm_c, dm_t);
    uint32_t surv = 0;
    for (size_t i = 0; i < n; ++i) {
        const float u = rng_f(seed, s[i], frame, 0, P_PRUNE, 0);
        if (prob > 0.0 && u < prob) mark[i] = 1;
        else ++surv;
    }
    for (size_t i = n; surv > dm_t && i-- > 0;)
        if (!mark[i]) { mark[i] = 1; --surv; }
    size_t k = 0;
    for (size_t i = 0; i < n; ++i)
        if (mark[i]) out[k++] = s[i];
    *count = k;
    free(s);
    free(mark);
    return 0;
}

/* ------------------------------------------------------------------ BVH (bvh.cpp) */
typedef struct { Box b; uint32_t left, first; uint16_t count, axis; } Node;

/* libstdc++'s std::nth_element (introselect with median-of-3 Hoare partitioning, heap
 * select fallback, final insertion sort) restated so the median-split partitions -- and
 * therefore the leaf order that fixes the BVH tie rule -- equal the reference's. */
typedef struct { const V* cent; int axis; } Cmp;
static int less_idx(const Cmp* c, uint32_t a, uint32_t b) {                               /* bvh.cpp:47-50 */
    const float ca = vget(c->cent[a], c->axis), cb = vget(c->cent[b], c->axis);
    if (ca != cb) return ca < cb;
    return a < b;
}
static void swp(uint32_t* a, uint32_t* b) { uint32_t t = *a; *a = *b; *b = t; }
static void median_to_first(const Cmp* c, uint32_t* r, uint32_t* a, uint32_t* b, uint32_t* d) {
    if (less_idx(c, *a, *b)) {
        if (less_idx(c, *b, *d)) swp(r, b);
        else if (less_idx(c, *a, *d)) swp(r, d);
        else swp(r, a);
    } else if (less_idx(c, *a, *d)) swp(r, a);
    else if (less_idx(c, *b, *d)) swp(r, d);
    else swp(r, b);
}
static uint32_t* unguarded_partition(const Cmp* c, uint32_t* first, uint32_t* last, uint32_t* pivot) {
    for (;;) {
        while (less_idx(c, *first, *pivot)) ++first;
        --last;
        while (less_idx(c, *pivot, *last)) --last;
        if (!(first < last)) return first;
        swp(first, last);
        ++first;
    }
}
static void push_heap_(const Cmp* c, uint32_t* f, long hole, long top, uint32_t val) {
    long parent = (hole - 1) / 2;
    while (hole > top && less_idx(c, f[parent], val)) {
        f[hole] = f[parent];
        hole = parent;
        parent = (hole - 1) / 2;
    }
    f[hole] = val;
}
static void adjust_heap(const Cmp* c, uint32_t* f, long hole, long len, uint32_t val) {
    const long top = hole;
    long second = hole;
    while (second < (len - 1) / 2) {
        second = 2 * (second + 1);
        if (less_idx(c, f[second], f[second - 1])) second--;
        f[hole] = f[second];
        hole = second;
    }
    if ((len & 1) == 0 && second == (len - 2) / 2) {
        second = 2 * (second + 1);
        f[hole] = f[second - 1];
        hole = second - 1;
    }
    push_heap_(c, f, hole, top, val);
}
static void make_heap_(const Cmp* c, uint32_t* f, uint32_t* l) {
    const long len = l - f;
    if (len < 2) return;
    long parent = (len - 2) / 2;
    for (;;) {
        adjust_heap(c, f, parent, len, f[parent]);
        if (parent == 0) return;
        parent--;
    }
}
static void heap_select(const Cmp* c, uint32_t* f, uint32_t* m, uint32_t* l) {
    make_heap_(c, f, m);
    for (uint32_t* i = m; i < l; ++i)
        if (less_idx(c, *i, *f)) {
            const uint32_t v = *i;
            *i = *f;
            adjust_heap(c, f, 0, m - f, v);
        }
}
static void insertion_sort(const Cmp* c, uint32_t* f, uint32_t* l) {
    if (f == l) return;
    for (uint32_t* i = f + 1; i != l; ++i) {
        const uint32_t v = *i;
        if (less_idx(c, v, *f)) {
            memmove(f + 1, f, (size_t)(i - f) * 4);
            *f = v;
        } else {
            uint32_t* last = i;
            uint32_t* next = i - 1;
            while (less_idx(c, v, *next)) { *last = *next; last = next; --next; }
            *last = v;
        }
    }
}
static void nth_element_(const Cmp* c, uint32_t* first, uint32_t* nth, uint32_t* last) {
    if (first == last || nth == last) return;
    long n = last - first, lg = 0;
    while (n >>= 1) ++lg;
    long depth = lg * 2;
    while (last - first > 3) {
        if (depth == 0) {
            heap_select(c, first, nth + 1, last);
            swp(first, nth);
            return;
        }
        --depth;
        uint32_t* mid = first + (last - first) / 2;
        median_to_first(c, first, first + 1, mid, last - 1);
        uint32_t* cut = unguarded_partition(c, first + 1, last, first);
        if (cut <= nth) first = cut;
        else last = cut;
    }
    insertion_sort(c, first, last);
}

typedef struct {
    Node* nodes;
    uint32_t n_nodes, cap;
    uint32_t* order;
    const Box* tb;
    const V* cent;
} Builder;
static uint32_t build_node(Builder* B, uint32_t begin, uint32_t end) {                     /* bvh.cpp:38-77 */
    const uint32_t idx = B->n_nodes++;
    Node* nd = &B->nodes[idx];
    memset(nd, 0, sizeof *nd);
    Box bounds = box_empty();
    for (uint32_t i = begin; i < end; ++i) box_box(&bounds, B->tb[B->order[i]]);
    B->nodes[idx].b = bounds;
    const uint32_t count = end - begin;
    if (count <= 4) {
        B->nodes[idx].first = begin;
        B->nodes[idx].count = (uint16_t)count;
        return idx;
    }
    Box cb = box_empty();
    for (uint32_t i = begin; i < end; ++i) box_pt(&cb, B->cent[B->order[i]]);
    const V ext = vsub(cb.hi, cb.lo);
    int axis = 0;
    if (ext.y > ext.x) axis = 1;
    if (ext.z > vget(ext, axis)) axis = 2;
    const uint32_t mid = begin + count / 2;
    Cmp c = {B->cent, axis};
    nth_element_(&c, B->order + begin, B->order + mid, B->order + end);
    B->nodes[idx].axis = (uint16_t)axis;
    const uint32_t l = build_node(B, begin, mid);
    const uint32_t r = build_node(B, mid, end);
    B->nodes[idx].left = l;
    B->nodes[idx].first = r;
    B->nodes[idx].count = 0;
    return idx;
}

/* ------------------------------------------------------------------ scene (scene.cpp) */
typedef struct {
    Tri* mesh;
    uint32_t n;
    int kind;
    V albedo;
    float gexp;
    KF* kf;
    uint32_t nkf;
    int dynamic;
    Box local;
} Obj;

struct po_scene {
    Obj* obj;
    uint32_t n_obj;
    Light* light;
    uint32_t n_light;
    prx_camera cam;
    int frames;
    Tri* st;          /* static world triangles, original order */
    uint32_t* st_obj;
    uint32_t n_st;
    Box world;
    Node* nodes;
    uint32_t n_nodes;
    uint32_t* perm;
    Tri* st_perm;     /* triangles in BVH order (bvh.cpp:24-26) */
};

static KF* copy_kf(const prx_keyframe* k, uint32_t n, uint32_t* n_out) {
    KF* out = (KF*)malloc(sizeof(KF) * (n ? n : 1));
    for (uint32_t i = 0; i < n; ++i) {
        out[i].frame = k[i].frame;
        out[i].xf.r.x = k[i].rotation.x;
        out[i].xf.r.y = k[i].rotation.y;
        out[i].xf.r.z = k[i].rotation.z;
        out[i].xf.r.w = k[i].rotation.w;
        out[i].xf.t = v3(k[i].translation.x, k[i].translation.y, k[i].translation.z);
        out[i].xf.s = k[i].scale;
    }
    if (n == 0) { out[0].frame = 0; out[0].xf = x_identity(); n = 1; }  /* scene.cpp:77 */
    *n_out = n;
    return out;
}

void po_scene_destroy(po_scene* s) {
    if (!s) return;
    for (uint32_t i = 0; i < s->n_obj; ++i) { free(s->obj[i].mesh); free(s->obj[i].kf); }
    for (uint32_t i = 0; i < s->n_light; ++i) free(s->light[i].kf);
    free(s->obj); free(s->light); free(s->st); free(s->st_obj); free(s->nodes); free(s->perm); free(s->st_perm);
    free(s);
}

/* finalize_scene, scene.cpp:63-113 (validation messages mirror the reference) */
int po_scene_create(const prx_scene_desc* d, po_scene** out) {
    if (d->n_objects == 0) return fail(PRX_E_SCENE, "scene: needs at least one object");
    if (d->n_lights == 0) return fail(PRX_E_SCENE, "scene: needs at least one light");
    po_scene* s = (po_scene*)calloc(1, sizeof *s);
    s->n_obj = d->n_objects;
    s->n_light = d->n_lights;
    s->obj = (Obj*)calloc(s->n_obj, sizeof(Obj));
    s->light = (Light*)calloc(s->n_light, sizeof(Light));
    s->cam = d->camera;
    s->frames = d->frames;
    uint32_t total = 0;
    for (uint32_t i = 0; i < s->n_obj; ++i) {
        const prx_object_desc* od = &d->objects[i];
        Obj* o = &s->obj[i];
        o->n = od->n_triangles;
        if (o->n == 0) { po_scene_destroy(s); return fail(PRX_E_SCENE, "object: empty mesh"); }
        o->mesh = (Tri*)malloc(sizeof(Tri) * o->n);
        for (uint32_t t = 0; t < o->n; ++t) {
            o->mesh[t].a = v3(od->mesh[t].a.x, od->mesh[t].a.y, od->mesh[t].a.z);
            o->mesh[t].b = v3(od->mesh[t].b.x, od->mesh[t].b.y, od->mesh[t].b.z);
            o->mesh[t].c = v3(od->mesh[t].c.x, od->mesh[t].c.y, od->mesh[t].c.z);
        }
        o->kind = od->material.kind;
        o->albedo = v3(od->material.albedo.x, od->material.albedo.y, od->material.albedo.z);
        o->gexp = od->material.glossy_exponent;
        o->kf = copy_kf(od->keyframes, od->n_keyframes, &o->nkf);
        o->dynamic = 0;
        for (uint32_t k = 1; k < o->nkf; ++k)
            if (!x_eq(o->kf[k].xf, o->kf[0].xf)) o->dynamic = 1;                /* animation.hpp:31 */
        o->local = box_empty();
        for (uint32_t t = 0; t < o->n; ++t) box_box(&o->local, tri_box(o->mesh[t]));
        if (!o->dynamic) total += o->n;
    }
    for (uint32_t i = 0; i < s->n_light; ++i) {
        const prx_light_desc* ld = &d->lights[i];
        Light* L = &s->light[i];
        L->kind = ld->kind;
        L->flux = v3(ld->flux.x, ld->flux.y, ld->flux.z);
        L->cone = ld->cone_angle_deg;
        L->radius = ld->radius;
        L->hx = ld->half_x;
        L->hy = ld->half_y;
        L->kf = copy_kf(ld->keyframes, ld->n_keyframes, &L->nkf);
    }
    s->st = (Tri*)malloc(sizeof(Tri) * (total ? total : 1));
    s->st_obj = (uint32_t*)malloc(4 * (total ? total : 1));
    s->world = box_empty();
    for (uint32_t i = 0; i < s->n_obj; ++i) {
        const Obj* o = &s->obj[i];
        const X xf0 = xform_at(o->kf, o->nkf, 0);
        if (o->dynamic) { box_box(&s->world, xform_box(o->local, xf0)); continue; }
        for (uint32_t t = 0; t < o->n; ++t) {
            Tri w = {apply(xf0, o->mesh[t].a), apply(xf0, o->mesh[t].b), apply(xf0, o->mesh[t].c)};
            s->st_obj[s->n_st] = i;
            s->st[s->n_st++] = w;
            box_box(&s->world, tri_box(w));
        }
    }
    if (s->n_st) {                                                                         /* bvh.cpp:13-36 */
        Box* tb = (Box*)malloc(sizeof(Box) * s->n_st);
        V* cent = (V*)malloc(sizeof(V) * s->n_st);
        for (uint32_t i = 0; i < s->n_st; ++i) {
            tb[i] = tri_box(s->st[i]);
            cent[i] = vdiv(vadd(vadd(s->st[i].a, s->st[i].b), s->st[i].c), 3.0f);
        }
        s->perm = (uint32_t*)malloc(4 * s->n_st);
        for (uint32_t i = 0; i < s->n_st; ++i) s->perm[i] = i;
        Builder B = {(Node*)malloc(sizeof(Node) * 2 * s->n_st), 0, 2 * s->n_st, s->perm, tb, cent};
        build_node(&B, 0, s->n_st);
        s->nodes = B.nodes;
        s->n_nodes = B.n_nodes;
        s->st_perm = (Tri*)malloc(sizeof(Tri) * s->n_st);
        for (uint32_t i = 0; i < s->n_st; ++i) s->st_perm[i] = s->st[s->perm[i]];
        free(tb);
        free(cent);
    }
    for (uint32_t i = 0; i < s->n_light; ++i) box_pt(&s->world, pose_at(&s->light[i], 0).pos);
    *out = s;
    return 0;
}

float po_scene_diagonal(const po_scene* s) { return len3(vsub(s->world.hi, s->world.lo)); }

int po_scene_bvh_permutation(const po_scene* s, uint32_t* out, size_t cap, size_t* count) {
    *count = s->n_st;
    if (out) memcpy(out, s->perm, 4 * (cap < s->n_st ? cap : s->n_st));
    return 0;
}

/* ------------------------------------------------------------------ placed state (state_at) */
typedef struct {
    uint32_t n_dyn;
    uint32_t* obj;      /* object id per placed dynamic */
    Tri** tris;         /* world triangles at the frame */
    Box* cur;
    Box* prev;
} Placed;

static void placed_free(Placed* P) {
    for (uint32_t j = 0; j < P->n_dyn; ++j) free(P->tris[j]);
    free(P->obj); free(P->tris); free(P->cur); free(P->prev);
    memset(P, 0, sizeof *P);
}

static void state_at(const po_scene* s, int frame, Placed* P) {                           /* scene.cpp:115-134 */
    placed_free(P);
    uint32_t n = 0;
    for (uint32_t i = 0; i < s->n_obj; ++i) n += s->obj[i].dynamic;
    P->n_dyn = n;
    P->obj = (uint32_t*)malloc(4 * (n ? n : 1));
    P->tris = (Tri**)malloc(sizeof(Tri*) * (n ? n : 1));
    P->cur = (Box*)malloc(sizeof(Box) * (n ? n : 1));
    P->prev = (Box*)malloc(sizeof(Box) * (n ? n : 1));
    uint32_t j = 0;
    for (uint32_t i = 0; i < s->n_obj; ++i) {
        const Obj* o = &s->obj[i];
        if (!o->dynamic) continue;
        const X now = xform_at(o->kf, o->nkf, frame);
        const X prv = xform_at(o->kf, o->nkf, frame > 0 ? frame - 1 : 0);
        P->obj[j] = i;
        P->tris[j] = (Tri*)malloc(sizeof(Tri) * o->n);
        for (uint32_t t = 0; t < o->n; ++t) {
            P->tris[j][t].a = apply(now, o->mesh[t].a);
            P->tris[j][t].b = apply(now, o->mesh[t].b);
            P->tris[j][t].c = apply(now, o->mesh[t].c);
        }
        P->cur[j] = xform_box(o->local, now);
        P->prev[j] = xform_box(o->local, prv);
        ++j;
    }
}

typedef struct { float t; uint32_t obj; V pos, n; } Hit;

/* Bvh::intersect, bvh.cpp:79-106 */
static int bvh_isect(const po_scene* s, V o, V d, float tmin, float* tmax, uint32_t* best, int any) {
    if (!s->n_nodes) return 0;
    uint32_t stack[64];
    int sp = 0, found = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        const Node* nd = &s->nodes[stack[--sp]];
        if (!ray_box(o, d, tmin, *tmax, nd->b)) continue;
        if (nd->count > 0) {
            for (uint32_t i = nd->first; i < nd->first + nd->count; ++i) {
                float t;
                if (isect_tri(o, d, tmin, *tmax, s->st_perm[i], &t)) {
                    found = 1;
                    *best = s->perm[i];
                    if (any) return 1;
                    *tmax = t;
                }
            }
        } else {
            stack[sp++] = nd->first;
            stack[sp++] = nd->left;
        }
    }
    return found;
}

/* brute_force_intersect, bvh.cpp:108-117 */
static int brute(const Tri* tris, uint32_t n, V o, V d, float tmin, float* tmax, uint32_t* best, int any) {
    int found = 0;
    for (uint32_t i = 0; i < n; ++i) {
        float t;
        if (isect_tri(o, d, tmin, *tmax, tris[i], &t)) {
            found = 1;
            *best = i;
            if (any) return 1;
            *tmax = t;
        }
    }
    return found;
}

static V geo_normal(Tri t) { return norm3(cross3(vsub(t.b, t.a), vsub(t.c, t.a))); }    /* geometry.hpp:64 */

/* intersect_scene, scene.cpp:136-168 */
static int isect_scene(const po_scene* s, const Placed* P, V o, V d, float tmin, Hit* h) {
    float tmax = FLT_MAX;
    uint32_t best;
    int found = 0;
    if (bvh_isect(s, o, d, tmin, &tmax, &best, 0)) {
        h->t = tmax;
        h->obj = s->st_obj[best];
        h->pos = vadd(o, vmul(d, tmax));
        h->n = geo_normal(s->st[best]);
        found = 1;
    }
    for (uint32_t j = 0; j < P->n_dyn; ++j) {
        if (!ray_box(o, d, tmin, tmax, P->cur[j])) continue;
        const uint32_t n = s->obj[P->obj[j]].n;
        if (brute(P->tris[j], n, o, d, tmin, &tmax, &best, 0)) {
            h->t = tmax;
            h->obj = P->obj[j];
            h->pos = vadd(o, vmul(d, tmax));
            h->n = geo_normal(P->tris[j][best]);
            found = 1;
        }
    }
    if (found && dot3(h->n, d) > 0.0f) h->n = vneg(h->n);
    return found;
}

/* occluded, scene.cpp:170-177 */
static int occluded(const po_scene* s, const Placed* P, V o, V d, float tmin, float tmax) {
    uint32_t best;
    float tm = tmax;
    if (bvh_isect(s, o, d, tmin, &tm, &best, 1)) return 1;
    for (uint32_t j = 0; j < P->n_dyn; ++j) {
        if (!ray_box(o, d, tmin, tmax, P->cur[j])) continue;
        tm = tmax;
        if (brute(P->tris[j], s->obj[P->obj[j]].n, o, d, tmin, &tm, &best, 1)) return 1;
    }
    return 0;
}

int po_intersect_batch(const po_scene* s, int frame, const float* rays, size_t n, float* hits) {
    Placed P;
    memset(&P, 0, sizeof P);
    state_at(s, frame, &P);
    for (size_t i = 0; i < n; ++i) {
        const float* r = rays + 8 * i;
        float* h = hits + 9 * i;
        Hit x;
        const V o = v3(r[0], r[1], r[2]), d = v3(r[3], r[4], r[5]);
        /* generic t_max: same procedure with the caller's bound */
        float tmax = r[7];
        uint32_t best;
        int found = 0;
        if (bvh_isect(s, o, d, r[6], &tmax, &best, 0)) {
            x.obj = s->st_obj[best]; x.n = geo_normal(s->st[best]); found = 1;
        }
        for (uint32_t j = 0; j < P.n_dyn; ++j) {
            if (!ray_box(o, d, r[6], tmax, P.cur[j])) continue;
            if (brute(P.tris[j], s->obj[P.obj[j]].n, o, d, r[6], &tmax, &best, 0)) {
                x.obj = P.obj[j]; x.n = geo_normal(P.tris[j][best]); found = 1;
            }
        }
        memset(h, 0, 9 * sizeof(float));
        if (!found) { uint32_t inv = 0xFFFFFFFFu; memcpy(&h[1], &inv, 4); continue; }
        if (dot3(x.n, d) > 0.0f) x.n = vneg(x.n);
        x.pos = vadd(o, vmul(d, tmax));
        h[0] = tmax;
        memcpy(&h[1], &x.obj, 4);
        h[3] = x.pos.x; h[4] = x.pos.y; h[5] = x.pos.z;
        h[6] = x.n.x; h[7] = x.n.y; h[8] = x.n.z;
    }
    placed_free(&P);
    return 0;
}

/* ------------------------------------------------------------------ engine (engine.cpp) */
enum { DEAD = 0, LIVE = 1, REPLACE = 2 };
typedef struct { float x, y, z, w; } F4;

typedef struct {
    const Light* L;
    uint32_t begin, end, nd, dims[4], cells;
    uint32_t *dm_t, *dm_c;
    V flux_pp;
    Pose prev, now;
    int moved;
} Block;

struct po_engine {
    const po_scene* s;
    prx_config cfg;
    uint32_t N, B;
    float eps;
    int frames_run;
    Block blk[PRX_MAX_LIGHTS];
    uint32_t n_blk;
    F4 *pos_obj, *energy, *in_dir, *out_dir, *origin, *emis, *canon;
    uint32_t *cell, *epoch, *path_info, *seg_flags, *pruned;
    uint8_t *meta, *rstart;
    uint32_t n_pruned;
    Placed placed;
    Box occ[256];
    uint32_t n_occ;
    uint32_t sb, se;   /* shard [sb, se) of the global path range (all paths by default) */
    uint8_t* mark;     /* sharded prune: 1 = marked, 2 = unmarked candidate */
};

/* block range intersected with the shard */
static uint32_t lo_of(const po_engine* e, const Block* b) { return b->begin > e->sb ? b->begin : e->sb; }
static uint32_t hi_of(const po_engine* e, const Block* b) { return b->end < e->se ? b->end : e->se; }

static size_t vi(const po_engine* e, uint32_t b, uint32_t p) { return (size_t)b * e->N + p; }
static V f4v(F4 f) { return v3(f.x, f.y, f.z); }
static F4 vf4(V v, float w) { F4 f = {v.x, v.y, v.z, w}; return f; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static uint32_t obj_of(const po_engine* e, size_t v) { return f2u(e->pos_obj[v].w); }

void po_engine_destroy(po_engine* e) {
    if (!e) return;
    for (uint32_t i = 0; i < e->n_blk; ++i) { free(e->blk[i].dm_t); free(e->blk[i].dm_c); }
    free(e->pos_obj); free(e->energy); free(e->in_dir); free(e->out_dir); free(e->origin); free(e->emis);
    free(e->canon); free(e->cell); free(e->epoch); free(e->path_info); free(e->seg_flags); free(e->pruned);
    free(e->meta); free(e->rstart); free(e->mark);
    placed_free(&e->placed);
    free(e);
}

/* Engine::Engine, engine.cpp:63-117 */
int po_engine_create(const po_scene* s, const prx_config* cfg, po_engine** out) {
    if (cfg->n_paths == 0) return fail(PRX_E_INVALID_ARGUMENT, "engine: n_paths must be positive");
    if (cfg->max_bounces < 1 || cfg->max_bounces > 16)
        return fail(PRX_E_INVALID_ARGUMENT, "engine: max_bounces must be in 1..16");
    po_engine* e = (po_engine*)calloc(1, sizeof *e);
    e->s = s;
    e->cfg = *cfg;
    e->N = cfg->n_paths;
    e->B = cfg->max_bounces;
    e->eps = 1e-4f * po_scene_diagonal(s);
    e->n_blk = s->n_light;
    const uint32_t base = e->N / s->n_light, extra = e->N % s->n_light;
    uint32_t next = 0;
    for (uint32_t li = 0; li < s->n_light; ++li) {
        Block* b = &e->blk[li];
        b->L = &s->light[li];
        const uint32_t count = base + (li < extra ? 1u : 0u);
        if (count == 0) { po_engine_destroy(e); return fail(PRX_E_INVALID_ARGUMENT, "engine: fewer paths than lights"); }
        b->begin = next;
        b->end = next + count;
        next = b->end;
        if (is_area(b->L->kind)) { b->nd = 4; for (int a = 0; a < 4; ++a) b->dims[a] = cfg->dm_dims[a]; }
        else { b->nd = 2; b->dims[0] = cfg->dm_dims[2]; b->dims[1] = cfg->dm_dims[3]; }
        uint64_t cells = 1;
        for (uint32_t a = 0; a < b->nd; ++a) {
            if (b->dims[a] == 0) { po_engine_destroy(e); return fail(PRX_E_INVALID_ARGUMENT, "init_dm_target: zero-sized DM axis"); }
            cells *= b->dims[a];
        }
        if (cells > (1u << 22)) { po_engine_destroy(e); return fail(PRX_E_INVALID_ARGUMENT, "init_dm_target: more than 2^22 DM cells"); }
        b->cells = (uint32_t)cells;
        b->dm_t = (uint32_t*)calloc(cells, 4);
        b->dm_c = (uint32_t*)calloc(cells, 4);
        for (uint32_t i = 0; i < count; ++i) {                                            /* light.cpp:230-252 */
            float c[4] = {0, 0, 0, 0};
            for (uint32_t a = 0; a < b->nd; ++a) c[a] = (float)rng_d(cfg->seed, i, 0, 0, P_DMT, a);
            b->dm_t[cell_of(b->dims, b->nd, c)]++;
        }
        b->flux_pp = vdiv(b->L->flux, (float)(double)count);                             /* engine.cpp:95-96 */
        b->now = pose_at(b->L, 0);
        b->prev = b->now;
    }
    const size_t nv = (size_t)e->N * e->B;
    e->pos_obj = (F4*)calloc(nv, sizeof(F4));
    e->energy = (F4*)calloc(nv, sizeof(F4));
    e->in_dir = (F4*)calloc(nv, sizeof(F4));
    e->out_dir = (F4*)calloc(nv, sizeof(F4));
    for (size_t v = 0; v < nv; ++v) e->pos_obj[v].w = u2f(0xFFFFFFFFu);
    e->origin = (F4*)calloc(e->N, sizeof(F4));
    e->emis = (F4*)calloc(e->N, sizeof(F4));
    for (uint32_t p = 0; p < e->N; ++p) e->emis[p].z = 1.0f;
    e->canon = (F4*)calloc(e->N, sizeof(F4));
    e->cell = (uint32_t*)calloc(e->N, 4);
    e->epoch = (uint32_t*)calloc(e->N, 4);
    e->path_info = (uint32_t*)calloc(e->N, 4);
    e->seg_flags = (uint32_t*)calloc(e->N, 4);
    e->pruned = (uint32_t*)calloc(e->N, 4);
    e->meta = (uint8_t*)calloc(e->N, 4);
    e->rstart = (uint8_t*)malloc(e->N);
    memset(e->rstart, 0xFF, e->N);
    e->mark = (uint8_t*)calloc(e->N, 1);
    e->sb = cfg->shard_begin;
    e->se = (cfg->shard_begin == 0 && cfg->shard_end == 0) ? e->N : cfg->shard_end;
    *out = e;
    return 0;
}

static const Block* block_of(const po_engine* e, uint32_t p) {
    for (uint32_t i = 0; i < e->n_blk; ++i)
        if (p >= e->blk[i].begin && p < e->blk[i].end) return &e->blk[i];
    return &e->blk[0];
}

/* Engine::truncate_path, engine.cpp:141-147 */
static void truncate_path(po_engine* e, uint32_t p, uint32_t k, int escaped) {
    for (uint32_t b = k; b < e->B; ++b) {
        const size_t v = vi(e, b, p);
        e->in_dir[v] = vf4(v3(0, 0, 0), 0);
        e->pos_obj[v].w = u2f(0xFFFFFFFFu);
        e->energy[v] = vf4(v3(0, 0, 0), 0);
    }
    e->meta[4 * p] = (uint8_t)k;
    e->meta[4 * p + 1] = escaped ? 1 : 0;
}

static V seg_origin(const po_engine* e, uint32_t p, uint32_t i) {                          /* engine.cpp:125 */
    return i == 0 ? f4v(e->origin[p]) : f4v(e->pos_obj[vi(e, i - 1, p)]);
}
static V seg_dir(const po_engine* e, uint32_t p, uint32_t i) {                             /* engine.cpp:130 */
    return i == 0 ? f4v(e->emis[p]) : f4v(e->out_dir[vi(e, i - 1, p)]);
}

/* Engine::sample_bounce, engine.cpp:159-170 (cosine_sample :25-32, phong :34-42) */
static V bounce(const po_engine* e, uint32_t obj, V n, V in, uint32_t p, uint32_t key) {
    const uint64_t seed = e->cfg.seed;
    const float u1 = rng_f(seed, p, e->epoch[p], key, P_BOUNCE, 0);
    const float u2 = rng_f(seed, p, e->epoch[p], key, P_BOUNCE, 1);
    const Obj* o = &e->s->obj[obj];
    V t, b;
    if (o->kind != PRX_MATERIAL_GLOSSY) {
        const float r = sqrtf(u1);
        const float phi = 2.0f * (float)3.14159265358979323846 * u2;
        const float z = sqrtf(fmaxr(0.0f, 1.0f - u1));
        float sp, cp;
        sincosf(phi, &sp, &cp);
        basis(n, &t, &b);
        return norm3(vadd(vadd(vmul(t, r * cp), vmul(b, r * sp)), vmul(n, z)));
    }
    const V mirror = norm3(vsub(in, vmul(n, 2.0f * dot3(in, n))));
    const float ct = powf(u1, 1.0f / (o->gexp + 1.0f));
    const float st = sqrtf(fmaxr(0.0f, 1.0f - ct * ct));
    const float phi = 2.0f * (float)3.14159265358979323846 * u2;
    float sp, cp;
    sincosf(phi, &sp, &cp);
    basis(mirror, &t, &b);
    V out = norm3(vadd(vadd(vmul(t, st * cp), vmul(b, st * sp)), vmul(mirror, ct)));
    if (dot3(out, n) <= 0.0f) out = mirror;
    return out;
}

static int is_dyn(const po_engine* e, uint32_t obj) { return obj != 0xFFFFFFFFu && e->s->obj[obj].dynamic; }

/* compute_flag_mask, engine.cpp:172-199 */
static uint32_t flag_mask(const po_engine* e, uint32_t p) {
    const uint32_t k = e->meta[4 * p], segs = k + e->meta[4 * p + 1];
    const float two_diag = 2.0f * po_scene_diagonal(e->s);
    uint32_t mask = 0;
    for (uint32_t i = 0; i < segs; ++i) {
        int f = 0;
        if (i > 0 && is_dyn(e, obj_of(e, vi(e, i - 1, p)))) f = 1;
        if (!f && i < k && is_dyn(e, obj_of(e, vi(e, i, p)))) f = 1;
        if (!f) {
            const V a = seg_origin(e, p, i);
            const V b = i < k ? f4v(e->pos_obj[vi(e, i, p)]) : vadd(a, vmul(seg_dir(e, p, i), two_diag));
            for (uint32_t j = 0; j < e->n_occ; ++j)
                if (seg_box(a, b, e->occ[j])) { f = 1; break; }
        }
        if (f) mask |= 1u << i;
    }
    return mask;
}

/* run_frame prelude, engine.cpp:202-232 */
int po_frame_update(po_engine* e, prx_frame_stats* st) {
    const int frame = e->frames_run++;
    state_at(e->s, frame, &e->placed);
    for (uint32_t i = 0; i < e->n_blk; ++i) {
        Block* b = &e->blk[i];
        b->prev = b->now;
        b->now = pose_at(b->L, frame);
        b->moved = frame > 0 && !pose_eq(b->now, b->prev);
    }
    e->n_occ = 0;
    if (frame > 0) {
        for (uint32_t j = 0; j < e->placed.n_dyn; ++j) {
            Box bx = e->placed.prev[j];
            box_box(&bx, e->placed.cur[j]);
            bx.lo = vsub(bx.lo, v3(e->eps, e->eps, e->eps));
            bx.hi = vadd(bx.hi, v3(e->eps, e->eps, e->eps));
            e->occ[e->n_occ++] = bx;
        }
    }
    e->n_pruned = 0;
    for (uint32_t p = e->sb; p < e->se; ++p) {
        e->meta[4 * p + 3] = 0;
        e->rstart[p] = 0xFF;
        if (e->cfg.record_flags) e->seg_flags[p] = 0;
    }
    if (e->cfg.mode == PRX_MODE_BASELINE) {                                                /* release_all_paths :149-157 */
        for (uint32_t p = e->sb; p < e->se; ++p) {
            truncate_path(e, p, 0, 0);
            e->meta[4 * p + 2] = DEAD;
        }
        for (uint32_t i = 0; i < e->n_blk; ++i) memset(e->blk[i].dm_c, 0, 4 * e->blk[i].cells);
    }
    if (st) {
        memset(st, 0, sizeof *st);
        st->frame = frame;
        st->mode = e->cfg.mode;
    }
    return 0;
}

/* stage_update_origins, engine.cpp:244-304 */
static void update_origins(po_engine* e, prx_frame_stats* st) {
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        Block* b = &e->blk[li];
        if (!b->moved) continue;
        const Pose ps = b->now;
        for (uint32_t p = lo_of(e, b); p < hi_of(e, b); ++p) {
            if (e->meta[4 * p + 2] != LIVE) continue;
            if (!is_area(b->L->kind)) {
                e->origin[p] = vf4(ps.pos, 0);
                if (e->meta[4 * p] > 0) {
                    const V to = vsub(f4v(e->pos_obj[p]), ps.pos);
                    const float dist = len3(to);
                    if (dist <= e->eps) { e->meta[4 * p + 2] = REPLACE; continue; }
                    const V dir = vdiv(to, dist);
                    e->emis[p] = vf4(dir, 0);
                    st->visibility_rays++;
                    if (occluded(e->s, &e->placed, ps.pos, dir, e->eps, dist - e->eps)) e->meta[4 * p + 2] = REPLACE;
                }
            } else if (e->meta[4 * p] > 0) {
                const V d = f4v(e->emis[p]);
                const float denom = dot3(d, ps.n);
                if (denom <= 1e-6f) { e->meta[4 * p + 2] = REPLACE; continue; }
                const float s = dot3(vsub(f4v(e->pos_obj[p]), ps.pos), ps.n) / denom;
                if (s <= 0.0f) { e->meta[4 * p + 2] = REPLACE; continue; }
                e->origin[p] = vf4(vsub(f4v(e->pos_obj[p]), vmul(d, s)), 0);
            } else {
                const float c[4] = {e->canon[p].x, e->canon[p].y, e->canon[p].z, e->canon[p].w};
                V o, d;
                warp(b->L, ps, c, &o, &d);
                e->origin[p] = vf4(o, 0);
            }
        }
    }
}

/* verify_path_error_based, engine.cpp:339-403 */
static void verify_error(po_engine* e, const Block* blk, uint32_t p, uint32_t flags, prx_frame_stats* st) {
    const uint32_t k = e->meta[4 * p], segs = k + e->meta[4 * p + 1];
    int force = 0;
    uint32_t i = 0;
    while (i < segs) {
        const int flagged = force || ((flags >> i) & 1u);
        force = 0;
        if (!flagged) { ++i; continue; }
        const V o = seg_origin(e, p, i), d = seg_dir(e, p, i);
        st->visibility_rays++;
        Hit h;
        const int hit = isect_scene(e->s, &e->placed, o, d, e->eps, &h);
        if (i == k) { if (hit) e->rstart[p] = (uint8_t)i; return; }
        if (!hit) { truncate_path(e, p, i, 1); return; }
        const size_t v = vi(e, i, p);
        const V stored = f4v(e->energy[v]);
        const V eprev = i == 0 ? blk->flux_pp : f4v(e->energy[vi(e, i - 1, p)]);
        const Obj* mo = &e->s->obj[h.obj];
        const V enew = vmulv(eprev, mo->albedo);
        const float a[3] = {stored.x, stored.y, stored.z}, bb[3] = {enew.x, enew.y, enew.z};
        if (mo->kind == PRX_MATERIAL_GLOSSY || !po_energies_close(a, bb, e->cfg.threshold)) {
            e->in_dir[v] = vf4(d, 0);
            e->pos_obj[v] = vf4(h.pos, u2f(h.obj));
            e->energy[v] = vf4(enew, e->cfg.gather_radius);
            e->out_dir[v] = vf4(bounce(e, h.obj, h.n, d, p, i + 1), 0);
            e->rstart[p] = (uint8_t)(i + 1);
            return;
        }
        const int close_pos = len3(vsub(h.pos, f4v(e->pos_obj[v]))) <= e->eps;
        e->in_dir[v] = vf4(d, 0);
        e->pos_obj[v] = vf4(h.pos, u2f(h.obj));
        if (i + 1 >= segs) return;
        if (close_pos && !mo->dynamic && !((flags >> (i + 1)) & 1u)) { i += 2; continue; }
        if (i + 1 < k) e->out_dir[v] = vf4(norm3(vsub(f4v(e->pos_obj[vi(e, i + 1, p)]), h.pos)), 0);
        force = 1;
        ++i;
    }
}

/* stage_occlusions, engine.cpp:306-337 */
static void occlusions(po_engine* e, prx_frame_stats* st) {
    if (e->n_occ == 0) return;
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        const Block* b = &e->blk[li];
        for (uint32_t p = lo_of(e, b); p < hi_of(e, b); ++p) {
            if (e->meta[4 * p + 2] != LIVE) continue;
            const uint32_t flags = flag_mask(e, p);
            if (e->cfg.record_flags) e->seg_flags[p] = flags;
            if (!flags) continue;
            if (e->cfg.mode == PRX_MODE_NAIVE) {
                uint32_t first = 0;
                while (!(flags & (1u << first))) ++first;
                e->rstart[p] = (uint8_t)first;
            } else {
                verify_error(e, b, p, flags, st);
            }
        }
    }
}

/* stage_compute_dm, engine.cpp:405-441 */
static void compute_dm(po_engine* e, prx_frame_stats* st) {
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        Block* b = &e->blk[li];
        memset(b->dm_c, 0, 4 * b->cells);
        for (uint32_t p = lo_of(e, b); p < hi_of(e, b); ++p) {
            const uint8_t status = e->meta[4 * p + 2];
            if (status == DEAD) continue;
            int ok = status == LIVE;
            if (ok) {
                float c[4];
                ok = canon(b->L, b->now, f4v(e->origin[p]), f4v(e->emis[p]), c);
                if (ok) {
                    e->canon[p].x = c[0]; e->canon[p].y = c[1]; e->canon[p].z = c[2]; e->canon[p].w = c[3];
                    e->cell[p] = cell_of(b->dims, b->nd, c);
                    b->dm_c[e->cell[p]]++;
                }
            }
            if (!ok) {
                truncate_path(e, p, 0, 0);
                e->meta[4 * p + 2] = DEAD;
                st->paths_replaced++;
            }
        }
    }
}

/* stage_prune, engine.cpp:473-497 */
static void prune(po_engine* e, prx_frame_stats* st) {
    const uint32_t frame = (uint32_t)(e->frames_run - 1);
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        Block* b = &e->blk[li];
        /* per-cell path lists in ascending path order (counting sort) */
        uint32_t* start = (uint32_t*)calloc(b->cells + 1, 4);
        for (uint32_t p = b->begin; p < b->end; ++p)
            if (e->meta[4 * p + 2] == LIVE) start[e->cell[p] + 1]++;
        for (uint32_t c = 0; c < b->cells; ++c) start[c + 1] += start[c];
        uint32_t* list = (uint32_t*)malloc(4 * (start[b->cells] ? start[b->cells] : 1));
        uint32_t* cur = (uint32_t*)malloc(4 * (b->cells ? b->cells : 1));
        memcpy(cur, start, 4 * b->cells);
        for (uint32_t p = b->begin; p < b->end; ++p)
            if (e->meta[4 * p + 2] == LIVE) list[cur[e->cell[p]]++] = p;
        uint32_t* out = (uint32_t*)malloc(4 * (start[b->cells] ? start[b->cells] : 1));
        for (uint32_t c = 0; c < b->cells; ++c) {
            if (b->dm_c[c] <= b->dm_t[c]) continue;
            size_t n;
            po_select_paths_to_prune(list + start[c], start[c + 1] - start[c], b->dm_c[c], b->dm_t[c],
                                     e->cfg.seed, frame, out, &n);
            for (size_t k = 0; k < n; ++k) {
                const uint32_t p = out[k];
                --b->dm_c[e->cell[p]];
                truncate_path(e, p, 0, 0);
                e->meta[4 * p + 2] = DEAD;
                e->pruned[e->n_pruned++] = p;
            }
        }
        free(start); free(list); free(cur); free(out);
    }
    qsort(e->pruned, e->n_pruned, 4, cmp_u32);
    st->paths_pruned = e->n_pruned;
}

/* stage_fill, engine.cpp:499-546 */
static int fill(po_engine* e, prx_frame_stats* st) {
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        Block* b = &e->blk[li];
        uint32_t slot = b->begin;
        for (uint32_t c = 0; c < b->cells; ++c) {
            uint32_t need = b->dm_t[c] > b->dm_c[c] ? b->dm_t[c] - b->dm_c[c] : 0;
            while (need > 0) {
                while (slot < b->end && e->meta[4 * slot + 2] != DEAD) ++slot;
                if (slot >= b->end) return fail(PRX_E_LOGIC, "fill: ran out of free path slots");
                const uint32_t p = slot;
                e->epoch[p] += 1;
                float cc[4];
                V o, d;
                sample_cell(b->L, b->now, b->dims, b->nd, c, e->cfg.seed, p, e->epoch[p], cc, &o, &d);
                e->origin[p] = vf4(o, 0);
                e->emis[p] = vf4(d, 0);
                e->canon[p].x = cc[0]; e->canon[p].y = cc[1]; e->canon[p].z = cc[2]; e->canon[p].w = cc[3];
                e->cell[p] = c;
                e->meta[4 * p] = 0;
                e->meta[4 * p + 1] = 0;
                e->meta[4 * p + 2] = LIVE;
                e->meta[4 * p + 3] = 1;
                e->rstart[p] = 0;
                st->paths_filled++;
                ++slot;
                --need;
            }
            if (b->dm_c[c] < b->dm_t[c]) b->dm_c[c] = b->dm_t[c];
        }
    }
    return 0;
}

/* stage_trace + refresh_path_info, engine.cpp:548-610 */
static void trace(po_engine* e, prx_frame_stats* st) {
    uint64_t traced = 0, segments = 0;
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        const Block* blk = &e->blk[li];
        for (uint32_t p = lo_of(e, blk); p < hi_of(e, blk); ++p) {
            if (e->meta[4 * p + 2] != LIVE) continue;
            const uint8_t start = e->rstart[p];
            if (start != 0xFF) {
                uint32_t b = start;
                V pos = seg_origin(e, p, b), dir = seg_dir(e, p, b);
                V en = b == 0 ? blk->flux_pp : f4v(e->energy[vi(e, b - 1, p)]);
                int escaped = 0;
                while (b < e->B) {
                    ++traced;
                    Hit h;
                    if (!isect_scene(e->s, &e->placed, pos, dir, e->eps, &h)) { escaped = 1; break; }
                    en = vmulv(en, e->s->obj[h.obj].albedo);
                    const size_t v = vi(e, b, p);
                    e->in_dir[v] = vf4(dir, 0);
                    e->pos_obj[v] = vf4(h.pos, u2f(h.obj));
                    e->energy[v] = vf4(en, e->cfg.gather_radius);
                    const V out = bounce(e, h.obj, h.n, dir, p, b + 1);
                    e->out_dir[v] = vf4(out, 0);
                    pos = h.pos;
                    dir = out;
                    ++b;
                }
                truncate_path(e, p, b, escaped);
            }
            const uint32_t segs = e->meta[4 * p] + e->meta[4 * p + 1];
            segments += segs;
            const uint32_t rs = e->rstart[p];
            uint32_t w;
            po_encode_path_info(e->cell[p], segs > 1 ? segs : 1, rs == 0xFF ? 0 : (rs < 15 ? rs : 15), 0,
                                e->meta[4 * p + 3] == 0, &w);
            e->path_info[p] = w;
        }
    }
    st->rays_traced += traced;
    st->rays_reused = segments - st->rays_traced;
}

int po_run_stage(po_engine* e, int stage, prx_frame_stats* st) {
    const int active = e->cfg.mode != PRX_MODE_BASELINE && e->frames_run - 1 > 0;
    switch (stage) {
        case PRX_STAGE_UPDATE_ORIGINS: if (active) update_origins(e, st); return 0;
        case PRX_STAGE_OCCLUSIONS: if (active) occlusions(e, st); return 0;
        case PRX_STAGE_COMPUTE_DM: compute_dm(e, st); return 0;
        case PRX_STAGE_PRUNE: if (e->cfg.mode != PRX_MODE_BASELINE) prune(e, st); return 0;
        case PRX_STAGE_FILL: return fill(e, st);
        case PRX_STAGE_TRACE: trace(e, st); return 0;
    }
    return fail(PRX_E_INVALID_ARGUMENT, "unknown stage");
}

/* Engine::run_frame, engine.cpp:201-242 */
int po_run_frame(po_engine* e, prx_frame_stats* st) {
    int rc = po_frame_update(e, st);
    for (int stage = PRX_STAGE_UPDATE_ORIGINS; !rc && stage <= PRX_STAGE_TRACE; ++stage)
        rc = po_run_stage(e, stage, st);
    return rc;
}

/* ------------------------------------------------------------------ field I/O */
size_t po_field_bytes(const po_engine* e, int field, uint32_t index) {
    const size_t nv = (size_t)e->N * e->B;
    switch (field) {
        case PRX_FIELD_PHOTONS: return nv * 32;
        case PRX_FIELD_AUX: return nv * 24;
        case PRX_FIELD_POS_OBJ: case PRX_FIELD_ENERGY: case PRX_FIELD_IN_DIR: case PRX_FIELD_OUT_DIR: return nv * 16;
        case PRX_FIELD_ORIGIN: case PRX_FIELD_EMISSION_DIR: case PRX_FIELD_CANONICAL: return 16 * (size_t)e->N;
        case PRX_FIELD_CELL: case PRX_FIELD_EPOCH: case PRX_FIELD_PATH_INFO: case PRX_FIELD_META:
        case PRX_FIELD_SEGMENT_FLAGS: return 4 * (size_t)e->N;
        case PRX_FIELD_RETRACE_START: return e->N;
        case PRX_FIELD_DM_TARGET: case PRX_FIELD_DM_CURRENT:
            return index < e->n_blk ? 4 * (size_t)e->blk[index].cells : 0;
        case PRX_FIELD_PRUNED: return 4 * (size_t)e->n_pruned;
    }
    return 0;
}

static void* field_ptr(const po_engine* e, int field, uint32_t index) {
    switch (field) {
        case PRX_FIELD_POS_OBJ: return e->pos_obj;
        case PRX_FIELD_ENERGY: return e->energy;
        case PRX_FIELD_IN_DIR: return e->in_dir;
        case PRX_FIELD_OUT_DIR: return e->out_dir;
        case PRX_FIELD_ORIGIN: return e->origin;
        case PRX_FIELD_EMISSION_DIR: return e->emis;
        case PRX_FIELD_CANONICAL: return e->canon;
        case PRX_FIELD_CELL: return e->cell;
        case PRX_FIELD_EPOCH: return e->epoch;
        case PRX_FIELD_PATH_INFO: return e->path_info;
        case PRX_FIELD_META: return e->meta;
        case PRX_FIELD_SEGMENT_FLAGS: return e->seg_flags;
        case PRX_FIELD_RETRACE_START: return e->rstart;
        case PRX_FIELD_DM_TARGET: return e->blk[index].dm_t;
        case PRX_FIELD_DM_CURRENT: return e->blk[index].dm_c;
        case PRX_FIELD_PRUNED: return e->pruned;
    }
    return NULL;
}

int po_download(const po_engine* e, int field, uint32_t index, void* dst, size_t bytes) {
    if (bytes != po_field_bytes(e, field, index)) return fail(PRX_E_INVALID_ARGUMENT, "download: size mismatch");
    const size_t nv = (size_t)e->N * e->B;
    if (field == PRX_FIELD_PHOTONS) {                                                      /* photon_store.hpp:13 */
        float* o = (float*)dst;
        for (size_t v = 0; v < nv; ++v) {
            o[8 * v + 0] = e->in_dir[v].x; o[8 * v + 1] = e->in_dir[v].y; o[8 * v + 2] = e->in_dir[v].z;
            o[8 * v + 3] = e->pos_obj[v].w;
            o[8 * v + 4] = e->energy[v].x; o[8 * v + 5] = e->energy[v].y; o[8 * v + 6] = e->energy[v].z;
            o[8 * v + 7] = e->energy[v].w;
        }
        return 0;
    }
    if (field == PRX_FIELD_AUX) {
        float* o = (float*)dst;
        for (size_t v = 0; v < nv; ++v) {
            o[6 * v + 0] = e->pos_obj[v].x; o[6 * v + 1] = e->pos_obj[v].y; o[6 * v + 2] = e->pos_obj[v].z;
            o[6 * v + 3] = e->out_dir[v].x; o[6 * v + 4] = e->out_dir[v].y; o[6 * v + 5] = e->out_dir[v].z;
        }
        return 0;
    }
    const void* src = field_ptr(e, field, index);
    if (!src && bytes) return fail(PRX_E_INVALID_ARGUMENT, "unknown field");
    memcpy(dst, src, bytes);
    return 0;
}

int po_upload(po_engine* e, int field, uint32_t index, const void* src, size_t bytes) {
    if (bytes != po_field_bytes(e, field, index)) return fail(PRX_E_INVALID_ARGUMENT, "upload: size mismatch");
    if (field == PRX_FIELD_PHOTONS || field == PRX_FIELD_AUX || field == PRX_FIELD_PRUNED)
        return fail(PRX_E_INVALID_ARGUMENT, "upload: use the split vertex fields");
    void* dst = field_ptr(e, field, index);
    if (!dst) return fail(PRX_E_INVALID_ARGUMENT, "unknown field");
    memcpy(dst, src, bytes);
    return 0;
}

int po_set_frame_counter(po_engine* e, int frames_run) {
    e->frames_run = frames_run;
    const int last = frames_run > 0 ? frames_run - 1 : 0;
    for (uint32_t i = 0; i < e->n_blk; ++i) {
        e->blk[i].now = pose_at(e->blk[i].L, last);
        e->blk[i].prev = e->blk[i].now;
    }
    state_at(e->s, last, &e->placed);
    return 0;
}

/* ------------------------------------------------------------------ gather (gather.cpp) */
typedef struct { uint64_t key; uint32_t idx; } KeyIdx;
static int cmp_key(const void* a, const void* b) {
    const KeyIdx *x = (const KeyIdx*)a, *y = (const KeyIdx*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}
static int64_t gcoord(float v, float cs) { return (int64_t)floorf(v / cs); }              /* gather.hpp:63 */
static uint64_t gkey(int64_t x, int64_t y, int64_t z) {                                     /* gather.hpp:64-69 */
    return (((uint64_t)x & 0x1FFFFF) << 42) | (((uint64_t)y & 0x1FFFFF) << 21) | ((uint64_t)z & 0x1FFFFF);
}

/* gather_image, gather.cpp:35-75: a sorted (key, insertion index) array replaces the
 * unordered_map of per-cell vectors; per-cell visiting order is the same insertion order. */
int po_gather(po_engine* e, const prx_camera* cam, float radius, float* rgb) {
    if (!(radius > 0.0f)) return fail(PRX_E_INVALID_ARGUMENT, "gather: radius must be positive");
    const size_t nv = (size_t)e->N * e->B;
    size_t n = 0;
    for (size_t v = 0; v < nv; ++v) n += obj_of(e, v) != 0xFFFFFFFFu;
    V* pos = (V*)malloc(sizeof(V) * (n ? n : 1));
    V* en = (V*)malloc(sizeof(V) * (n ? n : 1));
    uint32_t* ob = (uint32_t*)malloc(4 * (n ? n : 1));
    KeyIdx* ki = (KeyIdx*)malloc(sizeof(KeyIdx) * (n ? n : 1));
    size_t k = 0;
    for (size_t v = 0; v < nv; ++v) {
        if (obj_of(e, v) == 0xFFFFFFFFu) continue;
        pos[k] = f4v(e->pos_obj[v]);
        en[k] = f4v(e->energy[v]);
        ob[k] = obj_of(e, v);
        ki[k].key = gkey(gcoord(pos[k].x, radius), gcoord(pos[k].y, radius), gcoord(pos[k].z, radius));
        ki[k].idx = (uint32_t)k;
        ++k;
    }
    qsort(ki, n, sizeof(KeyIdx), cmp_key);
    const float inv_area = 1.0f / ((float)3.14159265358979323846 * radius * radius);
    const float inv_pi = 1.0f / (float)3.14159265358979323846;
    const float r2 = radius * radius;
    /* camera_ray, gather.cpp:22-33 */
    const V cpos = v3(cam->position.x, cam->position.y, cam->position.z);
    const V fwd = norm3(vsub(v3(cam->look_at.x, cam->look_at.y, cam->look_at.z), cpos));
    V up = v3(0, 1, 0);
    if (fabsf(dot3(fwd, up)) > 0.999f) up = v3(1, 0, 0);
    const V right = norm3(cross3(fwd, up));
    const V upv = cross3(right, fwd);
    const float tan_half = tanf(cam->fov_deg * (float)3.14159265358979323846 / 360.0f);
    const float aspect = (float)cam->width / (float)cam->height;
    memset(rgb, 0, sizeof(float) * 3 * cam->width * cam->height);
    for (uint32_t pix = 0; pix < cam->width * cam->height; ++pix) {
        const uint32_t px = pix % cam->width, py = pix / cam->width;
        const float sx = (2.0f * (px + 0.5f) / cam->width - 1.0f) * tan_half * aspect;
        const float sy = (1.0f - 2.0f * (py + 0.5f) / cam->height) * tan_half;
        const V dir = norm3(vadd(vadd(fwd, vmul(right, sx)), vmul(upv, sy)));
        Hit h;
        if (!isect_scene(e->s, &e->placed, cpos, dir, 0.0f, &h)) continue;
        const V albedo = e->s->obj[h.obj].albedo;
        V rad = v3(0, 0, 0);
        const int64_t cx = gcoord(h.pos.x, radius), cy = gcoord(h.pos.y, radius), cz = gcoord(h.pos.z, radius);
        for (int64_t dz = -1; dz <= 1; ++dz)
            for (int64_t dy = -1; dy <= 1; ++dy)
                for (int64_t dx = -1; dx <= 1; ++dx) {
                    const uint64_t key = gkey(cx + dx, cy + dy, cz + dz);
                    size_t lo = 0, hi = n;                                                  /* lower_bound */
                    while (lo < hi) {
                        const size_t mid = (lo + hi) / 2;
                        if (ki[mid].key < key) lo = mid + 1;
                        else hi = mid;
                    }
                    for (size_t j = lo; j < n && ki[j].key == key; ++j) {
                        const uint32_t idx = ki[j].idx;
                        const V d = vsub(pos[idx], h.pos);
                        if (dot3(d, d) <= r2 && ob[idx] == h.obj) rad = vadd(rad, en[idx]);
                    }
                }
        const V out = vmul(vmul(vmulv(rad, albedo), inv_pi), inv_area);
        rgb[3 * pix] = out.x;
        rgb[3 * pix + 1] = out.y;
        rgb[3 * pix + 2] = out.z;
    }
    free(pos); free(en); free(ob); free(ki);
    return 0;
}

/* ------------------------------------------------------------------ sharded prune / fill
 * The single-engine stage_prune / stage_fill (engine.cpp:443-546) split at the exchange
 * points of SURVEY.md s8e; with one shard (prefix 0, total = local) they reduce to them. */
int po_prune_count(po_engine* e, uint32_t** unmarked) {
    const uint32_t frame = (uint32_t)(e->frames_run - 1);
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        const Block* b = &e->blk[li];
        memset(unmarked[li], 0, 4 * b->cells);
        for (uint32_t p = lo_of(e, b); p < hi_of(e, b); ++p) {
            e->mark[p] = 0;
            if (e->meta[4 * p + 2] != LIVE) continue;
            const uint32_t c = e->cell[p];
            if (b->dm_c[c] <= b->dm_t[c]) continue;
            const double prob = po_prune_probability(b->dm_c[c], b->dm_t[c]);
            const float u = rng_f(e->cfg.seed, p, frame, 0, P_PRUNE, 0);
            if (prob > 0.0 && u < prob) e->mark[p] = 1;
            else { e->mark[p] = 2; unmarked[li][c]++; }
        }
    }
    return 0;
}

int po_prune_apply(po_engine* e, const uint32_t** prefix, const uint32_t** total, prx_frame_stats* st) {
    e->n_pruned = 0;
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        Block* b = &e->blk[li];
        uint32_t* seen = (uint32_t*)calloc(b->cells, 4);
        for (uint32_t p = lo_of(e, b); p < hi_of(e, b); ++p) {  /* ascending ids = per-cell rank */
            if (e->mark[p] != 2) continue;
            const uint32_t c = e->cell[p];
            const uint32_t rank = prefix[li][c] + seen[c]++;
            if (total[li][c] > b->dm_t[c] && rank >= b->dm_t[c]) e->mark[p] = 1;
        }
        free(seen);
        for (uint32_t p = lo_of(e, b); p < hi_of(e, b); ++p) {
            if (e->mark[p] != 1) continue;
            truncate_path(e, p, 0, 0);
            e->meta[4 * p + 2] = DEAD;
            e->pruned[e->n_pruned++] = p;
        }
        for (uint32_t c = 0; c < b->cells; ++c)
            if (b->dm_c[c] > b->dm_t[c]) b->dm_c[c] = total[li][c] < b->dm_t[c] ? total[li][c] : b->dm_t[c];
    }
    qsort(e->pruned, e->n_pruned, 4, cmp_u32);
    st->paths_pruned = e->n_pruned;
    return 0;
}

int po_fill_count(po_engine* e, uint32_t* dead) {
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        const Block* b = &e->blk[li];
        dead[li] = 0;
        for (uint32_t p = lo_of(e, b); p < hi_of(e, b); ++p) dead[li] += e->meta[4 * p + 2] == DEAD;
    }
    return 0;
}

int po_fill_apply(po_engine* e, const uint64_t* prefix, const uint64_t* total, prx_frame_stats* st) {
    for (uint32_t li = 0; li < e->n_blk; ++li) {
        Block* b = &e->blk[li];
        uint64_t need_total = 0;
        for (uint32_t c = 0; c < b->cells; ++c) need_total += b->dm_t[c] > b->dm_c[c] ? b->dm_t[c] - b->dm_c[c] : 0;
        if (need_total > total[li]) return fail(PRX_E_LOGIC, "fill: ran out of free path slots");
        uint64_t u = 0;  /* global unit index */
        uint32_t slot = lo_of(e, b);
        for (uint32_t c = 0; c < b->cells; ++c) {
            const uint32_t need = b->dm_t[c] > b->dm_c[c] ? b->dm_t[c] - b->dm_c[c] : 0;
            for (uint32_t k = 0; k < need; ++k, ++u) {
                if (u < prefix[li]) continue;            /* unit owned by a lower shard */
                while (slot < hi_of(e, b) && e->meta[4 * slot + 2] != DEAD) ++slot;
                if (slot >= hi_of(e, b)) break;          /* owned by a higher shard */
                const uint32_t p = slot++;
                e->epoch[p] += 1;
                float cc[4];
                V o, d;
                sample_cell(b->L, b->now, b->dims, b->nd, c, e->cfg.seed, p, e->epoch[p], cc, &o, &d);
                e->origin[p] = vf4(o, 0);
                e->emis[p] = vf4(d, 0);
                e->canon[p].x = cc[0]; e->canon[p].y = cc[1]; e->canon[p].z = cc[2]; e->canon[p].w = cc[3];
                e->cell[p] = c;
                e->meta[4 * p] = 0; e->meta[4 * p + 1] = 0; e->meta[4 * p + 2] = LIVE; e->meta[4 * p + 3] = 1;
                e->rstart[p] = 0;
                st->paths_filled++;
            }
        }
        for (uint32_t c = 0; c < b->cells; ++c)
            if (b->dm_c[c] < b->dm_t[c]) b->dm_c[c] = b->dm_t[c];
    }
    return 0;
}
