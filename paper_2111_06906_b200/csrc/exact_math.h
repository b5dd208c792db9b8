// exact_math.h -- host/device scalar math with the reference's exact IEEE semantics.
//
// Every routine here reproduces the operation order and precision of the reference
// (/root/reference/proj) so that, compiled with --fmad=false and IEEE div/sqrt on the
// device and without FMA contraction on the host, the GPU engine produces bit-identical
// floats.  Citations are file:line of the reference function each routine follows.
#pragma once

#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define PRX_HD __host__ __device__ __forceinline__
#else
#define PRX_HD inline
#endif

namespace prx {

// ---------------------------------------------------------------- vectors (vec3.hpp)
struct V3 {
    float x, y, z;
};

PRX_HD V3 mk(float x, float y, float z) { return V3{x, y, z}; }
PRX_HD V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
PRX_HD V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
PRX_HD V3 mul(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
PRX_HD V3 mulv(V3 a, V3 b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
PRX_HD V3 divs(V3 a, float s) { return {a.x / s, a.y / s, a.z / s}; }
PRX_HD V3 neg(V3 a) { return {-a.x, -a.y, -a.z}; }
PRX_HD float comp(V3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }
PRX_HD bool eq(V3 a, V3 b) { return a.x == b.x && a.y == b.y && a.z == b.z; }

// vec3.hpp:45 -- ((ax*bx) + (ay*by)) + (az*bz)
PRX_HD float dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
// vec3.hpp:47-49
PRX_HD V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
// vec3.hpp:52
PRX_HD float length(V3 v) { return sqrtf(dot(v, v)); }
// vec3.hpp:54-57 -- sqrt then three true divisions (not a reciprocal multiply)
PRX_HD V3 normalized(V3 v) { return divs(v, length(v)); }

// std::min / std::max semantics (return the first argument unless the second is strictly
// smaller / larger) -- matters for signed zeros, used by Aabb::expand (geometry.hpp:28-35)
PRX_HD float fmin_std(float a, float b) { return (b < a) ? b : a; }
PRX_HD float fmax_std(float a, float b) { return (a < b) ? b : a; }
PRX_HD double dmin_std(double a, double b) { return (b < a) ? b : a; }
PRX_HD double dmax_std(double a, double b) { return (a < b) ? b : a; }
PRX_HD V3 vmin(V3 a, V3 b) { return {fmin_std(a.x, b.x), fmin_std(a.y, b.y), fmin_std(a.z, b.z)}; }
PRX_HD V3 vmax(V3 a, V3 b) { return {fmax_std(a.x, b.x), fmax_std(a.y, b.y), fmax_std(a.z, b.z)}; }

// vec3.hpp:74-80 (Duff et al. 2017 branchless basis)
PRX_HD void orthonormal_basis(V3 n, V3& t, V3& b) {
    const float sign = copysignf(1.0f, n.z);
    const float a = -1.0f / (sign + n.z);
    const float c = n.x * n.y * a;
    t = V3{1.0f + sign * n.x * n.x * a, sign * c, -sign * n.x};
    b = V3{c, sign + n.y * n.y * a, -n.y};
}

// ---------------------------------------------------------------- boxes (geometry.hpp)
struct Box {
    V3 lo, hi;
};
PRX_HD Box empty_box() {
    return Box{{3.402823466e+38f, 3.402823466e+38f, 3.402823466e+38f},
               {-3.402823466e+38f, -3.402823466e+38f, -3.402823466e+38f}};
}
PRX_HD void expand(Box& b, V3 p) {
    b.lo = vmin(b.lo, p);
    b.hi = vmax(b.hi, p);
}
PRX_HD void expand(Box& b, const Box& o) {
    b.lo = vmin(b.lo, o.lo);
    b.hi = vmax(b.hi, o.hi);
}
PRX_HD void inflate(Box& b, float amount) {  // geometry.hpp:36-39
    b.lo = sub(b.lo, mk(amount, amount, amount));
    b.hi = add(b.hi, mk(amount, amount, amount));
}

// ---------------------------------------------------------------- RNG (rng.hpp)
enum RngPurpose : uint32_t { kDmTargetInit = 1, kEmission = 2, kBounceDir = 3, kPruneMark = 4 };

// rng.hpp:27-32 (splitmix64 finaliser)
PRX_HD uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// rng.hpp:35-42, with the seed hash hoisted: seed_mix = mix64(seed)
PRX_HD uint64_t rng_bits_m(uint64_t seed_mix, uint32_t a, uint32_t b, uint32_t c,
                           uint32_t purpose, uint32_t lane) {
    uint64_t h = mix64(seed_mix ^ ((uint64_t)a | ((uint64_t)b << 32)));
    h = mix64(h ^ ((uint64_t)c | ((uint64_t)purpose << 32)));
    h = mix64(h ^ (uint64_t)lane);
    return h;
}
// rng.hpp:45-47: top 24 bits -> [0,1)
PRX_HD float rng_uniform_m(uint64_t seed_mix, uint32_t a, uint32_t b, uint32_t c,
                           uint32_t purpose, uint32_t lane) {
    return (float)(rng_bits_m(seed_mix, a, b, c, purpose, lane) >> 40) * 5.9604644775390625e-8f;
}
// The 24-bit integer behind rng_uniform (index into the exact-trig table).
PRX_HD uint32_t rng_u24_m(uint64_t seed_mix, uint32_t a, uint32_t b, uint32_t c,
                          uint32_t purpose, uint32_t lane) {
    return (uint32_t)(rng_bits_m(seed_mix, a, b, c, purpose, lane) >> 40);
}
// rng.hpp:51-53: 53 bits -> [0,1)
PRX_HD double rng_uniform_d_m(uint64_t seed_mix, uint32_t a, uint32_t b, uint32_t c,
                              uint32_t purpose, uint32_t lane) {
    return (double)(rng_bits_m(seed_mix, a, b, c, purpose, lane) >> 11) *
           1.1102230246251565404236316680908203125e-16;
}

// ---------------------------------------------------------------- primitives
// geometry.hpp:86-103 -- Moeller-Trumbore with the triangle pre-split into (a, e1, e2);
// e1 = b - a and e2 = c - a are exactly the reference's first two statements.
PRX_HD bool intersect_tri(V3 o, V3 d, float t_min, float t_max, V3 a, V3 e1, V3 e2,
                          float& t_out) {
    const float kEdgeEps = 1e-7f;
    const V3 pvec = cross(d, e2);
    const float det = dot(e1, pvec);
    if (fabsf(det) < 1e-12f) return false;
    const float inv_det = 1.0f / det;
    const V3 tvec = sub(o, a);
    const float u = dot(tvec, pvec) * inv_det;
    if (u < -kEdgeEps || u > 1.0f + kEdgeEps) return false;
    const V3 qvec = cross(tvec, e1);
    const float v = dot(d, qvec) * inv_det;
    if (v < -kEdgeEps || u + v > 1.0f + kEdgeEps) return false;
    const float t = dot(e2, qvec) * inv_det;
    if (t <= t_min || t >= t_max) return false;
    t_out = t;
    return true;
}

// geometry.hpp:107-134 -- closed segment vs closed box, double slab, lexicographic
// endpoint canonicalisation.
PRX_HD bool segment_box_exact(V3 a, V3 b, const Box& box) {
    bool swap = false;
    if (b.x != a.x) swap = b.x < a.x;
    else if (b.y != a.y) swap = b.y < a.y;
    else swap = b.z < a.z;
    if (swap) {
        const V3 t = a;
        a = b;
        b = t;
    }
    double t0 = 0.0, t1 = 1.0;
    for (int axis = 0; axis < 3; ++axis) {
        const double o = comp(a, axis);
        const double d = (double)comp(b, axis) - o;
        const double lo = comp(box.lo, axis);
        const double hi = comp(box.hi, axis);
        if (d == 0.0) {
            if (o < lo || o > hi) return false;
            continue;
        }
        double tn = (lo - o) / d;
        double tf = (hi - o) / d;
        if (tn > tf) {
            const double s = tn;
            tn = tf;
            tf = s;
        }
        t0 = dmax_std(t0, tn);
        t1 = dmin_std(t1, tf);
        if (t0 > t1) return false;
    }
    return true;
}

// geometry.hpp:136-154 -- ray vs closed box in double over [t_min, t_max].
PRX_HD bool ray_box_exact(V3 o3, V3 d3, float t_min, float t_max, const Box& box) {
    double t0 = t_min, t1 = t_max;
    for (int axis = 0; axis < 3; ++axis) {
        const double o = comp(o3, axis);
        const double d = comp(d3, axis);
        const double lo = comp(box.lo, axis);
        const double hi = comp(box.hi, axis);
        if (d == 0.0) {
            if (o < lo || o > hi) return false;
            continue;
        }
        double tn = (lo - o) / d;
        double tf = (hi - o) / d;
        if (tn > tf) {
            const double s = tn;
            tn = tf;
            tf = s;
        }
        t0 = dmax_std(t0, tn);
        t1 = dmin_std(t1, tf);
        if (t0 > t1) return false;
    }
    return true;
}

// engine.hpp:34-41 (Eq. 2)
PRX_HD bool energies_close(V3 e_old, V3 e_new, float threshold) {
    for (int ch = 0; ch < 3; ++ch) {
        const float delta = comp(e_new, ch) - comp(e_old, ch);
        const float bound = threshold * comp(e_old, ch);
        if (delta < -bound || delta > bound) return false;
    }
    return true;
}

// light.hpp:132-135 (Eq. 1)
PRX_HD double prune_probability(uint32_t dm_c, uint32_t dm_t) {
    if (dm_c == 0 || dm_c <= dm_t) return 0.0;
    return (double)(dm_c - dm_t) / (double)dm_c;
}

// photon_store.hpp:23-40 (range checks are the caller's; the GPU never violates them)
PRX_HD uint32_t pack_path_info(uint32_t cell, uint32_t seg_count, uint32_t retrace_start,
                               bool replace, bool reuse_light) {
    uint32_t w = cell;
    w |= (seg_count - 1u) << 22;
    w |= retrace_start << 26;
    if (replace) w |= 1u << 30;
    if (reuse_light) w |= 1u << 31;
    return w;
}

}  // namespace prx
