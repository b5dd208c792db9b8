// device_scene.cuh -- device-side scene, traversal and light math of the B200 engine.
//
// Everything here is __device__ code compiled with --fmad=false and IEEE div/sqrt, in the
// reference's operation order, so that the per-path results are bit-identical to the CPU
// reference.  Tie rules of intersect_scene (scene.cpp:136-168):
//   * static BVH first, visited in the reference tree's left-first DFS order with the
//     double-precision node test against the shrinking t_max (bvh.cpp:79-106);
//   * then every dynamic object in index order, gated by the double ray/box test of its
//     current bounds with the already-shrunk t_max (scene.cpp:153-155);
//   * inside a dynamic mesh the lexicographic minimum (t, triangle index) wins -- exactly
//     what brute_force_intersect's strict `<` yields (bvh.cpp:108-117).
#pragma once

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "dev_types.h"
#include "exact_trig.h"

namespace prx {

// --------------------------------------------------------------------------- rays
struct Hit {
    float t;
    uint32_t obj;
    V3 pos;
    V3 normal;
};

__device__ __forceinline__ V3 ld3(const float4 v) { return V3{v.x, v.y, v.z}; }

// Filtered exact ray/box test: a float slab test with a certified error margin decides
// the clear cases; anything inside the margin falls back to the reference's double test
// (ray_box_exact), so the boolean is always the reference's.
struct RayPre {
    V3 o, d;
    float inv[3];
    bool safe;  // all |d| components either 0 or large enough for the float filter
    bool regular;  // safe and no zero component: the fast culling slabs need no branches
};

// hide a per-ray flag from rematerialization (kept in a register instead of being re-derived
// from its inputs -- kernel parameters -- at every use in the traversal loop)
__device__ __forceinline__ void opaque_flag(bool& f) {
    uint32_t v = f ? 1u : 0u;
    asm volatile("mov.u32 %0, %0;" : "+r"(v));
    f = v != 0u;
}

__device__ __forceinline__ RayPre make_ray(V3 o, V3 d) {
    RayPre r;
    r.o = o;
    r.d = d;
    r.safe = true;
    r.regular = true;
    for (int a = 0; a < 3; ++a) {
        const float da = comp(d, a);
        r.inv[a] = da != 0.0f ? 1.0f / da : 0.0f;
        if (da != 0.0f && fabsf(da) < 1e-18f) r.safe = false;
        if (da == 0.0f) r.regular = false;
    }
    r.regular = r.regular && r.safe;
    return r;
}

// round(N / d) <= c (le) or c <= round(N / d) (!le) for the reference's double quotient
// (N = fl64(bound - o), d != 0) against a float c.  c * d is exact in double (24 x 24 bits),
// so one fma gives the exact sign of N - c * d, hence of N / d - c; rounding is monotone
// and c is representable, so that sign decides unless N / d lies within a few double ulps
// of c, where the quotient itself is computed.
static __device__ __noinline__ bool quot_cmp_const(double N, float d, float c, bool le) {
    const double dd = d, cd = c;
    const double res = fma(-cd, dd, N);  // sign(N - c d) exact
    if (fabs(res) <= fabs(cd) * fabs(dd) * 0x1p-48 + 0x1p-1000) {
        const double q = N / dd;
        return le ? (q <= cd) : (cd <= q);
    }
    const bool q_below_c = (dd > 0.0) ? (res < 0.0) : (res > 0.0);
    return le ? q_below_c : !q_below_c;
}

// Slow path of ray_box: decide max(lower) <= min(upper) pair by pair.  Lower candidates are
// t_min and the entry quotients, upper ones t_max and the exit quotients; a pair the float
// values settle is skipped, a float-vs-quotient pair is settled exactly by quot_cmp_const,
// and a quotient-vs-quotient pair falls back to the reference's double test.
static __device__ __noinline__ bool ray_box_refine(const RayPre r, float t_min, float t_max, const Box b) {
    float fn[3], ff[3];  // the float entry / exit quotients of ray_box
    for (int a = 0; a < 3; ++a) {
        const float da = comp(r.d, a), oa = comp(r.o, a);
        const float tn = (comp(b.lo, a) - oa) * r.inv[a];
        const float tf = (comp(b.hi, a) - oa) * r.inv[a];
        fn[a] = da == 0.0f ? 0.0f : (tn > tf ? tf : tn);
        ff[a] = da == 0.0f ? 0.0f : (tn > tf ? tn : tf);
    }
    for (int i = -1; i < 3; ++i) {
        if (i >= 0 && comp(r.d, i) == 0.0f) continue;
        const float li = i < 0 ? t_min : fn[i];
        for (int j = -1; j < 3; ++j) {
            if (j >= 0 && comp(r.d, j) == 0.0f) continue;
            const float uj = j < 0 ? t_max : ff[j];
            const float slack = 4.0e-7f * (fabsf(li) + fabsf(uj)) + 1e-30f;
            if (uj - li > slack) continue;  // certainly li <= uj
            if (li - uj > slack) return false;
            if (i < 0 && j < 0) {
                if (!(t_min <= t_max)) return false;
            } else if (i >= 0 && j >= 0) {
                return ray_box_exact(r.o, r.d, t_min, t_max, b);
            } else {
                const int a = i >= 0 ? i : j;
                const float da = comp(r.d, a), oa = comp(r.o, a);
                // entry bound is lo for d > 0, hi for d < 0; exit the other one
                const bool entry = i >= 0;
                const float bound = (entry == (da > 0.0f)) ? comp(b.lo, a) : comp(b.hi, a);
                const double N = (double)bound - (double)oa;
                // entry quotient <= t_max, or t_min <= exit quotient
                if (!quot_cmp_const(N, da, entry ? t_max : t_min, entry)) return false;
            }
        }
    }
    return true;
}

__device__ __forceinline__ bool ray_box(const RayPre& r, float t_min, float t_max, const Box& b) {
    if (!r.safe) return ray_box_exact(r.o, r.d, t_min, t_max, b);
    // Float slab: each quotient q = (bound - o) / d is approximated by f = fl(fl(bound - o)
    // * fl(1/d)), |f - q| <= 3 * 2^-24 * |f| (+ denormal slack).  The max/min over such
    // values inherit the bound, so |t0_f - t0| + |t1_f - t1| <= 1.8e-7 (|t0_f| + |t1_f|).
    float t0 = t_min, t1 = t_max;
    for (int a = 0; a < 3; ++a) {
        const float da = comp(r.d, a);
        const float oa = comp(r.o, a);
        const float lo = comp(b.lo, a), hi = comp(b.hi, a);
        if (da == 0.0f) {
            if (oa < lo || oa > hi) return false;
            continue;
        }
        float tn = (lo - oa) * r.inv[a];
        float tf = (hi - oa) * r.inv[a];
        if (tn > tf) {
            const float s = tn;
            tn = tf;
            tf = s;
        }
        t0 = fmax_std(t0, tn);
        t1 = fmin_std(t1, tf);
    }
    // reference: miss iff t0 > t1 (double); decide only outside the certified band
    const float slack = 4.0e-7f * (fabsf(t0) + fabsf(t1)) + 1e-30f;
    if (t0 - t1 > slack) return false;
    if (t1 - t0 > slack) return true;
    return ray_box_refine(r, t_min, t_max, b);
}

// Static BVH closest hit (bvh.cpp:79-106) -- identical visit order, identical culling.
__device__ __forceinline__ bool static_closest(const SceneDev& S, const RayPre& r, float t_min,
                                               float& t_max, uint32_t& best) {
    if (S.n_nodes == 0) return false;
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = 0;
    bool found = false;
    while (sp > 0) {
        const uint32_t ni = stack[--sp];
        const float4 A = __ldg(&S.nodes[2 * ni]);
        const float4 B = __ldg(&S.nodes[2 * ni + 1]);
        const Box box{{A.x, A.y, A.z}, {B.x, B.y, B.z}};
        if (!ray_box(r, t_min, t_max, box)) continue;
        const uint32_t a = __float_as_uint(A.w), b = __float_as_uint(B.w);
        if (a & kLeafBit) {
            const uint32_t first = a & ~kLeafBit;
            for (uint32_t i = first; i < first + b; ++i) {
                const float4 ta = __ldg(&S.stris[3 * i]);
                const float4 t1 = __ldg(&S.stris[3 * i + 1]);
                const float4 t2 = __ldg(&S.stris[3 * i + 2]);
                float t;
                if (intersect_tri(r.o, r.d, t_min, t_max, ld3(ta), ld3(t1), ld3(t2), t)) {
                    found = true;
                    best = i;
                    t_max = t;
                }
            }
        } else {
            stack[sp++] = b;  // right child
            stack[sp++] = a;  // left child (popped first)
        }
    }
    return found;
}

__device__ __forceinline__ bool static_any(const SceneDev& S, const RayPre& r, float t_min,
                                           float t_max) {
    if (S.n_nodes == 0) return false;
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        const uint32_t ni = stack[--sp];
        const float4 A = __ldg(&S.nodes[2 * ni]);
        const float4 B = __ldg(&S.nodes[2 * ni + 1]);
        const Box box{{A.x, A.y, A.z}, {B.x, B.y, B.z}};
        if (!ray_box(r, t_min, t_max, box)) continue;
        const uint32_t a = __float_as_uint(A.w), b = __float_as_uint(B.w);
        if (a & kLeafBit) {
            const uint32_t first = a & ~kLeafBit;
            for (uint32_t i = first; i < first + b; ++i) {
                const float4 ta = __ldg(&S.stris[3 * i]);
                const float4 t1 = __ldg(&S.stris[3 * i + 1]);
                const float4 t2 = __ldg(&S.stris[3 * i + 2]);
                float t;
                if (intersect_tri(r.o, r.d, t_min, t_max, ld3(ta), ld3(t1), ld3(t2), t)) return true;
            }
        } else {
            stack[sp++] = b;
            stack[sp++] = a;
        }
    }
    return false;
}

// Conservative float slab for LBVH culling (no exactness needed: the result of the
// object query is the lexicographic min (t, index), independent of visit order, so a
// node may only be skipped when it provably holds no accepted triangle).
__device__ __forceinline__ bool ray_box_conservative(const RayPre& r, float t_min, float t_max,
                                                     float4 lo, float4 hi) {
    float t0 = t_min, t1 = t_max;
    for (int a = 0; a < 3; ++a) {
        const float da = comp(r.d, a);
        const float oa = comp(r.o, a);
        const float l = a == 0 ? lo.x : (a == 1 ? lo.y : lo.z);
        const float h = a == 0 ? hi.x : (a == 1 ? hi.y : hi.z);
        if (da == 0.0f) {
            if (oa < l || oa > h) return false;
            continue;
        }
        if (!r.safe) continue;  // no culling on an axis the float filter cannot bound
        float tn = (l - oa) * r.inv[a];
        float tf = (h - oa) * r.inv[a];
        if (tn > tf) {
            const float s = tn;
            tn = tf;
            tf = s;
        }
        t0 = fmax_std(t0, tn);
        t1 = fmin_std(t1, tf);
    }
    return t0 - t1 <= 2.0e-6f * (fabsf(t0) + fabsf(t1)) + 1e-30f;
}


// Closest hit inside one dynamic object: the (t, index)-lexicographic minimum over its
// triangles with t in (t_min, t_max) -- brute_force_intersect's result (bvh.cpp:108-117).
// Postponed leaves: the node loop hands over to the leaf loop once PRX_LEAF_SHARE/8 of the
// active lanes hold a parked leaf (8: all of them, Aila & Laine's rule). Measured on C4:
// 3/8 beats "all" by ~4% (trace 5.17 -> 4.89 ms, occlusion stage 3.17 -> 2.89 ms); lanes
// without a leaf simply skip the leaf round and keep descending afterwards.
#ifndef PRX_LEAF_SHARE
#define PRX_LEAF_SHARE 3
#endif
__device__ __forceinline__ bool leaf_round_due(bool parked) {
    const unsigned act = __activemask();
    const unsigned have = __ballot_sync(act, parked);
    if (PRX_LEAF_SHARE >= 8) return have == act;
    return 8 * __popc(have) >= PRX_LEAF_SHARE * __popc(act);
}

template <bool kAny>
__device__ __forceinline__ bool fast_closest(const float4* __restrict__ nodes, const float4* __restrict__ tris,
                                             const RayPre& r, float t_min, float t_max, float& best_t,
                                             uint32_t& best_pos, float& t_cert, uint32_t root = 0);

__device__ __forceinline__ bool dyn_closest(const SceneDev& S, const DynObj& D, const RayPre& r,
                                            float t_min, float& t_max, uint32_t& best_tri) {
    if (S.fast && S.dfast && D.sah_root != kLbvhBrute) {
        // the (t, index) minimum over the object's triangles in the window: its subtree of the
        // combined SAH tree (fast_closest is exact over the triangles it is given)
        float bt, tc;
        uint32_t g;
        if (!fast_closest<false>(S.fnodes, S.datris, r, t_min, t_max, bt, g, tc, D.sah_root)) return false;
        best_tri = g - D.tri_begin;
        t_max = bt;
        return true;
    }
    bool found = false;
    const float4* T = S.dtris + 3ull * D.tri_begin;
    if (D.node_begin == kLbvhBrute) {
        for (uint32_t i = 0; i < D.tri_count; ++i) {
            float t;
            if (intersect_tri(r.o, r.d, t_min, t_max, ld3(__ldg(&T[3 * i])), ld3(__ldg(&T[3 * i + 1])),
                              ld3(__ldg(&T[3 * i + 2])), t)) {
                found = true;
                best_tri = i;
                t_max = t;
            }
        }
        return found;
    }
    // LBVH: nodes[node_begin + k], k < tri_count - 1 internal; children with kLeafBit are
    // leaves (index into the sorted leaf list).  Node = {lmin,l} {lmax,-} {rmin,r} {rmax,-}.
    const float4* N = S.dnodes + 4ull * D.node_begin;
    const uint32_t* L = S.dleaf + D.tri_begin;
    const float t_in = t_max;  // acceptance window is (t_min, t_in); ties -> lower index
    float best_t = t_in;
    uint32_t bi = 0xFFFFFFFFu;
    uint32_t stack[64];
    int sp = 0;
    if (D.tri_count == 1) {
        stack[sp++] = kLeafBit | 0;
    } else {
        stack[sp++] = 0;
    }
    while (sp > 0) {
        const uint32_t c = stack[--sp];
        if (c & kLeafBit) {
            const uint32_t i = L[c & ~kLeafBit];
            float t;
            // accept t < t_in; replace if t < best_t or (t == best_t and lower index)
            if (intersect_tri(r.o, r.d, t_min, t_in, ld3(__ldg(&T[3 * i])), ld3(__ldg(&T[3 * i + 1])),
                              ld3(__ldg(&T[3 * i + 2])), t)) {
                if (t < best_t || (t == best_t && i < bi)) {
                    best_t = t;
                    bi = i;
                }
            }
            continue;
        }
        const float4 lmin = __ldg(&N[4 * c]), lmax = __ldg(&N[4 * c + 1]);
        const float4 rmin = __ldg(&N[4 * c + 2]), rmax = __ldg(&N[4 * c + 3]);
        const bool hl = ray_box_conservative(r, t_min, best_t, lmin, lmax);
        const bool hr = ray_box_conservative(r, t_min, best_t, rmin, rmax);
        if (hr) stack[sp++] = __float_as_uint(rmin.w);
        if (hl) stack[sp++] = __float_as_uint(lmin.w);
    }
    if (bi != 0xFFFFFFFFu) {
        best_tri = bi;
        t_max = best_t;
        return true;
    }
    return false;
}

__device__ __forceinline__ bool dyn_any(const SceneDev& S, const DynObj& D, const RayPre& r,
                                        float t_min, float t_max) {
    if (S.fast && S.dfast && D.sah_root != kLbvhBrute) {
        float bt, tc;
        uint32_t g;
        return fast_closest<true>(S.fnodes, S.datris, r, t_min, t_max, bt, g, tc, D.sah_root);
    }
    const float4* T = S.dtris + 3ull * D.tri_begin;
    if (D.node_begin == kLbvhBrute) {
        for (uint32_t i = 0; i < D.tri_count; ++i) {
            float t;
            if (intersect_tri(r.o, r.d, t_min, t_max, ld3(__ldg(&T[3 * i])), ld3(__ldg(&T[3 * i + 1])),
                              ld3(__ldg(&T[3 * i + 2])), t))
                return true;
        }
        return false;
    }
    const float4* N = S.dnodes + 4ull * D.node_begin;
    const uint32_t* L = S.dleaf + D.tri_begin;
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = D.tri_count == 1 ? (kLeafBit | 0) : 0;
    while (sp > 0) {
        const uint32_t c = stack[--sp];
        if (c & kLeafBit) {
            const uint32_t i = L[c & ~kLeafBit];
            float t;
            if (intersect_tri(r.o, r.d, t_min, t_max, ld3(__ldg(&T[3 * i])), ld3(__ldg(&T[3 * i + 1])),
                              ld3(__ldg(&T[3 * i + 2])), t))
                return true;
            continue;
        }
        const float4 lmin = __ldg(&N[4 * c]), lmax = __ldg(&N[4 * c + 1]);
        const float4 rmin = __ldg(&N[4 * c + 2]), rmax = __ldg(&N[4 * c + 3]);
        if (ray_box_conservative(r, t_min, t_max, rmin, rmax)) stack[sp++] = __float_as_uint(rmin.w);
        if (ray_box_conservative(r, t_min, t_max, lmin, lmax)) stack[sp++] = __float_as_uint(lmin.w);
    }
    return false;
}

// --------------------------------------------------------------------------- resumable traversal
// One ray query of intersect_scene (scene.cpp:136-168) or occluded (:170-177) as a state
// machine advanced one BVH node (or one leaf) per trav_step().  Persistent kernels step
// many rays per lane and refill finished lanes, keeping SIMD lanes busy; visit order and
// culling are exactly those of the one-shot functions above, so results are identical.
struct Trav {
    RayPre r;
    float t_min, t_max;   // acceptance window (t_max shrinks in closest-hit mode)
    float t_in;           // dynamic object: window bound when the object started
    float obj_t;          // dynamic object: best t so far (lexicographic with obj_i)
    uint32_t obj_i;
    uint32_t best;        // static: BVH-order triangle; dynamic: object-local triangle
    uint32_t dj;          // dynamic object of `best`
    int32_t kind;         // -1 none, 0 static, 1 dynamic
    int32_t phase;        // -1 static BVH, j >= 0 dynamic object j, n_dyn = finished
    int32_t gate;         // dynamic: 0 = gate pending, 1 = inside the object's LBVH
    int32_t any;          // any-hit (occluded) mode
    int32_t sp;
    uint32_t stack[64];
};

__device__ __forceinline__ void trav_init(const SceneDev& S, Trav& T, V3 o, V3 d, float t_min, float t_max,
                                          bool any) {
    T.r = make_ray(o, d);
    if (!(t_min >= 0.0f)) T.r.regular = false;  // box_entry_fast's slack form assumes t_min >= 0
    T.t_min = t_min;
    T.t_max = t_max;
    T.kind = -1;
    T.any = any ? 1 : 0;
    T.gate = 0;
    T.sp = 0;
    if (S.n_nodes) {
        T.phase = -1;
        T.stack[T.sp++] = 0;
    } else {
        T.phase = 0;
    }
}

// Returns true when the query is finished (any-hit: T.kind >= 0 means occluded).
__device__ __forceinline__ bool trav_step(const SceneDev& S, Trav& T) {
    if (T.phase < 0) {  // static BVH, left-first DFS (bvh.cpp:79-106)
        if (T.sp == 0) {
            T.phase = 0;
            T.gate = 0;
            return S.fp->n_dyn == 0;
        }
        const uint32_t ni = T.stack[--T.sp];
        const float4 A = __ldg(&S.nodes[2 * ni]);
        const float4 B = __ldg(&S.nodes[2 * ni + 1]);
        const Box box{{A.x, A.y, A.z}, {B.x, B.y, B.z}};
        if (!ray_box(T.r, T.t_min, T.t_max, box)) return false;
        const uint32_t a = __float_as_uint(A.w), b = __float_as_uint(B.w);
        if (a & kLeafBit) {
            const uint32_t first = a & ~kLeafBit;
            for (uint32_t i = first; i < first + b; ++i) {
                const float4 ta = __ldg(&S.stris[3 * i]);
                const float4 t1 = __ldg(&S.stris[3 * i + 1]);
                const float4 t2 = __ldg(&S.stris[3 * i + 2]);
                float t;
                if (intersect_tri(T.r.o, T.r.d, T.t_min, T.t_max, ld3(ta), ld3(t1), ld3(t2), t)) {
                    T.kind = 0;
                    T.best = i;
                    if (T.any) return true;
                    T.t_max = t;
                }
            }
        } else {
            T.stack[T.sp++] = b;  // right child
            T.stack[T.sp++] = a;  // left child, popped first
        }
        return false;
    }
    const FrameParams* fp = S.fp;
    if ((uint32_t)T.phase >= fp->n_dyn) return true;
    const DynObj& D = fp->dyn[T.phase];
    const float4* Tr = S.dtris + 3ull * D.tri_begin;
    if (T.gate == 0) {  // scene.cpp:153-155 gate with the already-shrunk t_max
        if (!ray_box(T.r, T.t_min, T.t_max, D.cur)) {
            ++T.phase;
            return (uint32_t)T.phase >= fp->n_dyn;
        }
        if (D.node_begin == kLbvhBrute) {  // brute_force_intersect (bvh.cpp:108-117)
            for (uint32_t i = 0; i < D.tri_count; ++i) {
                float t;
                if (intersect_tri(T.r.o, T.r.d, T.t_min, T.t_max, ld3(__ldg(&Tr[3 * i])),
                                  ld3(__ldg(&Tr[3 * i + 1])), ld3(__ldg(&Tr[3 * i + 2])), t)) {
                    T.kind = 1;
                    T.dj = (uint32_t)T.phase;
                    T.best = i;
                    if (T.any) return true;
                    T.t_max = t;
                }
            }
            ++T.phase;
            return (uint32_t)T.phase >= fp->n_dyn;
        }
        T.gate = 1;
        T.sp = 0;
        T.stack[T.sp++] = D.tri_count == 1 ? (kLeafBit | 0u) : 0u;
        T.t_in = T.t_max;
        T.obj_t = T.t_max;
        T.obj_i = 0xFFFFFFFFu;
        return false;
    }
    if (T.sp == 0) {  // object finished: lexicographic (t, index) minimum
        if (T.obj_i != 0xFFFFFFFFu) {
            T.kind = 1;
            T.dj = (uint32_t)T.phase;
            T.best = T.obj_i;
            T.t_max = T.obj_t;
        }
        ++T.phase;
        T.gate = 0;
        return (uint32_t)T.phase >= fp->n_dyn;
    }
    const uint32_t c = T.stack[--T.sp];
    if (c & kLeafBit) {
        const uint32_t i = __ldg(&S.dleaf[D.tri_begin + (c & ~kLeafBit)]);
        float t;
        if (intersect_tri(T.r.o, T.r.d, T.t_min, T.t_in, ld3(__ldg(&Tr[3 * i])), ld3(__ldg(&Tr[3 * i + 1])),
                          ld3(__ldg(&Tr[3 * i + 2])), t)) {
            if (T.any) {
                T.kind = 1;
                T.dj = (uint32_t)T.phase;
                T.best = i;
                return true;
            }
            if (t < T.obj_t || (t == T.obj_t && i < T.obj_i)) {
                T.obj_t = t;
                T.obj_i = i;
            }
        }
        return false;
    }
    const float4* N = S.dnodes + 4ull * (D.node_begin + c);
    const float4 lmin = __ldg(&N[0]), lmax = __ldg(&N[1]);
    const float4 rmin = __ldg(&N[2]), rmax = __ldg(&N[3]);
    const float tb = T.any ? T.t_max : T.obj_t;
    if (ray_box_conservative(T.r, T.t_min, tb, rmin, rmax)) T.stack[T.sp++] = __float_as_uint(rmin.w);
    if (ray_box_conservative(T.r, T.t_min, tb, lmin, lmax)) T.stack[T.sp++] = __float_as_uint(lmin.w);
    return false;
}

// Hit record of a finished closest-hit query (scene.cpp:144-167)
__device__ __forceinline__ bool trav_hit(const SceneDev& S, const Trav& T, Hit& h) {
    if (T.kind < 0) return false;
    V3 e1, e2;
    if (T.kind == 0) {
        const float4 q1 = __ldg(&S.stris[3 * T.best + 1]);
        const float4 q2 = __ldg(&S.stris[3 * T.best + 2]);
        e1 = ld3(q1);
        e2 = ld3(q2);
        h.obj = __float_as_uint(q1.w);
    } else {
        const DynObj& D = S.fp->dyn[T.dj];
        const float4* Tr = S.dtris + 3ull * (D.tri_begin + T.best);
        e1 = ld3(__ldg(&Tr[1]));
        e2 = ld3(__ldg(&Tr[2]));
        h.obj = D.obj;
    }
    h.t = T.t_max;
    h.pos = add(T.r.o, mul(T.r.d, T.t_max));
    V3 n = normalized(cross(e1, e2));  // Triangle::geometric_normal (geometry.hpp:64)
    if (dot(n, T.r.d) > 0.0f) n = neg(n);
    h.normal = n;
    return true;
}

// --------------------------------------------------------------------------- fast exact static traversal
// The reference's Bvh::intersect (bvh.cpp:79-106) returns, among the triangles its left-first
// DFS visits, the one with the smallest (t, permutation position) -- DFS order IS permutation
// order.  If it visits the global (t, position)-minimum T*, that is its answer; it visits T*
// iff every ancestor of T*'s leaf passes the exact box test at the t_max it has there.  That
// t_max is the initial one or the t of a triangle found earlier, i.e. one with t > t* (an
// earlier hit with t <= t* would precede T* lexicographically), so it is at least the smallest
// accepted t above t*; the test is monotone in t_max, so it suffices that each ancestor passes
// at any bound tc <= that value (fast_closest's t_cert; at worst nextafter(t*)).
// static_fast finds T* with near-first ordering and conservative culling (boxes inflated by
// cull_pad, t window widened); static_cert tests T*'s reference leaf with the exact test,
// which implies every ancestor passes.  A ray whose certificate fails reruns the
// reference-order DFS (static_closest).
__device__ __forceinline__ float box_entry(const RayPre& r, float t_min, float t_lim, float4 A, float4 B,
                                           float pad) {
    float t0 = t_min, t1 = t_lim;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float d = comp(r.d, a), o = comp(r.o, a);
        const float lo = (a == 0 ? A.x : (a == 1 ? A.y : A.z)) - pad;
        const float hi = (a == 0 ? B.x : (a == 1 ? B.y : B.z)) + pad;
        if (d == 0.0f || !r.safe) {
            if (d == 0.0f && (o < lo || o > hi)) return INFINITY;
            continue;  // no culling on an axis the float slab cannot bound
        }
        float tn = (lo - o) * r.inv[a];
        float tf = (hi - o) * r.inv[a];
        if (tn > tf) {
            const float s = tn;
            tn = tf;
            tf = s;
        }
        t0 = fmax_std(t0, tn);
        t1 = fmin_std(t1, tf);
    }
    // relative slack covers the rounding of the slab quotients far from the ray origin
    return t0 - t1 <= 2.0e-6f * (fabsf(t0) + fabsf(t1)) ? t0 : INFINITY;
}

// box_entry for the fast (culling-only) walks.  Regular rays (no zero or tiny direction
// component) take a branch-free slab with single-instruction min/max; the others fall back
// to box_entry.  Same values and the same relative slack as box_entry.
#ifndef PRX_F32X2
#define PRX_F32X2 1
#endif
#ifndef PRX_SLACK_MUL
#define PRX_SLACK_MUL 1
#endif
#ifndef PRX_NODE_LD256
#define PRX_NODE_LD256 1
#endif
#ifndef PRX_NODE_L1_LAST
#define PRX_NODE_L1_LAST 1
#endif
#ifndef PRX_NODE_EVICT_LAST
#define PRX_NODE_EVICT_LAST 1
#endif
#ifndef PRX_SS_ADDR
#define PRX_SS_ADDR 1
#endif
#ifndef PRX_CACHE_CL
#define PRX_CACHE_CL 1  // the joint walk keeps cull_limit(best_t) instead of recomputing it
#endif
// packed fp32 pairs (sm_100 FADD2 / FMUL2): two IEEE single operations per instruction, the
// same per-lane rounding as the scalar forms
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2_slab(unsigned long long a, unsigned long long o,
                                                      unsigned long long inv) {  // (a - o) * inv
    return f2_mul(f2_sub(a, o), inv);
}

__device__ __forceinline__ float box_entry_fast(const RayPre& r, float t_min, float t_lim, float4 A, float4 B) {
    if (!r.regular) return box_entry(r, t_min, t_lim, A, B, 0.0f);
#if PRX_F32X2
    float tnx, tny, tfx, tfy;
    {
        const unsigned long long oxy = f2_pack(r.o.x, r.o.y), ixy = f2_pack(r.inv[0], r.inv[1]);
        f2_unpack(f2_slab(f2_pack(A.x, A.y), oxy, ixy), tnx, tny);
        f2_unpack(f2_slab(f2_pack(B.x, B.y), oxy, ixy), tfx, tfy);
    }
#else
    const float tnx = (A.x - r.o.x) * r.inv[0], tfx = (B.x - r.o.x) * r.inv[0];
    const float tny = (A.y - r.o.y) * r.inv[1], tfy = (B.y - r.o.y) * r.inv[1];
#endif
    const float tnz = (A.z - r.o.z) * r.inv[2], tfz = (B.z - r.o.z) * r.inv[2];
    const float t0 = fmaxf(fmaxf(t_min, fminf(tnx, tfx)), fmaxf(fminf(tny, tfy), fminf(tnz, tfz)));
    const float t1 = fminf(fminf(t_lim, fmaxf(tnx, tfx)), fminf(fmaxf(tny, tfy), fmaxf(tnz, tfz)));
#if PRX_SLACK_MUL
    // t0 >= t_min >= 0, so the relative slack t0 - t1 <= 2e-6 (|t0| + |t1|) is
    // t0 <= t1 (1 + 2e-6) / (1 - 2e-6) for t1 >= 0 (and a miss for t1 < 0): one product with a
    // slightly larger factor accepts a superset (the culling only has to be conservative)
    return t0 <= t1 * 1.000005f ? t0 : INFINITY;
#else
    return t0 - t1 <= 2.0e-6f * (fabsf(t0) + fabsf(t1)) ? t0 : INFINITY;
#endif
}

__device__ __forceinline__ float cull_limit(float best_t) { return best_t + 1e-4f * fabsf(best_t) + 1e-6f; }

#ifndef PRX_SHORT_STACK
#define PRX_SHORT_STACK 12
#endif
constexpr int kShortStack = PRX_SHORT_STACK;
constexpr int kMaxBlock = 256;  // every kernel that traverses launches <= 256 threads per block

// this thread's column of the block's shared short stack (entry k at [k * kMaxBlock])
__device__ __forceinline__ uint2* trav_short_stack() {
    __shared__ uint2 s_stack[kShortStack * kMaxBlock];
    return s_stack + threadIdx.x;
}

// a 64-byte node as two 256-bit loads (sm_100 LDG.256), optionally with an L2 evict-last hint
// that keeps the hot tree ahead of the streaming path records in L2
__device__ __forceinline__ void ld_node(const float4* N, float4& n0, float4& n1, float4& n2, float4& n3) {
#if PRX_NODE_EVICT_LAST && PRX_NODE_L1_LAST
#define PRX_LD256 "ld.global.nc.L1::evict_last.L2::evict_last.v8.f32"
#elif PRX_NODE_EVICT_LAST
#define PRX_LD256 "ld.global.nc.L2::evict_last.v8.f32"
#else
#define PRX_LD256 "ld.global.nc.v8.f32"
#endif
    asm(PRX_LD256 " {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(n0.x), "=f"(n0.y), "=f"(n0.z), "=f"(n0.w), "=f"(n1.x), "=f"(n1.y), "=f"(n1.z), "=f"(n1.w)
        : "l"(N));
    asm(PRX_LD256 " {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(n2.x), "=f"(n2.y), "=f"(n2.z), "=f"(n2.w), "=f"(n3.x), "=f"(n3.y), "=f"(n3.z), "=f"(n3.w)
        : "l"(N + 2));
#undef PRX_LD256
}

// a fast-tree triangle record (kFT = 4 float4: a, e1, e2, pad) as two 256-bit loads
__device__ __forceinline__ void ld_tri(const float4* T, float4& a, float4& e1, float4& e2) {
    float4 pad;
    ld_node(T, a, e1, e2, pad);
    (void)pad;
}

// global (t, position)-minimum over the triangles of a fast tree with t in (t_min, t_max).
// Static: the SAH tree (fast_bvh.cpp), position = reference permutation position; dynamic:
// the combined LBVH (lbvh.cu), position = global dynamic triangle index.  While-while
// traversal (Aila & Laine 2009) with postponed leaves: a lane that reaches a leaf parks it
// and keeps descending until every active lane of the warp holds a leaf, so triangle tests
// run warp-wide.  The result is the order-independent lexicographic minimum, so neither
// tree nor visit order matters.  kAny: stop at the first accepted triangle (any-hit).
//
// t_cert (closest mode) is a certificate bound: a value in (best_t, t_max] that does not exceed
// the smallest t > best_t of any accepted triangle.  Every hit with t <= cull_limit(best_t) is
// visited (culling only drops boxes entered beyond the limit at the time, which is larger),
// and the leaf window tracks the smallest such t above best_t, so
// min(that, cull_limit(best_t), t_max) is a valid bound.
#ifdef PRX_CERT_STATS  // diagnostic build only: [0] joint walks, [1] their certificate failures,
// [2]/[3] any-hit walks / failures, [4]/[5] static/dynamic inner nodes, [6]/[7] static/dynamic triangles
static __device__ unsigned long long g_cert_stats[8];
#define PRX_CERT_COUNT(k) atomicAdd(&g_cert_stats[k], 1ull)
#define PRX_CERT_ADD(k, v) atomicAdd(&g_cert_stats[k], (unsigned long long)(v))
#else
#define PRX_CERT_COUNT(k) ((void)0)
#define PRX_CERT_ADD(k, v) ((void)0)
#endif

template <bool kAny>
__device__ __forceinline__ bool fast_closest(const float4* __restrict__ nodes, const float4* __restrict__ tris,
                                             const RayPre& r, float t_min, float t_max, float& best_t,
                                             uint32_t& best_pos, float& t_cert, uint32_t root) {
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    best_t = t_max;
    best_pos = kNone;
    float second = t_max;  // smallest accepted t strictly above best_t seen so far
    bool found = false;
    // traversal stack {node, entry t}: the top kShortStack entries live in shared memory
    // (per-thread column, conflict-free), deeper ones in a local overflow array that the
    // usual traversal never touches -- a 64-deep local stack per thread would exceed L1 and
    // L2 at full occupancy and stream to DRAM.
    uint2* const ss = trav_short_stack();
    constexpr uint32_t stride = kMaxBlock;  // (compile-time: cheap shared addresses; blockDim.x <= kMaxBlock)
    uint2 overflow[64 - kShortStack];
    int sp = 0;
    uint32_t node = root;  // always an internal node
    uint32_t leaf = kNone;
    auto push = [&](uint32_t c, float ent) {
        const uint2 e = make_uint2(c, __float_as_uint(ent));
        if (sp < kShortStack) ss[sp * stride] = e;
        else overflow[sp - kShortStack] = e;
        ++sp;
    };
    auto pop = [&]() -> uint32_t {
        const float lim = cull_limit(best_t);
        while (sp > 0) {
            --sp;
            uint2 e;
            if (sp < kShortStack) e = ss[sp * stride];
            else e = overflow[sp - kShortStack];
            if (__uint_as_float(e.y) <= lim) return e.x;
        }
        return kNone;
    };
    while (node != kNone || leaf != kNone) {
        while (node != kNone && !(node & kLeafBit)) {
            const float4* N = nodes + 4ull * node;
            const float4 n0 = __ldg(&N[0]), n1 = __ldg(&N[1]), n2 = __ldg(&N[2]), n3 = __ldg(&N[3]);
            const uint32_t c0 = __float_as_uint(n0.w), c1 = __float_as_uint(n1.w);
            const float lim = cull_limit(best_t);
            const float tl = box_entry_fast(r, t_min, lim, n0, n1);  // boxes are pre-inflated
            const float tr = c1 != kNone ? box_entry_fast(r, t_min, lim, n2, n3) : INFINITY;
            const bool hl = tl != INFINITY, hr = tr != INFINITY, left_first = tl <= tr;
            uint32_t next = kNone;
            if (hl || hr) next = (hl && (left_first || !hr)) ? c0 : c1;
            if (hl && hr) push(left_first ? c1 : c0, left_first ? tr : tl);
            if (next != kNone && (next & kLeafBit) && leaf == kNone) {  // park the leaf
                leaf = next;
                next = kNone;
            }
            node = next != kNone ? next : pop();
            if (leaf_round_due(leaf != kNone)) break;
        }
        if (leaf == kNone && node != kNone && (node & kLeafBit)) {
            leaf = node;
            node = pop();
        }
        while (leaf != kNone) {
            const uint32_t first = (leaf & ~kLeafBit) >> 3, count = (leaf & 7u) + 1u;
            for (uint32_t k = first; k < first + count; ++k) {
                float4 ta, t1, t2;
                ld_tri(tris + (size_t)kFT * k, ta, t1, t2);
                const uint32_t pos = __float_as_uint(ta.w);
                float t;
                // window: (t_min, t_max) before the first hit, then up to the cull limit
                // (hits above best_t feed the certificate bound; ties go by position)
                const float lim = found ? fminf(cull_limit(best_t), t_max) : t_max;
                if (intersect_tri(r.o, r.d, t_min, lim, ld3(ta), ld3(t1), ld3(t2), t)) {
                    if (kAny) {
                        best_t = t;
                        best_pos = pos;
                        t_cert = t_max;
                        return true;
                    }
                    if (!found || t < best_t || (t == best_t && pos < best_pos)) {
                        if (found && t < best_t) second = best_t;
                        best_t = t;
                        best_pos = pos;
                        found = true;
                    } else if (t > best_t && t < second) {
                        second = t;
                    }
                }
            }
            leaf = kNone;
            if (node != kNone && (node & kLeafBit)) {
                leaf = node;
                node = pop();
            }
        }
    }
    t_cert = fminf(fminf(second, cull_limit(best_t)), t_max);
    return found;
}

// One walk over both fast trees (static SAH tree and combined dynamic LBVH): codes carry
// kTreeBit for the dynamic tree, and candidates compare as (t, tree, position) -- static
// before dynamic at equal t, which is intersect_scene's tie rule (the static hit shrinks
// t_max first and dynamic hits must be strictly nearer).  A hit in either tree culls both,
// so rays that hit a mover skip most of the static tree.  Returns the winner and a
// certificate bound as fast_closest (second = smallest accepted t above the winner over both
// trees, which bounds the reference's running t_max in either phase from below).
constexpr uint32_t kTreeBit = 0x40000000u;
#ifndef PRX_JOINT_STATIC_FIRST
#define PRX_JOINT_STATIC_FIRST 0
#endif
#ifndef PRX_LEAF_PREFETCH
#define PRX_LEAF_PREFETCH 0  // measured slower (profiles/r02_sweeps.md)
#endif
#ifndef PRX_FAR_PREFETCH
#define PRX_FAR_PREFETCH 0
#endif
// L1 prefetch of a parked leaf's triangles (48 B each, <= 8): the leaf round that tests them
// runs only once enough lanes hold a leaf, so the lines arrive while the node walk continues
__device__ __forceinline__ void prefetch_leaf(const SceneDev& S, uint32_t leaf) {
    const float4* tris = (leaf & kTreeBit) ? S.datris : S.ftris;
    const uint32_t first = (leaf & ~(kLeafBit | kTreeBit)) >> 3, count = (leaf & 7u) + 1u;
    const char* a = reinterpret_cast<const char*>(tris + (size_t)kFT * first);
    const char* e = a + 16u * kFT * count;
    for (const char* p = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(a) & ~uintptr_t(127)); p < e;
         p += 128)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <bool kAny>
__device__ __forceinline__ bool joint_closest(const SceneDev& S, const RayPre& r, float t_min, float t_max,
                                              float& best_t, uint32_t& best_tree, uint32_t& best_pos,
                                              float& t_cert, uint32_t& best_slot) {
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    best_t = t_max;
    best_pos = kNone;
    best_tree = 0;
    best_slot = 0;
    float second = t_max;
    bool found = false;
#if PRX_CACHE_CL
    float cl = cull_limit(best_t);  // cull_limit(best_t), updated with best_t
#define PRX_CL cl
#else
#define PRX_CL cull_limit(best_t)
#endif
#if PRX_SS_ADDR
    // the column's 32-bit shared address, kept (recomputing the generic->shared base costs
    // two S2R and a few ALU ops per push / pop)
    uint32_t ss_addr;  // (opaque to the compiler, so it is kept rather than rematerialized)
    asm volatile("mov.u32 %0, %1;" : "=r"(ss_addr) : "r"((uint32_t)__cvta_generic_to_shared(trav_short_stack())));
#else
    uint2* const ss = trav_short_stack();
#endif
    constexpr uint32_t stride = kMaxBlock;  // (compile-time: cheap shared addresses; blockDim.x <= kMaxBlock)
    uint2 overflow[64 - kShortStack];
    int sp = 0;
    auto push = [&](uint32_t c, float ent) {
        const uint2 e = make_uint2(c, __float_as_uint(ent));
#if PRX_SS_ADDR
        if (sp < kShortStack)
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(ss_addr + sp * stride * 8), "r"(e.x), "r"(e.y)
                         : "memory");
#else
        if (sp < kShortStack) ss[sp * stride] = e;
#endif
        else overflow[sp - kShortStack] = e;
        ++sp;
    };
    auto pop = [&]() -> uint32_t {
        const float lim = PRX_CL;
        while (sp > 0) {
            --sp;
            uint2 e;
#if PRX_SS_ADDR
            if (sp < kShortStack)
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(ss_addr + sp * stride * 8)
                             : "memory");
#else
            if (sp < kShortStack) e = ss[sp * stride];
#endif
            else e = overflow[sp - kShortStack];
            if (__uint_as_float(e.y) <= lim) return e.x;
        }
        return kNone;
    };
#if PRX_JOINT_STATIC_FIRST
    push(kTreeBit | S.dnode_off, t_min);  // dynamic root, after the static tree
    uint32_t node = 0u;        // static root
#else
    push(0u, t_min);                         // static root, after the (small) dynamic tree
    uint32_t node = kTreeBit | S.dnode_off;  // dynamic root
#endif
    uint32_t leaf = kNone;
#ifdef PRX_CERT_STATS
    uint32_t st_n[2] = {0, 0}, st_t[2] = {0, 0};
#endif
    while (node != kNone || leaf != kNone) {
        while (node != kNone && !(node & kLeafBit)) {
            const uint32_t tree = node & kTreeBit;
#ifdef PRX_CERT_STATS
            ++st_n[tree ? 1 : 0];
#endif
            const float4* N = S.fnodes + 4ull * (node & ~kTreeBit);  // (both trees: one node array)
#if PRX_NODE_LD256
            float4 n0, n1, n2, n3;
            ld_node(N, n0, n1, n2, n3);
#else
            const float4 n0 = __ldg(&N[0]), n1 = __ldg(&N[1]), n2 = __ldg(&N[2]), n3 = __ldg(&N[3]);
#endif
            const uint32_t c0 = __float_as_uint(n0.w) | tree, c1r = __float_as_uint(n1.w);
            const uint32_t c1 = c1r | tree;
            const float lim = PRX_CL;
            const float tl = box_entry_fast(r, t_min, lim, n0, n1);  // boxes are pre-inflated
            const float tr = c1r != kNone ? box_entry_fast(r, t_min, lim, n2, n3) : INFINITY;
            // near child next, far child pushed; one pop site for "both missed" and "parked"
            const bool hl = tl != INFINITY, hr = tr != INFINITY, left_first = tl <= tr;
            uint32_t next = kNone;
            if (hl || hr) next = (hl && (left_first || !hr)) ? c0 : c1;
            if (hl && hr) {
                const uint32_t far = left_first ? c1 : c0;
                push(far, left_first ? tr : tl);
#if PRX_FAR_PREFETCH
                if (!(far & kLeafBit))  // the deferred child's node, for when it is popped
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(
                        S.fnodes + 4ull * (far & ~kTreeBit)));
#endif
            }
            if (next != kNone && (next & kLeafBit) && leaf == kNone) {  // park the leaf
                leaf = next;
                next = kNone;
#if PRX_LEAF_PREFETCH
                prefetch_leaf(S, leaf);  // its triangles stream into L1 while the walk goes on
#endif
            }
            node = next != kNone ? next : pop();
            if (leaf_round_due(leaf != kNone)) break;
        }
        if (leaf == kNone && node != kNone && (node & kLeafBit)) {
            leaf = node;
            node = pop();
        }
        while (leaf != kNone) {
            const uint32_t tree = (leaf & kTreeBit) ? 1u : 0u;
            const float4* tris = tree ? S.datris : S.ftris;
            const uint32_t first = (leaf & ~(kLeafBit | kTreeBit)) >> 3, count = (leaf & 7u) + 1u;
#ifdef PRX_CERT_STATS
            st_t[tree] += count;
#endif
            for (uint32_t k = first; k < first + count; ++k) {
                float4 ta, t1, t2;
                ld_tri(tris + (size_t)kFT * k, ta, t1, t2);
                const uint32_t pos = __float_as_uint(ta.w);
                float t;
                const float lim = found ? fminf(PRX_CL, t_max) : t_max;
                if (intersect_tri(r.o, r.d, t_min, lim, ld3(ta), ld3(t1), ld3(t2), t)) {
                    if (kAny) {
                        best_t = t;
                        best_tree = tree;
                        best_pos = pos;
                        best_slot = k;
                        t_cert = t_max;
                        return true;
                    }
                    if (!found || t < best_t ||
                        (t == best_t && (tree < best_tree || (tree == best_tree && pos < best_pos)))) {
                        if (found && t < best_t) second = best_t;
                        best_t = t;
                        best_tree = tree;
                        best_pos = pos;
                        best_slot = k;
                        found = true;
#if PRX_CACHE_CL
                        cl = cull_limit(t);
#endif
                    } else if (t > best_t && t < second) {
                        second = t;
                    }
                }
            }
            leaf = kNone;
            if (node != kNone && (node & kLeafBit)) {
                leaf = node;
                node = pop();
            }
        }
    }
    t_cert = fminf(fminf(second, cull_limit(best_t)), t_max);
#undef PRX_CL
#ifdef PRX_CERT_STATS
    PRX_CERT_ADD(4, st_n[0]);
    PRX_CERT_ADD(5, st_n[1]);
    PRX_CERT_ADD(6, st_t[0]);
    PRX_CERT_ADD(7, st_t[1]);
#endif
    return found;
}

__device__ __forceinline__ bool static_fast(const SceneDev& S, const RayPre& r, float t_min, float t_max,
                                            float& best_t, uint32_t& best_pos, float& t_cert) {
    return fast_closest<false>(S.fnodes, S.ftris, r, t_min, t_max, best_t, best_pos, t_cert);
}

// Every ancestor of permutation position `pos` passes the reference's exact box test at
// t_lim iff its leaf does: node boxes are unions of their triangles' float bounds, so an
// ancestor box contains the leaf box, and the double slab test is monotone under box
// inclusion (fl(lo' - o) <= fl(lo - o) for lo' <= lo, division by d keeps the order, so the
// entry bound can only drop and the exit bound only rise).
// (the joint walk's form: the winner's fast-tree slot carries its reference leaf in ftris[kFT k + 2].w,
// one dependent load less than leaf_of[position])
__device__ __forceinline__ bool static_cert_slot(const SceneDev& S, const RayPre& r, float t_min, float t_lim,
                                                 uint32_t slot) {
    if (S.cert_off || !(t_min >= 0.0f)) return false;  // (t_min < 0: exact paths only)
    const uint32_t leaf = __float_as_uint(__ldg(&S.ftris[kFT * slot + 2]).w);
    const float4 A = __ldg(&S.nodes[2 * leaf]);
    const float4 B = __ldg(&S.nodes[2 * leaf + 1]);
    return ray_box(r, t_min, t_lim, Box{{A.x, A.y, A.z}, {B.x, B.y, B.z}});
}

__device__ __forceinline__ bool static_cert(const SceneDev& S, const RayPre& r, float t_min, float t_lim,
                                            uint32_t pos) {
    if (S.cert_off || !(t_min >= 0.0f)) return false;
    const uint32_t leaf = __ldg(&S.leaf_of[pos]);
    const float4 A = __ldg(&S.nodes[2 * leaf]);
    const float4 B = __ldg(&S.nodes[2 * leaf + 1]);
    return ray_box(r, t_min, t_lim, Box{{A.x, A.y, A.z}, {B.x, B.y, B.z}});
}

// static part of intersect_scene with the reference's exact result
__device__ __forceinline__ bool static_closest_exact(const SceneDev& S, const RayPre& r, float t_min, float& t_max,
                                                     uint32_t& best) {
    if (S.n_nodes == 0) return false;
    if (!S.fast) return static_closest(S, r, t_min, t_max, best);
    float bt, tc;
    uint32_t bp;
    if (!static_fast(S, r, t_min, t_max, bt, bp, tc)) return false;
    // the reference visits T*'s leaf with a t_max >= tc (see fast_closest)
    if (static_cert(S, r, t_min, tc, bp)) {
        t_max = bt;
        best = bp;
        return true;
    }
    return static_closest(S, r, t_min, t_max, best);
}

// static part of occluded: the reference answers true iff some accepted triangle has all
// ancestors passing the exact test at the (fixed) t_max, so the first accepted triangle the
// fast walk meets certifies a hit whenever its own path does.
__device__ __forceinline__ bool static_any_exact(const SceneDev& S, const RayPre& r, float t_min, float t_max) {
    if (S.n_nodes == 0) return false;
    if (!S.fast) return static_any(S, r, t_min, t_max);
    float bt, tc;
    uint32_t bp;
    if (!fast_closest<true>(S.fnodes, S.ftris, r, t_min, t_max, bt, bp, tc)) return false;
    if (static_cert(S, r, t_min, t_max, bp)) return true;
    return static_any(S, r, t_min, t_max);
}

// Dynamic phase of intersect_scene (scene.cpp:153-165): objects in order, each behind its
// exact gate at the running t_max, brute-force (t, index) minimum inside.
__device__ __forceinline__ int dyn_closest_seq(const SceneDev& S, const RayPre& r, float t_min, float& t_max,
                                               uint32_t& dj, uint32_t& dtri) {
    const FrameParams* fp = S.fp;
    int kind = -1;
    for (uint32_t j = 0; j < fp->n_dyn; ++j) {
        const DynObj& D = fp->dyn[j];
        if (!ray_box(r, t_min, t_max, D.cur)) continue;
        uint32_t bt;
        if (dyn_closest(S, D, r, t_min, t_max, bt)) {
            kind = 1;
            dj = j;
            dtri = bt;
        }
    }
    return kind;
}

// Certified fast form of the dynamic phase.  Without gates the sequential loop returns the
// (t, object, index)-lexicographic minimum over all dynamic triangles with t in (t_min, t_max):
// an object replaces the running winner only with a strictly smaller t, and triangle order
// inside an object breaks ties.  With gates, let (t*, j*, i*) be that minimum: every object
// before j* holds only hits with t > t*, so when j* is reached the running t_max is at least
// min(t_max, smallest dynamic hit above t*) >= tc (fast_closest's certificate bound), and if
// j*'s gate passes at tc it passes there too (the test is monotone in t_max); later objects
// cannot beat t* strictly.  So the minimum, found by one walk over the combined LBVH (global
// index order == (object, index) order), is the reference's answer whenever its object's
// gate passes at tc; otherwise rerun the sequential loop.
__device__ __forceinline__ int dyn_closest_exact(const SceneDev& S, const RayPre& r, float t_min, float& t_max,
                                                 uint32_t& dj, uint32_t& dtri) {
    const FrameParams* fp = S.fp;
    if (fp->n_dyn == 0) return -1;
    if (!S.fast || !S.dfast) return dyn_closest_seq(S, r, t_min, t_max, dj, dtri);
    float bt, tc;
    uint32_t g;
    if (!fast_closest<false>(S.fnodes, S.datris, r, t_min, t_max, bt, g, tc, S.dnode_off)) return -1;
    const uint32_t j = __ldg(&S.dtri_obj[g]);
    const DynObj& D = fp->dyn[j];
    if (!S.cert_off && t_min >= 0.0f && ray_box(r, t_min, tc, D.cur)) {
        t_max = bt;
        dj = j;
        dtri = g - D.tri_begin;
        return 1;
    }
    return dyn_closest_seq(S, r, t_min, t_max, dj, dtri);
}

// Hit of intersect_scene for the winner: kind 0 static triangle at BVH position sbest,
// kind 1 dynamic object dj, triangle dtri of its mesh; t is the hit distance.
__device__ __forceinline__ void make_hit(const SceneDev& S, V3 o, V3 d, int kind, uint32_t sbest, uint32_t dj,
                                         uint32_t dtri, float t, Hit& h) {
    V3 e1, e2;
    if (kind == 0) {
        const float4 q1 = __ldg(&S.stris[3 * sbest + 1]);
        const float4 q2 = __ldg(&S.stris[3 * sbest + 2]);
        e1 = ld3(q1);
        e2 = ld3(q2);
        h.obj = __float_as_uint(q1.w);
    } else {
        const DynObj& D = S.fp->dyn[dj];
        const float4* T = S.dtris + 3ull * (D.tri_begin + dtri);
        e1 = ld3(__ldg(&T[1]));
        e2 = ld3(__ldg(&T[2]));
        h.obj = D.obj;
    }
    h.t = t;
    h.pos = add(o, mul(d, t));
    V3 n = normalized(cross(e1, e2));  // Triangle::geometric_normal (geometry.hpp:64)
    if (dot(n, d) > 0.0f) n = neg(n);
    h.normal = n;
}

// make_hit for a winner of the joint walk, from the fast tree's own triangle copy (the same
// e1/e2 floats as S.stris / S.dtris, already touched by the walk) -- no random access into
// the reference-order arrays on the hot path
__device__ __forceinline__ void make_hit_slot(const float4* __restrict__ tris, uint32_t slot, uint32_t obj, V3 o,
                                              V3 d, float t, Hit& h) {
    const V3 e1 = ld3(__ldg(&tris[kFT * slot + 1]));
    const V3 e2 = ld3(__ldg(&tris[kFT * slot + 2]));
    h.obj = obj;
    h.t = t;
    h.pos = add(o, mul(d, t));
    V3 n = normalized(cross(e1, e2));  // Triangle::geometric_normal (geometry.hpp:64)
    if (dot(n, d) > 0.0f) n = neg(n);
    h.normal = n;
}

// intersect_scene (scene.cpp:136-168), one-shot form: static phase, then the dynamic phase.
// `t_max` is the ray's (Ray::t_max, FLT_MAX in every engine query); `tri` (optional) receives
// Hit::triangle: the static triangle's index in scene order, or the index inside its mesh.
__device__ __forceinline__ bool intersect_scene(const SceneDev& S, V3 o, V3 d, float t_min, Hit& h,
                                                float t_max = FLT_MAX, uint32_t* tri = nullptr) {
    RayPre r = make_ray(o, d);
    if (!(t_min >= 0.0f)) r.regular = false;  // box_entry_fast's slack form assumes t_min >= 0
    opaque_flag(r.regular);
    if (S.fast && S.dfast && S.n_nodes > 0 && S.fp->n_dyn > 0) {
        // one walk over both trees; the winner's certificate makes it the two-phase answer:
        // a static winner beats every dynamic hit, so the dynamic phase adds nothing; a
        // dynamic winner is strictly nearer than every static hit, and its gate is certified
        // at the bound (which the reference's running t_max at that object exceeds)
        float bt, tc;
        uint32_t tree, pos, slot;
        PRX_CERT_COUNT(0);
        if (!joint_closest<false>(S, r, t_min, t_max, bt, tree, pos, tc, slot)) return false;
        bool ok;
        uint32_t dj = 0;
        if (tree == 0) {
            ok = static_cert_slot(S, r, t_min, tc, slot);
        } else {
            dj = __float_as_uint(__ldg(&S.datris[kFT * slot + 1]).w);  // dynamic object of the winner
            ok = !S.cert_off && t_min >= 0.0f && ray_box(r, t_min, tc, S.fp->dyn[dj].cur);
        }
        if (ok) {
            if (tri) *tri = tree == 0 ? __float_as_uint(__ldg(&S.stris[3 * pos]).w) : pos - S.fp->dyn[dj].tri_begin;
            if (tree == 0)
                make_hit_slot(S.ftris, slot, __float_as_uint(__ldg(&S.ftris[kFT * slot + 1]).w), o, d, bt, h);
            else
                make_hit_slot(S.datris, slot, S.fp->dyn[dj].obj, o, d, bt, h);
            return true;
        }
        PRX_CERT_COUNT(1);
    }
    uint32_t sbest = 0;
    const bool found = static_closest_exact(S, r, t_min, t_max, sbest);
    uint32_t dj = 0, dtri = 0;
    int kind = dyn_closest_exact(S, r, t_min, t_max, dj, dtri);
    if (kind < 0) kind = found ? 0 : -1;
    if (kind < 0) return false;
    if (tri) *tri = kind == 0 ? __float_as_uint(__ldg(&S.stris[3 * sbest]).w) : dtri;
    make_hit(S, o, d, kind, sbest, dj, dtri, t_max, h);
    return true;
}

// occluded (scene.cpp:170-177).  Dynamic phase: true iff some object whose gate passes at
// t_max holds an accepted triangle; the first accepted triangle of the combined walk
// certifies when its own object's gate passes, else the sequential loop decides.
__device__ __forceinline__ bool occluded(const SceneDev& S, V3 o, V3 d, float t_min, float t_max) {
    RayPre r = make_ray(o, d);
    if (!(t_min >= 0.0f)) r.regular = false;  // box_entry_fast's slack form assumes t_min >= 0
    opaque_flag(r.regular);
    if (S.fast && S.dfast && S.n_nodes > 0 && S.fp->n_dyn > 0) {
        // one walk over both trees to the first accepted triangle; it decides when its own
        // reference path (static leaf, or its object's gate) passes at the fixed t_max
        float bt, tc;
        uint32_t tree, pos, slot;
        PRX_CERT_COUNT(2);
        if (!joint_closest<true>(S, r, t_min, t_max, bt, tree, pos, tc, slot)) return false;
        if (tree == 0 ? static_cert_slot(S, r, t_min, t_max, slot)
                      : !S.cert_off && t_min >= 0.0f &&
                            ray_box(r, t_min, t_max, S.fp->dyn[__float_as_uint(__ldg(&S.datris[kFT * slot + 1]).w)].cur))
            return true;
        PRX_CERT_COUNT(3);
    }
    if (static_any_exact(S, r, t_min, t_max)) return true;
    const FrameParams* fp = S.fp;
    if (fp->n_dyn == 0) return false;
    if (S.fast && S.dfast) {
        float bt, tc;
        uint32_t g;
        if (!fast_closest<true>(S.fnodes, S.datris, r, t_min, t_max, bt, g, tc, S.dnode_off)) return false;
        if (!S.cert_off && t_min >= 0.0f && ray_box(r, t_min, t_max, fp->dyn[__ldg(&S.dtri_obj[g])].cur)) return true;
    }
    for (uint32_t j = 0; j < fp->n_dyn; ++j) {
        const DynObj& D = fp->dyn[j];
        if (!ray_box(r, t_min, t_max, D.cur)) continue;
        if (dyn_any(S, D, r, t_min, t_max)) return true;
    }
    return false;
}

// --------------------------------------------------------------------------- bounces
// cosine_sample (engine.cpp:25-32); cos/sin(phi) come from the host-libm table when
// available (phi = fl(2pi_f) * k * 2^-24 is a function of the 24-bit draw k).
__device__ __forceinline__ V3 cosine_sample(const SceneDev& S, V3 normal, float u1, uint32_t k2) {
    const float u2 = (float)k2 * 5.9604644775390625e-8f;
    const float r = sqrtf(u1);
    float cphi, sphi;
    if (S.trig) {
        const float2 cs = __ldcs(&S.trig[k2]);  // random 1-in-2^24 lookups: evict-first
        cphi = cs.x;
        sphi = cs.y;
    } else {
        const float phi = 2.0f * 3.14159265358979323846f * u2;
        cphi = cosf(phi);
        sphi = sinf(phi);
    }
    const float z = sqrtf(fmax_std(0.0f, 1.0f - u1));
    V3 t, b;
    orthonormal_basis(normal, t, b);
    return normalized(add(add(mul(t, r * cphi), mul(b, r * sphi)), mul(normal, z)));
}

// phong_lobe_sample (engine.cpp:34-42) -- glossy only (device powf: tolerance class C)
__device__ __forceinline__ V3 phong_sample(const SceneDev& S, V3 mirror, float exponent, float u1,
                                           uint32_t k1, uint32_t k2, uint32_t flags) {
    const float u2 = (float)k2 * 5.9604644775390625e-8f;
    // host-libm powf by table lookup (bit-exact) when the engine built the table
    const float cos_theta = (flags & 4u) ? __ldcs(&S.pow_tabs[flags >> 8][k1]) : powf(u1, 1.0f / (exponent + 1.0f));
    const float sin_theta = sqrtf(fmax_std(0.0f, 1.0f - cos_theta * cos_theta));
    float cphi, sphi;
    if (S.trig) {
        const float2 cs = __ldcs(&S.trig[k2]);  // random 1-in-2^24 lookups: evict-first
        cphi = cs.x;
        sphi = cs.y;
    } else {
        const float phi = 2.0f * 3.14159265358979323846f * u2;
        cphi = cosf(phi);
        sphi = sinf(phi);
    }
    V3 t, b;
    orthonormal_basis(mirror, t, b);
    return normalized(add(add(mul(t, sin_theta * cphi), mul(b, sin_theta * sphi)), mul(mirror, cos_theta)));
}

// Engine::sample_bounce (engine.cpp:159-170)
__device__ __forceinline__ V3 sample_bounce(const SceneDev& S, uint32_t obj, V3 normal, V3 incoming,
                                            uint32_t path, uint32_t epoch, uint32_t bounce_key) {
    const uint32_t k1 = rng_u24_m(S.seed_mix, path, epoch, bounce_key, kBounceDir, 0);
    const float u1 = (float)k1 * 5.9604644775390625e-8f;  // rng_uniform (rng.hpp:45-49)
    const uint32_t k2 = rng_u24_m(S.seed_mix, path, epoch, bounce_key, kBounceDir, 1);
    const uint32_t flags = __ldg(&S.oflags[obj]);
    if (!(flags & 2u)) return cosine_sample(S, normal, u1, k2);
    const float4 m = __ldg(&S.mat[obj]);
    const V3 mirror = normalized(sub(incoming, mul(normal, 2.0f * dot(incoming, normal))));
    V3 out = phong_sample(S, mirror, m.w, u1, k1, k2, flags);
    if (dot(out, normal) <= 0.0f) out = mirror;
    return out;
}

// --------------------------------------------------------------------------- lights
__device__ __forceinline__ double wrap_unit(double v) {  // light.cpp:49-53
    v -= floor(v);
    if (v >= 1.0) v = 0.0;
    return v;
}

__device__ __forceinline__ double dclamp(double v, double lo, double hi) {
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// dir_from_angles (light.cpp:40-47).  cos/sin(phi) come from CUDA's libm unless the
// narrowing (float)(cos(phi) * sin_theta) is not decided by it (exact_trig.h); then from the
// correctly rounded double-double evaluation.
__device__ __forceinline__ V3 dir_from_angles(const LightDev& L, double cos_theta, double phi) {
    const double sin_theta = sqrt(dmax_std(0.0, 1.0 - cos_theta * cos_theta));
    double sp, cp;
    sincos(phi, &sp, &cp);
    if (L.xt_force || !xt::product_narrows_stably(cp, sin_theta) || !xt::product_narrows_stably(sp, sin_theta))
        xt::sincos_rn(phi, sp, cp);
    const double cx = cp * sin_theta;
    const double cy = sp * sin_theta;
    return normalized(add(add(mul(L.tangent, (float)cx), mul(L.bitangent, (float)cy)),
                          mul(L.normal, (float)cos_theta)));
}

// wrap_unit(atan2(y, x) / 2pi) narrowed to float, with the same checked narrowing
__device__ __forceinline__ float wrapped_angle(const LightDev& L, double y, double x) {
    double a = atan2(y, x);
    if (L.xt_force || (float)wrap_unit(xt::win_lo(a) / kTwoPiD) != (float)wrap_unit(xt::win_hi(a) / kTwoPiD))
        a = xt::atan2_rn(y, x, a);
    return (float)wrap_unit(a / kTwoPiD);
}

// warp_canonical (light.cpp:70-117): canonical coords -> (origin, dir)
__device__ __forceinline__ void warp_canonical(const LightDev& L, const float c[4], V3& origin,
                                               V3& dir) {
    switch (L.kind) {
        case PRX_LIGHT_POINT: {
            const double cos_theta = 1.0 - 2.0 * (double)c[0];
            origin = L.position;
            dir = dir_from_angles(L, cos_theta, kTwoPiD * (double)c[1]);
            break;
        }
        case PRX_LIGHT_SPOT: {
            const double cos_theta = 1.0 - (double)c[0] * (1.0 - L.cos_half);
            origin = L.position;
            dir = dir_from_angles(L, cos_theta, kTwoPiD * (double)c[1]);
            break;
        }
        case PRX_LIGHT_DISC_AREA: {
            const double r_max = (double)L.radius * (double)L.scale;
            const double r = r_max * sqrt((double)c[0]);
            const double phi_s = kTwoPiD * (double)c[1];
            double sp, cp;
            sincos(phi_s, &sp, &cp);
            if (L.xt_force || !xt::product_narrows_stably(cp, r) || !xt::product_narrows_stably(sp, r))
                xt::sincos_rn(phi_s, sp, cp);
            origin = add(add(L.position, mul(L.tangent, (float)(r * cp))), mul(L.bitangent, (float)(r * sp)));
            const double cos_theta = sqrt(dmax_std(0.0, 1.0 - (double)c[2]));
            dir = dir_from_angles(L, cos_theta, kTwoPiD * (double)c[3]);
            break;
        }
        default: {  // rect
            const float hx = L.half_x * L.scale;
            const float hy = L.half_y * L.scale;
            origin = add(add(L.position, mul(L.tangent, (2.0f * c[0] - 1.0f) * hx)),
                         mul(L.bitangent, (2.0f * c[1] - 1.0f) * hy));
            const double cos_theta = sqrt(dmax_std(0.0, 1.0 - (double)c[2]));
            dir = dir_from_angles(L, cos_theta, kTwoPiD * (double)c[3]);
            break;
        }
    }
}

// canonical_of (light.cpp:119-175); returns false when the configuration does not
// parametrise (off-surface / outside the emission domain).
__device__ __forceinline__ bool canonical_of(const LightDev& L, V3 origin, V3 dir, float c[4]) {
    c[0] = c[1] = c[2] = c[3] = 0.0f;
    const double dn = dot(dir, L.normal);
    const double dt = dot(dir, L.tangent);
    const double db = dot(dir, L.bitangent);
    const float phi = wrapped_angle(L, db, dt);  // wrap_unit(atan2(db, dt) / 2pi), narrowed
    const double kTol = 1e-4;
    switch (L.kind) {
        case PRX_LIGHT_POINT:
            c[0] = (float)dclamp((1.0 - dn) / 2.0, 0.0, 1.0);
            c[1] = phi;
            return true;
        case PRX_LIGHT_SPOT: {
            const double q = (1.0 - dn) / (1.0 - L.cos_half);
            if (q < 0.0 || q > 1.0) return false;
            c[0] = (float)dmin_std(q, 1.0);
            c[1] = phi;
            return true;
        }
        default: {
            const V3 rel = sub(origin, L.position);
            const double lz = dot(rel, L.normal);
            const double lx = dot(rel, L.tangent);
            const double ly = dot(rel, L.bitangent);
            if (L.kind == PRX_LIGHT_DISC_AREA) {
                const double r_max = (double)L.radius * (double)L.scale;
                if (fabs(lz) > kTol * r_max) return false;
                const double q = (lx * lx + ly * ly) / (r_max * r_max);
                if (q > 1.0 + kTol) return false;
                c[0] = (float)dmin_std(q, 1.0);
                c[1] = wrapped_angle(L, ly, lx);
            } else {
                const double hx = (double)L.half_x * (double)L.scale;
                const double hy = (double)L.half_y * (double)L.scale;
                if (fabs(lz) > kTol * dmax_std(hx, hy)) return false;
                const double u = (lx / hx + 1.0) / 2.0;
                const double v = (ly / hy + 1.0) / 2.0;
                if (u < -kTol || u > 1.0 + kTol || v < -kTol || v > 1.0 + kTol) return false;
                c[0] = (float)dclamp(u, 0.0, 1.0);
                c[1] = (float)dclamp(v, 0.0, 1.0);
            }
            if (dn <= 0.0) return false;
            c[2] = (float)dclamp(1.0 - dn * dn, 0.0, 1.0);
            c[3] = phi;
            return true;
        }
    }
}

// cell_of_canonical (light.cpp:177-186)
__device__ __forceinline__ uint32_t cell_of(const LightDev& L, const float c[4]) {
    uint32_t cell = 0;
    for (uint32_t a = 0; a < L.ndims; ++a) {
        const uint32_t dim = L.dims[a];
        uint32_t idx = (uint32_t)(c[a] * (float)dim);
        if (idx >= dim) idx = dim - 1;
        cell = cell * dim + idx;
    }
    return cell;
}

// sample_in_cell (light.cpp:211-228) with key {path, epoch, 0, Emission, lane 0}
__device__ __forceinline__ void sample_in_cell(const LightDev& L, uint32_t cell, uint64_t seed_mix,
                                               uint32_t path, uint32_t epoch, float c[4], V3& origin,
                                               V3& dir) {
    float lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
    uint32_t rest = cell;
    for (int a = (int)L.ndims - 1; a >= 0; --a) {
        const uint32_t dim = L.dims[a];
        const uint32_t idx = rest % dim;
        rest /= dim;
        lo[a] = (float)idx / (float)dim;
        hi[a] = (float)(idx + 1) / (float)dim;
    }
    c[0] = c[1] = c[2] = c[3] = 0.0f;
    for (uint32_t a = 0; a < L.ndims; ++a) {
        const double u = rng_uniform_d_m(seed_mix, path, epoch, 0, kEmission, a);
        const double width = (double)hi[a] - (double)lo[a];
        const double m0 = 2e-5 / width;
        const double margin = (m0 < 0.4) ? m0 : 0.4;
        const double t = margin + u * (1.0 - 2.0 * margin);
        c[a] = (float)((double)lo[a] + t * width);
    }
    warp_canonical(L, c, origin, dir);
}

__device__ __forceinline__ uint32_t light_of(const FrameParams* fp, uint32_t p) {
    uint32_t li = 0;
    for (uint32_t k = 1; k < fp->n_lights; ++k)
        if (p >= fp->lights[k].begin) li = k;
    return li;
}

}  // namespace prx

namespace prx {

// segment_intersects_aabb (geometry.hpp:107-134), filtered: a float slab test with a
// certified margin decides clear cases; borderline cases run the reference's double test.
__device__ __forceinline__ bool segment_box(V3 a, V3 b, const Box& box) {
    bool swap;
    if (b.x != a.x) swap = b.x < a.x;
    else if (b.y != a.y) swap = b.y < a.y;
    else swap = b.z < a.z;
    if (swap) {
        const V3 t = a;
        a = b;
        b = t;
    }
    float t0 = 0.0f, t1 = 1.0f;
    for (int axis = 0; axis < 3; ++axis) {
        const float o = comp(a, axis), e = comp(b, axis);
        const float lo = comp(box.lo, axis), hi = comp(box.hi, axis);
        if (o == e) {  // d == 0 in double as well
            if (o < lo || o > hi) return false;
            continue;
        }
        const float d = e - o;
        if (fabsf(d) < 1e-30f) return segment_box_exact(a, b, box);
        const float inv = __frcp_rn(d);  // == 1.0f / d (both correctly rounded), cheaper
        float tn = (lo - o) * inv;
        float tf = (hi - o) * inv;
        if (tn > tf) {
            const float s = tn;
            tn = tf;
            tf = s;
        }
        t0 = fmax_std(t0, tn);
        t1 = fmin_std(t1, tf);
    }
    // each quotient carries <= 4 roundings (2.4e-7 relative) vs the double reference
    const float slack = 6.0e-7f * (fabsf(t0) + fabsf(t1)) + 1e-30f;
    if (t0 - t1 > slack) return false;
    if (t1 - t0 > slack) return true;
    return segment_box_exact(a, b, box);
}

}  // namespace prx
