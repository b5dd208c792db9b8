// kernels.cu -- per-frame stage kernels of the B200 path-reuse engine.
//
// One thread per path (grid-stride), bounce-major vertex streams so that every warp
// access to bounce b of 32 consecutive paths is one coalesced 512-byte float4 load.
// Citations: reference function each kernel restates (paths under /root/reference/proj).
#include <cstdio>
#include "device_scene.cuh"
#include "kernels.h"

namespace prx {

std::atomic<uint64_t> g_launches{0};

int launch_grid(uint64_t n, int threads) {
    const uint64_t blocks = (n + threads - 1) / threads;
    const uint64_t cap = 148ull * 16ull;  // 16 resident 256-thread CTAs per SM
    return static_cast<int>(blocks == 0 ? 1 : (blocks < cap ? blocks : cap));
}

namespace {

constexpr int kT = 256;
#ifndef PRX_TRACE_MINB
#define PRX_TRACE_MINB 5  // resident CTAs per SM requested for the traversal kernels
#endif

// Block-wide sum of a per-thread counter, one atomic per CTA (a per-warp atomic on one
// address serialises ~20K warps in the path-wide kernels).  Every thread of the block must
// call it (the kernels call it once, after their grid-stride loop).
__device__ __forceinline__ void warp_add(unsigned long long* dst, unsigned long long v) {
    __shared__ unsigned long long s_part[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) s_part[w] = v;
    __syncthreads();
    if (w == 0) {
        unsigned long long x = lane < (int)(blockDim.x >> 5) ? s_part[lane] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0 && x) atomicAdd(dst, x);
    }
    __syncthreads();
}

__device__ __forceinline__ size_t vix(const PathDev& P, uint32_t b, uint32_t i) {
    return (size_t)b * P.n + i;
}

// Engine::truncate_path (engine.cpp:141-147): photon records >= new_count become empty
// Photon{} (aux untouched), count/escaped updated.
__device__ __forceinline__ void truncate_path(const PathDev& P, uint32_t i, uint32_t new_count,
                                              bool escaped, uchar4& m) {
    for (uint32_t b = new_count; b < P.B; ++b) {
        const size_t v = vix(P, b, i);
        __stcs(&P.in_dir[kVS * (v)], make_float4(0.f, 0.f, 0.f, 0.f));
        __stcs(&P.pos_obj[kVS * (v)].w, __uint_as_float(kInvalidObj));
        __stcs(&P.energy[kVS * (v)], make_float4(0.f, 0.f, 0.f, 0.f));
    }
    m.x = (unsigned char)new_count;
    m.y = escaped ? 1 : 0;
}

// ---------------------------------------------------------------- init / placement
__global__ void k_init_dm_target(LightDev L, uint32_t n, uint64_t seed_mix, uint32_t* dm_t) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        float c[4] = {0, 0, 0, 0};
        for (uint32_t a = 0; a < L.ndims; ++a)
            c[a] = (float)rng_uniform_d_m(seed_mix, i, 0, 0, kDmTargetInit, a);
        atomicAdd(&dm_t[cell_of(L, c)], 1u);
    }
}

// transform.hpp:72,98-100: p' = rotate(q, p * s) + t, then (a, b - a, c - a)
__global__ void k_transform_dynamic(const float4* __restrict__ local, const uint32_t* __restrict__ tri_xf,
                                    const float4* __restrict__ xf, uint32_t n, float4* __restrict__ world) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t k = tri_xf[i];
        const float4 q = xf[2 * k], ts = xf[2 * k + 1];
        const V3 u{q.x, q.y, q.z};
        V3 w[3];
        for (int j = 0; j < 3; ++j) {
            const float4 p4 = local[3 * i + j];
            const V3 v = mul(V3{p4.x, p4.y, p4.z}, ts.w);
            const V3 t = mul(cross(u, v), 2.0f);
            w[j] = add(add(add(v, mul(t, q.w)), cross(u, t)), V3{ts.x, ts.y, ts.z});
        }
        const V3 e1 = sub(w[1], w[0]), e2 = sub(w[2], w[0]);
        world[3 * i] = make_float4(w[0].x, w[0].y, w[0].z, 0.f);
        world[3 * i + 1] = make_float4(e1.x, e1.y, e1.z, 0.f);
        world[3 * i + 2] = make_float4(e2.x, e2.y, e2.z, 0.f);
    }
}

// Four paths per thread with whole-word accesses: clearing only meta.w per path compiles to
// stride-4 byte stores (partial sectors, ~85 GB/s); 16-byte meta and 4-byte rstart words
// write whole sectors.  Buffers are cudaMalloc-aligned, so the word views are aligned.
__device__ __forceinline__ uint32_t reset_meta_word(uint32_t m, unsigned long long& segs) {
    if (((m >> 16) & 0xFFu) == kLive) segs += (m & 0xFFu) + ((m >> 8) & 0xFFu);  // {count, escaped, status, filled}
    return m & 0x00FFFFFFu;
}
__global__ void k_frame_reset(PathDev P, int record, Counters* ctr) {
    unsigned long long segs = 0;
    const uint32_t n4 = P.n / 4;
    uint4* meta4 = reinterpret_cast<uint4*>(P.meta);
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += gridDim.x * blockDim.x) {
        uint4 m = __ldcs(&meta4[q]);
        m.x = reset_meta_word(m.x, segs);
        m.y = reset_meta_word(m.y, segs);
        m.z = reset_meta_word(m.z, segs);
        m.w = reset_meta_word(m.w, segs);
        __stcs(&meta4[q], m);
        __stcs(reinterpret_cast<uint32_t*>(P.rstart) + q, 0x01010101u * kNoRetrace);
        if (record) __stcs(reinterpret_cast<uint4*>(P.seg_flags) + q, make_uint4(0u, 0u, 0u, 0u));
    }
    for (uint32_t i = 4 * n4 + blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        uint32_t* mw = reinterpret_cast<uint32_t*>(P.meta) + i;
        __stcs(mw, reset_meta_word(*mw, segs));
        P.rstart[i] = kNoRetrace;
        if (record) P.seg_flags[i] = 0;
    }
    warp_add(&ctr->live_segments, segs);
}

__global__ void k_release_all(PathDev P) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        uchar4 m = P.meta[i];
        truncate_path(P, i, 0, false, m);
        m.z = kDead;
        P.meta[i] = m;
    }
}

// ---------------------------------------------------------------- verify_paths
__global__ void __launch_bounds__(kT) k_update_origins(SceneDev S, PathDev P, Counters* ctr) {
    const FrameParams* fp = S.fp;
    unsigned long long vis = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        const uint32_t p = P.base + i;
        const LightDev& L = fp->lights[light_of(fp, p)];
        if (!L.moved) continue;
        uchar4 m = P.meta[i];
        if (m.z != kLive) continue;
        if (L.kind == PRX_LIGHT_POINT || L.kind == PRX_LIGHT_SPOT) {
            P.origin[i] = make_float4(L.position.x, L.position.y, L.position.z, 0.f);
            if (m.x > 0) {
                const V3 primary = ld3(P.pos_obj[kVS * (i)]);
                const V3 to = sub(primary, L.position);
                const float dist = length(to);
                if (dist <= S.eps) {
                    m.z = kReplace;
                    P.meta[i] = m;
                    continue;
                }
                const V3 dir = divs(to, dist);
                P.emis[i] = make_float4(dir.x, dir.y, dir.z, 0.f);
                ++vis;
                if (occluded(S, L.position, dir, S.eps, dist - S.eps)) {
                    m.z = kReplace;
                    P.meta[i] = m;
                }
            }
        } else {
            if (m.x > 0) {
                const V3 d = ld3(P.emis[i]);
                const V3 primary = ld3(P.pos_obj[kVS * (i)]);
                const float denom = dot(d, L.normal);
                if (denom <= 1e-6f) {
                    m.z = kReplace;
                    P.meta[i] = m;
                    continue;
                }
                const float s = dot(sub(primary, L.position), L.normal) / denom;
                if (s <= 0.0f) {
                    m.z = kReplace;
                    P.meta[i] = m;
                    continue;
                }
                const V3 o = sub(primary, mul(d, s));
                P.origin[i] = make_float4(o.x, o.y, o.z, 0.f);
            } else {
                const float4 c4 = P.canon[i];
                const float c[4] = {c4.x, c4.y, c4.z, c4.w};
                V3 o, d;
                warp_canonical(L, c, o, d);
                P.origin[i] = make_float4(o.x, o.y, o.z, 0.f);
            }
        }
    }
    warp_add(&ctr->vis, vis);
}

// compute_flag_mask (engine.cpp:172-199) with segment ends per Engine::segment_end
// (engine.cpp:135-139); occlusion boxes staged in shared memory.
#ifndef PRX_OCC_MINB
#define PRX_OCC_MINB 4
#endif
#ifndef PRX_OCC_PREFETCH2
#define PRX_OCC_PREFETCH2 1
#endif
__global__ void __launch_bounds__(kT, PRX_OCC_MINB) k_occlusion_flags(SceneDev S, PathDev P, int mode, int record,
                                                        uint32_t* list, uint32_t* masks, Counters* ctr) {
    __shared__ Box boxes[kMaxDyn];
    __shared__ float4 wide[2 * kMaxDyn];  // boxes pre-widened by the reject tolerance at ext_bound
    // per warp: a queue of (segment, box) pairs that passed the reject; the exact tests run 32
    // at a time, one pair per lane, whichever lane's path they belong to (the segment flag is
    // an OR over boxes, so order and early exit do not matter)
    constexpr uint32_t kQ = 64;
    __shared__ float4 q_a[kT / 32][kQ], q_b[kT / 32][kQ];  // {a, owner << 16 | s << 8 | box} {b, -}
    __shared__ uint32_t q_mask[kT];
    const FrameParams* fp = S.fp;
    const uint32_t nb = fp->n_boxes;
    // Bounding-box reject before the slab test: a segment whose box misses an occlusion box by
    // more than tol = 1e-6 (segment extent + |lo| + |hi|) per axis cannot pass the double test
    // (its quotients err by ~1e-16 relative).  The tolerance is evaluated once per box at an
    // extent bound (every step is monotone, so it only grows and the reject stays sound);
    // segments longer than the bound skip the reject.
    const float ext_bound = 2.0f * S.two_diag;
    for (uint32_t k = threadIdx.x; k < nb; k += blockDim.x) {
        const Box B = fp->boxes[k];
        boxes[k] = B;
        float lo[3], hi[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float tol = 1e-6f * (ext_bound + fabsf(comp(B.lo, a)) + fabsf(comp(B.hi, a))) + 1e-30f;
            lo[a] = comp(B.lo, a) - tol;
            hi[a] = comp(B.hi, a) + tol;
        }
        wide[2 * k] = make_float4(lo[0], lo[1], lo[2], 0.f);
        wide[2 * k + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float4* const QA = q_a[warp];
    float4* const QB = q_b[warp];
    uint32_t* const QM = q_mask + 32 * warp;
    uint32_t qn = 0;  // warp-uniform queue length
    auto test_front = [&](uint32_t cnt) {  // exact tests of queue entries [0, cnt), cnt <= 32
        if (lane < cnt) {
            const float4 a = QA[lane], b = QB[lane];
            const uint32_t code = __float_as_uint(a.w);
            if (segment_box(V3{a.x, a.y, a.z}, V3{b.x, b.y, b.z}, boxes[code & 0xFFu]))
                atomicOr(&QM[code >> 16], 1u << ((code >> 8) & 0xFFu));
        }
        __syncwarp();
    };
    for (uint32_t i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < P.n; i0 += gridDim.x * blockDim.x) {
        const uint32_t i = i0 + lane;
        const uchar4 m = i < P.n ? P.meta[i] : make_uchar4(0, 0, kDead, 0);
        const bool live = m.z == kLive;
        const uint32_t k = live ? m.x : 0u, segs = live ? m.x + m.y : 0u;
        QM[lane] = 0u;
        uint32_t mask = 0;
        V3 prev = live ? ld3(P.origin[i]) : V3{0.f, 0.f, 0.f};
        uint32_t prev_obj = kInvalidObj;
        // vertices s+1 (and s+2, PRX_OCC_PREFETCH2) are loaded while segment s is tested (the
        // loop is load-latency bound)
        float4 nextv = k > 0 ? __ldcs(&P.pos_obj[kVS * (vix(P, 0, i))]) : make_float4(0.f, 0.f, 0.f, 0.f);
#if PRX_OCC_PREFETCH2
        float4 next2 = k > 1 ? __ldcs(&P.pos_obj[kVS * (vix(P, 1, i))]) : make_float4(0.f, 0.f, 0.f, 0.f);
#endif
        const uint32_t s_end = __reduce_max_sync(0xffffffffu, segs);
        for (uint32_t s = 0; s < s_end; ++s) {
            const bool act = s < segs;
            V3 cur{0, 0, 0};
            uint32_t cur_obj = kInvalidObj;
            if (act && s < k) {
                const float4 v = nextv;
#if PRX_OCC_PREFETCH2
                nextv = next2;
                if (s + 2 < k) next2 = __ldcs(&P.pos_obj[kVS * (vix(P, s + 2, i))]);
#else
                if (s + 1 < k) nextv = __ldcs(&P.pos_obj[kVS * (vix(P, s + 1, i))]);
#endif
                cur = ld3(v);
                cur_obj = __float_as_uint(v.w);
            }
            bool flagged = false;
            if (act && s > 0 && prev_obj != kInvalidObj && (__ldg(&S.oflags[prev_obj]) & 1u)) flagged = true;
            if (act && !flagged && s < k && cur_obj != kInvalidObj && (__ldg(&S.oflags[cur_obj]) & 1u)) flagged = true;
            if (flagged) mask |= 1u << s;
            const bool probe = act && !flagged;
            V3 b = cur, smin{}, smax{};
            bool bounded = false;
            if (probe) {
                if (s >= k) {  // escape segment, clipped to twice the diagonal
                    const V3 dir = s == 0 ? ld3(P.emis[i]) : ld3(P.out_dir[kVS * (vix(P, s - 1, i))]);
                    b = add(prev, mul(dir, S.two_diag));
                }
                smin = V3{fminf(prev.x, b.x), fminf(prev.y, b.y), fminf(prev.z, b.z)};
                smax = V3{fmaxf(prev.x, b.x), fmaxf(prev.y, b.y), fmaxf(prev.z, b.z)};
                bounded = smax.x - smin.x <= ext_bound && smax.y - smin.y <= ext_bound && smax.z - smin.z <= ext_bound;
            }
            for (uint32_t base = 0; base < nb; base += 32) {
                const uint32_t cnt = nb - base < 32 ? nb - base : 32;
                uint32_t cand = 0;
                if (probe) {
                    for (uint32_t q = 0; q < cnt; ++q) {
                        const float4 lo = wide[2 * (base + q)], hi = wide[2 * (base + q) + 1];
                        const bool apart = bounded && (smax.x < lo.x || smax.y < lo.y || smax.z < lo.z ||
                                                       smin.x > hi.x || smin.y > hi.y || smin.z > hi.z);
                        cand |= apart ? 0u : 1u << q;
                    }
                }
                while (__any_sync(0xffffffffu, cand != 0u)) {  // append one candidate per lane
                    const bool has = cand != 0u;
                    const unsigned who = __ballot_sync(0xffffffffu, has);
                    if (has) {
                        const uint32_t q = __ffs(cand) - 1;
                        cand &= cand - 1;
                        const uint32_t at = qn + __popc(who & ((1u << lane) - 1u));
                        QA[at] = make_float4(prev.x, prev.y, prev.z, __uint_as_float(lane << 16 | s << 8 | (base + q)));
                        QB[at] = make_float4(b.x, b.y, b.z, 0.f);
                    }
                    qn += __popc(who);
                    __syncwarp();
                    if (qn >= 32) {
                        test_front(32);
                        qn -= 32;
                        float4 ta, tb;
                        if (lane < qn) {
                            ta = QA[32 + lane];
                            tb = QB[32 + lane];
                        }
                        __syncwarp();
                        if (lane < qn) {
                            QA[lane] = ta;
                            QB[lane] = tb;
                        }
                        __syncwarp();
                    }
                }
            }
            prev = cur;
            prev_obj = cur_obj;
        }
        if (qn > 0) {
            test_front(qn);
            qn = 0;
        }
        mask |= QM[lane];
        __syncwarp();
        if (!live) continue;
        if (record) P.seg_flags[i] = mask;
        if (mask == 0) continue;
        if (mode == PRX_MODE_NAIVE) {
            P.rstart[i] = (uint8_t)(__ffs(mask) - 1);
        } else {
            const uint32_t slot = (uint32_t)atomicAdd(&ctr->flagged, 1ull);
            list[slot] = i;
            masks[slot] = mask;
        }
    }
}

// Warp-aggregated work fetch for persistent kernels: every lane that needs work gets the
// next index of a global queue; one atomic per warp and call.
__device__ __forceinline__ uint32_t fetch_work(uint32_t* counter) {
    const unsigned m = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    const unsigned rank = __popc(m & ((1u << lane) - 1u));
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned)__popc(m));
    base = __shfl_sync(m, base, leader);
    return base + rank;
}

// Batched refill for the persistent ray-granularity kernels: the warp stays converged at the
// loop head; once at least PRX_REFILL lanes are idle (or nobody is working) the idle lanes
// take consecutive queue slots with one atomic, so the state-load latency is paid once per
// batch instead of once per lane.
#ifndef PRX_REFILL
#define PRX_REFILL 24
#endif
__device__ __forceinline__ bool refill_due(bool idle, bool working) {
    const unsigned iw = __ballot_sync(0xffffffffu, idle);
    const unsigned ww = __ballot_sync(0xffffffffu, working);
    return iw != 0u && (__popc(iw) >= PRX_REFILL || ww == 0u);
}
// queue slot of this lane among the idle ones (>= queue length: exhausted)
__device__ __forceinline__ uint32_t refill_slot(uint32_t* counter, bool idle) {
    const unsigned iw = __ballot_sync(0xffffffffu, idle);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(iw) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned)__popc(iw));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + (uint32_t)__popc(iw & ((1u << lane) - 1u));
}

// verify_path_error_based (engine.cpp:339-403): Alg. 1 walk over the flagged segments,
// persistent: each lane walks one path at a time and advances its visibility ray one BVH
// node per iteration, fetching the next flagged path as soon as its walk ends.
__global__ void __launch_bounds__(kT) k_verify_error(SceneDev S, PathDev P, float threshold,
                                                     const uint32_t* __restrict__ list,
                                                     const uint32_t* __restrict__ masks,
                                                     const Counters* cnt, uint32_t* work, Counters* ctr) {
    const FrameParams* fp = S.fp;
    const uint32_t n_list = (uint32_t)cnt->flagged;
    unsigned long long vis = 0;
    bool has = false, ray = false, force = false;
    uint32_t i = 0, p = 0, flags = 0, k = 0, segs = 0, s = 0, epoch = 0, li = 0;
    uchar4 m = make_uchar4(0, 0, 0, 0);
    Trav T;
    while (true) {
        if (!has) {
            const uint32_t j = fetch_work(work);
            if (j >= n_list) break;
            i = list[j];
            flags = masks[j];
            p = P.base + i;
            li = light_of(fp, p);
            m = P.meta[i];
            k = m.x;
            segs = m.x + m.y;
            epoch = P.epoch[i];
            s = 0;
            force = false;
            ray = false;
            has = true;
        }
        if (!ray) {  // next flagged segment (engine.cpp:345-351)
            while (s < segs) {
                const bool flagged = force || ((flags >> s) & 1u);
                force = false;
                if (flagged) break;
                ++s;
            }
            if (s >= segs) {
                has = false;
                continue;
            }
            const V3 o = s == 0 ? ld3(P.origin[i]) : ld3(P.pos_obj[kVS * (vix(P, s - 1, i))]);
            const V3 d = s == 0 ? ld3(P.emis[i]) : ld3(P.out_dir[kVS * (vix(P, s - 1, i))]);
            ++vis;
            trav_init(S, T, o, d, S.eps, FLT_MAX, false);
            ray = true;
        }
        if (!trav_step(S, T)) continue;
        ray = false;
        Hit h;
        const bool hit = trav_hit(S, T, h);
        const V3 d = T.r.d;
        if (s == k) {  // escape segment: a new blocker -> retrace from here
            if (hit) P.rstart[i] = (uint8_t)s;
            has = false;
            continue;
        }
        if (!hit) {  // destination gone: truncate and escape
            truncate_path(P, i, s, true, m);
            P.meta[i] = m;
            has = false;
            continue;
        }
        const size_t v = vix(P, s, i);
        const float4 stored = P.energy[kVS * (v)];
        const V3 e_prev = s == 0 ? fp->lights[li].flux_pp : ld3(P.energy[kVS * (vix(P, s - 1, i))]);
        const float4 am = __ldg(&S.mat[h.obj]);
        const V3 e_new = mulv(e_prev, V3{am.x, am.y, am.z});
        const bool glossy = (__ldg(&S.oflags[h.obj]) & 2u) != 0;
        if (glossy || !energies_close(ld3(stored), e_new, threshold)) {
            __stcs(&P.in_dir[kVS * (v)], make_float4(d.x, d.y, d.z, 0.f));
            __stcs(&P.pos_obj[kVS * (v)], make_float4(h.pos.x, h.pos.y, h.pos.z, __uint_as_float(h.obj)));
            __stcs(&P.energy[kVS * (v)], make_float4(e_new.x, e_new.y, e_new.z, S.gather_radius));
            const V3 out = sample_bounce(S, h.obj, h.normal, d, p, epoch, s + 1);
            __stcs(&P.out_dir[kVS * (v)], make_float4(out.x, out.y, out.z, 0.f));
            P.rstart[i] = (uint8_t)(s + 1);
            has = false;
            continue;
        }
        const V3 old_pos = ld3(P.pos_obj[kVS * (v)]);
        const bool close_pos = length(sub(h.pos, old_pos)) <= S.eps;
        __stcs(&P.in_dir[kVS * (v)], make_float4(d.x, d.y, d.z, 0.f));
        __stcs(&P.pos_obj[kVS * (v)], make_float4(h.pos.x, h.pos.y, h.pos.z, __uint_as_float(h.obj)));
        if (s + 1 >= segs) {
            has = false;
            continue;
        }
        const bool hit_dyn = (__ldg(&S.oflags[h.obj]) & 1u) != 0;
        if (close_pos && !hit_dyn && !((flags >> (s + 1)) & 1u)) {
            s += 2;  // the next segment is provably unchanged
            continue;
        }
        if (s + 1 < k) {
            const V3 next = ld3(P.pos_obj[kVS * (vix(P, s + 1, i))]);
            const V3 od = normalized(sub(next, h.pos));
            __stcs(&P.out_dir[kVS * (v)], make_float4(od.x, od.y, od.z, 0.f));
        }
        force = true;
        ++s;
    }
    warp_add(&ctr->vis, vis);
}

// verify_path_error_based (engine.cpp:339-403) with one-shot intersect_scene queries (fast
// traversal + certificate).  Persistent lanes at ray granularity: a lane skips its path's
// unflagged segments, traces one visibility ray per iteration and fetches the next flagged
// path as soon as its walk ends.
__global__ void __launch_bounds__(kT, PRX_TRACE_MINB) k_verify_error_walk(SceneDev S, PathDev P, float threshold,
                                                          const uint32_t* __restrict__ list,
                                                          const uint32_t* __restrict__ masks, const Counters* cnt,
                                                          uint32_t* work, Counters* ctr) {
    const FrameParams* fp = S.fp;
    const uint32_t n_list = (uint32_t)cnt->flagged;
    unsigned long long vis = 0;
    uint32_t i = 0, flags = 0, p = 0, k = 0, segs = 0, epoch = 0, s = 0;
    uchar4 m = make_uchar4(0, 0, 0, 0);
    bool force = false, have = false, done = false;
    while (true) {
        if (refill_due(!have && !done, have)) {
            const uint32_t j = refill_slot(work, !have && !done);
            if (!have && !done) {
                if (j >= n_list) {
                    done = true;
                } else {
                    i = list[j];
                    flags = masks[j];
                    p = P.base + i;
                    m = P.meta[i];
                    k = m.x;
                    segs = m.x + m.y;
                    epoch = P.epoch[i];
                    force = false;
                    s = 0;
                    have = true;
                }
            }
        }
        if (__all_sync(0xffffffffu, done)) break;
        if (!have) continue;
        if (!force)
            while (s < segs && !((flags >> s) & 1u)) ++s;
        force = false;
        if (s >= segs) {
            have = false;
            continue;
        }
        const V3 o = s == 0 ? ld3(P.origin[i]) : ld3(P.pos_obj[kVS * (vix(P, s - 1, i))]);
        const V3 d = s == 0 ? ld3(P.emis[i]) : ld3(P.out_dir[kVS * (vix(P, s - 1, i))]);
        ++vis;
        Hit h;
        const bool hit = intersect_scene(S, o, d, S.eps, h);
        have = false;  // every branch below ends the walk unless it continues explicitly
        if (s == k) {  // escape segment: a new blocker -> retrace from here
            if (hit) P.rstart[i] = (uint8_t)s;
            continue;
        }
        if (!hit) {  // destination gone: truncate and escape
            truncate_path(P, i, s, true, m);
            P.meta[i] = m;
            continue;
        }
        const size_t v = vix(P, s, i);
        const float4 stored = P.energy[kVS * (v)];
        const V3 e_prev = s == 0 ? fp->lights[light_of(fp, p)].flux_pp : ld3(P.energy[kVS * (vix(P, s - 1, i))]);
        const float4 am = __ldg(&S.mat[h.obj]);
        const V3 e_new = mulv(e_prev, V3{am.x, am.y, am.z});
        const bool glossy = (__ldg(&S.oflags[h.obj]) & 2u) != 0;
        if (glossy || !energies_close(ld3(stored), e_new, threshold)) {
            __stcs(&P.in_dir[kVS * (v)], make_float4(d.x, d.y, d.z, 0.f));
            __stcs(&P.pos_obj[kVS * (v)], make_float4(h.pos.x, h.pos.y, h.pos.z, __uint_as_float(h.obj)));
            __stcs(&P.energy[kVS * (v)], make_float4(e_new.x, e_new.y, e_new.z, S.gather_radius));
            const V3 out = sample_bounce(S, h.obj, h.normal, d, p, epoch, s + 1);
            __stcs(&P.out_dir[kVS * (v)], make_float4(out.x, out.y, out.z, 0.f));
            P.rstart[i] = (uint8_t)(s + 1);
            continue;
        }
        const V3 old_pos = ld3(P.pos_obj[kVS * (v)]);
        const bool close_pos = length(sub(h.pos, old_pos)) <= S.eps;
        __stcs(&P.in_dir[kVS * (v)], make_float4(d.x, d.y, d.z, 0.f));
        __stcs(&P.pos_obj[kVS * (v)], make_float4(h.pos.x, h.pos.y, h.pos.z, __uint_as_float(h.obj)));
        if (s + 1 >= segs) continue;
        have = true;
        const bool hit_dyn = (__ldg(&S.oflags[h.obj]) & 1u) != 0;
        if (close_pos && !hit_dyn && !((flags >> (s + 1)) & 1u)) {
            s += 2;
            continue;
        }
        if (s + 1 < k) {
            const V3 next = ld3(P.pos_obj[kVS * (vix(P, s + 1, i))]);
            const V3 od = normalized(sub(next, h.pos));
            __stcs(&P.out_dir[kVS * (v)], make_float4(od.x, od.y, od.z, 0.f));
        }
        force = true;
        ++s;
    }
    warp_add(&ctr->vis, vis);
}

#ifndef PRX_DM_MINB
#define PRX_DM_MINB 4
#endif
__global__ void __launch_bounds__(kT, PRX_DM_MINB) k_compute_dm(SceneDev S, PathDev P, Counters* ctr) {
    const FrameParams* fp = S.fp;
    unsigned long long replaced = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        uchar4 m = P.meta[i];
        if (m.z == kDead) continue;
        bool ok = m.z == kLive;
        if (ok) {
            const LightDev& L = fp->lights[light_of(fp, P.base + i)];
            float c[4];
            ok = canonical_of(L, ld3(P.origin[i]), ld3(P.emis[i]), c);
            if (ok) {
                P.canon[i] = make_float4(c[0], c[1], c[2], c[3]);
                const uint32_t cell = cell_of(L, c);
                P.cell[i] = cell;
                atomicAdd(&L.dm_c[cell], 1u);
            }
        }
        if (!ok) {
            truncate_path(P, i, 0, false, m);
            m.z = kDead;
            P.meta[i] = m;
            ++replaced;
        }
    }
    warp_add(&ctr->replaced, replaced);
}

// ---------------------------------------------------------------- prune (engine.cpp:443-497)
__global__ void k_prune_mark(SceneDev S, PathDev P, const uint32_t* frame_dev, uint32_t* const* unmarked,
                             uint8_t* pruned, uint8_t* cand) {
    const FrameParams* fp = S.fp;
    const uint32_t frame = *frame_dev;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        pruned[i] = 0;
        cand[i] = 0;
        if (P.meta[i].z != kLive) continue;
        const uint32_t p = P.base + i;
        const uint32_t li = light_of(fp, p);
        const LightDev& L = fp->lights[li];
        const uint32_t c = P.cell[i];
        const uint32_t dmc = L.dm_c[c], dmt = L.dm_t[c];
        if (dmc <= dmt) continue;
        const double prob = prune_probability(dmc, dmt);
        const float u = rng_uniform_m(S.seed_mix, p, frame, 0, kPruneMark, 0);
        if (prob > 0.0 && (double)u < prob) {
            pruned[i] = 1;
        } else {
            cand[i] = 1;
            atomicAdd(&unmarked[li][c], 1u);
        }
    }
}

// candidates in cells whose (global) survivor count exceeds the target need a trim
__global__ void k_prune_trim_flags(PathDev P, const FrameParams* fp, uint32_t* const* unm_total,
                                   const uint8_t* cand, uint8_t* trim) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        uint8_t f = 0;
        if (cand[i]) {
            const uint32_t li = light_of(fp, P.base + i);
            const uint32_t c = P.cell[i];
            f = unm_total[li][c] > fp->lights[li].dm_t[c] ? 1 : 0;
        }
        trim[i] = f;
    }
}

__global__ void k_prune_keys(PathDev P, const FrameParams* fp, const uint32_t* list, const uint32_t* count,
                             uint32_t* keys, uint32_t* vals) {
    const uint32_t n = *count;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t i = list[j];
        keys[j] = (light_of(fp, P.base + i) << 22) | P.cell[i];
        vals[j] = i;
    }
}

// keys sorted by (light, cell), stable in path id: survivors are the dm_t lowest ids
// (select_paths_to_prune trims "from the top path id down", engine.cpp:459-466).
__global__ void k_prune_heads(const uint32_t* keys, const uint32_t* count, uint32_t* const* seg_start) {
    const uint32_t n = *count;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t k = keys[j];
        if (j == 0 || keys[j - 1] != k) seg_start[k >> 22][k & 0x3FFFFFu] = j;
    }
}

__global__ void k_prune_trim(const FrameParams* fp, const uint32_t* keys, const uint32_t* vals,
                             const uint32_t* count, uint32_t* const* seg_start, uint32_t* const* prefix,
                             uint8_t* pruned) {
    const uint32_t n = *count;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t k = keys[j];
        const uint32_t li = k >> 22, c = k & 0x3FFFFFu;
        const uint32_t rank = j - seg_start[li][c] + (prefix ? prefix[li][c] : 0u);
        if (rank >= fp->lights[li].dm_t[c]) pruned[vals[j]] = 1;
    }
}

// clear_records == 0 inside a full frame: every dead slot is refilled and retraced by the same
// frame (sum of fill deficits == dead slots, engine.cpp:499-546), and the retrace rewrites all
// of the path's records, so the scattered record clears (sector read-modify-writes) are skipped;
// only the stage-by-stage entry points need the intermediate state materialised.
__global__ void k_prune_apply(PathDev P, const uint8_t* pruned, int clear_records) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        if (!pruned[i]) continue;
        uchar4 m = P.meta[i];
        if (clear_records) {
            truncate_path(P, i, 0, false, m);
        } else {
            m.x = 0;
            m.y = 0;
        }
        m.z = kDead;
        P.meta[i] = m;
    }
}

__global__ void k_dm_after_prune(uint32_t* dm_c, const uint32_t* dm_t, const uint32_t* unm, uint32_t cells) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x) {
        const uint32_t a = dm_c[c], t = dm_t[c];
        if (a > t) dm_c[c] = unm[c] < t ? unm[c] : t;
    }
}

// ---------------------------------------------------------------- fill (engine.cpp:499-546)
__global__ void k_fill_need(const uint32_t* dm_t, const uint32_t* dm_c, uint32_t* need, uint32_t cells) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x)
        need[c] = dm_t[c] > dm_c[c] ? dm_t[c] - dm_c[c] : 0u;
}

__global__ void k_dead_flags(PathDev P, uint32_t lb, uint32_t le, uint8_t* flags) {
    for (uint32_t i = lb + blockIdx.x * blockDim.x + threadIdx.x; i < le; i += gridDim.x * blockDim.x)
        flags[i - lb] = P.meta[i].z == kDead ? 1 : 0;
}

__global__ void __launch_bounds__(kT) k_fill_assign(SceneDev S, PathDev P, uint32_t li,
                                                    const uint32_t* dead, const uint32_t* dead_count,
                                                    uint64_t dead_prefix, const uint64_t* dead_prefix_dev,
                                                    const uint32_t* need_off,
                                                    const uint32_t* need_total, uint32_t cells,
                                                    Counters* ctr) {
    const LightDev& L = S.fp->lights[li];
    const uint32_t nd = *dead_count;
    const uint64_t total = *need_total;
    unsigned long long filled = 0;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nd; j += gridDim.x * blockDim.x) {
        const uint64_t u = (dead_prefix_dev ? dead_prefix_dev[li] : dead_prefix) + j;
        if (u >= total) continue;
        // cell c with need_off[c] <= u < need_off[c] + need[c]: last c with need_off[c] <= u
        uint32_t lo = 0, hi = cells;  // invariant: need_off[lo] <= u, answer in [lo, hi)
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if ((uint64_t)need_off[mid] <= u) lo = mid;
            else hi = mid;
        }
        const uint32_t c = lo;
        const uint32_t i = dead[j];
        const uint32_t p = P.base + i;
        const uint32_t epoch = P.epoch[i] + 1;
        P.epoch[i] = epoch;
        float cc[4];
        V3 o, d;
        sample_in_cell(L, c, S.seed_mix, p, epoch, cc, o, d);
        P.origin[i] = make_float4(o.x, o.y, o.z, 0.f);
        P.emis[i] = make_float4(d.x, d.y, d.z, 0.f);
        P.canon[i] = make_float4(cc[0], cc[1], cc[2], cc[3]);
        P.cell[i] = c;
        P.meta[i] = make_uchar4(0, 0, kLive, 1);
        P.rstart[i] = 0;
        ++filled;
    }
    warp_add(&ctr->filled, filled);
}

// fill's slot-exhaustion check (engine.cpp:512-513): single-shard form (dead_count), or the
// all-shard dead-slot total (host value, or device value of light li when sharded in-engine)
__global__ void k_fill_check(const uint32_t* dead_count, uint64_t dead_total, const uint64_t* dead_total_dev,
                             uint32_t li, const uint32_t* need_total, Counters* ctr) {
    const uint64_t avail = dead_count ? (uint64_t)*dead_count : (dead_total_dev ? dead_total_dev[li] : dead_total);
    if ((uint64_t)*need_total > avail) atomicAdd(&ctr->fill_overflow, 1ull);
}

// Sharded exchange: per-rank counts gathered as g[r * n + i]; prefix = the
// counts of the lower ranks (their paths have the lower ids), total = all ranks.
__global__ void k_rank_prefix_u32(const uint32_t* g, uint32_t n, uint32_t world, uint32_t rank, uint32_t* prefix,
                                  uint32_t* total) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t p = 0, t = 0;
        for (uint32_t r = 0; r < world; ++r) {
            const uint32_t v = g[(size_t)r * n + i];
            if (r < rank) p += v;
            t += v;
        }
        prefix[i] = p;
        total[i] = t;
    }
}
__global__ void k_rank_prefix_u64(const uint32_t* g, uint32_t n, uint32_t world, uint32_t rank, uint64_t* prefix,
                                  uint64_t* total) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint64_t p = 0, t = 0;
        for (uint32_t r = 0; r < world; ++r) {
            const uint64_t v = g[(size_t)r * n + i];
            if (r < rank) p += v;
            t += v;
        }
        prefix[i] = p;
        total[i] = t;
    }
}

__global__ void k_dm_after_fill(uint32_t* dm_c, const uint32_t* dm_t, uint32_t cells) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x)
        dm_c[c] = dm_c[c] < dm_t[c] ? dm_t[c] : dm_c[c];
}

// Verify-walk queue order (PRX_WALK_ORDER): sort keys of the flagged list, most expected rays
// first -- 1: most flagged segments, 2: earliest flagged segment, 3: most flagged segments,
// then earliest flagged segment.  Each walk depends on its own
// path only, so the order changes the persistent kernel's tail, not its results.
__global__ void k_walk_keys(const uint32_t* __restrict__ masks, const Counters* cnt, uint32_t* n32, uint32_t top,
                            int how, uint32_t n_max, uint32_t* keys, uint32_t* vals) {
    const uint32_t n = (uint32_t)cnt->flagged;
    if (blockIdx.x == 0 && threadIdx.x == 0) *n32 = n;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n && j < n_max; j += gridDim.x * blockDim.x) {
        const uint32_t f = masks[j];
        const uint32_t c = (uint32_t)__popc(f), first = f ? (uint32_t)(__ffs(f) - 1) : top;
        const uint32_t more = c < top ? top - c : 0u;
        keys[j] = how == 1 ? more : (how == 2 ? first : (more << 4 | (first < 15u ? first : 15u)));
        vals[j] = j;
    }
}
__global__ void k_walk_permute(const uint32_t* __restrict__ list, const uint32_t* __restrict__ masks,
                               const uint32_t* __restrict__ order, const uint32_t* n32, uint32_t* list2,
                               uint32_t* masks2) {
    const uint32_t n = *n32;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t o = order[j];
        list2[j] = list[o];
        masks2[j] = masks[o];
    }
}

// ---------------------------------------------------------------- trace (engine.cpp:548-598)
__global__ void k_retrace_flags(PathDev P, uint8_t* flags, uint32_t* start_of) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        const uint8_t r = P.rstart[i];
        const bool f = P.meta[i].z == kLive && r != kNoRetrace;
        flags[i] = f ? 1 : 0;
        if (start_of && f) start_of[i] = r;
    }
}

// stage_trace's per-path bounce loop (engine.cpp:557-586).  Persistent lanes at ray
// granularity: each lane traces one bounce of its current path per iteration and fetches the
// next queued path as soon as its own ends, so lanes whose paths escape early keep tracing
// instead of idling until the warp's longest path is done.
__global__ void __launch_bounds__(kT, PRX_TRACE_MINB) k_trace(SceneDev S, PathDev P, const uint32_t* __restrict__ list,
                                              const uint32_t* count, uint32_t* work, Counters* ctr) {
    const FrameParams* fp = S.fp;
    const uint32_t n = *count;
    unsigned long long traced = 0;
    uint32_t i = 0, p = 0, epoch = 0, b = 0;
    uchar4 m = make_uchar4(0, 0, 0, 0);
    V3 pos{}, dir{}, energy{};
    bool have = false, done = false;
    while (true) {
        if (refill_due(!have && !done, have)) {
            const uint32_t j = refill_slot(work, !have && !done);
            if (!have && !done) {
                if (j >= n) {
                    done = true;
                } else {
                    i = list[j];
                    p = P.base + i;
                    m = P.meta[i];
                    epoch = P.epoch[i];
                    b = P.rstart[i];
                    pos = b == 0 ? ld3(P.origin[i]) : ld3(P.pos_obj[kVS * (vix(P, b - 1, i))]);
                    dir = b == 0 ? ld3(P.emis[i]) : ld3(P.out_dir[kVS * (vix(P, b - 1, i))]);
                    energy = b == 0 ? fp->lights[light_of(fp, p)].flux_pp : ld3(P.energy[kVS * (vix(P, b - 1, i))]);
                    if (b >= P.B) {
                        truncate_path(P, i, b, false, m);
                        P.meta[i] = m;
                    } else {
                        have = true;
                    }
                }
            }
        }
        if (__all_sync(0xffffffffu, done)) break;
        if (!have) continue;
        ++traced;
        Hit h;
        bool escaped = false;
        if (!intersect_scene(S, pos, dir, S.eps, h)) {
            escaped = true;
        } else {
            const float4 am = __ldg(&S.mat[h.obj]);
            energy = mulv(energy, V3{am.x, am.y, am.z});
            const size_t v = vix(P, b, i);
            __stcs(&P.in_dir[kVS * (v)], make_float4(dir.x, dir.y, dir.z, 0.f));
            __stcs(&P.pos_obj[kVS * (v)], make_float4(h.pos.x, h.pos.y, h.pos.z, __uint_as_float(h.obj)));
            __stcs(&P.energy[kVS * (v)], make_float4(energy.x, energy.y, energy.z, S.gather_radius));
            const V3 out = sample_bounce(S, h.obj, h.normal, dir, p, epoch, b + 1);
            __stcs(&P.out_dir[kVS * (v)], make_float4(out.x, out.y, out.z, 0.f));
            pos = h.pos;
            dir = out;
            ++b;
        }
        if (escaped || b >= P.B) {
            truncate_path(P, i, b, escaped, m);
            P.meta[i] = m;
            have = false;
        }
    }
    warp_add(&ctr->traced, traced);
}

// segment accounting + refresh_path_info (engine.cpp:586-610) for every live path
__global__ void k_finalize(PathDev P, Counters* ctr) {
    unsigned long long segs_sum = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
        const uchar4 m = P.meta[i];
        if (m.z != kLive) continue;
        const uint32_t segs = m.x + m.y;
        segs_sum += segs;
        const uint8_t st = P.rstart[i];
        const uint32_t start = st == kNoRetrace ? 0u : (st < 15 ? st : 15u);
        P.path_info[i] = pack_path_info(P.cell[i], segs > 1 ? segs : 1u, start, false, m.w == 0);
    }
    warp_add(&ctr->segments, segs_sum);
}

// ---------------------------------------------------------------- scene queries
// intersect_scene / occluded (scene.cpp:136-177) for a batch of rays {o, d, t_min, t_max}:
// closest -> 9 floats {t, object, triangle, position, normal}; any-hit -> 1 float.
__global__ void __launch_bounds__(kT, PRX_TRACE_MINB) k_intersect_batch(SceneDev S, const float* __restrict__ rays,
                                                                        uint32_t n, int any_hit, float* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float* q = rays + 8ull * i;
        const V3 o{q[0], q[1], q[2]}, d{q[3], q[4], q[5]};
        if (any_hit) {
            out[i] = occluded(S, o, d, q[6], q[7]) ? 1.0f : 0.0f;
            continue;
        }
        Hit h;
        uint32_t tri = 0;
        float* w = out + 9ull * i;
        if (intersect_scene(S, o, d, q[6], h, q[7], &tri)) {
            w[0] = h.t;
            w[1] = __uint_as_float(h.obj);
            w[2] = __uint_as_float(tri);
            w[3] = h.pos.x, w[4] = h.pos.y, w[5] = h.pos.z;
            w[6] = h.normal.x, w[7] = h.normal.y, w[8] = h.normal.z;
        } else {
            w[0] = 0.0f;
            w[1] = __uint_as_float(kInvalidObj);
            for (int k = 2; k < 9; ++k) w[k] = 0.0f;
        }
    }
}

// ---------------------------------------------------------------- layout conversion
struct PhotonRec {  // photon_store.hpp:13-21
    float dx, dy, dz;
    uint32_t obj;
    float ex, ey, ez;
    float radius;
};
struct AuxRec {  // photon_store.hpp:75-78
    float px, py, pz, ox, oy, oz;
};

__global__ void k_pack(PathDev P, PhotonRec* ph, AuxRec* aux) {
    const size_t total = (size_t)P.n * P.B;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < total; v += (size_t)gridDim.x * blockDim.x) {
        const float4 po = P.pos_obj[kVS * (v)], en = P.energy[kVS * (v)], in = P.in_dir[kVS * (v)], od = P.out_dir[kVS * (v)];
        if (ph) ph[v] = PhotonRec{in.x, in.y, in.z, __float_as_uint(po.w), en.x, en.y, en.z, en.w};
        if (aux) aux[v] = AuxRec{po.x, po.y, po.z, od.x, od.y, od.z};
    }
}

__global__ void k_unpack(PathDev P, const PhotonRec* ph, const AuxRec* aux) {
    const size_t total = (size_t)P.n * P.B;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < total; v += (size_t)gridDim.x * blockDim.x) {
        if (ph) {
            const PhotonRec r = ph[v];
            __stcs(&P.in_dir[kVS * (v)], make_float4(r.dx, r.dy, r.dz, 0.f));
            __stcs(&P.energy[kVS * (v)], make_float4(r.ex, r.ey, r.ez, r.radius));
            P.pos_obj[kVS * (v)].w = __uint_as_float(r.obj);
        }
        if (aux) {
            const AuxRec a = aux[v];
            P.pos_obj[kVS * (v)].x = a.px;
            P.pos_obj[kVS * (v)].y = a.py;
            P.pos_obj[kVS * (v)].z = a.pz;
            __stcs(&P.out_dir[kVS * (v)], make_float4(a.ox, a.oy, a.oz, 0.f));
        }
    }
}

}  // namespace

#define LAUNCH(kernel, n, ...)                                                   \
    do {                                                                         \
        kernel<<<launch_grid((n), kT), kT, 0, st>>>(__VA_ARGS__);               \
        ++g_launches;                                                            \
    } while (0)

void launch_init_dm_target(const LightDev* L, uint32_t n, uint64_t seed_mix, uint32_t* dm_t,
                           cudaStream_t st) {
    LAUNCH(k_init_dm_target, n, *L, n, seed_mix, dm_t);
}
void launch_transform_dynamic(const float4* local, const uint32_t* tri_xf, const float4* xf, uint32_t n,
                              float4* world, cudaStream_t st) {
    if (n) LAUNCH(k_transform_dynamic, n, local, tri_xf, xf, n, world);
}
void launch_frame_reset(PathDev P, int record, Counters* ctr, cudaStream_t st) {
    LAUNCH(k_frame_reset, (P.n + 3) / 4, P, record, ctr);
}
void launch_release_all(PathDev P, cudaStream_t st) { LAUNCH(k_release_all, P.n, P); }
void launch_update_origins(SceneDev S, PathDev P, Counters* ctr, cudaStream_t st) {
    LAUNCH(k_update_origins, P.n, S, P, ctr);
}
void launch_occlusion_flags(SceneDev S, PathDev P, int mode, int record, uint32_t* list, uint32_t* masks,
                            Counters* ctr, cudaStream_t st) {
    LAUNCH(k_occlusion_flags, P.n, S, P, mode, record, list, masks, ctr);
}
template <typename K>
static int persistent_grid(K kernel) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kT, 0);
    return sms * (per_sm > 0 ? per_sm : 1);
}

#ifdef PRX_CERT_STATS
static void cert_report(const char* stage, cudaStream_t st) {
    unsigned long long c[8] = {};
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(c, g_cert_stats, sizeof(c));
    std::fprintf(stderr, "[cert] %s: closest %llu fail %llu | any %llu fail %llu | nodes s %llu d %llu | tris s %llu d %llu\n",
                 stage, c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]);
    const unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_cert_stats, z, sizeof(z));
}
#define CERT_REPORT(stage) cert_report(stage, st)
#else
#define CERT_REPORT(stage) ((void)0)
#endif

void launch_walk_keys(const uint32_t* masks, const Counters* cnt, uint32_t* n32, uint32_t top, int how,
                      uint32_t n_max, uint32_t* keys, uint32_t* vals, cudaStream_t st) {
    LAUNCH(k_walk_keys, n_max, masks, cnt, n32, top, how, n_max, keys, vals);
}
void launch_walk_permute(const uint32_t* list, const uint32_t* masks, const uint32_t* order, const uint32_t* n32,
                         uint32_t n_max, uint32_t* list2, uint32_t* masks2, cudaStream_t st) {
    LAUNCH(k_walk_permute, n_max, list, masks, order, n32, list2, masks2);
}
void launch_verify_error(SceneDev S, PathDev P, float threshold, const uint32_t* list, const uint32_t* masks,
                         const Counters* cnt, uint32_t* work, Counters* ctr, cudaStream_t st) {
    if (S.fast) {  // one-shot walks on the fast traversal
        static int grid = persistent_grid(k_verify_error_walk);
        cudaMemsetAsync(work, 0, 4, st);
        CERT_REPORT("before verify");
        k_verify_error_walk<<<grid, kT, 0, st>>>(S, P, threshold, list, masks, cnt, work, ctr);
        CERT_REPORT("verify walk");
    } else {  // resumable reference-order traversal, persistent lanes
        static int grid = persistent_grid(k_verify_error);
        cudaMemsetAsync(work, 0, 4, st);
        k_verify_error<<<grid, kT, 0, st>>>(S, P, threshold, list, masks, cnt, work, ctr);
    }
    ++g_launches;
}
void launch_compute_dm(SceneDev S, PathDev P, Counters* ctr, cudaStream_t st) {
    LAUNCH(k_compute_dm, P.n, S, P, ctr);
}
void launch_prune_mark(SceneDev S, PathDev P, const uint32_t* frame, uint32_t* const* unmarked, uint8_t* pruned,
                       uint8_t* cand, cudaStream_t st) {
    LAUNCH(k_prune_mark, P.n, S, P, frame, unmarked, pruned, cand);
}
void launch_prune_trim_flags(PathDev P, const FrameParams* fp, uint32_t* const* unm_total, const uint8_t* cand,
                             uint8_t* trim, cudaStream_t st) {
    LAUNCH(k_prune_trim_flags, P.n, P, fp, unm_total, cand, trim);
}
void launch_prune_keys(PathDev P, const FrameParams* fp, const uint32_t* list, const uint32_t* count,
                       uint32_t* keys, uint32_t* vals, uint32_t n_max, cudaStream_t st) {
    LAUNCH(k_prune_keys, n_max, P, fp, list, count, keys, vals);
}
void launch_prune_trim(PathDev P, const FrameParams* fp, const uint32_t* keys, const uint32_t* vals,
                       const uint32_t* count, uint32_t n_max, uint32_t* const* seg_start,
                       uint32_t* const* prefix, uint8_t* pruned, cudaStream_t st) {
    (void)P;
    LAUNCH(k_prune_heads, n_max, keys, count, seg_start);
    LAUNCH(k_prune_trim, n_max, fp, keys, vals, count, seg_start, prefix, pruned);
}
void launch_prune_apply(PathDev P, const uint8_t* pruned, int clear_records, cudaStream_t st) {
    LAUNCH(k_prune_apply, P.n, P, pruned, clear_records);
}
void launch_dm_after_prune(uint32_t* dm_c, const uint32_t* dm_t, const uint32_t* unm, uint32_t cells,
                           cudaStream_t st) {
    LAUNCH(k_dm_after_prune, cells, dm_c, dm_t, unm, cells);
}
void launch_fill_need(const uint32_t* dm_t, const uint32_t* dm_c, uint32_t* need, uint32_t cells,
                      cudaStream_t st) {
    LAUNCH(k_fill_need, cells, dm_t, dm_c, need, cells);
}
void launch_dead_flags(PathDev P, uint32_t lb, uint32_t le, uint8_t* flags, cudaStream_t st) {
    if (le > lb) LAUNCH(k_dead_flags, le - lb, P, lb, le, flags);
}
void launch_fill_assign(SceneDev S, PathDev P, uint32_t li, const uint32_t* dead, const uint32_t* dead_count,
                        uint32_t n_max, uint64_t dead_prefix, const uint64_t* dead_prefix_dev,
                        const uint32_t* need_off, const uint32_t* need_total, uint32_t cells, Counters* ctr,
                        cudaStream_t st) {
    LAUNCH(k_fill_assign, n_max, S, P, li, dead, dead_count, dead_prefix, dead_prefix_dev, need_off, need_total,
           cells, ctr);
}
void launch_fill_check(const uint32_t* dead_count, uint64_t dead_total, const uint64_t* dead_total_dev, uint32_t li,
                       const uint32_t* need_total, Counters* ctr, cudaStream_t st) {
    k_fill_check<<<1, 1, 0, st>>>(dead_count, dead_total, dead_total_dev, li, need_total, ctr);
    ++g_launches;
}
void launch_rank_prefix_u32(const uint32_t* g, uint32_t n, uint32_t world, uint32_t rank, uint32_t* prefix,
                            uint32_t* total, cudaStream_t st) {
    LAUNCH(k_rank_prefix_u32, n, g, n, world, rank, prefix, total);
}
void launch_rank_prefix_u64(const uint32_t* g, uint32_t n, uint32_t world, uint32_t rank, uint64_t* prefix,
                            uint64_t* total, cudaStream_t st) {
    LAUNCH(k_rank_prefix_u64, n, g, n, world, rank, prefix, total);
}
void launch_dm_after_fill(uint32_t* dm_c, const uint32_t* dm_t, uint32_t cells, cudaStream_t st) {
    LAUNCH(k_dm_after_fill, cells, dm_c, dm_t, cells);
}
void launch_retrace_flags(PathDev P, uint8_t* flags, uint32_t* start_of, cudaStream_t st) {
    LAUNCH(k_retrace_flags, P.n, P, flags, start_of);
}
void launch_trace(SceneDev S, PathDev P, const uint32_t* list, const uint32_t* count, uint32_t* work,
                  Counters* ctr, cudaStream_t st) {
    static int grid = persistent_grid(k_trace);
    cudaMemsetAsync(work, 0, 4, st);
    CERT_REPORT("before trace");
    k_trace<<<grid, kT, 0, st>>>(S, P, list, count, work, ctr);
    CERT_REPORT("trace");
    ++g_launches;
}
void launch_intersect_batch(SceneDev S, const float* rays, uint32_t n, int any_hit, float* out, cudaStream_t st) {
    LAUNCH(k_intersect_batch, n, S, rays, n, any_hit, out);
}
void launch_finalize(PathDev P, Counters* ctr, cudaStream_t st) { LAUNCH(k_finalize, P.n, P, ctr); }
void launch_pack_photons(PathDev P, void* photons, void* aux, cudaStream_t st) {
    LAUNCH(k_pack, (uint64_t)P.n * P.B, P, static_cast<PhotonRec*>(photons), static_cast<AuxRec*>(aux));
}
void launch_unpack_photons(PathDev P, const void* photons, const void* aux, cudaStream_t st) {
    LAUNCH(k_unpack, (uint64_t)P.n * P.B, P, static_cast<const PhotonRec*>(photons),
           static_cast<const AuxRec*>(aux));
}

}  // namespace prx
