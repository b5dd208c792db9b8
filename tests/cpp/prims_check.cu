// Randomised check of the device primitives (prims.cu) against host references:
// stable LSD radix sort of (key, value) pairs, stable compaction and exclusive scan, with
// element counts on the device below the host-side capacity (the engine's usage).
// usage: prims_check [seed]   -- prints "ok <cases>" or the first mismatch, exit code != 0
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#include "prims.h"

namespace prx {
std::atomic<uint64_t> g_launches{0};
}

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::printf("cuda error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(2);                                                                       \
        }                                                                                       \
    } while (0)

template <typename T>
T* dev(const std::vector<T>& h, size_t extra = 0) {
    T* p = nullptr;
    CK(cudaMalloc(&p, sizeof(T) * (h.size() + extra + 1)));
    if (!h.empty()) CK(cudaMemcpy(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
    return p;
}

template <typename T>
std::vector<T> host(const T* p, size_t n) {
    std::vector<T> h(n);
    if (n) CK(cudaMemcpy(h.data(), p, sizeof(T) * n, cudaMemcpyDeviceToHost));
    return h;
}

static int fail(const char* what, uint32_t n_max, uint32_t n, int bits, size_t at) {
    std::printf("FAIL %s n_max=%u n=%u bits=%d at %zu\n", what, n_max, n, bits, at);
    return 1;
}

// sort: keys with `bits` random low bits (plus garbage above, which must be ignored only if
// the caller masks -- the engine's keys never carry bits above `bits`), values = positions
static int check_sort(std::mt19937_64& rng, uint32_t n_max, uint32_t n, int bits, int skew) {
    std::vector<uint32_t> k(n_max), v(n_max);
    const uint32_t kmask = bits >= 32 ? 0xFFFFFFFFu : ((1u << bits) - 1u);
    for (uint32_t i = 0; i < n_max; ++i) {
        uint32_t x = static_cast<uint32_t>(rng()) & kmask;
        if (skew == 1) x &= 0x7u;                           // few distinct keys: long runs
        if (skew == 2) x = (rng() % 8 == 0) ? x : 5u & kmask;  // one dominant key
        k[i] = x;
        v[i] = i;
    }
    uint32_t *dk = dev(k), *dv = dev(v), *dk2 = dev(k), *dv2 = dev(v), *dn = dev(std::vector<uint32_t>{n});
    void* scratch = nullptr;
    CK(cudaMalloc(&scratch, prx::prim_scratch_bytes(n_max)));
    prx::radix_sort_pairs(dk, dv, dk2, dv2, n_max, dn, bits, scratch, 0);
    CK(cudaDeviceSynchronize());
    const auto gk = host(dk, n), gv = host(dv, n);
    std::vector<uint32_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0u);
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return k[a] < k[b]; });
    for (uint32_t j = 0; j < n; ++j)
        if (gk[j] != k[idx[j]] || gv[j] != idx[j]) return fail("radix_sort_pairs", n_max, n, bits, j);
    // the same sort gathering two float4 payload streams (stride 2) in its last pass
    {
        std::vector<float4> pay(2 * (size_t)n_max);
        for (size_t q = 0; q < pay.size(); ++q)
            pay[q] = make_float4((float)q, (float)(q * 3), (float)(q & 1023), (float)(q % 7));
        float4 *dp = dev(pay), *oa = dev(std::vector<float4>(n_max)), *ob = dev(std::vector<float4>(n_max));
        uint32_t *k2 = dev(k), *v2 = dev(v);
        prx::SortGather g;
        g.a = dp;
        g.b = dp + 1;
        g.stride = 2;
        g.out_a = oa;
        g.out_b = ob;
        prx::radix_sort_gather(k2, v2, dk2, dv2, n_max, dn, bits, g, scratch, 0);
        CK(cudaDeviceSynchronize());
        const auto ga = host(oa, n), gb = host(ob, n);
        for (uint32_t j = 0; j < n; ++j) {
            const float4 a = pay[2 * (size_t)idx[j]], b = pay[2 * (size_t)idx[j] + 1];
            if (ga[j].x != a.x || ga[j].y != a.y || ga[j].z != a.z || ga[j].w != a.w || gb[j].x != b.x ||
                gb[j].w != b.w)
                return fail("radix_sort_gather", n_max, n, bits, j);
        }
        cudaFree(dp), cudaFree(oa), cudaFree(ob), cudaFree(k2), cudaFree(v2);
    }
    // ragged tiles: tile t of kSortTile slots holds a random in-order subset of its pairs
    {
        const uint32_t T = prx::kSortTile, tiles = (n_max + T - 1) / T;
        std::vector<uint32_t> rk(n_max, 0xDEADBEEFu), rv(n_max, 0xDEADBEEFu), cnt(tiles, 0), sub_k, sub_v;
        for (uint32_t t = 0; t < tiles; ++t)
            for (uint32_t i = t * T; i < std::min<uint64_t>((uint64_t)(t + 1) * T, n_max); ++i)
                if (rng() % 3 != 0) {
                    rk[t * T + cnt[t]] = k[i];
                    rv[t * T + cnt[t]] = i;
                    ++cnt[t];
                    sub_k.push_back(k[i]);
                    sub_v.push_back(i);
                }
        const uint32_t tot = static_cast<uint32_t>(sub_k.size());
        std::vector<float4> pay(n_max);
        for (uint32_t q = 0; q < n_max; ++q) pay[q] = make_float4((float)q, 0.f, 0.f, (float)(q & 4095));
        uint32_t *k2 = dev(rk), *v2 = dev(rv), *dc = dev(cnt), *dt = dev(std::vector<uint32_t>{tot});
        float4 *dp = dev(pay), *oa = dev(std::vector<float4>(n_max)), *ob = dev(std::vector<float4>(n_max));
        prx::SortGather g;
        g.a = dp;
        g.b = dp;
        g.stride = 1;
        g.out_a = oa;
        g.out_b = ob;
        prx::radix_sort_gather(k2, v2, dk2, dv2, n_max, dt, bits, g, scratch, 0, dc);
        CK(cudaDeviceSynchronize());
        std::vector<uint32_t> o(tot);
        std::iota(o.begin(), o.end(), 0u);
        std::stable_sort(o.begin(), o.end(), [&](uint32_t a, uint32_t b) { return sub_k[a] < sub_k[b]; });
        const auto ga = host(oa, tot);
        for (uint32_t j = 0; j < tot; ++j)
            if (ga[j].x != pay[sub_v[o[j]]].x || ga[j].w != pay[sub_v[o[j]]].w)
                return fail("radix_sort_gather ragged", n_max, tot, bits, j);
        cudaFree(k2), cudaFree(v2), cudaFree(dc), cudaFree(dt), cudaFree(dp), cudaFree(oa), cudaFree(ob);
    }
    // elements beyond n stay untouched in keys/vals
    const auto tail = host(dk + n, n_max - n);
    for (uint32_t j = 0; j < n_max - n; ++j)
        if (tail[j] != k[n + j]) return fail("radix tail", n_max, n, bits, j);
    cudaFree(dk), cudaFree(dv), cudaFree(dk2), cudaFree(dv2), cudaFree(dn), cudaFree(scratch);
    return 0;
}

static int check_compact_scan(std::mt19937_64& rng, uint32_t n_max, uint32_t n, int density) {
    std::vector<uint8_t> f(n_max);
    std::vector<uint32_t> x(n_max);
    for (uint32_t i = 0; i < n_max; ++i) {
        f[i] = (rng() % 100) < (uint64_t)density ? 1 : 0;
        x[i] = static_cast<uint32_t>(rng() % 1000);
    }
    uint8_t* df = dev(f);
    uint32_t *dx = dev(x), *dout = dev(std::vector<uint32_t>(n_max)), *dn = dev(std::vector<uint32_t>{n}),
             *dcnt = dev(std::vector<uint32_t>{0}), *dtot = dev(std::vector<uint32_t>{0});
    void* scratch = nullptr;
    CK(cudaMalloc(&scratch, prx::prim_scratch_bytes(n_max)));
    prx::compact_u8(df, n_max, dn, 7, dout, dcnt, scratch, 0);
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> want;
    for (uint32_t i = 0; i < n; ++i)
        if (f[i]) want.push_back(7 + i);
    const uint32_t cnt = host(dcnt, 1)[0];
    if (cnt != want.size()) return fail("compact count", n_max, n, 0, cnt);
    const auto got = host(dout, cnt);
    for (uint32_t j = 0; j < cnt; ++j)
        if (got[j] != want[j]) return fail("compact_u8", n_max, n, 0, j);
    {  // pairs form: keys from a per-element table, all n_max elements
        std::vector<uint32_t> key_of(n_max);
        for (uint32_t i = 0; i < n_max; ++i) key_of[i] = static_cast<uint32_t>(rng());
        uint32_t *dko = dev(key_of), *pk = dev(std::vector<uint32_t>(n_max)), *pv = dev(std::vector<uint32_t>(n_max));
        prx::compact_u8_pairs(df, dko, n_max, pk, pv, dcnt, scratch, 0);
        CK(cudaDeviceSynchronize());
        std::vector<uint32_t> wi;
        for (uint32_t i = 0; i < n_max; ++i)
            if (f[i]) wi.push_back(i);
        const uint32_t c2 = host(dcnt, 1)[0];
        if (c2 != wi.size()) return fail("compact_u8_pairs count", n_max, n_max, 0, c2);
        const auto gk = host(pk, c2), gv = host(pv, c2);
        for (uint32_t j = 0; j < c2; ++j)
            if (gv[j] != wi[j] || gk[j] != key_of[wi[j]]) return fail("compact_u8_pairs", n_max, n_max, 0, j);
        cudaFree(dko), cudaFree(pk), cudaFree(pv);
    }
    prx::scan_exclusive_u32(dx, dx, n_max, dn, dtot, scratch, 0);
    CK(cudaDeviceSynchronize());
    const auto sc = host(dx, n);
    uint32_t run = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (sc[i] != run) return fail("scan", n_max, n, 0, i);
        run += x[i];
    }
    if (host(dtot, 1)[0] != run) return fail("scan total", n_max, n, 0, 0);
    cudaFree(df), cudaFree(dx), cudaFree(dout), cudaFree(dn), cudaFree(dcnt), cudaFree(dtot), cudaFree(scratch);
    return 0;
}

int main(int argc, char** argv) {
    std::mt19937_64 rng(argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1);
    int cases = 0, bad = 0;
    const uint32_t sizes[][2] = {{1, 1},         {5, 3},           {4095, 4095},   {4096, 4096},   {4097, 4097},
                                 {10000, 0},     {10000, 1},       {65537, 40000}, {300000, 299999},
                                 {1u << 20, 777777}, {3000000, 2500001}};
    const int bit_list[] = {1, 4, 8, 9, 16, 20, 23, 31};
    for (auto& sz : sizes)
        for (int bits : bit_list)
            for (int skew = 0; skew < 3; ++skew) {
                if (sz[0] > 300000 && (skew != 0 || (bits != 20 && bits != 23))) continue;
                bad += check_sort(rng, sz[0], sz[1], bits, skew);
                ++cases;
                if (bad) return 1;
            }
    for (auto& sz : sizes)
        for (int density : {0, 3, 50, 100}) {
            bad += check_compact_scan(rng, sz[0], sz[1], density);
            ++cases;
            if (bad) return 1;
        }
    std::printf("ok %d\n", cases);
    return 0;
}
