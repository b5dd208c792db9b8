// Timing of the radix sort passes on synthetic keys (profiling aid): nvcc -std=c++17 -O2
// -gencode arch=compute_100a,code=sm_100a -Ipaper_2111_06906_b200/csrc profiles/prims_bench.cu
// paper_2111_06906_b200/csrc/prims.cu -o /tmp/pb;
// prims_bench n bits ragged_fill(0 = dense input, else percent of each tile kept)
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "prims.h"

namespace prx {
std::atomic<uint64_t> g_launches{0};
}

int main(int argc, char** argv) {
    const uint32_t n = argc > 1 ? std::atoi(argv[1]) : 25000000;
    const int bits = argc > 2 ? std::atoi(argv[2]) : 16;
    const int fill = argc > 3 ? std::atoi(argv[3]) : 0;
    std::mt19937_64 rng(1);
    const uint32_t T = prx::kSortTile, tiles = (n + T - 1) / T;
    std::vector<uint32_t> k(n), v(n), cnt(tiles, 0);
    uint32_t tot = 0;
    for (uint32_t t = 0; t < tiles; ++t)
        for (uint32_t i = t * T; i < std::min<uint64_t>((uint64_t)(t + 1) * T, n); ++i) {
            if (fill && (int)(rng() % 100) >= fill) continue;
            const uint32_t o = fill ? t * T + cnt[t] : i;
            k[o] = static_cast<uint32_t>(rng()) & ((1u << bits) - 1u);
            v[o] = i;
            ++cnt[t];
            ++tot;
        }
    uint32_t *dk, *dv, *dk2, *dv2, *dc, *dn;
    float4 *pa, *oa, *ob;
    void* scratch;
    cudaMalloc(&dk, 4ull * n), cudaMalloc(&dv, 4ull * n), cudaMalloc(&dk2, 4ull * n), cudaMalloc(&dv2, 4ull * n);
    cudaMalloc(&dc, 4ull * tiles), cudaMalloc(&dn, 4);
    cudaMalloc(&pa, 32ull * n), cudaMalloc(&oa, 16ull * n), cudaMalloc(&ob, 16ull * n);
    cudaMalloc(&scratch, prx::prim_scratch_bytes(n));
    cudaMemcpy(dc, cnt.data(), 4ull * tiles, cudaMemcpyHostToDevice);
    cudaMemcpy(dn, &tot, 4, cudaMemcpyHostToDevice);
    prx::SortGather g;
    g.a = pa;
    g.b = pa + 1;
    g.stride = 2;
    g.out_a = oa;
    g.out_b = ob;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemcpy(dk, k.data(), 4ull * n, cudaMemcpyHostToDevice);
        cudaMemcpy(dv, v.data(), 4ull * n, cudaMemcpyHostToDevice);
        cudaEventRecord(e0);
        prx::radix_sort_gather(dk, dv, dk2, dv2, n, dn, bits, g, scratch, 0, fill ? dc : nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    std::printf("n=%u live=%u bits=%d fill=%d sort+gather %.3f ms (%s)\n", n, tot, bits, fill, best,
                cudaGetErrorString(cudaGetLastError()));
    return 0;
}
