// splat.cu -- screen-space photon splatting (north_star subsystem 6), replacing the
// reference's per-pixel gather_image (gather.cpp:35-75).
//
//   K11 gbuffer:  per pixel, camera_ray (gather.cpp:22-33) + intersect_scene -> hit
//                 position and object (same float ops as the reference).
//   K12 splat:    per live photon, the screen rectangle that can contain pixels whose
//                 hit point lies within r is derived from the photon's bounding box in
//                 camera space; every pixel in it passes the reference's own filters
//                 (same object, |x_ph - x_px|^2 <= r^2, photon in the 27-cell grid
//                 neighbourhood of the pixel, gather.hpp:45-58) and atomically adds the
//                 photon energy -- into a CTA-private shared-memory image when the frame
//                 fits (120x90x3 fp32 = 130 KB), else straight into global memory.
//   resolve:      L = sum(E) * albedo / pi / (pi r^2) (gather.cpp:71).
// Only the fp32 summation order differs from the reference (tolerance class C).
#include "device_scene.cuh"
#include "kernels.h"

namespace prx {

namespace {

constexpr int kT = 256;

__global__ void k_gbuffer(SceneDev S, CamDev C, float4* gbuf) {
    const uint32_t n = C.w * C.h;
    for (uint32_t pix = blockIdx.x * blockDim.x + threadIdx.x; pix < n; pix += gridDim.x * blockDim.x) {
        const uint32_t px = pix % C.w, py = pix / C.w;
        const float sx = (2.0f * ((float)px + 0.5f) / (float)C.w - 1.0f) * C.tan_half * C.aspect;
        const float sy = (1.0f - 2.0f * ((float)py + 0.5f) / (float)C.h) * C.tan_half;
        const V3 dir = normalized(add(add(C.fwd, mul(C.right, sx)), mul(C.up, sy)));
        Hit h;
        if (intersect_scene(S, C.pos, dir, 0.0f, h))
            gbuf[pix] = make_float4(h.pos.x, h.pos.y, h.pos.z, __uint_as_float(h.obj));
        else
            gbuf[pix] = make_float4(0.f, 0.f, 0.f, __uint_as_float(kInvalidObj));
    }
}

__device__ __forceinline__ long long cell_coord(float v, float r) { return (long long)floorf(v / r); }

template <bool kShared>
__global__ void __launch_bounds__(kT) k_splat(PathDev P, CamDev C, float radius,
                                              const float4* __restrict__ gbuf, float* __restrict__ img) {
    extern __shared__ float simg[];
    const uint32_t npx = C.w * C.h;
    if (kShared) {
        for (uint32_t k = threadIdx.x; k < 3 * npx; k += blockDim.x) simg[k] = 0.0f;
        __syncthreads();
    }
    float* acc = kShared ? simg : img;
    const float r2 = radius * radius;
    const float ta = C.tan_half * C.aspect;
    const size_t total = (size_t)P.n * P.B;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < total; v += (size_t)gridDim.x * blockDim.x) {
        const float4 po = P.pos_obj[v];
        const uint32_t obj = __float_as_uint(po.w);
        if (obj == kInvalidObj) continue;
        const float4 en = P.energy[v];
        const V3 ph{po.x, po.y, po.z};
        const V3 q = sub(ph, C.pos);
        const float z = dot(q, C.fwd), x = dot(q, C.right), y = dot(q, C.up);
        int x0 = 0, x1 = (int)C.w - 1, y0 = 0, y1 = (int)C.h - 1;
        if (z > radius * 1.001f + 1e-4f) {
            const float zl = z - radius, zh = z + radius;
            const float sxa = fminf((x - radius) / zl, (x - radius) / zh);
            const float sxb = fmaxf((x + radius) / zl, (x + radius) / zh);
            const float sya = fminf((y - radius) / zl, (y - radius) / zh);
            const float syb = fmaxf((y + radius) / zl, (y + radius) / zh);
            const float fx0 = (sxa / ta + 1.0f) * 0.5f * (float)C.w - 0.5f;
            const float fx1 = (sxb / ta + 1.0f) * 0.5f * (float)C.w - 0.5f;
            const float fy0 = (1.0f - syb / C.tan_half) * 0.5f * (float)C.h - 0.5f;
            const float fy1 = (1.0f - sya / C.tan_half) * 0.5f * (float)C.h - 0.5f;
            if (fx1 < -2.0f || fy1 < -2.0f || fx0 > (float)C.w + 1.0f || fy0 > (float)C.h + 1.0f) continue;
            x0 = max(0, (int)floorf(fx0) - 1);
            x1 = min((int)C.w - 1, (int)ceilf(fx1) + 1);
            y0 = max(0, (int)floorf(fy0) - 1);
            y1 = min((int)C.h - 1, (int)ceilf(fy1) + 1);
        }
        const long long cx = cell_coord(ph.x, radius), cy = cell_coord(ph.y, radius), cz = cell_coord(ph.z, radius);
        for (int py = y0; py <= y1; ++py) {
            for (int px = x0; px <= x1; ++px) {
                const uint32_t pix = (uint32_t)py * C.w + (uint32_t)px;
                const float4 g = __ldg(&gbuf[pix]);
                if (__float_as_uint(g.w) != obj) continue;
                const V3 d = sub(ph, V3{g.x, g.y, g.z});
                if (dot(d, d) > r2) continue;
                const long long gx = cell_coord(g.x, radius), gy = cell_coord(g.y, radius), gz = cell_coord(g.z, radius);
                if (llabs(cx - gx) > 1 || llabs(cy - gy) > 1 || llabs(cz - gz) > 1) continue;
                atomicAdd(&acc[3 * pix], en.x);
                atomicAdd(&acc[3 * pix + 1], en.y);
                atomicAdd(&acc[3 * pix + 2], en.z);
            }
        }
    }
    if (kShared) {
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < 3 * npx; k += blockDim.x) {
            const float s = simg[k];
            if (s != 0.0f) atomicAdd(&img[k], s);
        }
    }
}

__global__ void k_resolve(const float4* __restrict__ gbuf, const float4* __restrict__ mat, float* img,
                          uint32_t n, float inv_pi, float inv_area) {
    for (uint32_t pix = blockIdx.x * blockDim.x + threadIdx.x; pix < n; pix += gridDim.x * blockDim.x) {
        const uint32_t obj = __float_as_uint(gbuf[pix].w);
        if (obj == kInvalidObj) {
            img[3 * pix] = img[3 * pix + 1] = img[3 * pix + 2] = 0.0f;
            continue;
        }
        const float4 a = mat[obj];
        const V3 rad{img[3 * pix], img[3 * pix + 1], img[3 * pix + 2]};
        const V3 out = mul(mul(mulv(rad, V3{a.x, a.y, a.z}), inv_pi), inv_area);
        img[3 * pix] = out.x;
        img[3 * pix + 1] = out.y;
        img[3 * pix + 2] = out.z;
    }
}

}  // namespace

void launch_splat(SceneDev S, PathDev P, const CamDev& C, float radius, float4* gbuf, float* img,
                  float inv_pi, float inv_area, cudaStream_t st) {
    const uint32_t npx = C.w * C.h;
    k_gbuffer<<<launch_grid(npx, kT), kT, 0, st>>>(S, C, gbuf);
    cudaMemsetAsync(img, 0, 12ull * npx, st);
    const size_t smem = 12ull * npx;
    int dev = 0;
    cudaGetDevice(&dev);
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (smem <= 200u * 1024u) {
        cudaFuncSetAttribute(k_splat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_splat<true><<<n_sm, kT, smem, st>>>(P, C, radius, gbuf, img);
    } else {
        k_splat<false><<<launch_grid((uint64_t)P.n * P.B, kT), kT, 0, st>>>(P, C, radius, gbuf, img);
    }
    k_resolve<<<launch_grid(npx, kT), kT, 0, st>>>(gbuf, S.mat, img, npx, inv_pi, inv_area);
    g_launches += 3;
}

}  // namespace prx
