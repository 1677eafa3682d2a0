// Speed-of-light of the 3F2N traffic mix on one B200: 4 B read + 12 B
// written per pixel (planar fp32 normals), no arithmetic, the strip kernel's geometry (warp =
// 128 columns x strip rows, lane = 4 columns).  Store paths compared:
//   stg_cs   three st.global.cs.v4 per lane-row (the production epilogue)
//   stg_wb   three st.global.v4 (write-back)
//   bulk     the row's three 512-B plane segments staged in shared memory (STS.128) and written
//            by cp.async.bulk.global.shared::cta (TMA bulk store), double-buffered per warp
//   tma_ld   rows in through a TMA tensor ring (as tfn_tma.cuh), st.global.cs out
// plus references: copy (4 B in / 4 B out), write-only (12 B/px), read-only (4 B/px).
// Prints one JSON object (GB/s of algorithmic bytes, best of 10 after warm-up).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int STRIP = 48;
struct Geo { int B, H, W; };

__device__ __forceinline__ int items_of(const Geo& g) { return ((g.W + 127) / 128) * ((g.H + STRIP - 1) / STRIP) * g.B; }

template <int MODE>   // 0 stg_cs, 1 stg_wb, 2 write-only, 3 read-only, 4 copy
__global__ void __launch_bounds__(128) k_stg(const float* __restrict__ in, float* __restrict__ out, Geo g, float* sink) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const long long HW = (long long)g.H * g.W;
    const int sxn = (g.W + 127) / 128, syn = (g.H + STRIP - 1) / STRIP;
    float acc = 0.f;
    for (int it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items_of(g); it += nw) {
        const int sx = it % sxn, t = it / sxn, sy = t % syn, b = t / syn;
        const int c0 = sx * 128 + lane * 4;
        if (c0 >= g.W) continue;
        const int y1 = min((sy + 1) * STRIP, g.H);
        for (int v = sy * STRIP; v < y1; ++v) {
            const long long p = (long long)b * HW + (long long)v * g.W + c0;
            float4 x = make_float4(1.f, 2.f, 3.f, 4.f);
            if (MODE != 2) x = __ldg(reinterpret_cast<const float4*>(in + p));
            if (MODE == 3) { acc += x.x + x.y + x.z + x.w; continue; }
            float* o = out + (long long)b * 3 * HW + (long long)v * g.W + c0;
            if (MODE == 4) { __stcs(reinterpret_cast<float4*>(out + p), x); continue; }
            if (MODE == 1) {
                *reinterpret_cast<float4*>(o) = x; *reinterpret_cast<float4*>(o + HW) = x;
                *reinterpret_cast<float4*>(o + 2 * HW) = x;
            } else {
                __stcs(reinterpret_cast<float4*>(o), x); __stcs(reinterpret_cast<float4*>(o + HW), x);
                __stcs(reinterpret_cast<float4*>(o + 2 * HW), x);
            }
        }
    }
    if (acc == 123.456f) sink[0] = acc;
}

// TMA bulk stores: each warp stages a row's three 512-B plane segments in shared memory and one
// lane issues three cp.async.bulk.global.shared::cta; two staging buffers per warp
__global__ void __launch_bounds__(128) k_bulk(const float* __restrict__ in, float* __restrict__ out, Geo g) {
    __shared__ __align__(128) float st[4][2][3][128];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const long long HW = (long long)g.H * g.W;
    const int sxn = (g.W + 127) / 128, syn = (g.H + STRIP - 1) / STRIP;
    int buf = 0;
    for (int it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items_of(g); it += nw) {
        const int sx = it % sxn, t = it / sxn, sy = t % syn, b = t / syn;
        const int c0w = sx * 128, c0 = c0w + lane * 4;
        const int ncol = min(128, g.W - c0w);
        const int y1 = min((sy + 1) * STRIP, g.H);
        for (int v = sy * STRIP; v < y1; ++v) {
            const long long p = (long long)b * HW + (long long)v * g.W + c0;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c0 < g.W) x = __ldg(reinterpret_cast<const float4*>(in + p));
            // the buffer written two rows ago must have been read by its bulk copy
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            float* s = &st[w][buf][0][0];
            *reinterpret_cast<float4*>(s + lane * 4) = x;
            *reinterpret_cast<float4*>(s + 128 + lane * 4) = x;
            *reinterpret_cast<float4*>(s + 256 + lane * 4) = x;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                float* o = out + (long long)b * 3 * HW + (long long)v * g.W + c0w;
                const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
                for (int c = 0; c < 3; ++c)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                 :: "l"(o + c * HW), "r"(sa + c * 512), "r"(ncol * 4) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            buf ^= 1;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA tensor loads (136-column x 4-row boxes, 4-slot ring per warp, as tfn_tma.cuh) + st.global.cs
__global__ void __launch_bounds__(128) k_tmald(const __grid_constant__ CUtensorMap tm, float* __restrict__ out, Geo g) {
    __shared__ __align__(128) float ring[4][4][4][136];
    __shared__ __align__(8) unsigned long long bar[4][4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const long long HW = (long long)g.H * g.W;
    const int sxn = (g.W + 127) / 128, syn = (g.H + STRIP - 1) / STRIP;
    const unsigned b0 = (unsigned)__cvta_generic_to_shared(&bar[w][0]);
    const unsigned r0 = (unsigned)__cvta_generic_to_shared(&ring[w][0][0][0]);
    if (lane == 0) {
        for (int k = 0; k < 4; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b0 + 8 * k));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned kq = 0;
    auto issue = [&](int k, int x, int y, int b) {
        const unsigned slot = (kq + k) & 3;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b0 + 8 * slot), "r"(4 * 136 * 4) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     :: "r"(r0 + slot * 4 * 136 * 4), "l"(&tm), "r"(x), "r"(y + 4 * k), "r"(b), "r"(b0 + 8 * slot) : "memory");
    };
    for (int it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items_of(g); it += nw) {
        const int sx = it % sxn, t = it / sxn, sy = t % syn, b = t / syn;
        const int c0 = sx * 128 + lane * 4;
        const int ya = sy * STRIP, y1 = min(ya + STRIP, g.H);
        const int nch = (y1 - ya + 3) / 4;
        __syncwarp();
        if (lane == 0) for (int k = 0; k < 4 && k < nch; ++k) issue(k, sx * 128 - 4, ya, b);
        for (int rr = 0; rr < y1 - ya; ++rr) {
            const int k = rr >> 2, rw = rr & 3;
            const unsigned slot = (kq + k) & 3;
            if (rw == 0) {
                if (k > 0 && k + 3 < nch) { __syncwarp(); if (lane == 0) issue(k + 3, sx * 128 - 4, ya, b); }
                unsigned done = 0;
                do {
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(done) : "r"(b0 + 8 * slot), "r"(((kq + k) >> 2) & 1u) : "memory");
                } while (!done);
            }
            const float4 x = *reinterpret_cast<const float4*>(&ring[w][slot][rw][4 + lane * 4]);
            if (c0 < g.W) {
                float* o = out + (long long)b * 3 * HW + (long long)(ya + rr) * g.W + c0;
                __stcs(reinterpret_cast<float4*>(o), x); __stcs(reinterpret_cast<float4*>(o + HW), x);
                __stcs(reinterpret_cast<float4*>(o + 2 * HW), x);
            }
        }
        kq += nch;
    }
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const Geo g{1024, 480, 640};
    const size_t px = (size_t)g.B * g.H * g.W;
    float *in, *out, *sink;
    CK(cudaMalloc(&in, px * 4)); CK(cudaMalloc(&out, px * 12)); CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(in, 0, px * 4));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap tm;
    const cuuint64_t dims[3] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.B};
    const cuuint64_t strides[2] = {(cuuint64_t)g.W * 4, (cuuint64_t)g.H * g.W * 4};
    const cuuint32_t box[3] = {136, 4, 1}, es[3] = {1, 1, 1};
    if (((EncodeTiled)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("{\"error\": \"tensor map\"}\n"); return 1;
    }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    printf("{\"what\": \"4 B read + 12 B write per px SOL (1024 x 480x640, fp32 planar), GB/s of algorithmic bytes, best of 10\"");
    for (int ctas = 3; ctas <= 8; ctas += 5) {
        auto time = [&](const char* name, double bpp, auto launch) {
            for (int i = 0; i < 3; ++i) launch();
            float best = 1e30f;
            for (int i = 0; i < 10; ++i) {
                cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
            }
            printf(", \"%s_ctas%d\": %.1f", name, ctas, bpp * px / (best * 1e-3) / 1e9);
        };
        const int grid = sms * ctas;
        time("stg_cs", 16, [&] { k_stg<0><<<grid, 128>>>(in, out, g, sink); });
        time("stg_wb", 16, [&] { k_stg<1><<<grid, 128>>>(in, out, g, sink); });
        time("bulk_store", 16, [&] { k_bulk<<<grid, 128>>>(in, out, g); });
        time("tma_load_stg_cs", 16, [&] { k_tmald<<<grid, 128>>>(tm, out, g); });
        time("write_only_12B", 12, [&] { k_stg<2><<<grid, 128>>>(in, out, g, sink); });
        time("read_only_4B", 4, [&] { k_stg<3><<<grid, 128>>>(in, out, g, sink); });
        time("copy_4B_4B", 8, [&] { k_stg<4><<<grid, 128>>>(in, out, g, sink); });
    }
    CK(cudaGetLastError());
    printf("}\n");
    return 0;
}
