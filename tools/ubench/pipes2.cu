// Pipe-throughput microbenchmark, part 2 (sm_100a): the XU / MIO / FP64 side of the 3F2N
// kernels — MUFU.RCP, MUFU.RSQ, MUFU.RCP64H, F2F.F32.F64, DFMA, DADD, SHFL — and mixes of
// them with the ALU min/max (do XU and ALU overlap?).  8 independent chains per thread,
// 16 warps/SM, one CTA per SM.  Prints warp-instructions of the listed ops per cycle per SM.
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 2048
__device__ __forceinline__ float rcpa(float x) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x) : "memory"); return r; }
__device__ __forceinline__ float rsqa(float x) { float r; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x) : "memory"); return r; }
__device__ __forceinline__ double rcp64(double x) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x) : "memory"); return r; }
__device__ __forceinline__ float f2f(double x) { float r; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(r) : "d"(x) : "memory"); return r; }
__device__ __forceinline__ float mn(float a, float b) { float r; asm volatile("min.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }

template <int OP>
__global__ void k(float* out, float s, long long* cyc) {
    float a[8]; double d[8];
    for (int i = 0; i < 8; ++i) { a[i] = 1.f + threadIdx.x * 1e-3f + i; d[i] = a[i]; }
    __syncthreads();
    long long t0; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");
#pragma unroll 2
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            // results feed back (dependency on the previous iteration only: 8-way ILP)
            if (OP == 0) a[i] = rcpa(__uint_as_float(__float_as_uint(a[i]) ^ 1u));        // MUFU.RCP (+LOP3: stops rcp(rcp(x)) folding)
            if (OP == 1) a[i] = rsqa(a[i]);                                             // MUFU.RSQ
            if (OP == 2) d[i] = rcp64(d[i]);                                            // MUFU.RCP64H (+ moves)
            if (OP == 3) { d[i] = d[i] * (double)s; a[(i + 1) & 7] += f2f(d[i]); }     // F2F.F32.F64 (+DMUL +FADD)
            if (OP == 4) d[i] = __fma_rn(d[i], (double)s, d[(i + 1) & 7]);              // DFMA
            if (OP == 5) d[i] = __dadd_rn(d[i], d[(i + 3) & 7]);                        // DADD
            if (OP == 6) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1) + 0.f;            // SHFL (+FADD)
            if (OP == 7) { a[i] = rcpa(__uint_as_float(__float_as_uint(a[i]) ^ 1u)); a[(i + 4) & 7] = mn(a[(i + 4) & 7], a[(i + 5) & 7]); }   // MUFU || FMNMX
            if (OP == 8) { a[i] = rcpa(__uint_as_float(__float_as_uint(a[i]) ^ 1u)); a[(i + 4) & 7] = mn(a[(i + 4) & 7], a[(i + 5) & 7]);
                           a[(i + 2) & 7] = mn(a[(i + 2) & 7], a[(i + 6) & 7]); a[(i + 3) & 7] = __fmaf_rn(a[(i + 3) & 7], s, 0.5f); }  // 1 MUFU : 2 FMNMX : 1 FFMA
            if (OP == 9) { a[i] = rcpa(__uint_as_float(__float_as_uint(a[i]) ^ 1u)); d[i] = d[i] * (double)s; a[(i + 4) & 7] += f2f(d[i]); }  // MUFU || F2F (+LOP3 DMUL FADD)
            if (OP == 10) { d[i] = __fma_rn(d[i], (double)s, d[(i + 1) & 7]); a[i] = mn(a[i], a[(i + 3) & 7]); }  // DFMA || FMNMX
        }
    }
    long long t1; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) :: "memory");
    float acc = 0;
    for (int i = 0; i < 8; ++i) acc += a[i] + (float)d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name, int per_it, float* out, long long* cyc, int blocks) {
    k<OP><<<blocks, 512>>>(out, 0.999f, cyc);
    k<OP><<<blocks, 512>>>(out, 0.999f, cyc);
    cudaDeviceSynchronize();
    long long h[1024]; cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double mean = 0; for (int i = 0; i < blocks; ++i) mean += h[i]; mean /= blocks;
    double wi = 16.0 * N_IT * 8 * per_it;      // counted warp-instructions per SM
    printf("%-34s %6.3f warp-instr/clk/SM  (%5.2f per SMSP; %5.1f clk per warp-instr per SMSP)\n", name, wi / mean,
           wi / mean / 4, 4 * mean / wi);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; long long* cyc;
    cudaMalloc(&out, sms * 512 * 4); cudaMalloc(&cyc, sms * 8);
    run<0>("MUFU.RCP", 1, out, cyc, sms);
    run<1>("MUFU.RSQ", 1, out, cyc, sms);
    run<2>("MUFU.RCP64H (counted 1/op)", 1, out, cyc, sms);
    run<3>("F2F.F32.F64 (counted 1/op)", 1, out, cyc, sms);
    run<4>("DFMA", 1, out, cyc, sms);
    run<5>("DADD", 1, out, cyc, sms);
    run<6>("SHFL (counted 1/op, +FADD)", 1, out, cyc, sms);
    run<7>("MUFU + FMNMX (counted 2/op)", 2, out, cyc, sms);
    run<8>("MUFU+2 FMNMX+FFMA (counted 4/op)", 4, out, cyc, sms);
    run<9>("MUFU + F2F (counted 2/op, +FADD)", 2, out, cyc, sms);
    run<10>("DFMA + FMNMX (counted 2/op)", 2, out, cyc, sms);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
