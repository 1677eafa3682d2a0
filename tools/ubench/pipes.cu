// Pipe-throughput microbenchmark (sm_100a): warp-instructions per cycle per SM for the
// arithmetic the 3F2N kernels use.  8 independent chains per thread, 16 warps/SM.
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 4096
template <int OP>
__global__ void k(float* out, float s, long long* cyc) {
    float a[8]; float2 b[8];
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i; b[i] = make_float2(a[i], a[i] + 1.f); }
    const float2 s2 = make_float2(s, s * 0.5f);
    unsigned u[8];
    for (int i = 0; i < 8; ++i) u[i] = __float_as_uint(a[i]);
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 4
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = __fmaf_rn(a[i], s, a[(i + 1) & 7]);            // FFMA 3-reg
            if (OP == 1) a[i] = __fmul_rn(a[i], a[(i + 3) & 7]);              // FMUL 2-reg
            if (OP == 2) a[i] = __fadd_rn(a[i], a[(i + 3) & 7]);              // FADD 2-reg
            if (OP == 3) b[i] = __ffma2_rn(b[i], s2, b[(i + 1) & 7]);         // FFMA2
            if (OP == 4) b[i] = __fadd2_rn(b[i], b[(i + 3) & 7]);             // FADD2
            if (OP == 5) a[i] = fminf(a[i], a[(i + 3) & 7]);                  // FMNMX
            if (OP == 6) a[i] = fminf(fminf(a[i], a[(i + 3) & 7]), a[(i + 5) & 7]);   // FMNMX3
            if (OP == 7) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[i])); a[i] = r; }   // MUFU
            if (OP == 8) u[i] = (u[i] ^ u[(i + 3) & 7]) + 0x9e3779b9u;        // LOP3+IADD (2 ALU)
            if (OP == 9) a[i] = __fmaf_rn(a[i], 1.0001f, 0.5f);              // FFMA imm
            if (OP == 10) b[i] = __fmul2_rn(b[i], b[(i + 3) & 7]);            // FMUL2
            if (OP == 11) { a[i] = __fmaf_rn(a[i], s, a[(i + 1) & 7]); u[i] = (u[i] ^ u[(i + 3) & 7]) + 1u; }  // FFMA || ALU mix
        }
    }
    long long t1 = clock64();
    float acc = 0;
    for (int i = 0; i < 8; ++i) acc += a[i] + b[i].x + b[i].y + __uint_as_float(u[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name, int per_it, float* out, long long* cyc, int blocks) {
    k<OP><<<blocks, 512>>>(out, 0.999f, cyc);
    k<OP><<<blocks, 512>>>(out, 0.999f, cyc);
    cudaDeviceSynchronize();
    long long h[1024]; cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double mean = 0; for (int i = 0; i < blocks; ++i) mean += h[i]; mean /= blocks;
    // warp-instructions of the op per SM per cycle (16 warps per block, 1 block per SM)
    double wi = 16.0 * N_IT * 8 * per_it;
    printf("%-28s %6.3f warp-instr/clk/SM  (%5.2f per SMSP)\n", name, wi / mean, wi / mean / 4);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; long long* cyc;
    cudaMalloc(&out, sms * 512 * 4); cudaMalloc(&cyc, sms * 8);
    run<0>("FFMA r,r,r", 1, out, cyc, sms);
    run<9>("FFMA r,imm,imm", 1, out, cyc, sms);
    run<1>("FMUL r,r", 1, out, cyc, sms);
    run<2>("FADD r,r", 1, out, cyc, sms);
    run<3>("FFMA2", 1, out, cyc, sms);
    run<10>("FMUL2", 1, out, cyc, sms);
    run<4>("FADD2", 1, out, cyc, sms);
    run<5>("FMNMX", 1, out, cyc, sms);
    run<6>("FMNMX3 (1 instr)", 1, out, cyc, sms);
    run<7>("MUFU.RCP", 1, out, cyc, sms);
    run<8>("LOP3+IADD (2 instr)", 2, out, cyc, sms);
    run<11>("FFMA + LOP3 + IADD (3 instr)", 3, out, cyc, sms);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
