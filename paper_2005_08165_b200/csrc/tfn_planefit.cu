// tfn_planefit.cu — SURVEY §8(f) N4: the paper's accuracy yardsticks PlanePCA (PAPER.md
// Eq. 3) and PlaneSVD (Eq. 2) as a GPU comparator, following SPEC
// S:251-258 (3x3 window, k >= 3 valid neighbours, 1-px border invalid, camera-facing).
//
// One thread per pixel, everything in fp64 (the B200's fp64 pipe): back-project the valid
// samples of the 3x3 window (Eq. 13), form the 3x3 scatter matrix about the mean (PCA) or
// the 4x4 normal matrix of [Q+ 1] (SVD), and take the smallest-eigenvalue eigenvector by
// cyclic Jacobi (Golub & Van Loan's symmetric Schur rotations; stop when the off-diagonal
// norm is below 1e-12 of the matrix norm, <= 50 sweeps) — the same algorithm as the
// oracle's orc_smallest_eigvec_sym, written independently here.  An ALU / fp64-bound
// workload (no tensor-core shape: 9 points per pixel), unlike the HBM-shaped 3F2N path.
#include <cuda_runtime.h>

#include "tfn_device.cuh"
#include "tfn_kernels.h"

namespace tfn {

template <int D>
__device__ __forceinline__ void jacobi_smallest(double a[D][D], double out[D]) {
    double v[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) v[i][j] = (i == j) ? 1.0 : 0.0;
    double fro = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) fro += a[i][j] * a[i][j];
    fro = sqrt(fro);
    for (int sweep = 0; sweep < 50; ++sweep) {
        double off = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j)
                if (i != j) off += a[i][j] * a[i][j];
        if (sqrt(off) <= 1e-12 * fro) break;
#pragma unroll
        for (int p = 0; p < D - 1; ++p)
#pragma unroll
            for (int q = p + 1; q < D; ++q) {
                const double apq = a[p][q];
                if (apq == 0.0) continue;
                const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                const double c = rsqrt(1.0 + t * t), s = t * c;
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const double akp = a[k][p], akq = a[k][q];
                    a[k][p] = c * akp - s * akq;
                    a[k][q] = s * akp + c * akq;
                }
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = c * apk - s * aqk;
                    a[q][k] = s * apk + c * aqk;
                }
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const double vkp = v[k][p], vkq = v[k][q];
                    v[k][p] = c * vkp - s * vkq;
                    v[k][q] = s * vkp + c * vkq;
                }
            }
    }
    double lmin = a[0][0];
#pragma unroll
    for (int i = 1; i < D; ++i) lmin = fmin(lmin, a[i][i]);
    const double tie = 1e-12 * (fro > 0 ? fro : 1.0);
    int best = 0;
    double best_mag = -1.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        double first = 0.0;
#pragma unroll
        for (int k = D - 1; k >= 0; --k) if (v[k][j] != 0.0) first = v[k][j];
        if (a[j][j] - lmin <= tie && fabs(first) > best_mag) { best_mag = fabs(first); best = j; }
    }
    double first = 0.0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) if (v[k][best] != 0.0) first = v[k][best];
    const double sg = first < 0 ? -1.0 : 1.0;
#pragma unroll
    for (int k = 0; k < D; ++k) out[k] = sg * v[k][best];
}

template <int METHOD>      // 0 = PlanePCA, 1 = PlaneSVD
__global__ void __launch_bounds__(256) tfn_planefit_kernel(const float* __restrict__ depth, float* __restrict__ out,
                                                           int H, int W, double fx, double fy, double u0,
                                                           double v0, int layout) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y * blockDim.y + threadIdx.y;
    const long long b = blockIdx.z;
    if (u >= W || v >= H) return;
    const long long HW = (long long)H * W;
    const float* z = depth + b * HW;
    double n[3] = {NAN, NAN, NAN};
    const double zc = (u >= 1 && v >= 1 && u <= W - 2 && v <= H - 2) ? (double)sanitize(__ldg(z + (long long)v * W + u))
                                                                       : (double)NAN;
    if (!isnan(zc)) {
        // all 9 window points with a 0/1 weight instead of a compacted list (no dynamic
        // indexing, no local memory); an invalid point is (0,0,0) with weight 0, and adding
        // exact zeros leaves every sum bit-identical to skipping it
        double q[9][3], wgt[9];
        int k = 0;
#pragma unroll
        for (int dv = -1; dv <= 1; ++dv)
#pragma unroll
            for (int du = -1; du <= 1; ++du) {
                const int i = (dv + 1) * 3 + (du + 1);
                const double zz = (double)sanitize(__ldg(z + (long long)(v + dv) * W + (u + du)));
                const bool ok = !isnan(zz);
                wgt[i] = ok ? 1.0 : 0.0;
                q[i][0] = ok ? ((double)(u + du) - u0) * zz / fx : 0.0;       // Eq. 13
                q[i][1] = ok ? ((double)(v + dv) - v0) * zz / fy : 0.0;
                q[i][2] = ok ? zz : 0.0;
                if (ok && (du != 0 || dv != 0)) ++k;
            }
        const double cnt = (double)(k + 1);
        if (k >= 3) {
            double e[4];
            if (METHOD == 0) {
                double m[3] = {0, 0, 0};
#pragma unroll
                for (int i = 0; i < 9; ++i)
#pragma unroll
                    for (int c = 0; c < 3; ++c) m[c] += q[i][c];
#pragma unroll
                for (int c = 0; c < 3; ++c) m[c] /= cnt;
                double a[3][3];
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        double s = 0.0;
#pragma unroll
                        for (int i = 0; i < 9; ++i) s += wgt[i] * ((q[i][r] - m[r]) * (q[i][c] - m[c]));
                        a[r][c] = s;
                    }
                jacobi_smallest<3>(a, e);
            } else {
                double a[4][4];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        double s = 0.0;
#pragma unroll
                        for (int i = 0; i < 9; ++i) s += (r < 3 ? q[i][r] : wgt[i]) * (c < 3 ? q[i][c] : wgt[i]);
                        a[r][c] = s;
                    }
                jacobi_smallest<4>(a, e);
            }
            // normalise, orient toward the camera (Q11): flip iff <n,p> > 0, tie -> n_z > 0
            const double len = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
            n[0] = e[0] / len; n[1] = e[1] / len; n[2] = e[2] / len;
            const double px = ((double)u - u0) * zc / fx, py = ((double)v - v0) * zc / fy;
            const double sdot = n[0] * px + n[1] * py + n[2] * zc;
            if (sdot > 0.0 || (sdot == 0.0 && n[2] > 0.0)) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; }
        }
    }
    const long long pix = (long long)v * W + u;
    if (layout == 0) {
        float* o = out + b * 3 * HW + pix;
        o[0] = (float)n[0]; o[HW] = (float)n[1]; o[2 * HW] = (float)n[2];
    } else {
        float* o = out + (b * HW + pix) * 3;
        o[0] = (float)n[0]; o[1] = (float)n[1]; o[2] = (float)n[2];
    }
}

cudaError_t launch_planefit(const float* depth, float* out, long long B, int H, int W, double fx, double fy,
                            double u0, double v0, int layout, int method, cudaStream_t st) {
    const long long HW = (long long)H * W;
    for (long long b0 = 0; b0 < B; b0 += 65535) {          // frames on grid z, <= 65535 per launch
        const long long n = (B - b0 < 65535) ? B - b0 : 65535;
        dim3 blk(32, 8, 1);
        dim3 grd((W + 31) / 32, (H + 7) / 8, (unsigned)n);
        if (method == 0) tfn_planefit_kernel<0><<<grd, blk, 0, st>>>(depth + b0 * HW, out + b0 * 3 * HW, H, W, fx, fy, u0, v0, layout);
        else tfn_planefit_kernel<1><<<grd, blk, 0, st>>>(depth + b0 * HW, out + b0 * 3 * HW, H, W, fx, fy, u0, v0, layout);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace tfn
