/*
 * tfn_oracle.c — fp64 CPU ORACLE for the 3F2N per-pixel hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2005_08165_b200/csrc/) and
 * neither side includes the other.
 *
 * What it computes: the paper's equations, literally, step by step, in IEEE fp64
 * round-to-nearest, in the order and notation of PAPER.md §III:
 *
 *   Eq. 13  z [u v 1]^T = K p            -> back-projection of the 3x3
 *   P:197               "gradient filters ... on the inverse depth image (1/z)"
 *   Eq. 18  n_x = fx d(1/z)/du,  n_y = fy d(1/z)/dv,
 *                       n_z = -Phi{ (dx_j n_x + dy_j n_y) / dz_j },  j = 1..k
 *   P:218               Phi = mean or median; flat neighbourhood -> [0,0,-1]
 *   Eq. 19-21 disparity: z = f t_c / d, n_x = dd/du, n_y = dd/dv
 *
 * The closed form the GPU uses is deliberately NOT used
 * here: candidates are formed from explicitly back-projected neighbours.
 *
 * Readings of silent / ambiguous passages (SURVEY.md §8(c) ledger):
 *   Q1  kernels [p q p]^T (x) [-1 0 1]: FD (0,1), Sobel (1,2), Scharr (3,10),
 *       Prewitt (1,1); vertical = transpose; unnormalised.
 *   Q2  correlation orientation (g_u > 0 when x grows with u).
 *   Q3  1-px image border is invalid.
 *   Q4  output valid <=> interior, centre valid, every NONZERO-weight tap valid.
 *   Q5  a depth (disparity) is valid iff finite and >= FLT_MIN (2^-126): zero,
 *       negative, NaN, +-Inf and fp32-subnormal values are "no measurement".
 *   Q6  candidate j skipped iff its neighbour is invalid or z_j == z_c exactly.
 *   Q7  even-count median = mean of the two middle order statistics.
 *   Q8  mean divides by k, the number of candidates used.
 *   Q9  flat rule: g_u == 0 && g_v == 0  ->  [0,0,-1]  (covers k == 0).
 *   Q10 gradient taps grouped pairwise: g_u = sum_r k_r (x(v+r,u+1) - x(v+r,u-1)),
 *       summed r = -1, 0, +1 in that order (zero-weight terms omitted).
 *   Q11 orientation: flip iff <n,p> > 0; tie <n,p> == 0 -> flip iff n_z > 0.
 *   Q12 true per-pixel back-projection of every neighbour (Eq. 13).
 *   Q13 u = column, v = row, 0-based, pixel centres at integers.
 *   Q14 disparity requires fx == fy (checked by the caller); t_c*f enters only
 *       through z = f t_c / d.
 *
 * Parity pins for every function below live in tests/test_oracle_*.py (closed
 * forms, SPEC examples, invariants, brute-force PlaneSVD).  See DESIGN.md §4.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <float.h>

#define ORC_EXPORT __attribute__((visibility("default")))

typedef struct { double fx, fy, u0, v0; } orc_intrinsics;

/* ---- Q5: validity of one input sample --------------------------------------- */
ORC_EXPORT int orc_valid_sample(double z)
{
    return isfinite(z) && z >= (double)FLT_MIN;
}

/* ---- Eq. 13: back-projection  p = z K^{-1} [u v 1]^T -------------------------- */
ORC_EXPORT void orc_backproject(const orc_intrinsics* K, double u, double v, double z,
                                double p[3])
{
    p[0] = (u - K->u0) * z / K->fx;
    p[1] = (v - K->v0) * z / K->fy;
    p[2] = z;
}

/* ---- the point cloud of a depth image — Eq. 13 at every pixel,
 *      NaN for an invalid sample (Q5).  z: fp64 [B,H,W] depth; out: planar [B,3,H,W]. ---- */
ORC_EXPORT void orc_backproject_image(const orc_intrinsics* K, const double* z, int B, int H, int W,
                                      double* out)
{
    const size_t hw = (size_t)H * W;
    for (int b = 0; b < B; ++b)
        for (int v = 0; v < H; ++v)
            for (int u = 0; u < W; ++u) {
                const size_t i = (size_t)v * W + u;
                double* o = out + (size_t)b * 3 * hw + i;
                const double zz = z[(size_t)b * hw + i];
                if (!orc_valid_sample(zz)) { o[0] = o[hw] = o[2 * hw] = NAN; continue; }
                double p[3];
                orc_backproject(K, (double)u, (double)v, zz, p);
                o[0] = p[0]; o[hw] = p[1]; o[2 * hw] = p[2];
            }
}

/* ---- P:197 inverse depth; Eq. 19 disparity -> depth -------------------------- */
ORC_EXPORT double orc_inverse_depth(double z) { return 1.0 / z; }
ORC_EXPORT double orc_disparity_to_depth(double f_times_tc, double d) { return f_times_tc / d; }

/* ---- Q1: smoothing weights (k_{-1} = k_{+1} = kp, k_0 = k0) of the gradient
 *      kernels [kp k0 kp]^T (x) [-1 0 1] ------------------------------------------ */
ORC_EXPORT int orc_filter_weights(int filter, double* kp, double* k0)
{
    switch (filter) {
    case 0: *kp = 0.0; *k0 = 1.0;  return 0;   /* FD [-1,0,1]      */
    case 1: *kp = 1.0; *k0 = 2.0;  return 0;   /* Sobel                     */
    case 2: *kp = 3.0; *k0 = 10.0; return 0;   /* Scharr                    */
    case 3: *kp = 1.0; *k0 = 1.0;  return 0;   /* Prewitt                   */
    default: return -1;
    }
}

/* ---- Eq. 15 / P:197: horizontal and vertical gradient filters at (v,u) of the
 *      image x (inverse depth or disparity), correlation orientation (Q2),
 *      pairwise grouping, r = -1,0,+1 (Q10).  Zero-weight taps are not read.  ----- */
ORC_EXPORT void orc_gradient_at(const double* x, int H, int W, int v, int u,
                                double kp, double k0, double* gu, double* gv)
{
    (void)H;
    double w[3] = { kp, k0, kp };
    double su = 0.0, sv = 0.0;
    for (int r = -1; r <= 1; ++r) {
        double k = w[r + 1];
        if (k == 0.0) continue;
        su += k * (x[(size_t)(v + r) * W + (u + 1)] - x[(size_t)(v + r) * W + (u - 1)]);
    }
    for (int c = -1; c <= 1; ++c) {
        double k = w[c + 1];
        if (k == 0.0) continue;
        sv += k * (x[(size_t)(v + 1) * W + (u + c)] - x[(size_t)(v - 1) * W + (u + c)]);
    }
    *gu = su;
    *gv = sv;
}

/* ---- Eq. 17/18: one n_z candidate (dx n_x + dy n_y) / dz for r = q - p --------- */
ORC_EXPORT double orc_nz_candidate(const double p[3], const double q[3], double nx, double ny)
{
    double dx = q[0] - p[0];
    double dy = q[1] - p[1];
    double dz = q[2] - p[2];
    return (dx * nx + dy * ny) / dz;
}

/* ---- P:218 Phi: mean (Q8) and median (Q7) of k values (sorted in place) -------- */
ORC_EXPORT double orc_mean(const double* c, int k)
{
    double s = 0.0;
    for (int i = 0; i < k; ++i) s += c[i];
    return s / (double)k;
}

ORC_EXPORT double orc_median(double* c, int k)
{
    for (int i = 1; i < k; ++i) {            /* insertion sort, ascending */
        double t = c[i];
        int j = i - 1;
        while (j >= 0 && c[j] > t) { c[j + 1] = c[j]; --j; }
        c[j + 1] = t;
    }
    if (k & 1) return c[k / 2];
    return 0.5 * (c[k / 2 - 1] + c[k / 2]);
}

/* ---- Q11: normalise n and orient it toward the camera -------------- */
ORC_EXPORT void orc_orient_toward_camera(double n[3], const double p[3])
{
    double len = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    n[0] /= len; n[1] /= len; n[2] /= len;
    double s = n[0] * p[0] + n[1] * p[1] + n[2] * p[2];
    if (s > 0.0 || (s == 0.0 && n[2] > 0.0)) {
        n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2];
    }
}

/* ---- one frame ------------------------------------------------------------------
 * sample: [H,W] fp64 depth (is_disp = 0) or disparity (is_disp = 1).
 * f_tc  : f * t_c for the disparity path (Eq. 19); ignored for depth.
 * out   : [3,H,W] planar fp64; NaN triple for invalid pixels.
 * kp,k0 : smoothing weights (Q1); mode 0 = mean, 1 = median.
 * work  : scratch of 3*H*W doubles (x image, z image, validity as 0/1).
 * ------------------------------------------------------------------------------ */
static void estimate_frame(const double* sample, int H, int W, const orc_intrinsics* K,
                           int is_disp, double f_tc, double kp, double k0, int mode,
                           double* out, double* work)
{
    const size_t HW = (size_t)H * W;
    double* x = work;            /* inverse depth 1/z or disparity d (Eq. 21) */
    double* z = work + HW;       /* depth (Eq. 19 for disparity)                      */
    double* ok = work + 2 * HW;  /* Q5 validity                                        */
    for (size_t i = 0; i < HW; ++i) {
        double s = sample[i];
        ok[i] = orc_valid_sample(s) ? 1.0 : 0.0;
        if (ok[i] != 0.0) {
            if (is_disp) { x[i] = s; z[i] = orc_disparity_to_depth(f_tc, s); }
            else         { x[i] = orc_inverse_depth(s); z[i] = s; }
        } else {
            x[i] = NAN; z[i] = NAN;
        }
    }
    const double NaN = NAN;
    const double wt[3] = { kp, k0, kp };
    for (int v = 0; v < H; ++v) {
        for (int u = 0; u < W; ++u) {
            size_t i = (size_t)v * W + u;
            double* o0 = out + i;
            double* o1 = out + HW + i;
            double* o2 = out + 2 * HW + i;
            *o0 = NaN; *o1 = NaN; *o2 = NaN;
            /* Q3: border invalid */
            if (u < 1 || v < 1 || u > W - 2 || v > H - 2) continue;
            if (ok[i] == 0.0) continue;
            /* Q4: every nonzero-weight tap of both gradient kernels valid */
            int taps_ok = 1;
            for (int r = -1; r <= 1; ++r) {
                if (wt[r + 1] == 0.0) continue;
                if (ok[(size_t)(v + r) * W + u + 1] == 0.0 || ok[(size_t)(v + r) * W + u - 1] == 0.0) taps_ok = 0;
                if (ok[(size_t)(v + 1) * W + u + r] == 0.0 || ok[(size_t)(v - 1) * W + u + r] == 0.0) taps_ok = 0;
            }
            if (!taps_ok) continue;

            /* Eq. 15-16 / Eq. 21: gradients of 1/z (or d) */
            double gu, gv;
            orc_gradient_at(x, H, W, v, u, kp, k0, &gu, &gv);

            /* Q9 / P:218 flat rule */
            if (gu == 0.0 && gv == 0.0) { *o0 = 0.0; *o1 = 0.0; *o2 = -1.0; continue; }

            /* Eq. 18 first line (depth) / Eq. 21 first line (disparity) */
            double nx = is_disp ? gu : K->fx * gu;
            double ny = is_disp ? gv : K->fy * gv;

            /* Eq. 13: back-project centre and neighbours; Eq. 17-18 candidates */
            double p[3];
            orc_backproject(K, (double)u, (double)v, z[i], p);
            double cand[8];
            int k = 0;
            for (int dv = -1; dv <= 1; ++dv) {
                for (int du = -1; du <= 1; ++du) {
                    if (du == 0 && dv == 0) continue;
                    size_t j = (size_t)(v + dv) * W + (u + du);
                    if (ok[j] == 0.0) continue;             /* Q6 invalid neighbour */
                    if (z[j] == z[i]) continue;             /* Q6 dz == 0           */
                    double q[3];
                    orc_backproject(K, (double)(u + du), (double)(v + dv), z[j], q);
                    cand[k++] = orc_nz_candidate(p, q, nx, ny);
                }
            }
            if (k == 0) { *o0 = 0.0; *o1 = 0.0; *o2 = -1.0; continue; }   /* Q9 */

            /* P:218 / Eq. 18 second line: n_z = -Phi{candidates} */
            double phi = (mode == 0) ? orc_mean(cand, k) : orc_median(cand, k);
            double n[3] = { nx, ny, -phi };

            /* normalise + orient toward the camera (Q11) */
            orc_orient_toward_camera(n, p);
            *o0 = n[0]; *o1 = n[1]; *o2 = n[2];
        }
    }
}

/* ---- public entry points ------------------------------------------------------- */

/* depth (fp64 samples), generic smoothing weights; out [B,3,H,W] fp64 */
ORC_EXPORT int orc_estimate_depth_f64(const double* depth, int B, int H, int W,
                                      const orc_intrinsics* K, double kp, double k0, int mode,
                                      double* out, double* work)
{
    if (B < 0 || H <= 0 || W <= 0) return 1;
    size_t HW = (size_t)H * W;
    for (int b = 0; b < B; ++b)
        estimate_frame(depth + b * HW, H, W, K, 0, 0.0, kp, k0, mode, out + 3 * b * HW, work);
    return 0;
}

ORC_EXPORT int orc_estimate_disparity_f64(const double* disp, double f_tc, int B, int H, int W,
                                          const orc_intrinsics* K, double kp, double k0, int mode,
                                          double* out, double* work)
{
    if (B < 0 || H <= 0 || W <= 0) return 1;
    if (K->fx != K->fy) return 2;                  /* Q14 / Eq. 19 single focal length */
    size_t HW = (size_t)H * W;
    for (int b = 0; b < B; ++b)
        estimate_frame(disp + b * HW, H, W, K, 1, f_tc, kp, k0, mode, out + 3 * b * HW, work);
    return 0;
}

/* fp32 input (the same buffer the GPU reads), upcast exactly to fp64 per frame.
 * work must hold 4*H*W doubles. */
ORC_EXPORT int orc_estimate_f32(const float* sample, int is_disp, double f_tc, int B, int H, int W,
                                const orc_intrinsics* K, double kp, double k0, int mode,
                                double* out, double* work)
{
    if (B < 0 || H <= 0 || W <= 0) return 1;
    if (is_disp && K->fx != K->fy) return 2;
    size_t HW = (size_t)H * W;
    double* up = work + 3 * HW;
    for (int b = 0; b < B; ++b) {
        for (size_t i = 0; i < HW; ++i) up[i] = (double)sample[b * HW + i];
        estimate_frame(up, H, W, K, is_disp, f_tc, kp, k0, mode, out + 3 * b * HW, work);
    }
    return 0;
}

/* One output pixel only (for sampled parity at full sizes): reads the 3x3
 * neighbourhood of (v,u) from an fp32 frame, writes n[3] (NaN if invalid). */
ORC_EXPORT int orc_estimate_pixel_f32(const float* frame, int is_disp, double f_tc, int H, int W,
                                      const orc_intrinsics* K, double kp, double k0, int mode,
                                      int v, int u, double n_out[3])
{
    /* copy the 5x5 window (zero = invalid outside the image) into a tiny frame and
     * run the same per-frame routine on it; the centre of a 5x5 is interior and
     * its 3x3 neighbourhood is exact. */
    double win[25], work[75], out[75];
    if (u < 0 || v < 0 || u >= W || v >= H) return 1;
    if (is_disp && K->fx != K->fy) return 2;
    orc_intrinsics Kw = *K;
    Kw.u0 = K->u0 - (double)(u - 2);
    Kw.v0 = K->v0 - (double)(v - 2);
    for (int dv = -2; dv <= 2; ++dv)
        for (int du = -2; du <= 2; ++du) {
            int vv = v + dv, uu = u + du;
            win[(dv + 2) * 5 + (du + 2)] =
                (vv >= 0 && vv < H && uu >= 0 && uu < W) ? (double)frame[(size_t)vv * W + uu] : 0.0;
        }
    estimate_frame(win, 5, 5, &Kw, is_disp, f_tc, kp, k0, mode, out, work);
    int border = (u < 1 || v < 1 || u > W - 2 || v > H - 2);
    for (int c = 0; c < 3; ++c) n_out[c] = border ? NAN : out[c * 25 + 12];
    return 0;
}

/* ================================================================================
 * the comparison estimators PlaneSVD (Eq. 2) and
 * PlanePCA (Eq. 3), as SPEC S:251-258 specifies them: per pixel, the centre
 * point and its valid 8-neighbours Q_i^+ (k >= 3 neighbours, else invalid; 1-px border
 * invalid), back-projected with Eq. 13; PlaneSVD = the smallest-eigenvalue eigenvector of
 * the 4x4 normal matrix [Q+ 1]^T [Q+ 1], n = its first three components; PlanePCA = the
 * smallest-eigenvalue eigenvector of the 3x3 scatter matrix of Q+ about its mean; then
 * normalised and oriented toward the camera (Q11).
 * ================================================================================ */

/* cyclic Jacobi on a symmetric d x d matrix (d = 3 or 4), sweeps until the
 * off-diagonal Frobenius norm is below 1e-12 x the matrix's Frobenius norm (reading: the
 * SPEC's 1e-12 taken relative, so the test does not depend on the depth unit), at most 50
 * sweeps; returns the unit eigenvector of the smallest eigenvalue, ties broken toward the
 * candidate whose first nonzero component has the largest magnitude (lowest index among
 * equals), made positive.  Returns 1 if M is not symmetric within 1e-9 (relative). */
ORC_EXPORT int orc_smallest_eigvec_sym(const double* M, int d, double* out)
{
    double a[16], v[16];
    double fro = 0.0;
    for (int i = 0; i < d * d; ++i) fro += M[i] * M[i];
    fro = sqrt(fro);
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
            if (fabs(M[i * d + j] - M[j * d + i]) > 1e-9 * (fro > 0 ? fro : 1.0)) return 1;
    for (int i = 0; i < d * d; ++i) { a[i] = M[i]; v[i] = (i / d == i % d) ? 1.0 : 0.0; }
    for (int sweep = 0; sweep < 50; ++sweep) {
        double off = 0.0;
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j)
                if (i != j) off += a[i * d + j] * a[i * d + j];
        if (sqrt(off) <= 1e-12 * fro) break;
        for (int p = 0; p < d - 1; ++p)
            for (int q = p + 1; q < d; ++q) {
                const double apq = a[p * d + q];
                if (apq == 0.0) continue;
                /* Golub & Van Loan, symmetric Schur: zero a_pq */
                const double theta = (a[q * d + q] - a[p * d + p]) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                for (int k = 0; k < d; ++k) {          /* A <- J^T A J */
                    const double akp = a[k * d + p], akq = a[k * d + q];
                    a[k * d + p] = c * akp - s * akq;
                    a[k * d + q] = s * akp + c * akq;
                }
                for (int k = 0; k < d; ++k) {
                    const double apk = a[p * d + k], aqk = a[q * d + k];
                    a[p * d + k] = c * apk - s * aqk;
                    a[q * d + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < d; ++k) {          /* V <- V J */
                    const double vkp = v[k * d + p], vkq = v[k * d + q];
                    v[k * d + p] = c * vkp - s * vkq;
                    v[k * d + q] = s * vkp + c * vkq;
                }
            }
    }
    double lmin = a[0];
    for (int i = 1; i < d; ++i) if (a[i * d + i] < lmin) lmin = a[i * d + i];
    const double tie = 1e-12 * (fro > 0 ? fro : 1.0);
    int best = -1;
    double best_mag = -1.0;
    for (int j = 0; j < d; ++j) {
        if (a[j * d + j] - lmin > tie) continue;
        double first = 0.0;
        for (int k = 0; k < d; ++k) if (v[k * d + j] != 0.0) { first = v[k * d + j]; break; }
        if (fabs(first) > best_mag) { best_mag = fabs(first); best = j; }
    }
    double first = 0.0;
    for (int k = 0; k < d; ++k) if (v[k * d + best] != 0.0) { first = v[k * d + best]; break; }
    const double sg = first < 0 ? -1.0 : 1.0;
    for (int k = 0; k < d; ++k) out[k] = sg * v[k * d + best];
    return 0;
}

/* method 0 = PlanePCA (Eq. 3), 1 = PlaneSVD (Eq. 2).  depth fp64 [B,H,W]; out planar
 * [B,3,H,W] fp64, NaN triple where invalid. */
ORC_EXPORT int orc_plane_fit(const double* depth, int B, int H, int W, const orc_intrinsics* K, int method,
                             double* out)
{
    if (method != 0 && method != 1) return 1;
    const size_t hw = (size_t)H * W;
    for (int b = 0; b < B; ++b) {
        const double* z = depth + (size_t)b * hw;
        for (int v = 0; v < H; ++v)
            for (int u = 0; u < W; ++u) {
                double* o = out + (size_t)b * 3 * hw + (size_t)v * W + u;
                o[0] = o[hw] = o[2 * hw] = NAN;
                if (u < 1 || v < 1 || u > W - 2 || v > H - 2) continue;      /* border */
                const double zc = z[(size_t)v * W + u];
                if (!orc_valid_sample(zc)) continue;
                double q[9][3];
                int n = 0, k = 0;
                for (int dv = -1; dv <= 1; ++dv)
                    for (int du = -1; du <= 1; ++du) {
                        const double zz = z[(size_t)(v + dv) * W + (u + du)];
                        if (!orc_valid_sample(zz)) continue;
                        orc_backproject(K, (double)(u + du), (double)(v + dv), zz, q[n]);
                        ++n;
                        if (du != 0 || dv != 0) ++k;
                    }
                if (k < 3) continue;
                double nrm[4], M[16];
                if (method == 0) {
                    double mean[3] = {0, 0, 0};
                    for (int i = 0; i < n; ++i) for (int c = 0; c < 3; ++c) mean[c] += q[i][c];
                    for (int c = 0; c < 3; ++c) mean[c] /= n;
                    for (int r = 0; r < 3; ++r)
                        for (int c = 0; c < 3; ++c) {
                            double s = 0.0;
                            for (int i = 0; i < n; ++i) s += (q[i][r] - mean[r]) * (q[i][c] - mean[c]);
                            M[r * 3 + c] = s;
                        }
                    if (orc_smallest_eigvec_sym(M, 3, nrm)) continue;
                } else {
                    for (int r = 0; r < 4; ++r)
                        for (int c = 0; c < 4; ++c) {
                            double s = 0.0;
                            for (int i = 0; i < n; ++i) s += (r < 3 ? q[i][r] : 1.0) * (c < 3 ? q[i][c] : 1.0);
                            M[r * 4 + c] = s;
                        }
                    if (orc_smallest_eigvec_sym(M, 4, nrm)) continue;
                }
                double nn[3] = {nrm[0], nrm[1], nrm[2]};
                double p[3];
                orc_backproject(K, (double)u, (double)v, zc, p);
                orc_orient_toward_camera(nn, p);
                o[0] = nn[0]; o[hw] = nn[1]; o[2 * hw] = nn[2];
            }
    }
    return 0;
}
