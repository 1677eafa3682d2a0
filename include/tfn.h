/*
 * tfn.h — C ABI of the B200-native 3F2N ("three-filters-to-normal") surface-normal
 * estimator: libtfn.so (paper_2005_08165_b200/libtfn.so), sm_100a only.
 *
 * The operation (§III): for every
 * pixel (u = column, v = row, 0-based) of a batch of depth images Z (or disparity
 * images d), with pinhole intrinsics K = (fx, fy, u0, v0) (Eq. 13):
 *   1. g_u, g_v = horizontal / vertical gradient filter (FD, Sobel, Scharr or
 *      Prewitt) of the inverse depth 1/Z (disparity: of d, Eq. 21);
 *   2. n_x = fx g_u, n_y = fy g_v  (Eq. 18; disparity Eq. 21: n_x = g_u, n_y = g_v);
 *   3. n_z = -Phi_j{ (dX_j n_x + dY_j n_y) / dZ_j } over the 8-neighbourhood, the
 *      neighbours back-projected with K (Eq. 13, 17, 18), Phi = mean or median
 *      (P:218), skipping invalid neighbours and dZ_j == 0;
 *   4. flat rule: g_u == g_v == 0 -> n = [0,0,-1];
 *   5. n normalised and oriented toward the camera (<n, p> <= 0).
 * The readings of everything the paper leaves open (validity, border, even-count
 * median, orientation tie, ...) are DESIGN.md §3 (Q1-Q19); they are identical to
 * the fp64 oracle's (oracle/tfn_oracle.c).
 *
 * Data layout.  Inputs are contiguous fp32 [batch, H, W] row-major (or, for
 * tfn_estimate_u16, uint16 depth codes: Z = code x depth_scale, code 0 = no
 * measurement — SURVEY §8(f) N1).  A fp32 sample is VALID iff it is finite and
 * >= FLT_MIN (zero, negative, NaN, Inf and fp32 subnormals mean "no measurement").
 * Outputs are unit normals, fp32 (default) or IEEE half (TFN_OPT_OUT_DTYPE =
 * TFN_OUT_F16: each component the fp32 result rounded to nearest; NaN stays NaN):
 *   TFN_LAYOUT_PLANAR  [batch, 3, H, W]  (n_x plane, n_y plane, n_z plane)
 *   TFN_LAYOUT_PACKED  [batch, H, W, 3]
 * or octahedral int16 pairs (TFN_OUT_OCT16, 4 B/pixel; [batch,2,H,W] planar / [batch,H,W,2]
 * packed): (u, v) = round(32767 * octahedral map of (n_x, n_y, -n_z)) — p = v/|v|_1, the
 * far hemisphere (n_z > 0) folded as (1-|p_y|, 1-|p_x|) with the signs of p — so
 * camera-facing normals sit in the inner diamond; decode p = q/32767, v = (p_x, p_y,
 * 1-|p_x|-|p_y|), unfold if negative, normalise, n = (v_x, v_y, -v_z).  Direction error
 * <= 0.005 deg.  Invalid pixels: (-32768, -32768).
 * An output pixel is VALID iff it is not on the 1-pixel image border, its centre
 * sample is valid and every tap with a nonzero weight in either gradient kernel is
 * valid (FD: the 4 edge neighbours; Sobel/Scharr/Prewitt: all 8).  Invalid output
 * pixels are written as (NaN, NaN, NaN) — invalid pixels are data, not errors.
 *
 * Ownership.  The caller owns every buffer.  Device pointers must be cudaMalloc'd
 * (or torch) memory on the current device; inputs and outputs must not overlap.
 * With W % 4 == 0 and buffers aligned to 4 elements (16 B fp32, 8 B uint16 / half)
 * the strip kernel runs (the fast path); anything else (element-aligned) takes the
 * per-pixel kernel, same results.
 * A handle holds only its parameters (plus, for tfn_estimate_host, a lazily
 * allocated device workspace guarded by a mutex); set options before the first
 * estimate.  Device calls are asynchronous on `stream` (a cudaStream_t passed as
 * void*; NULL = legacy default stream); kernel faults surface at the caller's
 * next synchronisation.  batch == 0 is a no-op returning TFN_OK.  H or W < 3 is
 * valid and yields an all-invalid (NaN) output.
 *
 * Errors: every entry point returns a tfn_status; nothing is thrown or printed.
 */
#ifndef TFN_H
#define TFN_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TFN_OK = 0,
    TFN_ERR_INVALID_ARGUMENT = 1, /* null pointer, batch < 0, H or W <= 0, overflow, overlap, bad enum */
    TFN_ERR_CONFIG = 2,           /* fx, fy not finite or <= 0; disparity with fx != fy or bad baseline*f */
    TFN_ERR_CUDA = 3              /* CUDA launch/runtime error, or the device is not sm_100 */
} tfn_status;

typedef enum {
    TFN_FILTER_FD = 0, TFN_FILTER_SOBEL = 1, TFN_FILTER_SCHARR = 2, TFN_FILTER_PREWITT = 3,
    TFN_FILTER_CUSTOM = 4   /* [kp k0 kp]^T (x) [-1 0 1] with run-time weights (tfn_set_filter_weights) */
} tfn_filter;
typedef enum { TFN_NZ_MEAN = 0, TFN_NZ_MEDIAN = 1 } tfn_nz_mode;
typedef enum { TFN_LAYOUT_PLANAR = 0, TFN_LAYOUT_PACKED = 1 } tfn_layout;
typedef enum { TFN_OUT_F32 = 0, TFN_OUT_F16 = 1, TFN_OUT_OCT16 = 2 } tfn_out_dtype;

/* Options for tfn_set_option (tuning / testing; defaults are the production path) */
typedef enum {
    TFN_OPT_KERNEL = 0,     /* 0 auto, 1 per-pixel kernel, 2 strip kernel (needs W%4==0, 16-B alignment),  */
                            /* 3 general strip kernel (same results; no special path: for holes / quantized), */
                            /* 4 masked strip kernel (same results; special path only for pixels whose taps  */
                            /*   are all valid: for depth with holes / dropout)                               */
                            /* 5 fp32 unit-step kernel (round 2 production path: within the  */
                            /*   parity tolerance of the others, not bit-identical), 6 its masked variant    */
    TFN_OPT_STRIP_H = 1,    /* rows per warp strip, 0 = auto (>= 4)                                        */
    TFN_OPT_GRID = 2,       /* CTAs of the strip kernel, 0 = auto (resident CTAs x SMs)                    */
    TFN_OPT_DYNAMIC = 3,    /* 1 (default): strips claimed from a per-call work counter; 0: static stride  */
    TFN_OPT_OUT_DTYPE = 4,  /* tfn_out_dtype of the normals every estimate call writes (default F32)        */
    TFN_OPT_COUNT_SPECIAL = 5  /* 1: the fp32 kernel counts the pixels it sends to the exact path            */
                               /*    (read back with tfn_debug_special_count); 0 (default): not counted     */
} tfn_option;

/* Pinhole intrinsics in pixels (Eq. 13): u = column, v = row, 0-based, pixel
 * centres at integer coordinates. */
typedef struct { double fx, fy, u0, v0; } tfn_intrinsics;

typedef struct tfn_ctx* tfn_handle;

/* Create an estimator for intrinsics K, gradient kernel `filter` (tfn_filter) and
 * n_z filter `nz_mode` (tfn_nz_mode).  Checks that the current device is sm_100.
 * Errors: K or out NULL, bad enum -> INVALID_ARGUMENT; fx/fy/u0/v0 non-finite or
 * fx, fy <= 0 -> CONFIG; no CUDA device / not sm_100 -> CUDA. */
int tfn_create(const tfn_intrinsics* K, int filter, int nz_mode, tfn_handle* out);

/* Weights of a TFN_FILTER_CUSTOM handle: the smoothing column [kp k0 kp] of the gradient
 * kernels [kp k0 kp]^T (x) [-1 0 1] (horizontal; vertical = transpose) — the paper's 3x3
 * kernel search space.  kp > 0 and k0 > 0, finite (CONFIG
 * otherwise; kp = 0 is TFN_FILTER_FD).  Only the ratio matters for the direction; the
 * gradient is summed in the oracle's order ((kp D- + k0 D0) + kp D+), so (1,2), (3,10)
 * and (1,1) reproduce Sobel, Scharr and Prewitt bit for bit.  Default (1, 2).
 * INVALID_ARGUMENT if h is NULL or not a CUSTOM handle. */
int tfn_set_filter_weights(tfn_handle h, double kp, double k0);

/* Output layout (tfn_layout); default PLANAR. */
int tfn_set_layout(tfn_handle h, int layout);

/* Tuning/testing option (tfn_option). */
int tfn_set_option(tfn_handle h, int option, long long value);

/* 3F2N from depth (Eq. 13-18).  depth: device fp32 [batch,H,W] in metres
 * (any positive unit); out_normals: device, 3*batch*H*W components of the handle's
 * output dtype (fp32 or half) in the handle's layout.  Asynchronous on stream. */
int tfn_estimate(tfn_handle h, const float* depth, int batch, int H, int W,
                 void* stream, void* out_normals);

/* 3F2N from integer depth codes (e.g. millimetre depth from RGB-D
 * sensors): depth_codes device uint16 [batch,H,W], Z = code * depth_scale, code 0 =
 * no measurement.  depth_scale > 0 and finite (CONFIG otherwise); it cancels from the
 * normal direction (Appendix A.4) and is only validated.  Same output as
 * tfn_estimate on the fp32 depths code * depth_scale up to rounding (<= 1e-3 deg; the
 * oracle parity bar), bit-identical to tfn_estimate on the fp32 values (float)code.
 * Quantized depth makes dZ == 0 common, so the general strip variant runs. */
int tfn_estimate_u16(tfn_handle h, const unsigned short* depth_codes, double depth_scale, int batch, int H,
                     int W, void* stream, void* out_normals);

/* 3F2N from disparity (Eq. 19-21): z = f t_c / d.  Requires fx == fy
 * (CONFIG otherwise).  baseline_times_f = f * t_c > 0 and finite (CONFIG otherwise);
 * it cancels from the normal direction and is only validated. */
int tfn_estimate_disparity(tfn_handle h, const float* disparity, double baseline_times_f,
                           int batch, int H, int W, void* stream, void* out_normals);

/* End-to-end from HOST memory: copies host_in (fp32 [batch,H,W], depth or
 * disparity) to the device in chunks, runs the same kernel, copies the normals back
 * to host_out (3*batch*H*W components of the output dtype), overlapping H2D / kernel /
 * D2H on two internal streams.  Pinned host memory gives full overlap.  Blocking:
 * returns when host_out is complete (or on the first error).  `stream` orders the
 * work after prior work on that stream. */
int tfn_estimate_host(tfn_handle h, const float* host_in, int is_disparity, double baseline_times_f,
                      int batch, int H, int W, void* host_out, void* stream);

/* normals AND the point cloud in one pass (the downstream consumers:
 * registration / SLAM).  input_kind (tfn_input_kind): fp32 depth
 * (Z = scale * sample), fp32 disparity (Z = scale / d, scale = f * t_c, needs fx == fy),
 * or uint16 depth codes (Z = scale * code).  scale > 0 and finite (CONFIG otherwise).
 * out_normals as for tfn_estimate (same bits); out_points: device fp32, 3*batch*H*W
 * floats in the handle's layout, p = Z (  (u-u0)/fx, (v-v0)/fy, 1 ) (Eq. 13), each
 * coordinate rounded as fl(fl(a * Z) * fl(1/fx)) (<= 3 ulp of the fp64 value); NaN where
 * the sample is invalid (the point needs no neighbours: border pixels get points).
 * out_points must not overlap the other buffers; 16-B aligned for the strip kernel. */
typedef enum { TFN_INPUT_DEPTH_F32 = 0, TFN_INPUT_DISPARITY_F32 = 1, TFN_INPUT_DEPTH_U16 = 2 } tfn_input_kind;
int tfn_estimate_points(tfn_handle h, const void* input, int input_kind, double scale, int batch, int H, int W,
                        void* stream, void* out_normals, float* out_points);

/* tfn_estimate_host for uint16 depth codes (see tfn_estimate_u16). */
int tfn_estimate_host_u16(tfn_handle h, const unsigned short* host_codes, double depth_scale, int batch, int H,
                          int W, void* host_out, void* stream);

/* the paper's accuracy yardsticks on the GPU: PlanePCA (Eq. 3,
 * method TFN_PLANE_PCA) or PlaneSVD (Eq. 2, TFN_PLANE_SVD) normals of fp32 depth, per SPEC
 * the centre and its valid 8-neighbours back-projected (Eq. 13), >= 3 valid
 * neighbours else invalid, 1-px border invalid, smallest-eigenvalue eigenvector of the 3x3
 * scatter / 4x4 normal matrix (cyclic Jacobi, fp64), oriented toward the camera.
 * out_normals: fp32 in the handle's layout (the output dtype option does not apply).
 * Uses the handle's intrinsics; its filter / Phi are irrelevant.  One thread per pixel. */
typedef enum { TFN_PLANE_PCA = 0, TFN_PLANE_SVD = 1 } tfn_plane_method;
int tfn_plane_fit(tfn_handle h, const float* depth, int method, int batch, int H, int W, void* stream,
                  float* out_normals);

/* angular-error statistics (Eq. 22-24) of est (device,
 * layout `layout`) against gt (device, planar [batch,3,H,W], NaN = invalid), ADDED
 * into stats_dev (device int64[8]): [0] sum of psi in 1e-6 degree units, [1] m =
 * pixels valid in both, [2..4] count psi <= 10/20/30 deg, [5] valid estimates,
 * [6] valid GT, [7] pixels.  psi = atan2(|a x b|, a.b) in fp64. */
int tfn_stats(const float* est, const float* gt, int batch, int H, int W, int layout,
              void* stream, long long* stats_dev);

/* Probe of the device Phi (P8): for n groups of 8 candidates (device fp32 [n,8];
 * a non-finite candidate is skipped) writes Phi (mean or median of the finite ones)
 * to out_dev[n] and their count to k_dev[n], through the kernel's own code path.
 * nz_mode: TFN_NZ_MEAN, TFN_NZ_MEDIAN (the per-pixel / general path), or 2 = the median as
 * the strip kernel's fast and masked variants decide it (NaN-propagating network and its
 * extreme-magnitude finiteness test; same results).  INVALID_ARGUMENT otherwise. */
int tfn_debug_phi8(const float* cand_dev, long long n, int nz_mode, float* out_dev, int* k_dev,
                   void* stream);

/* Speed-of-light reference for the roofline: moves exactly the 3F2N
 * traffic mix — reads in_dev fp32 [batch,H,W], writes every sample three times into
 * out_dev fp32 [batch,3,H,W] (planar), 4 B in + 12 B out per pixel, with the strip
 * kernel's access pattern and no arithmetic.  H*W % 4 == 0 and 16-B aligned buffers
 * (INVALID_ARGUMENT otherwise).  Asynchronous on stream. */
int tfn_debug_sol(const float* in_dev, int batch, int H, int W, void* stream, float* out_dev);

/* Release a handle (and its workspace, work counters and AUTO read-back word).  NULL is
 * OK.  Frees device memory with cudaFree (which waits for the device), so work already
 * submitted with h completes first; no call may use h afterwards. */
int tfn_destroy(tfn_handle h);

/* Static string for a status code. */
const char* tfn_status_string(int status);

/* Number of kernels this library has launched in the process (for bench accounting). */
unsigned long long tfn_kernel_launches(void);

/* The strip variant TFN_OPT_KERNEL = 0 (AUTO) currently picks for handle h: *variant = 2
 * (fast strip kernel + exact per-pixel special path), 4 (masked: the fast kernel whose
 * special path skips pixels with an invalid tap — their NaN is already exact) or 3 (general
 * strip kernel).  AUTO starts fast; the fast and masked kernels count the row steps that
 * needed their special path, the count returns asynchronously (pinned word + event, read at
 * a later call, never a sync), and above 20 % of row steps AUTO steps fast -> masked ->
 * general (below 10 % back; masked mode re-probes the fast kernel every 256th call,
 * general mode the masked one every 32nd).  Results are bit-identical either way; only speed differs.
 * uint16 input and the point cloud always run the general kernel.  Returns
 * TFN_ERR_INVALID_ARGUMENT for NULLs. */
int tfn_auto_variant(tfn_handle h, int* variant);

/* Host-only probe of the AUTO state machine (no device needed; for tests): states 0 fast,
 * 1 masked, 2 general.  *next_state = the state after a probe of variant `probed` (0 fast,
 * 1 masked) reported `rate` (fraction of its row steps that needed the special path);
 * *run (0/1/2) and *probe (0/1) = the variant call number `call` runs in `state` and whether
 * it counts its special row steps, when a read-back is possible (`can_probe`).  Returns
 * TFN_ERR_INVALID_ARGUMENT for NULL outputs or states / variants out of range. */
int tfn_debug_auto(int state, int probed, double rate, unsigned call, int can_probe,
                   int* next_state, int* run, int* probe);

/* Pixels the fp32 unit-step kernel (TFN_OPT_KERNEL 5/6) sent to the exact per-pixel path in
 * the last launch on h made with TFN_OPT_COUNT_SPECIAL = 1 (*count = -1 if none).
 * Synchronous (waits for that launch).  INVALID_ARGUMENT for NULLs, CUDA on a copy error. */
int tfn_debug_special_count(tfn_handle h, long long* count);

/* ABI version (major*10000 + minor*100 + patch). */
int tfn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TFN_H */
