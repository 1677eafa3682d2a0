// tfn_abi.cu — the C ABI declared in include/tfn.h: argument validation, kernel
// selection, launch-geometry, the pipelined host-buffer path, status strings.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <new>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/tfn.h"
#include "tfn_kernels.h"
#ifndef TFN_STRIP_TMA
#define TFN_STRIP_TMA 1
#endif

#define TFN_API extern "C" __attribute__((visibility("default")))

namespace {

std::atomic<unsigned long long> g_launches{0};

struct Workspace {
    void* in[2] = {nullptr, nullptr};
    void* out[2] = {nullptr, nullptr};
    size_t frames = 0;        // capacity in frames of one chunk
    size_t frame_in = 0;      // bytes per frame the buffers were sized for
    size_t frame_out = 0;
    cudaStream_t s[2] = {nullptr, nullptr};
    cudaEvent_t start = nullptr;
};

}  // namespace

struct tfn_ctx {
    tfn_intrinsics K;
    int filter;
    int mode;
    int layout = TFN_LAYOUT_PLANAR;
    int out_kind = 0;                    // TFN_OPT_OUT_DTYPE: 0 fp32, 1 half, 2 oct16
    double kp = 1.0, k0 = 2.0;           // TFN_FILTER_CUSTOM weights (tfn_set_filter_weights)
    int kernel = tfn::TFN_KERNEL_AUTO;
    int strip_h = 0;
    int grid = 0;
    int dynamic = 1;
    int device = 0;
    int sms = 148;
    int strip_ctas_per_sm[3][2] = {{0, 0}, {0, 0}, {0, 0}};   // fp32 input: [fast, general, masked][depth, disparity]
    int strip_ctas_u16 = 0;                           // uint16 depth codes (general variant)
    int f32_ctas[2][2] = {{0, 0}, {0, 0}};            // fp32 unit-step kernel: [depth, disparity][fast, masked]
    int count_special = 0;               // TFN_OPT_COUNT_SPECIAL: fp32 kernel counts its special pixels
    std::atomic<int*> last_fired{nullptr};   //   (device counter of the last such launch)
    std::mutex ws_mu;
    Workspace ws;
    int* work = nullptr;                 // ring of per-call {work, fired} counter pairs
    std::atomic<unsigned> call_seq{0};
    std::atomic<unsigned> capture_seq{0};    // next dedicated capture slot (after the ring)
    // AUTO kernel selection: the fast and masked strip variants count their special row
    // steps; the count comes back through a pinned word a few calls later and moves the
    // choice fast -> masked -> general (and back)
    std::mutex auto_mu;
    int* fb_host = nullptr;              // pinned: fired row steps of the last probed launch
    cudaEvent_t fb_ev = nullptr;
    bool fb_pending = false;
    double fb_steps = 0;                 // row steps of that launch
    int auto_state = 0;                  // current AUTO choice: 0 fast, 1 masked, 2 general
    int fb_variant = 0;                  // variant of the pending probe: 0 fast, 1 masked
    unsigned auto_calls = 0;
};
#define TFN_WORK_RING 4096
#define TFN_CAPTURE_SLOTS 1024           // counter pairs reserved for CUDA-graph captures (never reused)
// AUTO: step to the next variant (fast -> masked -> general) when more than this fraction
// of the probed variant's row steps needed the special path (measured break-even ~0.24:
// config 2 has 0.011 and runs 217 fast vs 210 masked vs 167 general; config 4 (holes + 1 %
// salt) fires on 0.98 of the fast variant's row steps but few of the masked one's, and
// runs 94 fast vs 191 masked vs 164 general); back below TFN_AUTO_FAST_BELOW
#define TFN_AUTO_GENERAL_ABOVE 0.20
#define TFN_AUTO_FAST_BELOW 0.10
#define TFN_AUTO_PROBE_FAST 8            // fast / masked mode: read the counter back every 8th call
#define TFN_AUTO_PROBE_GENERAL 32        // general mode: every 32nd call probes the masked variant
#define TFN_AUTO_PROBE_MASKED 256        // masked mode: every 256th call probes the fast variant (on
                                         // holey data a fast call costs ~2x; back to fast gains ~3 %)

namespace {
// AUTO state machine, pure host logic (pinned by tests/test_abi.py through tfn_debug_auto).
// state: 0 fast, 1 masked, 2 general.  auto_next: the state after the feedback of a probe
// of `probed` (0 fast, 1 masked) that fired on `rate` of its row steps.
int auto_next(int state, int probed, double rate) {
    if (probed == 0) {
        if (rate > TFN_AUTO_GENERAL_ABOVE) return state == 0 ? 1 : state;
        if (rate < TFN_AUTO_FAST_BELOW) return 0;
        return state;
    }
    if (rate > TFN_AUTO_GENERAL_ABOVE) return 2;
    if (rate < TFN_AUTO_FAST_BELOW && state == 2) return 1;
    return state;
}
// auto_pick: the variant call n runs in `state` (0 fast, 1 masked, 2 general) and whether it
// counts its special row steps (a probe), given whether a probe can be read back
void auto_pick(int state, unsigned n, bool can_probe, int* run, bool* probe) {
    int r = state;
    bool want = (n % TFN_AUTO_PROBE_FAST) == 0;
    if (state == 1 && can_probe && (n % TFN_AUTO_PROBE_MASKED) == 0) r = 0;   // clean again?
    if (state == 2) {
        const bool reprobe = can_probe && (n % TFN_AUTO_PROBE_GENERAL) == 0;
        r = reprobe ? 1 : 2;
        want = reprobe;
    }
    *run = r;
    *probe = can_probe && r != 2 && want;
}
}  // namespace

namespace {

bool is_fin(double x) { return std::isfinite(x); }

int check_device(int* dev, int* sms) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) { cudaGetLastError(); return TFN_ERR_CUDA; }
    int major = 0, minor = 0, n = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, d) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) {
        cudaGetLastError();
        return TFN_ERR_CUDA;
    }
    if (major != 10 || minor != 0) return TFN_ERR_CUDA;   // built for sm_100a only
    *dev = d;
    *sms = n;
    return TFN_OK;
}

bool overlap(const void* a, size_t na, const void* b, size_t nb) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
}

// bytes per sample in / per normal component out
size_t in_bytes(int in_u16) { return in_u16 ? 2 : 4; }
// bytes per output pixel (normals) and the alignment the strip kernel's vector stores need
size_t out_px_bytes(const tfn_ctx* h) { return h->out_kind == 0 ? 12 : h->out_kind == 1 ? 6 : 4; }
uintptr_t out_align(const tfn_ctx* h) { return h->out_kind == 0 ? 15 : h->out_kind == 1 ? 7 : 15; }

// ---- fp32 unit-step kernel (tfn_f32.cuh): TMA descriptor and guard constants ----------------
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_tiled() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
        cudaGetLastError();
    });
    return fn;
}
// the input [B,H,W] fp32 as a 3-D tensor (W, H, B); boxes of 136 columns x RC rows, zero fill
// outside (= invalid samples, Q3)
bool f32_tensor_map(CUtensorMap* tm, const void* in, int B, int H, int W) {
    EncodeTiled enc = encode_tiled();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)H * W * 4};
    const cuuint32_t box[3] = {(cuuint32_t)tfn::ring::BOXW, (cuuint32_t)tfn::ring::RC, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(in), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// with u = 2^-24, a multiplier whose three terms share one sign is accurate to
// c1 (depth 16u incl. margin, disparity 6u); the pixel's angular error is then at most
//   (c1 + 2u)(2 + |a|/fx + |b|/fy) + 4u + sqrt(3) u + 6u (1/fx + 1/fy) + (c1 + 14u) V/|n'|
// and the orientation is certain when |Phi| >= 2 (c1 + 12u) V + 12u (1/fx + 1/fy) |n'|.
// Budget: 0.8e-3 deg (the parity gate is 1e-3 deg).  Returns false when even V <= 1.5 |n'| cannot
// be certified (tiny focal lengths): the fp32 kernel is not used then.
bool f32_consts(const tfn_ctx* h, bool disp, tfn::F32Consts* k) {
    const double u = std::ldexp(1.0, -24);
    const double c1 = disp ? 6 * u : 16 * u, Ac = c1 + 2 * u, B = c1 + 14 * u;
    const double fx = h->K.fx, fy = h->K.fy;
    const double teff = 0.8e-3 * 3.14159265358979323846 / 180.0;
    const double inv = 1.0 / fx + 1.0 / fy;
    const double k0lim = (teff - 4 * u - std::sqrt(3.0) * u - 6 * u * inv - 2 * Ac) / B;
    k->kp = (float)h->kp;
    k->k0 = (float)h->k0;
    k->k0lim = (float)(k0lim * (1 - 1e-6));
    k->kca = (float)(Ac / (fx * B) * (1 + 1e-6));
    k->kr = (float)(Ac / (fy * B) * (1 + 1e-6));
    k->cg = (float)(12 * u * inv * (1 + 1e-6));
    k->tb = (float)(2 * (c1 + 12 * u) * (1 + 1e-6));
    return k0lim >= 1.5;
}

// The {work, fired} counter pair a launch uses.  Direct calls take the next pair of a ring of
// TFN_WORK_RING (zeroed by a memset on the launch's stream just before the kernel).  A launch
// being captured into a CUDA graph gets a pair of its own that no other launch ever uses: the
// graph's memset node re-zeroes it at every replay, so a replay can run concurrently with any
// direct call (a ring slot baked into a graph was handed out again 4096 calls
// later).  When the capture pairs run out, captured launches schedule strips statically
// (no counter; same results).  nullptr: no counter available.
int* counter_pair(tfn_ctx* h, bool capturing) {
    if (!h->work) return nullptr;
    if (!capturing) return h->work + 2 * (h->call_seq.fetch_add(1) % TFN_WORK_RING);
    const unsigned k = h->capture_seq.fetch_add(1);
    if (k >= TFN_CAPTURE_SLOTS) return nullptr;
    return h->work + 2 * (TFN_WORK_RING + k);
}

int validate(tfn_handle h, const void* in, int in_u16, int batch, int H, int W, const void* out) {
    if (!h) return TFN_ERR_INVALID_ARGUMENT;
    if (batch < 0 || H <= 0 || W <= 0) return TFN_ERR_INVALID_ARGUMENT;
    if (batch == 0) return TFN_OK;
    if (!in || !out) return TFN_ERR_INVALID_ARGUMENT;
    const unsigned long long px = (unsigned long long)batch * (unsigned long long)H * (unsigned long long)W;
    if (px > (1ull << 60) / 12) return TFN_ERR_INVALID_ARGUMENT;
    const size_t ib = in_bytes(in_u16), ob = h->out_kind == 0 ? 4 : 2;
    if (((uintptr_t)in & (ib - 1)) || ((uintptr_t)out & (ob - 1))) return TFN_ERR_INVALID_ARGUMENT;
    if (overlap(in, px * ib, out, px * out_px_bytes(h))) return TFN_ERR_INVALID_ARGUMENT;
    return TFN_OK;
}

int run(tfn_handle h, const void* in, int in_u16, bool disp, int batch, int H, int W, cudaStream_t st,
        void* out, float* pts = nullptr, double pscale = 1.0) {
    tfn::KernelArgs a;
    a.tmap = nullptr;
    a.in = in;
    a.out = out;
    a.in_u16 = in_u16;
    a.out_kind = h->out_kind;
    a.pts = pts;
    a.pscale = (float)pscale;
    a.ifx = (float)(1.0 / h->K.fx);
    a.ify = (float)(1.0 / h->K.fy);
    a.kp = h->kp;
    a.k0 = h->k0;
    a.B = batch;
    a.H = H;
    a.W = W;
    a.fx = (float)h->K.fx;
    a.fy = (float)h->K.fy;
    a.u0 = (float)h->K.u0;
    a.v0 = (float)h->K.v0;
    a.layout = h->layout;
    // strip kernel: 4-sample vectors in and 4-component vectors out (16 B fp32, 8 B for
    // uint16 / half), and (frame, strip-row, strip-col) items indexed in 32 bits
    const long long max_items = (long long)((W + TFN_STRIP_COLS - 1) / TFN_STRIP_COLS) * (long long)batch;   // at strip_h = H
    const uintptr_t in_al = 4 * in_bytes(in_u16) - 1, out_al = out_align(h);
    const bool strip_ok = (W % 4 == 0) && (((uintptr_t)in & in_al) == 0) && (((uintptr_t)out & out_al) == 0) &&
                          (((uintptr_t)pts & 15) == 0) && max_items < (1LL << 31);
    int kernel = h->kernel;
    bool probe = false;
    // CUDA-graph capture: no host-side event query or read-back while capturing (the AUTO
    // choice made so far is baked into the graph; the work counter memset is a graph node)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) { cudaGetLastError(); cap = cudaStreamCaptureStatusNone; }
    const bool capturing = cap != cudaStreamCaptureStatusNone;
    // the fp32 unit-step kernel: fp32 in / fp32 normals, no points, frames below 65536 x 65536
    // (special-pixel queue entries pack v and u in 16 bits each), a certifiable guard
    tfn::F32Consts f32k;
    const bool f32_ok = strip_ok && !in_u16 && !pts && h->out_kind == 0 && H < 65536 && W < 65536 &&
                        f32_consts(h, disp, &f32k);
    // (not picked by AUTO: measured slower than the strip kernel on configs[1])
    if ((kernel == tfn::TFN_KERNEL_F32 || kernel == tfn::TFN_KERNEL_F32_MASKED) && !f32_ok)
        kernel = strip_ok ? tfn::TFN_KERNEL_STRIP : tfn::TFN_KERNEL_PIXEL;
    if (kernel == tfn::TFN_KERNEL_F32 || kernel == tfn::TFN_KERNEL_F32_MASKED) {
        const bool vm = kernel == tfn::TFN_KERNEL_F32_MASKED;
        CUtensorMap tm;
        if (!f32_tensor_map(&tm, in, batch, H, W)) return TFN_ERR_CUDA;
        const int ctas_sm = h->f32_ctas[disp][vm];
        const long long resident_warps = (long long)h->sms * ctas_sm * (TFN_F32_THREADS / 32);
        const long long sx_n = (W + 127) / 128;
        int sh = h->strip_h;
        if (sh <= 0) {
            sh = (H % 48 == 0) ? 48 : 24;
            while (sh > 6 && sx_n * ((H + sh - 1) / sh) * (long long)batch < 3 * resident_warps) sh /= 2;
        }
        while (sx_n * ((H + sh - 1) / sh) * (long long)batch >= (1LL << 31) && sh < H) sh = sh * 2 < H ? sh * 2 : H;
        const long long items = sx_n * ((H + sh - 1) / sh) * (long long)batch;
        if (items >= (1LL << 31)) return TFN_ERR_INVALID_ARGUMENT;
        a.strip_h = sh;
        a.work = nullptr;
        a.fired = nullptr;
        long long ctas = h->grid > 0 ? h->grid : (long long)h->sms * ctas_sm;
        const long long need = (items + (TFN_F32_THREADS / 32) - 1) / (TFN_F32_THREADS / 32);
        if (ctas > need) ctas = need;
        if (ctas < 1) ctas = 1;
        const bool dyn = h->dynamic && items > ctas * (TFN_F32_THREADS / 32);
        int* ctr = (dyn || h->count_special) ? counter_pair(h, capturing) : nullptr;
        if (ctr) {
            if (cudaMemsetAsync(ctr, 0, 2 * sizeof(int), st) != cudaSuccess) return TFN_ERR_CUDA;
            a.work = dyn ? ctr : nullptr;
            a.fired = h->count_special ? ctr + 1 : nullptr;     // special pixels of this launch
            h->last_fired.store(a.fired);
        }
        if (tfn::launch_f32_any(tm, a, f32k, h->filter, h->mode, disp, vm, (int)ctas, st) != cudaSuccess)
            return TFN_ERR_CUDA;
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return TFN_OK;
    }
    if (kernel == tfn::TFN_KERNEL_AUTO) {
        if (!strip_ok) {
            kernel = tfn::TFN_KERNEL_PIXEL;
        } else if (in_u16 || pts) {
            kernel = tfn::TFN_KERNEL_STRIP_GENERAL;     // the only strip variant built for these
        } else {
            std::lock_guard<std::mutex> lk(h->auto_mu);
            if (!capturing && h->fb_pending && cudaEventQuery(h->fb_ev) == cudaSuccess) {
                const double rate = h->fb_steps > 0 ? *h->fb_host / h->fb_steps : 0.0;
                h->auto_state = auto_next(h->auto_state, h->fb_variant, rate);
                h->fb_pending = false;
            }
            cudaGetLastError();           // a not-ready query is not an error
            const unsigned n = h->auto_calls++;
            const bool can_probe = !capturing && h->fb_host && !h->fb_pending;
            int run = 0;
            auto_pick(h->auto_state, n, can_probe, &run, &probe);
            kernel = run == 0 ? tfn::TFN_KERNEL_STRIP : run == 1 ? tfn::TFN_KERNEL_STRIP_MASKED
                                                                 : tfn::TFN_KERNEL_STRIP_GENERAL;
            if (probe) h->fb_variant = run;
        }
    }
    // the fast and masked strip variants are built for fp32 input without points; the general
    // one has the same results (bit for bit) and runs everything else
    if ((in_u16 || pts) && (kernel == tfn::TFN_KERNEL_STRIP || kernel == tfn::TFN_KERNEL_STRIP_MASKED))
        kernel = tfn::TFN_KERNEL_STRIP_GENERAL;
    const bool strip = (kernel == tfn::TFN_KERNEL_STRIP || kernel == tfn::TFN_KERNEL_STRIP_GENERAL ||
                        kernel == tfn::TFN_KERNEL_STRIP_MASKED);
    if (strip && !strip_ok) return TFN_ERR_INVALID_ARGUMENT;
    const int gen = (kernel == tfn::TFN_KERNEL_STRIP_GENERAL) ? 1 : (kernel == tfn::TFN_KERNEL_STRIP_MASKED) ? 2 : 0;
    int grid = 0;
    if (strip) {
        const int ctas_sm = in_u16 ? h->strip_ctas_u16 : h->strip_ctas_per_sm[gen][disp];
        const long long resident_warps = (long long)h->sms * ctas_sm * (TFN_STRIP_THREADS / 32);
        int sh = h->strip_h;
        const long long sx_n = (W + TFN_STRIP_COLS - 1) / TFN_STRIP_COLS;
        if (sh <= 0) {
            // 48 rows per strip (a multiple of the 3-row unroll; measured best on config 2 with
            // dynamic scheduling: 12 -> 192.7, 24 -> 201.1, 48 -> 203.3 Gpx/s) when it divides H;
            // 24 when it does not (fast and masked variants).  r01h sweep (bench --strip-h, --hw,
            // 2 reps): 1080x1920 x128 runs 198.9 at 24 vs 191.5 at 48 masked, 206.2 vs 199.3 fast
            // (with or without holes), while 2160x3840 x32 (45 bands of 48) keeps 48: 216.9 vs 213.5
            // fast, 210.3 vs 207.0 masked; 480x640 keeps 48 (216.7 vs 213.9).  The general
            // variant keeps 48 (166.6 at 24 vs 167.9 at 48 on configs[3]).  Then halved while the
            // batch gives fewer than 3 strips per resident warp (the tail: 32 x 720x1280 frames,
            // 2.7 strips per warp at 48, run 181.1 at 24 vs 167.5 at 48)
            sh = (H % 48 == 0 || gen == 1) ? 48 : 24;
            while (sh > 6 && sx_n * ((H + sh - 1) / sh) * (long long)batch < 3 * resident_warps) sh /= 2;
        }
        // (frame, strip-row, strip-col) items are indexed in 32 bits: raise a small requested
        // strip height until they fit (results do not depend on it)
        while (sx_n * ((H + sh - 1) / sh) * (long long)batch >= (1LL << 31) && sh < H) sh = sh * 2 < H ? sh * 2 : H;
        a.strip_h = sh;
        a.work = nullptr;
        a.fired = nullptr;
        const long long items = sx_n * ((H + sh - 1) / sh) * (long long)batch;
        long long ctas = h->grid > 0 ? h->grid : (long long)h->sms * ctas_sm;
        const long long need = (items + (TFN_STRIP_THREADS / 32) - 1) / (TFN_STRIP_THREADS / 32);
        if (ctas > need) ctas = need;
        if (ctas < 1) ctas = 1;
        grid = (int)ctas;
        // the work counter only hands out items beyond each warp's first (static) one: with
        // no more items than warps it is pure overhead (a memset node per call: single
        // frames 14.5 -> 12.5 us per graph-replayed call measured)
        const bool dyn = h->dynamic && items > ctas * (TFN_STRIP_THREADS / 32);
        int* ctr = (dyn || probe) ? counter_pair(h, capturing) : nullptr;
        if (ctr) {
            if (cudaMemsetAsync(ctr, 0, 2 * sizeof(int), st) != cudaSuccess) return TFN_ERR_CUDA;
            a.work = dyn ? ctr : nullptr;
            a.fired = probe ? ctr + 1 : nullptr;
        }
    } else {
        a.strip_h = 0;
    }
    // strip kernels on fp32 input read their rows through the TMA ring (tfn_tma.cuh)
    static const CUtensorMap zero_tm = {};
    CUtensorMap tmv;
    a.tmap = &zero_tm;
    if (strip && !in_u16 && TFN_STRIP_TMA) {
        if (!f32_tensor_map(&tmv, in, batch, H, W)) return TFN_ERR_CUDA;
        a.tmap = &tmv;
    }
    cudaError_t e = tfn::launch_3f2n(a, h->filter, h->mode, disp, kernel, grid, st);
    if (e != cudaSuccess) return TFN_ERR_CUDA;
    if (a.fired) {
        std::lock_guard<std::mutex> lk(h->auto_mu);
        if (!h->fb_pending &&
            cudaMemcpyAsync(h->fb_host, a.fired, sizeof(int), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
            cudaEventRecord(h->fb_ev, st) == cudaSuccess) {
            h->fb_steps = (double)((W + TFN_STRIP_COLS - 1) / TFN_STRIP_COLS) * H * (double)batch;
            h->fb_pending = true;
        }
        cudaGetLastError();
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return TFN_OK;
}

}  // namespace


TFN_API int tfn_create(const tfn_intrinsics* K, int filter, int nz_mode, tfn_handle* out) {
    if (!K || !out) return TFN_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    if (filter < 0 || filter > 4 || nz_mode < 0 || nz_mode > 1) return TFN_ERR_INVALID_ARGUMENT;
    if (!is_fin(K->fx) || !is_fin(K->fy) || !is_fin(K->u0) || !is_fin(K->v0) || K->fx <= 0 || K->fy <= 0)
        return TFN_ERR_CONFIG;
    int dev = 0, sms = 0;
    const int st = check_device(&dev, &sms);
    if (st != TFN_OK) return st;
    tfn_ctx* h = new (std::nothrow) tfn_ctx();
    if (!h) return TFN_ERR_CUDA;
    h->K = *K;
    h->filter = filter;
    h->mode = nz_mode;
    h->device = dev;
    h->sms = sms;
    for (int g = 0; g < 3; ++g)
        for (int d = 0; d < 2; ++d) {
            int& n = h->strip_ctas_per_sm[g][d];
            n = tfn::strip_occupancy(filter, nz_mode, d != 0, g, 0);
            if (n <= 0) n = 1;
        }
    for (int d = 0; d < 2; ++d)
        for (int m = 0; m < 2; ++m) {
            int& n = h->f32_ctas[d][m];
            n = tfn::f32_occupancy(filter, nz_mode, d != 0, m != 0);
            if (n <= 0) n = 1;
        }
    h->strip_ctas_u16 = tfn::strip_occupancy(filter, nz_mode, false, 1, 1);
    if (h->strip_ctas_u16 <= 0) h->strip_ctas_u16 = 1;
    if (cudaMalloc(&h->work, 2 * (TFN_WORK_RING + TFN_CAPTURE_SLOTS) * sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        h->work = nullptr;                // static scheduling (and the fast AUTO choice) still work
    }
    if (cudaMallocHost(&h->fb_host, sizeof(int)) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->fb_ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        if (h->fb_host) cudaFreeHost(h->fb_host);
        h->fb_host = nullptr;             // AUTO then always picks the fast variant
    }
    *out = h;
    return TFN_OK;
}

TFN_API int tfn_set_filter_weights(tfn_handle h, double kp, double k0) {
    if (!h || h->filter != TFN_FILTER_CUSTOM) return TFN_ERR_INVALID_ARGUMENT;
    if (!is_fin(kp) || !is_fin(k0) || kp <= 0 || k0 <= 0) return TFN_ERR_CONFIG;
    h->kp = kp;
    h->k0 = k0;
    return TFN_OK;
}

TFN_API int tfn_set_layout(tfn_handle h, int layout) {
    if (!h || (layout != TFN_LAYOUT_PLANAR && layout != TFN_LAYOUT_PACKED)) return TFN_ERR_INVALID_ARGUMENT;
    h->layout = layout;
    return TFN_OK;
}

TFN_API int tfn_set_option(tfn_handle h, int option, long long value) {
    if (!h) return TFN_ERR_INVALID_ARGUMENT;
    switch (option) {
    case TFN_OPT_KERNEL:
        if (value < 0 || value > 6) return TFN_ERR_INVALID_ARGUMENT;
        h->kernel = (int)value;
        return TFN_OK;
    case TFN_OPT_STRIP_H:
        if (value < 0 || value > 1 << 20) return TFN_ERR_INVALID_ARGUMENT;
        h->strip_h = (int)value;
        return TFN_OK;
    case TFN_OPT_GRID:
        if (value < 0 || value > 1 << 24) return TFN_ERR_INVALID_ARGUMENT;
        h->grid = (int)value;
        return TFN_OK;
    case TFN_OPT_DYNAMIC:
        h->dynamic = value ? 1 : 0;
        return TFN_OK;
    case TFN_OPT_COUNT_SPECIAL:
        h->count_special = value ? 1 : 0;
        return TFN_OK;
    case TFN_OPT_OUT_DTYPE:
        if (value != TFN_OUT_F32 && value != TFN_OUT_F16 && value != TFN_OUT_OCT16) return TFN_ERR_INVALID_ARGUMENT;
        h->out_kind = (int)value;
        return TFN_OK;
    default:
        return TFN_ERR_INVALID_ARGUMENT;
    }
}

TFN_API int tfn_estimate(tfn_handle h, const float* depth, int batch, int H, int W, void* stream,
                         void* out_normals) {
    int st = validate(h, depth, 0, batch, H, W, out_normals);
    if (st != TFN_OK || batch == 0) return st;
    return run(h, depth, 0, false, batch, H, W, (cudaStream_t)stream, out_normals);
}

TFN_API int tfn_estimate_u16(tfn_handle h, const unsigned short* depth_codes, double depth_scale, int batch, int H,
                             int W, void* stream, void* out_normals) {
    if (!h) return TFN_ERR_INVALID_ARGUMENT;
    if (!is_fin(depth_scale) || depth_scale <= 0) return TFN_ERR_CONFIG;   // validated; cancels (A.4)
    int st = validate(h, depth_codes, 1, batch, H, W, out_normals);
    if (st != TFN_OK || batch == 0) return st;
    return run(h, depth_codes, 1, false, batch, H, W, (cudaStream_t)stream, out_normals);
}

TFN_API int tfn_estimate_disparity(tfn_handle h, const float* disparity, double baseline_times_f,
                                   int batch, int H, int W, void* stream, void* out_normals) {
    if (!h) return TFN_ERR_INVALID_ARGUMENT;
    if (h->K.fx != h->K.fy) return TFN_ERR_CONFIG;                       // Eq. 19: one f
    if (!is_fin(baseline_times_f) || baseline_times_f <= 0) return TFN_ERR_CONFIG;
    int st = validate(h, disparity, 0, batch, H, W, out_normals);
    if (st != TFN_OK || batch == 0) return st;
    return run(h, disparity, 0, true, batch, H, W, (cudaStream_t)stream, out_normals);
}

TFN_API int tfn_estimate_points(tfn_handle h, const void* input, int input_kind, double scale, int batch, int H,
                                int W, void* stream, void* out_normals, float* out_points) {
    if (!h) return TFN_ERR_INVALID_ARGUMENT;
    if (input_kind != TFN_INPUT_DEPTH_F32 && input_kind != TFN_INPUT_DISPARITY_F32 &&
        input_kind != TFN_INPUT_DEPTH_U16)
        return TFN_ERR_INVALID_ARGUMENT;
    if (!is_fin(scale) || scale <= 0) return TFN_ERR_CONFIG;
    const bool disp = input_kind == TFN_INPUT_DISPARITY_F32;
    if (disp && h->K.fx != h->K.fy) return TFN_ERR_CONFIG;
    const int u16 = input_kind == TFN_INPUT_DEPTH_U16 ? 1 : 0;
    int st = validate(h, input, u16, batch, H, W, out_normals);
    if (st != TFN_OK || batch == 0) return st;
    if (!out_points || ((uintptr_t)out_points & 3)) return TFN_ERR_INVALID_ARGUMENT;
    const size_t px = (size_t)batch * H * W;
    if (overlap(out_points, px * 12, input, px * in_bytes(u16)) ||
        overlap(out_points, px * 12, out_normals, px * out_px_bytes(h)))
        return TFN_ERR_INVALID_ARGUMENT;
    return run(h, input, u16, disp, batch, H, W, (cudaStream_t)stream, out_normals, out_points, scale);
}

namespace {

// the pipelined host-buffer path shared by tfn_estimate_host / tfn_estimate_host_u16:
// ~48 MB chunks alternate between two streams (H2D copy, kernel, D2H copy)
int host_run(tfn_handle h, const void* host_in, int in_u16, bool disp, int batch, int H, int W, void* host_out,
             void* stream) {
    if (batch < 0 || H <= 0 || W <= 0) return TFN_ERR_INVALID_ARGUMENT;
    if (batch == 0) return TFN_OK;
    if (!host_in || !host_out) return TFN_ERR_INVALID_ARGUMENT;
    const size_t fpx = (size_t)H * (size_t)W;
    if ((unsigned long long)batch * fpx > (1ull << 60) / 12) return TFN_ERR_INVALID_ARGUMENT;
    const size_t fin = fpx * in_bytes(in_u16), fout = fpx * out_px_bytes(h);
    // chunk k+1's H2D would read input that chunk k's D2H already overwrote
    if (overlap(host_in, (size_t)batch * fin, host_out, (size_t)batch * fout)) return TFN_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lock(h->ws_mu);
    Workspace& ws = h->ws;
    size_t chunk = (48u << 20) / fin;
    if (chunk < 1) chunk = 1;
    if (chunk > (size_t)batch) chunk = batch;
    if (ws.frames < chunk || ws.frame_in < fin || ws.frame_out < fout) {
        for (int i = 0; i < 2; ++i) {
            if (ws.in[i]) cudaFree(ws.in[i]);
            if (ws.out[i]) cudaFree(ws.out[i]);
            ws.in[i] = ws.out[i] = nullptr;
        }
        ws.frames = 0;
        for (int i = 0; i < 2; ++i) {
            if (cudaMalloc(&ws.in[i], chunk * fin) != cudaSuccess || cudaMalloc(&ws.out[i], chunk * fout) != cudaSuccess) {
                cudaGetLastError();
                return TFN_ERR_CUDA;
            }
        }
        ws.frames = chunk;
        ws.frame_in = fin;
        ws.frame_out = fout;
    }
    if (!ws.s[0]) {
        for (int i = 0; i < 2; ++i)
            if (cudaStreamCreateWithFlags(&ws.s[i], cudaStreamNonBlocking) != cudaSuccess) return TFN_ERR_CUDA;
        if (cudaEventCreateWithFlags(&ws.start, cudaEventDisableTiming) != cudaSuccess) return TFN_ERR_CUDA;
    }
    cudaStream_t user = (cudaStream_t)stream;
    if (cudaEventRecord(ws.start, user) != cudaSuccess) return TFN_ERR_CUDA;
    for (int i = 0; i < 2; ++i)
        if (cudaStreamWaitEvent(ws.s[i], ws.start, 0) != cudaSuccess) return TFN_ERR_CUDA;
    int rc = TFN_OK;
    size_t done = 0;
    int k = 0;
    const char* hin = static_cast<const char*>(host_in);
    char* hout = static_cast<char*>(host_out);
    while (done < (size_t)batch) {
        const size_t n = ((size_t)batch - done < chunk) ? (size_t)batch - done : chunk;
        cudaStream_t s = ws.s[k & 1];
        if (cudaMemcpyAsync(ws.in[k & 1], hin + done * fin, n * fin, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            rc = TFN_ERR_CUDA;
            break;
        }
        rc = run(h, ws.in[k & 1], in_u16, disp, (int)n, H, W, s, ws.out[k & 1]);
        if (rc != TFN_OK) break;
        if (cudaMemcpyAsync(hout + done * fout, ws.out[k & 1], n * fout, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
            rc = TFN_ERR_CUDA;
            break;
        }
        done += n;
        ++k;
    }
    for (int i = 0; i < 2; ++i)
        if (cudaStreamSynchronize(ws.s[i]) != cudaSuccess) rc = TFN_ERR_CUDA;
    return rc;
}

}  // namespace

TFN_API int tfn_estimate_host(tfn_handle h, const float* host_in, int is_disparity, double baseline_times_f,
                              int batch, int H, int W, void* host_out, void* stream) {
    if (!h) return TFN_ERR_INVALID_ARGUMENT;
    if (is_disparity) {
        if (h->K.fx != h->K.fy) return TFN_ERR_CONFIG;
        if (!is_fin(baseline_times_f) || baseline_times_f <= 0) return TFN_ERR_CONFIG;
    }
    return host_run(h, host_in, 0, is_disparity != 0, batch, H, W, host_out, stream);
}

TFN_API int tfn_estimate_host_u16(tfn_handle h, const unsigned short* host_codes, double depth_scale, int batch, int H,
                                  int W, void* host_out, void* stream) {
    if (!h) return TFN_ERR_INVALID_ARGUMENT;
    if (!is_fin(depth_scale) || depth_scale <= 0) return TFN_ERR_CONFIG;
    return host_run(h, host_codes, 1, false, batch, H, W, host_out, stream);
}

TFN_API int tfn_plane_fit(tfn_handle h, const float* depth, int method, int batch, int H, int W, void* stream,
                          float* out_normals) {
    if (!h || (method != TFN_PLANE_PCA && method != TFN_PLANE_SVD)) return TFN_ERR_INVALID_ARGUMENT;
    if (batch < 0 || H <= 0 || W <= 0) return TFN_ERR_INVALID_ARGUMENT;
    if (batch == 0) return TFN_OK;
    if (!depth || !out_normals || ((uintptr_t)depth & 3) || ((uintptr_t)out_normals & 3)) return TFN_ERR_INVALID_ARGUMENT;
    const size_t px = (size_t)batch * H * W;
    if (overlap(depth, px * 4, out_normals, px * 12)) return TFN_ERR_INVALID_ARGUMENT;
    if (tfn::launch_planefit(depth, out_normals, batch, H, W, h->K.fx, h->K.fy, h->K.u0, h->K.v0, h->layout,
                             method, (cudaStream_t)stream) != cudaSuccess)
        return TFN_ERR_CUDA;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return TFN_OK;
}

TFN_API int tfn_stats(const float* est, const float* gt, int batch, int H, int W, int layout, void* stream,
                      long long* stats_dev) {
    if (batch < 0 || H <= 0 || W <= 0 || (layout != 0 && layout != 1)) return TFN_ERR_INVALID_ARGUMENT;
    if (batch == 0) return TFN_OK;
    if (!est || !gt || !stats_dev) return TFN_ERR_INVALID_ARGUMENT;
    if (tfn::launch_stats(est, gt, batch, H, W, layout, stats_dev, (cudaStream_t)stream) != cudaSuccess)
        return TFN_ERR_CUDA;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return TFN_OK;
}

TFN_API int tfn_debug_phi8(const float* cand_dev, long long n, int nz_mode, float* out_dev, int* k_dev,
                           void* stream) {
    if (n < 0 || nz_mode < 0 || nz_mode > 2) return TFN_ERR_INVALID_ARGUMENT;
    if (n == 0) return TFN_OK;
    if (!cand_dev || !out_dev || !k_dev) return TFN_ERR_INVALID_ARGUMENT;
    if (tfn::launch_phi8(cand_dev, n, nz_mode, out_dev, k_dev, (cudaStream_t)stream) != cudaSuccess)
        return TFN_ERR_CUDA;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return TFN_OK;
}

TFN_API int tfn_debug_sol(const float* in_dev, int batch, int H, int W, void* stream, float* out_dev) {
    if (batch < 0 || H <= 0 || W <= 0) return TFN_ERR_INVALID_ARGUMENT;
    if (batch == 0) return TFN_OK;
    if (!in_dev || !out_dev || ((long long)H * W) % 4 || ((uintptr_t)in_dev & 15) || ((uintptr_t)out_dev & 15))
        return TFN_ERR_INVALID_ARGUMENT;
    int dev = 0, sms = 0;
    if (check_device(&dev, &sms) != TFN_OK) return TFN_ERR_CUDA;
    if (tfn::launch_sol(in_dev, out_dev, batch, H, W, sms, (cudaStream_t)stream) != cudaSuccess) return TFN_ERR_CUDA;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return TFN_OK;
}

TFN_API int tfn_destroy(tfn_handle h) {
    if (!h) return TFN_OK;
    {
        std::lock_guard<std::mutex> lock(h->ws_mu);
        for (int i = 0; i < 2; ++i) {
            if (h->ws.in[i]) cudaFree(h->ws.in[i]);
            if (h->ws.out[i]) cudaFree(h->ws.out[i]);
            if (h->ws.s[i]) cudaStreamDestroy(h->ws.s[i]);
        }
        if (h->ws.start) cudaEventDestroy(h->ws.start);
    }
    if (h->work) cudaFree(h->work);
    if (h->fb_ev) cudaEventDestroy(h->fb_ev);
    if (h->fb_host) cudaFreeHost(h->fb_host);
    delete h;
    return TFN_OK;
}

TFN_API const char* tfn_status_string(int status) {
    switch (status) {
    case TFN_OK: return "TFN_OK";
    case TFN_ERR_INVALID_ARGUMENT: return "TFN_ERR_INVALID_ARGUMENT";
    case TFN_ERR_CONFIG: return "TFN_ERR_CONFIG";
    case TFN_ERR_CUDA: return "TFN_ERR_CUDA";
    default: return "TFN_UNKNOWN_STATUS";
    }
}

TFN_API unsigned long long tfn_kernel_launches(void) { return g_launches.load(); }

TFN_API int tfn_auto_variant(tfn_handle h, int* variant) {
    if (!h || !variant) return TFN_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(h->auto_mu);
    *variant = h->auto_state == 2 ? tfn::TFN_KERNEL_STRIP_GENERAL
             : h->auto_state == 1 ? tfn::TFN_KERNEL_STRIP_MASKED : tfn::TFN_KERNEL_STRIP;
    return TFN_OK;
}

TFN_API int tfn_debug_auto(int state, int probed, double rate, unsigned call, int can_probe,
                           int* next_state, int* run, int* probe) {
    if (!next_state || !run || !probe || state < 0 || state > 2 || probed < 0 || probed > 1)
        return TFN_ERR_INVALID_ARGUMENT;
    *next_state = auto_next(state, probed, rate);
    bool pr = false;
    auto_pick(state, call, can_probe != 0, run, &pr);
    *probe = pr ? 1 : 0;
    return TFN_OK;
}

TFN_API int tfn_debug_special_count(tfn_handle h, long long* count) {
    if (!h || !count) return TFN_ERR_INVALID_ARGUMENT;
    *count = -1;
    int* const lf = h->last_fired.load();
    if (!lf) return TFN_OK;
    int n = 0;
    if (cudaMemcpy(&n, lf, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return TFN_ERR_CUDA;
    *count = n;
    return TFN_OK;
}

TFN_API int tfn_version(void) { return 201; }
