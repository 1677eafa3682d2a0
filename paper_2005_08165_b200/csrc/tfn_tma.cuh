// tfn_tma.cuh — per-warp TMA row ring shared by the strip kernels (tfn_strip.cuh, tfn_f32.cuh).
//
// A warp's strip is 128 columns x strip_h rows of one frame.  Its input rows (plus one halo row
// above and below) arrive as TMA 2D boxes of 136 columns (c0-4 .. c0+131: the 16-B lane vectors
// stay aligned and every lane has its two halo columns) x TFN_RING_RC rows, zero-filled outside
// the image (a zero sample is invalid: Q3 / Q5 make out-of-image taps invalid for free), into a
// ring of TFN_RING_NS slots with one mbarrier each.  Lane 0 issues; every lane waits on the
// slot's barrier at the first row of a box and reads its 4 samples (LDS.128) and 2 halos (LDS).
// The box of chunk k-1 is reissued as chunk k-1+NS when chunk k starts (the warp has read all
// of k-1 by then: rows are consumed in order, once).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

// Bounds-checked debug build (-DTFN_BOUNDS_CHECK; compute-sanitizer is closed on the GPU pool):
// every global row / column index and shared-memory ring / queue index is checked on the device
// and a violation traps (the launch fails with an unspecified-launch error).
#ifndef TFN_CHECK
#ifdef TFN_BOUNDS_CHECK
#define TFN_CHECK(cond)                                                             \
    do {                                                                            \
        if (!(cond)) {                                                              \
            printf("TFN_CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);    \
            __trap();                                                               \
        }                                                                           \
    } while (0)
#else
#define TFN_CHECK(cond) ((void)0)
#endif
#endif

#ifndef TFN_RING_RC
#define TFN_RING_RC 8             // rows per TMA box (r02 A/B: 8 x 2 slots beats 4 x 4 by 1-2 %, same shared memory)
#endif
#ifndef TFN_RING_NS
#define TFN_RING_NS 2             // slots per warp
#endif

namespace tfn {
namespace ring {

constexpr int RC = TFN_RING_RC;
constexpr int NS = TFN_RING_NS;
constexpr int BOXW = 136;
constexpr int SLOT_FLOATS = RC * BOXW;
static_assert((SLOT_FLOATS * 4) % 128 == 0, "TMA box destinations must stay 128-B aligned: TFN_RING_RC % 4 == 0");

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

struct Ring {
    const float* base;         // this warp's slot 0, row 0, lane vector (generic pointer into shared memory)
    unsigned sbase;            // the same slot 0 row 0 (shared address, box origin)
    unsigned bar;              // barrier of slot 0 (shared address; slot s at bar + 8 s)
    unsigned kq;               // boxes this warp consumed before the current strip
    int nch;                   // boxes of the current strip
    int x, y, b;               // origin of box 0 of the current strip (column, row, frame)
};

// per-warp setup: slots at `slots` (NS * SLOT_FLOATS floats, 16-B aligned), NS barriers at `bars`
__device__ __forceinline__ void ring_init(Ring& r, float* slots, unsigned long long* bars, int lane) {
    r.sbase = smem_u32(slots);
    r.base = slots + 4 + 4 * lane;
    r.bar = smem_u32(bars);
    r.kq = 0;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NS; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(r.bar + 8 * k) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
}

// issue box k of the current strip into its slot (lane 0 only)
__device__ __forceinline__ void ring_issue(const CUtensorMap* tm, const Ring& r, int k) {
    const unsigned slot = (r.kq + (unsigned)k) % NS;
    const unsigned dst = r.sbase + slot * (SLOT_FLOATS * 4), bar = r.bar + slot * 8;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(SLOT_FLOATS * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 :: "r"(dst), "l"(tm), "r"(r.x), "r"(r.y + k * RC), "r"(r.b), "r"(bar) : "memory");
}

// start a strip: rows y0-1 .. y1 (inclusive) of frame b, columns from x; issue the first boxes
__device__ __forceinline__ void ring_strip(const CUtensorMap* tm, Ring& r, int x, int y0, int y1, int b, int lane) {
    r.nch = (y1 - y0 + 2 + RC - 1) / RC;
    r.x = x; r.y = y0 - 1; r.b = b;
    __syncwarp();
    if (lane == 0)
        for (int k = 0; k < NS && k < r.nch; ++k) ring_issue(tm, r, k);
}
__device__ __forceinline__ void ring_strip_done(Ring& r) { r.kq += (unsigned)r.nch; }

__device__ __forceinline__ void bar_wait(unsigned bar, unsigned parity) {
    unsigned done = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    } while (!done);
}

// row rr (0 = the strip's first row - 1) into the lane's 6-sample window (columns c0-1 .. c0+4)
__device__ __forceinline__ void ring_row(const CUtensorMap* tm, const Ring& r, int rr, int lane, float zr[6]) {
    const int k = rr / RC, rw = rr - k * RC;
    const unsigned g = r.kq + (unsigned)k, slot = g % NS;
    if (rw == 0) {
        if (k > 0 && k - 1 + NS < r.nch) {
            __syncwarp();
            if (lane == 0) ring_issue(tm, r, k - 1 + NS);
        }
        bar_wait(r.bar + slot * 8, (g / NS) & 1u);
    }
    TFN_CHECK(slot < (unsigned)NS && rw >= 0 && rw < RC && k < r.nch && lane >= 0 && lane < 32);
    const float* p = r.base + slot * SLOT_FLOATS + rw * BOXW;
    const float4 m = *reinterpret_cast<const float4*>(p);
    zr[0] = p[-1]; zr[1] = m.x; zr[2] = m.y; zr[3] = m.z; zr[4] = m.w; zr[5] = p[4];
}

}  // namespace ring
}  // namespace tfn
