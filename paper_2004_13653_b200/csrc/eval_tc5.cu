// Step a4, the tensor-core path -- per-warp pipelines.  Used for the plain
// fp16 mode when a group's window is one MMA tile of N <= 64 columns; the split-fp16 mode and
// larger windows use eval_tc.cu.
//
// Every Table-1 kernel is a product k(s) k(t), so a group's block is the dense
// contraction S = A . B^T, A[row][p] = ky_p(row), B[col][p] = kx_p(col), both masked by the
// point's fp64-decided integer ranges (R3).
//
// One CTA per SM: kW worker warps (10 when N <= 48, else 8), each an independent pipeline with
// its OWN TMEM accumulator (a 48- or 64-column slice of the SM's 512) and its own two operand
// buffers, plus 4 epilogue warps.
// A worker pops (group, segment) items and walks them in BUCKET-HOMOGENEOUS chunks of 32
// points (lane = point; a chunk's rows lie in its bucket's (B + 2F)-row window, so NA = NB =
// (B + 2F)/8 units carry every nonzero factor); per chunk it loads the next chunk's points
// (one chunk ahead), waits for its buffer's previous MMAs (tcgen05.commit -> mbarrier),
// evaluates its NA + NB units in straight-line code (the Gaussian: the A and B exact-ratio
// chains advanced together by packed FMUL2), RN to fp16 (R11), stores them into
// the UMMA layouts (A: MN-major 128-byte swizzle; B: MN-major unswizzled), and one elected
// lane issues its two tcgen05.mma.kind::f16 (M = 128, N, K = 16) -- no CTA barrier and no
// cross-warp ordering: the workers never wait on each other.  At an item's end the worker
// commits its accumulator and posts a drain request (a ready bit per epilogue warp + an
// mbarrier doorbell the idle epilogue warps sleep on); the 4 epilogue warps (TMEM lanes
// 32e..32e+31 each) read it with tcgen05.ld into the item's splat slot and release it.
// Per (item, pixel) the accumulation order is the item's chunk order (deterministic); the
// combine pass sums the slots in a fixed order (bitwise sharding).
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>

#include "internal.cuh"
#include "kernels.cuh"

namespace kde {
namespace tc5 {

// worker warps per CTA (one CTA per SM): as many 48- or 64-column accumulators as the SM's 512
// TMEM columns hold (10 for N <= 48, 8 for N = 64)
template <int N> struct Workers { static constexpr int kW = N <= 48 ? 10 : 8, kAcc = N <= 48 ? 48 : 64; };
// M = 64 tiles (group windows of <= 64 rows, N <= 48): an accumulator holds its rows 16q..16q+15
// in TMEM lanes 32q + 16h .. 32q + 16h + 15 (lane half h = 0, 1; measured with
// tools/tmem_m64_lane_probe.cu), so two share each 48-column slice: 16 workers in 8 slices,
// their double-buffered 4 + 3 KB operands filling the shared memory
template <int N, int MR> struct Tc5Shape {
    static constexpr int kW = MR == 64 ? 16 : Workers<N>::kW, kAcc = Workers<N>::kAcc;
};
constexpr int kEpi = 4;                    // epilogue warps
constexpr int kPts = 32;                   // points per chunk (K of two MMAs)
constexpr int kABytes = kTcM * kPts * 2;   // A: 128 rows x 32 fp16
constexpr uint32_t kALBO = 4096;           // A: bytes between the two 64-row atoms
constexpr int kSBO = 512;                  // B: bytes between 8-column core-matrix groups

struct Args {
    Geom g;
    PathGeom pg;
    const uint32_t* __restrict__ offsets;
    const float2* __restrict__ xy;
    const uint2* __restrict__ rng;
    const int4* __restrict__ items;
    int* __restrict__ totals;  // plan totals (kTot*): item count, work-queue head
    float* __restrict__ splat;
    int n;           // MMA N
    int buf_bytes;   // operand bytes per buffer
    float kq, q2;    // Gaussian: -log2(e)/(2 h^2), 2^(2 kq)
    float twoc;      // Cosine: 2 cos(pi / (2 h))
    KConst k;        // 1-D factor constants (kernels.cuh)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor, MN-major canonical layouts (layout = 0: no swizzle, 2:
// 128-byte swizzle; for the swizzled layout LBO is the stride between 64-element MN atoms and
// SBO the stride between 8-row K groups, for the unswizzled one LBO is the K-group stride and
// SBO the stride between 8-element MN core matrices -- cute's make_umma_desc<Major::MN>).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    d |= (uint64_t)layout << 61;
    return d;                // base offset 0 (atoms are 1024-byte aligned), lbo mode 0
}

// A operand (M = 128 rows x K = 32 points per stage), MN-major with the 128-byte swizzle: a
// swizzle atom is 64 rows (128 B) x 8 points = 1 KB; the 4 point groups of an atom are
// kASBO apart, the two 64-row atoms kALBO apart.  The 16-byte chunk holding rows 8c..8c+7
// of point k sits at chunk c ^ (k mod 8) of the point's 128-byte atom row (bank-conflict
// free for the tensor core's reads and for the producers' one-16-B-per-lane stores).
constexpr uint32_t kASBO = 1024;
__device__ __forceinline__ uint32_t a_unit_addr(uint32_t base_lane, int u, int r, uint32_t albo) {
    return base_lane + (uint32_t)(u >> 3) * albo + ((uint32_t)((u & 7) ^ r) << 4);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

// Wait for the phase of the given parity to complete.  A pipeline wait here lasts at most
// milliseconds; one that spins for ~2^26 polls (seconds) is a protocol bug: trap (the launch
// fails with an error) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0, n = 0;
    for (;;) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (++n > (1u << 26)) __trap();
    }
}

// one bounded wait: true once the phase of the given parity has completed; otherwise the
// thread is suspended for up to ~ns nanoseconds (a doorbell that does not spin)
__device__ __forceinline__ bool mbar_try_wait_ns(uint64_t* bar, uint32_t parity, uint32_t ns) {
    uint32_t ok = 0;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// 1-D TMA: bytes (multiple of 16, 16-B aligned both ends) global -> shared, completing on bar
__device__ __forceinline__ void tma_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// one lane of the (converged) warp: true on exactly one lane
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 16; k++) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ void sts128(uint32_t saddr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}


__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {  // packed fp32x2 multiply (FMUL2)
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
    return make_uint4(pack_half2(f[0], f[1]), pack_half2(f[2], f[3]), pack_half2(f[4], f[5]), pack_half2(f[6], f[7]));
}

// 8 factors -> masked to [lo, lo + span] (relative to c0) -> fp16 x 8
__device__ __forceinline__ uint4 mask_pack(float (&f)[8], int c0, int lo, int span) {
    const int l0 = max(lo - c0, 0), h0 = min(lo + span - c0, 7);
    const uint32_t m = l0 <= h0 ? (2u << h0) - (1u << l0) : 0u;
#pragma unroll
    for (int e = 0; e < 8; e++) f[e] = (m & (1u << e)) ? f[e] : 0.f;
    return make_uint4(pack_half2(f[0], f[1]), pack_half2(f[2], f[3]), pack_half2(f[4], f[5]), pack_half2(f[6], f[7]));
}

// the factors khat((c + 1/2 - P) / h) of one unit [c0, c0 + 8): d0 = c0 - (P - 1/2)
template <int K, bool REC>
__device__ __forceinline__ void factors(float d0, const Args& a, float (&f)[8]) {
    if constexpr (K == KDE_GAUSSIAN && REC) {
        float gv = ex2_ftz(d0 * d0 * a.kq);
        float r = ex2_ftz(fmaf(2.0f, d0, 1.0f) * a.kq);
#pragma unroll
        for (int e = 0; e < 8; e++) {
            f[e] = gv;
            gv *= r;
            r *= a.q2;
        }
    } else if constexpr (K == KDE_COSINE) {
        f[0] = __cosf(d0 * a.k.kc);
        f[1] = __cosf((d0 + 1.0f) * a.k.kc);
#pragma unroll
        for (int e = 2; e < 8; e++) f[e] = fmaf(a.twoc, f[e - 1], -f[e - 2]);
#pragma unroll
        for (int e = 0; e < 8; e++) f[e] = fmaxf(f[e], 0.0f);  // DESIGN.md R8
    } else {
#pragma unroll
        for (int e = 0; e < 8; e++) f[e] = khat<K>(d0 + (float)e, a.k);
    }
}

// two units' Gaussian factors at once: both exact-ratio chains in one packed FMUL2 stream
__device__ __forceinline__ void factors2(float d0, float d1, const Args& a, float (&f0)[8], float (&f1)[8]) {
    uint64_t G = pk2(ex2_ftz(d0 * d0 * a.kq), ex2_ftz(d1 * d1 * a.kq));
    uint64_t R = pk2(ex2_ftz(fmaf(2.0f, d0, 1.0f) * a.kq), ex2_ftz(fmaf(2.0f, d1, 1.0f) * a.kq));
    const uint64_t Q = pk2(a.q2, a.q2);
#pragma unroll
    for (int e = 0; e < 8; e++) {
        upk2(G, f0[e], f1[e]);
        G = fmul2(G, R);
        R = fmul2(R, Q);
    }
}



template <int K, bool REC, int NU, int NC, int MR>
__global__ void __launch_bounds__(32 * (Tc5Shape<NC, MR>::kW + kEpi), 1) tc5_kernel(const Args a) {
    constexpr int kW = Tc5Shape<NC, MR>::kW, kAccCols = Tc5Shape<NC, MR>::kAcc, kThreads = 32 * (kW + kEpi);
    constexpr int kAB = MR * kPts * 2;  // A bytes per buffer
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) uint64_t bar_buf[kW][2];    // MMAs done reading worker w's buffer b
    __shared__ __align__(8) uint64_t bar_acc[kW];       // worker w's accumulator complete
    __shared__ __align__(8) uint64_t bar_drained[kW];   // ... read back by the 4 epilogue warps
    __shared__ int s_slot[kW];                          // the posted item's splat slot
    __shared__ unsigned s_ready[kEpi];                  // bit w: worker w's posted item not yet
                                                        // drained by epilogue warp e
    __shared__ unsigned s_fin;                          // bit w: worker w has no more items
    __shared__ __align__(8) uint64_t bar_post[kEpi];    // doorbell of epilogue warp e (a post or a
                                                        // finish arrives; phases may merge: the
                                                        // waits are bounded and re-check s_ready)
    __shared__ uint32_t s_tmem;

    const Geom& g = a.g;
    const PathGeom& pg = a.pg;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t sm0 = (smem_u32(smem) + 1023u) & ~1023u;  // worker w's buffers at 2 w buf_bytes
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int w = 0; w < kW; w++) {
            mbar_init(&bar_buf[w][0], 1);
            mbar_init(&bar_buf[w][1], 1);
            mbar_init(&bar_acc[w], 1);
            mbar_init(&bar_drained[w], kEpi);
        }
        for (int e = 0; e < kEpi; e++) {
            s_ready[e] = 0u;
            mbar_init(&bar_post[e], 1);
        }
        s_fin = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = t; e < kW * 2 * a.buf_bytes / 16; e += kThreads) sts128(sm0 + 16u * e, make_uint4(0u, 0u, 0u, 0u));
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    if (warp < kW) {
        // ------------------------------------------------------------------ worker
        constexpr int NA = NU, NB = NU;
        const int w = warp;
        // the accumulator: M = 128, slice w; M = 64, slice w / 2 at lane offset 16 (w % 2)
        const uint32_t acc = MR == 64 ? tmem + ((uint32_t)(16 * (w & 1)) << 16) + (uint32_t)((w >> 1) * kAccCols)
                                      : tmem + (uint32_t)(w * kAccCols);
        const uint32_t idesc = (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(a.n >> 3) << 17) |
                               ((uint32_t)(MR >> 4) << 24);
        const uint32_t a_lane = (uint32_t)((lane >> 3) * kASBO + (lane & 7) * 128);
        const uint32_t b_lane = (uint32_t)((lane >> 3) * 128 + (lane & 7) * 16);
        const int r8 = lane & 7;
        const int nitems = a.totals[kTotSlots];
        int q = 0;                  // chunks so far: buffer q & 1
        int prev_ua[2] = {-1, -1};  // first A unit each buffer holds (-1: all zero)
        int nitem = 0;
        for (;;) {
            int wi = 0;
            if (lane == 0) wi = atomicAdd(&a.totals[kTotQueue], 1);
            wi = __shfl_sync(0xffffffffu, wi, 0);
            if (wi >= nitems) break;
            const int4 it = a.items[wi];
            const int gx = it.x % pg.ngx, gy = it.x / pg.ngx;
            const int ox = gx * pg.px - g.F, oy = gy * pg.py - g.F;
            const int ns = min(pg.s, g.nby - gy * pg.s);
            const int key0 = gx * g.nby + gy * pg.s;
            int lo = 0, hi = 0;  // lane b: bucket b's points within [k0, k1)
            if (lane < ns) {
                lo = max((int)a.offsets[key0 + lane], it.y);
                hi = min((int)a.offsets[key0 + lane + 1], it.z);
            }
            unsigned live = __ballot_sync(0xffffffffu, hi > lo);
            if (!live) {  // (cannot happen for a planned item): its slot is all zero
                float* sp = a.splat + (size_t)it.w * (pg.slot_w * pg.slot_h);
                for (int e = lane; e < pg.slot_w * pg.slot_h; e += 32) sp[e] = 0.f;
                continue;
            }
            const float adx = (float)(gx * g.B - ox) - 0.5f;
            // chunk cursor (b, p): bucket b, first point p; the next one is prefetched
            int b = live ? __ffs(live) - 1 : 0;
            int p = __shfl_sync(0xffffffffu, lo, b);
            int bh = __shfl_sync(0xffffffffu, hi, b);
            float2 nl = make_float2(0.f, 0.f);
            uint2 nr = make_uint2(1u, 0u);  // lo > hi: empty
            if (live && p + lane < bh) {
                nl = a.xy[p + lane];
                nr = a.rng[p + lane];
            }
            bool first = true;
            while (live) {
                const int cb = b, cp = p, cbh = bh;
                const float2 cl = nl;
                const uint2 cr = nr;
                // advance the cursor and prefetch the next chunk's points
                p += kPts;
                if (p >= bh) {
                    live &= ~(1u << b);
                    if (live) {
                        b = __ffs(live) - 1;
                        p = __shfl_sync(0xffffffffu, lo, b);
                        bh = __shfl_sync(0xffffffffu, hi, b);
                    }
                }
                const bool more = live != 0;
                nl = make_float2(0.f, 0.f);
                nr = make_uint2(1u, 0u);
                if (more && p + lane < bh) {
                    nl = a.xy[p + lane];
                    nr = a.rng[p + lane];
                }
                // this chunk: bucket cb, points [cp, min(cp + 32, cbh))
                const int ua0 = (cb * g.B) >> 3;
                const float pyh = cl.y + ((float)((gy * pg.s + cb) * g.B - oy) - 0.5f);
                const float pxh = cl.x + adx;
                const bool valid = cp + lane < cbh;
                const int jlo = valid ? (int)(cr.y & 0xffffu) - oy : 1 << 29;
                const int jsp = (int)(cr.y >> 16) - (int)(cr.y & 0xffffu);
                const int ilo = valid ? (int)(cr.x & 0xffffu) - ox : 1 << 29;
                const int isp = (int)(cr.x >> 16) - (int)(cr.x & 0xffffu);
                const int bf = q & 1;
                if (q >= 2) mbar_wait(&bar_buf[w][bf], (uint32_t)((q >> 1) - 1) & 1u);
                const uint32_t base = sm0 + (uint32_t)((2 * w + bf) * a.buf_bytes);
                const uint32_t ab = base + a_lane, bb = base + (uint32_t)kAB + b_lane;
                const int old = bf ? prev_ua[1] : prev_ua[0];
                if (old >= 0 && old != ua0) {  // A units the buffer's last chunk (another bucket) wrote
#pragma unroll
                    for (int k = 0; k < NA; k++) {
                        const int u = old + k;
                        if (u < ua0 || u >= ua0 + NA) sts128(a_unit_addr(ab, u, r8, kALBO), make_uint4(0u, 0u, 0u, 0u));
                    }
                }
                if (bf) prev_ua[1] = ua0;
                else prev_ua[0] = ua0;
                // the NA row units and NB column units of this chunk, straight-line.  When all 32
                // points' ranges cover units 1 .. NU-2 on both axes (a full chunk away from the
                // raster edges: the usual case), those units need no mask.
                const bool inner = __all_sync(0xffffffffu, jlo <= (ua0 + 1) * 8 && jlo + jsp >= (ua0 + NU - 1) * 8 - 1 &&
                                                               ilo <= 8 && ilo + isp >= (NU - 1) * 8 - 1);
#pragma unroll
                for (int k = 0; k < NU; k++) {
                    float fa[8], fb[8];
                    const float da = (float)((ua0 + k) * 8) - pyh, db = (float)(k * 8) - pxh;
                    if constexpr (K == KDE_GAUSSIAN && REC) {
                        factors2(da, db, a, fa, fb);
                    } else {
                        factors<K, REC>(da, a, fa);
                        factors<K, REC>(db, a, fb);
                    }
                    if (k >= 1 && k <= NU - 2 && inner) {
                        sts128(a_unit_addr(ab, ua0 + k, r8, kALBO), pack8(fa));
                        sts128(bb + k * kSBO, pack8(fb));
                    } else {
                        sts128(a_unit_addr(ab, ua0 + k, r8, kALBO), mask_pack(fa, (ua0 + k) * 8, jlo, jsp));
                        sts128(bb + k * kSBO, mask_pack(fb, k * 8, ilo, isp));
                    }
                }
                fence_async_smem();
                __syncwarp();
                if (first && nitem > 0) mbar_wait(&bar_drained[w], (uint32_t)(nitem - 1) & 1u);  // acc reused
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 2; kk++)
                        mma_f16(acc, umma_desc(base + kk * 2 * kASBO, kALBO, kASBO, 2),
                                umma_desc(base + kAB + kk * 256, 128, kSBO), idesc, (!first || kk > 0) ? 1u : 0u);
                    mma_commit(&bar_buf[w][bf]);
                    if (!more) mma_commit(&bar_acc[w]);
                }
                __syncwarp();
                first = false;
                q++;
            }
            if (lane == 0) {  // the item's accumulator completes on bar_acc[w]: post it
                s_slot[w] = it.w;
                __threadfence_block();
#pragma unroll
                for (int e = 0; e < kEpi; e++) atomicOr(&s_ready[e], 1u << w);
#pragma unroll
                for (int e = 0; e < kEpi; e++) mbar_arrive(&bar_post[e]);
            }
            nitem++;
        }
        if (lane == 0) {
            if (q) atomicAdd(&a.totals[kTotChunksExec], q);  // executed chunks (kde_stats.tc_mma_flops)
            __threadfence_block();
            atomicOr(&s_fin, 1u << w);  // (after its last post)
#pragma unroll
            for (int e = 0; e < kEpi; e++) mbar_arrive(&bar_post[e]);
        }
    } else {
        // ------------------------------------------------------------------ epilogue
        const int quad = warp & 3;  // tcgen05.ld: warp reaches TMEM lanes 32 (warp % 4) .. + 31
        // the accumulator row of this lane (M = 64: of the worker whose lane half it is)
        const int row = MR == 64 ? quad * 16 + (lane & 15) : quad * 32 + lane;
        const int slot_floats = pg.slot_w * pg.slot_h;
        const int e = warp - kW;  // this epilogue warp's ready word
        volatile unsigned* ready = &s_ready[e];
        volatile unsigned* fin = &s_fin;
        uint32_t par = 0;   // bit w: parity of worker w's next accumulator phase
        uint32_t bell = 0;  // parity of the doorbell's next phase
        for (;;) {
            unsigned m = __shfl_sync(0xffffffffu, *ready, 0);  // warp-uniform (tcgen05.ld is .aligned)
            if (m == 0u) {  // nothing posted: done when every worker is, else sleep on the doorbell
                const unsigned f = __shfl_sync(0xffffffffu, *fin, 0);
                __threadfence_block();
                if (f == (1u << kW) - 1u && __shfl_sync(0xffffffffu, *ready, 0) == 0u) break;
                if (mbar_try_wait_ns(&bar_post[e], bell, 2000u)) bell ^= 1u;
                __syncwarp();
                continue;
            }
            while (m) {
                const int w = __ffs(m) - 1;
                m &= m - 1;
                mbar_wait(&bar_acc[w], (par >> w) & 1u);
                par ^= 1u << w;
                tc_fence_after();
                const int slot = s_slot[w];
                float* dst = a.splat + (size_t)slot * slot_floats + (size_t)row * pg.slot_w;
                const bool mine = MR != 64 || (lane >> 4) == (w & 1);  // M = 64: this worker's lane half
                const uint32_t col = (uint32_t)((MR == 64 ? (w >> 1) : w) * kAccCols);
                for (int c0 = 0; c0 < a.n; c0 += 16) {
                    float v[16];
                    tmem_ld16(tmem + ((uint32_t)(quad * 32) << 16) + col + (uint32_t)c0, v);
#pragma unroll
                    for (int k = 0; k < 16; k += 4)
                        if (mine && c0 + k < pg.slot_w)
                            *reinterpret_cast<float4*>(dst + c0 + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    atomicAnd(&s_ready[e], ~(1u << w));  // before the release: the next post sets it again
                    mbar_arrive(&bar_drained[w]);
                }
                __syncwarp();
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int K, bool REC, int NU, int NC, int MR>
static int launch(kde_ctx* c, EvalPlan& pl, Args& a, cudaStream_t s) {
    a.buf_bytes = MR * kPts * 2 + a.n * kPts * 2;
    const size_t smem = (size_t)Tc5Shape<NC, MR>::kW * 2 * a.buf_bytes + 1024;
    auto kern = tc5_kernel<K, REC, NU, NC, MR>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "tensor-core kernel attribute");
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->p.device);
    if (getenv("KDE_DEBUG"))
        fprintf(stderr, "[kde] tc5: NU=%d smem=%zu grid=%d n=%d\n", NU, smem, nsm, a.n);
    cudaMemsetAsync(pl.d_totals + kTotQueue, 0, sizeof(int), s);  // work-queue head
    tmark(c, 3, s);
    kern<<<nsm, 32 * (Tc5Shape<NC, MR>::kW + kEpi), smem, s>>>(a);  // persistent: one CTA per SM
    return KDE_OK;
}

template <int K, bool REC>
static int launch_nu(kde_ctx* c, EvalPlan& pl, Args& a, cudaStream_t s, int nu) {
    // N = window rounded up to 16: <= 48 up to 6 units, else 64; M = 64 tiles when the plan's
    // group windows have <= 64 rows (PathGeom::mrows)
    if (pl.pg.mrows == 64) {
        switch (nu) {
        case 2: return launch<K, REC, 2, 48, 64>(c, pl, a, s);
        case 3: return launch<K, REC, 3, 48, 64>(c, pl, a, s);
        case 4: return launch<K, REC, 4, 48, 64>(c, pl, a, s);
        case 5: return launch<K, REC, 5, 48, 64>(c, pl, a, s);
        default: return launch<K, REC, 6, 48, 64>(c, pl, a, s);
        }
    }
    switch (nu) {
    case 2: return launch<K, REC, 2, 48, 128>(c, pl, a, s);
    case 3: return launch<K, REC, 3, 48, 128>(c, pl, a, s);
    case 4: return launch<K, REC, 4, 48, 128>(c, pl, a, s);
    case 5: return launch<K, REC, 5, 48, 128>(c, pl, a, s);
    case 6: return launch<K, REC, 6, 48, 128>(c, pl, a, s);
    case 7: return launch<K, REC, 7, 64, 128>(c, pl, a, s);
    default: return launch<K, REC, 8, 64, 128>(c, pl, a, s);
    }
}

}  // namespace tc5

// The per-warp-pipeline tensor-core kernel for plain fp16 evaluations whose group window is
// one MMA tile of N <= 64 columns (eval_tc.cu's launch_tc falls back to its own kernel
// otherwise).  Returns KDE_EUNSUPPORTED (nothing launched) for geometries it does not take.
int launch_tc5(kde_ctx* c, cudaStream_t s) {
    EvalPlan& pl = c->plan[KDE_PATH_TENSOR];
    const PathGeom& pg = pl.pg;
    const char* env = getenv("KDE_TC5");
    if (env && atoi(env) == 0) return KDE_EUNSUPPORTED;
    const int win = c->g.B + 2 * c->g.F;
    const int nu = (win + 7) / 8;
    if (pg.nsub() != 1 || c->g.B % 8 != 0 || pg.mma_n > 64 || (nu <= 6 && pg.mma_n > 48) || nu < 2 || nu > 8 ||
        nu * 8 > pg.mma_n || (pg.mrows == 64 && (nu > 6 || pg.wh > 64)))
        return KDE_EUNSUPPORTED;
    tc5::Args a;
    a.g = c->g;
    a.pg = pg;
    a.offsets = c->d_offsets;
    a.xy = c->pb.xy;
    a.rng = c->pb.rng;
    a.items = pl.d_items;
    a.totals = pl.d_totals;
    a.splat = pl.d_splat;
    a.n = pg.mma_n;
    a.kq = (float)(-0.5 * 1.4426950408889634074 / (c->hpx * c->hpx));
    a.q2 = (float)exp2(2.0 * (double)a.kq);
    a.twoc = (float)(2.0 * cos(3.14159265358979323846 / (2.0 * c->hpx)));
    a.k = make_kconst(c->hpx);
    const double dmax = c->g.F + c->g.B + 8.0;  // a unit starts within F + B + 7.5 px of its points
    const bool rec = -(double)a.kq * dmax * dmax < 120.0;
    using Fn = int (*)(kde_ctx*, EvalPlan&, tc5::Args&, cudaStream_t, int);
    static const Fn kL[8] = {tc5::launch_nu<0, true>, tc5::launch_nu<1, true>, tc5::launch_nu<2, true>,
                             tc5::launch_nu<3, true>, tc5::launch_nu<4, true>, tc5::launch_nu<5, true>,
                             tc5::launch_nu<6, true>, tc5::launch_nu<7, true>};
    if (c->kern == KDE_GAUSSIAN && !rec) return tc5::launch_nu<6, false>(c, pl, a, s, nu);
    return kL[c->kern](c, pl, a, s, nu);
}

}  // namespace kde
