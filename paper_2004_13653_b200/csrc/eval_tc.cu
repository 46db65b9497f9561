// Step a4: tensor-core Gaussian path.
//
// Table 1's Gaussian is a product kernel f(s,t) = k(s) k(t), so the block a group
// of points adds to its window is a genuine dense contraction:
//     S[row][col] = sum_p ky_p(row) * kx_p(col) = (A . B^T)[row][col],
//     A[row][p] = ky_p(row) (masked by the point's integer row range),
//     B[col][p] = kx_p(col) (masked by its column range).
// A group is a vertical stack of s buckets whose window (B + 2F columns, sB + 2F rows)
// fills the M = 128 TMEM lanes; N = B + 2F rounded up to 16.
//
// One persistent CTA (4 warps) per SM slot pops (group, segment of <= 512 points) items:
//   * operand generation, all warps: lane = point; for each 8-row (or 8-column) unit the
//     lane evaluates 8 Gaussian factors by the exact-ratio recurrence (2 SFU + 14 FMUL),
//     rounds them to fp16 (RN; 10-bit mantissa like tf32) and stores one 16-byte vector
//     straight into the UMMA operand layout (MN-major, no swizzle: an 8x8 core matrix is
//     128 contiguous bytes, k-groups 128 B apart (LBO), 8-row groups 512 B apart (SBO));
//   * one elected thread issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N, K=16) twice
//     per 32-point chunk, accumulating fp32 in TMEM, and tcgen05.commit's an mbarrier that
//     frees the operand buffer (double-buffered: generation overlaps the MMAs);
//   * epilogue: tcgen05.ld (32x32b) of the accumulator, each warp its 32 TMEM lanes, into
//     the segment's splat slot; the combine pass (shared with the direct path) then sums,
//     for every pixel, the slots of all groups and segments covering it in a fixed order
//     and applies C/(n h^2).
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>

#include "internal.cuh"
#include "kernels.cuh"

namespace kde {

constexpr int kTcThreads = 128;
constexpr int kIssuer = 96;  // the thread that issues the MMAs and commits
constexpr int kMaxStack = 32;
// H points per lane per chunk: a chunk is 32 H points = 2 H MMAs of K = 16; the A buffer
// is 128 x 32H fp16 (8H KB); 8-row core-matrix groups are 512 H bytes apart (SBO)
template <int H> struct TcShape {
    static constexpr int kChunk = 32 * H;
    static constexpr int kABytes = kTcM * kChunk * 2;
    static constexpr int kSBO = 512 * H;
    static constexpr int kMinBlocks = H == 1 ? 7 : 5;  // CTAs per SM (smem, TMEM, registers)
};

struct TcArgs {
    Geom g;
    PathGeom pg;
    const uint32_t* __restrict__ offsets;
    const float2* __restrict__ xy;
    const uint2* __restrict__ rng;
    const int4* __restrict__ items;
    const int2* __restrict__ group;
    int* __restrict__ totals;  // plan totals (kTot*): item count, work-queue head
    float* __restrict__ splat;
    int n;          // MMA N
    int tmem_cols;  // allocated TMEM columns (power of two >= n)
    float kq, q2;   // Gaussian: -log2(e)/(2 h^2), 2^(2 kq)
    float twoc;     // Cosine: 2 cos(pi / (2 h))
    KConst k;       // 1-D factor constants (kernels.cuh)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory descriptor: no swizzle, MN-major canonical layout.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
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

// 8 masked 1-D kernel factors khat((c + 1/2 - P) / h) of one point for the unit
// [c0, c0+8) -> fp16 x 8, stored as one 16-byte vector at the point's slot of the operand
// core matrix (shared address dst).  Every Table-1 kernel is a product k(s) k(t),
// so the same contraction serves all eight (NEXT-F2); only the factor generation differs:
//   Gaussian  exact-ratio recurrence g(d+1) = g(d) r, r(d+1) = r(d) q^2 (2 SFU + 14 FMUL)
//   Cosine    Chebyshev recurrence cos(a + (e+1)b) = 2 cos(b) cos(a + eb) - cos(a + (e-1)b)
//             (2 SFU + 6 FFMA)
//   others    the polynomial of kernels.cuh per element (FMA pipe)
// Support membership is the fp64-decided integer range [lo, lo + span] (R3).
// SPLIT (KDE_PATH_TENSOR_SPLIT, NEXT-F4): each factor f is also written as its fp16
// residual lo = RN16(f - RN16(f)) into a second operand plane lo_off bytes further, so that
// A_hi B_hi + A_hi B_lo + A_lo B_hi carries ~22 mantissa bits (the lo*lo term is 2^-22 of
// the product): the fp32 path's 1e-5 bar on the tensor pipe.
template <int K, bool SPLIT, bool REC>
__device__ __forceinline__ void kern_unit(uint32_t dst, uint32_t lo_off, int c0, float ph, int lo, int span,
                                          const TcArgs& a) {
    const int l0 = max(lo - c0, 0), h0 = min(lo + span - c0, 7);
    uint4 o = make_uint4(0u, 0u, 0u, 0u);
    uint4 ol = make_uint4(0u, 0u, 0u, 0u);
    if (l0 <= h0) {
        const uint32_t m = (2u << h0) - (1u << l0);
        const float d0 = (float)c0 - ph;
        float f[8];
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
#pragma unroll
        for (int e = 0; e < 8; e++) f[e] = (m & (1u << e)) ? f[e] : 0.f;
        o = make_uint4(pack_half2(f[0], f[1]), pack_half2(f[2], f[3]), pack_half2(f[4], f[5]),
                       pack_half2(f[6], f[7]));
        if constexpr (SPLIT) {
            const uint32_t hw[4] = {o.x, o.y, o.z, o.w};
            uint32_t lw[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const float2 hv = __half22float2(*reinterpret_cast<const __half2*>(&hw[q]));
                lw[q] = pack_half2(f[2 * q] - hv.x, f[2 * q + 1] - hv.y);
            }
            ol = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
    }
    sts128(dst, o);
    if constexpr (SPLIT) sts128(dst + lo_off, ol);
}

template <int H, int K, bool SPLIT, bool REC>
__global__ void __launch_bounds__(kTcThreads, TcShape<H>::kMinBlocks) tc_splat_kernel(const TcArgs a) {
    using SH = TcShape<H>;
    constexpr int kTcChunk = SH::kChunk, kTcABytes = SH::kABytes, kSBO = SH::kSBO;
    extern __shared__ __align__(1024) char tc_smem[];
    // [A0 | A1 | B0 | B1] operand buffers, then bookkeeping
    __shared__ __align__(8) uint64_t s_bar[3];  // operand buffers 0/1 freed; accumulator ready
    __shared__ uint32_t s_tmem;
    __shared__ int s_w;
    __shared__ uint32_t s_pre[kMaxStack + 1];   // first sorted position of each stack bucket

    const Geom& g = a.g;
    const PathGeom& pg = a.pg;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int bbytes = a.n * kTcChunk * 2;  // B buffer: N x 32H fp16
    const uint32_t idesc = (1u << 4)                       // D: f32
                           | (1u << 15) | (1u << 16)        // A, B: MN-major
                           | ((uint32_t)(a.n >> 3) << 17)   // N
                           | ((uint32_t)(kTcM >> 4) << 24); // M = 128
    const int slot_floats = pg.slot_w * pg.slot_h;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&s_tmem)),
                     "r"(a.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        mbar_init(&s_bar[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    uint32_t nuse[2] = {0u, 0u};  // commits issued per operand buffer (same on all threads)
    uint32_t nacc = 0;            // accumulator-ready commits

    // A buffer b at sm_a + b * astride (SPLIT: its lo plane kTcABytes further), B buffer b
    // at sm_b + b * bstride (lo plane bbytes further)
    constexpr int kPlanes = SPLIT ? 2 : 1;
    const int astride = kPlanes * kTcABytes, bstride = kPlanes * bbytes;
    const uint32_t sm_a = smem_u32(tc_smem);
    const uint32_t sm_b = sm_a + 2 * astride;
    const uint32_t koff = (uint32_t)((lane >> 3) * 128 + (lane & 7) * 16);  // point = k index
    const int nbu = a.n / 8;                                // B column units
    const int nitems = a.totals[kTotSlots];
    if (t == 0) s_w = atomicAdd(&a.totals[kTotQueue], 1);
    for (;;) {
        __syncthreads();
        const int w = s_w;
        if (w >= nitems) break;
        const int4 it = a.items[w];
        __syncthreads();                                         // everyone has read s_w
        if (t == 0) s_w = atomicAdd(&a.totals[kTotQueue], 1);  // pop the next item early
        const int gx = it.x % pg.ngx, gy = it.x / pg.ngx;
        // window origin (pixels): the group's window, or its sub-window (windows wider than
        // the 128 TMEM lanes / MMA N are cut into nsubx x nsuby pieces, slot = seg*nsub + sub)
        const int sub = it.w % pg.nsub();
        const int ox = gx * pg.px - g.F + (sub % pg.nsubx) * pg.sx;
        const int oy = gy * pg.py - g.F + (sub / pg.nsubx) * pg.sy;
        // the stack's buckets are the contiguous keys gx*nby + gy*s + k (column-major keys):
        // s_pre[k] = first sorted position of bucket k of the stack (items are absolute)
        const int key0 = gx * g.nby + gy * pg.s;
        const int ns = min(pg.s, g.nby - gy * pg.s);
        if (t <= ns) s_pre[t] = a.offsets[key0 + t];
        __syncthreads();
        const int cnt = it.z - it.y;
        const int nch = (cnt + kTcChunk - 1) / kTcChunk;  // (partial chunks: zero operands)
        const float shx = (float)(gx * g.B - ox) - 0.5f;   // (c + 1/2) - P = c - (P - 1/2)
        // the lane's points q + 32h of each chunk, their buckets within the stack (kb is
        // nondecreasing in q), prefetched one chunk ahead
        int q = it.y + lane;
        int kb = 0;
        float2 nl[H];
        uint2 nr[H];
        int nk[H];
#pragma unroll
        for (int h = 0; h < H; h++) {
            const int qh = q + 32 * h;
            nl[h] = make_float2(0.f, 0.f);
            nr[h] = make_uint2(0u, 0u);
            nk[h] = 0;
            if (qh < it.z) {
                while (kb + 1 < ns && (uint32_t)qh >= s_pre[kb + 1]) kb++;
                nl[h] = a.xy[qh];
                nr[h] = a.rng[qh];
                nk[h] = kb;
            }
        }
        for (int ch = 0; ch < nch; ch++) {
            const int b = ch & 1;
            float pxh[H], pyh[H];
            int ilo[H], ispan[H], jlo[H], jspan[H];
#pragma unroll
            for (int h = 0; h < H; h++) {
                const float2 l = nl[h];
                const uint2 rr = nr[h];
                const int by = gy * pg.s + nk[h];
                const bool valid = q + 32 * h < it.z;
                pxh[h] = pyh[h] = 0.f;
                ilo[h] = jlo[h] = 1 << 29;
                ispan[h] = jspan[h] = 0;
                if (valid) {
                    pxh[h] = l.x + shx;
                    pyh[h] = l.y + ((float)(by * g.B - oy) - 0.5f);
                    ilo[h] = (int)(rr.x & 0xffffu) - ox;
                    ispan[h] = (int)(rr.x >> 16) - (int)(rr.x & 0xffffu);
                    jlo[h] = (int)(rr.y & 0xffffu) - oy;
                    jspan[h] = (int)(rr.y >> 16) - (int)(rr.y & 0xffffu);
                }
            }
            q += kTcChunk;
#pragma unroll
            for (int h = 0; h < H; h++) {  // prefetch the next chunk's points
                const int qh = q + 32 * h;
                if (qh < it.z) {
                    while (kb + 1 < ns && (uint32_t)qh >= s_pre[kb + 1]) kb++;
                    nl[h] = a.xy[qh];
                    nr[h] = a.rng[qh];
                    nk[h] = kb;
                }
            }
            // the MMAs that last read this buffer must be done
            if (nuse[b] > 0) mbar_wait(&s_bar[b], (nuse[b] - 1) & 1);
            const uint32_t ab = sm_a + b * astride + koff;
            const uint32_t bb = sm_b + b * bstride + koff;
#pragma unroll
            for (int j = 0; j < kTcM / 32; j++) {  // A: 16 row units, 4 per warp
                const int u = warp + 4 * j;
#pragma unroll
                for (int h = 0; h < H; h++)
                    kern_unit<K, SPLIT, REC>(ab + u * kSBO + h * 512, kTcABytes, u * 8, pyh[h], jlo[h], jspan[h], a);
            }
            for (int u = warp; u < nbu; u += 4)  // B: N/8 column units
#pragma unroll
                for (int h = 0; h < H; h++)
                    kern_unit<K, SPLIT, REC>(bb + u * kSBO + h * 512, bbytes, u * 8, pxh[h], ilo[h], ispan[h], a);
            fence_async_smem();
            __syncthreads();
            if (t == kIssuer) {  // warp 3 generates the fewest B units
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 2 * H; kk++) {
                    const uint64_t ad = umma_desc(sm_a + b * astride + kk * 256, 128, kSBO);
                    const uint64_t bd = umma_desc(sm_b + b * bstride + kk * 256, 128, kSBO);
                    mma_f16(tmem, ad, bd, idesc, (ch > 0 || kk > 0) ? 1u : 0u);
                    if constexpr (SPLIT) {  // + A_hi B_lo + A_lo B_hi
                        mma_f16(tmem, ad, umma_desc(sm_b + b * bstride + bbytes + kk * 256, 128, kSBO), idesc, 1u);
                        mma_f16(tmem, umma_desc(sm_a + b * astride + kTcABytes + kk * 256, 128, kSBO), bd, idesc, 1u);
                    }
                }
                mma_commit(&s_bar[b]);
                if (ch == nch - 1) mma_commit(&s_bar[2]);
            }
            nuse[b]++;
        }
        // accumulator ready -> registers -> splat slot (warp w reads TMEM lanes 32w..32w+31)
        mbar_wait(&s_bar[2], nacc & 1);
        nacc++;
        tc_fence_after();
        {
            const int row = warp * 32 + lane;  // (slots of M = 64 plans hold rows < 64: the rest are zero)
            float* dst = a.splat + (size_t)it.w * slot_floats + (size_t)row * pg.slot_w;
            for (int c0 = 0; c0 < a.n; c0 += 16) {  // only the window's slot_w columns
                float v[16];
                tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
                for (int k = 0; k < 16; k += 4)
                    if (row < pg.slot_h && c0 + k < pg.slot_w)
                        *reinterpret_cast<float4*>(dst + c0 + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
            }
        }
        tc_fence_before();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
    }
}

template <int H, int K, bool SPLIT, bool REC>
static void launch_tc_h(kde_ctx* c, EvalPlan& pl, const TcArgs& a, cudaStream_t s) {
    const size_t smem =
        (SPLIT ? 2 : 1) * (2 * (size_t)TcShape<H>::kABytes + 2 * (size_t)a.n * TcShape<H>::kChunk * 2) + 1024;
    int& grid = SPLIT ? pl.grid_split : pl.grid;
    if (grid <= 0) {
        cudaFuncSetAttribute(tc_splat_kernel<H, K, SPLIT, REC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int nsm = 148, per = 0;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->p.device);
        const cudaError_t oe =
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tc_splat_kernel<H, K, SPLIT, REC>, kTcThreads, smem);
        if (getenv("KDE_DEBUG"))
            fprintf(stderr, "[kde] tc occupancy query: err=%d per=%d smem=%zu\n", (int)oe, per, smem);
        // (the occupancy API reports 1 CTA/SM for this kernel; size from the real limits:
        //  shared memory, registers, and TMEM columns below)
        if (oe != cudaSuccess) cudaGetLastError();
        per = std::max(per, std::min(TcShape<H>::kMinBlocks, (int)((200u << 10) / (smem + 2048))));
        // persistent CTAs hold their TMEM allocation for the whole launch: never
        // oversubscribe the 512 columns of an SM
        per = std::max(1, std::min(per, 512 / a.tmem_cols));
        grid = nsm * per;
    }
    cudaMemsetAsync(pl.d_totals + kTotQueue, 0, sizeof(int), s);  // work-queue head
    tmark(c, 3, s);
    tc_splat_kernel<H, K, SPLIT, REC><<<grid, kTcThreads, smem, s>>>(a);  // persistent; item count on device
}

int launch_tc(kde_ctx* c, float* out, cudaStream_t s, bool split) {
    EvalPlan& pl = c->plan[KDE_PATH_TENSOR];
    TcArgs a;
    a.g = c->g;
    a.pg = pl.pg;
    a.offsets = c->d_offsets;
    a.xy = c->pb.xy;
    a.rng = c->pb.rng;
    a.items = pl.d_items;
    a.group = pl.d_group;
    a.totals = pl.d_totals;
    a.splat = pl.d_splat;
    a.n = pl.pg.mma_n;
    a.tmem_cols = 32;
    while (a.tmem_cols < a.n) a.tmem_cols <<= 1;
    a.kq = (float)(-0.5 * 1.4426950408889634074 / (c->hpx * c->hpx));
    a.q2 = (float)exp2(2.0 * (double)a.kq);
    a.twoc = (float)(2.0 * cos(3.14159265358979323846 / (2.0 * c->hpx)));
    a.k = make_kconst(c->hpx);
    // chunk_pts is 32 (H = 1): 64-point chunks measured slower.  The Gaussian's
    // recurrence starts at a unit's first pixel, up to F + B + 7.5 px from the point: while
    // 2^(kq d^2) stays a normal float there it is exact-ratio; otherwise (small h with a
    // large cutoff) one exp2 per factor (REC = false).
    const double dmax = c->g.F + c->g.B + 8.0;
    const bool rec = -(double)a.kq * dmax * dmax < 120.0;
    using Fn = void (*)(kde_ctx*, EvalPlan&, const TcArgs&, cudaStream_t);
    static const Fn kLaunch[2][8] = {
        {launch_tc_h<1, 0, false, true>, launch_tc_h<1, 1, false, true>, launch_tc_h<1, 2, false, true>,
         launch_tc_h<1, 3, false, true>, launch_tc_h<1, 4, false, true>, launch_tc_h<1, 5, false, true>,
         launch_tc_h<1, 6, false, true>, launch_tc_h<1, 7, false, true>},
        {launch_tc_h<1, 0, true, true>, launch_tc_h<1, 1, true, true>, launch_tc_h<1, 2, true, true>,
         launch_tc_h<1, 3, true, true>, launch_tc_h<1, 4, true, true>, launch_tc_h<1, 5, true, true>,
         launch_tc_h<1, 6, true, true>, launch_tc_h<1, 7, true, true>}};
    cudaMemsetAsync(pl.d_totals + kTotChunksExec, 0, sizeof(int), s);  // set by eval_tc5.cu only
    const int rc5 = split ? KDE_EUNSUPPORTED : launch_tc5(c, s);  // eval_tc5.cu when it applies
    if (rc5 != KDE_OK && rc5 != KDE_EUNSUPPORTED) return rc5;
    c->main_kernel = rc5 == KDE_OK ? 3 : 2;
    if (rc5 == KDE_OK)
        ;
    else if (c->kern == KDE_GAUSSIAN && !rec)
        (split ? launch_tc_h<1, 6, true, false> : launch_tc_h<1, 6, false, false>)(c, pl, a, s);
    else
        kLaunch[split ? 1 : 0][c->kern](c, pl, a, s);
    c->launches += 1;
    tmark(c, 4, s);
    launch_combine(c, pl, out, s);
    tmark(c, 5, s);
    c->tev_eval = c->timing;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "tensor-core eval launch");
    return KDE_OK;
}

}  // namespace kde
