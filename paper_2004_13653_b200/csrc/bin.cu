// Steps a1/a2 of the hot path: fp64 convert + integer support
// ranges + bucket keys, a stable LSD counting sort of the keys, and the gather of the
// sorted points into bucket-local fp32 SoA.
//
// a1 follows Eqs. 5-6 in spirit -- each point is projected to raster
// coordinates -- but onto a fixed world grid (R5); the per-point count of
// Alg. 3 step 2 (atomicAdd into M_D) is replaced by a deterministic counting
// sort whose offsets are the exclusive scan of the bucket counts (the scan role of
// §IV-A-3).  Everything here is integer or fp64-RN work: bit-exact against
// oracle/kde_oracle.c:oracle_bin by construction of the written formulas (not code).
#include "internal.cuh"

namespace kde {

// ---------------------------------------------------------------------------------
// a1: one point -> (kept?, key, ranges, bucket-local coordinates).  Same fp64 RN
// operations in the same order as the documented formulas (kde.h).
struct Binned {
    int status;  // 0 non-finite, 1 finite but dropped, 2 kept
    uint32_t key;
    int ilo, ihi, jlo, jhi;
    float lx, ly;
};

// fp64 floor / ceil to int by the round-to-integer of an add to 1.5 * 2^52 (ulp 1 there):
// exact for |a| < 2^31, on the FP64 pipe instead of the XU pipe's F2I/FRND.
__device__ __forceinline__ int dfloor_i(double a) {
    return (int)(uint32_t)__double_as_longlong(__dadd_rd(a, 6755399441055744.0));
}
__device__ __forceinline__ int dceil_i(double a) {
    return (int)(uint32_t)__double_as_longlong(__dadd_ru(a, 6755399441055744.0));
}

__device__ __forceinline__ Binned bin_point(double x, double y, const Geom& g, uint32_t sentinel) {
    Binned b;
    b.key = sentinel;
    b.status = 0;
    b.ilo = b.ihi = b.jlo = b.jhi = 0;
    b.lx = b.ly = 0.f;
    if (!isfinite(x) || !isfinite(y)) return b;
    b.status = 1;
    const double u = __ddiv_rn(__dsub_rn(x, g.x0), g.res);
    const double v = __ddiv_rn(__dsub_rn(y, g.y0), g.res);
    const double ilo_a = __dsub_rn(__dsub_rn(u, 0.5), g.R), ihi_a = __dadd_rn(__dsub_rn(u, 0.5), g.R);
    const double jlo_a = __dsub_rn(__dsub_rn(v, 0.5), g.R), jhi_a = __dadd_rn(__dsub_rn(v, 0.5), g.R);
    int ilo, ihi, jlo, jhi, hx, hy;
    if (fabs(u) + g.R < 1073741824.0 && fabs(v) + g.R < 1073741824.0) {
        // |every rounded value| < 2^31: integer floor/ceil by the add-to-1.5*2^52 rounding
        // (the same values as ceil/floor of the same fp64 operands), clamps in integers
        ilo = max(dceil_i(ilo_a), 0);
        ihi = min(dfloor_i(ihi_a), g.W - 1);
        jlo = max(dceil_i(jlo_a), 0);
        jhi = min(dfloor_i(jhi_a), g.H - 1);
        if (ilo > ihi || jlo > jhi) return b;  // window misses the raster
        hx = min(max(dfloor_i(u), 0), g.W - 1);
        hy = min(max(dfloor_i(v), 0), g.H - 1);
    } else {  // far outside (or a huge support): the written fp64 formulas
        const double ilod = fmax(ceil(ilo_a), 0.0), ihid = fmin(floor(ihi_a), (double)(g.W - 1));
        const double jlod = fmax(ceil(jlo_a), 0.0), jhid = fmin(floor(jhi_a), (double)(g.H - 1));
        if (ilod > ihid || jlod > jhid) return b;  // window misses the raster
        ilo = (int)ilod;
        ihi = (int)ihid;
        jlo = (int)jlod;
        jhi = (int)jhid;
        const double fu = floor(u), fv = floor(v);
        hx = fu < 0.0 ? 0 : (fu > (double)(g.W - 1) ? g.W - 1 : (int)fu);
        hy = fv < 0.0 ? 0 : (fv > (double)(g.H - 1) ? g.H - 1 : (int)fv);
    }
    const int bx = hx >> g.lgB, by = hy >> g.lgB;  // B is a power of two
    if (by < g.band_lo || by > g.band_hi) return b;  // outside the band's reach
    b.status = 2;
    b.key = (uint32_t)(bx * g.nby + by);  // column-major: a vertical bucket stack is contiguous
    b.ilo = ilo;
    b.ihi = ihi;
    b.jlo = jlo;
    b.jhi = jhi;
    b.lx = __double2float_rn(__dsub_rn(u, (double)(bx * g.B)));
    b.ly = __double2float_rn(__dsub_rn(v, (double)(by * g.B)));
    return b;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------------------------
// a2 constants
constexpr int kRsThreads = 256;
constexpr int kRsMaxBits = 10;  // digits of <= 10 bits: <= 1025 digits per pass (incl. sentinel)
constexpr int kRsMaxDigits = 1025;
constexpr int kRsMaxPasses = 3;   // keys < 2^30
// A sort tile is kRsThreads x rounds keys, rounds = max(8, nbins / 64) rounded up to a
// power of two: tiles hold at least 4 keys per digit.
inline int rs_rounds(int nbins) {
    int r = 8;
    while (r * 64 + 64 < nbins) r *= 2;  // (a last digit set of 2^k + 1 keeps 2^k / 64)
    return r;
}

// the first tile of radix CTA c's range (os_pass_kernel)
__host__ __device__ inline int os_tile_begin(int c, int ntiles, int nctas) {
    return (int)(((int64_t)c * ntiles) / nctas);
}

// a1 kernel: each CTA converts (a part of) the contiguous range of whole sort tiles the
// first radix pass's CTA of the same index sorts.  Keys, the point's record (bucket-local
// fp32 coordinates + packed int16 ranges, read back by the gather), the integer stats (n_finite, n_outside, useful_pairs), and the GLOBAL histogram of every radix
// pass's digit (shared-memory counts, one global add per nonzero count per CTA): the
// radix passes take the digit offsets from these totals; the first pass's range histogram
// is this CTA's count of its digit.
__global__ void __launch_bounds__(kRsThreads, 4) bin_convert_kernel(
    const double* __restrict__ x, const double* __restrict__ y, int n, Geom g, uint32_t sentinel,
    uint32_t* __restrict__ key, uint4* __restrict__ rec, unsigned long long* __restrict__ stats, int passes,
    int dbits, uint32_t* __restrict__ ghist, int tile, int ntiles, uint32_t* __restrict__ rowhist0, int nbins0,
    int split) {
    constexpr int hpasses = 1;  // the first pass's digit totals (later passes total their own columns)
    __shared__ uint32_t h[kRsMaxDigits];
    for (int d = threadIdx.x; d < hpasses * kRsMaxDigits; d += kRsThreads) h[d] = 0;
    unsigned long long nf = 0, no = 0, up = 0;
    const int rb = g.rb, re = g.re;
    const uint32_t lmask = (1u << dbits) - 1u;
    // part blockIdx.x % split of the range of the first radix pass's CTA blockIdx.x / split
    // (os_pass_kernel): whole tiles
    const int pc = blockIdx.x / split, part = blockIdx.x % split, nc = gridDim.x / split;
    const int tb = os_tile_begin(pc, ntiles, nc), te = os_tile_begin(pc + 1, ntiles, nc);
    const int beg = (tb + (int)(((int64_t)part * (te - tb)) / split)) * tile;
    const int end = min(n, (tb + (int)(((int64_t)(part + 1) * (te - tb)) / split)) * tile);
    __syncthreads();
    constexpr int kHalf = 4;  // batches of loads-then-compute
    for (int b0 = beg + threadIdx.x; b0 < end; b0 += kHalf * kRsThreads) {
        double xv[kHalf], yv[kHalf];
#pragma unroll
        for (int r = 0; r < kHalf; r++) {
            const int i = b0 + r * kRsThreads;
            xv[r] = i < end ? x[i] : 0.0;
            yv[r] = i < end ? y[i] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < kHalf; r++) {
            const int i = b0 + r * kRsThreads;
            if (i >= end) break;
            const Binned b = bin_point(xv[r], yv[r], g, sentinel);
            key[i] = b.key;
            rec[i] = make_uint4(__float_as_uint(b.lx), __float_as_uint(b.ly),
                                ((uint32_t)b.ilo & 0xffffu) | ((uint32_t)b.ihi << 16),
                                ((uint32_t)b.jlo & 0xffffu) | ((uint32_t)b.jhi << 16));
            for (int ps = 0; ps < hpasses; ps++) {
                const uint32_t dg = b.key >> (ps * dbits);
                atomicAdd(&h[ps * kRsMaxDigits + (ps == passes - 1 ? dg : dg & lmask)], 1u);
            }
            nf += b.status > 0;
            no += b.status == 1;
            if (b.status == 2) {
                const int jl = max(b.jlo, rb), jh = min(b.jhi, re - 1);
                if (jh >= jl) up += (unsigned long long)(b.ihi - b.ilo + 1) * (unsigned long long)(jh - jl + 1);
            }
        }
    }
    __shared__ unsigned long long s[3][kRsThreads / 32];
    nf = warp_sum_u64(nf);
    no = warp_sum_u64(no);
    up = warp_sum_u64(up);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        s[0][w] = nf;
        s[1][w] = no;
        s[2][w] = up;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long t = 0;
        for (int k = 0; k < kRsThreads / 32; k++) t += s[threadIdx.x][k];
        if (t) atomicAdd(&stats[threadIdx.x], t);
    }
    for (int d = threadIdx.x; d < hpasses * kRsMaxDigits; d += kRsThreads)
        if (h[d]) atomicAdd(&ghist[d], h[d]);
    for (int d = threadIdx.x; d < nbins0; d += kRsThreads)  // the first pass's range histogram
        if (h[d]) atomicAdd(&rowhist0[(size_t)pc * nbins0 + d], h[d]);
}

// exclusive scan of a[0..nb) in shared memory, in place (all kRsThreads threads call it)
__device__ __forceinline__ void block_scan_smem(uint32_t* a, int nb, uint32_t* s_ws) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int per = (nb + kRsThreads - 1) / kRsThreads;  // consecutive entries per thread
    uint32_t tot = 0;
    for (int k = 0; k < per; k++) {
        const int d = t * per + k;
        if (d < nb) tot += a[d];
    }
    uint32_t inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) s_ws[warp] = inc;
    __syncthreads();
    uint32_t pre = inc - tot;
    for (int w = 0; w < warp; w++) pre += s_ws[w];
    for (int k = 0; k < per; k++) {
        const int d = t * per + k;
        if (d < nb) {
            const uint32_t v = a[d];
            a[d] = pre;
            pre += v;
        }
    }
    __syncthreads();
}

// per pass (one CTA each): the global digit totals -> their exclusive scan (the digit's
// first output position)
__global__ void __launch_bounds__(kRsThreads) os_scan_kernel(const uint32_t* __restrict__ ghist,
                                                            uint32_t* __restrict__ gofs, int dbits, int passes,
                                                            int nlast) {
    __shared__ uint32_t a[kRsMaxDigits];
    __shared__ uint32_t s_ws[kRsThreads / 32];
    const int ps = blockIdx.x;
    const int nb = ps == passes - 1 ? nlast : 1 << dbits;
    for (int d = threadIdx.x; d < nb; d += kRsThreads) a[d] = ghist[ps * kRsMaxDigits + d];
    __syncthreads();
    block_scan_smem(a, nb, s_ws);
    for (int d = threadIdx.x; d < nb; d += kRsThreads) gofs[ps * kRsMaxDigits + d] = a[d];
}

// ---------------------------------------------------------------------------------
// a2: stable LSD counting sort, ONE persistent cooperative kernel per pass.  Keys lie in
// [0, nb] (nb = dropped); passes = ceil(bits/10) with digits of ceil(bits/passes) <= 10
// bits, the LAST pass taking all the remaining high bits (its digit set (nb >> shift) + 1
// holds the sentinel).
//
// The C CTAs of a pass are all resident (cooperative launch); CTA c owns the contiguous
// tiles [c T / C, (c+1) T / C) of the keys, so the stable order is CTA order, then tile
// order, then position within the tile:
//   A. range histogram: the digit counts of the CTA's whole range -> rowhist[c][d] (for the
//      first pass the convert kernel, which walks the same ranges, has written them);
//   B. grid barrier; CTA c scans the columns d = c, c + C, ... over the C ranges (one warp per
//      column) -> colpre[c'][d] = count of digit d in the ranges before c'; grid barrier;
//   C. running offsets boff[d] = digit offset (the convert's global totals, scanned) +
//      colpre[c][d]; then per tile, with no inter-CTA traffic:
//      1. per round, warp match_any ranks equal digits among the lanes; a warp-private digit
//         counter (shared memory, uint16) orders the rounds -> rank of each key within its
//         warp's keys of that digit (warp w owns the contiguous sub-range
//         [w*32*ROUNDS, (w+1)*32*ROUNDS) of the tile; loads stay coalesced);
//      2. per digit, an exclusive scan of the 8 warp counters (warp order = index order)
//         -> the tile's digit counts -> their exclusive scan = tile-local run starts;
//      3. the tile is written digit-sorted into shared memory, then out coalesced, each run
//         to boff[d]; boff[d] += the tile's count.
// The result is the stable order (index order within equal digits), as the oracle's
// std::stable_sort-equivalent definition requires.
struct OsArgs {
    const uint32_t* kin;   // first pass: the keys (values = input positions)
    const uint2* pin;      // later passes: (key, value) pairs
    uint2* pout;           // (key, value) pairs, sorted by this pass's digit
    int n, shift, nbins, ntiles, nctas;
    uint32_t dmask;
    const uint32_t* gofs;  // [nbins] exclusive scan of the digit totals (first pass)
    uint32_t* dtot;        // [nbins] later passes: the digit totals, from the column scans
    uint32_t* rowhist;     // [nctas][nbins] range histograms
    uint32_t* colpre;      // [nctas][nbins] their column-wise exclusive scans
    uint32_t* bar;         // grid-barrier arrival counter (zero at launch)
};

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

// mbarrier + 1-D TMA (cp.async.bulk) for the radix passes' tile prefetch
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void os_mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n\tfence.mbarrier_init.release.cluster;" ::"r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void os_mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0, polls = 0;
    for (;;) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (++polls > (1u << 26)) __trap();  // a copy that never lands is a bug: fail, don't hang
    }
}
// bytes (multiple of 16, 16-byte aligned ends) global -> shared, completing on bar
__device__ __forceinline__ void os_tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void os_mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

// all CTAs of a cooperative launch: every thread's prior global writes are visible to
// every CTA after the call (the k-th barrier of the launch waits for k * gridDim.x arrivals)
__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        uint32_t polls = 0;
        while (ld_volatile(bar) < target) {  // (all CTAs are resident: a hang is a bug -> trap)
            __nanosleep(64);
            if (++polls > (1u << 26)) __trap();
        }
        __threadfence();
    }
    __syncthreads();
}

template <int ROUNDS, bool UPSWEEP>
__global__ void __launch_bounds__(kRsThreads, ROUNDS >= 16 ? 2 : 3) os_pass_kernel(OsArgs a) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ uint32_t s_ws[kRsThreads / 32];
    __shared__ __align__(8) uint64_t s_bar;  // the prefetched tile has landed
    constexpr int kW = kRsThreads / 32;
    constexpr int tile = kRsThreads * ROUNDS;
    const int nbins = a.nbins, shift = a.shift, n = a.n;
    const uint32_t dmask = a.dmask;
    uint2* pre = reinterpret_cast<uint2*>(sm);            // [tile] the next tile (TMA): pairs, or keys
    uint2* spair = pre + tile;                            // [tile] the tile, digit-sorted
    uint32_t* boff = reinterpret_cast<uint32_t*>(spair + tile);  // [nbins] running global base
    uint32_t* dstart = boff + nbins;                      // [nbins] tile count -> tile-local run start
    uint16_t* wcnt = reinterpret_cast<uint16_t*>(dstart + nbins);  // [kW][nbins]
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int c = blockIdx.x, C = a.nctas;
    const int tb = os_tile_begin(c, a.ntiles, C), te = os_tile_begin(c + 1, a.ntiles, C);
    // A. the range histogram (the keys are the pairs' first words)
    if (UPSWEEP) {
        for (int d = t; d < nbins; d += kRsThreads) boff[d] = 0u;
        __syncthreads();
        const int i0 = tb * tile, i1 = min(n, te * tile);  // i0 even
        constexpr int kU = 4;                              // 16-byte loads (2 pairs) in flight per thread
        for (int i = i0 + 2 * t; i < i1; i += 2 * kU * kRsThreads) {
            uint4 p4[kU];
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const int j = i + u * 2 * kRsThreads;
                p4[u] = j + 1 < i1 ? __ldcg(reinterpret_cast<const uint4*>(a.pin + j)) : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const int j = i + u * 2 * kRsThreads;
                if (j + 1 < i1) {
                    atomicAdd(&boff[(p4[u].x >> shift) & dmask], 1u);
                    atomicAdd(&boff[(p4[u].z >> shift) & dmask], 1u);
                } else if (j < i1) {
                    atomicAdd(&boff[(a.pin[j].x >> shift) & dmask], 1u);
                }
            }
        }
        __syncthreads();
        for (int d = t; d < nbins; d += kRsThreads) a.rowhist[(size_t)c * nbins + d] = boff[d];
    }
    // B. column scans over the ranges, between two grid barriers
    grid_barrier(a.bar, (uint32_t)C);
    for (int d = c + warp * C; d < nbins; d += kW * C) {
        const int per = (C + 31) / 32;  // consecutive ranges per lane
        uint32_t tot = 0;
        for (int k = 0; k < per; k++) {
            const int r = lane * per + k;
            if (r < C) tot += __ldcg(a.rowhist + (size_t)r * nbins + d);
        }
        uint32_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        if (UPSWEEP && lane == 31) a.dtot[d] = inc;  // the digit's total over all ranges
        uint32_t pre_ = inc - tot;
        for (int k = 0; k < per; k++) {
            const int r = lane * per + k;
            if (r < C) {
                const uint32_t v = __ldcg(a.rowhist + (size_t)r * nbins + d);
                a.colpre[(size_t)r * nbins + d] = pre_;
                pre_ += v;
            }
        }
    }
    grid_barrier(a.bar, 2u * (uint32_t)C);
    // C. the range's tiles in order, from running offsets = the digit's first position (the
    // first pass: the convert's totals, scanned; later passes: the column totals of phase B,
    // scanned here) + the column prefix of this range
    if (UPSWEEP) {
        for (int d = t; d < nbins; d += kRsThreads) boff[d] = __ldcg(a.dtot + d);
        __syncthreads();
        block_scan_smem(boff, nbins, s_ws);
        for (int d = t; d < nbins; d += kRsThreads) boff[d] += __ldcg(a.colpre + (size_t)c * nbins + d);
    } else {
        for (int d = t; d < nbins; d += kRsThreads) boff[d] = a.gofs[d] + __ldcg(a.colpre + (size_t)c * nbins + d);
    }
    uint16_t* my = wcnt + warp * nbins;
    const uint32_t lt = (1u << lane) - 1u;
    const bool pairs_in = a.pin != nullptr;
    // tile b (keys, or pairs) streams into `pre` by TMA while tile b - 1 is ranked
    auto prefetch = [&](int b) {  // (thread 0)
        const int cnt = min(tile, n - b * tile);
        const uint32_t bytes = (uint32_t)((cnt * (pairs_in ? 8 : 4) + 15) & ~15);  // (+ slack in the buffers)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the generic reads
        os_mbar_expect(&s_bar, bytes);
        if (pairs_in) os_tma_load(pre, a.pin + (size_t)b * tile, bytes, &s_bar);
        else os_tma_load(pre, a.kin + (size_t)b * tile, bytes, &s_bar);
    };
    if (t == 0) {
        os_mbar_init(&s_bar);
        if (tb < te) prefetch(tb);
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    for (int b = tb; b < te; b++) {
        for (int e = t; e < kW * nbins; e += kRsThreads) wcnt[e] = 0;
        const int wbase = b * tile + warp * 32 * ROUNDS + lane;
        const int lbase = warp * 32 * ROUNDS + lane;
        uint32_t kb[ROUNDS], vb[ROUNDS], rk[ROUNDS];
        os_mbar_wait(&s_bar, (uint32_t)(b - tb) & 1u);
        if (pairs_in) {
#pragma unroll
            for (int r = 0; r < ROUNDS; r++) {
                const uint2 pr = pre[lbase + r * 32];
                kb[r] = pr.x;
                vb[r] = pr.y;
            }
        } else {
            const uint32_t* pk = reinterpret_cast<const uint32_t*>(pre);
#pragma unroll
            for (int r = 0; r < ROUNDS; r++) {
                kb[r] = pk[lbase + r * 32];
                vb[r] = (uint32_t)(wbase + r * 32);
            }
        }
        // the lanes holding each key's digit in its round: independent of the counters
#pragma unroll
        for (int r = 0; r < ROUNDS; r++) {
            const bool valid = wbase + r * 32 < n;
            const uint32_t d = valid ? ((kb[r] >> shift) & dmask) : (0x10000u + lane);  // unique if invalid
            rk[r] = __match_any_sync(0xffffffffu, d);
        }
        __syncthreads();  // wcnt zeroed; the previous tile's staging read out; `pre` read
        if (t == 0 && b + 1 < te) prefetch(b + 1);
        // the warp's counters, round by round: rank = counter + earlier peers in the round
#pragma unroll
        for (int r = 0; r < ROUNDS; r++) {
            const bool valid = wbase + r * 32 < n;
            const uint32_t d = (kb[r] >> shift) & dmask;
            const uint32_t peers = rk[r];
            const uint32_t pre_ = valid ? (uint32_t)my[d] : 0u;
            rk[r] = pre_ + __popc(peers & lt);
            __syncwarp();
            if (valid && (peers & lt) == 0) my[d] = (uint16_t)(pre_ + __popc(peers));
            __syncwarp();
        }
        __syncthreads();
        for (int d = t; d < nbins; d += kRsThreads) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kW; w++) {
                const uint32_t cnt = wcnt[w * nbins + d];
                wcnt[w * nbins + d] = (uint16_t)run;
                run += cnt;
            }
            dstart[d] = run;
        }
        __syncthreads();
        block_scan_smem(dstart, nbins, s_ws);
#pragma unroll
        for (int r = 0; r < ROUNDS; r++) {
            if (wbase + r * 32 >= n) break;
            const uint32_t d = (kb[r] >> shift) & dmask;
            spair[dstart[d] + (uint32_t)my[d] + rk[r]] = make_uint2(kb[r], vb[r]);
        }
        __syncthreads();
        const int cnt = min(tile, n - b * tile);
        for (int e = t; e < cnt; e += kRsThreads) {
            const uint2 pr = spair[e];
            const uint32_t d = (pr.x >> shift) & dmask;
            a.pout[boff[d] + (uint32_t)e - dstart[d]] = pr;
        }
        __syncthreads();
        for (int d = t; d < nbins; d += kRsThreads)  // + the tile's count of d
            boff[d] += (d + 1 < nbins ? dstart[d + 1] : (uint32_t)cnt) - dstart[d];
    }
}

// Exclusive scan of one row of counts in place + its total (band compaction's block
// offsets), one CTA: coalesced uint4 loads of 1024 entries per step, a block scan, a carry.
__global__ void __launch_bounds__(256) rs_scan_digits(uint32_t* __restrict__ hist, int nbins, int ntiles,
                                                      int stride, uint32_t* __restrict__ dtot) {
    __shared__ uint32_t s_ws[8];
    const int d = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t* row = hist + (size_t)d * stride;
    uint32_t carry = 0;
    for (int base = 0; base < ntiles; base += 1024) {
        const int i = base + 4 * t;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (i + 3 < ntiles) {
            v = *reinterpret_cast<const uint4*>(row + i);
        } else {
            if (i < ntiles) v.x = row[i];
            if (i + 1 < ntiles) v.y = row[i + 1];
            if (i + 2 < ntiles) v.z = row[i + 2];
        }
        const uint32_t sum = v.x + v.y + v.z + v.w;
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) s_ws[warp] = inc;
        __syncthreads();
        uint32_t pre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) {
            const uint32_t x = s_ws[w];
            pre += w < warp ? x : 0u;
            tot += x;
        }
        __syncthreads();  // s_ws is rewritten by the next step
        uint4 o;
        o.x = carry + pre + inc - sum;
        o.y = o.x + v.x;
        o.z = o.y + v.y;
        o.w = o.z + v.z;
        if (i + 3 < ntiles) {
            *reinterpret_cast<uint4*>(row + i) = o;
        } else {
            if (i < ntiles) row[i] = o.x;
            if (i + 1 < ntiles) row[i + 1] = o.y;
            if (i + 2 < ntiles) row[i + 2] = o.z;
        }
        carry += tot;
    }
    if (t == 0) dtot[d] = carry;
    (void)nbins;
}

// a2 gather + bucket offsets, one pass over the sorted keys.  Position d in [0, n]:
//   offsets: offsets[b] = first position with key >= b -- the thread of position d writes the
//            buckets (key[d-1], key[d]] (empty buckets take the next occupied bucket's start;
//            long runs of empty buckets are written by the whole warp);
//   gather:  a kept point (key < nb) at sorted position d gets its bucket-local fp32 SoA and
//            packed int16 ranges from the record the convert kernel wrote in input order
//            (measured: recomputing them from the fp64 coordinates instead is slower).
// Kept keys (< nb) sort before the dropped sentinel nb, so positions [0, n_binned) are the
// binned points.
__global__ void __launch_bounds__(256) gather_offsets_kernel(const uint4* __restrict__ rec,
                                                             const uint2* __restrict__ sp, int n, uint32_t nb,
                                                             uint32_t* __restrict__ offsets,
                                                             float2* __restrict__ xy, uint2* __restrict__ rng) {
    const int lane = threadIdx.x & 31;
    constexpr int U = 4;
    const int tile = blockDim.x * U;
    for (int d0 = blockIdx.x * tile; d0 <= n; d0 += gridDim.x * tile) {  // warp-uniform trip count
        uint32_t kc[U], kp[U], q[U];
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int d = d0 + u * blockDim.x + (threadIdx.x & ~31) + lane;
            const uint2 pc = d < n ? sp[d] : make_uint2(nb, 0u);
            kc[u] = pc.x;
            kp[u] = (d > 0 && d <= n) ? sp[d - 1].x : 0xffffffffu;
            q[u] = (d < n && kc[u] < nb) ? pc.y : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int d = d0 + u * blockDim.x + (threadIdx.x & ~31) + lane;
            r[u] = (d < n && kc[u] < nb) ? rec[q[u]] : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int d = d0 + u * blockDim.x + (threadIdx.x & ~31) + lane;
            int64_t lo = 0, hi = -1;  // buckets [lo, hi] take position d
            if (d <= n) {
                lo = (d > 0 ? (int64_t)kp[u] : -1) + 1;
                hi = d < n ? (int64_t)min(kc[u], nb) : (int64_t)nb;
            }
            const bool big = hi - lo >= 8;
            if (!big)
                for (int64_t b = lo; b <= hi; b++) offsets[b] = (uint32_t)d;
            uint32_t m = __ballot_sync(0xffffffffu, big);
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const int64_t s0 = __shfl_sync(0xffffffffu, lo, src), s1 = __shfl_sync(0xffffffffu, hi, src);
                const int dv = __shfl_sync(0xffffffffu, d, src);
                for (int64_t b = s0 + lane; b <= s1; b += 32) offsets[b] = (uint32_t)dv;
            }
            if (d < n && kc[u] < nb) {
                xy[d] = make_float2(__uint_as_float(r[u].x), __uint_as_float(r[u].y));
                rng[d] = make_uint2(r[u].z, r[u].w);
            }
        }
    }
}

// ---------------------------------------------------------------------------------
// Banded contexts (row-band sharding): only the points whose home-bucket row is
// within the band's reach are binned.  They are compacted IN INPUT ORDER before the sort
// (per-block counts -> scan -> write), so a rank sorts ~n/P + halo keys instead of all n, and
// the sort's stability still orders equal keys by original index (the values carried through
// the sort are compacted positions; cidx maps them back).
constexpr int kBcThreads = 256, kBcPer = 4, kBcTile = kBcThreads * kBcPer;

// the band filter: finite, and the home-bucket row (bin_point's fp64 v, the same RN
// operations) within the band's kept rows.  Points that pass but miss the raster are
// dropped by the convert kernel as usual.
__device__ __forceinline__ int band_status(double x, double y, const Geom& g) {
    if (!isfinite(x) || !isfinite(y)) return 0;
    const double v = __ddiv_rn(__dsub_rn(y, g.y0), g.res);
    const double fv = floor(v);
    const int hy = fv < 0.0 ? 0 : (fv > (double)(g.H - 1) ? g.H - 1 : (int)fv);
    const int by = hy >> g.lgB;
    return (by < g.band_lo || by > g.band_hi) ? 1 : 2;
}

__global__ void __launch_bounds__(kBcThreads) band_count_kernel(const double* __restrict__ x,
                                                                const double* __restrict__ y, int n, Geom g,
                                                                uint32_t* __restrict__ bcnt,
                                                                unsigned long long* __restrict__ nfin) {
    __shared__ uint32_t s_k[kBcThreads / 32], s_f[kBcThreads / 32];
    uint32_t kept = 0, fin = 0;
#pragma unroll
    for (int r = 0; r < kBcPer; r++) {
        const int i = blockIdx.x * kBcTile + r * kBcThreads + threadIdx.x;
        if (i < n) {
            const int st = band_status(x[i], y[i], g);
            kept += st == 2;
            fin += st > 0;
        }
    }
    kept = __reduce_add_sync(0xffffffffu, kept);
    fin = __reduce_add_sync(0xffffffffu, fin);
    if ((threadIdx.x & 31) == 0) {
        s_k[threadIdx.x >> 5] = kept;
        s_f[threadIdx.x >> 5] = fin;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t k = 0, f = 0;
        for (int w = 0; w < kBcThreads / 32; w++) {
            k += s_k[w];
            f += s_f[w];
        }
        bcnt[blockIdx.x] = k;
        if (f) atomicAdd(nfin, (unsigned long long)f);
    }
}

__global__ void __launch_bounds__(kBcThreads) band_compact_kernel(const double* __restrict__ x,
                                                                  const double* __restrict__ y, int n, Geom g,
                                                                  const uint32_t* __restrict__ boff,
                                                                  double* __restrict__ cx, double* __restrict__ cy,
                                                                  uint32_t* __restrict__ cidx) {
    __shared__ uint32_t s_w[kBcThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t base = boff[blockIdx.x];
#pragma unroll
    for (int r = 0; r < kBcPer; r++) {  // rounds in input order; within a round, warp order
        const int i = blockIdx.x * kBcTile + r * kBcThreads + threadIdx.x;
        double xv = 0.0, yv = 0.0;
        bool keep = false;
        if (i < n) {
            xv = x[i];
            yv = y[i];
            keep = band_status(xv, yv, g) == 2;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_w[warp] = __popc(m);
        __syncthreads();
        uint32_t pre = 0, tot = 0;
        for (int w = 0; w < kBcThreads / 32; w++) {
            pre += w < warp ? s_w[w] : 0u;
            tot += s_w[w];
        }
        if (keep) {
            const uint32_t o = base + pre + __popc(m & ((1u << lane) - 1u));
            cx[o] = xv;
            cy[o] = yv;
            cidx[o] = (uint32_t)i;
        }
        base += tot;
        __syncthreads();
    }
}

// after binning a compacted set: n_finite counts every finite point passed in (the
// normalisation, R4), n_outside the finite ones not binned
__global__ void band_stats_kernel(unsigned long long* __restrict__ stats, const unsigned long long* __restrict__ nfin,
                                  const uint32_t* __restrict__ binned) {
    stats[0] = *nfin;
    stats[1] = *nfin - (unsigned long long)*binned;
}

static int grow(void** p, size_t bytes) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    const cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
    if (e != cudaSuccess) {
        set_error("cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
        cudaGetLastError();
        return KDE_ENOMEM;
    }
    return KDE_OK;
}

static int bin_sorted(kde_ctx* c, const double* d_x, const double* d_y, int n);

int bin_points(kde_ctx* c, const double* d_x, const double* d_y, int64_t n64) {
    const int n = (int)n64;
    PointBufs& pb = c->pb;
    const Geom& g = c->g;
    const bool banded = g.band_lo > 0 || g.band_hi < g.nby - 1;
    pb.compacted = false;
    if (!banded || n == 0) return bin_sorted(c, d_x, d_y, n);
    cudaStream_t s = c->stream;
    const int nbk = (n + kBcTile - 1) / kBcTile;
    if (n64 > pb.ccap) {
        int rc = KDE_OK;
        rc |= grow((void**)&pb.cx, sizeof(double) * n64);
        rc |= grow((void**)&pb.cy, sizeof(double) * n64);
        rc |= grow((void**)&pb.cidx, sizeof(uint32_t) * n64);
        if (rc) return KDE_ENOMEM;
        pb.ccap = n64;
    }
    if (nbk + 8 > pb.bcap) {
        if (grow((void**)&pb.bcnt, sizeof(uint32_t) * ((nbk + 8 + 3) & ~3))) return KDE_ENOMEM;
        if (!pb.nfin && grow((void**)&pb.nfin, sizeof(unsigned long long) * 2)) return KDE_ENOMEM;
        pb.bcap = nbk + 8;
    }
    if (!pb.scan_tmp && grow((void**)&pb.scan_tmp, sizeof(uint32_t) * 4096)) return KDE_ENOMEM;
    cudaMemsetAsync(pb.nfin, 0, sizeof(unsigned long long), s);
    band_count_kernel<<<nbk, kBcThreads, 0, s>>>(d_x, d_y, n, g, pb.bcnt, pb.nfin);
    rs_scan_digits<<<1, 256, 0, s>>>(pb.bcnt, 1, nbk, nbk, pb.scan_tmp);  // one row: block offsets; total = m
    band_compact_kernel<<<nbk, kBcThreads, 0, s>>>(d_x, d_y, n, g, pb.bcnt, pb.cx, pb.cy, pb.cidx);
    c->launches += 3;
    uint32_t m = 0;  // the kept count sizes the sort: one readback per banded load
    cudaError_t e = cudaMemcpyAsync(c->h_totals + 28, pb.scan_tmp, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(c->h_totals + 30, pb.nfin, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "band compaction");
    m = (uint32_t)c->h_totals[28];
    c->plan_n = (int64_t)*reinterpret_cast<const unsigned long long*>(c->h_totals + 30);
    const int rc = bin_sorted(c, pb.cx, pb.cy, (int)m);  // sorts compacted positions (cidx: originals)
    if (rc) return rc;
    band_stats_kernel<<<1, 1, 0, s>>>(c->d_stats, pb.nfin, c->d_offsets + (size_t)g.nbx * g.nby);
    c->launches += 1;
    pb.compacted = true;
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "band compaction launch");
    return KDE_OK;
}

// a1/a2 over n points (the sort carries each point's position in d_x / d_y)
static int bin_sorted(kde_ctx* c, const double* d_x, const double* d_y, int n) {
    const int64_t n64 = n;
    PointBufs& pb = c->pb;
    const Geom& g = c->g;
    cudaStream_t s = c->stream;
    const uint32_t nb = (uint32_t)g.nbx * (uint32_t)g.nby;
    // LSD passes over the keys [0, nb] (nb = dropped).  The real keys [0, nb) need kb bits;
    // passes = ceil(kb / 10), digits of db = ceil(kb / passes) bits, and the LAST pass takes
    // all the remaining high bits, key >> shift in [0, nb >> shift] -- a digit set of
    // (nb >> shift) + 1 that holds the dropped sentinel without an extra pass (C4: 2^20
    // buckets -> 1024 + 1025 digits, two passes instead of three).
    int kb = 1;
    while ((1ull << kb) < nb) kb++;
    const int passes = (kb + kRsMaxBits - 1) / kRsMaxBits;
    const int dbits = (kb + passes - 1) / passes;
    if (passes > kRsMaxPasses || n64 >= (1ll << 30)) {
        set_error("binning: %d key bits / %lld points not supported", kb, (long long)n64);
        return KDE_EUNSUPPORTED;
    }
    auto pass_bins = [&](int ps) {
        return ps == passes - 1 ? (int)(nb >> (ps * dbits)) + 1 : 1 << dbits;
    };
    auto pass_mask = [&](int ps) { return ps == passes - 1 ? 0xffffffffu : (1u << dbits) - 1u; };
    int nbins = 0;  // the largest digit set
    for (int ps = 0; ps < passes; ps++) nbins = std::max(nbins, pass_bins(ps));
    // tuning knob (A/B experiments): KDE_RS_ROUNDS = 8|16 forces the tile rounds.  Default:
    // 4096-key tiles from 8 M points on (C2 prefers 2048-key tiles: more CTAs for its 2 M
    // keys); tiles hold >= 4 keys per digit
    static const int env_rounds = getenv("KDE_RS_ROUNDS") ? atoi(getenv("KDE_RS_ROUNDS")) : 0;
    const int rounds = (env_rounds == 8 || env_rounds == 16) ? std::max(env_rounds, rs_rounds(nbins))
                       : (n >= (8 << 20) ? std::max(16, rs_rounds(nbins)) : rs_rounds(nbins));
    if (rounds != 8 && rounds != 16) {
        set_error("binning: %d digits per pass not supported", nbins);
        return KDE_EUNSUPPORTED;
    }
    const int tile = kRsThreads * rounds;
    const int nblk = (n + tile - 1) / tile;
    if (n64 > pb.cap || pb.key[0] == nullptr) {
        const int64_t cap = n64 > 1024 ? n64 : 1024;
        int rc = KDE_OK;
        rc |= grow((void**)&pb.key[0], sizeof(uint32_t) * (cap + 4));  // + TMA tail slack
        rc |= grow((void**)&pb.pair[0], sizeof(uint2) * (cap + 2));
        rc |= grow((void**)&pb.pair[1], sizeof(uint2) * (cap + 2));
        rc |= grow((void**)&pb.xy, sizeof(float2) * cap);
        rc |= grow((void**)&pb.rng, sizeof(uint2) * cap);
        rc |= grow((void**)&pb.rec, sizeof(uint4) * cap);
        if (rc) return KDE_ENOMEM;
        pb.cap = cap;
    }
    // hist: [1025] first-pass digit totals, [1025] their scan, [passes][1025] later passes'
    // totals (column scans), a grid-barrier counter per pass
    constexpr int kHistWords = (2 + kRsMaxPasses) * kRsMaxDigits + kRsMaxPasses + 1;
    if (!pb.hist && grow((void**)&pb.hist, sizeof(uint32_t) * kHistWords)) return KDE_ENOMEM;
    uint32_t* ghist = pb.hist;
    uint32_t* gofs = pb.hist + kRsMaxDigits;  // then the later passes' totals (OsArgs::dtot)
    uint32_t* bars = pb.hist + (2 + kRsMaxPasses) * kRsMaxDigits;
    // the passes' CTA count: every CTA resident (cooperative launch), at most one per tile
    const size_t dsmem = sizeof(uint2) * 2 * tile + sizeof(uint32_t) * 2 * nbins + sizeof(uint16_t) * 8 * nbins;
    auto k_first = rounds == 8 ? os_pass_kernel<8, false> : os_pass_kernel<16, false>;
    auto k_next = rounds == 8 ? os_pass_kernel<8, true> : os_pass_kernel<16, true>;
    int nsm = 148, occ0 = 0, occ1 = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->p.device);
    // the shared-memory opt-in is per device and cheap: set it on every load (no
    // process-global state)
    cudaFuncSetAttribute(k_first, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
    cudaFuncSetAttribute(k_next, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, k_first, kRsThreads, dsmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k_next, kRsThreads, dsmem);
    const int nctas = std::max(1, std::min(nblk, nsm * std::min(occ0, occ1)));
    if (std::min(occ0, occ1) < 1) {
        set_error("binning: radix pass kernel does not fit an SM");
        return KDE_EUNSUPPORTED;
    }
    const int64_t sneed = (int64_t)nctas * nbins;  // range histograms / column scans
    if (sneed > pb.ost_cap) {
        const int64_t cap = std::max<int64_t>(sneed, (int64_t)nsm * 3 * kRsMaxDigits);
        for (int k = 0; k < 2; k++)
            if (grow((void**)&pb.ost[k], sizeof(uint32_t) * cap)) return KDE_ENOMEM;
        pb.ost_cap = cap;
    }
    cudaMemsetAsync(c->d_stats, 0, 3 * sizeof(unsigned long long), s);
    if (n > 0) {
        cudaMemsetAsync(ghist, 0, sizeof(uint32_t) * kRsMaxDigits, s);
        cudaMemsetAsync(bars, 0, sizeof(uint32_t) * kRsMaxPasses, s);
        // the convert: each pass-0 range cut into `split` parts (~4 CTAs per SM), the parts'
        // digit counts added into the range histogram
        const int split = std::max(1, std::min(4, (nsm * 4) / nctas));
        cudaMemsetAsync(pb.ost[0], 0, sizeof(uint32_t) * (size_t)nctas * pass_bins(0), s);
        bin_convert_kernel<<<nctas * split, kRsThreads, 0, s>>>(d_x, d_y, n, g, nb, pb.key[0], pb.rec, c->d_stats,
                                                                passes, dbits, ghist, tile, nblk, pb.ost[0],
                                                                pass_bins(0), split);
        os_scan_kernel<<<1, kRsThreads, 0, s>>>(ghist, gofs, dbits, passes, pass_bins(passes - 1));  // pass 0's
        c->launches += 2;
        int cur = 0;
        for (int ps = 0; ps < passes; ps++) {
            OsArgs oa;
            oa.kin = ps == 0 ? pb.key[0] : nullptr;
            oa.pin = ps == 0 ? nullptr : pb.pair[cur];
            if (ps > 0) cur ^= 1;
            oa.pout = pb.pair[cur];
            oa.n = n;
            oa.shift = ps * dbits;
            oa.nbins = pass_bins(ps);
            oa.ntiles = nblk;
            oa.nctas = nctas;
            oa.dmask = pass_mask(ps);
            oa.gofs = gofs;                             // pass 0: the convert's totals, scanned
            oa.dtot = gofs + (1 + ps) * kRsMaxDigits;  // later passes (ps >= 1): their column totals
            oa.rowhist = pb.ost[0];
            oa.colpre = pb.ost[1];
            oa.bar = bars + ps;
            void* args[] = {&oa};
            const cudaError_t le = cudaLaunchCooperativeKernel((const void*)(ps == 0 ? k_first : k_next), dim3(nctas),
                                                               dim3(kRsThreads), args, dsmem, s);
            if (le != cudaSuccess) return cuda_fail(le, "radix pass (cooperative launch)");
            c->launches += 1;
        }
        pb.sorted = pb.pair[cur];
        const int gg = (n + 1 + 1023) / 1024 < 148 * 8 ? (n + 1 + 1023) / 1024 : 148 * 8;
        gather_offsets_kernel<<<gg, 256, 0, s>>>(pb.rec, pb.sorted, n, nb, c->d_offsets, pb.xy, pb.rng);
        c->launches += 1;
    } else {
        cudaMemsetAsync(c->d_offsets, 0, sizeof(uint32_t) * (nb + 1), s);
        pb.sorted = pb.pair[0];
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "binning launch");
    return KDE_OK;
}

}  // namespace kde
