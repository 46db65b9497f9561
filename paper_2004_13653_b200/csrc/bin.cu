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
    double ilo = ceil(__dsub_rn(__dsub_rn(u, 0.5), g.R));
    double ihi = floor(__dadd_rn(__dsub_rn(u, 0.5), g.R));
    double jlo = ceil(__dsub_rn(__dsub_rn(v, 0.5), g.R));
    double jhi = floor(__dadd_rn(__dsub_rn(v, 0.5), g.R));
    ilo = fmax(ilo, 0.0);
    ihi = fmin(ihi, (double)(g.W - 1));
    jlo = fmax(jlo, 0.0);
    jhi = fmin(jhi, (double)(g.H - 1));
    if (ilo > ihi || jlo > jhi) return b;  // window misses the raster
    const double fu = floor(u), fv = floor(v);
    const int hx = fu < 0.0 ? 0 : (fu > (double)(g.W - 1) ? g.W - 1 : (int)fu);
    const int hy = fv < 0.0 ? 0 : (fv > (double)(g.H - 1) ? g.H - 1 : (int)fv);
    const int bx = hx >> g.lgB, by = hy >> g.lgB;  // B is a power of two
    if (by < g.band_lo || by > g.band_hi) return b;  // outside the band's reach
    b.status = 2;
    b.key = (uint32_t)(bx * g.nby + by);  // column-major: a vertical bucket stack is contiguous
    b.ilo = (int)ilo;
    b.ihi = (int)ihi;
    b.jlo = (int)jlo;
    b.jhi = (int)jhi;
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
// a2 constants (the convert kernel below already works in sort tiles)
constexpr int kRsThreads = 256;
constexpr int kRsMaxBits = 10;  // (11-bit digits need 8192-key tiles in registers: slower at C5)
// A sort tile is kRsThreads x rounds keys, rounds = max(8, nbins / 64) rounded up to a
// power of two: tiles hold at least 4 keys per digit, so the per-tile histograms stay <= 1/4
// of the keys.
inline int rs_rounds(int nbins) {
    int r = 8;
    while (r * 64 + 64 < nbins) r *= 2;  // (a last digit set of 2^k + 1 keeps 2^k / 64)
    return r;
}

// a1 kernel, one sort tile (kRsThreads x rounds points) per CTA: keys, the point's record (bucket-
// local fp32 coordinates + packed int16 ranges, read back by the gather), the integer
// stats (n_finite, n_outside, useful_pairs) and the tile's histogram of the first radix
// digit (the first pass's upsweep, fused).
__global__ void __launch_bounds__(kRsThreads, 4) bin_convert_kernel(
    const double* __restrict__ x, const double* __restrict__ y, int n, Geom g, uint32_t sentinel,
    uint32_t* __restrict__ key, uint4* __restrict__ rec, unsigned long long* __restrict__ stats,
    uint32_t dmask, int nbins, uint32_t* __restrict__ hist, int hstride, int rounds) {
    extern __shared__ uint32_t h[];  // [nbins]
    for (int d = threadIdx.x; d < nbins; d += kRsThreads) h[d] = 0;
    unsigned long long nf = 0, no = 0, up = 0;
    const int rb = g.rb, re = g.re;
    const int base = blockIdx.x * kRsThreads * rounds + threadIdx.x;
    __syncthreads();
    constexpr int kHalf = 4;  // batches of loads-then-compute
    for (int hb = 0; hb < rounds / kHalf; hb++) {
        double xv[kHalf], yv[kHalf];
#pragma unroll
        for (int r = 0; r < kHalf; r++) {
            const int i = base + (hb * kHalf + r) * kRsThreads;
            xv[r] = i < n ? x[i] : 0.0;
            yv[r] = i < n ? y[i] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < kHalf; r++) {
            const int i = base + (hb * kHalf + r) * kRsThreads;
            if (i >= n) break;
            const Binned b = bin_point(xv[r], yv[r], g, sentinel);
            key[i] = b.key;
            rec[i] = make_uint4(__float_as_uint(b.lx), __float_as_uint(b.ly),
                                ((uint32_t)b.ilo & 0xffffu) | ((uint32_t)b.ihi << 16),
                                ((uint32_t)b.jlo & 0xffffu) | ((uint32_t)b.jhi << 16));
            atomicAdd(&h[b.key & dmask], 1u);
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
    for (int d = threadIdx.x; d < nbins; d += kRsThreads) hist[(size_t)d * hstride + blockIdx.x] = h[d];
}

// ---------------------------------------------------------------------------------
// a2: stable LSD counting sort.  Keys lie in [0, nb] (nb = dropped); passes =
// ceil(bits/10) with digits of ceil(bits/passes) <= 10 bits (two passes up to 2^20
// buckets, three up to 2^30).  Per pass: per-tile digit histograms (pass 0: fused into
// the convert kernel) -> per-digit exclusive scan over the tiles + digit totals (one
// kernel) -> stable in-tile ranking into a digit-sorted shared-memory copy of the tile
// -> coalesced write-out, each tile adding the exclusive scan of the digit totals.

__global__ void __launch_bounds__(kRsThreads) rs_upsweep(const uint32_t* __restrict__ keys, int n,
                                                         int shift, uint32_t dmask, int nbins,
                                                         uint32_t* __restrict__ hist, int hstride, int rounds) {
    extern __shared__ uint32_t h[];  // [nbins]
    for (int d = threadIdx.x; d < nbins; d += kRsThreads) h[d] = 0;
    __syncthreads();
    const int base = blockIdx.x * kRsThreads * rounds;
#pragma unroll 8
    for (int r = 0; r < rounds; r++) {
        const int i = base + r * kRsThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < nbins; d += kRsThreads) hist[(size_t)d * hstride + blockIdx.x] = h[d];
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

// Stable scatter of one tile (kRsThreads x ROUNDS keys, ROUNDS = rs_rounds(nbins)).  Warp w
// owns the contiguous sub-range [w*32*ROUNDS, (w+1)*32*ROUNDS) of the tile (loads stay
// coalesced: 32 consecutive keys per round), so ranking needs no CTA barrier per round:
//   1. per round, warp match_any ranks equal digits among the lanes; a warp-private digit
//      counter (shared memory, uint16) orders the rounds -> rank of each key within its
//      warp's keys of that digit (kept in registers);
//   2. one barrier; per digit, an exclusive scan of the 8 warp counters (warp order =
//      index order) and of the tile's digit counts (tile-local run starts);
//   3. each key's tile-local position = run start + warp prefix + in-warp rank: STAGED
//      writes the tile digit-sorted into shared memory and then out coalesced (small digit
//      sets), otherwise keys scatter straight to their global positions.
// The result is the stable order (index order within equal digits), as the oracle's
// std::stable_sort-equivalent definition requires.
template <bool STAGED, int ROUNDS>
__global__ void __launch_bounds__(kRsThreads) rs_downsweep(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
    uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, int n, int shift, uint32_t dmask, int nbins,
    const uint32_t* __restrict__ hscan, const uint32_t* __restrict__ dtot, int hstride) {
    extern __shared__ uint32_t sm[];
    __shared__ uint32_t s_ws[kRsThreads / 32];
    constexpr int kW = kRsThreads / 32;
    constexpr int tile = kRsThreads * ROUNDS;
    uint32_t* boff = sm;                    // [nbins] global base of the tile's digit run
    uint32_t* dstart = sm + nbins;          // [nbins] tile-local start of the digit run
    uint32_t* skey = sm + 2 * nbins;        // [tile] (STAGED)
    uint32_t* sval = skey + tile;           // [tile] (STAGED)
    uint16_t* wcnt = reinterpret_cast<uint16_t*>(STAGED ? sval + tile : sm + 2 * nbins);  // [kW][nbins]
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int b = blockIdx.x;
    for (int e = t; e < kW * nbins; e += kRsThreads) wcnt[e] = 0;
    // this warp's keys (index order: round-major within the warp's sub-range)
    const int wbase = b * tile + warp * 32 * ROUNDS + lane;
    uint32_t kb[ROUNDS], vb[ROUNDS], rk[ROUNDS];
#pragma unroll
    for (int r = 0; r < ROUNDS; r++) {
        const int i = wbase + r * 32;
        kb[r] = i < n ? kin[i] : 0u;
        vb[r] = i < n ? (vin ? vin[i] : (uint32_t)i) : 0u;
    }
    __syncthreads();
    uint16_t* my = wcnt + warp * nbins;
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < ROUNDS; r++) {
        const bool valid = wbase + r * 32 < n;
        const uint32_t d = valid ? ((kb[r] >> shift) & dmask) : (0x10000u + lane);  // unique if invalid
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t pre = valid ? (uint32_t)my[d] : 0u;
        rk[r] = pre + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) my[d] = (uint16_t)(pre + __popc(peers));
        __syncwarp();
    }
    __syncthreads();
    // per digit: warp counters -> exclusive prefixes over warps; tile count -> dstart
    for (int d = t; d < nbins; d += kRsThreads) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kW; w++) {
            const uint32_t c = wcnt[w * nbins + d];
            wcnt[w * nbins + d] = (uint16_t)run;
            run += c;
        }
        dstart[d] = run;
        boff[d] = dtot[d];  // -> exclusive scan of the digit totals
    }
    __syncthreads();
    block_scan_smem(boff, nbins, s_ws);
    if (STAGED) block_scan_smem(dstart, nbins, s_ws);
    for (int d = t; d < nbins; d += kRsThreads) boff[d] += hscan[(size_t)d * hstride + b];  // + tile prefix
    __syncthreads();
#pragma unroll
    for (int r = 0; r < ROUNDS; r++) {
        if (wbase + r * 32 >= n) break;
        const uint32_t d = (kb[r] >> shift) & dmask;
        const uint32_t pos = (uint32_t)my[d] + rk[r];
        if (STAGED) {
            const uint32_t lp = dstart[d] + pos;
            skey[lp] = kb[r];
            sval[lp] = vb[r];
        } else {
            const uint32_t dst = boff[d] + pos;
            kout[dst] = kb[r];
            vout[dst] = vb[r];
        }
    }
    if (!STAGED) return;
    __syncthreads();
    const int base = b * tile;
    const int cnt = min(tile, n - base);
    for (int e = t; e < cnt; e += kRsThreads) {
        const uint32_t k = skey[e];
        const uint32_t d = (k >> shift) & dmask;
        const uint32_t dst = boff[d] + (uint32_t)e - dstart[d];
        kout[dst] = k;
        vout[dst] = sval[e];
    }
}

// Per-digit exclusive scan over the tiles, in place (hist is digit-major [d][stride], rows
// 16-byte aligned), one CTA per digit: coalesced uint4 loads of 1024 tiles per step, a block
// scan, a running carry; dtot[d] = the digit's total.
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
}

// a2 gather + bucket offsets, one pass over the sorted keys.  Position d in [0, n]:
//   offsets: offsets[b] = first position with key >= b -- the thread of position d writes the
//            buckets (key[d-1], key[d]] (empty buckets take the next occupied bucket's start;
//            long runs of empty buckets are written by the whole warp);
//   gather:  a kept point (key < nb) at sorted position d gets its bucket-local fp32 SoA and
//            packed int16 ranges from the record the convert kernel wrote in input order.
// Kept keys (< nb) sort before the dropped sentinel nb, so positions [0, n_binned) are the
// binned points.
__global__ void __launch_bounds__(256) gather_offsets_kernel(const uint4* __restrict__ rec,
                                                             const uint32_t* __restrict__ perm,
                                                             const uint32_t* __restrict__ skey, int n, uint32_t nb,
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
            kc[u] = d < n ? skey[d] : nb;
            kp[u] = (d > 0 && d <= n) ? skey[d - 1] : 0xffffffffu;
            q[u] = (d < n && kc[u] < nb) ? perm[d] : 0u;
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
    // passes = ceil(kb / 11), digits of db = ceil(kb / passes) bits, and the LAST pass takes
    // all the remaining high bits, key >> shift in [0, nb >> shift] -- a digit set of
    // (nb >> shift) + 1 that holds the dropped sentinel without an extra pass (C4: 2^20
    // buckets -> 1024 + 1025 digits, two passes instead of three).
    int kb = 1;
    while ((1ull << kb) < nb) kb++;
    const int passes = (kb + kRsMaxBits - 1) / kRsMaxBits;
    const int dbits = (kb + passes - 1) / passes;
    auto pass_bins = [&](int ps) {
        return ps == passes - 1 ? (int)(nb >> (ps * dbits)) + 1 : 1 << dbits;
    };
    auto pass_mask = [&](int ps) { return ps == passes - 1 ? 0xffffffffu : (1u << dbits) - 1u; };
    int nbins = 0;  // the largest digit set
    for (int ps = 0; ps < passes; ps++) nbins = std::max(nbins, pass_bins(ps));
    const uint32_t dmask0 = pass_mask(0);
    const int nbins0 = pass_bins(0);
    // tuning knobs (A/B experiments): KDE_RS_ROUNDS = 8|16 forces the tile rounds,
    // KDE_RS_STAGED = the largest digit count that stages the tile in shared memory
    static const int env_rounds = getenv("KDE_RS_ROUNDS") ? atoi(getenv("KDE_RS_ROUNDS")) : 0;
    static const int env_staged = getenv("KDE_RS_STAGED") ? atoi(getenv("KDE_RS_STAGED")) : 1100;
    // default: 4096-key tiles from 8 M points on (measured: C4 binning 0.96 -> 0.91 ms; C2
    // prefers 2048-key tiles: more CTAs for its 2 M keys); tiles hold >= 4 keys per digit
    const int rounds = (env_rounds == 8 || env_rounds == 16) ? std::max(env_rounds, rs_rounds(nbins))
                       : (n >= (8 << 20) ? std::max(16, rs_rounds(nbins)) : rs_rounds(nbins));
    if (rounds != 8 && rounds != 16 && rounds != 32) {
        set_error("binning: %d digits per pass not supported", nbins);
        return KDE_EUNSUPPORTED;
    }
    const int tile = kRsThreads * rounds;
    const int nblk = (n + tile - 1) / tile;
    const int hstride = (nblk + 3) & ~3;  // histogram rows: 16-byte aligned (rs_scan_digits)
    if (n64 > pb.cap || pb.key[0] == nullptr) {
        const int64_t cap = n64 > 1024 ? n64 : 1024;
        int rc = KDE_OK;
        rc |= grow((void**)&pb.key[0], sizeof(uint32_t) * cap);
        rc |= grow((void**)&pb.key[1], sizeof(uint32_t) * cap);
        rc |= grow((void**)&pb.val[0], sizeof(uint32_t) * cap);
        rc |= grow((void**)&pb.val[1], sizeof(uint32_t) * cap);
        rc |= grow((void**)&pb.xy, sizeof(float2) * cap);
        rc |= grow((void**)&pb.rng, sizeof(uint2) * cap);
        rc |= grow((void**)&pb.rec, sizeof(uint4) * cap);
        if (rc) return KDE_ENOMEM;
        pb.cap = cap;
    }
    const int64_t hneed = (int64_t)nbins * (hstride > 0 ? hstride : 4);
    if (hneed > pb.hist_cap) {
        if (grow((void**)&pb.hist, sizeof(uint32_t) * hneed)) return KDE_ENOMEM;
        if (grow((void**)&pb.scan_tmp, sizeof(uint32_t) * 4096)) return KDE_ENOMEM;  // digit totals
        pb.hist_cap = hneed;
    }
    cudaMemsetAsync(c->d_stats, 0, 3 * sizeof(unsigned long long), s);
    if (n > 0) {
        // small digit sets scatter short runs: stage the tile digit-sorted in shared memory
        // and write it out coalesced; large ones scatter directly
        auto dn_smem = [&](int nbp, bool stg) {
            return sizeof(uint32_t) * (2 * nbp + (stg ? 2 * tile : 0)) + sizeof(uint16_t) * 8 * nbp;
        };
        {   // the shared-memory opt-in is per device and cheap: set it on every load (no
            // process-global state).  Largest case: 2049 digits, tile 8192.
            const int mx = (int)std::max(dn_smem(2049, false), dn_smem(1100, true));
            cudaFuncSetAttribute(rs_downsweep<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
            cudaFuncSetAttribute(rs_downsweep<true, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
            cudaFuncSetAttribute(rs_downsweep<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
            cudaFuncSetAttribute(rs_downsweep<false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
            cudaFuncSetAttribute(rs_downsweep<false, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        }
        bin_convert_kernel<<<nblk, kRsThreads, sizeof(uint32_t) * nbins0, s>>>(
            d_x, d_y, n, g, nb, pb.key[0], pb.rec, c->d_stats, dmask0, nbins0, pb.hist, hstride, rounds);
        c->launches += 1;
        int cur = 0;
        for (int ps = 0; ps < passes; ps++) {
            const int shift = ps * dbits;
            const uint32_t dmask = pass_mask(ps);
            const int nbp = pass_bins(ps);
            if (ps > 0) {
                rs_upsweep<<<nblk, kRsThreads, sizeof(uint32_t) * nbp, s>>>(pb.key[cur], n, shift, dmask, nbp,
                                                                           pb.hist, hstride, rounds);
                c->launches += 1;
            }
            rs_scan_digits<<<nbp, 256, 0, s>>>(pb.hist, nbp, nblk, hstride, pb.scan_tmp);
            const bool staged = nbp <= env_staged && rounds <= 16;
            auto dsw = staged ? (rounds == 8 ? rs_downsweep<true, 8> : rs_downsweep<true, 16>)
                              : (rounds == 8 ? rs_downsweep<false, 8>
                                             : rounds == 16 ? rs_downsweep<false, 16> : rs_downsweep<false, 32>);
            dsw<<<nblk, kRsThreads, dn_smem(nbp, staged), s>>>(pb.key[cur], ps == 0 ? nullptr : pb.val[cur],
                                                                 pb.key[cur ^ 1], pb.val[cur ^ 1], n, shift, dmask,
                                                                 nbp, pb.hist, pb.scan_tmp, hstride);
            c->launches += 2;
            cur ^= 1;
        }
        pb.perm = pb.val[cur];
        const int gg = (n + 1 + 1023) / 1024 < 148 * 8 ? (n + 1 + 1023) / 1024 : 148 * 8;
        gather_offsets_kernel<<<gg, 256, 0, s>>>(pb.rec, pb.perm, pb.key[cur], n, nb, c->d_offsets, pb.xy, pb.rng);
        c->launches += 1;
    } else {
        cudaMemsetAsync(c->d_offsets, 0, sizeof(uint32_t) * (nb + 1), s);
        pb.perm = pb.val[0];
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "binning launch");
    return KDE_OK;
}

}  // namespace kde
