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
    const int bx = hx / g.B, by = hy / g.B;
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

// a1 kernel: keys + integer stats (n_finite, n_outside, useful_pairs).
__global__ void __launch_bounds__(256) bin_convert_kernel(const double* __restrict__ x,
                                                          const double* __restrict__ y, int n,
                                                          Geom g, uint32_t sentinel,
                                                          uint32_t* __restrict__ key,
                                                          unsigned long long* __restrict__ stats) {
    unsigned long long nf = 0, no = 0, up = 0;
    const int rb = g.rb, re = g.re;
    constexpr int U = 4;  // points per thread per iteration: loads issued before use
    const int tile = blockDim.x * U;
    for (int i0 = blockIdx.x * tile + threadIdx.x; i0 < n; i0 += gridDim.x * tile) {
        double xv[U], yv[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = i0 + u * blockDim.x;
            xv[u] = i < n ? x[i] : 0.0;
            yv[u] = i < n ? y[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = i0 + u * blockDim.x;
            if (i >= n) break;
            const Binned b = bin_point(xv[u], yv[u], g, sentinel);
            key[i] = b.key;
            nf += b.status > 0;
            no += b.status == 1;
            if (b.status == 2) {
                const int jl = max(b.jlo, rb), jh = min(b.jhi, re - 1);
                if (jh >= jl)
                    up += (unsigned long long)(b.ihi - b.ilo + 1) * (unsigned long long)(jh - jl + 1);
            }
        }
    }
    __shared__ unsigned long long s[3][8];
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
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) t += s[threadIdx.x][k];
        if (t) atomicAdd(&stats[threadIdx.x], t);
    }
}

// ---------------------------------------------------------------------------------
// a2: stable LSD counting sort.  Keys lie in [0, nb] (nb = dropped); passes =
// ceil(bits/11) with digits of ceil(bits/passes) <= 11 bits (two passes up to 2^22
// buckets).  Per pass: per-block digit histograms -> exclusive scan (digit-major) ->
// stable in-block ranking (warp match_any; per-warp digit counts; leaders only clear what
// they set) + scatter.
constexpr int kRsThreads = 256;
constexpr int kRsRounds = 8;
constexpr int kRsChunk = kRsThreads * kRsRounds;
constexpr int kRsMaxBits = 11;

__global__ void __launch_bounds__(kRsThreads) rs_upsweep(const uint32_t* __restrict__ keys, int n,
                                                         int shift, uint32_t dmask,
                                                         uint32_t* __restrict__ hist, int nblk) {
    extern __shared__ uint32_t h[];  // [dmask + 1]
    const int nbins = (int)dmask + 1;
    for (int d = threadIdx.x; d < nbins; d += kRsThreads) h[d] = 0;
    __syncthreads();
    const int base = blockIdx.x * kRsChunk;
#pragma unroll
    for (int r = 0; r < kRsRounds; r++) {
        const int i = base + r * kRsThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < nbins; d += kRsThreads) hist[(size_t)d * nblk + blockIdx.x] = h[d];
}

__global__ void __launch_bounds__(kRsThreads) rs_downsweep(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
    uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, int n, int shift, uint32_t dmask,
    const uint32_t* __restrict__ hscan, int nblk) {
    extern __shared__ uint32_t sm[];
    const int nbins = (int)dmask + 1;
    uint32_t* run = sm;                                   // [nbins] running count per digit
    uint32_t* boff = sm + nbins;                          // [nbins] block base per digit
    uint16_t* wcnt = reinterpret_cast<uint16_t*>(sm + 2 * nbins);  // [8][nbins]
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int d = t; d < nbins; d += kRsThreads) {
        run[d] = 0;
        boff[d] = hscan[(size_t)d * nblk + blockIdx.x];
    }
    for (int e = t; e < (kRsThreads / 32) * nbins; e += kRsThreads) wcnt[e] = 0;
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    const int base = blockIdx.x * kRsChunk;
    for (int r = 0; r < kRsRounds; r++) {
        const int i = base + r * kRsThreads + t;
        const bool valid = i < n;
        const uint32_t k = valid ? kin[i] : 0u;
        const uint32_t v = valid ? (vin ? vin[i] : (uint32_t)i) : 0u;
        const uint32_t d = valid ? ((k >> shift) & dmask) : (0x10000u + lane);  // unique if invalid
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t lrank = __popc(peers & lt);
        const bool leader = valid && lrank == 0;
        if (leader) wcnt[warp * nbins + d] = (uint16_t)__popc(peers);
        __syncthreads();
        if (valid) {
            uint32_t pos = run[d] + lrank;
            for (int w = 0; w < warp; w++) pos += wcnt[w * nbins + d];
            const uint32_t dst = boff[d] + pos;
            kout[dst] = k;
            vout[dst] = v;
        }
        __syncthreads();
        if (leader) {
            atomicAdd(&run[d], (uint32_t)__popc(peers));
            wcnt[warp * nbins + d] = 0;
        }
        __syncthreads();
    }
}

// Exclusive scan of a u32 array (length L) in place: block sums -> scan -> apply.
constexpr int kScanChunk = 2048;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

__global__ void __launch_bounds__(256) scan_sums_kernel(const uint32_t* __restrict__ a, int64_t L,
                                                        uint32_t* __restrict__ sums) {
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    uint32_t s = 0;
    for (int k = threadIdx.x; k < kScanChunk; k += 256) {
        const int64_t i = base + k;
        if (i < L) s += a[i];
    }
    s = warp_incl_scan(s);  // lane 31 holds the warp total
    __shared__ uint32_t ws[8];
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; w++) t += ws[w];
        sums[blockIdx.x] = t;
    }
}

// single block: exclusive scan of the block sums (sequential over 256-wide slabs)
__global__ void __launch_bounds__(256) scan_block_sums_kernel(uint32_t* __restrict__ sums, int nb) {
    __shared__ uint32_t carry;
    __shared__ uint32_t ws[8];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 256) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < nb ? sums[i] : 0u;
        const uint32_t inc = warp_incl_scan(v);
        if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = inc;
        __syncthreads();
        uint32_t wpre = 0, tot = 0;
        for (int w = 0; w < 8; w++) {
            if (w < (int)(threadIdx.x >> 5)) wpre += ws[w];
            tot += ws[w];
        }
        const uint32_t c0 = carry;
        if (i < nb) sums[i] = c0 + wpre + inc - v;
        __syncthreads();
        if (threadIdx.x == 0) carry = c0 + tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) scan_apply_kernel(uint32_t* __restrict__ a, int64_t L,
                                                         const uint32_t* __restrict__ sums) {
    // each thread owns 8 consecutive elements of the 2048-chunk
    const int64_t base = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * 8;
    uint32_t v[8];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        v[k] = (base + k < L) ? a[base + k] : 0u;
        s += v[k];
    }
    const uint32_t inc = warp_incl_scan(s);
    __shared__ uint32_t ws[8];
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = inc;
    __syncthreads();
    uint32_t wpre = 0;
    for (int w = 0; w < (int)(threadIdx.x >> 5); w++) wpre += ws[w];
    uint32_t run = sums[blockIdx.x] + wpre + inc - s;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        if (base + k < L) a[base + k] = run;
        run += v[k];
    }
}

// bucket offsets from the sorted keys: offsets[b] = first position with key >= b
__global__ void offsets_kernel(const uint32_t* __restrict__ skey, int n, uint32_t nb,
                               uint32_t* __restrict__ offsets) {
    for (int d = blockIdx.x * blockDim.x + threadIdx.x; d <= n; d += gridDim.x * blockDim.x) {
        const int64_t kprev = d > 0 ? (int64_t)skey[d - 1] : -1;
        const int64_t k = d < n ? (int64_t)min(skey[d], nb) : (int64_t)nb;
        for (int64_t b = kprev + 1; b <= k && b <= (int64_t)nb; b++) offsets[b] = (uint32_t)d;
    }
}

// a2 gather: sorted position -> bucket-local fp32 SoA + packed int16 ranges
__global__ void __launch_bounds__(256) gather_kernel(const double* __restrict__ x,
                                                     const double* __restrict__ y,
                                                     const uint32_t* __restrict__ perm,
                                                     const uint32_t* __restrict__ offsets,
                                                     uint32_t nb, Geom g,
                                                     float2* __restrict__ xy,
                                                     uint2* __restrict__ rng) {
    const int nbin = (int)offsets[nb];
    constexpr int U = 4;
    const int tile = blockDim.x * U;
    for (int d0 = blockIdx.x * tile + threadIdx.x; d0 < nbin; d0 += gridDim.x * tile) {
        uint32_t q[U];
        double xv[U], yv[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int d = d0 + u * blockDim.x;
            q[u] = d < nbin ? perm[d] : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int d = d0 + u * blockDim.x;
            xv[u] = d < nbin ? x[q[u]] : 0.0;
            yv[u] = d < nbin ? y[q[u]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int d = d0 + u * blockDim.x;
            if (d >= nbin) break;
            const Binned b = bin_point(xv[u], yv[u], g, nb);
            xy[d] = make_float2(b.lx, b.ly);
            rng[d] = make_uint2(((uint32_t)b.ilo & 0xffffu) | ((uint32_t)b.ihi << 16),
                                ((uint32_t)b.jlo & 0xffffu) | ((uint32_t)b.jhi << 16));
        }
    }
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

int scan_excl_u32(uint32_t* a, int64_t L, uint32_t* tmp, cudaStream_t s) {
    if (L <= 0) return 0;
    const int nblk = (int)((L + kScanChunk - 1) / kScanChunk);
    scan_sums_kernel<<<nblk, 256, 0, s>>>(a, L, tmp);
    scan_block_sums_kernel<<<1, 256, 0, s>>>(tmp, nblk);
    scan_apply_kernel<<<nblk, 256, 0, s>>>(a, L, tmp);
    return 3;
}

int bin_points(kde_ctx* c, const double* d_x, const double* d_y, int64_t n64) {
    const int n = (int)n64;
    PointBufs& pb = c->pb;
    const Geom& g = c->g;
    cudaStream_t s = c->stream;
    const uint32_t nb = (uint32_t)g.nbx * (uint32_t)g.nby;
    const int nblk = (n + kRsChunk - 1) / kRsChunk;
    if (n64 > pb.cap || pb.key[0] == nullptr) {
        const int64_t cap = n64 > 1024 ? n64 : 1024;
        int rc = KDE_OK;
        rc |= grow((void**)&pb.key[0], sizeof(uint32_t) * cap);
        rc |= grow((void**)&pb.key[1], sizeof(uint32_t) * cap);
        rc |= grow((void**)&pb.val[0], sizeof(uint32_t) * cap);
        rc |= grow((void**)&pb.val[1], sizeof(uint32_t) * cap);
        rc |= grow((void**)&pb.xy, sizeof(float2) * cap);
        rc |= grow((void**)&pb.rng, sizeof(uint2) * cap);
        if (rc) return KDE_ENOMEM;
        pb.cap = cap;
    }
    const int64_t hneed = (int64_t)2048 * (nblk > 0 ? nblk : 1);
    if (hneed > pb.hist_cap) {
        if (grow((void**)&pb.hist, sizeof(uint32_t) * hneed)) return KDE_ENOMEM;
        if (grow((void**)&pb.scan_tmp, sizeof(uint32_t) * (hneed / kScanChunk + 2))) return KDE_ENOMEM;
        pb.hist_cap = hneed;
    }
    cudaMemsetAsync(c->d_stats, 0, 3 * sizeof(unsigned long long), s);
    if (n > 0) {
        const int grid = (n + 1023) / 1024 < 148 * 8 ? (n + 1023) / 1024 : 148 * 8;
        bin_convert_kernel<<<grid, 256, 0, s>>>(d_x, d_y, n, g, nb, pb.key[0], c->d_stats);
        c->launches += 1;
        // LSD passes over the key bits of [0, nb]
        int bits = 1;
        while ((1ull << bits) <= nb) bits++;
        const int passes = (bits + kRsMaxBits - 1) / kRsMaxBits;
        const int dbits = (bits + passes - 1) / passes;
        const uint32_t dmask = (1u << dbits) - 1u;
        const size_t up_smem = sizeof(uint32_t) * (dmask + 1);
        const size_t dn_smem = sizeof(uint32_t) * 2 * (dmask + 1) + sizeof(uint16_t) * 8 * (dmask + 1);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(rs_downsweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(uint32_t) * 2 * 2048 + sizeof(uint16_t) * 8 * 2048));
            attr = true;
        }
        int cur = 0;
        for (int ps = 0; ps < passes; ps++) {
            const int shift = ps * dbits;
            rs_upsweep<<<nblk, kRsThreads, up_smem, s>>>(pb.key[cur], n, shift, dmask, pb.hist, nblk);
            c->launches += 2 + scan_excl_u32(pb.hist, (int64_t)(dmask + 1) * nblk, pb.scan_tmp, s);
            rs_downsweep<<<nblk, kRsThreads, dn_smem, s>>>(pb.key[cur], ps == 0 ? nullptr : pb.val[cur],
                                                          pb.key[cur ^ 1], pb.val[cur ^ 1], n, shift,
                                                          dmask, pb.hist, nblk);
            cur ^= 1;
        }
        pb.perm = pb.val[cur];
        const int og = (n + 1 + 255) / 256 < 148 * 16 ? (n + 1 + 255) / 256 : 148 * 16;
        offsets_kernel<<<og, 256, 0, s>>>(pb.key[cur], n, nb, c->d_offsets);
        const int gg = (n + 1023) / 1024 < 148 * 8 ? (n + 1023) / 1024 : 148 * 8;
        gather_kernel<<<gg, 256, 0, s>>>(d_x, d_y, pb.perm, c->d_offsets, nb, g, pb.xy, pb.rng);
        c->launches += 2;
    } else {
        cudaMemsetAsync(c->d_offsets, 0, sizeof(uint32_t) * (nb + 1), s);
        pb.perm = pb.val[0];
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "binning launch");
    return KDE_OK;
}

}  // namespace kde
