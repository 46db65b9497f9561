// NEXT-F3: GPU Douglas-Peucker over a batch of trajectories (kde_dp in include/kde.h).
//
// The recursion of the serial DP (the paper's own motivation for
// removing it) is replaced by level-synchronous rounds over ALL points of ALL
// trajectories at once.  Every point carries the kept points (s, e) bracketing it -- its
// current curve segment (the role of the paper's label set Lp, Fig. 5) -- and a round is
//   dp_ved16_kernel   VED (Eq. 9) of every unkept point to its chord, fp64 with
//                     one IEEE rounding per operation in the oracle's order; the
//                     segment's maximum by atomicMax on the bits (VED >= 0, so the bit
//                     patterns order like the values) -- the paper's segmented max-scan
//   dp_argmax16_kernel the earliest index attaining that maximum, when it exceeds eps
//                     (strict) -- the argmax of the segmented scan
//   dp_split16_kernel the chosen point becomes a kept point; the others of the segment
//                     move to the half they lie in (the paper's Eq. 11 relabelling)
// Segments are independent, so processing a whole level at once keeps exactly the point
// set the recursion keeps (same VED arithmetic, same tie rule).  Rounds run in batches of
// kDpBatch between one 4-byte convergence readback (a converged round changes nothing).
#include <math.h>
#include <string.h>

#include "internal.cuh"

namespace kde {

constexpr int kDpThreads = 256;
constexpr int kDpBatch = 4;
constexpr int kNoSplit = 0x7f7f7f7f;
constexpr int kLocalMax = 4096;     // trajectories up to this length: one CTA, shared memory
constexpr size_t local_smem(int lmax) { return (size_t)lmax * (8 + 8 + 8 + 4 + 4 + 1); }  // bidx after the per-round memset of 0x7f bytes (> any index)

// Eq. 9: |P_sP_n x P_sP_e| / |P_sP_e|; a degenerate chord uses |P_n - P_s| (R14)
__device__ __forceinline__ double dp_ved(double px, double py, double sx, double sy, double ex, double ey) {
    const double dx = __dsub_rn(ex, sx), dy = __dsub_rn(ey, sy);
    const double L = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    const double ax = __dsub_rn(px, sx), ay = __dsub_rn(py, sy);
    if (L == 0.0) return __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    const double cr = __dsub_rn(__dmul_rn(ax, dy), __dmul_rn(ay, dx));
    return __ddiv_rn(fabs(cr), L);
}

// The bits a VED takes part in the segment maximum with.  The serial recursion keeps a
// point only if `d > dmax` (dp_oracle.c), so a NaN VED (a non-finite coordinate) never
// becomes the maximum: NaN maps to the bits of 0.0, which never exceeds eps >= 0 and never
// equals a positive maximum -- the kept set stays the recursion's.
__device__ __forceinline__ unsigned long long ved_bits(double d) {
    return isnan(d) ? 0ull : (unsigned long long)__double_as_longlong(d);
}

// segment of every point: its trajectory's end points; end points are kept
__global__ void dp_init_kernel(const int64_t* __restrict__ offs, int ntraj, int n, int2* __restrict__ seg,
                               uint8_t* __restrict__ keep) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int lo = 0, hi = ntraj;  // trajectory t with offs[t] <= i < offs[t+1]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (offs[mid] <= i) lo = mid;
        else hi = mid;
    }
    const int a = (int)offs[lo], b = (int)offs[lo + 1] - 1;
    seg[i] = make_int2(a, b);
    // trajectories of <= kLocalMax points are finished by dp_local_kernel: inactive here
    keep[i] = (i == a || i == b || b - a + 1 <= kLocalMax) ? 1 : 0;
}

// A whole trajectory of <= kLocalMax points per CTA, every round in shared memory (the same
// VED arithmetic and tie rule as the global rounds, so the same kept set): no global
// traffic per round, only CTA barriers.  Writes keep[] for its trajectory.
template <int LMIN, int LMAX, int T>
__global__ void __launch_bounds__(T) dp_local_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                     const int64_t* __restrict__ offs, double eps,
                                                     uint8_t* __restrict__ keep, int* __restrict__ rounds) {
    extern __shared__ __align__(16) unsigned char dsm[];
    double* sx = reinterpret_cast<double*>(dsm);                       // [LMAX]
    double* sy = sx + LMAX;                                             // [LMAX]
    unsigned long long* sb = reinterpret_cast<unsigned long long*>(sy + LMAX);  // per segment start: max VED bits
    int* si = reinterpret_cast<int*>(sb + LMAX);                        // per segment start: earliest argmax
    short2* sg = reinterpret_cast<short2*>(si + LMAX);                  // per point: its segment (start, end)
    uint8_t* fl = reinterpret_cast<uint8_t*>(sg + LMAX);                // 0 active, 1 kept, 2 retired
    __shared__ int s_changed;
    constexpr int kLocalThreads = T;
    const int a = (int)offs[blockIdx.x], L = (int)offs[blockIdx.x + 1] - a;
    if (L > LMAX || L < LMIN || L <= 0) return;
    const int tid = threadIdx.x;
    for (int i = tid; i < L; i += kLocalThreads) {
        sx[i] = x[a + i];
        sy[i] = y[a + i];
        fl[i] = (i == 0 || i == L - 1) ? 1 : 0;
        sg[i] = make_short2(0, (short)(L - 1));
        sb[i] = 0ull;
        si[i] = 0x7fffffff;
    }
    __syncthreads();
    int nround = 0;
    for (;;) {
        nround++;
        if (tid == 0) s_changed = 0;
        for (int i = tid; i < L; i += kLocalThreads) {  // VED, segment maxima
            if (fl[i] != 0) continue;
            const short2 se = sg[i];
            const double d = dp_ved(sx[i], sy[i], sx[se.x], sy[se.x], sx[se.y], sy[se.y]);
            atomicMax(&sb[se.x], ved_bits(d));
        }
        __syncthreads();
        for (int i = tid; i < L; i += kLocalThreads) {  // earliest argmax above eps
            if (fl[i] != 0) continue;
            const short2 se = sg[i];
            const double d = dp_ved(sx[i], sy[i], sx[se.x], sy[se.x], sx[se.y], sy[se.y]);
            const unsigned long long b = sb[se.x];
            if (ved_bits(d) == b && __longlong_as_double((long long)b) > eps)
                atomicMin(&si[se.x], i);
        }
        __syncthreads();
        for (int i = tid; i < L; i += kLocalThreads) {  // split / retire
            if (fl[i] != 0) continue;
            const short2 se = sg[i];
            const int k = si[se.x];
            if (k == 0x7fffffff) fl[i] = 2;
            else if (i == k) {
                fl[i] = 1;
                s_changed = 1;
            } else if (i > k) sg[i] = make_short2((short)k, se.y);
            else sg[i] = make_short2(se.x, (short)k);
        }
        __syncthreads();
        const int changed = s_changed;
        for (int i = tid; i < L; i += kLocalThreads) {
            sb[i] = 0ull;
            si[i] = 0x7fffffff;
        }
        __syncthreads();
        if (!changed) break;
    }
    for (int i = tid; i < L; i += kLocalThreads) keep[a + i] = fl[i] == 1 ? 1 : 0;
    if (tid == 0) atomicMax(rounds, nround - 1);  // the last round kept nothing
}

// Working flags: 0 active, 1 retained, 2 retired for good (its segment's maximum VED was
// <= eps: the segment never splits again, so its points leave the rounds).

// Packed round kernels: one thread per 16 consecutive points (one uint4 of the padded
// keep flags).  After the first rounds most points are retired, and a thread whose 16
// flags are all non-zero does nothing but one 16-byte load -- the per-point kernels above
// pay a CTA launch per 256 points every round instead.
__device__ __forceinline__ bool any_zero_byte(uint4 v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t z = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) z |= (w[q] - 0x01010101u) & ~w[q] & 0x80808080u;
    return z != 0;
}
__device__ __forceinline__ uint32_t flag_byte(uint4 v, int q) {
    const uint32_t w = q < 4 ? v.x : q < 8 ? v.y : q < 12 ? v.z : v.w;
    return (w >> (8 * (q & 3))) & 0xffu;
}

__global__ void __launch_bounds__(kDpThreads) dp_ved16_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                              const int2* __restrict__ seg, const uint4* __restrict__ kp,
                                                              int nv, unsigned long long* __restrict__ dbits,
                                                              unsigned long long* __restrict__ best) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nv) return;
    const uint4 kv = kp[t];
    if (!any_zero_byte(kv)) return;
    int cs = -1;                 // current segment run (points of a segment are contiguous)
    unsigned long long cb = 0;   // its running maximum
#pragma unroll 4
    for (int q = 0; q < 16; q++) {
        if (flag_byte(kv, q) != 0) continue;
        const int i = 16 * t + q;
        const int2 se = seg[i];
        const double d = dp_ved(x[i], y[i], x[se.x], y[se.x], x[se.y], y[se.y]);
        const unsigned long long b = ved_bits(d);
        dbits[i] = b;
        if (se.x != cs) {
            if (cs >= 0) atomicMax(&best[cs], cb);
            cs = se.x;
            cb = b;
        } else if (b > cb) {
            cb = b;
        }
    }
    if (cs >= 0) atomicMax(&best[cs], cb);
}

__global__ void __launch_bounds__(kDpThreads) dp_argmax16_kernel(const int2* __restrict__ seg, const uint4* __restrict__ kp,
                                                                 int nv, const unsigned long long* __restrict__ dbits,
                                                                 const unsigned long long* __restrict__ best, double eps,
                                                                 int* __restrict__ bidx) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nv) return;
    const uint4 kv = kp[t];
    if (!any_zero_byte(kv)) return;
    int done = -1;  // segment whose earliest maximum this thread already reported
    for (int q = 0; q < 16; q++) {
        if (flag_byte(kv, q) != 0) continue;
        const int i = 16 * t + q;
        const int s = seg[i].x;
        if (s == done) continue;
        const unsigned long long b = best[s];
        if (dbits[i] == b && __longlong_as_double((long long)b) > eps) {
            atomicMin(&bidx[s], i);
            done = s;
        }
    }
}

__global__ void __launch_bounds__(kDpThreads) dp_split16_kernel(int2* __restrict__ seg, uint4* __restrict__ kp, int nv,
                                                                const int* __restrict__ bidx, int* __restrict__ changed) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nv) return;
    const uint4 kv = kp[t];
    if (!any_zero_byte(kv)) return;
    uint32_t w[4] = {kv.x, kv.y, kv.z, kv.w};
    bool any_kept = false;
    for (int q = 0; q < 16; q++) {
        if (((w[q >> 2] >> (8 * (q & 3))) & 0xffu) != 0) continue;
        const int i = 16 * t + q;
        const int2 se = seg[i];
        const int k = bidx[se.x];
        uint32_t nb = 0;
        if (k == kNoSplit) {  // max VED <= eps: the segment is final
            nb = 2;
        } else if (i == k) {
            nb = 1;
            any_kept = true;
        } else if (i > k) {
            seg[i] = make_int2(k, se.y);
        } else {
            seg[i] = make_int2(se.x, k);
        }
        w[q >> 2] |= nb << (8 * (q & 3));
    }
    kp[t] = make_uint4(w[0], w[1], w[2], w[3]);
    if (any_kept) *changed = 1;
}

__global__ void dp_export_kernel(const uint8_t* __restrict__ kp, int n, uint8_t* __restrict__ keep) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // 2 (retired) -> 0
    if (i < n) keep[i] = kp[i] == 1 ? 1 : 0;
}

__global__ void dp_count_kernel(const uint8_t* __restrict__ keep, int n, unsigned long long* __restrict__ cnt) {
    unsigned long long c = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) c += keep[i] == 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

int dp_run(const double* x, const double* y, const int64_t* offs, int ntraj, int n, double eps, uint8_t* keep,
           cudaStream_t s, int64_t* n_kept, int64_t* rounds_out) {
    int2* seg = nullptr;
    unsigned long long *dbits = nullptr, *best = nullptr;
    int *bidx = nullptr, *changed = nullptr;
    int* h_changed = nullptr;
    uint8_t* kp = nullptr;  // padded working flags: 0 active, 1 retained, 2 retired
    const int nv = (n + 15) / 16;
    {   // keep the stream-ordered pool's memory between calls (no re-mapping of ~0.5 GB of
        // scratch on every call)
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
    }
    cudaError_t e = cudaMallocAsync(&seg, sizeof(int2) * (size_t)n, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&kp, 16 * (size_t)nv, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&dbits, sizeof(unsigned long long) * (size_t)n, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&best, sizeof(unsigned long long) * (size_t)n, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&bidx, sizeof(int) * (size_t)n, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&changed, sizeof(int) * kDpBatch, s);
    if (e == cudaSuccess) e = cudaMallocHost(&h_changed, sizeof(int) * kDpBatch);
    int rc = KDE_OK;
    int64_t rounds = 0;
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("kde_dp: scratch allocation failed (%d points)", n);
        rc = KDE_ENOMEM;
    } else {
        const int gb = (n + kDpThreads - 1) / kDpThreads;
        const int gv = (nv + kDpThreads - 1) / kDpThreads;
        cudaMemsetAsync(kp, 1, 16 * (size_t)nv, s);  // padding: retained (never active)
        dp_init_kernel<<<gb, kDpThreads, 0, s>>>(offs, ntraj, n, seg, kp);
        for (;;) {
            cudaMemsetAsync(changed, 0, sizeof(int) * kDpBatch, s);
            for (int r = 0; r < kDpBatch; r++) {
                cudaMemsetAsync(best, 0, sizeof(unsigned long long) * (size_t)n, s);
                cudaMemsetAsync(bidx, 0x7f, sizeof(int) * (size_t)n, s);  // kNoSplit
                const uint4* kp4 = reinterpret_cast<const uint4*>(kp);
                dp_ved16_kernel<<<gv, kDpThreads, 0, s>>>(x, y, seg, kp4, nv, dbits, best);
                dp_argmax16_kernel<<<gv, kDpThreads, 0, s>>>(seg, kp4, nv, dbits, best, eps, bidx);
                dp_split16_kernel<<<gv, kDpThreads, 0, s>>>(seg, reinterpret_cast<uint4*>(kp), nv, bidx,
                                                            changed + r);
            }
            cudaMemcpyAsync(h_changed, changed, sizeof(int) * kDpBatch, cudaMemcpyDeviceToHost, s);
            e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) {
                rc = cuda_fail(e, "kde_dp");
                break;
            }
            e = cudaGetLastError();  // the round kernels' launches
            if (e != cudaSuccess) {
                rc = cuda_fail(e, "kde_dp: round launch");
                break;
            }
            int last = -1;
            for (int r = 0; r < kDpBatch; r++)
                if (h_changed[r]) last = r;
            rounds += last + 1;
            if (last < kDpBatch - 1) break;  // a round changed nothing: converged
        }
    }
    if (rc == KDE_OK) {
        dp_export_kernel<<<(n + kDpThreads - 1) / kDpThreads, kDpThreads, 0, s>>>(kp, n, keep);
        if (ntraj > 0) {  // short trajectories: 256 threads, 6 CTAs/SM; long: 1024 threads
            // the shared-memory opt-in is per device: set it on every call (cheap), and
            // check both launches (a failed launch must not leave the pre-marked keep flags)
            e = cudaFuncSetAttribute(dp_local_kernel<0, 1024, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)local_smem(1024));
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(dp_local_kernel<1025, kLocalMax, 1024>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)local_smem(kLocalMax));
            int* d_lr = changed;  // scratch reuse: the local kernels' deepest round count
            if (e == cudaSuccess) e = cudaMemsetAsync(d_lr, 0, sizeof(int), s);
            if (e == cudaSuccess) {
                dp_local_kernel<0, 1024, 256><<<ntraj, 256, local_smem(1024), s>>>(x, y, offs, eps, keep, d_lr);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) {
                dp_local_kernel<1025, kLocalMax, 1024><<<ntraj, 1024, local_smem(kLocalMax), s>>>(x, y, offs, eps,
                                                                                                  keep, d_lr);
                e = cudaGetLastError();
            }
            int lr = 0;
            if (e == cudaSuccess) e = cudaMemcpyAsync(&lr, d_lr, sizeof(int), cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) rc = cuda_fail(e, "kde_dp: local rounds");
            rounds = std::max<int64_t>(rounds, lr);
        }
    }
    if (rc == KDE_OK && n_kept) {  // the kept count, read back once
        unsigned long long* d_cnt = dbits;  // scratch reuse
        cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), s);
        dp_count_kernel<<<std::min((n + kDpThreads - 1) / kDpThreads, 148 * 8), kDpThreads, 0, s>>>(keep, n, d_cnt);
        static_assert(sizeof(int) * kDpBatch >= sizeof(unsigned long long), "readback buffer");
        e = cudaMemcpyAsync(h_changed, d_cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) rc = cuda_fail(e, "kde_dp: count");
        unsigned long long hk = 0;
        memcpy(&hk, h_changed, sizeof hk);
        *n_kept = (int64_t)hk;
    }
    if (rounds_out) *rounds_out = rounds;
    cudaFreeAsync(seg, s);
    cudaFreeAsync(kp, s);
    cudaFreeAsync(dbits, s);
    cudaFreeAsync(best, s);
    cudaFreeAsync(bidx, s);
    cudaFreeAsync(changed, s);
    cudaStreamSynchronize(s);
    if (h_changed) cudaFreeHost(h_changed);
    return rc;
}

}  // namespace kde
