// NEXT-F3: GPU Douglas-Peucker over a batch of trajectories (kde_dp in include/kde.h).
//
// The recursion of the serial DP (the paper's own motivation for
// removing it) is replaced by level-synchronous rounds over ALL points of ALL
// trajectories at once.  Every point carries the kept points (s, e) bracketing it -- its
// current curve segment (the role of the paper's label set Lp, Fig. 5) -- and a round is
//   dp_ved_kernel     VED (Eq. 9) of every unkept point to its chord, fp64 with
//                     one IEEE rounding per operation in the oracle's order; the
//                     segment's maximum by atomicMax on the bits (VED >= 0, so the bit
//                     patterns order like the values) -- the paper's segmented max-scan
//   dp_argmax_kernel  the earliest index attaining that maximum, when it exceeds eps
//                     (strict) -- the argmax of the segmented scan
//   dp_split_kernel   the chosen point becomes a kept point; the others of the segment
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
constexpr int kNoSplit = 0x7f7f7f7f;  // bidx after the per-round memset of 0x7f bytes (> any index)

// Eq. 9: |P_sP_n x P_sP_e| / |P_sP_e|; a degenerate chord uses |P_n - P_s| (R14)
__device__ __forceinline__ double dp_ved(double px, double py, double sx, double sy, double ex, double ey) {
    const double dx = __dsub_rn(ex, sx), dy = __dsub_rn(ey, sy);
    const double L = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    const double ax = __dsub_rn(px, sx), ay = __dsub_rn(py, sy);
    if (L == 0.0) return __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    const double cr = __dsub_rn(__dmul_rn(ax, dy), __dmul_rn(ay, dx));
    return __ddiv_rn(fabs(cr), L);
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
    keep[i] = (i == a || i == b) ? 1 : 0;
}

// keep[i]: 0 active, 1 retained, 2 dropped for good (its segment's maximum VED was <= eps:
// the segment never splits again, so its points leave the rounds)
__global__ void dp_ved_kernel(const double* __restrict__ x, const double* __restrict__ y,
                              const int2* __restrict__ seg, const uint8_t* __restrict__ keep, int n,
                              unsigned long long* __restrict__ dbits, unsigned long long* __restrict__ best) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool act = i < n && keep[i] == 0;
    int s = -1 - lane;  // unique per inactive lane: never grouped
    unsigned long long b = 0;
    if (act) {
        const int2 se = seg[i];
        const double d = dp_ved(x[i], y[i], x[se.x], y[se.x], x[se.y], y[se.y]);
        b = (unsigned long long)__double_as_longlong(d);
        dbits[i] = b;
        s = se.x;
    }
    // lanes of one segment are contiguous: segmented max towards the run's first lane, so
    // one atomic per (warp, segment) instead of one per point
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long bo = __shfl_down_sync(0xffffffffu, b, o);
        const int so = __shfl_down_sync(0xffffffffu, s, o);
        if (lane + o < 32 && so == s) b = bo > b ? bo : b;
    }
    const int sp = __shfl_up_sync(0xffffffffu, s, 1);
    if (act && (lane == 0 || sp != s)) atomicMax(&best[s], b);
}

__global__ void dp_argmax_kernel(const int2* __restrict__ seg, const uint8_t* __restrict__ keep, int n,
                                 const unsigned long long* __restrict__ dbits,
                                 const unsigned long long* __restrict__ best, double eps,
                                 int* __restrict__ bidx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || keep[i] != 0) return;
    const int s = seg[i].x;
    const unsigned long long b = best[s];
    if (dbits[i] == b && __longlong_as_double((long long)b) > eps) atomicMin(&bidx[s], i);
}

__global__ void dp_split_kernel(int2* __restrict__ seg, uint8_t* __restrict__ keep, int n,
                                const int* __restrict__ bidx, int* __restrict__ changed) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || keep[i] != 0) return;
    const int2 se = seg[i];
    const int k = bidx[se.x];
    if (k == kNoSplit) {  // max VED <= eps: the segment is final
        keep[i] = 2;
        return;
    }
    if (i == k) {
        keep[i] = 1;
        *changed = 1;
    } else if (i > k) {
        seg[i] = make_int2(k, se.y);
    } else {
        seg[i] = make_int2(se.x, k);
    }
}

__global__ void dp_count_kernel(const uint8_t* __restrict__ keep, int n, unsigned long long* __restrict__ cnt) {
    unsigned long long c = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) c += keep[i] == 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

__global__ void dp_finish_kernel(uint8_t* __restrict__ keep, int n) {  // 2 -> 0
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && keep[i] == 2) keep[i] = 0;
}

int dp_run(const double* x, const double* y, const int64_t* offs, int ntraj, int n, double eps, uint8_t* keep,
           cudaStream_t s, int64_t* n_kept, int64_t* rounds_out) {
    int2* seg = nullptr;
    unsigned long long *dbits = nullptr, *best = nullptr;
    int *bidx = nullptr, *changed = nullptr;
    int* h_changed = nullptr;
    cudaError_t e = cudaMallocAsync(&seg, sizeof(int2) * (size_t)n, s);
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
        dp_init_kernel<<<gb, kDpThreads, 0, s>>>(offs, ntraj, n, seg, keep);
        for (;;) {
            cudaMemsetAsync(changed, 0, sizeof(int) * kDpBatch, s);
            for (int r = 0; r < kDpBatch; r++) {
                cudaMemsetAsync(best, 0, sizeof(unsigned long long) * (size_t)n, s);
                cudaMemsetAsync(bidx, 0x7f, sizeof(int) * (size_t)n, s);  // kNoSplit
                dp_ved_kernel<<<gb, kDpThreads, 0, s>>>(x, y, seg, keep, n, dbits, best);
                dp_argmax_kernel<<<gb, kDpThreads, 0, s>>>(seg, keep, n, dbits, best, eps, bidx);
                dp_split_kernel<<<gb, kDpThreads, 0, s>>>(seg, keep, n, bidx, changed + r);
            }
            cudaMemcpyAsync(h_changed, changed, sizeof(int) * kDpBatch, cudaMemcpyDeviceToHost, s);
            e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) {
                rc = cuda_fail(e, "kde_dp");
                break;
            }
            int last = -1;
            for (int r = 0; r < kDpBatch; r++)
                if (h_changed[r]) last = r;
            rounds += last + 1;
            if (last < kDpBatch - 1) break;  // a round changed nothing: converged
        }
    }
    if (rc == KDE_OK) dp_finish_kernel<<<(n + kDpThreads - 1) / kDpThreads, kDpThreads, 0, s>>>(keep, n);
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
    cudaFreeAsync(dbits, s);
    cudaFreeAsync(best, s);
    cudaFreeAsync(bidx, s);
    cudaFreeAsync(changed, s);
    cudaStreamSynchronize(s);
    if (h_changed) cudaFreeHost(h_changed);
    return rc;
}

}  // namespace kde
