// NEXT-F1: the paper's own KDE pipeline (Alg. 3 + Eq. 7), kde_snap in include/kde.h.
//
//   snap_extent_kernel   x_min/x_max/y_min/y_max of the finite points (order-preserving
//                        uint64 encoding of fp64, warp reduce + one atomic per warp)
//   snap_project_kernel  Eqs. 5-6 per point (fp64 RN, as written) -> integer atomics into
//                        M_D (Alg. 3 step 2: exact, so deterministic); the point's
//                        thread also adds the Eq. 12-13 interpolated cells between it and
//                        its successor when both carry the same label (Alg. 3 step 3)
//   snap_rows_kernel     Eq. 7, pass 1: tmp(x, y) = sum_s k(s/h) M_D(x - s, y)   (shared-
//                        memory row segment + halo, fp32, fixed order)
//   snap_cols_kernel     Eq. 7, pass 2: out(x, y) = sum_t k(t/h) tmp(x, y - t)
// Product kernels only: f(s,t) = k(s) k(t) makes the 2-D sum of Eq. 7 two 1-D sums
// (O(W H a) instead of O(W H a^2)); the factor constants are folded into the 1-D weights.
#include <math.h>

#include "internal.cuh"

namespace kde {

constexpr int kSnapThreads = 256;
constexpr int kRowSeg = 1024;   // row pass: outputs per CTA (4 per thread, 256 apart)
constexpr int kColW = 32;       // column pass: columns per CTA
constexpr int kColRows = 64;    // column pass: output rows per CTA
constexpr int kMaxTaps = 1025;  // 2a + 1 <= 1025 (a <= 512 px)

__device__ __forceinline__ unsigned long long ord64(double d) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord64(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// ext[0..3] = ord(x_min), ord(x_max), ord(y_min), ord(y_max); initialised to (~0, 0, ~0, 0)
__global__ void __launch_bounds__(kSnapThreads) snap_extent_kernel(const double* __restrict__ x,
                                                                   const double* __restrict__ y, int n,
                                                                   unsigned long long* __restrict__ ext) {
    unsigned long long mn[2] = {~0ull, ~0ull}, mx[2] = {0ull, 0ull};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double a = x[i], b = y[i];
        if (!isfinite(a) || !isfinite(b)) continue;
        const unsigned long long ka = ord64(a), kb = ord64(b);
        mn[0] = min(mn[0], ka);
        mx[0] = max(mx[0], ka);
        mn[1] = min(mn[1], kb);
        mx[1] = max(mx[1], kb);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < 2; k++) {
            mn[k] = min(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], o));
            mx[k] = max(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], o));
        }
    __shared__ unsigned long long s_r[4][kSnapThreads / 32];  // per warp, then one atomic per CTA
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_r[0][w] = mn[0];
        s_r[1][w] = mx[0];
        s_r[2][w] = mn[1];
        s_r[3][w] = mx[1];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        const int k = threadIdx.x;
        unsigned long long r = s_r[k][0];
        for (int q = 1; q < kSnapThreads / 32; q++) r = (k & 1) ? max(r, s_r[k][q]) : min(r, s_r[k][q]);
        const bool any = (k & 1) ? r != 0ull : r != ~0ull;
        if (any) {
            if (k & 1) atomicMax(&ext[k], r);
            else atomicMin(&ext[k], r);
        }
    }
}

// Eq. 5 (Eq. 6 alike): 1-based cell of coordinate z
__device__ __forceinline__ int snap_cell(double z, double zmin, double zmax, int m) {
    if (zmax == zmin) return 1;
    const double q = __dmul_rn(__ddiv_rn(__dsub_rn(z, zmin), __dsub_rn(zmax, zmin)), (double)(m - 1));
    return (int)ceil(q) + 1;
}

// [num / den] = floor(num/den + 1/2), den > 0, exactly (R17)
__device__ __forceinline__ int round_half_up_ratio(int num, int den) {
    const long long p = 2ll * num + den, q = 2ll * den;
    return (int)(p >= 0 ? p / q : -((-p + q - 1) / q));
}

__global__ void __launch_bounds__(kSnapThreads) snap_project_kernel(
    const double* __restrict__ x, const double* __restrict__ y, const int32_t* __restrict__ label, int n,
    const unsigned long long* __restrict__ ext, int u, int v, uint32_t* __restrict__ M) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const double x0 = unord64(ext[0]), x1 = unord64(ext[1]);
    const double y0 = unord64(ext[2]), y1 = unord64(ext[3]);
    int cx = 0, cy = 0, dx = 0, dy = 0, cmax = 0;  // cmax > 1: this point opens a gap
    if (i < n) {
        const double xa = x[i], ya = y[i];
        if (isfinite(xa) && isfinite(ya)) {
            cx = snap_cell(xa, x0, x1, u);
            cy = snap_cell(ya, y0, y1, v);
            atomicAdd(&M[(size_t)(cy - 1) * u + (cx - 1)], 1u);  // Alg. 3 step 2
            if (label && i + 1 < n && label[i] == label[i + 1]) {
                const double xb = x[i + 1], yb = y[i + 1];
                if (isfinite(xb) && isfinite(yb)) {
                    dx = snap_cell(xb, x0, x1, u) - cx;
                    dy = snap_cell(yb, y0, y1, v) - cy;
                    cmax = max(abs(dx), abs(dy));
                }
            }
        }
    }
    // Eqs. 12-13, c = 1 .. c_max - 1 (R18): short gaps by their own lane, long ones (AIS
    // reports up to 180 s apart span hundreds of cells) by the whole warp
    const bool big = cmax > 32;
    if (!big)
        for (int c = 1; c < cmax; c++)
            atomicAdd(&M[(size_t)(cy + round_half_up_ratio(c * dy, cmax) - 1) * u +
                         (cx + round_half_up_ratio(c * dx, cmax) - 1)], 1u);
    unsigned m = __ballot_sync(0xffffffffu, big);
    while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int gx = __shfl_sync(0xffffffffu, cx, src), gy = __shfl_sync(0xffffffffu, cy, src);
        const int gdx = __shfl_sync(0xffffffffu, dx, src), gdy = __shfl_sync(0xffffffffu, dy, src);
        const int gm = __shfl_sync(0xffffffffu, cmax, src);
        for (int c = 1 + lane; c < gm; c += 32)
            atomicAdd(&M[(size_t)(gy + round_half_up_ratio(c * gdy, gm) - 1) * u +
                         (gx + round_half_up_ratio(c * gdx, gm) - 1)], 1u);
    }
}

// pass 1: one CTA per (row, 256-column segment); the segment plus its a-wide halo is
// staged in shared memory as fp32
__global__ void __launch_bounds__(kSnapThreads) snap_rows_kernel(const uint32_t* __restrict__ M,
                                                                 const float* __restrict__ w, int a, int u,
                                                                 float* __restrict__ tmp) {
    extern __shared__ float sh[];  // [2a + 1] weights, then [kRowSeg + 2a] counts
    float* sw = sh;
    float* sr = sh + 2 * a + 1;
    const int y = blockIdx.y, x0 = blockIdx.x * kRowSeg;
    for (int k = threadIdx.x; k < 2 * a + 1; k += blockDim.x) sw[k] = w[k];
    const uint32_t* row = M + (size_t)y * u;
    for (int k = threadIdx.x; k < kRowSeg + 2 * a; k += blockDim.x) {
        const int xs = x0 - a + k;
        sr[k] = (xs >= 0 && xs < u) ? (float)row[xs] : 0.f;
    }
    __syncthreads();
    // tmp(x) = sum_{s=-a..a} k(s) M(x - s): sr[xl + a - s] = M(x - s); each weight read
    // once for the thread's 4 outputs
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s = -a; s <= a; s++) {
        const float w = sw[s + a];
#pragma unroll
        for (int q = 0; q < 4; q++) acc[q] = fmaf(w, sr[threadIdx.x + 256 * q + a - s], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int xo = x0 + threadIdx.x + 256 * q;
        if (xo < u) tmp[(size_t)y * u + xo] = acc[q];
    }
}

// pass 2: one CTA per (32 columns, 64 rows); the 64 + 2a rows of the 32 columns are
// staged in shared memory; thread (tx, ty) computes rows ty, ty + 8, ...
__global__ void __launch_bounds__(kSnapThreads) snap_cols_kernel(const float* __restrict__ tmp,
                                                                 const float* __restrict__ w, int a, int u, int v,
                                                                 float* __restrict__ out) {
    extern __shared__ float sh[];  // [2a + 1] weights, then [(kColRows + 2a) x kColW]
    float* sw = sh;
    float* sc = sh + 2 * a + 1;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int xc = blockIdx.x * kColW + tx, y0 = blockIdx.y * kColRows;
    for (int k = threadIdx.x; k < 2 * a + 1; k += blockDim.x) sw[k] = w[k];
    for (int r = ty; r < kColRows + 2 * a; r += kSnapThreads / 32) {
        const int ys = y0 - a + r;
        sc[r * kColW + tx] = (xc < u && ys >= 0 && ys < v) ? tmp[(size_t)ys * u + xc] : 0.f;
    }
    __syncthreads();
    if (xc >= u) return;
    constexpr int kR = kColRows / (kSnapThreads / 32);  // 8 output rows per thread
    float acc[kR];
#pragma unroll
    for (int q = 0; q < kR; q++) acc[q] = 0.f;
    for (int t = -a; t <= a; t++) {  // each weight read once for the thread's 8 outputs
        const float w = sw[t + a];
#pragma unroll
        for (int q = 0; q < kR; q++) acc[q] = fmaf(w, sc[(ty + 8 * q + a - t) * kColW + tx], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < kR; q++) {
        const int yo = y0 + ty + 8 * q;
        if (yo < v) out[(size_t)yo * u + xc] = acc[q];
    }
}

void snap_free(kde_ctx* c) {
    SnapBufs& sb = c->snap;
    cudaFree(sb.x);
    cudaFree(sb.y);
    cudaFree(sb.lab);
    cudaFree(sb.counts);
    cudaFree(sb.tmp);
    cudaFree(sb.ext);
    cudaFree(sb.w);
    if (sb.done) cudaEventDestroy(sb.done);
    sb = SnapBufs();
}

static int grow_snap(void** p, size_t bytes, const char* what) {
    cudaFree(*p);
    *p = nullptr;
    if (cudaMalloc(p, bytes ? bytes : 16) != cudaSuccess) {
        cudaGetLastError();
        set_error("kde_snap: cudaMalloc for %s failed (%zu bytes)", what, bytes);
        return KDE_ENOMEM;
    }
    return KDE_OK;
}

// 1-D weights k(s / h_px) with Table 1's constant, s = -a..a (host, fp64 -> fp32)
static void snap_weights(int kern, double hpx, int a, float* w) {
    const double pi = 3.14159265358979323846;
    const double c1[8] = {0.5, 1.0, 0.75, 15.0 / 16.0, 35.0 / 32.0, 70.0 / 81.0,
                          0.39894228040143267794, pi / 4.0};
    for (int s = -a; s <= a; s++) {
        const double z = s / hpx, z2 = z * z, az = fabs(z);
        double k;
        switch (kern) {
        case 0: k = 1.0; break;
        case 1: k = 1.0 - az; break;
        case 2: k = 1.0 - z2; break;
        case 3: k = (1.0 - z2) * (1.0 - z2); break;
        case 4: k = (1.0 - z2) * (1.0 - z2) * (1.0 - z2); break;
        case 5: { const double q = 1.0 - az * az * az; k = q * q * q; } break;
        case 6: k = exp(-0.5 * z2); break;
        default: k = cos(0.5 * pi * z); break;
        }
        w[s + a] = (float)(c1[kern] * (k > 0.0 ? k : 0.0));
    }
}

int snap_run(kde_ctx* c, const double* x, const double* y, const int32_t* label, int64_t n64,
             uint32_t* counts, float* out, cudaStream_t s, bool host) {
    SnapBufs& sb = c->snap;
    const int n = (int)n64, u = c->g.W, v = c->g.H;
    const size_t npx = (size_t)u * v;
    const int a = (int)floor(c->ceff * c->hpx);
    if (2 * a + 1 > kMaxTaps) {
        set_error("kde_snap: window 2a+1 = %d exceeds %d taps", 2 * a + 1, kMaxTaps);
        return KDE_EUNSUPPORTED;
    }
    if (!sb.done && cudaEventCreateWithFlags(&sb.done, cudaEventDisableTiming) != cudaSuccess)
        return cuda_fail(cudaGetLastError(), "kde_snap: event");
    // the scratch below (staging, extent, weights, M_D, row pass) is per context: a snap on
    // another stream must not overwrite it while the previous one still reads it
    if (sb.used) {
        if (host) {
            const cudaError_t we = cudaEventSynchronize(sb.done);  // its buffers are reallocated/overwritten
            if (we != cudaSuccess) return cuda_fail(we, "kde_snap: previous call");
        }
        cudaStreamWaitEvent(s, sb.done, 0);
    }
    if (host && n > sb.cap) {
        if (grow_snap((void**)&sb.x, sizeof(double) * n, "x") || grow_snap((void**)&sb.y, sizeof(double) * n, "y") ||
            grow_snap((void**)&sb.lab, sizeof(int32_t) * n, "labels"))
            return KDE_ENOMEM;
        sb.cap = n;
    }
    if (!sb.tmp) {
        if (grow_snap((void**)&sb.tmp, sizeof(float) * npx, "row pass") ||
            grow_snap((void**)&sb.ext, 4 * sizeof(unsigned long long), "extent") ||
            grow_snap((void**)&sb.w, sizeof(float) * kMaxTaps, "weights"))
            return KDE_ENOMEM;
    }
    if (!counts) {
        if (!sb.counts && grow_snap((void**)&sb.counts, sizeof(uint32_t) * npx, "M_D")) return KDE_ENOMEM;
        counts = sb.counts;
    }
    if (host && n > 0) {
        cudaMemcpyAsync(sb.x, x, sizeof(double) * n, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(sb.y, y, sizeof(double) * n, cudaMemcpyHostToDevice, s);
        if (label) cudaMemcpyAsync(sb.lab, label, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s);
        x = sb.x;
        y = sb.y;
        if (label) label = sb.lab;
    }
    float hw[kMaxTaps];
    snap_weights(c->kern, c->hpx, a, hw);
    cudaMemcpyAsync(sb.w, hw, sizeof(float) * (2 * a + 1), cudaMemcpyHostToDevice, s);
    const unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
    cudaMemcpyAsync(sb.ext, init, sizeof init, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(counts, 0, sizeof(uint32_t) * npx, s);
    if (n > 0) {
        const int gb = std::min((n + kSnapThreads - 1) / kSnapThreads, 148 * 4);
        snap_extent_kernel<<<gb, kSnapThreads, 0, s>>>(x, y, n, sb.ext);
        snap_project_kernel<<<(n + kSnapThreads - 1) / kSnapThreads, kSnapThreads, 0, s>>>(x, y, label, n, sb.ext,
                                                                                           u, v, counts);
        c->launches += 2;
    }
    const size_t rs = sizeof(float) * (2 * a + 1 + kRowSeg + 2 * a);
    const size_t cs = sizeof(float) * (2 * a + 1 + (size_t)(kColRows + 2 * a) * kColW);
    cudaFuncSetAttribute(snap_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs);
    cudaFuncSetAttribute(snap_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs);
    snap_rows_kernel<<<dim3((u + kRowSeg - 1) / kRowSeg, v), kSnapThreads, rs, s>>>(counts, sb.w, a, u, sb.tmp);
    snap_cols_kernel<<<dim3((u + kColW - 1) / kColW, (v + kColRows - 1) / kColRows), kSnapThreads, cs, s>>>(
        sb.tmp, sb.w, a, u, v, out);
    c->launches += 2;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "kde_snap launch");
    cudaEventRecord(sb.done, s);
    sb.used = true;
    if (host) {  // the caller's host buffers must outlive the copies
        const cudaError_t se = cudaStreamSynchronize(s);
        if (se != cudaSuccess) return cuda_fail(se, "kde_snap");
    }
    return KDE_OK;
}

}  // namespace kde
