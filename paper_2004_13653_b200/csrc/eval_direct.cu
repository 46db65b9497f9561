// Step a3 (+ fused a5): direct tiled evaluation for all 8 Table-1 kernels, product or
// radial form, fp32.
//
// Prior art: the paper's §IV-B-2 convolution tiles the output in a thread
// grid, stages the input tile + halo in shared memory, keeps the kernel in constant
// memory and unrolls for ILP.  Here the input is the continuous point set, so per
// 64x64 output tile one CTA:
//   1. streams the tile's neighbourhood buckets (contiguous ranges of the sorted SoA,
//      coalesced), culls points whose integer box misses the tile and compacts the
//      survivors IN ORDER into shared memory (ballot + warp prefix);
//   2. per chunk of 64 survivors, evaluates the 1-D factors khat(s) for the tile's 64
//      columns and khat(t) for its 64 rows once per CTA into shared memory (masked by
//      the fp64-decided integer ranges);
//   3. each warp owns a 32x16 sub-tile, skips points whose box misses it (warp-uniform
//      ballot masks), and each lane accumulates a 4x4 register micro-tile with one FFMA
//      per (pixel, point) pair: acc += ky[r] * kx[c];
//   4. blocked fp32 accumulation: per-chunk partials are added into running totals
//      (R10), and the epilogue multiplies by C/(n h_px^2) (step a5).
// Heavy tiles are split along the candidate list into fixed-size segments (split-K);
// segment partials are summed in segment order by reduce_kernel -> deterministic.
#include "internal.cuh"
#include "kernels.cuh"

namespace kde {

struct DirectArgs {
    Geom g;
    const uint32_t* __restrict__ offsets;
    const float2* __restrict__ xy;
    const uint2* __restrict__ rng;
    const WorkItem* __restrict__ items;
    float* __restrict__ out;
    float* __restrict__ partial;
    KConst k;
    float c2;     // radial: c_eff^2
    float scale;  // C / (n h_px^2)
};

constexpr int kT = kDirTile;     // 64
constexpr int kCh = 64;          // points per factor chunk
constexpr int kLd = kT + 4;      // padded factor row (floats)
constexpr int kStage = 256;      // candidates examined per staging step
constexpr int kMaxRowB = 64;     // max buckets per neighbourhood row held in smem

template <int KERN, bool RADIAL>
__global__ void __launch_bounds__(256, 2) direct_kernel(const DirectArgs a) {
    __shared__ __align__(16) float s_fx[kCh][kLd];
    __shared__ __align__(16) float s_fy[kCh][kLd];
    __shared__ float2 s_cxy[kCh + kStage];
    __shared__ int4 s_crng[kCh + kStage];
    __shared__ uint32_t s_rowb[kMaxRowB + 1];
    __shared__ int s_wsum[8];

    const Geom& g = a.g;
    const WorkItem w = a.items[blockIdx.x];
    const int X0 = w.tx * kT, Y0 = w.ty * kT;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int wx = warp & 1, wy = warp >> 1;     // warp sub-tile 32 cols x 16 rows
    const int lx = lane & 7, ly = lane >> 3;     // lane micro-tile 4 cols x 4 rows
    const int c0 = wx * 32 + lx * 4, r0 = wy * 16 + ly * 4;
    const uint32_t lt_mask = (1u << lane) - 1u;

    const int bx0 = max(X0 / kBucket - g.nr, 0);
    const int bx1 = min((X0 + kT - 1) / kBucket + g.nr, g.nbx - 1);
    const int by0 = max(Y0 / kBucket - g.nr, 0);
    const int by1 = min((Y0 + kT - 1) / kBucket + g.nr, g.nby - 1);
    const int nbr = bx1 - bx0 + 1;

    float acc[4][4], tot[4][4];
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[r][c] = tot[r][c] = 0.f;

    // --- one chunk of m <= 64 compacted points at s_cxy/s_crng[base..base+m) ---------
    auto process_chunk = [&](int base, int m) {
        {  // factors: thread -> point p = t/4, 16 columns and 16 rows
            const int p = t >> 2, q = (t & 3) * 16;
            if (p < m) {
                const float2 P = s_cxy[base + p];
                const int4 rr = s_crng[base + p];
#pragma unroll
                for (int k = 0; k < 16; k += 4) {
                    float4 fx, fy;
                    float* px = &fx.x;
                    float* py = &fy.x;
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int c = q + k + e;
                        const float dx = ((float)c + 0.5f) - P.x;
                        const float dy = ((float)c + 0.5f) - P.y;
                        const bool inx = (unsigned)(c - rr.x) <= (unsigned)(rr.y - rr.x);
                        const bool iny = (unsigned)(c - rr.z) <= (unsigned)(rr.w - rr.z);
                        if constexpr (RADIAL) {
                            px[e] = inx ? dx * dx * a.k.inv_h2 : __int_as_float(0x7f800000);
                            py[e] = iny ? dy * dy * a.k.inv_h2 : __int_as_float(0x7f800000);
                        } else {
                            px[e] = inx ? khat<KERN>(dx, a.k) : 0.f;
                            py[e] = iny ? khat<KERN>(dy, a.k) : 0.f;
                        }
                    }
                    *reinterpret_cast<float4*>(&s_fx[p][q + k]) = fx;
                    *reinterpret_cast<float4*>(&s_fy[p][q + k]) = fy;
                }
            }
        }
        // warp culling masks: which of the chunk's points touch this warp's sub-tile
        uint32_t mk[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int p = lane + 32 * h;
            bool hit = false;
            if (p < m) {
                const int4 rr = s_crng[base + p];
                hit = rr.x <= wx * 32 + 31 && rr.y >= wx * 32 && rr.z <= wy * 16 + 15 &&
                      rr.w >= wy * 16;
            }
            mk[h] = __ballot_sync(0xffffffffu, hit);
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; h++) {
            uint32_t msk = mk[h];
            while (msk) {
                const int p = __ffs(msk) - 1 + 32 * h;
                msk &= msk - 1;
                const float4 fx = *reinterpret_cast<const float4*>(&s_fx[p][c0]);
                const float4 fy = *reinterpret_cast<const float4*>(&s_fy[p][r0]);
                const float vx[4] = {fx.x, fx.y, fx.z, fx.w};
                const float vy[4] = {fy.x, fy.y, fy.z, fy.w};
#pragma unroll
                for (int r = 0; r < 4; r++)
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        if constexpr (RADIAL) {
                            const float r2 = vx[c] + vy[r];
                            acc[r][c] += (r2 <= a.c2) ? khat_r<KERN>(r2) : 0.f;
                        } else {
                            acc[r][c] = fmaf(vy[r], vx[c], acc[r][c]);
                        }
                    }
            }
        }
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int c = 0; c < 4; c++) {
                tot[r][c] += acc[r][c];
                acc[r][c] = 0.f;
            }
        __syncthreads();
    };

    int cnt = 0;  // compacted points waiting in s_cxy/s_crng
    int pos = 0;  // candidate position of the current row's first point
    for (int by = by0; by <= by1; by++) {
        const uint32_t* orow = a.offsets + (size_t)by * g.nbx;
        const int rlo = (int)orow[bx0], rhi = (int)orow[bx1 + 1];
        const int len = rhi - rlo;
        const int lo = max(w.k0 - pos, 0), hi = min(w.k1 - pos, len);
        pos += len;
        if (lo >= hi) continue;
        __syncthreads();
        if (t <= nbr && t <= kMaxRowB) s_rowb[t] = orow[bx0 + t];
        __syncthreads();
        for (int sb = lo; sb < hi; sb += kStage) {
            const int i = sb + t;
            bool keep = false;
            float2 P = make_float2(0.f, 0.f);
            int4 rr = make_int4(0, 0, 0, 0);
            if (i < hi) {
                const uint32_t d = (uint32_t)(rlo + i);
                const uint2 q = a.rng[d];
                rr = make_int4((int)(q.x & 0xffffu) - X0, (int)(q.x >> 16) - X0,
                               (int)(q.y & 0xffffu) - Y0, (int)(q.y >> 16) - Y0);
                keep = rr.x <= kT - 1 && rr.y >= 0 && rr.z <= kT - 1 && rr.w >= 0;
                if (keep) {
                    int bx = bx0;
                    if (nbr <= kMaxRowB) {
                        for (int b = 1; b < nbr; b++) bx += (d >= s_rowb[b]);
                    } else {
                        for (int b = 1; b < nbr; b++) bx += (d >= orow[bx0 + b]);
                    }
                    const float2 l = a.xy[d];
                    P = make_float2(l.x + (float)(bx * kBucket - X0), l.y + (float)(by * kBucket - Y0));
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) s_wsum[warp] = __popc(bal);
            __syncthreads();
            int wpre = 0, add = 0;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const int v = s_wsum[k];
                wpre += (k < warp) ? v : 0;
                add += v;
            }
            if (keep) {
                const int slot = cnt + wpre + __popc(bal & lt_mask);
                s_cxy[slot] = P;
                s_crng[slot] = rr;
            }
            __syncthreads();
            cnt += add;
            int done = 0;
            while (cnt - done >= kCh) {
                process_chunk(done, kCh);
                done += kCh;
            }
            if (done > 0) {  // move the (< 64) leftovers to the front, order kept
                const int rem = cnt - done;
                float2 tp = make_float2(0.f, 0.f);
                int4 tr = make_int4(0, 0, 0, 0);
                if (t < rem) {
                    tp = s_cxy[done + t];
                    tr = s_crng[done + t];
                }
                __syncthreads();
                if (t < rem) {
                    s_cxy[t] = tp;
                    s_crng[t] = tr;
                }
                __syncthreads();
                cnt = rem;
            }
        }
    }
    if (cnt > 0) process_chunk(0, cnt);

    // epilogue (a5): scale + store own band rows, or write the raw partial
    if (w.slot < 0) {
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int gy = Y0 + r0 + r;
            if (gy < g.rb || gy >= g.re) continue;
            float* orow = a.out + (size_t)(gy - g.rb) * g.W;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int gx = X0 + c0 + c;
                if (gx < g.W) orow[gx] = tot[r][c] * a.scale;
            }
        }
    } else {
        float* pp = a.partial + (size_t)w.slot * kT * kT;
#pragma unroll
        for (int r = 0; r < 4; r++)
            *reinterpret_cast<float4*>(&pp[(r0 + r) * kT + c0]) =
                make_float4(tot[r][0], tot[r][1], tot[r][2], tot[r][3]);
    }
}

// split-K reduction: fixed segment order -> deterministic
__global__ void __launch_bounds__(256) reduce_kernel(const ReduceItem* __restrict__ reds,
                                                     const float* __restrict__ partial, Geom g,
                                                     int tw, int th, float scale,
                                                     float* __restrict__ out) {
    const ReduceItem ri = reds[blockIdx.x];
    const int X0 = ri.tx * tw, Y0 = ri.ty * th;
    for (int e = threadIdx.x; e < tw * th; e += blockDim.x) {
        const int r = e / tw, c = e % tw;
        const int gy = Y0 + r, gx = X0 + c;
        float s = 0.f;
        for (int k = 0; k < ri.nseg; k++) s += partial[(size_t)(ri.slot0 + k) * tw * th + e];
        if (gx < g.W && gy >= g.rb && gy < g.re) out[(size_t)(gy - g.rb) * g.W + gx] = s * scale;
    }
}

template <int K, bool RAD>
static void launch_one(const DirectArgs& a, int nitems, cudaStream_t s) {
    direct_kernel<K, RAD><<<nitems, 256, 0, s>>>(a);
}

using LaunchFn = void (*)(const DirectArgs&, int, cudaStream_t);
static const LaunchFn kDirect[2][8] = {
    {launch_one<0, false>, launch_one<1, false>, launch_one<2, false>, launch_one<3, false>,
     launch_one<4, false>, launch_one<5, false>, launch_one<6, false>, launch_one<7, false>},
    {launch_one<0, true>, launch_one<1, true>, launch_one<2, true>, launch_one<3, true>,
     launch_one<4, true>, launch_one<5, true>, launch_one<6, true>, launch_one<7, true>}};

KConst make_kconst(double hpx) {
    KConst k;
    k.inv_h = (float)(1.0 / hpx);
    k.inv_h2 = (float)(1.0 / (hpx * hpx));
    k.inv_h3 = (float)(1.0 / (hpx * hpx * hpx));
    k.kq = (float)(-0.5 * 1.4426950408889634074 / (hpx * hpx));
    k.kc = (float)(3.14159265358979323846 / (2.0 * hpx));
    return k;
}

float make_scale(const kde_ctx* c) {
    const double n = (double)c->stats.n_finite;
    if (n <= 0) return 0.f;
    return (float)(kernel_constant(c->kern, c->radial) / (n * c->hpx * c->hpx));
}

int launch_direct(kde_ctx* c, float* out, cudaStream_t s) {
    EvalPlan& pl = c->plan_dir;
    const size_t rows = (size_t)(c->g.re - c->g.rb);
    if (pl.any_empty || pl.items.empty())
        cudaMemsetAsync(out, 0, rows * c->g.W * sizeof(float), s);
    if (!pl.items.empty()) {
        DirectArgs a;
        a.g = c->g;
        a.offsets = c->d_offsets;
        a.xy = c->pb.xy;
        a.rng = c->pb.rng;
        a.items = pl.d_items;
        a.out = out;
        a.partial = pl.d_partial;
        a.k = make_kconst(c->hpx);
        a.c2 = (float)(c->ceff * c->ceff);
        a.scale = make_scale(c);
        kDirect[c->radial ? 1 : 0][c->kern](a, (int)pl.items.size(), s);
        c->launches += 1 + (pl.reds.empty() ? 0 : 1);
        if (!pl.reds.empty())
            reduce_kernel<<<(int)pl.reds.size(), 256, 0, s>>>(pl.d_reds, pl.d_partial, c->g, kT, kT,
                                                             a.scale, out);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "direct eval launch");
    return KDE_OK;
}

}  // namespace kde
