// Step a3 (+ fused a5): direct fp32 evaluation for all 8 Table-1 kernels, product or
// radial form.
//
// Prior art: the paper's §IV-B-2 convolution tiles the output in a thread
// grid, stages input tile + halo in shared memory, keeps the kernel in constant memory
// and unrolls for ILP.  On B200 with continuous point coordinates the cost that matters
// is geometric waste: a SIMT lane owns fixed pixels, so a point's (2R+1)^2 window must be
// computed over every register tile it touches.  AIS points are concentrated (lanes,
// anchorages: >90% of points share an 8x8-pixel home bucket with >=128 others), so the
// register tiles are aligned to the POINT GROUPS instead of the output grid:
//
//   splat pass   one CTA per (bucket g, segment of <= 1024 of its points, 64x64 sub-window
//                of g's window [bx*B - F, bx*B + B - 1 + F]^2, F = floor(R + 1/2)).  Per
//                chunk of 32 points the CTA evaluates the 1-D factors khat(s) for the
//                window's columns and khat(t) for its rows once into shared memory
//                (masked by the fp64-decided integer ranges; double-buffered, one barrier
//                per chunk), and each thread accumulates a 4x4 register micro-tile with one
//                FFMA per (pixel, point) pair: acc += ky[r] * kx[c].  Blocked fp32
//                accumulation (per-chunk partials into running totals, R10).
//                The block is written to its splat slot.
//   combine pass one CTA per 32x32 output tile sums, for every pixel, the splat blocks of
//                the groups whose window covers it, in a fixed order (group row-major, then
//                segment), and multiplies by C/(n h_px^2) (step a5).  Deterministic; a band
//                computes exactly the same splats, so sharded == unsharded bitwise.
#include "internal.cuh"
#include "kernels.cuh"

namespace kde {

struct SplatArgs {
    Geom g;
    const uint32_t* __restrict__ offsets;
    const float2* __restrict__ xy;
    const uint2* __restrict__ rng;
    const int4* __restrict__ items;   // (bucket, k0, k1, slot)
    const int2* __restrict__ group;   // per bucket: (slot of segment 0, #segments)
    int* __restrict__ done;           // per slot arrival counters; done[nslots] = work queue
    float* __restrict__ splat;
    PathGeom pg;
    int nitems, nslots;
    KConst k;
    float c2;     // radial: c_eff^2
    float q2;     // Gaussian recurrence step 2^(2 kq)
    bool recur;   // recurrence safe: 2^(kq (R + 8)^2) stays a normal float
    int ld;       // factor row stride (floats)
};

constexpr int kChunk = 32;         // points per factor chunk (one per lane)

__device__ __forceinline__ int floor_div(int a, int b) {
    return a >= 0 ? a / b : -((-a + b - 1) / b);
}

// factor-row stride per micro-tile column group (floats): keeps vector loads aligned
template <int MT>
constexpr int mt_stride() { return MT <= 4 ? 4 : 8; }

template <int MT>
__device__ __forceinline__ void lds_mt(const float* p, float (&v)[MT]) {
    if constexpr (MT == 3) {
        const float2 a = *reinterpret_cast<const float2*>(p);
        v[0] = a.x; v[1] = a.y; v[2] = p[2];
    } else if constexpr (MT == 4) {
        const float4 a = *reinterpret_cast<const float4*>(p);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else if constexpr (MT == 5) {
        const float4 a = *reinterpret_cast<const float4*>(p);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = p[4];
    } else {
        const float4 a = *reinterpret_cast<const float4*>(p);
        const float2 b = *reinterpret_cast<const float2*>(p + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y;
    }
}

template <int MT>
__device__ __forceinline__ void sts_mt(float* p, const float (&v)[MT]) {
    if constexpr (MT == 3) {
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
        p[2] = v[2];
    } else if constexpr (MT == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else if constexpr (MT == 5) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        p[4] = v[4];
    } else {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float2*>(p + 4) = make_float2(v[4], v[5]);
    }
}

// Factors of one point for units u = warp, warp + nwarps, ... of MT consecutive columns:
// row[u*ST + e] = [c in range] * khat(c + 1/2 - P) for c = u*MT + e; ph = P - 1/2 in
// sub-window coordinates, [lo, lo + span] the point's integer range (lo huge: no point).
// The range test is a per-unit bitmask; the Gaussian uses the exact-ratio recurrence
// g(d+1) = g(d) * r(d), r(d+1) = r(d) * 2^(2 kq) (2 FMUL per factor, 2 SFU ops per unit).
template <int KERN, bool RADIAL, int MT>
__device__ __forceinline__ void factor_units(float* row, int nunits, int warp, int nwarps, float ph,
                                             int lo, int span, const SplatArgs& a) {
    constexpr int ST = mt_stride<MT>();
    for (int u = warp; u < nunits; u += nwarps) {
        const int c0 = u * MT;
        const int l0 = max(lo - c0, 0), h0 = min(lo + span - c0, MT - 1);
        const uint32_t m = (l0 <= h0) ? ((2u << h0) - (1u << l0)) : 0u;
        const float d0 = (float)c0 - ph;
        float f[MT];
        if (!RADIAL && KERN == 6 && a.recur) {
            float gv = ex2_ftz(d0 * d0 * a.k.kq);
            float r = ex2_ftz(fmaf(2.0f, d0, 1.0f) * a.k.kq);
            const float q = a.q2;
#pragma unroll
            for (int e = 0; e < MT; e++) {
                f[e] = (m & (1u << e)) ? gv : 0.f;
                gv *= r;
                r *= q;
            }
        } else {
#pragma unroll
            for (int e = 0; e < MT; e++) {
                const float d = d0 + (float)e;
                if constexpr (RADIAL) f[e] = (m & (1u << e)) ? d * d * a.k.inv_h2 : __int_as_float(0x7f800000);
                else f[e] = (m & (1u << e)) ? khat<KERN>(d, a.k) : 0.f;
            }
        }
        sts_mt<MT>(row + u * ST, f);
    }
}

// Splat pass (see the header comment).  MT x MT register micro-tile per thread; the plan
// picks MT in {3,4,5,6} so that ceil(S/MT)^2 threads tile the sub-window S x S with full
// warps.  Dynamic shared memory: one factor buffer of kChunk x ld floats for columns and
// one for rows, ld = ceil(S/MT) * mt_stride + 4 (two barriers per chunk).
template <int KERN, bool RADIAL, int MT>
__global__ void __launch_bounds__(256) splat_kernel(const SplatArgs a) {
    constexpr int ST = mt_stride<MT>();
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_w;
    const Geom& g = a.g;
    const int ld = a.ld;
    float* s_fx = smem;                      // [kChunk][ld]
    float* s_fy = smem + kChunk * ld;        // [kChunk][ld]
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, nwarps = blockDim.x >> 5;
    const int nsubx = a.pg.nsubx, nsub = a.pg.nsub(), S = a.pg.sx, slot_ld = a.pg.slot_w;
    const int slot_floats = slot_ld * slot_ld;

    for (;;) {  // persistent: items from the queue, full segments first (equal work)
        if (t == 0) s_w = atomicAdd(&a.done[a.nslots], 1);
        __syncthreads();
        const int w = s_w;
        if (w >= a.nitems) break;
        const int4 it = a.items[w];
        const int gx = it.x % a.pg.ngx, gy = it.x / a.pg.ngx;  // group = one bucket (s = 1)
        const int key = gx * g.nby + gy, sub = it.w % nsub;
        const int sx0 = (sub % nsubx) * S, sy0 = (sub / nsubx) * S;
        const int Wd = a.pg.ww;
        const int sw = min(S, Wd - sx0), sh = min(S, Wd - sy0);
        const int bx = gx, by = gy;
        const int ox = bx * g.B - g.F + sx0;  // global pixel origin of the sub-window
        const int oy = by * g.B - g.F + sy0;
        const int ncx = (sw + MT - 1) / MT, ncy = (sh + MT - 1) / MT;
        const bool active = t < ncx * ncy;
        const int mx = active ? t % ncx : 0, my = active ? t / ncx : 0;
        // bucket-local -> sub-window coordinates (exact small-integer shift), minus 1/2
        const float shx = (float)(bx * g.B - ox) - 0.5f, shy = (float)(by * g.B - oy) - 0.5f;
        const uint32_t base = a.offsets[key] + (uint32_t)it.y;
        const int cnt = it.z - it.y;

        float acc[MT][MT];
#pragma unroll
        for (int r = 0; r < MT; r++)
#pragma unroll
            for (int c = 0; c < MT; c++) acc[r][c] = 0.f;

        // lane p of every warp holds point p of the current chunk (coalesced, prefetched)
        float2 nxy = make_float2(0.f, 0.f);
        uint2 nrg = make_uint2(1u, 0u);
        if (lane < cnt) {
            nxy = a.xy[base + lane];
            nrg = a.rng[base + lane];
        }
        const int nch = (cnt + kChunk - 1) / kChunk;
        for (int ch = 0; ch < nch; ch++) {
            const int np = min(kChunk, cnt - ch * kChunk);
            const float pxh = nxy.x + shx, pyh = nxy.y + shy;
            const int ilo = (int)(nrg.x & 0xffffu) - ox, ihi = (int)(nrg.x >> 16) - ox;
            const int jlo = (int)(nrg.y & 0xffffu) - oy, jhi = (int)(nrg.y >> 16) - oy;
            const bool valid = lane < np;
            {  // prefetch the next chunk's point
                const int q = (ch + 1) * kChunk + lane;
                if (q < cnt) {
                    nxy = a.xy[base + q];
                    nrg = a.rng[base + q];
                }
            }
            __syncthreads();  // previous chunk's factors consumed (and s_w read)
            // 1-D factors of the lane's own point, MT columns (then MT rows) per unit
            factor_units<KERN, RADIAL, MT>(s_fx + lane * ld, ncx, warp, nwarps, pxh,
                                           valid ? ilo : (1 << 29), ihi - ilo, a);
            factor_units<KERN, RADIAL, MT>(s_fy + lane * ld, ncy, warp, nwarps, pyh,
                                           valid ? jlo : (1 << 29), jhi - jlo, a);
            __syncthreads();
            if (active) {
                const float* fxp = s_fx + mx * ST;
                const float* fyp = s_fy + my * ST;
#pragma unroll 4
                for (int p = 0; p < np; p++) {
                    float vx[MT], vy[MT];
                    lds_mt<MT>(fxp + p * ld, vx);
                    lds_mt<MT>(fyp + p * ld, vy);
#pragma unroll
                    for (int r = 0; r < MT; r++)
#pragma unroll
                        for (int c = 0; c < MT; c++) {
                            if constexpr (RADIAL) {
                                const float r2 = vx[c] + vy[r];
                                acc[r][c] += (r2 <= a.c2) ? khat_r<KERN>(r2) : 0.f;
                            } else {
                                acc[r][c] = fmaf(vy[r], vx[c], acc[r][c]);
                            }
                        }
                }
            }
        }
        if (active) {
            float* sp = a.splat + (size_t)it.w * slot_floats + (my * MT) * slot_ld + mx * MT;
#pragma unroll
            for (int r = 0; r < MT; r++)
#pragma unroll
                for (int c = 0; c < MT; c++) sp[r * slot_ld + c] = acc[r][c];
        }
    }
}

// Segment reduce: for every split group (listed by the planner) and sub-window, the
// segment blocks are summed IN SEGMENT ORDER into segment 0's slot.  One CTA per
// (group x sub-window, 1024-float chunk of the slot); float4, 4 segments in flight.
__global__ void __launch_bounds__(256) segreduce_kernel(const int* __restrict__ hot,
                                                        const int2* __restrict__ group, int nsub,
                                                        int slot_floats, float* __restrict__ splat) {
    const int gsub = blockIdx.y;
    const int2 gr = group[hot[gsub / nsub]];
    const int sub = gsub % nsub;
    const int e = (blockIdx.x * 256 + threadIdx.x) * 4;
    if (e >= slot_floats) return;
    float* d0 = splat + ((size_t)gr.x * nsub + sub) * slot_floats + e;
    const size_t stride = (size_t)nsub * slot_floats;
    float4 acc = *reinterpret_cast<const float4*>(d0);
    int k = 1;
    for (; k + 4 <= gr.y; k += 4) {
        const float4 v0 = *reinterpret_cast<const float4*>(d0 + k * stride);
        const float4 v1 = *reinterpret_cast<const float4*>(d0 + (k + 1) * stride);
        const float4 v2 = *reinterpret_cast<const float4*>(d0 + (k + 2) * stride);
        const float4 v3 = *reinterpret_cast<const float4*>(d0 + (k + 3) * stride);
        acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w;
        acc.x += v1.x; acc.y += v1.y; acc.z += v1.z; acc.w += v1.w;
        acc.x += v2.x; acc.y += v2.y; acc.z += v2.z; acc.w += v2.w;
        acc.x += v3.x; acc.y += v3.y; acc.z += v3.z; acc.w += v3.w;
    }
    for (; k < gr.y; k++) {
        const float4 v = *reinterpret_cast<const float4*>(d0 + k * stride);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    *reinterpret_cast<float4*>(d0) = acc;
}

// Combine pass: out(i,j) = scale * sum, in order, of the splat blocks covering (i,j).
// Works for any path geometry (groups of pitch px x py, windows ww x wh, sub-windows).
// One CTA per 32x32 tile.  Warp 0 lists the (slot, sub-window origin, size) entries of the
// non-empty groups whose window meets the tile -- group row-major, then sub-window
// (row-major) -- at most ((32 + ww)/px + 2)((32 + wh)/py + 2) groups x 4 sub-windows
// (checked at create); then every thread (column t&31, rows (t>>5)+8k) walks the list
// kBatch entries at a time so that 4 x kBatch independent loads are in flight.
constexpr int kMaxEnt = 2048;
constexpr int kBatch = 4;

struct CombineArgs {
    Geom g;
    PathGeom pg;
    const int2* __restrict__ group;  // per group: (first segment, #segments)
    const float* __restrict__ splat;
    float* __restrict__ out;
    const unsigned long long* __restrict__ stats;  // n_finite = stats[0] (device)
    double c_over_h2;  // kernel constant / h_px^2: scale = c_over_h2 / n_finite
};

__global__ void __launch_bounds__(256) combine_kernel(const CombineArgs a) {
    __shared__ int4 s_ent[kMaxEnt];  // (slot of segment 0, origin x, origin y, sw | sh << 16)
    __shared__ int s_n;
    const Geom& g = a.g;
    const PathGeom& pg = a.pg;
    const int X0 = blockIdx.x * kCombTile, Y0 = g.rb + blockIdx.y * kCombTile;
    const int Y1 = min(Y0 + kCombTile, g.re) - 1, X1 = X0 + kCombTile - 1;
    const int F = g.F;
    const int gxa = max(floor_div(X0 - F, pg.px), 0), gxb = min(floor_div(X1 + F, pg.px), pg.ngx - 1);
    const int gya = max(floor_div(Y0 - F, pg.py), 0), gyb = min(floor_div(Y1 + F, pg.py), pg.ngy - 1);
    const int ngxr = gxb - gxa + 1, ng = ngxr * (gyb - gya + 1);
    const int nsub = pg.nsub();
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        int n = 0;
        for (int gi0 = 0; gi0 < ng; gi0 += 32) {
            const int gi = gi0 + lane;
            const int gy = gya + gi / ngxr, gx = gxa + gi % ngxr;
            int2 gr = make_int2(0, 0);
            if (gi < ng) gr = a.group[gy * pg.ngx + gx];
            const int wx0 = gx * pg.px - F, wy0 = gy * pg.py - F;
            // sub-windows of this group meeting the tile
            const int sxa = max(X0 - wx0, 0) / pg.sx, sxb = min(min(X1 - wx0, pg.ww - 1) / pg.sx, pg.nsubx - 1);
            const int sya = max(Y0 - wy0, 0) / pg.sy, syb = min(min(Y1 - wy0, pg.wh - 1) / pg.sy, pg.nsuby - 1);
            const int nx = (gr.y > 0 && X1 >= wx0) ? sxb - sxa + 1 : 0;
            const int ny = (gr.y > 0 && Y1 >= wy0) ? syb - sya + 1 : 0;
            const int cntl = (nx > 0 && ny > 0) ? nx * ny : 0;
            int incl = cntl;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            int pos = n + incl - cntl;
            for (int sy = 0; sy < ny; sy++)
                for (int sx = 0; sx < nx; sx++) {
                    const int ssx = sxa + sx, ssy = sya + sy;
                    const int sw = min(pg.sx, pg.ww - ssx * pg.sx), sh = min(pg.sy, pg.wh - ssy * pg.sy);
                    if (pos < kMaxEnt)
                        s_ent[pos] = make_int4(gr.x * nsub + ssy * pg.nsubx + ssx, wx0 + ssx * pg.sx,
                                               wy0 + ssy * pg.sy, sw | (sh << 16));
                    pos++;
                }
            n += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_n = min(n, kMaxEnt);
    }
    __syncthreads();
    const int n = s_n;
    const int i = X0 + lane;
    const int jb = Y0 + (threadIdx.x >> 5);
    const int sl = pg.slot_w;
    const size_t sf = (size_t)pg.slot_floats();
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int e0 = 0; e0 < n; e0 += kBatch) {
        float v[kBatch][4];
#pragma unroll
        for (int b = 0; b < kBatch; b++) {
            const int e = e0 + b;
            const int4 en = e < n ? s_ent[e] : make_int4(0, 0, 0, 0);
            const int li = i - en.y;
            const int sw = en.w & 0xffff, sh = en.w >> 16;
            const bool inx = e < n && (unsigned)li < (unsigned)sw;
            const float* sp = a.splat + (size_t)en.x * sf + li;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int lj = jb + 8 * k - en.z;
                float x = 0.f;
                if (inx && (unsigned)lj < (unsigned)sh) x = sp[(size_t)lj * sl];
                v[b][k] = x;
            }
        }
#pragma unroll
        for (int b = 0; b < kBatch; b++)
#pragma unroll
            for (int k = 0; k < 4; k++) acc[k] += v[b][k];
    }
    if (i >= g.W) return;
    const unsigned long long nf = a.stats[0];
    const float scale = nf ? (float)(a.c_over_h2 / (double)nf) : 0.f;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int j = jb + 8 * k;
        if (j <= Y1) a.out[(size_t)(j - g.rb) * g.W + i] = acc[k] * scale;
    }
}

template <int K, bool RAD, int MT>
static void launch_mt(const SplatArgs& a, int grid, int threads, cudaStream_t s) {
    const size_t smem = sizeof(float) * 2 * kChunk * a.ld;
    splat_kernel<K, RAD, MT><<<grid, threads, smem, s>>>(a);
}

template <int K, bool RAD, int MT>
static int occ_mt(int threads, size_t smem) {
    int nb = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, splat_kernel<K, RAD, MT>, threads, smem);
    return nb > 0 ? nb : 1;
}

template <int K, bool RAD>
static int launch_one(const SplatArgs& a, int mt, int grid, int threads, cudaStream_t s) {
    const size_t smem = sizeof(float) * 2 * kChunk * a.ld;
    if (grid <= 0) {  // query: persistent CTAs per SM
        switch (mt) {
        case 3: return occ_mt<K, RAD, 3>(threads, smem);
        case 4: return occ_mt<K, RAD, 4>(threads, smem);
        case 5: return occ_mt<K, RAD, 5>(threads, smem);
        default: return occ_mt<K, RAD, 6>(threads, smem);
        }
    }
    switch (mt) {
    case 3: launch_mt<K, RAD, 3>(a, grid, threads, s); break;
    case 4: launch_mt<K, RAD, 4>(a, grid, threads, s); break;
    case 5: launch_mt<K, RAD, 5>(a, grid, threads, s); break;
    default: launch_mt<K, RAD, 6>(a, grid, threads, s); break;
    }
    return 0;
}

using LaunchFn = int (*)(const SplatArgs&, int, int, int, cudaStream_t);
static const LaunchFn kSplat[2][8] = {
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

int launch_combine(kde_ctx* c, const EvalPlan& pl, float* out, cudaStream_t s) {
    const Geom& g = c->g;
    if (pl.nhot > 0) {  // split groups: sum their segments first (fixed order)
        const int sf = (int)pl.pg.slot_floats();
        dim3 grid((sf / 4 + 255) / 256, pl.nhot * pl.pg.nsub());
        segreduce_kernel<<<grid, 256, 0, s>>>(pl.d_hot, pl.d_group, pl.pg.nsub(), sf, pl.d_splat);
        c->launches += 1;
    }
    CombineArgs a;
    a.g = g;
    a.pg = pl.pg;
    a.group = pl.d_group;
    a.splat = pl.d_splat;
    a.out = out;
    a.stats = c->d_stats;
    a.c_over_h2 = kernel_constant(c->kern, c->radial) / (c->hpx * c->hpx);
    dim3 grid((g.W + kCombTile - 1) / kCombTile, (g.re - g.rb + kCombTile - 1) / kCombTile);
    combine_kernel<<<grid, 256, 0, s>>>(a);
    c->launches += 1;
    return KDE_OK;
}

int launch_direct(kde_ctx* c, float* out, cudaStream_t s) {
    EvalPlan& pl = c->plan[KDE_PATH_DIRECT];
    if (pl.nitems > 0) {
        SplatArgs a;
        a.g = c->g;
        a.offsets = c->d_offsets;
        a.xy = c->pb.xy;
        a.rng = c->pb.rng;
        a.items = pl.d_items;
        a.group = pl.d_group;
        a.done = pl.d_done;
        a.splat = pl.d_splat;
        a.pg = pl.pg;
        a.nitems = pl.nitems;
        a.nslots = pl.nslots;
        a.k = make_kconst(c->hpx);
        a.c2 = (float)(c->ceff * c->ceff);
        a.ld = pl.ld;
        a.q2 = (float)exp2(2.0 * (double)a.k.kq);
        a.recur = -(double)a.k.kq * (c->g.R + 8.0) * (c->g.R + 8.0) < 120.0;
        LaunchFn fn = kSplat[c->radial ? 1 : 0][c->kern];
        if (pl.grid <= 0) {
            int nsm = 148;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->p.device);
            pl.grid = nsm * fn(a, pl.mt, 0, pl.threads, s);
        }
        // arrival counters + queue head (done[nslots]) start at zero
        cudaMemsetAsync(pl.d_done, 0, sizeof(int) * ((size_t)pl.nslots + 1), s);
        tmark(c, 3, s);
        fn(a, pl.mt, pl.nitems < pl.grid ? pl.nitems : pl.grid, pl.threads, s);
        c->launches += 1;
    } else {
        tmark(c, 3, s);
    }
    tmark(c, 4, s);
    launch_combine(c, pl, out, s);
    tmark(c, 5, s);
    c->tev_eval = c->timing;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "direct eval launch");
    return KDE_OK;
}

}  // namespace kde
