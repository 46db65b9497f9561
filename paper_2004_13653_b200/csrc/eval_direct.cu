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
//   splat pass   persistent CTAs of 8 warps pop work items (bucket g, segment of <= 512
//                of its points, sub-window S x S of g's window [bx*B - F, bx*B+B-1+F]^2,
//                F = floor(R + 1/2)).  The warps split the segment into 16-point chunks
//                (warp w takes chunks w, w+8, ...) and work without CTA barriers: per
//                chunk the warp evaluates the 1-D factors of its 16 points into its own
//                shared-memory buffer (lanes 0-15: the S column factors khat(s) of point
//                lane, lanes 16-31: the S row factors khat(t); masked by the fp64-decided
//                integer ranges), __syncwarp, and every lane accumulates a TY x 2TY
//                register tile (lanes = 4 column groups x 8 row groups, S = 8 TY) with one
//                FFMA per (pixel, point) pair: acc += ky[r] * kx[c] -- 5 vector LDS per
//                50 FFMA at S = 40.  At the end of the item the warps' tiles are summed in
//                a fixed order (warp 0..7) through shared memory into the segment's slot.
//   combine pass one CTA per 32x32 output tile sums, for every pixel, the splat blocks of
//                the groups whose window covers it, in a fixed order (group row-major, then
//                segment), and multiplies by C/(n h_px^2) (step a5).  Deterministic; a band
//                computes exactly the same splats, so sharded == unsharded bitwise.
#include <algorithm>

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
    int* __restrict__ totals;         // plan totals (kTot*): item count, work-queue head
    float* __restrict__ splat;
    PathGeom pg;
    KConst k;
    float c2;     // radial: c_eff^2
    float q2;     // Gaussian recurrence step 2^(2 kq)
    bool recur;   // recurrence safe: 2^(kq (R + 8)^2) stays a normal float
};

constexpr int kWarps = 8;     // warps per splat CTA
constexpr int kWChunk = 16;   // points per warp chunk

__device__ __forceinline__ int floor_div(int a, int b) {
    return a >= 0 ? a / b : -((-a + b - 1) / b);
}

// Shared-memory layout of one warp's factor buffer for lane tile TY x TX (TX = 2 TY):
// per point, 4 column groups of TX floats (stride TXP) then 8 row groups of TY floats
// (stride TYP, skewed by 4 floats after group 3 when TYP = 8) -- every vector load of the
// consume loop is 16-byte aligned and the 4 (8) groups a warp reads hit distinct banks.
template <int TY>
struct WLayout {
    static constexpr int TX = 2 * TY, S = 8 * TY;
    static constexpr int TXP = (TX + 3) / 4 * 4, TYP = (TY + 3) / 4 * 4;
    static constexpr int COLS = 4 * TXP;
    static constexpr int SKEW = TYP == 8 ? 4 : 0;
    static constexpr int LDP = COLS + 8 * TYP + SKEW;  // floats per point (multiple of 4)
    static constexpr int FACT_FLOATS = kWarps * kWChunk * LDP;
    static constexpr int RED_FLOATS = kWarps * S * S;
    static constexpr int SMEM_FLOATS = FACT_FLOATS > RED_FLOATS ? FACT_FLOATS : RED_FLOATS;
    __device__ static int rowoff(int my) { return COLS + my * TYP + (my >= 4 ? SKEW : 0); }
};

// acc.{x,y} += a.{x,y} * b as one packed FFMA2 (fma.rn.f32x2: same FMA rate as FFMA,
// half the issue slots; each half is an ordinary RN fp32 fma)
__device__ __forceinline__ void ffma2(float2& acc, float2 a, float b) {
    unsigned long long c = *reinterpret_cast<unsigned long long*>(&acc);
    const float2 bb = make_float2(b, b);
    asm("fma.rn.f32x2 %0, %1, %2, %0;"
        : "+l"(c)
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&bb)));
    acc = *reinterpret_cast<float2*>(&c);
}

// N consecutive floats from a 16-byte aligned shared address, widest loads first
template <int N>
__device__ __forceinline__ void lds_n(const float* p, float* v) {
#pragma unroll
    for (int k = 0; k + 4 <= N; k += 4) {
        const float4 a = *reinterpret_cast<const float4*>(p + k);
        v[k] = a.x; v[k + 1] = a.y; v[k + 2] = a.z; v[k + 3] = a.w;
    }
    constexpr int k2 = N / 4 * 4;
    if constexpr (N - k2 >= 2) {
        const float2 a = *reinterpret_cast<const float2*>(p + k2);
        v[k2] = a.x; v[k2 + 1] = a.y;
    }
    if constexpr ((N - k2) % 2 == 1) v[N - 1] = p[N - 1];
}

// The 8 units of TY factors of one point along one axis: unit u covers sub-window
// coordinates c = u*TY + e; f = [c in range] * khat(c + 1/2 - P), ph = P - 1/2 in
// sub-window coordinates, [lo, hi] the point's integer range along the axis (as a 64-bit
// mask over the 8 TY <= 48 coordinates).  The Gaussian uses the exact-ratio recurrence
// g(d+1) = g(d) r(d), r(d+1) = r(d) 2^(2kq) (2 FMUL per factor, reseeded per unit);
// radial forms store s^2 (or +inf when masked).
template <int KERN, bool RADIAL, int TY, bool RECUR>
__device__ __forceinline__ void factor_axis(float* dst_pt, bool yaxis, float ph, int lo, int hi,
                                            const SplatArgs& a) {
    using L = WLayout<TY>;
    // bits lo..hi of the sub-window coordinates (clipped to [0, 64))
    const int l = max(lo, 0), h = min(hi, 63);
    const uint64_t m64 = (l <= h) ? ((~0ull >> (63 - h)) & (~0ull << l)) : 0ull;
#pragma unroll
    for (int u = 0; u < 8; u++) {
        const int c0 = u * TY;
        const uint32_t m = (uint32_t)(m64 >> c0);
        const float d0 = (float)c0 - ph;
        float f[TY];
        if constexpr (RECUR) {
            float gv = ex2_ftz(d0 * d0 * a.k.kq);
            float r = ex2_ftz(fmaf(2.0f, d0, 1.0f) * a.k.kq);
#pragma unroll
            for (int e = 0; e < TY; e++) {
                f[e] = (m & (1u << e)) ? gv : 0.f;
                gv *= r;
                r *= a.q2;
            }
        } else {
#pragma unroll
            for (int e = 0; e < TY; e++) {
                const float d = d0 + (float)e;
                if constexpr (RADIAL) f[e] = (m & (1u << e)) ? d * d * a.k.inv_h2 : __int_as_float(0x7f800000);
                else f[e] = (m & (1u << e)) ? khat<KERN>(d, a.k) : 0.f;
            }
        }
        float* dst = dst_pt + (yaxis ? L::rowoff(u) : (u >> 1) * L::TXP + (u & 1) * TY);
#pragma unroll
        for (int e = 0; e < TY; e++) dst[e] = f[e];
    }
}

// Item geometry shared by the two phases of the splat kernel.
struct ItemGeo {
    uint32_t base;  // first sorted position of the item's points
    int cnt;        // points
    int oo;         // sub-window origin along this lane's generation axis (pixels)
    float sh;       // bucket-local -> sub-window coordinate shift minus 1/2, same axis
};

__device__ __forceinline__ ItemGeo item_geo(const SplatArgs& a, const int4& it, bool yaxis) {
    const Geom& g = a.g;
    const int nsub = a.pg.nsub(), SX = a.pg.sx;
    const int gx = it.x % a.pg.ngx, gy = it.x / a.pg.ngx;  // group = one bucket (s = 1)
    const int sub = it.w % nsub;
    const int ox = gx * g.B - g.F + (sub % a.pg.nsubx) * SX;  // global pixel origin of the
    const int oy = gy * g.B - g.F + (sub / a.pg.nsubx) * SX;  // sub-window
    ItemGeo r;
    r.base = (uint32_t)it.y;  // items hold absolute sorted positions
    r.cnt = it.z - it.y;
    r.oo = yaxis ? oy : ox;
    // exact small-integer shift, minus 1/2
    r.sh = yaxis ? (float)(gy * g.B - oy) - 0.5f : (float)(gx * g.B - ox) - 0.5f;
    return r;
}

// Accumulate chunks ch0, ch0 + step, ... of an item into the lane's register tile, using
// this warp's factor buffer wbuf (warp-synchronous; no CTA barrier).  The next chunk's
// point is loaded while the current one is evaluated.
template <int KERN, bool RADIAL, int TY, bool RECUR>
__device__ __forceinline__ void run_chunks(float2 (&acc)[TY][TY], const SplatArgs& a, const ItemGeo& ig,
                                           float* wbuf, int ch0, int step, int lane) {
    using L = WLayout<TY>;
    constexpr int TX = L::TX;
    const int mx = lane & 3, my = lane >> 2;  // lane tile: columns mx*TX.., rows my*TY..
    const int gp = lane & 15;                 // generation: point of this lane
    const bool yaxis = lane >= 16;            //             and its axis
    const int nch = (ig.cnt + kWChunk - 1) / kWChunk;
    const float* fxp = wbuf + mx * L::TXP;
    const float* fyp = wbuf + L::rowoff(my);
    float npos = 0.f;
    uint32_t nrg = 1u;  // lo = 1 > hi = 0: empty
    {
        const int q = ch0 * kWChunk + gp;
        if (ch0 < nch && q < ig.cnt) {
            const float2 l = a.xy[ig.base + q];
            const uint2 rr = a.rng[ig.base + q];
            npos = yaxis ? l.y : l.x;
            nrg = yaxis ? rr.y : rr.x;
        }
    }
    for (int ch = ch0; ch < nch; ch += step) {
        const float pos = npos;
        const uint32_t pr = nrg;
        const bool valid = ch * kWChunk + gp < ig.cnt;
        {   // prefetch the next chunk's point
            const int q = (ch + step) * kWChunk + gp;
            if (q < ig.cnt) {
                const float2 l = a.xy[ig.base + q];
                const uint2 rr = a.rng[ig.base + q];
                npos = yaxis ? l.y : l.x;
                nrg = yaxis ? rr.y : rr.x;
            }
        }
        if (valid)  // 1-D factors of this lane's point along its axis
            factor_axis<KERN, RADIAL, TY, RECUR>(wbuf + gp * L::LDP, yaxis, pos + ig.sh,
                                                 (int)(pr & 0xffffu) - ig.oo, (int)(pr >> 16) - ig.oo, a);
        __syncwarp();
        const int np = min(kWChunk, ig.cnt - ch * kWChunk);
#pragma unroll 2
        for (int p = 0; p < np; p++) {
            float vx[TX], vy[TY];
            lds_n<TX>(fxp + p * L::LDP, vx);
            lds_n<TY>(fyp + p * L::LDP, vy);
#pragma unroll
            for (int r = 0; r < TY; r++)
#pragma unroll
                for (int c = 0; c < TX; c += 2) {
                    if constexpr (RADIAL) {
                        const float r0 = vx[c] + vy[r], r1 = vx[c + 1] + vy[r];
                        acc[r][c / 2].x += (r0 <= a.c2) ? khat_r<KERN>(r0) : 0.f;
                        acc[r][c / 2].y += (r1 <= a.c2) ? khat_r<KERN>(r1) : 0.f;
                    } else {
                        ffma2(acc[r][c / 2], make_float2(vx[c], vx[c + 1]), vy[r]);
                    }
                }
        }
        __syncwarp();
    }
}

// Splat pass.  Phase 1: the CTA's 8 warps share each full segment (warp w takes chunks
// w, w+8, ...; tiles summed in warp order through shared memory).  Phase 2: every warp
// alone pops remainder pieces (<= 128 points) and writes its tile straight to the slot.
template <int KERN, bool RADIAL, int TY, bool RECUR>
__global__ void __launch_bounds__(kWarps * 32, 2) splat_kernel(const SplatArgs a) {
    using L = WLayout<TY>;
    constexpr int TX = L::TX, S = L::S;
    extern __shared__ __align__(16) float smem[];
    __shared__ int s_w;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int mx = lane & 3, my = lane >> 2;
    const bool yaxis = lane >= 16;
    const int slot_floats = S * S;
    const int nsub = a.pg.nsub();
    const int ncoop = a.totals[kTotFull] * nsub;  // full-segment items come first
    const int nitems = a.totals[kTotSlots];
    float* wbuf = smem + warp * (kWChunk * L::LDP);  // this warp's factor buffer

    for (;;) {  // phase 1 (persistent, CTA-cooperative)
        if (t == 0) s_w = atomicAdd(&a.totals[kTotQueue], 1);
        __syncthreads();
        const int w = s_w;
        if (w >= ncoop) break;
        const int4 it = a.items[w];
        const ItemGeo ig = item_geo(a, it, yaxis);
        float2 acc[TY][TY];  // column pairs
#pragma unroll
        for (int r = 0; r < TY; r++)
#pragma unroll
            for (int c = 0; c < TY; c++) acc[r][c] = make_float2(0.f, 0.f);
        run_chunks<KERN, RADIAL, TY, RECUR>(acc, a, ig, wbuf, warp, kWarps, lane);
        __syncthreads();  // every warp is done with its factor buffer
        {
            float* red = smem + warp * (S * S) + (my * TY) * S + mx * TX;
#pragma unroll
            for (int r = 0; r < TY; r++)
#pragma unroll
                for (int c = 0; c < TX; c += 2) *reinterpret_cast<float2*>(red + r * S + c) = acc[r][c / 2];
        }
        __syncthreads();
        float* sp = a.splat + (size_t)it.w * slot_floats;
        for (int e = t * 4; e < slot_floats; e += kWarps * 32 * 4) {
            float4 v = *reinterpret_cast<const float4*>(smem + e);
#pragma unroll
            for (int k = 1; k < kWarps; k++) {
                const float4 u = *reinterpret_cast<const float4*>(smem + k * (S * S) + e);
                v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
            }
            *reinterpret_cast<float4*>(sp + e) = v;
        }
        // (the next pop's barrier orders these reads before any buffer rewrite)
    }
    for (;;) {  // phase 2 (per warp): remainder pieces
        int w = 0;
        if (lane == 0) w = ncoop + atomicAdd(&a.totals[kTotQueue2], 1);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= nitems) break;
        const int4 it = a.items[w];
        const ItemGeo ig = item_geo(a, it, yaxis);
        float2 acc[TY][TY];
#pragma unroll
        for (int r = 0; r < TY; r++)
#pragma unroll
            for (int c = 0; c < TY; c++) acc[r][c] = make_float2(0.f, 0.f);
        run_chunks<KERN, RADIAL, TY, RECUR>(acc, a, ig, wbuf, 0, 1, lane);
        float* sp = a.splat + (size_t)it.w * slot_floats + (my * TY) * S + mx * TX;
#pragma unroll
        for (int r = 0; r < TY; r++)
#pragma unroll
            for (int c = 0; c < TX; c += 2) *reinterpret_cast<float2*>(sp + r * S + c) = acc[r][c / 2];
    }
}

// Segment reduce: for every split group (listed by the planner) and sub-window, the
// segment blocks are summed IN SEGMENT ORDER into segment 0's slot.  One CTA per
// (group x sub-window, 1024-float chunk of the slot); float4, 8 segments in flight.
__global__ void __launch_bounds__(256) segreduce_kernel(const int* __restrict__ hot,
                                                        const int* __restrict__ totals,
                                                        const int2* __restrict__ group, int nsub,
                                                        int slot_floats, float* __restrict__ splat) {
    const int e = (blockIdx.x * 256 + threadIdx.x) * 4;
    if (e >= slot_floats) return;
    const int nwork = totals[kTotHot] * nsub;
    const size_t stride = (size_t)nsub * slot_floats;
    for (int gsub = blockIdx.y; gsub < nwork; gsub += gridDim.y) {
        const int2 gr = group[hot[gsub / nsub]];
        const int sub = gsub % nsub;
        float* d0 = splat + ((size_t)gr.x * nsub + sub) * slot_floats + e;
        // 8 loads in flight, 4 partial sums (segment k goes to partial k mod 4 within each
        // group of 8), combined pairwise: a fixed order, so the result is deterministic and
        // band-invariant; the dependent-load chain of the hottest group is n/8 long
        float4 p[4] = {*reinterpret_cast<const float4*>(d0), make_float4(0.f, 0.f, 0.f, 0.f),
                       make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
        int k = 1;
        for (; k + 8 <= gr.y; k += 8) {
            float4 v[8];
#pragma unroll
            for (int q = 0; q < 8; q++) v[q] = *reinterpret_cast<const float4*>(d0 + (k + q) * stride);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                float4& t = p[q & 3];
                t.x += v[q].x; t.y += v[q].y; t.z += v[q].z; t.w += v[q].w;
            }
        }
        for (; k < gr.y; k++) {
            const float4 v = *reinterpret_cast<const float4*>(d0 + k * stride);
            p[0].x += v.x; p[0].y += v.y; p[0].z += v.z; p[0].w += v.w;
        }
        float4 acc;
        acc.x = (p[0].x + p[1].x) + (p[2].x + p[3].x);
        acc.y = (p[0].y + p[1].y) + (p[2].y + p[3].y);
        acc.z = (p[0].z + p[1].z) + (p[2].z + p[3].z);
        acc.w = (p[0].w + p[1].w) + (p[2].w + p[3].w);
        *reinterpret_cast<float4*>(d0) = acc;
    }
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
    const uint8_t* __restrict__ tflag;  // per tile: a planned group's window meets it
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
    if (!a.tflag[(size_t)blockIdx.y * gridDim.x + blockIdx.x]) {  // no group reaches the tile: zeros
        const int i = X0 + (threadIdx.x & 31);
        if (i < g.W)
            for (int j = Y0 + (threadIdx.x >> 5); j <= Y1; j += 8) a.out[(size_t)(j - g.rb) * g.W + i] = 0.f;
        return;
    }
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

// Combine pass for bucket-pitch groups (px = 8, one block per group): one CTA per 8-column
// strip x kStripH rows, each warp 8 columns x kStripH / 8 rows (lane = column lane % 8, rows
// lane / 8 + 4k).
// The strip is one bucket column wide, so a group window covers all of a warp's columns or
// none (for F a multiple of 8; the column test stays for the rest), and a warp skips, as a
// whole, every block whose rows miss its 16: each pixel adds only the blocks that can cover
// it, in the list's order -- the same sum, bit for bit, as combine_kernel (the skipped blocks
// add +0).
constexpr int kStripEnt = 512;

template <int kStripH>  // rows per strip: 256 for tall group pitches (tensor path), else 128
__global__ void __launch_bounds__(256) combine_strip_kernel(const CombineArgs a) {
    constexpr int kStripRW = kStripH / 8, kStripK = kStripRW / 4;  // rows per warp, rows per thread
    __shared__ int4 s_ent[kStripEnt];
    __shared__ int s_n;
    const Geom& g = a.g;
    const PathGeom& pg = a.pg;
    const int X0 = blockIdx.x * 8, X1 = X0 + 7;
    const int Y0 = g.rb + blockIdx.y * kStripH, Y1 = min(Y0 + kStripH, g.re) - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = X0 + (lane & 7);
    const int R0 = Y0 + kStripRW * warp;
    {   // planner flags of the 32 x 32 tiles the strip meets: all clear -> zeros
        const int tx = X0 / kCombTile, ty0 = (Y0 - g.rb) / kCombTile, ty1 = (Y1 - g.rb) / kCombTile;
        const int tfx = (g.W + kCombTile - 1) / kCombTile;
        bool any = false;
        for (int ty = ty0; ty <= ty1; ty++) any |= a.tflag[(size_t)ty * tfx + tx] != 0;
        if (!any) {
            if (i < g.W)
                for (int k = 0; k < kStripK; k++) {
                    const int j = R0 + (lane >> 3) + 4 * k;
                    if (j <= Y1) a.out[(size_t)(j - g.rb) * g.W + i] = 0.f;
                }
            return;
        }
    }
    const int F = g.F;
    const int gxa = max(floor_div(X0 - F, pg.px), 0), gxb = min(floor_div(X1 + F, pg.px), pg.ngx - 1);
    const int gya = max(floor_div(Y0 - F, pg.py), 0), gyb = min(floor_div(Y1 + F, pg.py), pg.ngy - 1);
    const int ngxr = gxb - gxa + 1, ng = ngxr * (gyb - gya + 1);
    if (threadIdx.x < 32) {  // the blocks meeting the strip, group row-major (as combine_kernel)
        int n = 0;
        for (int gi0 = 0; gi0 < ng; gi0 += 32) {
            const int gi = gi0 + lane;
            const int gy = gya + gi / ngxr, gx = gxa + gi % ngxr;
            int2 gr = make_int2(0, 0);
            if (gi < ng) gr = a.group[gy * pg.ngx + gx];
            const int wx0 = gx * pg.px - F, wy0 = gy * pg.py - F;
            const bool meet = gi < ng && gr.y > 0 && X1 >= wx0 && X0 <= wx0 + pg.ww - 1 && Y1 >= wy0 &&
                              Y0 <= wy0 + pg.wh - 1;
            const unsigned m = __ballot_sync(0xffffffffu, meet);
            if (meet) {
                const int pos = n + __popc(m & ((1u << lane) - 1u));
                if (pos < kStripEnt) s_ent[pos] = make_int4(gr.x, wx0, wy0, pg.ww | (pg.wh << 16));
            }
            n += __popc(m);
        }
        if (lane == 0) s_n = min(n, kStripEnt);
    }
    __syncthreads();
    const int n = s_n;
    const int sl = pg.slot_w;
    const size_t sf = (size_t)pg.slot_floats();
    const int r0 = lane >> 3;
    float acc[kStripK];
#pragma unroll
    for (int k = 0; k < kStripK; k++) acc[k] = 0.f;
    for (int e = 0; e < n; e++) {
        const int4 en = s_ent[e];
        const int sh = en.w >> 16;
        if (en.z > R0 + kStripRW - 1 || en.z + sh <= R0) continue;  // warp-uniform: the block misses its rows
        const int li = i - en.y;
        const bool inx = (unsigned)li < (unsigned)(en.w & 0xffff);
        const float* sp = a.splat + (size_t)en.x * sf + li;
        float v[kStripK];
#pragma unroll
        for (int k = 0; k < kStripK; k++) {
            const int lj = R0 + r0 + 4 * k - en.z;
            v[k] = (inx && (unsigned)lj < (unsigned)sh) ? sp[(size_t)lj * sl] : 0.f;
        }
#pragma unroll
        for (int k = 0; k < kStripK; k++) acc[k] += v[k];
    }
    if (i >= g.W) return;
    const unsigned long long nf = a.stats[0];
    const float scale = nf ? (float)(a.c_over_h2 / (double)nf) : 0.f;
#pragma unroll
    for (int k = 0; k < kStripK; k++) {
        const int j = R0 + r0 + 4 * k;
        if (j <= Y1) a.out[(size_t)(j - g.rb) * g.W + i] = acc[k] * scale;
    }
}

template <int K, bool RAD, int TY, bool REC>
static int launch_ty(const SplatArgs& a, int grid, cudaStream_t s) {
    const size_t smem = sizeof(float) * WLayout<TY>::SMEM_FLOATS;
    if (grid <= 0) {  // configure + query: persistent CTAs per SM
        cudaFuncSetAttribute(splat_kernel<K, RAD, TY, REC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int nb = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, splat_kernel<K, RAD, TY, REC>, kWarps * 32, smem);
        return nb > 0 ? nb : 1;
    }
    splat_kernel<K, RAD, TY, REC><<<grid, kWarps * 32, smem, s>>>(a);
    return 0;
}

template <int K, bool RAD, int TY>
static int launch_ty(const SplatArgs& a, int grid, cudaStream_t s) {
    // the Gaussian's exact-ratio recurrence, when its range stays normal (a.recur)
    if constexpr (K == 6 && !RAD)
        if (a.recur) return launch_ty<K, RAD, TY, true>(a, grid, s);
    return launch_ty<K, RAD, TY, false>(a, grid, s);
}

template <int K, bool RAD>
static int launch_one(const SplatArgs& a, int ty, int grid, cudaStream_t s) {
    switch (ty) {
    case 2: return launch_ty<K, RAD, 2>(a, grid, s);
    case 3: return launch_ty<K, RAD, 3>(a, grid, s);
    case 4: return launch_ty<K, RAD, 4>(a, grid, s);
    case 5: return launch_ty<K, RAD, 5>(a, grid, s);
    default: return launch_ty<K, RAD, 6>(a, grid, s);
    }
}

using LaunchFn = int (*)(const SplatArgs&, int, int, cudaStream_t);
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
    {   // split groups (count on the device): sum their segments first, in segment order
        const int sf = (int)pl.pg.slot_floats();
        const int gx = (sf / 4 + 255) / 256;
        dim3 grid(gx, std::max(1, 148 * 16 / gx));
        segreduce_kernel<<<grid, 256, 0, s>>>(pl.d_hot, pl.d_totals, pl.d_group, pl.pg.nsub(), sf, pl.d_splat);
        c->launches += 1;
    }
    CombineArgs a;
    a.g = g;
    a.pg = pl.pg;
    a.group = pl.d_group;
    a.tflag = pl.d_tflag;
    a.splat = pl.d_splat;
    a.out = out;
    a.stats = c->d_stats;
    a.c_over_h2 = kernel_constant(c->kern, c->radial) / (c->hpx * c->hpx);
    const PathGeom& pg = pl.pg;
    // strips of 256 rows when the group pitch is tall (tensor-core stacks: fewer block lists
    // per pixel), else 128 (measured: C4 tensor 0.174 -> 0.167 ms at 256, direct 0.255 -> 0.264)
    const int sh = pg.py >= 32 ? 256 : 128;
    const int strip_ent = ((8 + 2 * g.F) / pg.px + 2) * ((sh + 2 * g.F) / pg.py + 2);
    const char* env_s = getenv("KDE_COMBINE_STRIP");  // 0: the 32 x 32-tile kernel (tests, A/B)
    const bool env_strip = !env_s || atoi(env_s) != 0;
    if (env_strip && pg.px == 8 && pg.nsub() == 1 && strip_ent <= kStripEnt) {
        dim3 grid((g.W + 7) / 8, (g.re - g.rb + sh - 1) / sh);
        if (sh == 256) combine_strip_kernel<256><<<grid, 256, 0, s>>>(a);
        else combine_strip_kernel<128><<<grid, 256, 0, s>>>(a);
    } else {
        dim3 grid((g.W + kCombTile - 1) / kCombTile, (g.re - g.rb + kCombTile - 1) / kCombTile);
        combine_kernel<<<grid, 256, 0, s>>>(a);
    }
    c->launches += 1;
    return KDE_OK;
}

int launch_direct(kde_ctx* c, float* out, cudaStream_t s) {
    EvalPlan& pl = c->plan[KDE_PATH_DIRECT];
    SplatArgs a;
    a.g = c->g;
    a.offsets = c->d_offsets;
    a.xy = c->pb.xy;
    a.rng = c->pb.rng;
    a.items = pl.d_items;
    a.group = pl.d_group;
    a.totals = pl.d_totals;
    a.splat = pl.d_splat;
    a.pg = pl.pg;
    a.k = make_kconst(c->hpx);
    a.c2 = (float)(c->ceff * c->ceff);
    a.q2 = (float)exp2(2.0 * (double)a.k.kq);
    a.recur = -(double)a.k.kq * (c->g.R + 8.0) * (c->g.R + 8.0) < 120.0;
    LaunchFn fn = kSplat[c->radial ? 1 : 0][c->kern];
    if (pl.grid <= 0) {
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->p.device);
        pl.grid = nsm * fn(a, pl.mt, 0, s);
    }
    cudaMemsetAsync(pl.d_totals + kTotQueue, 0, 2 * sizeof(int), s);  // work-queue heads
    tmark(c, 3, s);
    fn(a, pl.mt, pl.grid, s);  // persistent; the item count is on the device
    c->launches += 1;
    c->main_kernel = 1;
    tmark(c, 4, s);
    launch_combine(c, pl, out, s);
    tmark(c, 5, s);
    c->tev_eval = c->timing;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "direct eval launch");
    return KDE_OK;
}

}  // namespace kde
