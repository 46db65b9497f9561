// Device-side evaluation plan, three kernels per path, built lazily by the
// first kde_eval of a path after a load, and no host round trip: the totals stay on the
// device (kTot* in internal.cuh) and the buffers are reserved at their upper bounds.  A
// path's group is a vertical stack of pg.s buckets (1 for the direct path).
//
//   plan_local    per group g whose window meets the band: cnt_g = sum of its buckets'
//                 counts, full_g = cnt_g / pg.seg_pts full segments, part_g =
//                 ceil((cnt_g % pg.seg_pts) / pg.part_pts) remainder pieces;
//                 block-local exclusive scan of the packed pair (full_g << 32 | part_g)
//   plan_blocks   one CTA: exclusive scan of the block totals
//   plan_finish   global prefixes -> group[g] = (first segment, #segments), the item list
//                 (all full segments first -- equal work -- then the remainder pieces of
//                 <= pg.part_pts points, segment = full segment or remainder piece;
//                 item = (g, k0, k1, slot), slot = (first segment + seg)*nsub + sub, [k0, k1)
//                 absolute sorted positions: a group is one contiguous range) and totals
//
// The plan depends only on each group's own counts, so a banded context plans every group
// it shares with the unbanded one identically (bitwise sharding).
#include "internal.cuh"

namespace kde {

constexpr int kPlanThreads = 256;
constexpr int kPlanPer = 1;  // groups per thread (more CTAs: the plan is latency-bound)
constexpr int kPlanTile = kPlanThreads * kPlanPer;

// Bucket keys are column-major (key = bx * nby + by), so a group -- a vertical stack of
// pg.s buckets -- is the contiguous key range [gx*nby + gy*s, + min(s, nby - gy*s)).
__device__ __forceinline__ uint32_t group_count(const Geom& g, const PathGeom& pg,
                                                const uint32_t* __restrict__ off, int gx, int gy) {
    const int k0 = gx * g.nby + gy * pg.s;
    const int k1 = k0 + min(pg.s, g.nby - gy * pg.s);
    return off[k1] - off[k0];
}

__device__ __forceinline__ uint64_t group_pair(const Geom& g, const PathGeom& pg,
                                               const uint32_t* __restrict__ off, int i, uint32_t* cnt) {
    *cnt = 0;
    if (i >= pg.ngroups()) return 0;
    const int gx = i % pg.ngx, gy = i / pg.ngx;
    const int wy0 = gy * pg.py - g.F, wy1 = wy0 + pg.wh - 1;
    if (wy1 < g.rb || wy0 > g.re - 1) return 0;  // window misses the band
    const uint32_t c = group_count(g, pg, off, gx, gy);
    *cnt = c;
    const uint32_t rem = c % pg.seg_pts;
    return ((uint64_t)(c / pg.seg_pts) << 32) | (uint64_t)((rem + pg.part_pts - 1) / pg.part_pts);
}

// block-wide exclusive scan of one u64 per thread (kPlanThreads threads); returns the total
__device__ __forceinline__ uint64_t block_scan_u64(uint64_t v, uint64_t* s_warp, uint64_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += x;
    }
    if (lane == 31) s_warp[w] = inc;
    __syncthreads();
    uint64_t pre = 0, tot = 0;
    for (int k = 0; k < kPlanThreads / 32; k++) {
        pre += (k < w) ? s_warp[k] : 0;
        tot += s_warp[k];
    }
    *total = tot;
    return pre + inc - v;
}

__global__ void __launch_bounds__(kPlanThreads) plan_local_kernel(const Geom g, const PathGeom pg,
                                                                  const uint32_t* __restrict__ off,
                                                                  uint64_t* __restrict__ local,
                                                                  uint64_t* __restrict__ bsum) {
    __shared__ uint64_t s_warp[kPlanThreads / 32];
    const int i0 = blockIdx.x * kPlanTile + threadIdx.x * kPlanPer;
    uint64_t v[kPlanPer], sum = 0;
    uint32_t c;
#pragma unroll
    for (int k = 0; k < kPlanPer; k++) {
        v[k] = group_pair(g, pg, off, i0 + k, &c);
        sum += v[k];
    }
    uint64_t tot;
    uint64_t run = block_scan_u64(sum, s_warp, &tot);
#pragma unroll
    for (int k = 0; k < kPlanPer; k++) {
        if (i0 + k <= pg.ngroups()) local[i0 + k] = run;
        run += v[k];
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// one CTA: exclusive scan of the block totals, in place; bsum[nblk] = grand total.  Each
// thread owns a run of consecutive totals (sequential), one block scan joins the runs.
__global__ void __launch_bounds__(kPlanThreads) plan_blocks_kernel(uint64_t* __restrict__ bsum, int nblk) {
    __shared__ uint64_t s_warp[kPlanThreads / 32];
    const int per = (nblk + kPlanThreads - 1) / kPlanThreads;
    const int b0 = threadIdx.x * per, b1 = min(b0 + per, nblk);
    uint64_t sum = 0;
    for (int b = b0; b < b1; b++) sum += bsum[b];
    uint64_t tot;
    uint64_t run = block_scan_u64(sum, s_warp, &tot);
    for (int b = b0; b < b1; b++) {
        const uint64_t v = bsum[b];
        bsum[b] = run;
        run += v;
    }
    if (threadIdx.x == 0) bsum[nblk] = tot;
}

__global__ void __launch_bounds__(kPlanThreads) plan_finish_kernel(
    const Geom g, const PathGeom pg, const uint32_t* __restrict__ off, const uint64_t* __restrict__ local,
    const uint64_t* __restrict__ bsum, int nblk, int2* __restrict__ group, int4* __restrict__ items,
    int* __restrict__ totals, int* __restrict__ hot, uint8_t* __restrict__ tflag, int tfx, int tfy) {
    const uint64_t T = bsum[nblk];
    const int TF = (int)(T >> 32);
    const int nsub = pg.nsub(), ng = pg.ngroups();
    const int lane = threadIdx.x & 31;
    const int i0 = blockIdx.x * kPlanTile + threadIdx.x * kPlanPer;
    const uint64_t base = bsum[blockIdx.x];
    uint32_t chunks = 0;  // MMA chunks of this thread's groups (tensor-core flop count)
#pragma unroll
    for (int k = 0; k < kPlanPer; k++) {
        const int i = i0 + k;
        int fs = 0, ps = 0, nf = 0, np = 0, gst = 0;
        uint32_t cnt = 0;
        if (i < ng) {
            const uint64_t pre = base + local[i];
            const uint64_t own = group_pair(g, pg, off, i, &cnt);
            fs = (int)(pre >> 32);
            ps = (int)(pre & 0xffffffffu);
            nf = (int)(own >> 32);
            np = (int)(own & 0xffffffffu);
            group[i] = make_int2(fs + ps, nf + np);  // first segment (numbered group by group)
            gst = (int)off[(i % pg.ngx) * g.nby + (i / pg.ngx) * pg.s];  // group's first position
            if (nf + np > 1) hot[atomicAdd(&totals[kTotHot], 1)] = i;  // split group: segment reduce
            if (nf + np > 0) {  // the combine tiles (band-relative) its window meets are non-empty
                const int wx0 = (i % pg.ngx) * pg.px - g.F, wy0 = (i / pg.ngx) * pg.py - g.F - g.rb;
                const int tx0 = max(wx0, 0) / kCombTile, tx1 = min((wx0 + pg.ww - 1) / kCombTile, tfx - 1);
                const int ty0 = max(wy0, 0) / kCombTile;
                const int ty1 = wy0 + pg.wh - 1 >= 0 ? min((wy0 + pg.wh - 1) / kCombTile, tfy - 1) : -1;
                for (int ty = ty0; ty <= ty1; ty++)
                    for (int tx = tx0; tx <= tx1; tx++) tflag[(size_t)ty * tfx + tx] = 1;
            }
            chunks += ((uint32_t)nf * (pg.seg_pts / pg.chunk_pts) +
                       ((cnt % pg.seg_pts) + pg.chunk_pts - 1) / pg.chunk_pts) * (uint32_t)nsub;
        }
        // items: a group with few is written by its own thread; the rest (hot groups have
        // hundreds) by the whole warp, one group at a time
        const int nit = (nf + np) * nsub;
        const bool big = nit > 8;
        const int sb = fs + ps;
        if (!big) {
            for (int e = 0; e < nf * nsub; e++) {
                const int sg = e / nsub, sub = e % nsub;
                items[(fs + sg) * nsub + sub] =
                    make_int4(i, gst + sg * pg.seg_pts, gst + (sg + 1) * pg.seg_pts, (sb + sg) * nsub + sub);
            }
            for (int e = 0; e < np * nsub; e++) {
                const int kk = e / nsub, sub = e % nsub;
                const int k0 = nf * pg.seg_pts + kk * pg.part_pts, k1 = min(k0 + pg.part_pts, (int)cnt);
                items[(TF + ps + kk) * nsub + sub] = make_int4(i, gst + k0, gst + k1, (sb + nf + kk) * nsub + sub);
            }
        }
        uint32_t m = __ballot_sync(0xffffffffu, big);
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const int gi = __shfl_sync(0xffffffffu, i, src);
            const int gfs = __shfl_sync(0xffffffffu, fs, src), gps = __shfl_sync(0xffffffffu, ps, src);
            const int gnf = __shfl_sync(0xffffffffu, nf, src), gnp = __shfl_sync(0xffffffffu, np, src);
            const int gcnt = (int)__shfl_sync(0xffffffffu, cnt, src);
            const int ggst = __shfl_sync(0xffffffffu, gst, src);
            const int gsb = gfs + gps;
            for (int e = lane; e < gnf * nsub; e += 32) {  // full segments
                const int sg = e / nsub, sub = e % nsub;
                items[(gfs + sg) * nsub + sub] =
                    make_int4(gi, ggst + sg * pg.seg_pts, ggst + (sg + 1) * pg.seg_pts, (gsb + sg) * nsub + sub);
            }
            for (int e = lane; e < gnp * nsub; e += 32) {  // the remainder's pieces of <= part_pts
                const int kk = e / nsub, sub = e % nsub;
                const int k0 = gnf * pg.seg_pts + kk * pg.part_pts, k1 = min(k0 + pg.part_pts, gcnt);
                items[(TF + gps + kk) * nsub + sub] = make_int4(gi, ggst + k0, ggst + k1, (gsb + gnf + kk) * nsub + sub);
            }
        }
    }
    chunks = __reduce_add_sync(0xffffffffu, chunks);
    if (lane == 0 && chunks) atomicAdd(&totals[kTotChunks], (int)chunks);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        totals[kTotFull] = TF;
        totals[kTotPart] = (int)(T & 0xffffffffu);
        totals[kTotSlots] = (TF + (int)(T & 0xffffffffu)) * nsub;
        totals[kTotBinned] = (int)off[g.nbx * g.nby];
    }
}

int plan_nblk(const PathGeom& pg) { return (pg.ngroups() + 1 + kPlanTile - 1) / kPlanTile; }

// Enqueue the three plan kernels of one path on stream s; the item list must already have
// its upper-bound capacity; totals land in pl.d_totals.
int plan_device(kde_ctx* c, EvalPlan& pl, cudaStream_t s) {
    const PathGeom& pg = pl.pg;
    const int nblk = plan_nblk(pg);
    cudaMemsetAsync(pl.d_totals, 0, sizeof(int) * kTotInts, s);  // counters start at zero
    cudaMemsetAsync(pl.d_tflag, 0, (size_t)pl.tfx * pl.tfy, s);
    plan_local_kernel<<<nblk, kPlanThreads, 0, s>>>(c->g, pg, c->d_offsets, pl.d_local, pl.d_bsum);
    plan_blocks_kernel<<<1, kPlanThreads, 0, s>>>(pl.d_bsum, nblk);
    plan_finish_kernel<<<nblk, kPlanThreads, 0, s>>>(c->g, pg, c->d_offsets, pl.d_local, pl.d_bsum,
                                                     nblk, pl.d_group, pl.d_items, pl.d_totals, pl.d_hot,
                                                     pl.d_tflag, pl.tfx, pl.tfy);
    c->launches += 3;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "plan launch");
    return KDE_OK;
}

}  // namespace kde
