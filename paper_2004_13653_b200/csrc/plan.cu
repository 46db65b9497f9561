// Device-side evaluation plan: from the bucket offsets, with no host
// round trip except one 16-byte read of the totals.  One plan per evaluation path; a
// path's group is a vertical stack of pg.s buckets (1 for the direct path).
//
//   plan_count    per group g whose window meets the band: cnt_g = sum of its buckets'
//                 counts; full_g = cnt_g / kSegPts segments, part_g = [cnt_g % kSegPts != 0]
//   3 scans       exclusive scans of full_g, part_g, nseg_g = full_g + part_g
//   plan_finish   group[g] = (first segment, nseg_g) and the totals (TF, TP, nslots, binned)
//   plan_scatter  the item list: all full segments first (equal work), then the partial
//                 ones; item = (g, k0, k1, slot), slot = (seg_scan_g + seg)*nsub + sub, where
//                 [k0, k1) are positions in the concatenation of the group's bucket ranges
//
// The plan depends only on each group's own counts, so a banded context plans every group
// it shares with the unbanded one identically (bitwise sharding).
#include "internal.cuh"

namespace kde {

int scan_excl_u32(uint32_t* a, int64_t L, uint32_t* tmp, cudaStream_t s);  // bin.cu

__device__ __forceinline__ uint32_t group_count(const Geom& g, const PathGeom& pg,
                                                const uint32_t* __restrict__ off, int gx, int gy) {
    uint32_t c = 0;
    for (int k = 0; k < pg.s; k++) {
        const int by = gy * pg.s + k;
        if (by >= g.nby) break;
        const int key = by * g.nbx + gx;
        c += off[key + 1] - off[key];
    }
    return c;
}

__global__ void plan_count_kernel(const Geom g, const PathGeom pg, const uint32_t* __restrict__ off,
                                  uint32_t* __restrict__ full, uint32_t* __restrict__ part,
                                  uint32_t* __restrict__ nseg) {
    const int ng = pg.ngroups();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= ng; i += gridDim.x * blockDim.x) {
        uint32_t f = 0, p = 0;
        if (i < ng) {
            const int gx = i % pg.ngx, gy = i / pg.ngx;
            const int wy0 = gy * pg.py - g.F, wy1 = wy0 + pg.wh - 1;
            if (wy1 >= g.rb && wy0 <= g.re - 1) {  // window meets the band
                const uint32_t cnt = group_count(g, pg, off, gx, gy);
                f = cnt / kSegPts;
                p = (cnt % kSegPts) ? 1u : 0u;
            }
        }
        full[i] = f;  // entry ng stays 0: the exclusive scan then ends with the total
        part[i] = p;
        nseg[i] = f + p;
    }
}

__global__ void plan_finish_kernel(const uint32_t* __restrict__ off, int nb,
                                   const uint32_t* __restrict__ full_s,
                                   const uint32_t* __restrict__ part_s,
                                   const uint32_t* __restrict__ nseg_s, int ng, int nsub,
                                   int2* __restrict__ group, int* __restrict__ totals) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ng; i += gridDim.x * blockDim.x)
        group[i] = make_int2((int)nseg_s[i], (int)(nseg_s[i + 1] - nseg_s[i]));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        totals[0] = (int)full_s[ng];            // full segments
        totals[1] = (int)part_s[ng];            // partial segments
        totals[2] = (int)nseg_s[ng] * nsub;     // slots
        totals[3] = (int)off[nb];               // points binned
    }
}

// one thread per group: write its items (full segments into [0, TF*nsub), the partial one
// into [TF*nsub, (TF+TP)*nsub)), sub-window index fastest
__global__ void plan_scatter_kernel(const Geom g, const PathGeom pg, const uint32_t* __restrict__ off,
                                    const uint32_t* __restrict__ full_s,
                                    const uint32_t* __restrict__ part_s,
                                    const uint32_t* __restrict__ nseg_s, int TF,
                                    int4* __restrict__ items) {
    const int ng = pg.ngroups(), nsub = pg.nsub();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ng; i += gridDim.x * blockDim.x) {
        const int nf = (int)(full_s[i + 1] - full_s[i]);
        const int np = (int)(part_s[i + 1] - part_s[i]);
        if (nf + np == 0) continue;
        const int cnt = (int)group_count(g, pg, off, i % pg.ngx, i / pg.ngx);
        const int sb = (int)nseg_s[i];
        for (int sg = 0; sg < nf; sg++)
            for (int sub = 0; sub < nsub; sub++)
                items[((int)full_s[i] + sg) * nsub + sub] =
                    make_int4(i, sg * kSegPts, (sg + 1) * kSegPts, (sb + sg) * nsub + sub);
        if (np)
            for (int sub = 0; sub < nsub; sub++)
                items[(TF + (int)part_s[i]) * nsub + sub] =
                    make_int4(i, nf * kSegPts, cnt, (sb + nf) * nsub + sub);
    }
}

static int grid_for(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

// Enqueue plan_count, the scans and plan_finish on the context stream; totals land in
// pl.d_totals (device) -- the caller reads them back.
int plan_device(kde_ctx* c, EvalPlan& pl) {
    const Geom& g = c->g;
    const PathGeom& pg = pl.pg;
    const int ng = pg.ngroups();
    cudaStream_t s = c->stream;
    plan_count_kernel<<<grid_for(ng + 1), 256, 0, s>>>(g, pg, c->d_offsets, pl.d_full, pl.d_part,
                                                       pl.d_nseg);
    c->launches += 1;
    c->launches += scan_excl_u32(pl.d_full, ng + 1, pl.d_scan_tmp, s);
    c->launches += scan_excl_u32(pl.d_part, ng + 1, pl.d_scan_tmp, s);
    c->launches += scan_excl_u32(pl.d_nseg, ng + 1, pl.d_scan_tmp, s);
    plan_finish_kernel<<<grid_for(ng), 256, 0, s>>>(c->d_offsets, g.nbx * g.nby, pl.d_full,
                                                    pl.d_part, pl.d_nseg, ng, pg.nsub(),
                                                    pl.d_group, pl.d_totals);
    c->launches += 1;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "plan launch");
    return KDE_OK;
}

int plan_scatter(kde_ctx* c, EvalPlan& pl) {
    const int ng = pl.pg.ngroups();
    plan_scatter_kernel<<<grid_for(ng), 256, 0, c->stream>>>(c->g, pl.pg, c->d_offsets, pl.d_full,
                                                            pl.d_part, pl.d_nseg, pl.tf, pl.d_items);
    c->launches += 1;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "plan scatter launch");
    return KDE_OK;
}

}  // namespace kde
