// Device-side evaluation plan: from the bucket offsets, with no host
// round trip except one 16-byte read of the totals.
//
//   plan_count    per bucket b whose window meets the band: full_b = cnt/kSegPts full
//                 segments, part_b = [cnt % kSegPts != 0], nseg_b = full_b + part_b
//   3 scans       exclusive scans of full_b, part_b, nseg_b
//   plan_finish   group[b] = (first slot, nseg) and the totals (TF, TP, nslots)
//   plan_scatter  the item list: all full segments first (equal work), then the partial
//                 ones; item = (bucket, k0, k1, slot), slot = (seg_scan_b + seg)*nsub + sub
//
// The plan depends only on each bucket's own count, so a banded context plans every
// group it shares with the unbanded one identically (bitwise sharding).
#include "internal.cuh"

namespace kde {

int scan_excl_u32(uint32_t* a, int64_t L, uint32_t* tmp, cudaStream_t s);  // bin.cu

__device__ __forceinline__ bool window_meets_band(const Geom& g, int by) {
    const int wy0 = by * g.B - g.F, wy1 = wy0 + g.B + 2 * g.F - 1;
    return wy1 >= g.rb && wy0 <= g.re - 1;
}

__global__ void plan_count_kernel(const Geom g, const uint32_t* __restrict__ off, int nb,
                                  uint32_t* __restrict__ full, uint32_t* __restrict__ part,
                                  uint32_t* __restrict__ nseg) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += gridDim.x * blockDim.x) {
        uint32_t f = 0, p = 0;
        if (b < nb && window_meets_band(g, b / g.nbx)) {
            const uint32_t cnt = off[b + 1] - off[b];
            f = cnt / kSegPts;
            p = (cnt % kSegPts) ? 1u : 0u;
        }
        full[b] = f;  // entry nb stays 0: the exclusive scan then ends with the total
        part[b] = p;
        nseg[b] = f + p;
    }
}

__global__ void plan_finish_kernel(const uint32_t* __restrict__ off,
                                   const uint32_t* __restrict__ full_s,
                                   const uint32_t* __restrict__ part_s,
                                   const uint32_t* __restrict__ nseg_s, int nb, int nsub,
                                   int2* __restrict__ group, int* __restrict__ totals) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x)
        group[b] = make_int2((int)nseg_s[b] * nsub, (int)(nseg_s[b + 1] - nseg_s[b]));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        totals[0] = (int)full_s[nb];            // full segments
        totals[1] = (int)part_s[nb];            // partial segments
        totals[2] = (int)nseg_s[nb] * nsub;     // slots
        totals[3] = (int)off[nb];               // points binned
    }
}

// one thread per bucket: write its items (full segments into [0, TF*nsub), the partial
// one into [TF*nsub, (TF+TP)*nsub)), sub-window index fastest
__global__ void plan_scatter_kernel(const uint32_t* __restrict__ off,
                                    const uint32_t* __restrict__ full_s,
                                    const uint32_t* __restrict__ part_s,
                                    const uint32_t* __restrict__ nseg_s, int nb, int nsub,
                                    int TF, int4* __restrict__ items) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
        const int nf = (int)(full_s[b + 1] - full_s[b]);
        const int np = (int)(part_s[b + 1] - part_s[b]);
        if (nf + np == 0) continue;
        const int cnt = (int)(off[b + 1] - off[b]);
        const int sb = (int)nseg_s[b];
        for (int sg = 0; sg < nf; sg++)
            for (int sub = 0; sub < nsub; sub++)
                items[((int)full_s[b] + sg) * nsub + sub] =
                    make_int4(b, sg * kSegPts, (sg + 1) * kSegPts, (sb + sg) * nsub + sub);
        if (np)
            for (int sub = 0; sub < nsub; sub++)
                items[(TF + (int)part_s[b]) * nsub + sub] =
                    make_int4(b, nf * kSegPts, cnt, (sb + nf) * nsub + sub);
    }
}

static int grid_for(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

// Enqueue plan_count, the scans and plan_finish on the context stream; totals land in
// c->plan.d_totals (device) -- the caller reads them back.
int plan_device(kde_ctx* c) {
    EvalPlan& pl = c->plan;
    const Geom& g = c->g;
    const int nb = g.nbx * g.nby;
    cudaStream_t s = c->stream;
    plan_count_kernel<<<grid_for(nb + 1), 256, 0, s>>>(g, c->d_offsets, nb, pl.d_full, pl.d_part,
                                                       pl.d_nseg);
    c->launches += 1;
    c->launches += scan_excl_u32(pl.d_full, nb + 1, pl.d_scan_tmp, s);
    c->launches += scan_excl_u32(pl.d_part, nb + 1, pl.d_scan_tmp, s);
    c->launches += scan_excl_u32(pl.d_nseg, nb + 1, pl.d_scan_tmp, s);
    plan_finish_kernel<<<grid_for(nb), 256, 0, s>>>(c->d_offsets, pl.d_full, pl.d_part, pl.d_nseg, nb,
                                                    pl.nsubx * pl.nsubx, pl.d_group, pl.d_totals);
    c->launches += 1;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "plan launch");
    return KDE_OK;
}

int plan_scatter(kde_ctx* c) {
    EvalPlan& pl = c->plan;
    const int nb = c->g.nbx * c->g.nby;
    plan_scatter_kernel<<<grid_for(nb), 256, 0, c->stream>>>(c->d_offsets, pl.d_full, pl.d_part,
                                                            pl.d_nseg, nb, pl.nsubx * pl.nsubx,
                                                            pl.tf, pl.d_items);
    c->launches += 1;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "plan scatter launch");
    return KDE_OK;
}

}  // namespace kde
