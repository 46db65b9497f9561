// Internal declarations of libkde (not part of the ABI; include/kde.h is).
// DESIGN.md §6 describes the HBM layout and every kernel below.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "kde.h"

namespace kde {

constexpr int kBucket = 32;       // bucket edge B (pixels); divides every tile edge
constexpr int kDirTile = 64;      // direct-path tile edge (pixels)
constexpr int kSegCands = 8192;   // direct split-K: candidates per work item (fixed ->
                                  // plan is invariant under band sharding)
constexpr int kTcM = 128;         // tensor-core tile rows (TMEM lanes)
constexpr int kTcN = 256;         // tensor-core tile columns (TMEM fp32 columns)
constexpr int kTcSegCands = 16384;

// Geometry shared by every kernel (passed by value).
struct Geom {
    double x0, y0, res;   // raster origin / pixel edge (world units)
    double R;             // support half-width in pixels, c_eff * h/res (fp64)
    int W, H;             // raster
    int rb, re;           // band rows [rb, re)
    int nbx, nby;         // bucket grid
    int reach;            // ceil(R + 1/2) + 1 (pixels)
    int nr;               // neighbourhood radius in buckets, ceil(reach / B)
    int band_lo, band_hi; // kept bucket rows (home-bucket band filter)
};

// One CTA of an evaluation pass: tile (tx, ty), candidate positions [k0, k1) of the
// tile's neighbourhood list, partial slot (-1: write scaled result to the raster).
struct WorkItem {
    int tx, ty;
    int k0, k1;
    int slot;
    int pad_;
};
struct ReduceItem {
    int tx, ty;
    int slot0, nseg;
};

// Point-sized device buffers (capacity grows, never shrinks).
struct PointBufs {
    int64_t cap = 0;
    double *x = nullptr, *y = nullptr;         // staging of host inputs
    int64_t stage_cap = 0;
    uint32_t *key[2] = {nullptr, nullptr};     // radix ping-pong
    uint32_t *val[2] = {nullptr, nullptr};
    uint32_t *hist = nullptr;                  // radix per-(digit, block) counts
    int64_t hist_cap = 0;
    uint32_t *scan_tmp = nullptr;
    float2 *xy = nullptr;                      // sorted bucket-local coordinates
    uint2 *rng = nullptr;                      // sorted packed int16 ranges
    uint32_t *perm = nullptr;                  // sorted -> original index (alias)
};

struct EvalPlan {
    int ntx = 0, nty0 = 0, nty1 = 0;           // tile columns, tile rows [nty0, nty1)
    std::vector<WorkItem> items;
    std::vector<ReduceItem> reds;
    int nslots = 0;
    bool any_empty = false;
    WorkItem* d_items = nullptr;
    int d_items_cap = 0;
    ReduceItem* d_reds = nullptr;
    int d_reds_cap = 0;
    float* d_partial = nullptr;
    int64_t partial_cap = 0;                   // floats
};

}  // namespace kde

struct kde_ctx {
    kde_params p;
    kde::Geom g;
    double hpx = 0, ceff = 0;
    int kern = 0;
    bool radial = false;
    cudaStream_t stream = nullptr;             // internal stream (loads)
    kde::PointBufs pb;
    uint32_t* d_offsets = nullptr;             // nb + 1
    unsigned long long* d_stats = nullptr;     // n_finite, n_outside, useful_pairs
    std::vector<uint32_t> h_offsets;
    kde_stats stats{};
    bool loaded = false;
    int64_t launches = 0;                      // kernels launched (kde_stats.kernel_launches)
    kde::EvalPlan plan_dir, plan_tc;
};

namespace kde {

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

// binning (bin.cu)
int bin_points(kde_ctx* c, const double* d_x, const double* d_y, int64_t n);
// evaluation (eval_direct.cu, eval_tc.cu)
int launch_direct(kde_ctx* c, float* out, cudaStream_t s);
int launch_tc(kde_ctx* c, float* out, cudaStream_t s);
int build_plan(kde_ctx* c, int tile_w, int tile_h, int seg, EvalPlan& pl, int64_t slot_floats);

}  // namespace kde
