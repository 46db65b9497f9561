// Internal declarations of libkde (not part of the ABI; include/kde.h is).
// DESIGN.md §6 describes the HBM layout and every kernel below.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "kde.h"

namespace kde {

constexpr int kSubMax = 48;       // direct-path sub-window edge bound (pixels): S = 8 TY <= 48
// split-K: points per full splat work item ("segment"), chosen per load from the global
// point count (seg_pts_for below) -- the same on every rank, so the plan is invariant under
// band sharding; <= 4096 keeps every per-warp fp32 running sum of the direct
// path within 512 terms (R10)
constexpr int kSegMin = 512, kSegMax = 4096;
constexpr int64_t kSegShareCtas = 1184;  // 148 SMs x 8 work streams (direct path)
constexpr int64_t kSegShareTc = 4736;    // 148 SMs x 16 per-warp pipelines (eval_tc5.cu) x 2
inline int seg_pts_for(int64_t n, int64_t share = kSegShareCtas) {
    int seg = kSegMin;
    while (seg < kSegMax && 3 * (int64_t)(2 * seg) <= 2 * (n / share)) seg *= 2;
    return seg;
}
constexpr int kPartPtsDirect = 128;  // direct path: smallest remainder piece (one warp's work item)
constexpr int kCombTile = 32;     // combine-pass output tile edge
constexpr int kTcM = 128;         // tensor-core tile rows = TMEM lanes

// Geometry shared by every kernel (passed by value).
struct Geom {
    double x0, y0, res;   // raster origin / pixel edge (world units)
    double R;             // support half-width in pixels, c_eff * h/res (fp64)
    int W, H;             // raster
    int rb, re;           // band rows [rb, re)
    int B;                // bucket (point group) edge in pixels (power of two)
    int lgB;              // log2(B)
    int F;                // floor(R + 1/2): window half-extent beyond the bucket (pixels)
    int nbx, nby;         // bucket grid
    int reach;            // ceil(R + 1/2) + 1 (pixels)
    int nr;               // neighbourhood radius in buckets, ceil(reach / B)
    int band_lo, band_hi; // kept bucket rows (home-bucket band filter)
};

// Point-sized device buffers (capacity grows, never shrinks).
struct PointBufs {
    int64_t cap = 0;
    double *sx[2] = {nullptr, nullptr};        // double-buffered staging of host inputs
    double *sy[2] = {nullptr, nullptr};
    int64_t stage_cap[2] = {0, 0};
    int stage = 0;                             // staging buffer of the next host load
    uint32_t *key[1] = {nullptr};              // keys in input order (convert)
    uint2 *pair[2] = {nullptr, nullptr};       // radix ping-pong: (key, input position) pairs
    uint32_t *hist = nullptr;                  // radix: per-pass digit totals, their exclusive
                                               // scans, grid-barrier counters (bin.cu)
    uint32_t *ost[2] = {nullptr, nullptr};     // radix: per-CTA range histograms, their
                                               // column-wise exclusive scans [cta][digit]
    int64_t ost_cap = 0;                       // words per buffer
    uint32_t *scan_tmp = nullptr;                // band compaction: kept total
    float2 *xy = nullptr;                      // sorted bucket-local coordinates
    uint2 *rng = nullptr;                      // sorted packed int16 ranges
    uint4 *rec = nullptr;                      // per input point: lx, ly, packed ranges
    uint2 *sorted = nullptr;                   // sorted (key, original index) pairs (alias)
    // banded contexts: the points binning keeps, compacted in input order before the sort
    double *cx = nullptr, *cy = nullptr;       // their coordinates
    uint32_t *cidx = nullptr;                  // their original indices
    uint32_t *bcnt = nullptr;                  // per-block kept counts -> offsets
    unsigned long long *nfin = nullptr;        // finite points (the 1/n normalisation)
    int64_t ccap = 0, bcap = 0;
    bool compacted = false;                    // the last load went through the compaction
};

// Geometry of one evaluation path's work decomposition.  A group is a vertical stack of
// `s` buckets (pitch px x py = B x sB pixels); its window is (px + 2F) x (py + 2F) pixels,
// cut into nsubx x nsuby sub-windows of sx x sy; each (group, segment, sub-window) block
// lands in a slot of slot_h rows x slot_w floats.
struct PathGeom {
    int s = 1;
    int ngx = 0, ngy = 0;
    int px = 0, py = 0;
    int ww = 0, wh = 0;
    int nsubx = 1, nsuby = 1;
    int sx = 0, sy = 0;
    int slot_w = 0, slot_h = 0;
    int seg_pts = kSegMin;   // points per full segment (set per load, seg_pts_for)
    int chunk_pts = 32;      // tensor-core path: points per MMA chunk (K of one commit group)
    int mma_n = 0;           // tensor-core path: MMA N (window columns rounded up to 16)
    int mrows = 128;         // tensor-core path: MMA M = accumulator rows = slot rows (64 when the
                             // group window has <= 64 rows and N <= 48: eval_tc5.cu's M = 64 tiles)
    int part_pts = 0;        // a group's remainder (< seg_pts points) is cut into pieces of <=
                             // part_pts points, one work item each (direct: 128, one warp;
                             // 0: the whole remainder, = seg_pts)
    __host__ __device__ int nsub() const { return nsubx * nsuby; }
    __host__ __device__ int ngroups() const { return ngx * ngy; }
    __host__ __device__ int64_t slot_floats() const { return (int64_t)slot_w * slot_h; }
};

// Buffers of the snapped pipeline (kde_snap, snap.cu), allocated on first use.
struct SnapBufs {
    int64_t cap = 0;                 // staging capacity (points) for host inputs
    double *x = nullptr, *y = nullptr;
    int32_t* lab = nullptr;
    uint32_t* counts = nullptr;      // M_D when the caller passes no counts buffer
    float* tmp = nullptr;            // Eq. 7 row pass
    unsigned long long* ext = nullptr;  // encoded x/y extent
    float* w = nullptr;              // 1-D weights
    cudaEvent_t done = nullptr;      // end of the last kde_snap: the next one (on any stream)
    bool used = false;               // waits for it before rewriting the scratch above
};

struct EvalPlan {
    PathGeom pg;
    bool enabled = false;
    // SIMT splat launch shape (direct path)
    int mt = 4;                                // lane tile rows TY (columns 2 TY), S = 8 TY
    int grid = 0;                              // persistent grid (0: not yet queried)
    int grid_split = 0;                        // the same for the split-fp16 tensor-core kernel
    bool part_fixed = false;                   // remainder pieces of kPartPtsDirect (direct)
    int64_t planned_gen = -1;                  // load generation this plan belongs to
    // device buffers.  The plan's sizes stay on the device (kTot*): kernels read them, the
    // host never waits for them (buffers are reserved at their upper bounds).
    uint64_t* d_local = nullptr;               // block-local prefixes (full << 32 | part)
    uint64_t* d_bsum = nullptr;                // block totals -> their exclusive scan
    int2* d_group = nullptr;                   // per group: (first segment, #segments)
    int* d_totals = nullptr;                   // see kTot*
    int* d_hot = nullptr;                      // groups with > 1 segment (segment reduce)
    uint8_t* d_tflag = nullptr;                // per combine tile of the band: 1 if a planned
                                               // group's window meets it (else it is all zero)
    int tfx = 0, tfy = 0;                      // combine tiles (columns, band rows)
    int4* d_items = nullptr;                   // (group, k0, k1, slot)
    int64_t items_cap = 0;
    float* d_splat = nullptr;
    int64_t slots_cap = 0;
};

// d_totals layout (ints)
constexpr int kTotFull = 0;    // full segments
constexpr int kTotPart = 1;    // partial segments
constexpr int kTotSlots = 2;   // slots = work items = (full + partial) * nsub
constexpr int kTotBinned = 3;  // points binned
constexpr int kTotHot = 4;     // split groups (segment reduce list length)
constexpr int kTotChunks = 5;  // tensor-core path: chunk_pts-point MMA chunks (executed flops)
constexpr int kTotQueue = 6;   // persistent-kernel work-queue head (CTA items)
constexpr int kTotQueue2 = 7;  // second queue head (direct path: per-warp items)
constexpr int kTotChunksExec = 8;  // chunks the per-warp tensor-core kernel executed (eval_tc5.cu's
                                   // bucket-homogeneous chunks; 0 when the other kernel ran)
constexpr int kTotInts = 9;

// Upper bound on a path's items/slots for n points: every full segment, plus per
// non-empty group its remainder pieces (at most n / part_pts + one per group), times the
// sub-windows.
inline int64_t slot_bound(const PathGeom& pg, int64_t n) {
    const int64_t ng = (int64_t)pg.ngroups();
    const int64_t rem = pg.part_pts < pg.seg_pts ? n / pg.part_pts : 0;
    return (n / pg.seg_pts + rem + (n < ng ? n : ng)) * pg.nsub();
}

}  // namespace kde

struct kde_ctx {
    kde_params p;
    kde::Geom g;
    double hpx = 0, ceff = 0;
    int kern = 0;
    bool radial = false;
    cudaStream_t stream = nullptr;             // internal stream (loads)
    cudaStream_t copy_stream = nullptr;        // host-input uploads (overlap the binning)
    cudaEvent_t stage_free[2] = {};            // staging buffer k read by its binning
    cudaEvent_t stage_ready = nullptr;         // the last upload has landed
    kde::PointBufs pb;
    uint32_t* d_offsets = nullptr;             // nb + 1
    unsigned long long* d_stats = nullptr;     // n_finite, n_outside, useful_pairs
    cudaEvent_t loaded_ev = nullptr;           // end of the last load (eval waits on it)
    cudaEvent_t evald_ev = nullptr;            // end of the last eval (the next load's
                                               // binning waits on it: eval reads the bins)
    cudaEvent_t input_ev = nullptr;            // legacy-stream point for device inputs
    cudaEvent_t stats_ev = nullptr;            // the load's stats readback has landed
    bool evaluated = false;
    int* h_totals = nullptr;                   // pinned: stats readback (asynchronous)
    bool stats_pending = false;                // h_totals not yet folded into stats
    size_t splat_budget = 0;                   // max bytes a splat buffer may reserve unread
    kde_stats stats{};
    bool loaded = false;
    int64_t load_gen = 0;                      // bumped by every load (lazy per-path plans)
    int64_t plan_n = 0;                        // the point count that sizes the plan's segments:
                                               // n_in, or n_finite after a banded load (so a
                                               // NaN-padded point shard plans like the raw set)
    int64_t launches = 0;                      // kernels launched (kde_stats.kernel_launches)
    int main_kernel = 0;                       // kde_stats.main_kernel of the last eval
    bool timing = false;                       // record phase events (kde_set_timing)
    cudaEvent_t tev[6] = {};                   // bin0, bin1 (load); plan0, main0, main1, comb1 (eval)
    bool tev_load = false, tev_eval = false;
    kde::EvalPlan plan[2];                     // [KDE_PATH_DIRECT], [KDE_PATH_TENSOR]
    kde::SnapBufs snap;                        // kde_snap (NEXT-F1)
};

namespace kde {

void set_error(const char* fmt, ...);
inline void tmark(kde_ctx* c, int k, cudaStream_t s) {
    if (c->timing) cudaEventRecord(c->tev[k], s);
}
int cuda_fail(cudaError_t e, const char* what);

// binning (bin.cu)
int bin_points(kde_ctx* c, const double* d_x, const double* d_y, int64_t n);
// evaluation (eval_direct.cu, eval_tc.cu)
int launch_direct(kde_ctx* c, float* out, cudaStream_t s);
int launch_tc(kde_ctx* c, float* out, cudaStream_t s, bool split);
int launch_tc5(kde_ctx* c, cudaStream_t s);  // eval_tc5.cu: per-warp tensor-core pipelines
// planning (plan.cu)
int plan_device(kde_ctx* c, EvalPlan& pl, cudaStream_t s);
int plan_nblk(const PathGeom& pg);
int launch_combine(kde_ctx* c, const EvalPlan& pl, float* out, cudaStream_t s);
// snapped pipeline (snap.cu)
int snap_run(kde_ctx* c, const double* x, const double* y, const int32_t* label, int64_t n,
             uint32_t* counts, float* out, cudaStream_t s, bool host);
void snap_free(kde_ctx* c);
// GPU Douglas-Peucker (dp.cu); device pointers
int dp_run(const double* x, const double* y, const int64_t* offs, int ntraj, int n, double eps, uint8_t* keep,
           cudaStream_t s, int64_t* n_kept, int64_t* rounds);

}  // namespace kde
