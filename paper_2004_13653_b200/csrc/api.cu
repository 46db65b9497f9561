// The C ABI of include/kde.h: validation, context lifecycle, load (a1/a2 + plan),
// eval dispatch (a3/a4/a5), stats, and error reporting.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <numeric>

#include <dlfcn.h>

#include "internal.cuh"

namespace kde {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
    set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    return KDE_ECUDA;
}

// RAII device guard: select the context device, restore the caller's afterwards.
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

static int dalloc(void** p, size_t bytes, const char* what) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (cudaMalloc(p, bytes ? bytes : 16) != cudaSuccess) {
        cudaGetLastError();
        set_error("cudaMalloc for %s failed (%zu bytes)", what, bytes);
        return KDE_ENOMEM;
    }
    return KDE_OK;
}

// Direct-path geometry, fixed at create: groups are single buckets; the window B + 2F is
// cut into nsub x nsub equal sub-windows of <= 48 pixels, each computed by a lane grid of
// 4 x 8 register tiles of 2TY x TY pixels (S = 8 TY >= the sub-window edge, TY in 2..6).
static void plan_geometry_direct(EvalPlan& pl, const Geom& g) {
    PathGeom& pg = pl.pg;
    const int Wd = g.B + 2 * g.F;
    pg.s = 1;
    pg.ngx = g.nbx;
    pg.ngy = g.nby;
    pg.px = pg.py = g.B;
    pg.ww = pg.wh = Wd;
    pg.nsubx = pg.nsuby = (Wd + kSubMax - 1) / kSubMax;
    pg.sx = pg.sy = (Wd + pg.nsubx - 1) / pg.nsubx;  // the last sub-window may be smaller
    pl.mt = std::max(2, (pg.sx + 7) / 8);            // TY
    pg.slot_w = pg.slot_h = 8 * pl.mt;               // S x S slot (float4-aligned rows)
    pl.part_fixed = true;                            // remainders: one warp per 128 points
    pl.enabled = true;
}

// Tensor-core geometry (product kernels, all eight: NEXT-F2).  While the bucket window
// B + 2F fits the M = 128 TMEM lanes, a group is a vertical stack of s buckets whose window
// fills them (rows); columns N = B + 2F rounded up to 16.  Larger supports (C5 at h >= 16
// px) keep one bucket per group and cut its window into nsubx x nsuby sub-windows of
// <= 128 rows x <= 128 columns (equal pieces), one MMA tile each (TMEM <= 128 columns:
// 4 CTAs per SM).
static void plan_geometry_tc(EvalPlan& pl, const Geom& g, bool product) {
    PathGeom& pg = pl.pg;
    const int Wd = g.B + 2 * g.F;
    pl.enabled = product;
    if (!pl.enabled) return;
    // M = 64 tiles (eval_tc5.cu) when a stack of >= 1 bucket fits 64 rows and the window's
    // columns fit N = 48: half the MMA rows of M = 128 are padding for such windows anyway, and
    // two M = 64 accumulators share a TMEM column slice (16 workers instead of 10).
    const char* m64env = getenv("KDE_TC_M64");
    const bool m64 = Wd <= 48 && (64 - 2 * g.F) / g.B >= 1 && !(m64env && atoi(m64env) == 0);
    pg.mrows = m64 ? 64 : kTcM;
    pg.s = m64 ? (64 - 2 * g.F) / g.B : (Wd <= kTcM ? std::max(1, (kTcM - 2 * g.F) / g.B) : 1);
    pg.ngx = g.nbx;
    pg.ngy = (g.nby + pg.s - 1) / pg.s;
    pg.px = g.B;
    pg.py = pg.s * g.B;
    pg.ww = Wd;
    pg.wh = pg.py + 2 * g.F;
    pg.nsubx = (pg.ww + kTcM - 1) / kTcM;
    pg.nsuby = (pg.wh + kTcM - 1) / kTcM;
    pg.sx = (pg.ww + pg.nsubx - 1) / pg.nsubx;
    pg.sy = (pg.wh + pg.nsuby - 1) / pg.nsuby;
    pg.slot_w = ((pg.sx + 3) / 4) * 4;  // the sub-window's columns (float4 rows); MMA N = round16
    pg.mma_n = ((pg.sx + 15) / 16) * 16;
    pg.slot_h = pg.mrows;
    pg.chunk_pts = 32;                  // 2 MMAs per operand buffer (eval_tc.cu, H = 1; 64-point
                                        // chunks measured slower: 5 CTAs/SM instead of 8)
}

static int alloc_plan(EvalPlan& pl, const Geom& g) {
    if (!pl.enabled) return KDE_OK;
    pl.tfx = (g.W + kCombTile - 1) / kCombTile;
    pl.tfy = (g.re - g.rb + kCombTile - 1) / kCombTile;
    const size_t ng = (size_t)pl.pg.ngroups();
    const size_t nblk = (size_t)plan_nblk(pl.pg);
    cudaError_t e = cudaMalloc(&pl.d_local, sizeof(uint64_t) * nblk * 1024);
    if (e == cudaSuccess) e = cudaMalloc(&pl.d_bsum, sizeof(uint64_t) * (nblk + 1));
    if (e == cudaSuccess) e = cudaMalloc(&pl.d_group, sizeof(int2) * (ng > 0 ? ng : 1));
    if (e == cudaSuccess) e = cudaMalloc(&pl.d_totals, sizeof(int) * kTotInts);
    if (e == cudaSuccess) e = cudaMalloc(&pl.d_hot, sizeof(int) * (ng > 0 ? ng : 1));
    if (e == cudaSuccess) e = cudaMalloc(&pl.d_tflag, (size_t)pl.tfx * pl.tfy);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("kde_create: plan allocation failed");
        return KDE_ENOMEM;
    }
    return KDE_OK;
}

// Build path pl's plan for the current load on stream s.  The item list
// and the splat buffer are reserved at their upper bounds, so the plan needs no host round
// trip -- unless the splat bound exceeds the context's budget (very large windows): then
// the exact slot count is read back once and only that much is allocated.
static int plan_path(kde_ctx* c, EvalPlan& pl, cudaStream_t s) {
    // segment size from the global n (identical on every rank); the tensor-core path's 16
    // pipelines per SM want twice as many items (C4: 2048-point segments, kernel 0.49 ->
    // 0.46 ms, the busiest worker's tail shorter; 1024 slowed the segment reduce more)
    const bool tc = &pl == &c->plan[KDE_PATH_TENSOR];
    pl.pg.seg_pts = seg_pts_for(c->plan_n, tc && pl.pg.mrows == 64 ? kSegShareTc : kSegShareCtas);
    static const int env_tcseg = getenv("KDE_TC_SEG") ? atoi(getenv("KDE_TC_SEG")) : 0;  // A/B experiments
    if (tc && env_tcseg >= kSegMin && env_tcseg <= kSegMax) pl.pg.seg_pts = env_tcseg;
    // direct path: remainder pieces of a quarter segment (>= 128 points): fewer splat slots
    // to write, reduce and combine (C4: 128 -> 1024-point pieces, step 2.80 -> 2.62 ms;
    // C2: 128 -> 256, 0.377 -> 0.368 ms).  KDE_PART_PTS overrides (A/B experiments).
    static const int env_part = getenv("KDE_PART_PTS") ? atoi(getenv("KDE_PART_PTS")) : 0;
    const int part = env_part >= 16 ? env_part : std::max(kPartPtsDirect, pl.pg.seg_pts / 4);
    pl.pg.part_pts = pl.part_fixed ? std::min(part, pl.pg.seg_pts) : pl.pg.seg_pts;
    const int64_t bound = slot_bound(pl.pg, std::max(c->stats.n_in, c->plan_n));
    if (bound + 1 > pl.items_cap) {
        if (dalloc((void**)&pl.d_items, sizeof(int4) * (bound + 1), "plan items")) return KDE_ENOMEM;
        pl.items_cap = bound + 1;
    }
    const size_t slot_bytes = sizeof(float) * (size_t)pl.pg.slot_floats();
    const bool exact = (size_t)bound * slot_bytes > c->splat_budget;
    if (!exact && bound > pl.slots_cap) {
        if (dalloc((void**)&pl.d_splat, slot_bytes * (size_t)(bound > 0 ? bound : 1), "splat blocks"))
            return KDE_ENOMEM;
        pl.slots_cap = bound;
    }
    int rc = plan_device(c, pl, s);
    if (rc) return rc;
    if (exact) {
        int nslots = 0;
        cudaError_t e = cudaMemcpyAsync(c->h_totals, pl.d_totals + kTotSlots, sizeof(int),
                                        cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(e, "kde_eval: plan readback");
        nslots = c->h_totals[0];
        if (nslots > pl.slots_cap) {
            if (dalloc((void**)&pl.d_splat, slot_bytes * (size_t)nslots, "splat blocks")) return KDE_ENOMEM;
            pl.slots_cap = nslots;
        }
    }
    pl.planned_gen = c->load_gen;
    return KDE_OK;
}

// fold the load's asynchronous stats readback into c->stats (waits for it)
static int sync_stats(kde_ctx* c) {
    if (!c->stats_pending) return KDE_OK;
    const cudaError_t e = cudaEventSynchronize(c->stats_ev);
    if (e != cudaSuccess) return cuda_fail(e, "stats readback");
    const unsigned long long* st = reinterpret_cast<const unsigned long long*>(c->h_totals + 16);
    c->stats.n_finite = (int64_t)st[0];
    c->stats.n_outside = (int64_t)st[1];
    c->stats.useful_pairs = (int64_t)st[2];
    c->stats.n_binned = (int64_t)(uint32_t)c->h_totals[24];
    c->stats_pending = false;
    return KDE_OK;
}

static void free_plan(EvalPlan& pl) {
    cudaFree(pl.d_local);
    cudaFree(pl.d_bsum);
    cudaFree(pl.d_group);
    cudaFree(pl.d_totals);
    cudaFree(pl.d_hot);
    cudaFree(pl.d_tflag);
    cudaFree(pl.d_items);
    cudaFree(pl.d_splat);
    pl = EvalPlan();
}

// Bucket (point-group) edge B: small enough that the group window B + 2F stays close to
// the (2R+1) support, large enough that groups hold many points.
static int choose_bucket(double R) {
    const char* env = getenv("KDE_BUCKET");
    if (env) {
        const int b = atoi(env);
        if (b == 4 || b == 8 || b == 16 || b == 32 || b == 64) return b;
    }
    if (R < 24.0) return 8;
    if (R < 64.0) return 16;
    if (R < 160.0) return 32;
    return 64;
}

static bool is_device_ptr(const void* p, int* dev) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    *dev = at.device;
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace kde

using namespace kde;

extern "C" {

const char* kde_last_error(void) { return g_err; }

int kde_create(const kde_params* p, kde_ctx** out) {
    if (out) *out = nullptr;
    if (!p || !out) {
        set_error("kde_create: NULL argument");
        return KDE_EINVAL;
    }
    auto bad = [](double v) { return !(v > 0.0) || !isfinite(v); };
    if (bad(p->res) || bad(p->h) || bad(p->cutoff) || !isfinite(p->x0) || !isfinite(p->y0)) {
        set_error("kde_create: res, h, cutoff must be finite and > 0 (x0, y0 finite)");
        return KDE_EINVAL;
    }
    if (p->width < 1 || p->width > 32767 || p->height < 1 || p->height > 32767) {
        set_error("kde_create: width/height must be in 1..32767");
        return KDE_EINVAL;
    }
    const int kern = p->kernel & 0xff;
    if ((p->kernel & ~(0xff | KDE_RADIAL)) != 0 || kern > KDE_COSINE) {
        set_error("kde_create: unknown kernel id 0x%x", p->kernel);
        return KDE_EINVAL;
    }
    int rb = p->row_begin, re = p->row_end;
    if (!(rb == 0 && re == 0) && !(0 <= rb && rb < re && re <= p->height)) {
        set_error("kde_create: band [%d,%d) outside [0,%d]", rb, re, p->height);
        return KDE_EINVAL;
    }
    if (rb == 0 && re == 0) re = p->height;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || p->device < 0 || p->device >= ndev) {
        cudaGetLastError();
        set_error("kde_create: CUDA device %d not available (%d devices)", p->device, ndev);
        return KDE_ECUDA;
    }
    DeviceGuard dg(p->device);
    if (!dg.ok) return cuda_fail(cudaGetLastError(), "kde_create: cudaSetDevice");

    kde_ctx* c = new kde_ctx();
    c->p = *p;
    c->kern = kern;
    c->radial = (p->kernel & KDE_RADIAL) != 0;
    c->hpx = p->h / p->res;
    c->ceff = (kern == KDE_GAUSSIAN) ? p->cutoff : (p->cutoff < 1.0 ? p->cutoff : 1.0);
    Geom& g = c->g;
    g.x0 = p->x0;
    g.y0 = p->y0;
    g.res = p->res;
    g.R = c->ceff * c->hpx;  // R_px = c_eff * (h / res)
    g.W = p->width;
    g.H = p->height;
    g.rb = rb;
    g.re = re;
    g.B = choose_bucket(g.R);
    g.lgB = 0;
    while ((1 << g.lgB) < g.B) g.lgB++;
    g.F = (int)floor(g.R + 0.5);
    g.nbx = (g.W + g.B - 1) / g.B;
    g.nby = (g.H + g.B - 1) / g.B;
    const double reach = ceil(g.R + 0.5) + 1.0;
    if (!(reach < 1.0e6)) {
        delete c;
        set_error("kde_create: support R = %g px too large", g.R);
        return KDE_EINVAL;
    }
    g.reach = (int)reach;
    {   // combine-pass entry list bound: groups meeting a 32-px tile x <= 4 sub-windows
        const int Wd = g.B + 2 * g.F;
        const int per = (kCombTile + Wd) / g.B + 2;
        if (per * per * 4 > 2048) {
            delete c;
            set_error("kde_create: support R = %g px too large for bucket %d", g.R, g.B);
            return KDE_EINVAL;
        }
    }
    g.nr = (g.reach + g.B - 1) / g.B;
    plan_geometry_direct(c->plan[KDE_PATH_DIRECT], g);
    plan_geometry_tc(c->plan[KDE_PATH_TENSOR], g, !c->radial);
    {   // kept home-bucket rows, rounded out to whole tensor-core stacks so that every group
        // of either path meeting the band is complete (bitwise sharding)
        const int st = c->plan[KDE_PATH_TENSOR].enabled ? c->plan[KDE_PATH_TENSOR].pg.s : 1;
        auto fdiv = [](int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
        const int lo = rb / g.B - g.nr, hi = (re - 1) / g.B + g.nr;
        g.band_lo = fdiv(lo, st) * st;
        g.band_hi = (fdiv(hi, st) + 1) * st - 1;
        c->stats.stack = st;
        c->stats.band_lo = g.band_lo;
        c->stats.band_hi = g.band_hi;
    }
    const size_t nb = (size_t)g.nbx * g.nby;
    // a non-blocking stream: a host-input upload may overlap the previous evaluation; the
    // load orders itself explicitly (see kde_load_points)
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
    for (int k = 0; k < 2 && e == cudaSuccess; k++)
        e = cudaEventCreateWithFlags(&c->stage_free[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->stage_ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->loaded_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->evald_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->input_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->stats_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) {
        size_t fr = 0, tot = 0;
        e = cudaMemGetInfo(&fr, &tot);
        c->splat_budget = std::min<size_t>(tot / 8, (size_t)16 << 30);
    }
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_totals, 128);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_offsets, sizeof(uint32_t) * (nb + 1));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_stats, sizeof(unsigned long long) * 4);
    if (e != cudaSuccess) {
        kde_free(c);
        return cuda_fail(e, "kde_create: allocation");
    }
    for (int p = 0; p < 2; p++)
        if (alloc_plan(c->plan[p], g)) {
            kde_free(c);
            return KDE_ENOMEM;
        }
    c->stats.bucket = g.B;
    c->stats.nbx = g.nbx;
    c->stats.nby = g.nby;
    c->stats.reach_px = g.reach;
    *out = c;
    return KDE_OK;
}

int kde_load_points(kde_ctx* c, const double* x, const double* y, int64_t n) {
    if (!c) {
        set_error("kde_load_points: NULL context");
        return KDE_EINVAL;
    }
    if (n < 0 || n > 0x7fffffffLL - 4096) {
        set_error("kde_load_points: n = %lld outside [0, 2^31 - 4097]", (long long)n);
        return KDE_EINVAL;
    }
    if (n > 0 && (!x || !y)) {
        set_error("kde_load_points: NULL x or y");
        return KDE_EINVAL;
    }
    DeviceGuard dg(c->p.device);
    if (!dg.ok) return cuda_fail(cudaGetLastError(), "kde_load_points: cudaSetDevice");
    c->loaded = false;
    const double *dx = x, *dy = y;
    int stage_used = -1;
    if (n > 0) {
        int devx = -1, devy = -1;
        const bool xd = is_device_ptr(x, &devx), yd = is_device_ptr(y, &devy);
        if (xd != yd) {
            set_error("kde_load_points: x and y must both be host or both device pointers");
            return KDE_EINVAL;
        }
        if (xd && (devx != c->p.device || devy != c->p.device)) {
            set_error("kde_load_points: device pointers on device %d/%d, context on %d", devx, devy,
                      c->p.device);
            return KDE_EINVAL;
        }
        if (!xd) {  // host input: upload on the copy stream into a staging buffer pair
            const int j = c->pb.stage;
            if (c->pb.stage_cap[j] < n) {
                cudaFree(c->pb.sx[j]);
                cudaFree(c->pb.sy[j]);
                c->pb.sx[j] = c->pb.sy[j] = nullptr;
                c->pb.stage_cap[j] = 0;
                if (cudaMalloc(&c->pb.sx[j], sizeof(double) * n) != cudaSuccess ||
                    cudaMalloc(&c->pb.sy[j], sizeof(double) * n) != cudaSuccess) {
                    cudaGetLastError();
                    set_error("kde_load_points: staging allocation failed");
                    return KDE_ENOMEM;
                }
                c->pb.stage_cap[j] = n;
            }
            // the binning that last read buffer j must be done (a never-recorded event is
            // complete); the upload then overlaps the previous load's binning and eval
            cudaStreamWaitEvent(c->copy_stream, c->stage_free[j], 0);
            cudaMemcpyAsync(c->pb.sx[j], x, sizeof(double) * n, cudaMemcpyHostToDevice, c->copy_stream);
            cudaMemcpyAsync(c->pb.sy[j], y, sizeof(double) * n, cudaMemcpyHostToDevice, c->copy_stream);
            cudaEventRecord(c->stage_ready, c->copy_stream);
            cudaStreamWaitEvent(c->stream, c->stage_ready, 0);
            dx = c->pb.sx[j];
            dy = c->pb.sy[j];
            stage_used = j;
            c->pb.stage ^= 1;
        } else {
            // device inputs: read them after the work already queued on the legacy default
            // stream (where PyTorch's default stream puts their producers)
            cudaEventRecord(c->input_ev, cudaStreamLegacy);
            cudaStreamWaitEvent(c->stream, c->input_ev, 0);
        }
    }
    // the previous evaluation reads the sorted points and the plan that binning rewrites
    if (c->evaluated) cudaStreamWaitEvent(c->stream, c->evald_ev, 0);
    tmark(c, 0, c->stream);
    c->plan_n = n;  // (a banded load replaces it with n_finite)
    int rc = bin_points(c, dx, dy, n);
    if (rc) return rc;
    if (stage_used >= 0) cudaEventRecord(c->stage_free[stage_used], c->stream);
    tmark(c, 1, c->stream);
    c->tev_load = c->timing;
    // the integer stats come back asynchronously (kde_get_stats waits for them); the
    // per-path plans are built lazily by the first kde_eval of each path
    c->stats.n_in = n;
    c->stats.n_finite = c->stats.n_binned = c->stats.n_outside = c->stats.useful_pairs = 0;
    cudaMemcpyAsync(c->h_totals + 16, c->d_stats, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                    c->stream);
    cudaMemcpyAsync(c->h_totals + 24, c->d_offsets + (size_t)c->g.nbx * c->g.nby, sizeof(uint32_t),
                    cudaMemcpyDeviceToHost, c->stream);
    cudaError_t e = cudaEventRecord(c->stats_ev, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "kde_load_points: event");
    c->stats_pending = true;
    c->load_gen++;
    e = cudaEventRecord(c->loaded_ev, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "kde_load_points: event");
    c->loaded = true;
    return KDE_OK;
}

int kde_eval(kde_ctx* c, int32_t path, float* out, void* stream) {
    if (!c || !out) {
        set_error("kde_eval: NULL argument");
        return KDE_EINVAL;
    }
    if (path != KDE_PATH_DIRECT && path != KDE_PATH_TENSOR && path != KDE_PATH_TENSOR_SPLIT) {
        set_error("kde_eval: unknown path %d", path);
        return KDE_EINVAL;
    }
    if (!c->loaded) {
        set_error("kde_eval: no points loaded");
        return KDE_ESTATE;
    }
    if (path != KDE_PATH_DIRECT && !c->plan[KDE_PATH_TENSOR].enabled) {
        set_error("kde_eval: the tensor-core path implements the product kernels only "
                  "(a radial support is not rank one)");
        return KDE_EUNSUPPORTED;
    }
    DeviceGuard dg(c->p.device);
    if (!dg.ok) return cuda_fail(cudaGetLastError(), "kde_eval: cudaSetDevice");
    cudaError_t e = cudaGetLastError();  // surface earlier asynchronous faults
    if (e != cudaSuccess) return cuda_fail(e, "kde_eval: earlier asynchronous error");
    cudaStream_t s = (cudaStream_t)stream;
    e = cudaStreamWaitEvent(s, c->loaded_ev, 0);  // the bins of the last load
    if (e == cudaSuccess && c->evaluated) e = cudaStreamWaitEvent(s, c->evald_ev, 0);  // evals in order
    if (e != cudaSuccess) return cuda_fail(e, "kde_eval: wait for load");
    EvalPlan& pl = c->plan[path == KDE_PATH_DIRECT ? KDE_PATH_DIRECT : KDE_PATH_TENSOR];  // (split: same plan)
    tmark(c, 2, s);
    if (pl.planned_gen != c->load_gen) {
        const int prc = plan_path(c, pl, s);
        if (prc) return prc;
    }
    const int rc = path == KDE_PATH_DIRECT ? launch_direct(c, out, s)
                                           : launch_tc(c, out, s, path == KDE_PATH_TENSOR_SPLIT);
    if (rc == KDE_OK) {
        cudaEventRecord(c->evald_ev, s);
        c->evaluated = true;
    }
    return rc;
}

int kde_set_timing(kde_ctx* c, int enable) {
    if (!c) {
        set_error("kde_set_timing: NULL context");
        return KDE_EINVAL;
    }
    DeviceGuard dg(c->p.device);
    if (enable && !c->tev[0])
        for (int k = 0; k < 6; k++)
            if (cudaEventCreate(&c->tev[k]) != cudaSuccess) return cuda_fail(cudaGetLastError(), "kde_set_timing");
    c->timing = enable != 0;
    c->tev_load = c->tev_eval = false;
    return KDE_OK;
}

int kde_get_timing(kde_ctx* c, kde_timing* t) {
    if (!c || !t) {
        set_error("kde_get_timing: NULL argument");
        return KDE_EINVAL;
    }
    if (!c->timing || !c->tev_load || !c->tev_eval) {
        set_error("kde_get_timing: timing disabled or no load+eval recorded since enabling");
        return KDE_ESTATE;
    }
    DeviceGuard dg(c->p.device);
    cudaError_t e = cudaEventSynchronize(c->tev[5]);
    if (e == cudaSuccess) e = cudaEventSynchronize(c->tev[1]);
    if (e != cudaSuccess) return cuda_fail(e, "kde_get_timing");
    cudaEventElapsedTime(&t->bin_ms, c->tev[0], c->tev[1]);
    cudaEventElapsedTime(&t->plan_ms, c->tev[2], c->tev[3]);
    cudaEventElapsedTime(&t->main_ms, c->tev[3], c->tev[4]);
    cudaEventElapsedTime(&t->combine_ms, c->tev[4], c->tev[5]);
    return KDE_OK;
}

int kde_get_stats(const kde_ctx* c, kde_stats* s) {
    if (!c || !s) {
        set_error("kde_get_stats: NULL argument");
        return KDE_EINVAL;
    }
    kde_ctx* m = const_cast<kde_ctx*>(c);
    DeviceGuard dg(c->p.device);
    int rc = sync_stats(m);
    if (rc) return rc;
    *s = c->stats;
    s->kernel_launches = c->launches;
    s->main_kernel = c->main_kernel;
    s->tc_m = c->plan[KDE_PATH_TENSOR].enabled ? c->plan[KDE_PATH_TENSOR].pg.mrows : 0;
    s->tc_mma_flops = 0;
    const EvalPlan& tp = c->plan[KDE_PATH_TENSOR];
    if (c->loaded && tp.enabled && tp.planned_gen == c->load_gen) {  // executed MMA flops / eval
        int tot[kTotInts] = {};
        // the plan was built on the eval's (possibly non-blocking) stream: wait for that
        // eval before reading its totals
        cudaError_t e = c->evaluated ? cudaEventSynchronize(c->evald_ev) : cudaSuccess;
        if (e == cudaSuccess) e = cudaMemcpy(tot, tp.d_totals, sizeof(tot), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(e, "kde_get_stats");
        // the per-warp kernel (eval_tc5.cu) counts the chunks it executed; the other kernel
        // executes the plan's chunks
        const int chunks = tot[kTotChunksExec] > 0 ? tot[kTotChunksExec] : tot[kTotChunks];
        // per chunk: chunk_pts/16 MMAs of M=128 x N x K=16, 2 flops per MAC
        const int64_t m = tot[kTotChunksExec] > 0 ? tp.pg.mrows : kTcM;  // eval_tc.cu: always M = 128
        s->tc_mma_flops = (int64_t)chunks * (tp.pg.chunk_pts / 16) * 2 * m * tp.pg.mma_n * 16;
    }
    return KDE_OK;
}

int kde_get_bins(const kde_ctx* c, int64_t* offsets, int64_t* perm, float* lx, float* ly,
                 int32_t* ranges) {
    if (!c) {
        set_error("kde_get_bins: NULL context");
        return KDE_EINVAL;
    }
    if (!c->loaded) {
        set_error("kde_get_bins: no points loaded");
        return KDE_ESTATE;
    }
    DeviceGuard dg(c->p.device);
    if (int rc = sync_stats(const_cast<kde_ctx*>(c))) return rc;
    const size_t nb = (size_t)c->g.nbx * c->g.nby;
    const size_t m = (size_t)c->stats.n_binned;
    if (cudaEventSynchronize(c->loaded_ev) != cudaSuccess) return cuda_fail(cudaGetLastError(), "kde_get_bins");
    if (offsets) {
        std::vector<uint32_t> ov(nb + 1);
        const cudaError_t e0 = cudaMemcpy(ov.data(), c->d_offsets, sizeof(uint32_t) * (nb + 1),
                                          cudaMemcpyDeviceToHost);
        if (e0 != cudaSuccess) return cuda_fail(e0, "kde_get_bins");
        for (size_t b = 0; b <= nb; b++) offsets[b] = (int64_t)ov[b];
    }
    if (m == 0) return KDE_OK;
    std::vector<uint32_t> pv;
    std::vector<float2> xy;
    std::vector<uint2> rg;
    cudaError_t e = cudaSuccess;
    if (perm) {
        pv.resize(m);
        e = cudaMemcpy2D(pv.data(), sizeof(uint32_t), reinterpret_cast<const char*>(c->pb.sorted) + sizeof(uint32_t),
                         sizeof(uint2), sizeof(uint32_t), m, cudaMemcpyDeviceToHost);  // the pairs' second words
        if (e == cudaSuccess && c->pb.compacted) {  // banded: sorted compacted positions -> input indices
            std::vector<uint32_t> ci((size_t)c->stats.n_in);
            e = cudaMemcpy(ci.data(), c->pb.cidx, sizeof(uint32_t) * ci.size(), cudaMemcpyDeviceToHost);
            for (size_t k = 0; k < m && e == cudaSuccess; k++) pv[k] = ci[pv[k]];
        }
        for (size_t k = 0; k < m && e == cudaSuccess; k++) perm[k] = (int64_t)pv[k];
    }
    if (e == cudaSuccess && (lx || ly)) {
        xy.resize(m);
        e = cudaMemcpy(xy.data(), c->pb.xy, sizeof(float2) * m, cudaMemcpyDeviceToHost);
        for (size_t k = 0; k < m && e == cudaSuccess; k++) {
            if (lx) lx[k] = xy[k].x;
            if (ly) ly[k] = xy[k].y;
        }
    }
    if (e == cudaSuccess && ranges) {
        rg.resize(m);
        e = cudaMemcpy(rg.data(), c->pb.rng, sizeof(uint2) * m, cudaMemcpyDeviceToHost);
        for (size_t k = 0; k < m && e == cudaSuccess; k++) {
            ranges[4 * k + 0] = (int32_t)(rg[k].x & 0xffffu);
            ranges[4 * k + 1] = (int32_t)(rg[k].x >> 16);
            ranges[4 * k + 2] = (int32_t)(rg[k].y & 0xffffu);
            ranges[4 * k + 3] = (int32_t)(rg[k].y >> 16);
        }
    }
    if (e != cudaSuccess) return cuda_fail(e, "kde_get_bins");
    return KDE_OK;
}

int kde_snap(kde_ctx* c, const double* x, const double* y, const int32_t* label, int64_t n,
             uint32_t* counts, float* out, void* stream) {
    if (!c || !out || (n > 0 && (!x || !y))) {
        set_error("kde_snap: NULL argument");
        return KDE_EINVAL;
    }
    if (n < 0 || n > 2147483647ll - 4096) {
        set_error("kde_snap: n = %lld outside [0, 2^31 - 4097]", (long long)n);
        return KDE_EINVAL;
    }
    if (c->radial) {
        set_error("kde_snap: Eq. 7's separable window needs a product kernel");
        return KDE_EUNSUPPORTED;
    }
    if (c->g.rb != 0 || c->g.re != c->g.H) {
        set_error("kde_snap: banded contexts are not supported");
        return KDE_EUNSUPPORTED;
    }
    DeviceGuard dg(c->p.device);
    if (!dg.ok) return cuda_fail(cudaGetLastError(), "kde_snap: cudaSetDevice");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "kde_snap: earlier asynchronous error");
    bool host = false;
    if (n > 0) {
        int dx = -1, dy = -1, dl = -1;
        const bool xd = is_device_ptr(x, &dx), yd = is_device_ptr(y, &dy);
        const bool ld = label ? is_device_ptr(label, &dl) : xd;
        if (xd != yd || ld != xd) {
            set_error("kde_snap: x, y (and label) must all be host or all device pointers");
            return KDE_EINVAL;
        }
        if (xd && (dx != c->p.device || dy != c->p.device || (label && dl != c->p.device))) {
            set_error("kde_snap: device pointers on another device than the context's");
            return KDE_EINVAL;
        }
        host = !xd;
    }
    return snap_run(c, x, y, label, n, counts, out, (cudaStream_t)stream, host);
}

int kde_dp(const double* x, const double* y, const int64_t* traj_offsets, int64_t ntraj, double eps,
           uint8_t* keep, int32_t device, void* stream, int64_t* n_kept, int64_t* rounds) {
    if (ntraj < 0 || !(eps >= 0.0) || !isfinite(eps)) {
        set_error("kde_dp: ntraj = %lld, eps = %g (need ntraj >= 0, finite eps >= 0)", (long long)ntraj, eps);
        return KDE_EINVAL;
    }
    if (!traj_offsets) {
        set_error("kde_dp: NULL traj_offsets");
        return KDE_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        set_error("kde_dp: no CUDA device %d (no CPU fallback exists)", device);
        return KDE_ECUDA;
    }
    DeviceGuard dg(device);
    if (!dg.ok) return cuda_fail(cudaGetLastError(), "kde_dp: cudaSetDevice");
    cudaStream_t s = (cudaStream_t)stream;
    int dd = -1;
    const bool dev = is_device_ptr(traj_offsets, &dd);
    // the offsets decide every index the kernels touch: validate them on the host
    // (offsets[0] == 0, nondecreasing; n = offsets[ntraj]) -- device offsets are copied back
    // once (8 B per trajectory)
    std::vector<int64_t> ho((size_t)ntraj + 1);
    if (dev) {
        if (cudaMemcpyAsync(ho.data(), traj_offsets, sizeof(int64_t) * (ntraj + 1), cudaMemcpyDeviceToHost, s) !=
                cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return cuda_fail(cudaGetLastError(), "kde_dp: offsets readback");
    } else {
        memcpy(ho.data(), traj_offsets, sizeof(int64_t) * (ntraj + 1));
    }
    if (ho[0] != 0) {
        set_error("kde_dp: traj_offsets[0] = %lld (must be 0)", (long long)ho[0]);
        return KDE_EINVAL;
    }
    for (int64_t t = 0; t < ntraj; t++)
        if (ho[t + 1] < ho[t]) {
            set_error("kde_dp: traj_offsets decrease at %lld", (long long)t);
            return KDE_EINVAL;
        }
    const int64_t n = ho[ntraj];
    if (n < 0 || n > 2147483647ll - 4096) {
        set_error("kde_dp: %lld points outside [0, 2^31 - 4097]", (long long)n);
        return KDE_EINVAL;
    }
    if (n_kept) *n_kept = 0;
    if (rounds) *rounds = 0;
    if (n == 0) return KDE_OK;
    if (!x || !y || !keep) {
        set_error("kde_dp: NULL x, y or keep");
        return KDE_EINVAL;
    }
    int d1 = -1, d2 = -1, d3 = -1;
    if (is_device_ptr(x, &d1) != dev || is_device_ptr(y, &d2) != dev || is_device_ptr(keep, &d3) != dev) {
        set_error("kde_dp: x, y, traj_offsets and keep must all be host or all device pointers");
        return KDE_EINVAL;
    }
    if (dev && (d1 != device || d2 != device || d3 != device || dd != device)) {
        set_error("kde_dp: device pointers must be on device %d", device);
        return KDE_EINVAL;
    }
    if (dev) return dp_run(x, y, traj_offsets, (int)ntraj, (int)n, eps, keep, s, n_kept, rounds);
    // host inputs: stage on the device, copy the mask back
    double *dx = nullptr, *dy = nullptr;
    int64_t* doff = nullptr;
    uint8_t* dk = nullptr;
    cudaError_t e = cudaMalloc(&dx, sizeof(double) * n);
    if (e == cudaSuccess) e = cudaMalloc(&dy, sizeof(double) * n);
    if (e == cudaSuccess) e = cudaMalloc(&doff, sizeof(int64_t) * (ntraj + 1));
    if (e == cudaSuccess) e = cudaMalloc(&dk, n);
    int rc = KDE_OK;
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("kde_dp: staging allocation failed");
        rc = KDE_ENOMEM;
    } else {
        cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dy, y, sizeof(double) * n, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(doff, traj_offsets, sizeof(int64_t) * (ntraj + 1), cudaMemcpyHostToDevice, s);
        rc = dp_run(dx, dy, doff, (int)ntraj, (int)n, eps, dk, s, n_kept, rounds);
        if (rc == KDE_OK) {
            e = cudaMemcpyAsync(keep, dk, n, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) rc = cuda_fail(e, "kde_dp: mask readback");
        }
    }
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(doff);
    cudaFree(dk);
    return rc;
}

int kde_ipc_export(const void* dev_ptr, void* handle, int64_t* offset) {
    if (!dev_ptr || !handle || !offset) {
        set_error("kde_ipc_export: NULL argument");
        return KDE_EINVAL;
    }
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, dev_ptr) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        set_error("kde_ipc_export: not a device pointer");
        return KDE_EINVAL;
    }
    DeviceGuard dg(at.device);
    // the allocation's base (IPC handles name whole allocations; a torch tensor may sit inside
    // a larger cached block): the driver's cuMemGetAddressRange, looked up at run time so the
    // library keeps no link-time dependency on libcuda (CPU-only hosts still load it)
    using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
    void* drv = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!drv) drv = dlopen("libcuda.so.1", RTLD_NOW);
    GetRange get_range = drv ? reinterpret_cast<GetRange>(dlsym(drv, "cuMemGetAddressRange_v2")) : nullptr;
    unsigned long long base_u = 0;
    size_t size = 0;
    if (!get_range || get_range(&base_u, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0) {
        set_error("kde_ipc_export: cuMemGetAddressRange unavailable or failed");
        return KDE_ECUDA;
    }
    void* base = reinterpret_cast<void*>((uintptr_t)base_u);
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, base);
    if (e != cudaSuccess) return cuda_fail(e, "kde_ipc_export");
    memcpy(handle, &h, sizeof h);
    *offset = (int64_t)((const char*)dev_ptr - (const char*)base);
    return KDE_OK;
}

int kde_ipc_open(const void* handle, int32_t device, void** dev_ptr) {
    if (!handle || !dev_ptr) {
        set_error("kde_ipc_open: NULL argument");
        return KDE_EINVAL;
    }
    DeviceGuard dg(device);
    if (!dg.ok) return cuda_fail(cudaGetLastError(), "kde_ipc_open: cudaSetDevice");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "kde_ipc_open");
    return KDE_OK;
}

int kde_ipc_close(void* dev_ptr, int32_t device) {
    if (!dev_ptr) {
        set_error("kde_ipc_close: NULL argument");
        return KDE_EINVAL;
    }
    DeviceGuard dg(device);
    const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) return cuda_fail(e, "kde_ipc_close");
    return KDE_OK;
}

void kde_free(kde_ctx* c) {
    if (!c) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(c->p.device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    PointBufs& pb = c->pb;
    for (int k = 0; k < 2; k++) {
        cudaFree(pb.sx[k]);
        cudaFree(pb.sy[k]);
    }
    cudaFree(pb.key[0]);
    for (int k = 0; k < 2; k++) cudaFree(pb.pair[k]);
    cudaFree(pb.rec);
    cudaFree(pb.hist);
    cudaFree(pb.ost[0]);
    cudaFree(pb.ost[1]);
    cudaFree(pb.scan_tmp);
    cudaFree(pb.xy);
    cudaFree(pb.rng);
    cudaFree(pb.cx);
    cudaFree(pb.cy);
    cudaFree(pb.cidx);
    cudaFree(pb.bcnt);
    cudaFree(pb.nfin);
    cudaFree(c->d_offsets);
    cudaFree(c->d_stats);
    free_plan(c->plan[0]);
    free_plan(c->plan[1]);
    snap_free(c);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (int k = 0; k < 2; k++)
        if (c->stage_free[k]) cudaEventDestroy(c->stage_free[k]);
    if (c->stage_ready) cudaEventDestroy(c->stage_ready);
    if (c->loaded_ev) cudaEventDestroy(c->loaded_ev);
    if (c->evald_ev) cudaEventDestroy(c->evald_ev);
    if (c->input_ev) cudaEventDestroy(c->input_ev);
    if (c->stats_ev) cudaEventDestroy(c->stats_ev);
    for (int k = 0; k < 6; k++)
        if (c->tev[k]) cudaEventDestroy(c->tev[k]);
    if (c->h_totals) cudaFreeHost(c->h_totals);
    delete c;
    if (prev >= 0) cudaSetDevice(prev);
}

}  // extern "C"
