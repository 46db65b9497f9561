// The C ABI of include/kde.h: validation, context lifecycle, load (a1/a2 + plan),
// eval dispatch (a3/a4/a5), stats, and error reporting.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <numeric>

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

template <class T>
static int upload(T** dptr, int* cap, const std::vector<T>& v, cudaStream_t s) {
    const int need = (int)v.size();
    if (need > *cap) {
        if (*dptr) cudaFree(*dptr);
        *dptr = nullptr;
        if (cudaMalloc(dptr, sizeof(T) * need) != cudaSuccess) {
            cudaGetLastError();
            set_error("cudaMalloc for plan failed");
            return KDE_ENOMEM;
        }
        *cap = need;
    }
    if (need) cudaMemcpyAsync(*dptr, v.data(), sizeof(T) * need, cudaMemcpyHostToDevice, s);
    return KDE_OK;
}

// Work plan for one evaluation path: tiles of tile_w x tile_h over the band, each with its
// neighbourhood candidate count from the bucket offsets; tiles with more than `seg`
// candidates are split into fixed-size segments (split-K).  Depends only on the
// neighbourhood contents, so a banded context plans each tile exactly as the unbanded one.
int build_plan(kde_ctx* c, int tile_w, int tile_h, int seg, EvalPlan& pl, int64_t slot_floats) {
    const Geom& g = c->g;
    pl.items.clear();
    pl.reds.clear();
    pl.nslots = 0;
    pl.any_empty = false;
    pl.ntx = (g.W + tile_w - 1) / tile_w;
    pl.nty0 = g.rb / tile_h;
    pl.nty1 = (g.re + tile_h - 1) / tile_h;
    const std::vector<uint32_t>& off = c->h_offsets;
    for (int ty = pl.nty0; ty < pl.nty1; ty++) {
        const int Y0 = ty * tile_h;
        const int by0 = std::max(Y0 / kBucket - g.nr, 0);
        const int by1 = std::min((Y0 + tile_h - 1) / kBucket + g.nr, g.nby - 1);
        for (int tx = 0; tx < pl.ntx; tx++) {
            const int X0 = tx * tile_w;
            const int bx0 = std::max(X0 / kBucket - g.nr, 0);
            const int bx1 = std::min((X0 + tile_w - 1) / kBucket + g.nr, g.nbx - 1);
            int64_t cand = 0;
            for (int by = by0; by <= by1; by++)
                cand += (int64_t)off[(size_t)by * g.nbx + bx1 + 1] - off[(size_t)by * g.nbx + bx0];
            if (cand == 0) {
                pl.any_empty = true;
                continue;
            }
            const int nseg = (int)((cand + seg - 1) / seg);
            if (nseg == 1) {
                pl.items.push_back({tx, ty, 0, (int)cand, -1, 0});
            } else {
                const int slot0 = pl.nslots;
                pl.nslots += nseg;
                for (int k = 0; k < nseg; k++)
                    pl.items.push_back({tx, ty, k * seg, (int)std::min<int64_t>(cand, (int64_t)(k + 1) * seg),
                                        slot0 + k, 0});
                pl.reds.push_back({tx, ty, slot0, nseg});
            }
        }
    }
    // heaviest first: the block scheduler then approximates longest-processing-time order
    std::stable_sort(pl.items.begin(), pl.items.end(), [](const WorkItem& a, const WorkItem& b) {
        return (a.k1 - a.k0) > (b.k1 - b.k0);
    });
    int rc = upload(&pl.d_items, &pl.d_items_cap, pl.items, c->stream);
    if (rc) return rc;
    rc = upload(&pl.d_reds, &pl.d_reds_cap, pl.reds, c->stream);
    if (rc) return rc;
    const int64_t need = (int64_t)pl.nslots * slot_floats;
    if (need > pl.partial_cap) {
        if (pl.d_partial) cudaFree(pl.d_partial);
        pl.d_partial = nullptr;
        if (cudaMalloc(&pl.d_partial, sizeof(float) * need) != cudaSuccess) {
            cudaGetLastError();
            set_error("cudaMalloc for split-K partials failed");
            return KDE_ENOMEM;
        }
        pl.partial_cap = need;
    }
    return KDE_OK;
}

static void free_plan(EvalPlan& pl) {
    cudaFree(pl.d_items);
    cudaFree(pl.d_reds);
    cudaFree(pl.d_partial);
    pl = EvalPlan();
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
    g.nbx = (g.W + kBucket - 1) / kBucket;
    g.nby = (g.H + kBucket - 1) / kBucket;
    const double reach = ceil(g.R + 0.5) + 1.0;
    if (!(reach < 1.0e6)) {
        delete c;
        set_error("kde_create: support R = %g px too large", g.R);
        return KDE_EINVAL;
    }
    g.reach = (int)reach;
    g.nr = (g.reach + kBucket - 1) / kBucket;
    g.band_lo = rb / kBucket - g.nr;
    g.band_hi = (re - 1) / kBucket + g.nr;
    const size_t nb = (size_t)g.nbx * g.nby;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_offsets, sizeof(uint32_t) * (nb + 1));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_stats, sizeof(unsigned long long) * 4);
    if (e != cudaSuccess) {
        kde_free(c);
        return cuda_fail(e, "kde_create: allocation");
    }
    c->h_offsets.assign(nb + 1, 0u);
    c->stats.bucket = kBucket;
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
        if (!xd) {  // host input: copy into the context's staging buffers
            if (c->pb.stage_cap < n) {
                cudaFree(c->pb.x);
                cudaFree(c->pb.y);
                c->pb.x = c->pb.y = nullptr;
                if (cudaMalloc(&c->pb.x, sizeof(double) * n) != cudaSuccess ||
                    cudaMalloc(&c->pb.y, sizeof(double) * n) != cudaSuccess) {
                    cudaGetLastError();
                    set_error("kde_load_points: staging allocation failed");
                    return KDE_ENOMEM;
                }
                c->pb.stage_cap = n;
            }
            cudaMemcpyAsync(c->pb.x, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream);
            cudaMemcpyAsync(c->pb.y, y, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream);
            dx = c->pb.x;
            dy = c->pb.y;
        }
    }
    int rc = bin_points(c, dx, dy, n);
    if (rc) return rc;
    const size_t nb = (size_t)c->g.nbx * c->g.nby;
    unsigned long long st[3];
    cudaMemcpyAsync(c->h_offsets.data(), c->d_offsets, sizeof(uint32_t) * (nb + 1),
                    cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(st, c->d_stats, sizeof st, cudaMemcpyDeviceToHost, c->stream);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "kde_load_points");
    c->stats.n_in = n;
    c->stats.n_finite = (int64_t)st[0];
    c->stats.n_outside = (int64_t)st[1];
    c->stats.useful_pairs = (int64_t)st[2];
    c->stats.n_binned = (int64_t)c->h_offsets[nb];
    rc = build_plan(c, kDirTile, kDirTile, kSegCands, c->plan_dir, (int64_t)kDirTile * kDirTile);
    if (rc) return rc;
    if (c->kern == KDE_GAUSSIAN && !c->radial) {
        rc = build_plan(c, kTcN, kTcM, kTcSegCands, c->plan_tc, (int64_t)kTcM * kTcN);
        if (rc) return rc;
    }
    e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "kde_load_points: plan upload");
    c->loaded = true;
    return KDE_OK;
}

int kde_eval(kde_ctx* c, int32_t path, float* out, void* stream) {
    if (!c || !out) {
        set_error("kde_eval: NULL argument");
        return KDE_EINVAL;
    }
    if (path != KDE_PATH_DIRECT && path != KDE_PATH_TENSOR) {
        set_error("kde_eval: unknown path %d", path);
        return KDE_EINVAL;
    }
    if (!c->loaded) {
        set_error("kde_eval: no points loaded");
        return KDE_ESTATE;
    }
    if (path == KDE_PATH_TENSOR && (c->radial || c->kern != KDE_GAUSSIAN)) {
        set_error("kde_eval: the tensor-core path implements the product-form Gaussian only");
        return KDE_EUNSUPPORTED;
    }
    DeviceGuard dg(c->p.device);
    if (!dg.ok) return cuda_fail(cudaGetLastError(), "kde_eval: cudaSetDevice");
    cudaError_t e = cudaGetLastError();  // surface earlier asynchronous faults
    if (e != cudaSuccess) return cuda_fail(e, "kde_eval: earlier asynchronous error");
    cudaStream_t s = (cudaStream_t)stream;
    return path == KDE_PATH_DIRECT ? launch_direct(c, out, s) : launch_tc(c, out, s);
}

int kde_get_stats(const kde_ctx* c, kde_stats* s) {
    if (!c || !s) {
        set_error("kde_get_stats: NULL argument");
        return KDE_EINVAL;
    }
    *s = c->stats;
    s->kernel_launches = c->launches;
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
    const size_t nb = (size_t)c->g.nbx * c->g.nby;
    const size_t m = (size_t)c->stats.n_binned;
    if (offsets)
        for (size_t b = 0; b <= nb; b++) offsets[b] = (int64_t)c->h_offsets[b];
    if (m == 0) return KDE_OK;
    std::vector<uint32_t> pv;
    std::vector<float2> xy;
    std::vector<uint2> rg;
    cudaError_t e = cudaSuccess;
    if (perm) {
        pv.resize(m);
        e = cudaMemcpy(pv.data(), c->pb.perm, sizeof(uint32_t) * m, cudaMemcpyDeviceToHost);
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

void kde_free(kde_ctx* c) {
    if (!c) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(c->p.device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    PointBufs& pb = c->pb;
    cudaFree(pb.x);
    cudaFree(pb.y);
    for (int k = 0; k < 2; k++) {
        cudaFree(pb.key[k]);
        cudaFree(pb.val[k]);
    }
    cudaFree(pb.hist);
    cudaFree(pb.scan_tmp);
    cudaFree(pb.xy);
    cudaFree(pb.rng);
    cudaFree(c->d_offsets);
    cudaFree(c->d_stats);
    free_plan(c->plan_dir);
    free_plan(c->plan_tc);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    if (prev >= 0) cudaSetDevice(prev);
}

}  // extern "C"
