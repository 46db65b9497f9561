/*
 * kde.h -- C ABI of libkde.so, the B200 (sm_100a) gridded kernel density
 * estimate of arxiv 2004.13653's visualisation hot path.
 *
 * Citations: P:n = PAPER.md line n (the paper's LaTeX source).
 * §2 restates the operation; DESIGN.md §5 lists the readings (R1..R22).
 *
 * Entry points: kde_create / kde_load_points / kde_eval / kde_get_stats /
 * kde_get_bins / kde_set_timing / kde_get_timing / kde_free (the continuous KDE
 * below, steps a1-a5 of SURVEY.md §8), kde_snap (the paper's own Alg. 3 + Eq. 7
 * pipeline), kde_dp (GPU Douglas-Peucker), kde_last_error.
 *
 * What it computes (the north star's formula with the paper's Table 1
 * kernels, and Eq. 7's truncated window):
 *
 *   density(i,j) = 1/(n * h_px^2) * sum_{p : S(i,j,p)} K(s,t),
 *   s = (i + 1/2 - u_p)/h_px,  t = (j + 1/2 - v_p)/h_px,
 *   u_p = (x_p - x0)/res,  v_p = (y_p - y0)/res,  h_px = h/res,
 *   S: ceil(u_p - 1/2 - R) <= i <= floor(u_p - 1/2 + R), same for j,
 *      with R = c_eff * h_px, c_eff = min(cutoff,1) for the compact kernels,
 *      cutoff for the Gaussian (Eq. 8 P:175-181 inclusive "<=");
 *   K(s,t) = k(s) k(t)            (product form, Table 1 as printed; default)
 *   K(s,t) = c2 * khat(sqrt(s^2+t^2)) and s^2+t^2 <= c_eff^2   (KDE_RADIAL)
 *
 * Pixel (i,j) has centre (x0 + (i+1/2) res, y0 + (j+1/2) res); row j = 0 is
 * the smallest y (Eq. 6's y~ = 1 at y_min).  Output is fp32,
 * row-major out[(j - row_begin) * width + i].  n is the number of finite
 * points passed to kde_load_points (points outside the raster stay in n).
 * n = 0 gives an all-zero raster.
 *
 * Support decisions (S) are made once per point in IEEE fp64 (round to
 * nearest, no contraction) during kde_load_points and carried as integer
 * ranges, so the fp32 (DIRECT) and fp16-operand tensor-core (TENSOR)
 * evaluations never disagree with the fp64 oracle about which box pairs are
 * included.  The radial disk test is made per pair in fp32.
 *
 * Threading: one context per host thread; no global state except the
 * thread-local error message.  No CPU fallback exists: every entry point
 * that computes runs CUDA kernels on params.device.
 */
#ifndef KDE_H
#define KDE_H

#include <stdint.h>

#if defined(__GNUC__)
#define KDE_API __attribute__((visibility("default")))
#else
#define KDE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Kernel ids in Table 1 order. */
enum {
    KDE_UNIFORM = 0,
    KDE_TRIANGULAR = 1,
    KDE_EPANECHNIKOV = 2,
    KDE_QUARTIC = 3,
    KDE_TRIWEIGHT = 4,
    KDE_TRICUBE = 5,
    KDE_GAUSSIAN = 6,
    KDE_COSINE = 7
};
/* OR into kernel: radial form K = c2 * khat(||(s,t)||) (R1). */
#define KDE_RADIAL 0x100

/* Evaluation paths (kde_eval). */
enum {
    KDE_PATH_DIRECT = 0, /* fp32 FMA/MUFU tiled evaluation, all kernels, both forms   */
    KDE_PATH_TENSOR = 1, /* tcgen05 tensor-core A*B^T, product form of all 8 kernels
                            (Table 1 rows are k(s)k(t); fp16 operands,
                            10-bit mantissa like tf32, fp32 accumulation in TMEM)      */
    KDE_PATH_TENSOR_SPLIT = 2 /* the same contraction with split-fp16 operands
                            f = hi + lo (both fp16): A_hi B_hi + A_hi B_lo + A_lo B_hi,
                            3 MMAs per K step (3 x tc_mma_flops), ~fp32 accuracy: the
                            DIRECT path's 1e-5 bar (NEXT-F4 accuracy mode)           */
};

/* Return codes. */
enum {
    KDE_OK = 0,
    KDE_EINVAL = -1,        /* bad argument (see each call)                        */
    KDE_ENOMEM = -2,        /* device allocation failed                            */
    KDE_ECUDA = -3,         /* CUDA launch / runtime error (incl. earlier async)    */
    KDE_EUNSUPPORTED = -4,  /* valid request this build does not implement         */
    KDE_ESTATE = -5         /* call out of order (e.g. eval before load)           */
};

typedef struct kde_ctx kde_ctx; /* opaque; owns every device buffer it allocates */

typedef struct {
    double x0, y0;      /* raster lower-left corner, world units (e.g. Mercator metres)  */
    double res;         /* pixel edge, world units; > 0 and finite                        */
    int32_t width;      /* W columns (x), 1..32767                                        */
    int32_t height;     /* H rows (y), 1..32767                                           */
    double h;           /* bandwidth, world units; > 0 and finite                         */
    int32_t kernel;     /* KDE_UNIFORM..KDE_COSINE, optionally | KDE_RADIAL               */
    double cutoff;      /* support half-width in units of h; > 0 (compact kernels clamp
                           it to 1); e.g. 4 for the Gaussian                               */
    int32_t row_begin;  /* owned band [row_begin, row_end) for row-band sharding;          */
    int32_t row_end;    /*   0,0 = all rows.  Otherwise 0 <= row_begin < row_end <= H.     */
    int32_t device;     /* CUDA device ordinal                                            */
} kde_params;

typedef struct {
    int64_t n_in;          /* points passed to the last kde_load_points                    */
    int64_t n_finite;      /* finite points = the n of 1/(n h^2)                           */
    int64_t n_binned;      /* points kept for evaluation                                   */
    int64_t n_outside;     /* finite points dropped: window misses the raster, or (banded)
                              home bucket row outside [band_lo, band_hi]                   */
    int64_t useful_pairs;  /* sum over kept points of |box window clipped to raster
                              columns x band rows| = (pixel, point) pairs inside the box
                              support; the "kernel evaluations" of the metric              */
    int32_t bucket;        /* bucket edge B in pixels (power of two)                       */
    int32_t nbx, nby;      /* bucket grid ceil(W/B) x ceil(H/B)                            */
    int32_t reach_px;      /* ceil(R + 1/2) + 1: max pixel distance window <- home pixel   */
    int32_t stack;         /* bucket rows per tensor-core group (1 if that path is off); the
                              band filter keeps whole stacks                                */
    int32_t band_lo, band_hi; /* kept home-bucket rows: [floor(l/stack)*stack,
                              (floor(h/stack)+1)*stack - 1] with l = rb/B - nr,
                              h = (re-1)/B + nr, nr = ceil(reach_px/B)                      */
    int64_t kernel_launches; /* CUDA kernels this context has launched so far (cumulative)  */
    int64_t tc_mma_flops;  /* tensor-core flops one KDE_PATH_TENSOR eval of the last load
                              executes (2 per MMA multiply-add; 0 until that path has been
                              evaluated for the load): the tensor-pipe roofline numerator   */
    int32_t main_kernel;   /* the main (a3/a4) kernel of the last kde_eval: 0 none yet,
                              1 splat_kernel (direct), 2 tc_splat_kernel (tensor, eval_tc.cu),
                              3 tc5_kernel (tensor, per-warp pipelines, eval_tc5.cu)         */
    int32_t tc_m;          /* MMA M (accumulator and splat-slot rows) of the tensor-core path's
                              plan: 64 when a group window has <= 64 rows and <= 48 columns
                              (eval_tc5.cu's M = 64 tiles), else 128; 0 if the path is off  */
} kde_stats;

/*
 * kde_create: validate params, plan (bucket size, tiles), and bind the device.  The
 * parameters are the paper's problem statement (a u x v grid over the area, Eq. 7's
 * kernel window P:167-182, the Table 1 kernel P:150-157) with h explicit (R2).
 * Allocates no point-sized buffers and launches no kernels.
 *   p    [in]  parameters, copied.
 *   out  [out] new context; set to NULL on error.
 * Errors: KDE_EINVAL for NULL pointers, res/h/cutoff not > 0 or not finite,
 *   width/height outside 1..32767, unknown kernel id or flag bits, band not
 *   0,0 and not 0 <= row_begin < row_end <= height; KDE_ECUDA if the device
 *   cannot be selected.
 */
KDE_API int kde_create(const kde_params* p, kde_ctx** out);

/*
 * kde_load_points: replace the context's point set and bin it (steps a1/a2: the
 * projection of every point onto the grid, Eqs. 5-6 P:133-139 / Alg. 3 steps 1-2
 * P:359-373, here onto the fixed world grid with integer support ranges, R5,
 * and the counting sort that replaces Alg. 3's atomicAdd).
 * A banded context (row_begin/row_end set) first compacts, in input order, the points
 * whose home-bucket row lies within the band's reach, and sorts only those (one 4-byte
 * readback sizes the sort; n_finite still counts every finite point, R4/R22).
 *   x, y [in] n fp64 coordinates (world units), structure-of-arrays; either
 *             both host pointers (copied to the device through a pinned staging
 *             buffer) or both device pointers on params.device.  Not retained.
 *   n    [in] >= 0 (0 is legal: kde_eval then writes zeros); < 2^30 (the sort's counters;
 *             KDE_EUNSUPPORTED otherwise).
 * Enqueues a1 (fp64 convert, integer support ranges, bucket keys) and a2 (stable
 * LSD counting sort by bucket key -- one cooperative launch per radix pass, all of
 * whose CTAs must be co-resident: a device shared with other work can refuse it,
 * KDE_ECUDA -- and the gather to bucket-local fp32 SoA) on the
 * context's internal stream and returns without waiting for them (the integer
 * stats come back asynchronously; kde_get_stats waits).  Ordering: device
 * inputs are read after all work already queued on the legacy default stream
 * (PyTorch's default stream); binning starts after the context's previous
 * kde_eval has finished reading the bins; a host-input upload runs on the
 * context's copy stream into one of two staging buffers, overlapping the
 * previous load's binning and evaluation (pinned host memory makes it
 * asynchronous: the caller keeps pinned x, y unchanged until the load has
 * completed -- e.g. until a later kde_eval's stream reaches that eval, or
 * kde_get_stats returns; pageable memory is copied before the call returns).
 * Non-finite points are dropped and not counted in n.
 * Errors: KDE_EINVAL (NULL ctx, n < 0, NULL x/y with n > 0, mixed host/device),
 *   KDE_ENOMEM, KDE_ECUDA.
 */
KDE_API int kde_load_points(kde_ctx* c, const double* x, const double* y, int64_t n);

/*
 * kde_eval: evaluate the band's raster (steps a3/a4 + a5) into out: Eq. 7's kernel
 * smoothing as the continuous KDE of DESIGN.md §2, scale 1/(n h_px^2).
 *   path   [in] KDE_PATH_DIRECT or KDE_PATH_TENSOR.
 *   out    [out] device pointer on params.device, (row_end-row_begin)*width fp32
 *                (all H*W when the band is 0,0), caller-owned; fully overwritten.
 *   stream [in] cudaStream_t (NULL = legacy default stream).  Stream-ordered and
 *               asynchronous: results are ready when the stream reaches this point.
 * The first eval of a path after a load also builds that path's device-side plan
 * on `stream`, without a host round trip (buffers are reserved at
 * their upper bounds; only a window so large that the bound exceeds 1/8 of device
 * memory costs one 4-byte readback).  Evals of one context run in call order.
 * Deterministic: the same inputs give bitwise-identical output, and a banded
 * context gives exactly the rows of the unbanded raster.
 * Errors: KDE_EINVAL (NULL ctx/out, unknown path), KDE_ESTATE (no kde_load_points
 *   yet), KDE_EUNSUPPORTED (TENSOR or TENSOR_SPLIT with a radial kernel), KDE_ECUDA (launch error,
 *   or an earlier asynchronous fault).
 */
KDE_API int kde_eval(kde_ctx* c, int32_t path, float* out, void* stream);

/* kde_get_stats: counters of the last load (all zero before one); waits for the
 * load's asynchronous stats readback (and reads tc_mma_flops from the device).
 * Errors: KDE_EINVAL on NULL, KDE_ECUDA. */
KDE_API int kde_get_stats(const kde_ctx* c, kde_stats* s);

/*
 * kde_get_bins: copy the binning result of the last load to HOST memory for
 * inspection (bit-exact parity tests).  Any pointer may be NULL to skip it.
 *   offsets [nbx*nby+1] int64   bucket start positions (exclusive scan of counts); the
 *                               bucket key is column-major, key = bx * nby + by, with
 *                               (bx, by) = (clamp(floor(u))/B, clamp(floor(v))/B)
 *   perm    [n_binned]  int64   original index of each sorted point
 *   lx, ly  [n_binned]  float   bucket-local coordinates u - bx*B, v - by*B (fp64->RN fp32)
 *   ranges  [4*n_binned] int32  i_lo, i_hi, j_lo, j_hi (clipped to the raster)
 * Synchronous.  Errors: KDE_EINVAL, KDE_ESTATE, KDE_ECUDA.
 */
KDE_API int kde_get_bins(const kde_ctx* c, int64_t* offsets, int64_t* perm, float* lx, float* ly,
                 int32_t* ranges);

/*
 * Phase timing (CUDA events recorded on the streams the kernels run on), for the
 * benchmark's roofline: disabled by default; when enabled every load/eval records
 * events around its phases.  kde_get_timing synchronises on the last eval.
 *   bin_ms      a1 + a2 (convert, counting sort, gather) of the last load
 *   plan_ms     device-side plan built by the last eval (~0 when it was cached)
 *   main_ms     the evaluation kernel of the last eval (splat pass / tensor-core pass)
 *   combine_ms  the combine pass (a5) of the last eval
 * Errors: KDE_EINVAL (NULL), KDE_ESTATE (timing disabled or nothing recorded).
 */
typedef struct {
    float bin_ms, plan_ms, main_ms, combine_ms;
} kde_timing;
KDE_API int kde_set_timing(kde_ctx* c, int enable);
KDE_API int kde_get_timing(kde_ctx* c, kde_timing* t);

/*
 * kde_snap: the paper's own KDE pipeline, Alg. 3 + Eq. 7
 * (PAPER.md:133-142, 167-182, 340-390), on the context's u x v = width x height matrix:
 *   1. Eqs. 5-6: x~ = ceil((x - x_min)/(x_max - x_min) * (u - 1)) + 1 in [1, u] (y~ alike),
 *      x_min/x_max over the finite points of this call (fp64 RN, left to right); x_max =
 *      x_min maps every point to 1; non-finite points are skipped;
 *   2. M_D(x~, y~) = points projected there (Alg. 3 step 2, integer atomics: exact);
 *   3. Eqs. 12-13: adjacent points n, n+1 with label[n] == label[n+1] (Lt) and
 *      c_max = max(|dx~|, |dy~|) > 1 add the cells [x~ + c dx~/c_max], c = 1..c_max-1,
 *      [.] = round half up (R17-R19);
 *   4. Eq. 7: out = f (x) M_D, f(s,t) = K(s/h_px, t/h_px) with Table 1's constants (product
 *      form), |s|, |t| <= a = floor(c_eff h_px), zero padding; a separable two-pass fp32
 *      convolution (exact for product kernels).
 * Row r of M_D / out is y~ = r + 1 (row 0 = y_min), column i is x~ = i + 1.  x0, y0, res
 * only convert h to pixels (h_px = h/res).
 *   x, y    [in]  n fp64 coordinates, host or device (both the same kind).
 *   label   [in]  n int32 trajectory labels (same kind as x), or NULL: no interpolation.
 *   n       [in]  0 <= n < 2^31; n = 0 gives zeros.
 *   counts  [out] NULL, or device uint32[height*width]: M_D (caller-owned).
 *   out     [out] device fp32[height*width]: the Eq. 7 matrix (caller-owned).
 *   stream  [in]  cudaStream_t; stream-ordered (host inputs are copied on it first).
 * Errors: KDE_EINVAL (NULL ctx/x/y/out, n out of range, mixed host/device inputs),
 *   KDE_EUNSUPPORTED (radial kernel, or a banded context), KDE_ENOMEM, KDE_ECUDA.
 */
KDE_API int kde_snap(kde_ctx* c, const double* x, const double* y, const int32_t* label, int64_t n,
                     uint32_t* counts, float* out, void* stream);

/*
 * kde_dp: GPU Douglas-Peucker compression of a batch of trajectories (SURVEY.md §8f
 * NEXT-F3; PAPER.md:116-129 serial DP, §IV-A P:184-331 its GPU parallelisation), the
 * producer of the north star's "DP-compressed" inputs.  Level-synchronous: every round
 * computes the VED (Eq. 9, fp64, one rounding per operation) of every
 * unretained point to its current chord, keeps the earliest point of maximal VED of every
 * segment whose maximum is strictly larger than eps, and splits the segment there;
 * it stops when a round keeps nothing (trajectories of <= 4096 points run all their
 * rounds inside one CTA in shared memory).  The kept set equals the serial recursion's
 * (R14: strict >, earliest index on ties, degenerate chord -> point distance).
 *   x, y          [in]  n fp64 coordinates (n = traj_offsets[ntraj]), all trajectories
 *                       concatenated (the paper's merged store, TLen)
 *   traj_offsets  [in]  ntraj + 1 int64, nondecreasing, traj_offsets[0] = 0
 *   ntraj         [in]  >= 0
 *   eps           [in]  threshold, finite, >= 0 (same units as x, y)
 *   keep          [out] n uint8: 1 = retained (end points always)
 *   device        [in]  CUDA ordinal; stream [in] cudaStream_t
 *   n_kept, rounds [out] NULL or host int64: retained count, and the number of
 *                 levels that retained a point (the recursion depth)
 * Pointers: all device (on `device`) or all host (staged through the device).
 * Synchronous (one 4-byte readback per 4 rounds).  Errors: KDE_EINVAL (traj_offsets[0] != 0,
 * decreasing offsets, n out of range, pointers on another device), KDE_ENOMEM, KDE_ECUDA.
 * The offsets are validated on the host (device offsets are copied back once).  A point
 * with a non-finite coordinate has a NaN VED, which -- as in the serial recursion's
 * `d > dmax` -- never becomes a segment maximum.
 */
KDE_API int kde_dp(const double* x, const double* y, const int64_t* traj_offsets, int64_t ntraj, double eps,
                   uint8_t* keep, int32_t device, void* stream, int64_t* n_kept, int64_t* rounds);

/*
 * Peer-memory band assembly (NEXT-F4): rank 0 exports its H x W raster, every
 * other rank maps it and passes (mapped pointer + row_begin * width) as kde_eval's `out`, so
 * the combine kernel's epilogue stores the band straight into rank 0's memory -- over NVLink
 * P2P between GPUs (no separate gather), through the same device's memory in the one-GPU
 * tests.  The paper's SR counts every transfer; this removes the gather's.
 *   kde_ipc_export: handle [out] 64 bytes (cudaIpcMemHandle_t) of the allocation holding
 *                   dev_ptr [in] (a device pointer from cudaMalloc, e.g. a torch tensor's
 *                   storage); *offset [out] = dev_ptr minus the allocation's base.
 *   kde_ipc_open:   map another process's exported allocation on `device`; *dev_ptr [out]
 *                   = its base (add the exporter's offset).  Close with kde_ipc_close.
 * Synchronisation is the caller's: the exporter must not read the raster before every
 * writer's eval stream has completed (e.g. stream synchronise + a process-group barrier).
 * Errors: KDE_EINVAL (NULL), KDE_ECUDA.
 */
KDE_API int kde_ipc_export(const void* dev_ptr, void* handle, int64_t* offset);
KDE_API int kde_ipc_open(const void* handle, int32_t device, void** dev_ptr);
KDE_API int kde_ipc_close(void* dev_ptr, int32_t device);

/* Thread-local message describing the last non-OK return on this thread. */
KDE_API const char* kde_last_error(void);

/* Release the context and every device buffer it owns. NULL-safe. */
KDE_API void kde_free(kde_ctx* c);

#ifdef __cplusplus
}
#endif
#endif /* KDE_H */
