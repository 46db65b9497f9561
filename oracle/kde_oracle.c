/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU implementation of the gridded KDE
 * hot path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2004_13653_b200/csrc); it is compiled with -ffp-contract=off so every
 * fp64 operation is a single IEEE round-to-nearest step, in the written order.
 *
 * Citations: P:n = PAPER.md line n (arxiv 2004.13653 LaTeX source).
 *
 *   density(i,j) = 1/(n * h_px^2) * sum_{p : S(i,j,p)} K(s, t),
 *   s = (i + 1/2 - u_p)/h_px,  t = (j + 1/2 - v_p)/h_px          (R4)
 *   u_p = (x_p - x0)/res,      v_p = (y_p - y0)/res
 *   S: ceil(u_p - 1/2 - R) <= i <= floor(u_p - 1/2 + R), same for j (box,
 *      inclusive, Eq. 8 P:175-181 "|w| <= (w-1)/2"); radial adds s^2+t^2 <= c^2.
 *   R = c_eff * h_px, c_eff = min(cutoff, 1) for compact kernels, cutoff for
 *   the Gaussian (R3).
 *   K(s,t) = k(s) k(t) with k from Table 1 [product form], or
 *   K = c2 * khat(sqrt(s^2+t^2)) [radial form, R1].
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (closed forms, brute force, Eq. 7 convolution, properties) -- see DESIGN.md §4.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

typedef struct {
    double x0, y0, res;       /* grid lower-left corner, pixel edge (world units) */
    int32_t width, height;    /* W columns, H rows */
    double h;                 /* bandwidth (world units) */
    int32_t kernel;           /* 0..7 (Table 1 order), | 0x100 for radial */
    double cutoff;            /* support in units of h */
    int32_t row_begin, row_end; /* band [row_begin,row_end); 0,0 = all rows */
} oracle_params;

enum { UNIFORM = 0, TRIANGULAR, EPANECHNIKOV, QUARTIC, TRIWEIGHT, TRICUBE, GAUSSIAN, COSINE };
#define RADIAL_FLAG 0x100

/* Table 1: the 1-D factor k with f(s,t) = k(s) k(t). */
double oracle_k1(int kernel, double s)
{
    double a = fabs(s), q = 1.0 - s * s;
    switch (kernel) {
    case UNIFORM:      return 0.5;                                   /* (1/2)^2 I I */
    case TRIANGULAR:   return 1.0 - a;                               /* (1-|s|)(1-|t|) */
    case EPANECHNIKOV: return 0.75 * q;                              /* (3/4)^2 (1-s^2)(1-t^2) */
    case QUARTIC:      return (15.0 / 16.0) * q * q;                 /* (15/16)^2 (1-s^2)^2 .. */
    case TRIWEIGHT:    return (35.0 / 32.0) * q * q * q;             /* (35/32)^2 (1-s^2)^3 .. */
    case TRICUBE: {    double c = 1.0 - a * a * a;                    /* (70/81)^2 (1-|s|^3)^3 .. */
                       return (70.0 / 81.0) * c * c * c; }
    case GAUSSIAN:     return exp(-0.5 * s * s) / sqrt(2.0 * M_PI);  /* (1/sqrt(2pi))^2 exp(-(s^2+t^2)/2) */
    case COSINE:       return (M_PI / 4.0) * cos(0.5 * M_PI * s);    /* (pi/4)^2 cos(pi s/2) cos(pi t/2) */
    }
    return NAN;
}

/* Radial reading (R1): K = c2 * khat(r), c2 normalising the
 * integral over the unit disk (plane for the Gaussian) to 1. */
double oracle_kr(int kernel, double r)
{
    double q = 1.0 - r * r;
    switch (kernel) {
    case UNIFORM:      return 1.0 / M_PI;
    case TRIANGULAR:   return (3.0 / M_PI) * (1.0 - r);
    case EPANECHNIKOV: return (2.0 / M_PI) * q;
    case QUARTIC:      return (3.0 / M_PI) * q * q;
    case TRIWEIGHT:    return (4.0 / M_PI) * q * q * q;
    case TRICUBE: {    double c = 1.0 - r * r * r;
                       return (220.0 / (81.0 * M_PI)) * c * c * c; }
    case GAUSSIAN:     return exp(-0.5 * r * r) / (2.0 * M_PI);
    case COSINE:       return (M_PI / (4.0 * (M_PI - 2.0))) * cos(0.5 * M_PI * r);
    }
    return NAN;
}

/* c_eff (R3): compact kernels clamp the cutoff to their support 1. */
double oracle_ceff(const oracle_params *p)
{
    int k = p->kernel & 0xff;
    return (k == GAUSSIAN) ? p->cutoff : (p->cutoff < 1.0 ? p->cutoff : 1.0);
}

/* R_px = c_eff * (h / res): support half-width in pixels. */
double oracle_rpx(const oracle_params *p)
{
    double hpx = p->h / p->res;
    return oracle_ceff(p) * hpx;
}

/* ------------------------------------------------------------------------ */
/* Full / sampled pixel evaluation: the definition written out.              */

typedef struct {
    const oracle_params *p;
    const double *u, *v;        /* pixel coordinates of every finite point */
    const double *ilo, *ihi, *jlo, *jhi; /* unclipped support bounds (fp64 ints) */
    int64_t n;                  /* number of finite points */
    const int32_t *pi, *pj;
    double *out;
    uint8_t *tie;               /* radial near-tie flag per pixel, may be NULL */
    int64_t k0, k1;
} pix_job;

static void *pix_worker(void *arg)
{
    pix_job *J = (pix_job *)arg;
    const oracle_params *p = J->p;
    int kern = p->kernel & 0xff, radial = (p->kernel & RADIAL_FLAG) != 0;
    double hpx = p->h / p->res;
    double c = oracle_ceff(p);
    double c2 = c * c;
    for (int64_t k = J->k0; k < J->k1; k++) {
        double i = (double)J->pi[k], j = (double)J->pj[k];
        double acc = 0.0;
        int tie = 0;
        for (int64_t q = 0; q < J->n; q++) {      /* every point, input order */
            if (i < J->ilo[q] || i > J->ihi[q] || j < J->jlo[q] || j > J->jhi[q])
                continue;                          /* S(i,j,p): box, inclusive */
            double s = (i + 0.5 - J->u[q]) / hpx;
            double t = (j + 0.5 - J->v[q]) / hpx;
            if (!radial) {
                acc += oracle_k1(kern, s) * oracle_k1(kern, t);
            } else {
                double r2 = s * s + t * t;
                if (fabs(r2 - c2) <= 1e-6 * c2) tie = 1;
                if (r2 <= c2) acc += oracle_kr(kern, sqrt(r2));
            }
        }
        J->out[k] = acc;
        if (J->tie) J->tie[k] = (uint8_t)tie;
    }
    return NULL;
}

/*
 * Evaluate density at npix pixels (pi[k], pj[k]).  out[k] in density per
 * pixel area (R4).  tie (optional) flags pixels where a radial
 * pair lies within 1e-6*c^2 of the disk boundary (R3).
 * Returns the number of finite points n used for normalisation.
 */
int64_t oracle_kde_pixels(const oracle_params *p, const double *x, const double *y, int64_t n,
                          const int32_t *pi, const int32_t *pj, int64_t npix, double *out,
                          uint8_t *tie, int nthreads)
{
    double hpx = p->h / p->res;
    double R = oracle_rpx(p);
    double *u = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *v = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *b = malloc(sizeof(double) * 4 * (size_t)(n > 0 ? n : 1));
    int64_t m = 0;
    for (int64_t q = 0; q < n; q++) {
        if (!isfinite(x[q]) || !isfinite(y[q])) continue;   /* dropped, not counted in n */
        double uq = (x[q] - p->x0) / p->res;
        double vq = (y[q] - p->y0) / p->res;
        u[m] = uq;
        v[m] = vq;
        b[4 * m + 0] = ceil((uq - 0.5) - R);
        b[4 * m + 1] = floor((uq - 0.5) + R);
        b[4 * m + 2] = ceil((vq - 0.5) - R);
        b[4 * m + 3] = floor((vq - 0.5) + R);
        m++;
    }
    double *ilo = malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *ihi = malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *jlo = malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *jhi = malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    for (int64_t q = 0; q < m; q++) {
        ilo[q] = b[4 * q]; ihi[q] = b[4 * q + 1]; jlo[q] = b[4 * q + 2]; jhi[q] = b[4 * q + 3];
    }
    free(b);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    pix_job jobs[256];
    int64_t per = (npix + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; t++) {
        int64_t k0 = t * per, k1 = (t + 1) * per < npix ? (t + 1) * per : npix;
        jobs[t] = (pix_job){p, u, v, ilo, ihi, jlo, jhi, m, pi, pj, out, tie, k0, k1};
        if (k0 >= k1) continue;
        if (nthreads == 1) pix_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, pix_worker, &jobs[t]);
    }
    if (nthreads > 1)
        for (int t = 0; t < nthreads; t++)
            if (jobs[t].k0 < jobs[t].k1) pthread_join(th[t], NULL);
    /* normalisation 1/(n h_px^2), n = finite points (R4); n = 0 -> zeros (R9) */
    double scale = (m > 0) ? 1.0 / ((double)m * hpx * hpx) : 0.0;
    for (int64_t k = 0; k < npix; k++) out[k] = (m > 0) ? out[k] * scale : 0.0;
    free(u); free(v); free(ilo); free(ihi); free(jlo); free(jhi);
    return m;
}

/* ------------------------------------------------------------------------ */
/* Binning oracle (steps a1/a2): keys, support ranges,         */
/* bucket-local fp32 coordinates and a stable counting sort by key.          */

typedef struct {
    int64_t n_in, n_finite, n_binned, n_outside, useful_pairs;
} oracle_stats;

/* reach in pixels of a point's window from its home pixel (R12) */
int32_t oracle_reach_px(const oracle_params *p)
{
    return (int32_t)ceil(oracle_rpx(p) + 0.5) + 1;
}

/*
 * Bin n points into B x B pixel buckets.  For a band, keep points whose home bucket row is
 * in [floor(l/stack)*stack, (floor(h/stack)+1)*stack - 1], l = rb/B - nr, h = (re-1)/B + nr.
 *   outputs (caller-allocated, n entries / nb+1 entries):
 *   offsets[nb+1], perm[n], lx[n], ly[n] (float), rng[4n] (i_lo,i_hi,j_lo,j_hi; int32)
 * Returns n_binned.  nb = ceil(W/B) * ceil(H/B).
 */
static int32_t floordiv32(int32_t a, int32_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

int64_t oracle_bin(const oracle_params *p, int32_t B, int32_t stack, const double *x, const double *y,
                   int64_t n, int64_t *offsets, int64_t *perm, float *lx, float *ly, int32_t *rng,
                   oracle_stats *st)
{
    int32_t W = p->width, H = p->height;
    int32_t rb = p->row_begin, re = p->row_end;
    if (rb == 0 && re == 0) re = H;
    int32_t nbx = (W + B - 1) / B, nby = (H + B - 1) / B;
    int64_t nb = (int64_t)nbx * nby;
    double R = oracle_rpx(p);
    int32_t reach = oracle_reach_px(p);
    int32_t nr = (reach + B - 1) / B;                  /* neighbourhood in buckets */
    /* kept bucket rows: the band's reach, rounded out to whole stacks of `stack` rows */
    int32_t band_lo = floordiv32(rb / B - nr, stack) * stack;
    int32_t band_hi = (floordiv32((re - 1) / B + nr, stack) + 1) * stack - 1;

    int64_t *key = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int32_t *r4 = malloc(sizeof(int32_t) * 4 * (size_t)(n > 0 ? n : 1));
    double *uu = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *vv = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    memset(st, 0, sizeof(*st));
    st->n_in = n;
    for (int64_t q = 0; q < n; q++) {
        key[q] = -1;
        if (!isfinite(x[q]) || !isfinite(y[q])) continue;
        st->n_finite++;
        double u = (x[q] - p->x0) / p->res;
        double v = (y[q] - p->y0) / p->res;
        double ilo = ceil((u - 0.5) - R), ihi = floor((u - 0.5) + R);
        double jlo = ceil((v - 0.5) - R), jhi = floor((v - 0.5) + R);
        if (ilo < 0) ilo = 0;
        if (ihi > W - 1) ihi = W - 1;
        if (jlo < 0) jlo = 0;
        if (jhi > H - 1) jhi = H - 1;
        if (ilo > ihi || jlo > jhi) { st->n_outside++; continue; }   /* misses the grid */
        double fu = floor(u), fv = floor(v);
        int32_t hx = fu < 0 ? 0 : (fu > W - 1 ? W - 1 : (int32_t)fu);  /* home pixel, clamped */
        int32_t hy = fv < 0 ? 0 : (fv > H - 1 ? H - 1 : (int32_t)fv);
        int32_t bx = hx / B, by = hy / B;
        if (by < band_lo || by > band_hi) { st->n_outside++; continue; } /* outside band reach */
        key[q] = (int64_t)bx * nby + by;               /* column-major bucket key */
        r4[4 * q + 0] = (int32_t)ilo; r4[4 * q + 1] = (int32_t)ihi;
        r4[4 * q + 2] = (int32_t)jlo; r4[4 * q + 3] = (int32_t)jhi;
        uu[q] = u; vv[q] = v;
        /* useful pairs: window clipped to the grid columns and the band rows */
        int64_t jl = (int64_t)jlo < rb ? rb : (int64_t)jlo;
        int64_t jh = (int64_t)jhi > re - 1 ? re - 1 : (int64_t)jhi;
        if (jh >= jl) st->useful_pairs += ((int64_t)ihi - (int64_t)ilo + 1) * (jh - jl + 1);
    }
    /* stable counting sort by key (ties keep input order) */
    memset(offsets, 0, sizeof(int64_t) * (size_t)(nb + 1));
    for (int64_t q = 0; q < n; q++)
        if (key[q] >= 0) offsets[key[q] + 1]++;
    for (int64_t b = 0; b < nb; b++) offsets[b + 1] += offsets[b];
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(nb > 0 ? nb : 1));
    memcpy(fill, offsets, sizeof(int64_t) * (size_t)nb);
    for (int64_t q = 0; q < n; q++) {
        if (key[q] < 0) continue;
        int64_t d = fill[key[q]]++;
        int32_t bx = (int32_t)(key[q] / nby), by = (int32_t)(key[q] % nby);
        perm[d] = q;
        lx[d] = (float)(uu[q] - (double)(bx * B));  /* bucket-local, fp64 then RN to fp32 */
        ly[d] = (float)(vv[q] - (double)(by * B));
        memcpy(&rng[4 * d], &r4[4 * q], 4 * sizeof(int32_t));
    }
    st->n_binned = offsets[nb];
    free(fill); free(key); free(r4); free(uu); free(vv);
    return st->n_binned;
}
