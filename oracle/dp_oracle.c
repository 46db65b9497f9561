/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY (input generation for DP-compressed
 * workloads; never on the product path).
 *
 * Serial Douglas-Peucker (§III-B), explicit work stack in
 * place of recursion (the paper's own motivation).  Readings
 * (R14):
 *   - VED (Eq. 9): |P_sP_n x P_sP_e| / |P_sP_e|, distance to the
 *     chord's LINE; a degenerate chord (P_s == P_e) uses |P_n - P_s|;
 *   - split at the maximum VED, earliest index on ties;
 *   - a point is kept iff its VED is strictly larger than eps (P:125
 *     "larger than the pre-defined threshold").
 * Pinned by tests/test_oracle_dp.py (endpoints, threshold property,
 * monotonicity in eps, idempotence, brute-force recursion on small inputs).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

double oracle_ved(double px, double py, double sx, double sy, double ex, double ey)
{
    double dx = ex - sx, dy = ey - sy;
    double L = sqrt(dx * dx + dy * dy);
    if (L == 0.0) return sqrt((px - sx) * (px - sx) + (py - sy) * (py - sy));
    double cr = (px - sx) * dy - (py - sy) * dx;
    return fabs(cr) / L;
}

/* keep[k] = 1 for retained points of the trajectory x[0..n-1], y[0..n-1]. */
static void dp_one(const double *x, const double *y, int64_t n, double eps, uint8_t *keep,
                   int64_t *stack)
{
    for (int64_t k = 0; k < n; k++) keep[k] = 0;
    if (n <= 0) return;
    keep[0] = 1;
    keep[n - 1] = 1;
    if (n <= 2) return;
    int64_t top = 0;
    stack[top++] = 0;
    stack[top++] = n - 1;
    while (top > 0) {
        int64_t e = stack[--top];
        int64_t s = stack[--top];
        if (e - s < 2) continue;
        double dmax = -1.0;
        int64_t imax = -1;
        for (int64_t k = s + 1; k < e; k++) {
            double d = oracle_ved(x[k], y[k], x[s], y[s], x[e], y[e]);
            if (d > dmax) { dmax = d; imax = k; }   /* strict: earliest index wins ties */
        }
        if (dmax > eps) {
            keep[imax] = 1;
            stack[top++] = s; stack[top++] = imax;
            stack[top++] = imax; stack[top++] = e;
        }
    }
}

/* Compress every trajectory [offs[t], offs[t+1]) of the flat store. Returns kept count. */
int64_t oracle_dp_compress(const double *x, const double *y, const int64_t *offs, int64_t ntraj,
                           double eps, uint8_t *keep)
{
    int64_t maxlen = 0;
    for (int64_t t = 0; t < ntraj; t++)
        if (offs[t + 1] - offs[t] > maxlen) maxlen = offs[t + 1] - offs[t];
    int64_t *stack = malloc(sizeof(int64_t) * (size_t)(2 * maxlen + 4));
    int64_t kept = 0;
    for (int64_t t = 0; t < ntraj; t++) {
        int64_t a = offs[t], n = offs[t + 1] - a;
        dp_one(x + a, y + a, n, eps, keep + a, stack);
        for (int64_t k = 0; k < n; k++) kept += keep[a + k];
    }
    free(stack);
    return kept;
}
