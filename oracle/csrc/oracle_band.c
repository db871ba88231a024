/* oracle_band.c -- TEST INFRASTRUCTURE ONLY (part of the CPU oracle).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code with the CUDA path.
 *
 * "Oracle A" for the 2D fine solver: backward Euler
 * for the 5-point Laplacian on an n x n interior grid with
 * homogeneous Dirichlet conditions, h = 1/(n+1), unknown (ix, iy) at index
 * i = ix*n + iy (x index slowest).  Each step solves
 *
 *     (I + dt A) u_j = u_{j-1} + dt f(t_g),    A = (4 u_i - sum of the four
 *                                              neighbours) / h^2,
 *
 * by a banded Cholesky factorisation of the SPD matrix I + dt A (half
 * bandwidth n, Golub & Van Loan Alg. 4.3.5, row-oriented), computed once
 * and reused for every step and vector.  No sine transform, no eigenvalues:
 * the algorithm is independent of the separable ("oracle B", fine.py) and of
 * the GPU's sine-basis solver.
 *
 * Band storage: L[i*(bw+1) + (j - i + bw)] = L_ij for i - bw <= j <= i.
 */
#include <math.h>
#include <stdlib.h>

/* entry (i, j) of I + dt A, j in [i - n, i] */
static double band_entry(int n, double dt, double h2, long i, long j)
{
    if (i == j) return 1.0 + dt * 4.0 / h2;
    long d = i - j;
    long ix = i / n, iy = i % n;
    if (d == 1 && iy > 0) return -dt / h2;          /* (ix, iy-1) */
    if (d == n && ix > 0) return -dt / h2;          /* (ix-1, iy) */
    return 0.0;
}

/* Cholesky factor of I + dt A into L ((n*n) x (n+1) doubles), right-looking
 * (outer-product) order: for each column j, L_jj = sqrt(a_jj), L_ij = a_ij /
 * L_jj (j < i <= j + bw), then the trailing band update a_ik -= L_ij L_kj
 * (j < k <= i <= j + bw), rows in parallel.  Returns 0, or the 1-based row of
 * a non-positive pivot. */
long oracle_band_factor(int n, double dt, double *L)
{
    const long N = (long)n * n, bw = n, W = bw + 1;
    const double h = 1.0 / (n + 1), h2 = h * h;
    for (long i = 0; i < N; ++i)                     /* L := lower band of I + dt A */
        for (long j = i - bw; j <= i; ++j)
            L[i * W + (j - i + bw)] = (j >= 0) ? band_entry(n, dt, h2, i, j) : 0.0;
    double *col = (double *)malloc(sizeof(double) * (size_t)W);
    long bad = 0;
    for (long j = 0; j < N && !bad; ++j) {
        const double a = L[j * W + bw];
        if (!(a > 0.0)) { bad = j + 1; break; }
        const double d = sqrt(a);
        L[j * W + bw] = d;
        const long i1 = j + bw < N - 1 ? j + bw : N - 1;
        for (long i = j + 1; i <= i1; ++i) {
            L[i * W + (j - i + bw)] /= d;
            col[i - j] = L[i * W + (j - i + bw)];
        }
#pragma omp parallel for schedule(static) if (i1 - j > 64)
        for (long i = j + 1; i <= i1; ++i) {
            double *Li = L + i * W;
            const double lij = col[i - j];
            for (long k = j + 1; k <= i; ++k) Li[k - i + bw] -= lij * col[k - j];
        }
    }
    free(col);
    return bad;
}

/* x <- (L L^T)^{-1} x for nvec vectors x_v = X + v*N (forward, then back
 * substitution), OpenMP over vectors. */
void oracle_band_solve(int n, const double *L, long nvec, double *X)
{
    const long N = (long)n * n, bw = n, W = bw + 1;
#pragma omp parallel for schedule(static)
    for (long v = 0; v < nvec; ++v) {
        double *x = X + v * N;
        for (long i = 0; i < N; ++i) {               /* L y = x */
            const double *Li = L + i * W;
            const long j0 = i - bw > 0 ? i - bw : 0;
            double s = x[i];
            for (long j = j0; j < i; ++j) s -= Li[j - i + bw] * x[j];
            x[i] = s / Li[bw];
        }
        for (long i = N - 1; i >= 0; --i) {          /* L^T x = y, column by column */
            const double *Li = L + i * W;
            const long j0 = i - bw > 0 ? i - bw : 0;
            const double xi = x[i] / Li[bw];
            x[i] = xi;
            for (long j = j0; j < i; ++j) x[j] -= Li[j - i + bw] * xi;
        }
    }
}
