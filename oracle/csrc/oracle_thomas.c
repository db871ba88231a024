/* oracle_thomas.c -- TEST INFRASTRUCTURE ONLY (part of the CPU oracle).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code with the CUDA path.
 *
 * The Thomas algorithm (Gaussian elimination without pivoting on a
 * tridiagonal matrix: forward elimination, then back substitution), applied
 * to many independent systems.  The paper's fine solver is backward Euler
 * (P:648-650): each step solves (I + dt A) u_{j+1} = u_j + dt f(t_{j+1}); the
 * multi-right-hand-side direct solve of P:1074-1084 is this routine called on
 * a batch of vectors.
 *
 * System s (0 <= s < nsys) is
 *     sub[i] x[i-1] + (diag[i] + shift[s]) x[i] + sup[i] x[i+1] = rhs_s[i],
 * stored in place in X[s*n + i].  sub[0] and sup[n-1] are ignored.  shift may
 * be NULL (no shift).
 *
 * Pivots.  Elimination gives pivot_i = diag_i - sub_i sup_{i-1} / pivot_{i-1}.
 * If `rowsum` is given (rowsum_i = sub_i + diag_i + sup_i, supplied exactly by
 * the problem definition), the same pivots are computed from the row sums of
 * the reduced rows (reading R-ACC):
 *     r_0 = rowsum_0,  r_i = rowsum_i - sub_i r_{i-1} / pivot_{i-1},
 *     pivot_i = r_i - sup_i.
 * Algebraically identical; for diagonally dominant M-matrices (sub, sup <= 0,
 * rowsum >= 0 -- every operator here) all terms are non-negative, so the
 * pivots carry relative error O(u) instead of O(u * cond).  Without it the
 * coherent rounding of the pivots of I + dt A (dt/h^2 up to 2.5e4) shifts
 * the computed F' by ~ m u cond (4e-11 for C2, 1e-9 for C4).  The
 * elimination coefficients are recomputed for every system: plain and slow
 * by design.
 */
#include <stdlib.h>

void oracle_thomas_batch(int n, const double *sub, const double *diag, const double *sup,
                         const double *rowsum, const double *shift, long nsys, double *X)
{
#pragma omp parallel
    {
        double *cp = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(static)
        for (long s = 0; s < nsys; ++s) {
            double *x = X + s * (long)n;
            double sh = shift ? shift[s] : 0.0;
            double r = 0.0, den;
            /* forward elimination */
            if (rowsum) {
                r = rowsum[0] + sh;
                den = r - (n > 1 ? sup[0] : 0.0);
            } else {
                den = diag[0] + sh;
            }
            cp[0] = (n > 1 ? sup[0] : 0.0) / den;
            x[0] = x[0] / den;
            for (int i = 1; i < n; ++i) {
                double up = (i < n - 1 ? sup[i] : 0.0);
                if (rowsum) {
                    r = (rowsum[i] + sh) - sub[i] * (r / den);
                    den = r - up;
                } else {
                    den = (diag[i] + sh) - sub[i] * cp[i - 1];
                }
                cp[i] = up / den;
                x[i] = (x[i] - sub[i] * x[i - 1]) / den;
            }
            /* back substitution */
            for (int i = n - 2; i >= 0; --i)
                x[i] = x[i] - cp[i] * x[i + 1];
        }
        free(cp);
    }
}
