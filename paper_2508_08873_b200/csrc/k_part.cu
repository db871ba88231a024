// k_part.cu -- K1P: the cluster-partitioned 1D backward-Euler stepper (used
// for every 1D operator with 64 <= n <= 16384).
//
// The fused stepper (k_tridiag.cu) runs one vector per thread and streams the
// state through HBM once per step.  Here every vector's rows are split into
// P = CL * K chunks of L rows (rows >= n are decoupled identity rows): a
// thread-block cluster of CL CTAs owns a group of vectors, each CTA K chunks,
// each compute warp one chunk (H = 1, 32 vectors) or two adjacent chunks in its
// half-warps (H = 2, 16 vectors), and each lane keeps its chunk's L <= 64 state
// values in REGISTERS for all m steps.  One step (I + dt A) x = r
// by the partition method (reading R-PART):
//   x_c = T_c^{-1} r_c + V_c b_{c-1} + W_c t_{c+1}
//   V_c = T_c^{-1}(-a e_1), W_c = T_c^{-1}(-c e_L)     (spikes, fixed)
//   (t_c, b_c) = first / last unknown of chunk c, from the 2P x 2P interface
//   system z - V b - W t = g (rows at the chunk ends): a banded M-matrix.
// The interface system is solved in two levels: the K chunks of a CTA form a
// super-chunk with a local 2K x 2K system (band factors, two rows of its
// inverse, super-chunk spikes alpha = M_C^{-1} e_left, beta = M_C^{-1} e_right),
// and the CL super-chunks form a 2CL x 2CL system of the same shape whose
// inverse rows for each CTA's neighbours are stored.  All factorizations use
// row-sum (GTH-type) elimination of the M-matrices with row sums propagated
// exactly (reading R-ACC), so the inverses are entrywise accurate and
// non-negative.
//
// Pipelining.  Write the chunk solution of step j as
//   x_j = S_j + a_j V2 + c_j W2 + b_j V + t_j W,   V2 = T_c^{-1} V, W2 = T_c^{-1} W,
// with (a_j, c_j) = (b_{j-1}, t_{j-1}).  Then S_{j+1} = T_c^{-1}(S_j + a_j V2 + c_j W2
// + dt f_{j+1}) needs only the PREVIOUS step's interface values, so the sweep of
// step j+1 runs while the interface exchange of step j is in flight.  A
// dedicated interface warp per CTA forms the super-chunk values, sends them to
// every CTA of the cluster with st.async (distributed shared memory, completion
// counted on the receiver's mbarrier), gathers, and hands each chunk its
// neighbours' values through shared memory + mbarriers.  HBM is touched only
// to read the input and write the result.
#include <cooperative_groups.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>
#include <type_traits>

#include "pr_internal.cuh"

namespace cg = cooperative_groups;

namespace pr {

// dev aid: clock64 phase probes, compiled only with -DPR_PART_PROBES (they cost
// registers); PR_PART_PROF=1 then prints per-step phase cycles per CTA
#ifdef PR_PART_PROBES
#define PROBE_T(v) const long long v = clock64()
#define PROBE_DECL(v) long long v = 0
#define PROBE_SET(v) (v = clock64())
#define PROBE_ADD(slot, v) (pacc[slot] += (unsigned long long)(v))
#else
#define PROBE_T(v)
#define PROBE_DECL(v)
#define PROBE_SET(v)
#define PROBE_ADD(slot, v)
#endif
constexpr int PART_NPROBE = 16;
constexpr unsigned PART_IDLE_NS = 64;   // default interface-warp poll back-off

// per-CTA interface data (PART_CTAD doubles): band factors of the local
// interface matrix M_C (2K rows x 5) | alpha (2K) | beta (2K) | rows of the
// global inverse for B_{C-1} (2CL) and T_{C+1} (2CL) | rows 0 and 2K-1 of
// M_C^{-1} (2K each: the two values a CTA sends, off the band solve's chain)
constexpr int CTAD_A = 5 * 2 * PART_KMAX;
constexpr int CTAD_B = CTAD_A + 2 * PART_KMAX;
constexpr int CTAD_GB = CTAD_B + 2 * PART_KMAX;
constexpr int CTAD_GT = CTAD_GB + 2 * PART_CLMAX;
constexpr int CTAD_R0 = CTAD_GT + 2 * PART_CLMAX;     // row 0 of M_C^{-1} (T_C)
constexpr int CTAD_RM = CTAD_R0 + 2 * PART_KMAX;      // row 2K-1 of M_C^{-1} (B_C)
// split band solve (two halves of K rows each, R-PART): responses of the
// forward elimination of rows K..2K-1 to the carried values (y_{K-2}, y_{K-1})
// and of the back substitution of rows 0..K-1 to (x_K, x_{K+1})
constexpr int CTAD_FP = CTAD_RM + 2 * PART_KMAX;
constexpr int CTAD_FQ = CTAD_FP + PART_KMAX;
constexpr int CTAD_BR = CTAD_FQ + PART_KMAX;
constexpr int CTAD_BT = CTAD_BR + PART_KMAX;
// second half's back substitution (zero carried state) applied to the forward
// responses FP / FQ: with the forward and backward passes on separate warps
// (TM variants) the carried-pair correction of rows K..2K-1 is applied to the
// solution by the consumer, x_i += y_{K-2} PP_i + y_{K-1} PQ_i (linearity)
constexpr int CTAD_PP = CTAD_BT + PART_KMAX;
constexpr int CTAD_PQ = CTAD_PP + PART_KMAX;
static_assert(CTAD_PQ + PART_KMAX == PART_CTAD, "per-CTA interface data layout");

// ------------------------------------------------------------------ setup
// One thread per chunk c (rows s0..s0+L-1): local LU of T_c in row-sum form
// (pivots p_k, reading R-ACC), the local solves V, W (spikes),
// V2 = T_c^{-1} V, W2 = T_c^{-1} W and rho = T_c^{-1} s, and the chunk-local
// similarity scaling of the stepper (reading R-SCALE).
//
// Scaled form.  With x = D x~, D = diag(d_k), d_0 = 1, d_{k+1} = d_k p_k / (-c_k),
// the local solve T_c x = r becomes two one-coefficient recurrences
//   down  z~_k = r~_k + nl_k z~_{k-1},   nl_k = -(a_k / p_{k-1}) d_{k-1} / d_k
//   up    x~_k = w_k z~_k + x~_{k+1},    w_k  = 1 / p_k
// (the super-diagonal of the scaled U is -p_k, so its multiplier is exactly 1):
// 2 FMAs and 2 coefficients per row instead of 3 and 3.  Every term is
// non-negative for an M-matrix and non-negative data, as in the row-sum form.
// A chunk with a zero coupling c_k inside real rows (k < L-1, row < n-1) or a
// scale outside [2^-900, 2^900] cannot be scaled: *noscale is set and the
// operator uses the streaming stepper instead.  (c_k = 0 at row n-1 and on
// identity padding rows is harmless: the state there is exactly 0.)
//
// rowc row i (PART_ROWC): {w_i, nl_i, V2_i/d_i, W2_i/d_i, V_i, W_i, d_i, 1/d_i};
// ends[c] (PART_ENDS) = {rho, V, W at (top, bottom) of the chunk, 0, 0} (physical).
__global__ void k_part_setup(int n, int P, int L, const double *subA, const double *supA,
                             const double *rsA, const double *diagA, double dt, int transpose,
                             double *rowc, double *ends, int *bad, int *noscale)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P) return;
    const int s0 = c * L, e0 = s0 + L;
    auto a_of = [&](int i) -> double {              // (I + dt A)[i, i-1] (or of the transpose)
        if (i <= 0 || i >= n) return 0.0;
        return dt * (transpose ? supA[i - 1] : subA[i]);
    };
    auto c_of = [&](int i) -> double {              // (I + dt A)[i, i+1]
        if (i >= n - 1) return 0.0;
        return dt * (transpose ? subA[i + 1] : supA[i]);
    };
    auto s_of = [&](int i) -> double {              // row sums of I + dt A (1 on padding rows)
        if (i >= n) return 1.0;
        if (rsA) return 1.0 + dt * rsA[i];
        return a_of(i) + (1.0 + dt * diagA[i]) + c_of(i);
    };
    // local LU: T_c drops a_{s0} and c_{e0-1}; its row sums are s_i minus the
    // dropped (non-positive) entries
    double w[64], ga[64], cp[64], d[64];            // L <= 64
    double r = 0.0, den = 1.0;
    bool scal = true;
    for (int k = 0; k < L; ++k) {
        const int i = s0 + k;
        const double ai = (k == 0) ? 0.0 : a_of(i);
        const double ci = (k == L - 1) ? 0.0 : c_of(i);
        double sl = s_of(i);
        if (k == 0) sl -= a_of(i);
        if (k == L - 1) sl -= c_of(i);
        r = (k == 0) ? sl : sl - ai * (r / den);
        den = r - ci;
        if (!(den > 0.0) || !isfinite(den)) atomicExch(bad, 1);
        w[k] = 1.0 / den;
        ga[k] = w[k] * ai;
        cp[k] = w[k] * ci;
        if (k == 0) d[0] = 1.0;
        if (k + 1 < L) {
            if (ci != 0.0) {
                d[k + 1] = d[k] * (den / -ci);
            } else {
                d[k + 1] = d[k];
                if (i < n - 1) scal = false;
            }
            const double ad = fabs(d[k + 1]);
            if (!(ad < 0x1p900 && ad > 0x1p-900)) scal = false;
        }
    }
    if (!scal) atomicExch(noscale, 1);
    for (int k = 0; k < L; ++k) {
        double *R = rowc + (size_t)(s0 + k) * PART_ROWC;
        R[0] = w[k];
        R[1] = (k == 0) ? 0.0 : -(a_of(s0 + k) * w[k - 1]) * (d[k - 1] / d[k]);
        R[6] = d[k];
        R[7] = 1.0 / d[k];
    }
    // T_c x = rhs: forward y_k = w_k rhs_k - ga_k y_{k-1}, back x_k = y_k - cp_k x_{k+1}
    double y[64];
    double *E = ends + (size_t)c * PART_ENDS;
    for (int which = 0; which < 5; ++which) {       // 0 V, 1 W, 2 rho, 3 V2, 4 W2
        double yp = 0.0;
        for (int k = 0; k < L; ++k) {
            const double *R = rowc + (size_t)(s0 + k) * PART_ROWC;
            double rhs = 0.0;
            if (which == 0 && k == 0) rhs = -a_of(s0);
            if (which == 1 && k == L - 1) rhs = -c_of(e0 - 1);
            if (which == 2) rhs = s_of(s0 + k);
            if (which == 3) rhs = R[4];
            if (which == 4) rhs = R[5];
            yp = fma(-ga[k], yp, w[k] * rhs);
            y[k] = yp;
        }
        double xn = 0.0;
        for (int k = L - 1; k >= 0; --k) {
            double *R = rowc + (size_t)(s0 + k) * PART_ROWC;
            const double x = fma(-cp[k], xn, y[k]);
            if (which == 0) R[4] = x;
            if (which == 1) R[5] = x;
            if (which == 3) R[2] = x / d[k];
            if (which == 4) R[3] = x / d[k];
            if (which < 3) {
                const int top = which == 0 ? 2 : which == 1 ? 4 : 0;
                if (k == 0) E[top] = x;
                if (k == L - 1) E[top + 1] = x;
            }
            xn = x;
        }
    }
    E[6] = E[7] = 0.0;
}

// Banded M-matrix of order M <= 32 with offsets -2..+2 (A[i][d] at column
// i + d - 2, off-diagonals <= 0) and exact row sums rs[i] > 0, factored without
// pivoting: off-diagonals are updated with same-sign products, row sums with
// positive terms, and each pivot is (row sum) - (remaining off-diagonals).
// F[i] = {l_{i,i-2}, l_{i,i-1}, 1/u_ii, u_{i,i+1}, u_{i,i+2}}.
__device__ bool band_factor(int M, double (*A)[5], double *rs, double (*F)[5])
{
    bool ok = true;
    for (int i = 0; i < M; ++i) {
        double l2 = 0.0, l1 = 0.0;
        for (int dj = 2; dj >= 1; --dj) {
            const int j = i - dj;
            if (j < 0) continue;
            const double aij = A[i][2 - dj];
            if (aij == 0.0) continue;
            const double mult = aij * F[j][2];                 // a_ij / u_jj (<= 0)
            for (int e = 1; e <= 2; ++e) {
                const int di = j + e - i + 2;
                if (di >= 0 && di < 5) A[i][di] -= mult * F[j][2 + e];
            }
            rs[i] -= mult * rs[j];
            if (dj == 2) l2 = mult; else l1 = mult;
            A[i][2 - dj] = 0.0;
        }
        double off = 0.0;
        for (int e = 1; e <= 2; ++e)
            if (i + e < M) off += A[i][2 + e];
        const double piv = rs[i] - off;
        if (!(piv > 0.0) || !isfinite(piv)) ok = false;
        F[i][0] = l2;
        F[i][1] = l1;
        F[i][2] = 1.0 / piv;
        F[i][3] = (i + 1 < M) ? A[i][3] : 0.0;
        F[i][4] = (i + 2 < M) ? A[i][4] : 0.0;
    }
    return ok;
}

// x <- M^{-1} x with the factors (for x >= 0 every term is non-negative)
__device__ void band_solve(int M, const double (*F)[5], double *x)
{
    for (int i = 0; i < M; ++i) {
        if (i >= 2) x[i] -= F[i][0] * x[i - 2];
        if (i >= 1) x[i] -= F[i][1] * x[i - 1];
    }
    for (int i = M - 1; i >= 0; --i) {
        if (i + 1 < M) x[i] -= F[i][3] * x[i + 1];
        if (i + 2 < M) x[i] -= F[i][4] * x[i + 2];
        x[i] *= F[i][2];
    }
}

// Interface data (one thread).  Chunk-level rows of chunk c: row 2c (t_c) and
// 2c+1 (b_c):  z - V_c[end] b_{c-1} - W_c[end] t_{c+1} = g_c[end].
// Super-chunk C = chunks C*K .. C*K+K-1: local matrix M_C (couplings inside C)
// and its band factors, alpha_C = M_C^{-1} e_left (V of the first chunk),
// beta_C = M_C^{-1} e_right (W of the last chunk), rho_C = M_C^{-1} rho (row sums
// of the full rows).  Global rows of C:
//   T_C - alpha_C[0] B_{C-1} - beta_C[0] T_{C+1} = zloc_C[0]
//   B_C - alpha_C[2K-1] B_{C-1} - beta_C[2K-1] T_{C+1} = zloc_C[2K-1],  zloc_C = M_C^{-1} g_C.
// One block of 32 threads: thread C < CL prepares super-chunk C (local factors,
// responses, inverse rows, its two rows of the cluster-level system in shared
// memory); thread 0 then factors and inverts the cluster-level system.
__global__ void __launch_bounds__(32) k_part_iface(int CL, int K, const double *ends, double *ctad, int *bad)
{
    if (blockIdx.x != 0) return;
    constexpr int MX = 2 * (PART_KMAX > PART_CLMAX ? PART_KMAX : PART_CLMAX);
    double A[MX][5], rs[MX], F[MX][5], x[MX];
    __shared__ double gA[2 * PART_CLMAX][5], grs[2 * PART_CLMAX];
    const int M = 2 * K;
    bool ok = true;
    const int C = threadIdx.x;
    if (C < CL) {
        double *D = ctad + (size_t)C * PART_CTAD;
        for (int i = 0; i < PART_CTAD; ++i) D[i] = 0.0;
        for (int r = 0; r < M; ++r) {
            const int w = r / 2, e = r % 2;
            const double *E = ends + (size_t)(C * K + w) * PART_ENDS;
            for (int d = 0; d < 5; ++d) A[r][d] = 0.0;
            A[r][2] = 1.0;
            if (w > 0) A[r][(2 * w - 1) - r + 2] = -E[2 + e];
            if (w < K - 1) A[r][(2 * w + 2) - r + 2] = -E[4 + e];
            rs[r] = E[e] + (w == 0 ? E[2 + e] : 0.0) + (w == K - 1 ? E[4 + e] : 0.0);
        }
        ok = band_factor(M, A, rs, F) && ok;
        // stored for the stepper's interface warp with the back substitution
        // pre-scaled: {l2, l1, 1/u, u1/u, u2/u}, so its dependent chain is one
        // FMA per row in both directions
        for (int r = 0; r < M; ++r) {
            D[r * 5 + 0] = F[r][0];
            D[r * 5 + 1] = F[r][1];
            D[r * 5 + 2] = F[r][2];
            D[r * 5 + 3] = F[r][3] * F[r][2];
            D[r * 5 + 4] = F[r][4] * F[r][2];
        }
        if (K >= 2) {                                // split-solve responses (K rows per half)
            for (int e = 0; e < 2; ++e) {                // forward: carried (y_{K-2}, y_{K-1}) = unit
                double ym2 = e == 0 ? 1.0 : 0.0, ym1 = e == 0 ? 0.0 : 1.0;
                for (int r = K; r < M; ++r) {
                    const double y = -F[r][0] * ym2 - F[r][1] * ym1;
                    D[(e == 0 ? CTAD_FP : CTAD_FQ) + r - K] = y;
                    ym2 = ym1;
                    ym1 = y;
                }
            }
            for (int e = 0; e < 2; ++e) {                // backward: carried (x_K, x_{K+1}) = unit
                double xp1 = e == 0 ? 1.0 : 0.0, xp2 = e == 0 ? 0.0 : 1.0;
                for (int r = K - 1; r >= 0; --r) {
                    const double x = -(F[r][3] * F[r][2]) * xp1 - (F[r][4] * F[r][2]) * xp2;
                    D[(e == 0 ? CTAD_BR : CTAD_BT) + r] = x;
                    xp2 = xp1;
                    xp1 = x;
                }
            }
        }
        if (K >= 2) {                                // PP / PQ: back substitution of FP / FQ over rows K..2K-1
            for (int e = 0; e < 2; ++e) {
                double t1 = 0.0, t2 = 0.0;
                for (int r = M - 1; r >= K; --r) {
                    double t = D[(e == 0 ? CTAD_FP : CTAD_FQ) + r - K] * F[r][2];
                    if (r + 2 < M) t = fma(-(F[r][4] * F[r][2]), t2, t);
                    if (r + 1 < M) t = fma(-(F[r][3] * F[r][2]), t1, t);
                    D[(e == 0 ? CTAD_PP : CTAD_PQ) + r - K] = t;
                    t2 = t1;
                    t1 = t;
                }
            }
        }
        // rows 0 and M-1 of M_C^{-1}; for M = 32 the whole inverse (row-major)
        // for the tensor-core interface of the DM variant
        double *MI = ctad + (size_t)CL * PART_CTAD + (size_t)C * PART_MINV;
        for (int col = 0; col < M; ++col) {
            for (int r = 0; r < M; ++r) x[r] = (r == col) ? 1.0 : 0.0;
            band_solve(M, F, x);
            D[CTAD_R0 + col] = x[0];
            D[CTAD_RM + col] = x[M - 1];
            if (M * M == PART_MINV)
                for (int r = 0; r < M; ++r) MI[r * M + col] = x[r];
        }
        const double *E0 = ends + (size_t)(C * K) * PART_ENDS, *E1 = ends + (size_t)(C * K + K - 1) * PART_ENDS;
        for (int r = 0; r < M; ++r) x[r] = 0.0;
        x[0] = E0[2];
        x[1] = E0[3];
        band_solve(M, F, x);
        for (int r = 0; r < M; ++r) D[CTAD_A + r] = x[r];
        const double aT = x[0], aB = x[M - 1];
        for (int r = 0; r < M; ++r) x[r] = 0.0;
        x[M - 2] = E1[4];
        x[M - 1] = E1[5];
        band_solve(M, F, x);
        for (int r = 0; r < M; ++r) D[CTAD_B + r] = x[r];
        const double bT = x[0], bB = x[M - 1];
        for (int r = 0; r < M; ++r) x[r] = ends[(size_t)(C * K + r / 2) * PART_ENDS + r % 2];
        band_solve(M, F, x);
        // global rows 2C (T_C) and 2C+1 (B_C)
        for (int e = 0; e < 2; ++e) {
            const int r = 2 * C + e;
            for (int d = 0; d < 5; ++d) gA[r][d] = 0.0;
            gA[r][2] = 1.0;
            if (C > 0) gA[r][(2 * C - 1) - r + 2] = -(e ? aB : aT);
            if (C < CL - 1) gA[r][(2 * C + 2) - r + 2] = -(e ? bB : bT);
            grs[r] = e ? x[M - 1] : x[0];
        }
    }
    if (!ok) atomicExch(bad, 1);
    __syncthreads();
    if (threadIdx.x != 0) return;
    ok = true;
    const int MG = 2 * CL;
    ok = band_factor(MG, gA, grs, F) && ok;
    for (int col = 0; col < MG; ++col) {
        for (int r = 0; r < MG; ++r) x[r] = (r == col) ? 1.0 : 0.0;
        band_solve(MG, F, x);
        for (int C = 0; C < CL; ++C) {
            double *D = ctad + (size_t)C * PART_CTAD;
            D[CTAD_GB + col] = (C > 0) ? x[2 * C - 1] : 0.0;
            D[CTAD_GT + col] = (C < CL - 1) ? x[2 * C + 2] : 0.0;
        }
    }
    if (!ok) atomicExch(bad, 1);
}

// ------------------------------------------------------------------ stepper
struct PartArgs {
    int n, m;
    long B;
    const double *rowc;                // (P*L) x 8
    const double *ctad;                // CL x PART_CTAD, then CL x PART_MINV
    const double *in; long ld_in;      // null -> zero
    double *out; long ld_out;
    const double *off; long ld_off;
    // source (same convention as StepArgs): R == 0 none
    int R, RS;                         // RS: column stride of spaceT
    const double *spaceT;              // n x RS (zero padded)
    const double *time;
    const double *amp;
    int nsteps, nsrc, q0, vpi;
    long groups;                       // vector groups (VPG vectors each) over the persistent clusters
    double dt;
    unsigned long long *prof;          // dev aid (PR_PART_PROF): per-phase clock sums, or null
    unsigned idle_ns;                  // interface-warp poll back-off
    int noiface;                       // dev aid (PR_PART_NOIFACE): sweeps only, wrong results
};

constexpr int PART_RSM = 8;            // shared-memory stride of the source rows

// CTA shared memory (doubles): 8 mbarriers | gathered super-chunk values [2][CL][32]
// (double2) | chunk end values [2][K][32] (double2) | (B_{C-1}, T_{C+1}) [2][32]
// (double2) | interface data | per chunk: {w, -ga, V2, W2} [L] | -cp [L] | {V, W} [L] |
// source rows [L][8] (AFF) | cluster addresses [2][CL] (u32) | local solution [2][2K][32]
// (vector slots: 32 = the largest group, VPG <= 32)
// | carried pairs of the forward halves [2][32] (double2)
// | staged input of the next group [K*L][VPG] (when it fits; not AFF: the
// offsets launch has no input and its source rows take the space)
template <int CL, int W, int H, int L, int VPT, bool AFF>
__host__ __device__ constexpr size_t part_smem_base()
{
    constexpr int K = W * H;
    return (8 + (size_t)4 * CL * 32 + (size_t)4 * K * 32 + 4 * 32 + PART_CTAD +
            (size_t)K * (L * (4 + (AFF ? PART_RSM : 0)) + 4) + CL + (size_t)4 * K * 32 + 4 * 32 + 4 * 32) * sizeof(double);
}

template <int CL, int W, int H, int L, int VPT, bool AFF>
__host__ __device__ constexpr size_t part_stage_bytes()
{
    return (size_t)W * H * L * (32 / H) * VPT * sizeof(double);
}

template <int CL, int W, int H, int L, int VPT, bool AFF>
__host__ __device__ constexpr bool part_stage()
{
    return !AFF && part_smem_base<CL, W, H, L, VPT, AFF>() + part_stage_bytes<CL, W, H, L, VPT, AFF>() <= 227 * 1024;
}

template <int CL, int W, int H, int L, int VPT, bool AFF>
constexpr size_t part_smem_t()
{
    return part_smem_base<CL, W, H, L, VPT, AFF>() +
           (part_stage<CL, W, H, L, VPT, AFF>() ? part_stage_bytes<CL, W, H, L, VPT, AFF>() : 0);
}

__device__ __forceinline__ unsigned smem_u32(const void *p)
{
    return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ unsigned cluster_map(unsigned addr, unsigned rank)
{
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

__device__ __forceinline__ void st_async_v2(unsigned raddr, double x, double y, unsigned rbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 :: "r"(raddr), "d"(x), "d"(y), "r"(rbar) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity)
{
    unsigned done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    }
}

// the interface warps' waits span most of a sweep: back off between polls so
// the spinning warp does not take issue slots from the compute warps of its
// SM sub-partition
__device__ __forceinline__ void mbar_wait_idle(unsigned bar, unsigned parity, unsigned ns)
{
    unsigned done = 0;
    for (;;) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(bar), "r"(parity) : "memory");
        if (done) break;
        if (ns) __nanosleep(ns);
    }
}

__device__ __forceinline__ void mbar_arrive(unsigned bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory");
}

// ---- tensor memory (TMEM) as a per-lane coefficient store (TM variants).
// The sweeps are bound by the shared-memory coefficient stream (one LSU cycle
// per warp-wide LDS.64, broadcast or not): the two LU coefficients {nl, w} of
// a lane's chunk are kept in the SM's tensor memory instead (512 columns x
// 128 lanes x 32 bit; a warp reaches the 32 lanes of its quadrant, warps w and
// w + 4 share one: 256 columns = 128 doubles each) and read with
// tcgen05.ld.32x32b.x8 (4 rows per instruction, double buffered), which does
// not go through the LSU.  The spike coefficients stay in shared memory.
__device__ __forceinline__ void tm_ld8(unsigned addr, unsigned (&r)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
}

// the loaded registers are operands so that no consumer is scheduled above the
// wait (no memory clobber: shared-memory loads may move across TMEM reads)
__device__ __forceinline__ void tm_wait8(unsigned (&r)[8])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]));
}

__device__ __forceinline__ void tm_st8(unsigned addr, const unsigned (&r)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__device__ __forceinline__ double tm_dbl(const unsigned (&r)[8], int e)
{
    return __hiloint2double((int)r[2 * e + 1], (int)r[2 * e]);
}

// The interface warp's banded solve, streamed through shared memory: rows are
// processed in blocks of 8 whose operands are loaded (restrict: no aliasing
// with the stores) before the block's dependent chain runs, so each row
// costs one dependent FMA per direction.  g: raw ends of the K chunks
// (double2, stride 32), F: band factors (5 per row), z: the lane's column
// (stride 32).
template <int K>
__device__ __forceinline__ void band_forward(const double2 *__restrict__ g, const double *__restrict__ F,
                                             double *__restrict__ z, double &T0, double &T1, double &B0,
                                             double &B1)
{
    constexpr int BK = (K < 4) ? K : 4;   // chunks (2 BK rows) per block
    T0 = T1 = B0 = B1 = 0.0;
    double y1 = 0.0, y2 = 0.0;
#pragma unroll
    for (int u0 = 0; u0 < K; u0 += BK) {
        double2 gv[BK];
        double f0[2 * BK], f1[2 * BK];
#pragma unroll
        for (int b = 0; b < BK; ++b) {
            gv[b] = g[(u0 + b) * 32];
            f0[2 * b] = F[(2 * (u0 + b)) * 5 + 0];
            f1[2 * b] = F[(2 * (u0 + b)) * 5 + 1];
            f0[2 * b + 1] = F[(2 * (u0 + b) + 1) * 5 + 0];
            f1[2 * b + 1] = F[(2 * (u0 + b) + 1) * 5 + 1];
        }
        double out[2 * BK];
#pragma unroll
        for (int b = 0; b < BK; ++b) {
            const int i = 2 * (u0 + b);
            T0 = fma(F[CTAD_R0 + i], gv[b].x, T0);
            T1 = fma(F[CTAD_R0 + i + 1], gv[b].y, T1);
            B0 = fma(F[CTAD_RM + i], gv[b].x, B0);
            B1 = fma(F[CTAD_RM + i + 1], gv[b].y, B1);
            double y = gv[b].x;
            if (i >= 2) y = fma(-f0[2 * b], y2, y);
            if (i >= 1) y = fma(-f1[2 * b], y1, y);
            double yb = gv[b].y;
            if (i >= 1) yb = fma(-f0[2 * b + 1], y1, yb);
            yb = fma(-f1[2 * b + 1], y, yb);
            out[2 * b] = y;
            out[2 * b + 1] = yb;
            y2 = y;
            y1 = yb;
        }
#pragma unroll
        for (int r = 0; r < 2 * BK; ++r) z[(size_t)(2 * u0 + r) * 32] = out[r];
    }
}

template <int M>
__device__ __forceinline__ void band_backward(const double *__restrict__ F, double *__restrict__ z)
{
    constexpr int BR = (M < 8) ? M : 8;   // rows per block
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int i0 = M - BR; i0 >= 0; i0 -= BR) {
        double zv[BR], inv[BR], u1[BR], u2[BR];
#pragma unroll
        for (int r = 0; r < BR; ++r) {
            const int i = i0 + r;
            zv[r] = z[(size_t)i * 32];
            inv[r] = F[i * 5 + 2];
            u1[r] = F[i * 5 + 3];
            u2[r] = F[i * 5 + 4];
        }
#pragma unroll
        for (int r = BR - 1; r >= 0; --r) {
            const int i = i0 + r;
            double t = zv[r] * inv[r];
            if (i + 2 < M) t = fma(-u2[r], t2, t);
            if (i + 1 < M) t = fma(-u1[r], t1, t);
            zv[r] = t;
            t2 = t1;
            t1 = t;
        }
#pragma unroll
        for (int r = 0; r < BR; ++r) z[(size_t)(i0 + r) * 32] = zv[r];
    }
}

// Split band solve (K >= 2): the 2K rows of the local interface system in two
// halves of K rows.  Each half is eliminated from a zero carried state; the
// second half's forward values and the first half's back-substituted values
// are then corrected with the precomputed responses to the carried pair
// (CTAD_FP/FQ, CTAD_BR/BT), an exact rewriting (R-PART).  One lane per half
// (HI = 2: the two half-warps) or one lane doing both (HI = 1) performs the
// same operations in the same order, so the result does not depend on the
// group size.  Half hf: forward elimination over its rows from zero state.
template <int K>
__device__ __forceinline__ void half_forward(int hf, const double2 *__restrict__ g, const double *__restrict__ F,
                                             double *__restrict__ z, double &y2o, double &y1o)
{
    constexpr int NC = K / 2;                 // chunks per half
    constexpr int BK = (NC < 4) ? NC : 4;     // chunks per block
    const int c0 = hf * NC;
    double y1 = 0.0, y2 = 0.0;
#pragma unroll
    for (int u0 = 0; u0 < NC; u0 += BK) {
        double2 gv[BK];
        double f0[2 * BK], f1[2 * BK];
#pragma unroll
        for (int b = 0; b < BK; ++b) {
            const int i = 2 * (c0 + u0 + b);
            gv[b] = g[(c0 + u0 + b) * 32];
            f0[2 * b] = F[i * 5 + 0];
            f1[2 * b] = F[i * 5 + 1];
            f0[2 * b + 1] = F[(i + 1) * 5 + 0];
            f1[2 * b + 1] = F[(i + 1) * 5 + 1];
        }
        double out[2 * BK];
#pragma unroll
        for (int b = 0; b < BK; ++b) {
            const int r = 2 * (u0 + b);       // row within the half
            double y = gv[b].x;
            if (r >= 2) y = fma(-f0[2 * b], y2, y);
            if (r >= 1) y = fma(-f1[2 * b], y1, y);
            double yb = gv[b].y;
            if (r >= 1) yb = fma(-f0[2 * b + 1], y1, yb);
            yb = fma(-f1[2 * b + 1], y, yb);
            out[2 * b] = y;
            out[2 * b + 1] = yb;
            y2 = y;
            y1 = yb;
        }
#pragma unroll
        for (int r = 0; r < 2 * BK; ++r) z[(size_t)(2 * (c0 + u0) + r) * 32] = out[r];
    }
    y2o = y2;
    y1o = y1;
}

// back substitution over half hf from a zero carried state; returns the first
// two values of the half.  fix: the half's forward values first get the
// carried-pair correction y_i += y_{K-2} FP_i + y_{K-1} FQ_i (second half)
template <int K, bool NOFIX = false>
__device__ __forceinline__ void half_backward(int hf, const double *__restrict__ F, double *__restrict__ z,
                                              double &x0o, double &x1o, bool fix, double ym2, double ym1)
{
    constexpr int BR = (K < 8) ? K : 8;       // rows per block
    const int r0 = hf * K;
    if (!fix) ym2 = ym1 = 0.0;
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int i0 = K - BR; i0 >= 0; i0 -= BR) {
        double zv[BR], inv[BR], u1[BR], u2[BR];
#pragma unroll
        for (int r = 0; r < BR; ++r) {
            const int i = r0 + i0 + r;
            if constexpr (NOFIX) zv[r] = z[(size_t)i * 32];
            else zv[r] = fma(F[CTAD_FP + i0 + r], ym2, fma(F[CTAD_FQ + i0 + r], ym1, z[(size_t)i * 32]));
            inv[r] = F[i * 5 + 2];
            u1[r] = F[i * 5 + 3];
            u2[r] = F[i * 5 + 4];
        }
#pragma unroll
        for (int r = BR - 1; r >= 0; --r) {
            const int il = i0 + r;            // row within the half
            double t = zv[r] * inv[r];
            if (il + 2 < K) t = fma(-u2[r], t2, t);
            if (il + 1 < K) t = fma(-u1[r], t1, t);
            zv[r] = t;
            t2 = t1;
            t1 = t;
        }
#pragma unroll
        for (int r = 0; r < BR; ++r) z[(size_t)(r0 + i0 + r) * 32] = zv[r];
    }
    x0o = t1;
    x1o = t2;
}

// Interface super-values of a half (hf) of the local rows: the partial dot
// products of rows 0 / 2K-1 of M_C^{-1} with the raw ends (T_C, B_C), with
// four independent accumulators; sent before the band solve runs.
template <int K>
__device__ __forceinline__ void half_dots(int hf, const double2 *__restrict__ g, const double *__restrict__ F,
                                          double &T, double &B)
{
    constexpr int NC = K / 2;
    double T0 = 0.0, T1 = 0.0, B0 = 0.0, B1 = 0.0;
#pragma unroll
    for (int b = 0; b < NC; ++b) {
        const int cu = hf * NC + b, i = 2 * cu;
        const double2 gv = g[cu * 32];
        T0 = fma(F[CTAD_R0 + i], gv.x, T0);
        T1 = fma(F[CTAD_R0 + i + 1], gv.y, T1);
        B0 = fma(F[CTAD_RM + i], gv.x, B0);
        B1 = fma(F[CTAD_RM + i + 1], gv.y, B1);
    }
    T = T0 + T1;
    B = B0 + B1;
}

// Warps 0..W-1 each own H chunks (the warp's lanes split into H groups of
// LPC = 32/H lanes, one chunk each) and only sweep; each lane carries VPT
// vectors of its chunk, so a group of VPG = LPC * VPT vectors runs on a
// cluster and every shared-memory coefficient load feeds VPT independent
// recurrences.  Warps W (publish) and W+1 (gather) are the interface warps:
// the publish warp turns the chunks' raw end values into the super-chunk values
// (T_C, B_C) (two rows of the local inverse), sends them to every CTA of the
// cluster and then runs the banded local solve; the gather warp forms
// (B_{C-1}, T_{C+1}) from every CTA's values -- all while the compute warps
// run the next sweep (one-step lag, see the setup comment and R-PART).
// Hand-offs use mbarriers: ebar[p] (W compute warps arrive: raw ends of a
// step of parity p written), cbar[p] (publish + gather arrive: interface
// values of a step of parity p written); gbar[p] counts the gather bytes.
// TM variants (W = 8: every C4 / C2-sized launch) run 12 warps = 3 warpgroups:
// the two compute warpgroups raise their register budget to PART_TM_CREGS with
// setmaxnreg (room for the TMEM / spike-coefficient prefetch buffers next to the
// 128 state registers), the interface warpgroup (publish, gather, local solver,
// one idle warp) drops to PART_TM_IREGS.  setmaxnreg.inc blocks until the
// CTA's register pool (launch registers x threads) holds the increase, so the
// 8 compute warps may only take what the 4 interface warps released:
// 8 * (216 - 168) = 4 * (168 - 72).
constexpr int PART_TM_CREGS = 216, PART_TM_IREGS = 72, PART_TM_LREGS = 168;
static_assert(8 * (PART_TM_CREGS - PART_TM_LREGS) <= 4 * (PART_TM_LREGS - PART_TM_IREGS),
              "setmaxnreg.inc would wait forever for registers nobody releases");
template <bool TM> __host__ __device__ constexpr int part_ni() { return TM ? 4 : 2; }
template <int W, bool TM> __host__ __device__ constexpr int part_maxreg()
{
    constexpr int r = (65536 / (32 * (W + part_ni<TM>()))) / 8 * 8;
    return r > 255 ? 255 : r;
}

template <int CL, int W, int H, int L, int VPT, bool AFF, bool TM = false, bool DMV = true>
__global__ void __launch_bounds__(32 * (W + part_ni<TM>()), 1) __maxnreg__((part_maxreg<W, TM>())) k_part_step(PartArgs a)
{
    static_assert(!TM || (L == 64 && W == 8), "TMEM coefficient store: 2 x 64 doubles per lane, two warps per quadrant");
    static_assert(!TM || part_maxreg<W, TM>() == PART_TM_LREGS, "register pool accounting of the TM variants");
    __shared__ unsigned tm_slot;
    constexpr int LPC = 32 / H;          // lanes per chunk
    constexpr int VPG = LPC * VPT;       // vectors per cluster group
    static_assert(VPG == 16 || VPG == 32, "the interface warp splits 32 lanes over VPG vectors");
    constexpr int HI = 32 / VPG;         // interface-warp lanes per vector
    constexpr int K = W * H;             // chunks per CTA
    constexpr int M = 2 * K;             // local interface unknowns
    constexpr bool SPLIT = K >= 16;      // split band solve (two halves)
    constexpr bool SOLVER = TM && SPLIT; // the local band solve on its own warps, off the publish warp
    // DM: the local solve as a dense product z = M_C^{-1} g on the FP64 tensor cores
    // (32 x 32 inverse, 16 vectors), one 8-row tile per interface warp; T_C, B_C are
    // rows 0 and M-1 of the same product (DMV = false, PR_PART_NODM=1: the banded
    // solver warps instead)
    constexpr bool DM = DMV && SOLVER && M * M == PART_MINV && VPG == 16;
    constexpr int RSM = AFF ? PART_RSM : 0;
    constexpr bool STAGE = part_stage<CL, W, H, L, VPT, AFF>();   // next group's input prefetched into shared memory
    extern __shared__ __align__(16) double sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int C = (int)cluster.block_rank();
    // (measured: making the interface warps the hardware warps 0..3, the oldest of
    // each SM sub-partition, slows the C4 launch from 26.6 to 28.5 ms)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent clusters: cluster cid runs the vector groups cid, cid + ncl, ...
    // (its CTAs keep their coefficients in shared memory across groups)
    const long cid = (long)(blockIdx.x / CL), ncl = (long)(gridDim.x / CL);
    const long ngrp = (cid < a.groups) ? (a.groups - 1 - cid) / ncl + 1 : 0;
    unsigned long long *bar = reinterpret_cast<unsigned long long *>(sm);   // gbar[2] ebar[2] cbar[2] fbar[2]
    double2 *gth = reinterpret_cast<double2 *>(sm + 8);              // [2][CL][32]
    double2 *rawE = gth + 2 * CL * 32;                               // [2][K][32]
    double2 *coef = rawE + 2 * K * 32;                               // [2][32]: (B_{C-1}, T_{C+1})
    double *ctad = reinterpret_cast<double *>(coef + 2 * 32);
    double *regions = ctad + PART_CTAD;
    // chunk regions are padded by 4 doubles so that the chunks the lane groups
    // of one warp read fall in different shared-memory banks
    constexpr int RSTR = L * (4 + RSM) + 4;
    unsigned *rmap = reinterpret_cast<unsigned *>(regions + (size_t)K * RSTR);  // [2][CL]
    double *zs = reinterpret_cast<double *>(rmap + 2 * CL);                     // [2][M][32]
    double2 *zfx = reinterpret_cast<double2 *>(zs + 2 * M * 32);                // [2][32]
    double2 *zcar = zfx + 2 * 32;                                               // [2][32]
    double *stg = reinterpret_cast<double *>(zcar + 2 * 32);                    // [K*L][VPG] (STAGE)
    // chunk region: {V2~, W2~} [L] (double2) | nl [L] | w [L] | scaled source rows [L][RSM]
    auto cd_of = [&](int u) { return reinterpret_cast<double2 *>(regions + (size_t)u * RSTR); };
    const unsigned bar0 = smem_u32(bar), gth0 = smem_u32(gth);
    const unsigned gbar = bar0, ebar = bar0 + 16, cbar = bar0 + 32, fbar = bar0 + 48;

    for (int i = threadIdx.x; i < PART_CTAD; i += blockDim.x) ctad[i] = a.ctad[(size_t)C * PART_CTAD + i];
    if (threadIdx.x < CL) {        // cluster addresses of every CTA's gather buffer and barriers
        rmap[threadIdx.x] = cluster_map(gth0, threadIdx.x);
        rmap[CL + threadIdx.x] = cluster_map(bar0, threadIdx.x);
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2; ++q) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(gbar + 8 * q) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(ebar + 8 * q), "r"(W) : "memory");
            // interface values of a step are complete when both the publish warp
            // (local solution z) and the gather warp ((B_{C-1}, T_{C+1})) arrived
            // (DM: the four tile warps and the gather warp)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(cbar + 8 * q), "r"(DM ? 5 : 2) : "memory");
            // forward pass of a step done (solver warps of the TM variants)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(fbar + 8 * q) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (TM) {            // the publish warp allocates all 512 TMEM columns (one CTA per SM)
        if (w == W) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                         :: "r"(smem_u32(&tm_slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    // ctad / rmap are written by all warps and read below (neighbours) by
    // warps that may run ahead: make the copies visible before any use
    __syncthreads();
    unsigned tm_base = 0;
    if constexpr (TM) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tm_base = tm_slot;
    }

    if (w < W) {
        // ------------------------------------------------ compute warp: chunk c
        if constexpr (TM) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(PART_TM_CREGS));
        const int h = lane / LPC, li = lane % LPC;
        const int u = w * H + h;                     // chunk within the CTA
        const int c = C * K + u;
        const int s0 = c * L;
#pragma unroll 4
        for (int i = lane; i < H * L; i += 32) {     // this warp's H chunk regions
            const int uu = w * H + i / L, row = i % L;
            const double2 *R =
                reinterpret_cast<const double2 *>(a.rowc + ((size_t)(C * K + uu) * L + row) * PART_ROWC);
            const double2 r01 = R[0], r23 = R[1], r67 = R[3];
            double2 *cdu = cd_of(uu);
            cdu[row] = r23;                                              // {V2~, W2~}
            reinterpret_cast<double *>(cdu)[2 * L + row] = r01.y;        // nl
            reinterpret_cast<double *>(cdu)[3 * L + row] = r01.x;        // w
            if constexpr (AFF) {
                const int grow = (C * K + uu) * L + row;
                double *spu = reinterpret_cast<double *>(cdu) + 4 * L + row * RSM;
#pragma unroll
                for (int r = 0; r < RSM; ++r)
                    spu[r] = (grow < a.n && r < a.RS) ? a.spaceT[(size_t)grow * a.RS + r] * r67.y : 0.0;
            }
        }
        __syncwarp();
        const double2 *cd = cd_of(u);
        const double *nl = reinterpret_cast<const double *>(cd) + 2 * L;
        const double *wv = nl + L;
        const double *sp = wv + L;
        // TM: this lane's {nl, w} in its TMEM lane: columns 0..127 nl (rows 0..63), 128..255 w
        const unsigned tm_my = tm_base + ((unsigned)(32 * (w & 3)) << 16) + (unsigned)((w >> 2) * 256);
        if constexpr (TM) {
#pragma unroll 1
            for (int b = 0; b < 32; ++b) {
                unsigned r[8];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const double v = (b < 16) ? nl[b * 4 + e] : wv[(b - 16) * 4 + e];
                    r[2 * e] = (unsigned)__double2loint(v);
                    r[2 * e + 1] = (unsigned)__double2hiint(v);
                }
                tm_st8(tm_my + b * 8, r);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        const double *rowc_u = a.rowc + (size_t)c * L * PART_ROWC;     // this chunk's rows (global)
        const double dbot = rowc_u[(L - 1) * PART_ROWC + 6];            // d_{L-1} (d_0 = 1)
        // staged input of a group: this warp's H chunks, [H*L rows][VPG vectors]
        double *stw = stg + (size_t)w * H * L * VPG;
        // asynchronous copy of group grp's input rows into the staging buffer
        // (pairs of vectors by 16-byte cp.async where aligned and both valid,
        // else 8-byte copies; rows >= n and vectors >= B are zero-filled)
        auto prefetch = [&](long grp) {
            const long gb = grp * VPG;
            const bool al16 = ((a.ld_in & 1) == 0) && ((reinterpret_cast<size_t>(a.in) & 15) == 0);
#pragma unroll 4
            for (int e = lane; e < H * L * VPG / 2; e += 32) {
                const int r = e / (VPG / 2), vp = 2 * (e % (VPG / 2));
                const int grow = (w * H) * L + r + C * K * L;            // row of the vector
                const bool rok = grow < a.n;
                const long v0 = gb + vp;
                const double *src = a.in + (long)(rok ? grow : 0) * a.ld_in;
                const unsigned dst = smem_u32(stw + (size_t)r * VPG + vp);
                if (al16 && rok && v0 + 1 < a.B) {
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src + v0) : "memory");
                } else {
                    const int n0 = (rok && v0 < a.B) ? 8 : 0, n1 = (rok && v0 + 1 < a.B) ? 8 : 0;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;"
                                 :: "r"(dst), "l"(src + (n0 ? v0 : 0)), "r"(n0) : "memory");
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;"
                                 :: "r"(dst + 8), "l"(src + (n1 ? v0 + 1 : 0)), "r"(n1) : "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        // (b_{c-1}, t_{c+1}) of a step from the CTA's (B_{C-1}, T_{C+1}), this
        // chunk's super-spike entries and the local solution z.  Split solve:
        // the first half's z still lacks x_K BR + x_{K+1} BT, applied here.
        const double *zsb = zs;
        auto neighbours = [&](int pp, int vs, double &b, double &t) {
            const double2 bt = coef[pp * 32 + vs];
            const double *zz = zsb + (size_t)pp * M * 32 + vs;
            auto zval = [&](int pos) {
                double v = zz[pos * 32];
                if constexpr (SPLIT && !DM) {
                    if (pos < K) {
                        const double2 fx = zfx[pp * 32 + vs];
                        v = fma(ctad[CTAD_BR + pos], fx.x, fma(ctad[CTAD_BT + pos], fx.y, v));
                    } else if constexpr (SOLVER) {
                        const double2 ym = zcar[pp * 32 + vs];
                        v = fma(ctad[CTAD_PP + pos - K], ym.x, fma(ctad[CTAD_PQ + pos - K], ym.y, v));
                    }
                }
                return v;
            };
            b = (u == 0) ? bt.x : fma(ctad[CTAD_A + 2 * u - 1], bt.x, fma(ctad[CTAD_B + 2 * u - 1], bt.y, zval(2 * u - 1)));
            t = (u == K - 1) ? bt.y
                             : fma(ctad[CTAD_A + 2 * u + 2], bt.x, fma(ctad[CTAD_B + 2 * u + 2], bt.y, zval(2 * u + 2)));
        };
        if (STAGE && a.in && ngrp > 0) prefetch(cid);
        bool synced = false;
        for (long gi = 0; gi < ngrp; ++gi) {
            const long grp = cid + gi * ncl;
            const long gbase = grp * VPG;            // first vector of the group
            const long J0 = gi * a.m;                // global step index of step 0 of this group
            long vv[VPT];
            bool valid[VPT];
#pragma unroll
            for (int t = 0; t < VPT; ++t) {
                vv[t] = gbase + li + t * LPC;
                valid[t] = vv[t] < a.B;
            }
            // the state in the chunk's scaled coordinates x~ = x / d
            double S[VPT][L];
            if (a.in && STAGE) {
                // staged by the previous group (or above): wait, read, and start
                // the next group's copy into the same buffer
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
                const double *st = stw + (size_t)h * L * VPG;
#pragma unroll
                for (int i = 0; i < L; ++i) {
                    const double dinv = (s0 + i < a.n) ? rowc_u[i * PART_ROWC + 7] : 0.0;
#pragma unroll
                    for (int t = 0; t < VPT; ++t) S[t][i] = st[(size_t)i * VPG + li + t * LPC] * dinv;
                }
                __syncwarp();
                if (gi + 1 < ngrp) prefetch(grp + ncl);
            } else if (a.in) {
                // loads issued unconditionally from clamped addresses (no per-row
                // branch, so all rows are in flight together), masked afterwards
                long vc[VPT];
#pragma unroll
                for (int t = 0; t < VPT; ++t) vc[t] = valid[t] ? vv[t] : 0;
#pragma unroll
                for (int i = 0; i < L; ++i) {
                    const int row = (s0 + i < a.n) ? s0 + i : a.n - 1;
                    const double dinv = (s0 + i < a.n) ? rowc_u[i * PART_ROWC + 7] : 0.0;
#pragma unroll
                    for (int t = 0; t < VPT; ++t) {
                        const double v = __ldg(a.in + (long)row * a.ld_in + vc[t]);
                        S[t][i] = valid[t] ? v * dinv : 0.0;
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < L; ++i)
#pragma unroll
                    for (int t = 0; t < VPT; ++t) S[t][i] = 0.0;
            }
            if (!synced) {
                cluster.sync();
                synced = true;
            }
            int q[VPT], src[VPT];
#pragma unroll
            for (int t = 0; t < VPT; ++t) {
                q[t] = valid[t] ? a.q0 + (int)(vv[t] / a.vpi) : a.q0;
                src[t] = (AFF && valid[t]) ? (int)(vv[t] % a.nsrc) : 0;
            }
            double ca[VPT], cc[VPT];     // (b_{c-1}, t_{c+1}) of step j-1: coefficients of V2~, W2~
#pragma unroll
            for (int t = 0; t < VPT; ++t) ca[t] = cc[t] = 0.0;
#ifdef PR_PART_PROBES
            unsigned long long pacc[PART_NPROBE] = {};
            PROBE_T(tl0);
#endif
            for (int j = 1; j <= a.m; ++j) {
                PROBE_T(t0);
                const long J = J0 + j;                   // global step (mbarrier slot / phase)
                double alpha[VPT][AFF ? PART_RSM : 1];
                if constexpr (AFF) {
#pragma unroll
                    for (int t = 0; t < VPT; ++t)
#pragma unroll
                        for (int r = 0; r < PART_RSM; ++r) {
                            double al = 0.0;
                            if (r < a.R && valid[t])
                                al = a.dt * a.amp[(long)src[t] * a.R + r] *
                                     a.time[(long)r * a.nsteps + (long)q[t] * a.m + j - 1];
                            alpha[t][r] = al;
                        }
                }
                // S_j = T_c^{-1}(S_{j-1} + ca V2 + cc W2 + dt f_j) in scaled form:
                // down z_i = x_i + nl_i z_{i-1}, up S_i = w_i z_i + S_{i+1}
                double zp[VPT];
                double gn[VPT];
                PROBE_DECL(t1);
                if constexpr (TM) {
                    // {nl, w} from TMEM, 4 rows per load, the next block in flight
                    // while the current one is used
                    unsigned tb[2][8];
                    double2 qn[2][4];                        // spike coefficients, one block ahead
                    tm_ld8(tm_my, tb[0]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) qn[0][e] = cd[e];
#pragma unroll
                    for (int b = 0; b < L / 4; ++b) {
                        tm_wait8(tb[b & 1]);
                        // after the last nl block: the first w block of the up sweep
                        tm_ld8(b + 1 < L / 4 ? tm_my + (b + 1) * 8 : tm_my + 128 + (L / 4 - 1) * 8, tb[(b + 1) & 1]);
                        if (b + 1 < L / 4) {
#pragma unroll
                            for (int e = 0; e < 4; ++e) qn[(b + 1) & 1][e] = cd[(b + 1) * 4 + e];
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int i = b * 4 + e;
                            const double2 q2 = qn[b & 1][e];
                            const double nli = tm_dbl(tb[b & 1], e);
#pragma unroll
                            for (int t = 0; t < VPT; ++t) {
                                double x = fma(q2.x, ca[t], fma(q2.y, cc[t], S[t][i]));
                                if constexpr (AFF) {
#pragma unroll
                                    for (int r = 0; r < PART_RSM; ++r) x = fma(alpha[t][r], sp[i * RSM + r], x);
                                }
                                zp[t] = (i == 0) ? x : fma(nli, zp[t], x);
                                S[t][i] = zp[t];
                            }
                        }
                    }
                    PROBE_SET(t1);
                    PROBE_ADD(0, t1 - t0);
#pragma unroll
                    for (int b = L / 4 - 1; b >= 0; --b) {
                        constexpr int S0 = (L / 4) & 1;          // buffer of the first w block
                        const int sb = (S0 + (L / 4 - 1 - b)) & 1;
                        tm_wait8(tb[sb]);
                        if (b > 0) tm_ld8(tm_my + 128 + (b - 1) * 8, tb[sb ^ 1]);
#pragma unroll
                        for (int e = 3; e >= 0; --e) {
                            const int i = b * 4 + e;
                            const double wi = tm_dbl(tb[sb], e);
#pragma unroll
                            for (int t = 0; t < VPT; ++t) {
                                gn[t] = (i == L - 1) ? wi * S[t][i] : fma(wi, S[t][i], gn[t]);
                                S[t][i] = gn[t];
                            }
                        }
                    }
                } else {
#pragma unroll
                for (int i = 0; i < L; ++i) {
                    const double2 q2 = cd[i];
                    const double nli = nl[i];
#pragma unroll
                    for (int t = 0; t < VPT; ++t) {
                        double x = fma(q2.x, ca[t], fma(q2.y, cc[t], S[t][i]));
                        if constexpr (AFF) {
#pragma unroll
                            for (int r = 0; r < PART_RSM; ++r) x = fma(alpha[t][r], sp[i * RSM + r], x);
                        }
                        zp[t] = (i == 0) ? x : fma(nli, zp[t], x);
                        S[t][i] = zp[t];
                    }
                }
                PROBE_SET(t1);
                PROBE_ADD(0, t1 - t0);
#pragma unroll
                for (int i = L - 1; i >= 0; --i) {
                    const double wi = wv[i];
#pragma unroll
                    for (int t = 0; t < VPT; ++t) {
                        gn[t] = (i == L - 1) ? wi * S[t][i] : fma(wi, S[t][i], gn[t]);
                        S[t][i] = gn[t];
                    }
                }
                }
                const int p = (int)(J & 1);
                PROBE_T(t2);
                PROBE_ADD(1, t2 - t1);
                if (j >= 2 && !a.noiface) {   // interface values of step j-1 (formed during this sweep)
                    const int pp = (int)((J - 1) & 1);
                    mbar_wait(cbar + 8 * pp, (unsigned)(((J - 2) >> 1) & 1));
#pragma unroll
                    for (int t = 0; t < VPT; ++t) neighbours(pp, li + t * LPC, ca[t], cc[t]);
                }
                PROBE_T(t3);
                PROBE_ADD(2, t3 - t2);
                {                          // physical chunk ends of g_j = S_j + ca V2 + cc W2
                    const double2 q0 = cd[0], q1 = cd[L - 1];
#pragma unroll
                    for (int t = 0; t < VPT; ++t)
                        rawE[(p * K + u) * 32 + li + t * LPC] =
                            make_double2(fma(q0.x, ca[t], fma(q0.y, cc[t], S[t][0])),
                                         dbot * fma(q1.x, ca[t], fma(q1.y, cc[t], S[t][L - 1])));
                }
                __syncwarp();
                if (lane == 0 && !a.noiface) mbar_arrive(ebar + 8 * p);
                PROBE_T(t4);
                PROBE_ADD(3, t4 - t3);
            }
#ifdef PR_PART_PROBES
            PROBE_T(tl1);
            PROBE_ADD(11, tl1 - tl0);
            if (lane == 0 && w == 0 && a.prof)
                for (int k = 0; k < 4; ++k) atomicAdd(a.prof + k, pacc[k]);
            if (lane == 0 && w == 0 && a.prof) atomicAdd(a.prof + 11, pacc[11]);
            if (lane == 0 && w == 0 && a.prof) atomicAdd(a.prof + 10, (unsigned long long)a.m);
#endif
            // x_m = S_m + ca V2 + cc W2 + b_m V + t_m W, branch-free per row (the
            // row data loads are uniform over the chunk's lanes), masked stores
            const long Jm = J0 + a.m;
            const int pm = (int)(Jm & 1);
            double ex[VPT], ey[VPT];                     // (b_m, t_m) of the neighbours
#pragma unroll
            for (int t = 0; t < VPT; ++t) ex[t] = ey[t] = 0.0;
            if (!a.noiface) {
                mbar_wait(cbar + 8 * pm, (unsigned)(((Jm - 1) >> 1) & 1));
#pragma unroll
                for (int t = 0; t < VPT; ++t) neighbours(pm, li + t * LPC, ex[t], ey[t]);
            }
            // the stored offsets are read in blocks of EB rows from clamped
            // addresses BEFORE the block's stores (off may alias out, so loads
            // interleaved with the stores would be serialised behind them: one
            // HBM latency per row)
            constexpr int EB = 16;
            long vc[VPT];
#pragma unroll
            for (int t = 0; t < VPT; ++t) vc[t] = valid[t] ? vv[t] : 0;
#pragma unroll
            for (int i0 = 0; i0 < L; i0 += EB) {
                double ofs[VPT][EB];
#pragma unroll
                for (int r = 0; r < EB; ++r)
#pragma unroll
                    for (int t = 0; t < VPT; ++t) ofs[t][r] = 0.0;
                if (a.off) {
#pragma unroll
                    for (int r = 0; r < EB; ++r) {
                        const int row = (s0 + i0 + r < a.n) ? s0 + i0 + r : a.n - 1;
#pragma unroll
                        for (int t = 0; t < VPT; ++t) ofs[t][r] = a.off[(long)row * a.ld_off + vc[t]];
                    }
                }
#pragma unroll
                for (int r = 0; r < EB; ++r) {
                    const int i = i0 + r;
                    const double2 q2 = cd[i];
                    const double2 *R = reinterpret_cast<const double2 *>(rowc_u + i * PART_ROWC);
                    const double2 VW = __ldg(R + 2), dd = __ldg(R + 3);
                    const bool rok = s0 + i < a.n;
#pragma unroll
                    for (int t = 0; t < VPT; ++t) {
                        double x = fma(q2.x, ca[t], fma(q2.y, cc[t], S[t][i]));
                        x = fma(VW.x, ex[t], fma(VW.y, ey[t], dd.x * x));
                        if (rok && valid[t]) a.out[(long)(s0 + i) * a.ld_out + vv[t]] = x + ofs[t][r];
                    }
                }
            }
        }
        if (!synced) cluster.sync();
    } else {
        // ------------------------------------------------ interface warps
        // lane = (part hi, vector vl); with HI = 2 the two half-warps split the
        // cluster sends, the solve halves and the gather dot products
        if constexpr (TM) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(PART_TM_IREGS));
        const int hi = lane / VPG, vl = lane % VPG;
#ifdef PR_PART_PROBES
        unsigned long long pacc[PART_NPROBE] = {};
#endif
        cluster.sync();
        constexpr int CLH = CL / HI;                                     // CTAs per lane part
        // step j's values from every super-chunk -> (B_{C-1}, T_{C+1}) of step j
        auto gather = [&](long j) {
            const int p = (int)(j & 1);
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             :: "r"(gbar + 8 * p), "r"((unsigned)(CL * VPG * sizeof(double2))) : "memory");
            PROBE_T(g0);
            mbar_wait_idle(gbar + 8 * p, (unsigned)(((j - 1) >> 1) & 1), a.idle_ns);
            PROBE_T(g1);
            PROBE_ADD(8, g1 - g0);
            const double2 *Gt = gth + (size_t)p * CL * 32 + vl;
            // the two halves of the CTA list are summed separately and then
            // added, for HI = 1 and HI = 2 alike: the result does not depend on
            // the lane split the group size selects (bit-identical shards)
            auto half = [&](int hh, double &Bh, double &Th) {
                double b0 = 0.0, b1 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
                for (int rr = 0; rr < CL / 2; ++rr) {
                    const int r = hh * (CL / 2) + rr;
                    const double2 e = Gt[r * 32];
                    b0 = fma(ctad[CTAD_GB + 2 * r], e.x, b0);
                    b1 = fma(ctad[CTAD_GB + 2 * r + 1], e.y, b1);
                    t0 = fma(ctad[CTAD_GT + 2 * r], e.x, t0);
                    t1 = fma(ctad[CTAD_GT + 2 * r + 1], e.y, t1);
                }
                Bh = b0 + b1;
                Th = t0 + t1;
            };
            double Bx, Tx;
            if constexpr (HI == 2) {
                half(hi, Bx, Tx);
                Bx += __shfl_xor_sync(0xffffffffu, Bx, 16);
                Tx += __shfl_xor_sync(0xffffffffu, Tx, 16);
            } else {
                double B1, T1;
                half(0, Bx, Tx);
                half(1, B1, T1);
                Bx += B1;
                Tx += T1;
            }
            if (hi == 0) coef[p * 32 + vl] = make_double2(Bx, Tx);
            __syncwarp();
            if (lane == 0) mbar_arrive(cbar + 8 * p);
            PROBE_T(g2);
            PROBE_ADD(9, g2 - g1);
        };
        // chunk end values of step j -> (T_C, B_C) to every CTA, then the local
        // solve z = M_C^{-1} g_C (off the exchange's critical path)
        // Roles: SEND (super-values formed and sent), FWD / BWD (the two passes of
        // the band solve).  Without solver warps the publish warp does all three;
        // the TM variants (SOLVER) run them on warps W, W + 2 and W + 3, one per SM
        // sub-partition, so no sub-partition's compute warps lose much more FP64
        // issue than the others (the step ends with the slowest compute warp)
        auto publish = [&](long j, auto send_c, auto fwd_c, auto bwd_c) {
            constexpr bool SEND = decltype(send_c)::value, FWD = decltype(fwd_c)::value, BWD = decltype(bwd_c)::value;
            const int p = (int)(j & 1);
            const unsigned ph = (unsigned)(((j - 1) >> 1) & 1);
            PROBE_T(p0);
            if constexpr (SEND || FWD) mbar_wait_idle(ebar + 8 * p, ph, a.idle_ns);
            else mbar_wait_idle(fbar + 8 * p, ph, a.idle_ns);
            PROBE_T(p1);
            if (SEND) PROBE_ADD(4, p1 - p0);
            const double2 *rE = rawE + (size_t)p * K * 32 + vl;
            const unsigned off = (unsigned)(((p * CL + C) * 32 + vl) * sizeof(double2));
            if constexpr (SPLIT) {
                PROBE_DECL(p2);
                PROBE_SET(p2);
                if constexpr (SEND) {
                    // (T, B) partial sums of half 0 and half 1, added in that order
                    double T0h, T1h, B0h, B1h;
                    if constexpr (HI == 2) {
                        double Tm, Bm;
                        half_dots<K>(hi, rE, ctad, Tm, Bm);
                        const double To = __shfl_xor_sync(0xffffffffu, Tm, 16);
                        const double Bo = __shfl_xor_sync(0xffffffffu, Bm, 16);
                        T0h = hi ? To : Tm;
                        T1h = hi ? Tm : To;
                        B0h = hi ? Bo : Bm;
                        B1h = hi ? Bm : Bo;
                    } else {
                        half_dots<K>(0, rE, ctad, T0h, B0h);
                        half_dots<K>(1, rE, ctad, T1h, B1h);
                    }
                    const double Tv = T0h + T1h, Bv = B0h + B1h;
#pragma unroll
                    for (int rr = 0; rr < CLH; ++rr) {
                        const int r = hi * CLH + rr;
                        st_async_v2(rmap[r] + off, Tv, Bv, rmap[CL + r] + 8 * p);
                    }
                    PROBE_SET(p2);
                    PROBE_ADD(5, p2 - p1);
                }
                // split solve: all lanes write the common result slot vl
                double *zc = zs + (size_t)p * M * 32 + vl;
                double2 *zfix = zfx + p * 32 + vl;
                if constexpr (SOLVER) {
                    static_assert(!SOLVER || HI == 2, "solver warps: one half per half-warp");
                    if constexpr (FWD) {
                        double y2m, y1m;
                        half_forward<K>(hi, rE, ctad, zc, y2m, y1m);
                        if (hi == 0) zcar[p * 32 + vl] = make_double2(y2m, y1m);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(fbar + 8 * p);
                        PROBE_T(p3);
                        PROBE_ADD(6, p3 - p2);
                    }
                    if constexpr (BWD) {
                        // both halves from a zero carried state; the second half's
                        // carried-pair correction is the consumer's (PP / PQ), except
                        // for the two values the first half's consumers need
                        double x0m, x1m;
                        half_backward<K, true>(hi, ctad, zc, x0m, x1m, false, 0.0, 0.0);
                        if (hi == 1) {
                            const double2 ym = zcar[p * 32 + vl];
                            x0m = fma(ctad[CTAD_PP], ym.x, fma(ctad[CTAD_PQ], ym.y, x0m));
                            x1m = fma(ctad[CTAD_PP + 1], ym.x, fma(ctad[CTAD_PQ + 1], ym.y, x1m));
                            *zfix = make_double2(x0m, x1m);
                        }
                        __syncwarp();
                        PROBE_T(p4);
                        PROBE_ADD(7, p4 - p1);
                    }
                } else if constexpr (FWD && BWD) {
                    double y2c, y1c;                      // half 0's carried pair
                    if constexpr (HI == 2) {
                        double y2m, y1m;
                        half_forward<K>(hi, rE, ctad, zc, y2m, y1m);
                        y2c = __shfl_xor_sync(0xffffffffu, y2m, 16);
                        y1c = __shfl_xor_sync(0xffffffffu, y1m, 16);
                    } else {
                        double y2x, y1x;
                        half_forward<K>(0, rE, ctad, zc, y2c, y1c);
                        half_forward<K>(1, rE, ctad, zc, y2x, y1x);
                    }
                    PROBE_T(p3);
                    PROBE_ADD(6, p3 - p2);
                    if constexpr (HI == 2) {
                        double x0m, x1m;
                        half_backward<K>(hi, ctad, zc, x0m, x1m, hi == 1, y2c, y1c);
                        if (hi == 1) *zfix = make_double2(x0m, x1m);
                    } else {
                        double xk, xk1, x0x, x1x;
                        half_backward<K>(1, ctad, zc, xk, xk1, true, y2c, y1c);
                        half_backward<K>(0, ctad, zc, x0x, x1x, false, 0.0, 0.0);
                        *zfix = make_double2(xk, xk1);
                    }
                    __syncwarp();
                    PROBE_T(p4);
                    PROBE_ADD(7, p4 - p3);
                }
            } else {
                static_assert(SPLIT || !SOLVER, "the unsplit solve runs on the publish warp");
                double *zl = zs + (size_t)p * M * 32 + vl + VPG * hi;
                // forward elimination y = L^{-1} g (stored), and (T_C, B_C) from the
                // two stored rows of M_C^{-1} applied to g (independent FMAs)
                double T0, T1, B0, B1;
                band_forward<K>(rE, ctad, zl, T0, T1, B0, B1);
                const double Tv = T0 + T1, Bv = B0 + B1;
#pragma unroll
                for (int rr = 0; rr < CLH; ++rr) {
                    const int r = hi * CLH + rr;
                    st_async_v2(rmap[r] + off, Tv, Bv, rmap[CL + r] + 8 * p);
                }
                // back substitution with the pre-scaled factors {.., 1/u, u1/u, u2/u}
                band_backward<M>(ctad, zl);
                __syncwarp();
            }
        };
        // DM: interface warp q = w - W forms rows tile(q) of z = M_C^{-1} g with
        // mma.m8n8k4.f64 (A: 8 rows of the inverse, kept in registers; B: the raw
        // ends of 8 vectors, from shared memory), two column tiles (16 vectors),
        // the k range in two halves (four independent accumulator chains), summed
        // in fixed order.  Tile 0 holds rows {0, M-1, 1..6}: the publish warp owns
        // T_C and B_C and sends them right after its product.
        const int gq = lane >> 2, tq = lane & 3;
        const int dm_q = w - W;
        const int dm_row = (dm_q == 0) ? (gq == 0 ? 0 : (gq == 1 ? M - 1 : gq - 1)) : 7 + 8 * (dm_q - 1) + gq;
        constexpr int DKS = DM ? M / 4 : 1, DKH = DM ? M / 8 : 1;   // k steps (of 4), per accumulator half
        double afr[DKS] = {};
        if constexpr (DM) {
            const double *MI = a.ctad + (size_t)CL * PART_CTAD + (size_t)C * PART_MINV + (size_t)dm_row * M;
#pragma unroll
            for (int ks = 0; ks < DKS; ++ks) afr[ks] = __ldg(MI + 4 * ks + tq);
        }
        auto dm_tile = [&](auto j) {   // generic: instantiated for the DM variants only
            const int p = (int)(j & 1);
            const unsigned ph = (unsigned)(((j - 1) >> 1) & 1);
            PROBE_T(p0);
            mbar_wait_idle(ebar + 8 * p, ph, a.idle_ns);
            PROBE_T(p1);
            if (dm_q == 0) PROBE_ADD(4, p1 - p0);
            const double *gE = reinterpret_cast<const double *>(rawE + (size_t)p * K * 32);
            double bfr[DKS][2];
#pragma unroll
            for (int ks = 0; ks < DKS; ++ks)
#pragma unroll
                for (int ct = 0; ct < 2; ++ct)
                    bfr[ks][ct] = gE[(size_t)((2 * ks + (tq >> 1)) * 32 + ct * 8 + gq) * 2 + (tq & 1)];
            double acc[2][2][2];
#pragma unroll
            for (int ct = 0; ct < 2; ++ct)
#pragma unroll
                for (int kh = 0; kh < 2; ++kh) acc[ct][kh][0] = acc[ct][kh][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < DKS; ++ks)
#pragma unroll
                for (int ct = 0; ct < 2; ++ct)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(acc[ct][ks / DKH][0]), "+d"(acc[ct][ks / DKH][1])
                                 : "d"(afr[ks]), "d"(bfr[ks][ct]));
            double2 *zrow = reinterpret_cast<double2 *>(zs + ((size_t)p * M + dm_row) * 32);
#pragma unroll
            for (int ct = 0; ct < 2; ++ct)
                zrow[ct * 4 + tq] = make_double2(acc[ct][0][0] + acc[ct][1][0], acc[ct][0][1] + acc[ct][1][1]);
            __syncwarp();
            if (dm_q == 0) {           // (T_C, B_C) = rows 0 and M-1 to every CTA of the cluster
                const double Tv = zs[((size_t)p * M) * 32 + vl], Bv = zs[((size_t)p * M + M - 1) * 32 + vl];
                const unsigned off = (unsigned)(((p * CL + C) * 32 + vl) * sizeof(double2));
#pragma unroll
                for (int rr = 0; rr < CLH; ++rr) {
                    const int r = hi * CLH + rr;
                    st_async_v2(rmap[r] + off, Tv, Bv, rmap[CL + r] + 8 * p);
                }
            }
            if (lane == 0) mbar_arrive(cbar + 8 * p);
            PROBE_T(p2);
            if (dm_q == 0) PROBE_ADD(5, p2 - p1);
            if (dm_q == 2) PROBE_ADD(6, p2 - p1);
        };
        // global step index over this cluster's groups (mbarrier slots and phases)
        const long nJ = ngrp * (long)a.m;
        if (a.noiface) {
        } else if (DM) {
            if constexpr (DM) {
                for (long j = 1; j <= nJ; ++j) {
                    dm_tile(j);
                    if (w == W + 1) gather(j);
                }
            }
        } else if (w == W) {
            for (long j = 1; j <= nJ; ++j) {
                if constexpr (SOLVER) {
                    publish(j, std::true_type{}, std::false_type{}, std::false_type{});
                } else {
                    publish(j, std::true_type{}, std::true_type{}, std::true_type{});
                    if (lane == 0) mbar_arrive(cbar + 8 * (int)(j & 1));
                }
            }
        } else if (w == W + 1) {
            for (long j = 1; j <= nJ; ++j) gather(j);
        } else if (SOLVER && w == W + 2) {
            for (long j = 1; j <= nJ; ++j) publish(j, std::false_type{}, std::true_type{}, std::false_type{});
        } else if (SOLVER && w == W + 3) {
            for (long j = 1; j <= nJ; ++j) {
                publish(j, std::false_type{}, std::false_type{}, std::true_type{});
                if (lane == 0) mbar_arrive(cbar + 8 * (int)(j & 1));
            }
        }
#ifdef PR_PART_PROBES
        if (lane == 0 && a.prof)
            for (int k = 4; k < 10; ++k)
                if (pacc[k]) atomicAdd(a.prof + k, pacc[k]);
#endif
    }
    if constexpr (TM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster.sync();                // no CTA leaves while cluster peers may still target it
    if constexpr (TM) {
        if (w == W) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm_base) : "memory");
    }
}

// ---------------------------------------------------------------- driver
bool part_config(int n, int &P, int &L, int &CL, int &K)
{
    // chunks of L = 32 rows up to n = 512 (one warp per chunk, up to 16 CTAs),
    // else 64 rows in 16 CTAs of K = 1..16 chunks.  PR_PART_VPT2=1 selects for
    // n > 8192 32-row chunks with two vectors per lane instead (K = 32 chunks
    // per CTA: half the coefficient loads per DOF-step, but a 64-unknown local
    // interface solve per step, measured slower on C4).  P (a power of two)
    // chunks cover P*L >= n rows, the rest identity padding.
    if (n < 64 || n > PART_CLMAX * 32 * 32) return false;
    L = (n <= 512 || (n > 8192 && flags().part_vpt2)) ? 32 : 64;
    const int need = (n + L - 1) / L;
    P = 2;
    while (P < need) P *= 2;
    CL = P < PART_CLMAX ? P : PART_CLMAX;
    K = P / CL;
    return K <= PART_KMAX;
}

cudaError_t launch_part_setup(int n, int P, int L, int CL, int K, const double *subA, const double *supA,
                              const double *rsA, const double *diagA, double dt, int transpose, double *rowc,
                              double *ctad, double *ends, int *bad, int *noscale, cudaStream_t s)
{
    note_launch();
    k_part_setup<<<(P + 63) / 64, 64, 0, s>>>(n, P, L, subA, supA, rsA, diagA, dt, transpose, rowc, ends, bad,
                                              noscale);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    note_launch();
    k_part_iface<<<1, 32, 0, s>>>(CL, K, ends, ctad, bad);
    return cudaGetLastError();
}

template <int CL, int W, int H, int L, int VPT, bool AFF, bool TM = false, bool DMV = true>
static cudaError_t part_launch(const PartArgs &a, long groups, cudaStream_t s)
{
    constexpr size_t smem = part_smem_t<CL, W, H, L, VPT, AFF>();
    static_assert(smem <= 227 * 1024, "partitioned stepper shared memory");
    // function attributes are per device: set once for each device this
    // process launches on (bit d of the mask)
    static std::atomic<unsigned long long> attr_mask{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ULL << (dev & 63);
    if (!(attr_mask.load(std::memory_order_acquire) & bit)) {
        cudaError_t e = cudaFuncSetAttribute(k_part_step<CL, W, H, L, VPT, AFF, TM, DMV>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess && CL > 8)
            e = cudaFuncSetAttribute(k_part_step<CL, W, H, L, VPT, AFF, TM, DMV>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr_mask.fetch_or(bit, std::memory_order_release);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(groups * CL));
    cfg.blockDim = dim3(32 * (W + part_ni<TM>()));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // persistent clusters: as many as are co-resident (queried once per device),
    // each looping over vector groups; clusters never wait on one another, so
    // fewer resident clusters (another kernel sharing the GPU) only serialise
    static std::atomic<int> max_cl[64];
    int ncl = max_cl[dev & 63].load(std::memory_order_acquire);
    if (ncl == 0) {
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, (void *)k_part_step<CL, W, H, L, VPT, AFF, TM, DMV>, &cfg) != cudaSuccess ||
            nc < 1) {
            (void)cudaGetLastError();
            nc = -1;                   // unknown: one cluster per group
        }
        max_cl[dev & 63].store(nc, std::memory_order_release);
        ncl = nc;
    }
    if (flags().part_nopersist) ncl = -1;
    const long grid_cl = (ncl > 0 && ncl < groups) ? ncl : groups;
    cfg.gridDim = dim3((unsigned)(grid_cl * CL));
    PartArgs ag = a;
    ag.groups = groups;
    if (flags().part_prof) {
        int nc = -1;
        cudaError_t eo = cudaOccupancyMaxActiveClusters(&nc, (void *)k_part_step<CL, W, H, L, VPT, AFF, TM, DMV>, &cfg);
        fprintf(stderr, "part: max active clusters %d (%s), smem %zu B, groups %ld\n", nc,
                eo == cudaSuccess ? "ok" : cudaGetErrorString(eo), smem, groups);
        (void)cudaGetLastError();
    }
    note_launch();
#ifdef PR_PART_PROBES
    if (flags().part_prof) {
        PartArgs b = ag;
        cudaMalloc(&b.prof, PART_NPROBE * sizeof(unsigned long long));
        cudaMemsetAsync(b.prof, 0, PART_NPROBE * sizeof(unsigned long long), s);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_part_step<CL, W, H, L, VPT, AFF, TM, DMV>, b);
        unsigned long long h[PART_NPROBE];
        cudaMemcpyAsync(h, b.prof, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        cudaFree(b.prof);
        const double st = h[10] ? (double)h[10] : 1.0;   // steps x CTAs (compute warp 0)
        fprintf(stderr,
                "part probes (cycles per CTA-step): down %.0f up %.0f wait-iface %.0f ends %.0f | "
                "publish: wait %.0f dots+send %.0f fwd %.0f bwd %.0f | gather: wait %.0f dot %.0f | loop/step %.0f\n",
                h[0] / st, h[1] / st, h[2] / st, h[3] / st, h[4] / st, h[5] / st, h[6] / st, h[7] / st,
                h[8] / st, h[9] / st, h[11] / st);
        return e;
    }
#endif
    return cudaLaunchKernelEx(&cfg, k_part_step<CL, W, H, L, VPT, AFF, TM, DMV>, ag);
}

template <int CL, int W, int H, int L, int VPT = 1>
static cudaError_t part_launch_aff(const PartArgs &a, long B, cudaStream_t s)
{
    constexpr long VPG = (32 / H) * VPT;
    const long groups = (B + VPG - 1) / VPG;
    // TM: {nl, w} in tensor memory (64-row chunks, up to 8 compute warps);
    // PR_PART_NOTMEM=1 keeps every coefficient in shared memory
    if constexpr (L == 64 && VPT == 1 && W == 8) {
        if (!flags().part_notmem) {
            // PR_PART_NODM=1: the banded interface solve on the solver warps instead
            // of the tensor-core product (K = 16 chunks per CTA only)
            if constexpr (W * H == 16) {
                if (flags().part_nodm)
                    return a.R > 0 ? part_launch<CL, W, H, L, VPT, true, true, false>(a, groups, s)
                                   : part_launch<CL, W, H, L, VPT, false, true, false>(a, groups, s);
            }
            return a.R > 0 ? part_launch<CL, W, H, L, VPT, true, true>(a, groups, s)
                           : part_launch<CL, W, H, L, VPT, false, true>(a, groups, s);
        }
    }
    return a.R > 0 ? part_launch<CL, W, H, L, VPT, true>(a, groups, s)
                   : part_launch<CL, W, H, L, VPT, false>(a, groups, s);
}

bool part_preferred(const Op &op, long B, int m)
{
    // measured on B200 (C1, C2 shapes, B = 32 .. 20480): the partitioned stepper
    // beats the fused one at every batch size it supports
    (void)B;
    if (op.part_P == 0 || m < 1 || flags().no_part) return false;
    return true;
}

cudaError_t launch_stepper_part(const Op &op, const StepArgs &sa, int transpose, cudaStream_t s)
{
    PartArgs a{};
    a.n = sa.n; a.m = sa.m; a.B = sa.B;
    a.rowc = transpose ? op.part_rowc_tr : op.part_rowc_fw;
    a.ctad = transpose ? op.part_ctad_tr : op.part_ctad_fw;
    a.in = sa.in; a.ld_in = sa.ld_in; a.out = sa.out; a.ld_out = sa.ld_out;
    a.off = sa.off; a.ld_off = sa.ld_off;
    a.R = sa.R;
    a.RS = sa.R > 0 ? stepper_rs(sa.R) : 0;
    a.spaceT = sa.spaceT; a.time = sa.time; a.amp = sa.amp;
    a.nsteps = sa.nsteps; a.nsrc = sa.nsrc; a.q0 = sa.q0; a.vpi = sa.vpi; a.dt = sa.dt;
    a.idle_ns = flags().part_idle_ns >= 0 ? (unsigned)flags().part_idle_ns : PART_IDLE_NS;
    a.noiface = flags().part_noiface;
    if (sa.B == 0) return cudaSuccess;
    const int K = op.part_K;
    // two chunks per warp (16 vectors per warp) when that spreads a small batch
    // over more SMs, or when K chunks would need more than 8 compute warps
    int H = 1;
    if (K >= 2) {
        const long clusters32 = (sa.B + 31) / 32;
        if (K > 8 || clusters32 * op.part_CL * 2 <= num_sms()) H = 2;
        if (const int f = flags().part_h) {
            if ((f == 1 && K <= 8) || f == 2) H = f;
        }
    }
    const bool prof = profiling();
    if (prof) stepper_timed_begin(s);
    cudaError_t e = cudaErrorInvalidValue;
    if (op.part_L == 32 && K == 1) {
        switch (op.part_CL) {
        case 2: e = part_launch_aff<2, 1, 1, 32>(a, sa.B, s); break;
        case 4: e = part_launch_aff<4, 1, 1, 32>(a, sa.B, s); break;
        case 8: e = part_launch_aff<8, 1, 1, 32>(a, sa.B, s); break;
        case 16: e = part_launch_aff<16, 1, 1, 32>(a, sa.B, s); break;
        }
    } else if (op.part_L == 32) {
        // n > 8192: 32-row chunks, 4 chunks per warp (8 lanes each), two
        // vectors per lane: groups of 16 vectors
        if (op.part_CL == 16 && K == 32) e = part_launch_aff<16, 8, 4, 32, 2>(a, sa.B, s);
    } else if (op.part_CL == 16 && H == 1) {
        switch (K) {
        case 1: e = part_launch_aff<16, 1, 1, 64>(a, sa.B, s); break;
        case 2: e = part_launch_aff<16, 2, 1, 64>(a, sa.B, s); break;
        case 4: e = part_launch_aff<16, 4, 1, 64>(a, sa.B, s); break;
        case 8: e = part_launch_aff<16, 8, 1, 64>(a, sa.B, s); break;
        }
    } else if (op.part_CL == 16 && H == 2) {
        switch (K) {
        case 2: e = part_launch_aff<16, 1, 2, 64>(a, sa.B, s); break;
        case 4: e = part_launch_aff<16, 2, 2, 64>(a, sa.B, s); break;
        case 8: e = part_launch_aff<16, 4, 2, 64>(a, sa.B, s); break;
        case 16: e = part_launch_aff<16, 8, 2, 64>(a, sa.B, s); break;
        }
    }
    // algorithmic FP64 flops per DOF-step: Thomas with precomputed factors,
    // y = w r - ga y' (3) and x = y - cp x' (2), plus 2R for an R-term source
    // (bench.py roofline)
    if (prof) {
        const double dof = (double)sa.n * (double)sa.B * (double)sa.m;
        stepper_timed_end(s, dof, (5.0 + 2.0 * a.R) * dof);
    }
    return e;
}

}  // namespace pr
