// k_part.cu -- K1P: partitioned 1D backward-Euler stepper for small batches.
//
// The fused stepper (k_tridiag.cu) runs one vector per thread, so a batch of
// B vectors keeps only B/32 warps busy; with few vectors (Parareal fine solves
// of C1/C2: 16-64 vectors) each warp's row recurrence is latency-bound.  Here
// every vector's n rows are split into P chunks, one chunk per CTA of a
// P-CTA thread-block cluster, and the chunk state stays in shared memory for
// all m steps.  One step (I + dt A) x = r by the partition method:
//   g_c  = T_c^{-1} r_c                         (local LU, row-sum pivots)
//   x_c  = g_c + V_c b_{c-1} + W_c t_{c+1}      (spikes V_c = T_c^{-1}(-a e_1),
//                                                W_c = T_c^{-1}(-c e_L), fixed)
//   (t_c, b_c) = first / last unknown of chunk c, solved from the 2P x 2P
//   interface system  z_i - V b - W t = g_i,  a banded M-matrix factored once
//   with row-sum (GTH-type) elimination: its row sums 1 - V - W = T_c^{-1} s_c
//   are computed directly, so the pivots keep O(u) relative accuracy whatever
//   dt/h^2 (reading R-ACC).
// Per step a CTA sweeps its chunk down (forward elimination, after applying the
// previous step's spike correction and the source) and up (back substitution)
// in shared memory, publishes its two end values to the cluster leader through
// distributed shared memory, the leader solves the interface system (one lane
// per vector) and scatters (b_{c-1}, t_{c+1}) back.  Two cluster barriers per
// step; HBM is touched only to read the input and write the result.
#include <cooperative_groups.h>

#include "pr_internal.cuh"

namespace cg = cooperative_groups;

namespace pr {

// ------------------------------------------------------------------ setup
// One thread per chunk c (rows s0..e0-1): local LU of T_c in row-sum form and
// the three local solves V_c, W_c, rho_c.  rowc row i: {w_i, -ga_i, -cp_i, V_i, W_i};
// ends[c] = {rho_top, rho_bot, V_top, V_bot, W_top, W_bot, 0, 0}.
__global__ void k_part_setup(int n, int P, int L, const double *subA, const double *supA,
                             const double *rsA, const double *diagA, double dt, int transpose,
                             double *rowc, double *ends, int *bad)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= P) return;
    const int s0 = c * L, e0 = min(n, s0 + L);
    if (s0 >= e0 || e0 - s0 > PART_LMAX) { atomicExch(bad, 1); return; }
    auto a_of = [&](int i) -> double {              // (I + dt A)[i, i-1] (or of the transpose)
        if (i <= 0) return 0.0;
        return dt * (transpose ? supA[i - 1] : subA[i]);
    };
    auto c_of = [&](int i) -> double {              // (I + dt A)[i, i+1]
        if (i >= n - 1) return 0.0;
        return dt * (transpose ? subA[i + 1] : supA[i]);
    };
    auto s_of = [&](int i) -> double {              // row sums of I + dt A
        if (rsA) return 1.0 + dt * rsA[i];
        return a_of(i) + (1.0 + dt * diagA[i]) + c_of(i);
    };
    // local LU: T_c drops a_{s0} and c_{e0-1}; its row sums are s_i minus the
    // dropped (non-positive) entries, so they stay exact sums of the stencil
    double r = 0.0, den = 1.0;
    for (int i = s0; i < e0; ++i) {
        const double ai = (i == s0) ? 0.0 : a_of(i);
        const double ci = (i == e0 - 1) ? 0.0 : c_of(i);
        double sl = s_of(i);
        if (i == s0) sl -= a_of(i);
        if (i == e0 - 1) sl -= c_of(i);
        r = (i == s0) ? sl : sl - ai * (r / den);
        den = r - ci;
        if (!(den > 0.0) || !isfinite(den)) atomicExch(bad, 1);
        const double w = 1.0 / den;
        double *R = rowc + (size_t)i * 5;
        R[0] = w;
        R[1] = -(w * ai);
        R[2] = -(w * ci);
    }
    // T_c x = rhs: forward y_i = w_i rhs_i - ga_i y_{i-1}, back x_i = y_i - cp_i x_{i+1}
    double y[PART_LMAX];
    double *E = ends + (size_t)c * 8;
    for (int which = 0; which < 3; ++which) {       // 0: V, 1: W, 2: rho
        double yp = 0.0;
        for (int i = s0; i < e0; ++i) {
            double rhs = 0.0;
            if (which == 0 && i == s0) rhs = -a_of(s0);
            if (which == 1 && i == e0 - 1) rhs = -c_of(e0 - 1);
            if (which == 2) rhs = s_of(i);
            const double *R = rowc + (size_t)i * 5;
            yp = fma(R[1], yp, R[0] * rhs);
            y[i - s0] = yp;
        }
        double xn = 0.0;
        for (int i = e0 - 1; i >= s0; --i) {
            double *R = rowc + (size_t)i * 5;
            const double x = fma(R[2], xn, y[i - s0]);
            if (which < 2) R[3 + which] = x;
            if (i == s0) E[which == 0 ? 2 : which == 1 ? 4 : 0] = x;
            if (i == e0 - 1) E[which == 0 ? 3 : which == 1 ? 5 : 1] = x;
            xn = x;
        }
    }
    E[6] = E[7] = 0.0;
}

// Interface system of 2P unknowns z = (t_0, b_0, ..., t_{P-1}, b_{P-1}):
//   row 2c   : t_c - V_c[top] b_{c-1} - W_c[top] t_{c+1} = g_c[top]
//   row 2c+1 : b_c - V_c[bot] b_{c-1} - W_c[bot] t_{c+1} = g_c[bot]
// Banded M-matrix (offsets -2..+2), factored without pivoting; off-diagonals
// are updated with same-sign products, row sums with positive terms, and each
// pivot is (row sum) - (remaining off-diagonals): no cancellation.
// fac (per row i, 5 doubles): {l_{i,i-2}, l_{i,i-1}, 1/u_ii, u_{i,i+1}, u_{i,i+2}}.
__global__ void k_part_reduced(int P, const double *ends, double *fac, int *bad)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int M = 2 * P;
    double A[64][5];          // band: A[i][d], column i + d - 2
    double rs[64];
    for (int i = 0; i < M; ++i) {
        for (int d = 0; d < 5; ++d) A[i][d] = 0.0;
        const int c = i / 2;
        const bool top = (i % 2 == 0);
        const double *E = ends + (size_t)c * 8;
        const double V = top ? E[2] : E[3];
        const double W = top ? E[4] : E[5];
        A[i][2] = 1.0;
        // b_{c-1} is column 2c-1: offset (2c-1) - i + 2
        if (c > 0) A[i][(2 * c - 1) - i + 2] = -V;
        // t_{c+1} is column 2c+2
        if (c < P - 1) A[i][(2 * c + 2) - i + 2] = -W;
        rs[i] = top ? E[0] : E[1];
    }
    for (int i = 0; i < M; ++i) {
        double l2 = 0.0, l1 = 0.0;
        for (int dj = 2; dj >= 1; --dj) {              // eliminate columns i-2, i-1
            const int j = i - dj;
            if (j < 0) continue;
            const double aij = A[i][2 - dj];
            if (aij == 0.0) continue;
            const double mult = aij * fac[(size_t)j * 5 + 2];     // a_ij / u_jj  (<= 0)
            // row_i -= mult * row_j (columns > j): u_{j,j+1}, u_{j,j+2}
            for (int e = 1; e <= 2; ++e) {
                const int col = j + e;
                const int di = col - i + 2;
                if (di >= 0 && di < 5) A[i][di] -= mult * fac[(size_t)j * 5 + 2 + e];
            }
            rs[i] -= mult * rs[j];
            if (dj == 2) l2 = mult; else l1 = mult;
            A[i][2 - dj] = 0.0;
        }
        double off = 0.0;
        for (int e = 1; e <= 2; ++e)
            if (i + e < M) off += A[i][2 + e];
        const double piv = rs[i] - off;               // accurate diagonal
        if (!(piv > 0.0) || !isfinite(piv)) atomicExch(bad, 1);
        double *F = fac + (size_t)i * 5;
        F[0] = l2;
        F[1] = l1;
        F[2] = 1.0 / piv;
        F[3] = (i + 1 < M) ? A[i][3] : 0.0;
        F[4] = (i + 2 < M) ? A[i][4] : 0.0;
    }
}

// ------------------------------------------------------------------ stepper
struct PartArgs {
    int n, L, m;
    long B;
    const double *rowc;                // n x 5
    const double *fac;                 // 2P x 5
    const double *in; long ld_in;      // null -> zero
    double *out; long ld_out;
    const double *off; long ld_off;
    // source (same convention as StepArgs): R == 0 none
    int R, RS;
    const double *spaceT;              // n x RS (zero padded)
    const double *time;
    const double *amp;
    int nsteps, nsrc, q0, vpi;
    double dt;
};

// Shared memory of one CTA (chunk): state [L][32] | coefficients [L][5] |
// source rows [L][RS] | interface factors [2P][5] | interface rhs [2P][32]
// (used in the leader) | this chunk's (b_{c-1}, t_{c+1}) [2][32].
static size_t part_smem(int L, int P, int RS)
{
    return ((size_t)L * 32 + (size_t)L * 5 + (size_t)L * RS + (size_t)2 * P * 5 + (size_t)2 * P * 32 + 64) *
           sizeof(double);
}

template <int P, int RS>
__global__ void __launch_bounds__(32) k_part_step(PartArgs a)
{
    extern __shared__ __align__(16) double sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int c = (int)cluster.block_rank();             // chunk
    const long grp = blockIdx.x / P;                     // group of 32 vectors
    const int lane = threadIdx.x;
    const long v = grp * 32 + lane;
    const bool valid = v < a.B;
    const int L = a.L;
    const int s0 = c * L, nr = max(0, min(a.n, s0 + L) - s0);
    double *st = sm;
    double *co = st + (size_t)L * 32;
    double *sp = co + (size_t)L * 5;
    double *fac = sp + (size_t)L * RS;
    double *xg = fac + 2 * P * 5;
    double *mine = xg + 2 * P * 32;
    for (int i = lane; i < nr * 5; i += 32) co[i] = a.rowc[(size_t)s0 * 5 + i];
    if constexpr (RS > 0)
        for (int i = lane; i < nr * RS; i += 32) sp[i] = a.spaceT[(size_t)s0 * RS + i];
    if (c == 0)
        for (int i = lane; i < 2 * P * 5; i += 32) fac[i] = a.fac[i];
    for (int i = 0; i < nr; ++i)
        st[i * 32 + lane] = (a.in && valid) ? a.in[(long)(s0 + i) * a.ld_in + v] : 0.0;
    double bL = 0.0, tR = 0.0;
    const int q = valid ? a.q0 + (int)(v / a.vpi) : a.q0;
    const int src = (RS > 0 && valid) ? (int)(v % a.nsrc) : 0;
    double *lead = cluster.map_shared_rank(xg, 0);
    __syncwarp();
    for (int j = 1; j <= a.m; ++j) {
        double alpha[RS > 0 ? RS : 1];
        if constexpr (RS > 0) {
#pragma unroll
            for (int r = 0; r < RS; ++r) {
                double al = 0.0;
                if (r < a.R && valid)
                    al = a.dt * a.amp[(long)src * a.R + r] * a.time[(long)r * a.nsteps + (long)q * a.m + j - 1];
                alpha[r] = al;
            }
        }
        // down: x = g + V bL + W tR (previous step's solution), r = x + dt f_j,
        //       y_i = w_i r_i - ga_i y_{i-1}
        double yp = 0.0;
        const bool corr = j > 1;
#pragma unroll 4
        for (int i = 0; i < nr; ++i) {
            const double *C = co + i * 5;
            double x = st[i * 32 + lane];
            if (corr) x = fma(C[3], bL, fma(C[4], tR, x));
            if constexpr (RS > 0) {
#pragma unroll
                for (int r = 0; r < RS; ++r) x = fma(alpha[r], sp[i * RS + r], x);
            }
            yp = fma(C[1], yp, C[0] * x);
            st[i * 32 + lane] = yp;
        }
        // up: g_i = y_i - cp_i g_{i+1}
        double gn = 0.0;
#pragma unroll 4
        for (int i = nr - 1; i >= 0; --i) {
            const double g = fma(co[i * 5 + 2], gn, st[i * 32 + lane]);
            st[i * 32 + lane] = g;
            gn = g;
        }
        lead[(2 * c) * 32 + lane] = st[lane];
        lead[(2 * c + 1) * 32 + lane] = st[(nr - 1) * 32 + lane];
        cluster.sync();
        if (c == 0) {
            // banded forward / back substitution of the interface system
            constexpr int M = 2 * P;
            double z[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double zi = xg[i * 32 + lane];
                if (i >= 2) zi = fma(-fac[i * 5 + 0], z[i - 2], zi);
                if (i >= 1) zi = fma(-fac[i * 5 + 1], z[i - 1], zi);
                z[i] = zi;
            }
#pragma unroll
            for (int i = M - 1; i >= 0; --i) {
                double zi = z[i];
                if (i + 1 < M) zi = fma(-fac[i * 5 + 3], z[i + 1], zi);
                if (i + 2 < M) zi = fma(-fac[i * 5 + 4], z[i + 2], zi);
                z[i] = zi * fac[i * 5 + 2];
            }
#pragma unroll
            for (int cc = 0; cc < P; ++cc) {
                double *dst = cluster.map_shared_rank(mine, cc);
                dst[lane] = (cc > 0) ? z[2 * cc - 1] : 0.0;
                dst[32 + lane] = (cc < P - 1) ? z[2 * cc + 2] : 0.0;
            }
        }
        cluster.sync();
        bL = mine[lane];
        tR = mine[32 + lane];
    }
    if (valid) {
        for (int i = 0; i < nr; ++i) {
            const double *C = co + i * 5;
            double x = fma(C[3], bL, fma(C[4], tR, st[i * 32 + lane]));
            if (a.off) x += a.off[(long)(s0 + i) * a.ld_off + v];
            a.out[(long)(s0 + i) * a.ld_out + v] = x;
        }
    }
}

// ---------------------------------------------------------------- driver
int part_chunks(int n)
{
    // largest P in {16, 8, 4, 2} with chunks of >= 32 rows; chunks hold <= PART_LMAX rows
    for (int P = 16; P >= 2; P /= 2)
        if (n / P >= 32 && (n + P - 1) / P <= PART_LMAX) return P;
    return 0;
}

cudaError_t launch_part_setup(int n, int P, const double *subA, const double *supA, const double *rsA,
                              const double *diagA, double dt, int transpose, double *rowc, double *fac,
                              double *ends, int *bad, cudaStream_t s)
{
    const int L = (n + P - 1) / P;
    note_launch();
    k_part_setup<<<1, 32, 0, s>>>(n, P, L, subA, supA, rsA, diagA, dt, transpose, rowc, ends, bad);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    note_launch();
    k_part_reduced<<<1, 1, 0, s>>>(P, ends, fac, bad);
    return cudaGetLastError();
}

template <int P, int RS>
static cudaError_t part_launch(const PartArgs &a, long groups, cudaStream_t s)
{
    const size_t smem = part_smem(a.L, P, RS);
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(k_part_step<P, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)part_smem(PART_LMAX, P, RS));
        if (e == cudaSuccess && P > 8)
            e = cudaFuncSetAttribute(k_part_step<P, RS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(groups * P));
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    note_launch();
    return cudaLaunchKernelEx(&cfg, k_part_step<P, RS>, a);
}

template <int P>
static cudaError_t part_launch_rs(const PartArgs &a, long groups, cudaStream_t s)
{
    switch (a.RS) {
    case 0: return part_launch<P, 0>(a, groups, s);
    case 1: return part_launch<P, 1>(a, groups, s);
    case 2: return part_launch<P, 2>(a, groups, s);
    case 4: return part_launch<P, 4>(a, groups, s);
    default: return part_launch<P, 8>(a, groups, s);
    }
}

bool part_preferred(const Op &op, long B, int m)
{
    if (op.part_P == 0 || m < 1 || getenv("PR_NO_PART")) return false;
    if (getenv("PR_FORCE_PART")) return true;
    // the fused stepper wins once its one-vector-per-thread warps fill the GPU
    const long groups = (B + 31) / 32;
    return groups * 4 <= num_sms();
}

cudaError_t launch_stepper_part(const Op &op, const StepArgs &sa, int transpose, cudaStream_t s)
{
    const int P = op.part_P;
    PartArgs a{};
    a.n = sa.n; a.L = (sa.n + P - 1) / P; a.m = sa.m; a.B = sa.B;
    a.rowc = transpose ? op.part_rowc_tr : op.part_rowc_fw;
    a.fac = transpose ? op.part_fac_tr : op.part_fac_fw;
    a.in = sa.in; a.ld_in = sa.ld_in; a.out = sa.out; a.ld_out = sa.ld_out;
    a.off = sa.off; a.ld_off = sa.ld_off;
    a.R = sa.R; a.RS = sa.R > 0 ? stepper_rs(sa.R) : 0;
    a.spaceT = sa.spaceT; a.time = sa.time; a.amp = sa.amp;
    a.nsteps = sa.nsteps; a.nsrc = sa.nsrc; a.q0 = sa.q0; a.vpi = sa.vpi; a.dt = sa.dt;
    const long groups = (sa.B + 31) / 32;
    if (groups == 0) return cudaSuccess;
    const bool prof = profiling();
    if (prof) stepper_timed_begin(s);
    cudaError_t e;
    switch (P) {
    case 16: e = part_launch_rs<16>(a, groups, s); break;
    case 8: e = part_launch_rs<8>(a, groups, s); break;
    case 4: e = part_launch_rs<4>(a, groups, s); break;
    default: e = part_launch_rs<2>(a, groups, s); break;
    }
    if (prof) stepper_timed_end(s, (double)sa.n * (double)sa.B * (double)sa.m, 0.0);
    return e;
}

}  // namespace pr
