// k_pencil.cu -- K1T: batched 1D backward-Euler stepper for TIME-DEPENDENT
// pencils (eq. ex2), with an optional
// mass matrix (row 2; linear finite elements):
//
//     (M + dt A(t_g)) u_g = M u_{g-1} + dt l(t_g),      g = q*m + j,
//
// every step with its own tridiagonal left-hand side L_g = M + dt A(t_g)
// (Exp 2: kappa(x, t) = 1 + 0.9 sin(7 pi t + 2 pi x), Neumann rows), so the
// interval operators F_q' differ and are not normal.  The adjoint
// is the true transpose of the product, steps in REVERSE order (R-ADJ):
//     F_q'^T = (M^T L_{q,1}^{-T}) ... (M^T L_{q,m}^{-T}).
//
// Factorisation (k_pencil_factor, once per operator, one thread per step):
// L_g = L' U' with L' lower bidiagonal {sub a_i, diag p_i}, U' unit upper
// {super c'_i = c_i / p_i}; pivots from the exact row sums when given (reading
// R-ACC), else p_i = b_i - a_i c_{i-1} / p_{i-1}.  Per row and step:
//     {w_i = 1/p_i, ga_i = w_i a_i, cp_i = w_i c_i, gt_i = w_i a_{i+1}}
//   forward  L_g x = r:   y_i = w_i r_i - ga_i y_{i-1};  x_i = y_i - cp_i x_{i+1}
//   adjoint  L_g^T z = r: v_i = r_i - cp_{i-1} v_{i-1};  z_i = w_i v_i - gt_i z_{i+1}
//
// Stepper (k_pencil_step): one thread per vector of the interleaved (n x ld)
// batch (a warp's 32 vectors of one row are one 256-byte segment), two
// streaming passes per step over the state in the output buffer; the mass
// matrix product M x (or M^T z) is formed on the fly in the down pass from a
// three-row register window; the per-row factors of a step are warp-uniform
// loads (L1 broadcast).  HBM-bound: 32 B per DOF-step (+ 0 for M, formed from
// the window) -- no pass fusion here because consecutive steps have different
// factors (the time-independent K1/K1P paths fuse).
#include "pr_internal.cuh"

namespace pr {

__global__ void k_pencil_factor(int n, int nsteps, const double *__restrict__ lsub,
                                const double *__restrict__ ldiag, const double *__restrict__ lsup,
                                const double *__restrict__ lrs, Coef *fac, int *bad)
{
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nsteps) return;
    const double *a = lsub + (size_t)g * n, *b = ldiag + (size_t)g * n, *c = lsup + (size_t)g * n;
    const double *s = lrs ? lrs + (size_t)g * n : nullptr;
    Coef *F = fac + (size_t)g * n;
    double p = 1.0, r = 0.0;
    bool ok = true;
    for (int i = 0; i < n; ++i) {
        const double ai = (i > 0) ? a[i] : 0.0;
        const double ci = (i < n - 1) ? c[i] : 0.0;
        double piv;
        if (s) {
            r = (i == 0) ? s[0] : s[i] - ai * (r / p);
            piv = r - ci;
            if (!(piv > 0.0)) ok = false;
        } else {
            piv = (i == 0) ? b[0] : b[i] - ai * (c[i - 1] / p);
        }
        if (!(piv != 0.0) || !isfinite(piv)) ok = false;
        p = piv;
        const double w = 1.0 / piv;
        const double an = (i + 1 < n) ? a[i + 1] : 0.0;
        F[i] = Coef{w, w * ai, w * ci, w * an};
    }
    if (!ok) atomicExch(bad, 1);
}

struct PencilArgs {
    int n, m;
    long B;
    const Coef *fac;                   // nsteps x n
    const double *msub, *mdiag, *msup; // null: M = I
    const double *in; long ld_in;      // null -> zero input
    double *out; long ld_out;
    const double *off; long ld_off;
    int q0, vpi;
    int step0, mstride;                // global step of step j: q*mstride + step0 + j
    int R;                             // source terms (0: none)
    const double *spaceT; int rs;      // n x rs
    const double *time;                // R x nsteps
    const double *amp;                 // nsrc x R
    int nsteps, nsrc;
    double dt;
};

template <int MODE>                    // 0 linear, 1 affine, 2 adjoint
__global__ void __launch_bounds__(128) k_pencil_step(PencilArgs a)
{
    const long v = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= a.B) return;
    const int n = a.n;
    const int q = a.q0 + (int)(v / a.vpi);
    double *X = a.out + v;
    const long ldx = a.ld_out;
    const bool hasM = a.mdiag != nullptr;
    double al[8];
    for (int s = 0; s < a.m; ++s) {
        const int j = (MODE == 2) ? a.m - s : s + 1;       // 1-based step within the interval
        const long g = (long)q * a.mstride + a.step0 + j;   // 1-based global step
        const Coef *F = a.fac + (g - 1) * n;
        // input of this step's down pass: the previous state (or U_in)
        const double *Src = (s == 0) ? (a.in ? a.in + v : nullptr) : X;
        const long lds = (s == 0) ? a.ld_in : ldx;
        if (MODE == 1) {
            for (int r = 0; r < 8; ++r) al[r] = 0.0;
            const int src = (int)(v % a.nsrc);
            for (int r = 0; r < a.R && r < 8; ++r)
                al[r] = a.dt * a.amp[(long)src * a.R + r] * a.time[(long)r * a.nsteps + g - 1];
        }
        auto ld_src = [&](int i) -> double { return Src ? Src[(long)i * lds] : 0.0; };
        // down pass (rows ascending); window xm / x0 / xp of the input
        double xm = 0.0, x0 = ld_src(0), y = 0.0;
        for (int i = 0; i < n; ++i) {
            const double xp = (i + 1 < n) ? ld_src(i + 1) : 0.0;
            double r;
            if (MODE == 2) {
                // r = M^T z_prev after the first adjoint step, the input before it
                if (hasM && s > 0)
                    r = fma(a.mdiag[i], x0, (i > 0 ? a.msup[i - 1] * xm : 0.0) + (i + 1 < n ? a.msub[i + 1] * xp : 0.0));
                else
                    r = x0;
                const double cpm = (i > 0) ? F[i - 1].c : 0.0;
                y = fma(-cpm, y, r);                              // v_i = r_i - cp_{i-1} v_{i-1}
            } else {
                r = hasM ? fma(a.mdiag[i], x0, (i > 0 ? a.msub[i] * xm : 0.0) + (i + 1 < n ? a.msup[i] * xp : 0.0))
                         : x0;
                if (MODE == 1) {
                    double f = 0.0;
                    for (int k = 0; k < a.R && k < 8; ++k) f = fma(al[k], a.spaceT[(long)i * a.rs + k], f);
                    r += f;
                }
                const Coef c = F[i];
                y = fma(-c.b, y, c.a * r);                        // y_i = w_i r_i - ga_i y_{i-1}
            }
            X[(long)i * ldx] = y;
            xm = x0;
            x0 = xp;
        }
        // up pass (rows descending)
        double xn = 0.0;
        for (int i = n - 1; i >= 0; --i) {
            const Coef c = F[i];
            const double yi = X[(long)i * ldx];
            xn = (MODE == 2) ? fma(-c.d, xn, c.a * yi)             // z_i = w_i v_i - gt_i z_{i+1}
                             : fma(-c.c, xn, yi);                 // x_i = y_i - cp_i x_{i+1}
            X[(long)i * ldx] = xn;
        }
    }
    if (a.m == 0) {                    // F' = identity
        for (int i = 0; i < n; ++i) X[(long)i * ldx] = a.in ? a.in[v + (long)i * a.ld_in] : 0.0;
    }
    if (MODE == 2 && hasM && a.m > 0) {   // the last factor M^T of the adjoint
        double zm = 0.0, z0 = X[0];
        for (int i = 0; i < n; ++i) {
            const double zp = (i + 1 < n) ? X[(long)(i + 1) * ldx] : 0.0;
            X[(long)i * ldx] = fma(a.mdiag[i], z0, (i > 0 ? a.msup[i - 1] * zm : 0.0) + (i + 1 < n ? a.msub[i + 1] * zp : 0.0));
            zm = z0;
            z0 = zp;
        }
    }
    if (a.off)
        for (int i = 0; i < n; ++i) X[(long)i * ldx] += a.off[v + (long)i * a.ld_off];
}

// The Cholesky factor of the mass matrix (weighted views, R-WIP): one thread per
// vector, rows in the order the recurrence needs (in place safe).
template <int MODE>
__global__ void k_bidiag(int n, const double *__restrict__ cd, const double *__restrict__ ce, long B,
                         const double *in, long irs, long ivs, double *out, long ors, long ovs)
{
    const long v = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= B) return;
    const double *x = in ? in + v * ivs : nullptr;
    double *y = out + v * ovs;
    auto X = [&](int i) -> double { return x ? x[(long)i * irs] : 0.0; };
    if (MODE == BIDIAG_C) {              // y_i = c_ii x_i + c_{i,i+1} x_{i+1}   (ascending)
        double xi = X(0);
        for (int i = 0; i < n; ++i) {
            const double xn = (i + 1 < n) ? X(i + 1) : 0.0;
            y[(long)i * ors] = fma(cd[i], xi, (i + 1 < n) ? ce[i] * xn : 0.0);
            xi = xn;
        }
    } else if (MODE == BIDIAG_CT) {      // y_i = c_ii x_i + c_{i-1,i} x_{i-1}   (descending)
        double xi = X(n - 1);
        for (int i = n - 1; i >= 0; --i) {
            const double xp = (i > 0) ? X(i - 1) : 0.0;
            y[(long)i * ors] = fma(cd[i], xi, (i > 0) ? ce[i - 1] * xp : 0.0);
            xi = xp;
        }
    } else if (MODE == BIDIAG_CINV) {    // C y = x: back substitution
        double yn = 0.0;
        for (int i = n - 1; i >= 0; --i) {
            const double r = (i + 1 < n) ? fma(-ce[i], yn, X(i)) : X(i);
            yn = r / cd[i];
            y[(long)i * ors] = yn;
        }
    } else {                             // C^T y = x: forward substitution
        double yp = 0.0;
        for (int i = 0; i < n; ++i) {
            const double r = (i > 0) ? fma(-ce[i - 1], yp, X(i)) : X(i);
            yp = r / cd[i];
            y[(long)i * ors] = yp;
        }
    }
}

cudaError_t launch_bidiag(int mode, int n, const double *cdiag, const double *csup, long B, const double *in,
                          long irs, long ivs, double *out, long ors, long ovs, cudaStream_t s)
{
    if (B == 0) return cudaSuccess;
    note_launch();
    const unsigned blocks = (unsigned)((B + 127) / 128);
    switch (mode) {
    case BIDIAG_C: k_bidiag<BIDIAG_C><<<blocks, 128, 0, s>>>(n, cdiag, csup, B, in, irs, ivs, out, ors, ovs); break;
    case BIDIAG_CT: k_bidiag<BIDIAG_CT><<<blocks, 128, 0, s>>>(n, cdiag, csup, B, in, irs, ivs, out, ors, ovs); break;
    case BIDIAG_CINV: k_bidiag<BIDIAG_CINV><<<blocks, 128, 0, s>>>(n, cdiag, csup, B, in, irs, ivs, out, ors, ovs); break;
    default: k_bidiag<BIDIAG_CTINV><<<blocks, 128, 0, s>>>(n, cdiag, csup, B, in, irs, ivs, out, ors, ovs); break;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K1T-CTA: one thread block per vector for SMALL batches (the Parareal fine
// solves have one vector per interval and source).  The T threads of the block
// own RR consecutive rows each; the state stays in shared memory (row t*RR + i
// at xs[i*T + t], conflict-free) for all m steps.  Each step's two sweeps are
// first-order linear recurrences, y_i = a_i y_{i-1} + b_i, solved exactly by a
// block scan of the affine maps (a, b) of the thread segments: a local pass
// composes the segment map, a warp-shuffle + shared-memory scan gives every
// segment its carried-in value, a second local pass runs the recurrence from
// it (the same pivots and multipliers as the thread-per-vector kernel; all
// terms non-negative for an M-matrix, so no cancellation).
struct Aff {
    double A, B;                       // y -> A y + B
};

// inclusive scan over the block in thread order (REV: descending thread order)
// of maps composed as later o earlier; returns the EXCLUSIVE prefix applied to 0
template <int T, bool REV>
__device__ __forceinline__ double block_affine_carry(Aff f, Aff *sh)
{
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    constexpr int NW = T / 32;
    const int rl = REV ? 31 - lane : lane;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double pA = REV ? __shfl_down_sync(0xffffffffu, f.A, d) : __shfl_up_sync(0xffffffffu, f.A, d);
        const double pB = REV ? __shfl_down_sync(0xffffffffu, f.B, d) : __shfl_up_sync(0xffffffffu, f.B, d);
        if (rl >= d) f = Aff{f.A * pA, fma(f.A, pB, f.B)};
    }
    // warp totals (the last lane in scan order holds it)
    if (rl == 31) sh[w] = f;
    __syncthreads();
    if (t < 32) {
        const int rw = REV ? NW - 1 - t : t;          // warp index in scan order
        Aff g = (t < NW) ? sh[rw] : Aff{1.0, 0.0};
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            const double pA = __shfl_up_sync(0xffffffffu, g.A, d);
            const double pB = __shfl_up_sync(0xffffffffu, g.B, d);
            if (t >= d && t < NW) g = Aff{g.A * pA, fma(g.A, pB, g.B)};
        }
        if (t < NW) sh[NW + t] = g;                    // inclusive prefix at scan position t
    }
    __syncthreads();
    // exclusive prefix of this thread: own warp's inclusive up to the previous
    // lane, composed after the preceding warps' total
    const double eA = REV ? __shfl_down_sync(0xffffffffu, f.A, 1) : __shfl_up_sync(0xffffffffu, f.A, 1);
    const double eB = REV ? __shfl_down_sync(0xffffffffu, f.B, 1) : __shfl_up_sync(0xffffffffu, f.B, 1);
    const int rw = REV ? NW - 1 - w : w;
    const bool firstw = (rw == 0);
    const double carryw = firstw ? 0.0 : sh[NW + rw - 1].B;   // value entering this warp (scan position rw)
    double c;
    if (rl == 0) c = carryw;
    else c = fma(eA, carryw, eB);
    __syncthreads();                                    // sh reused by the next scan
    return c;
}

template <int MODE, int RR>            // MODE: 0 linear, 1 affine, 2 adjoint
__global__ void __launch_bounds__(256) k_pencil_cta(PencilArgs a)
{
    constexpr int T = 256;
    extern __shared__ __align__(16) double xs[];       // [RR][T]
    __shared__ Aff sh[2 * (T / 32)];
    const long v = blockIdx.x;
    const int t = threadIdx.x;
    const int n = a.n;
    const int q = a.q0 + (int)(v / a.vpi);
    const bool hasM = a.mdiag != nullptr;
    auto row_of = [&](int i) { return t * RR + i; };
    auto X = [&](int row) -> double {                  // state at a row (0 outside)
        if (row < 0 || row >= n) return 0.0;
        return xs[(row % RR) * T + row / RR];
    };
    for (int i = 0; i < RR; ++i) {
        const int row = row_of(i);
        xs[i * T + t] = (a.in && row < n) ? a.in[(long)row * a.ld_in + v] : 0.0;
    }
    __syncthreads();
    double al[8];
    for (int s = 0; s < a.m; ++s) {
        const int j = (MODE == 2) ? a.m - s : s + 1;
        const long g = (long)q * a.mstride + a.step0 + j;
        const Coef *F = a.fac + (g - 1) * n;
        if (MODE == 1) {
            const int src = (int)(v % a.nsrc);
            for (int r = 0; r < 8; ++r) al[r] = 0.0;
            for (int r = 0; r < a.R && r < 8; ++r)
                al[r] = a.dt * a.amp[(long)src * a.R + r] * a.time[(long)r * a.nsteps + g - 1];
        }
        // right-hand sides r_i (M x + dt f, or M^T z after the first adjoint step)
        double rv[RR], av[RR];
#pragma unroll
        for (int i = 0; i < RR; ++i) {
            const int row = row_of(i);
            double r = 0.0;
            if (row < n) {
                const double x0 = X(row);
                if (MODE == 2) {
                    r = (hasM && s > 0) ? fma(a.mdiag[row], x0, (row > 0 ? a.msup[row - 1] * X(row - 1) : 0.0) +
                                                                    (row + 1 < n ? a.msub[row + 1] * X(row + 1) : 0.0))
                                        : x0;
                } else {
                    r = hasM ? fma(a.mdiag[row], x0, (row > 0 ? a.msub[row] * X(row - 1) : 0.0) +
                                                         (row + 1 < n ? a.msup[row] * X(row + 1) : 0.0))
                             : x0;
                    if (MODE == 1) {
                        double f = 0.0;
                        for (int k = 0; k < a.R && k < 8; ++k) f = fma(al[k], a.spaceT[(long)row * a.rs + k], f);
                        r += f;
                    }
                }
            }
            rv[i] = r;
        }
        __syncthreads();                                // everyone read xs
        // down sweep: y_i = a_i y_{i-1} + b_i
        Aff f{1.0, 0.0};
#pragma unroll
        for (int i = 0; i < RR; ++i) {
            const int row = row_of(i);
            double ai = 0.0, bi = 0.0;
            if (row < n) {
                if (MODE == 2) {
                    ai = (row > 0) ? -F[row - 1].c : 0.0;          // v_i = r_i - cp_{i-1} v_{i-1}
                    bi = rv[i];
                } else {
                    const Coef c = F[row];
                    ai = -c.b;                                    // y_i = w_i r_i - ga_i y_{i-1}
                    bi = c.a * rv[i];
                }
            }
            av[i] = ai;
            rv[i] = bi;
            f = Aff{ai * f.A, fma(ai, f.B, bi)};
        }
        double y = block_affine_carry<T, false>(f, sh);
#pragma unroll
        for (int i = 0; i < RR; ++i) {
            y = fma(av[i], y, rv[i]);
            rv[i] = y;
        }
        // up sweep: x_i = c_i x_{i+1} + e_i (rows descending)
        Aff gb{1.0, 0.0};
#pragma unroll
        for (int i = RR - 1; i >= 0; --i) {
            const int row = row_of(i);
            double ci = 0.0, ei = 0.0;
            if (row < n) {
                const Coef c = F[row];
                if (MODE == 2) {
                    ci = -c.d;                                    // z_i = w_i v_i - gt_i z_{i+1}
                    ei = c.a * rv[i];
                } else {
                    ci = -c.c;                                    // x_i = y_i - cp_i x_{i+1}
                    ei = rv[i];
                }
            }
            av[i] = ci;
            rv[i] = ei;
            gb = Aff{ci * gb.A, fma(ci, gb.B, ei)};
        }
        double x = block_affine_carry<T, true>(gb, sh);
#pragma unroll
        for (int i = RR - 1; i >= 0; --i) {
            x = fma(av[i], x, rv[i]);
            xs[i * T + t] = x;
        }
        __syncthreads();
    }
    // output (adjoint: the last factor M^T first)
    double outv[RR];
#pragma unroll
    for (int i = 0; i < RR; ++i) {
        const int row = row_of(i);
        double x = (row < n) ? X(row) : 0.0;
        if (MODE == 2 && hasM && a.m > 0 && row < n)
            x = fma(a.mdiag[row], x, (row > 0 ? a.msup[row - 1] * X(row - 1) : 0.0) +
                                         (row + 1 < n ? a.msub[row + 1] * X(row + 1) : 0.0));
        outv[i] = x;
    }
#pragma unroll
    for (int i = 0; i < RR; ++i) {
        const int row = row_of(i);
        if (row < n) {
            double x = outv[i];
            if (a.off) x += a.off[(long)row * a.ld_off + v];
            a.out[(long)row * a.ld_out + v] = x;
        }
    }
}

template <int MODE>
static cudaError_t launch_cta_mode(const PencilArgs &a, cudaStream_t s)
{
    const int n = a.n;
    const unsigned blocks = (unsigned)a.B;
    if (n <= 256 * 2) { k_pencil_cta<MODE, 2><<<blocks, 256, 2 * 256 * 8, s>>>(a); return cudaGetLastError(); }
    if (n <= 256 * 4) { k_pencil_cta<MODE, 4><<<blocks, 256, 4 * 256 * 8, s>>>(a); return cudaGetLastError(); }
    if (n <= 256 * 8) { k_pencil_cta<MODE, 8><<<blocks, 256, 8 * 256 * 8, s>>>(a); return cudaGetLastError(); }
    if (n <= 256 * 16) { k_pencil_cta<MODE, 16><<<blocks, 256, 16 * 256 * 8, s>>>(a); return cudaGetLastError(); }
    return cudaErrorInvalidValue;
}

cudaError_t launch_pencil_factor(int n, int nsteps, const double *lsub, const double *ldiag,
                                 const double *lsup, const double *lrs, Coef *fac, int *bad,
                                 cudaStream_t s)
{
    note_launch();
    k_pencil_factor<<<(nsteps + 63) / 64, 64, 0, s>>>(n, nsteps, lsub, ldiag, lsup, lrs, fac, bad);
    return cudaGetLastError();
}

cudaError_t launch_stepper_pencil(const Op &op, int mode, const StepArgs &sa, cudaStream_t s)
{
    if (sa.B == 0) return cudaSuccess;
    PencilArgs a{};
    a.n = sa.n; a.m = sa.m; a.B = sa.B;
    a.fac = op.pen_fac;
    a.msub = op.pen_m; a.mdiag = op.pen_m ? op.pen_m + op.n : nullptr; a.msup = op.pen_m ? op.pen_m + 2 * op.n : nullptr;
    a.in = sa.in; a.ld_in = sa.ld_in; a.out = sa.out; a.ld_out = sa.ld_out;
    a.off = sa.off; a.ld_off = sa.ld_off;
    a.q0 = sa.q0; a.vpi = sa.vpi;
    a.step0 = sa.step0; a.mstride = sa.mstride > 0 ? sa.mstride : sa.m;
    a.R = sa.R; a.spaceT = sa.spaceT; a.rs = sa.R > 0 ? stepper_rs(sa.R) : 0;
    a.time = sa.time; a.amp = sa.amp; a.nsteps = sa.nsteps; a.nsrc = sa.nsrc > 0 ? sa.nsrc : 1;
    a.dt = sa.dt;
    const int threads = 128;
    const unsigned blocks = (unsigned)((sa.B + threads - 1) / threads);
    const bool prof = profiling();
    if (prof) stepper_timed_begin(s);
    note_launch();
    // a block per vector while the batch leaves the thread-per-vector kernel
    // with fewer than ~4 resident warps per SM (and n fits the block's rows)
    const bool cta = sa.n >= 256 && sa.n <= 256 * 16 && sa.B <= 4L * num_sms() * 32 && !flags().no_part;
    cudaError_t e = cudaSuccess;
    if (cta) {
        if (mode == PR_ADJOINT) e = launch_cta_mode<2>(a, s);
        else if (sa.R > 0) e = launch_cta_mode<1>(a, s);
        else e = launch_cta_mode<0>(a, s);
    } else if (mode == PR_ADJOINT) k_pencil_step<2><<<blocks, threads, 0, s>>>(a);
    else if (sa.R > 0) k_pencil_step<1><<<blocks, threads, 0, s>>>(a);
    else k_pencil_step<0><<<blocks, threads, 0, s>>>(a);
    if (e != cudaSuccess) return e;
    if (prof) {
        const double dof = (double)sa.n * (double)sa.B * (double)sa.m;
        stepper_timed_end(s, dof, (5.0 + (op.pen_m ? 5.0 : 0.0) + 2.0 * sa.R) * dof);
    }
    return cudaGetLastError();
}

}  // namespace pr
