// k_sep2d.cu -- K2: separable 2D backward-Euler stepper on FP64 tensor cores.
//
// A = T (x) I + I (x) T (5-point Laplacian, Dirichlet, n x n interior points),
// T = S diag(lam) S with the orthogonal symmetric sine matrix S.  One fine
// step (I + dt A) u_j = u_{j-1} + dt f_j is, in the eigenbasis,
// the elementwise update  u^_j = D o (u^_{j-1} + dt f^_j),
// D_ac = 1 / (1 + dt (lam_a + lam_c)).  A fine solve of m steps is therefore
//     X^ = S X S  (2 GEMM passes),  m diagonal steps (fused in the epilogue of
//     the 2nd pass, executed step by step -- SURVEY rule R1),  out = S X^ S.
//
// Storage: P = n + 1, vectors are P x P row-major with a zero ghost row and
// column 0.  S_ij = sqrt(2/P) sin(i j pi / P), i, j in [0, P): row/column 0 of
// S vanish, so ghosts stay exactly zero through every pass.
//
// GEMM pass: out_b = (S X_b)^T for every vector b -- two passes give
// ((S X)^T S)^T ... = S X S because S = S^T.  Tensor cores: legacy DMMA
// (mma.sync.m8n8k4.f64; tcgen05 has no f64 kind).  CTA tile
// 64 x 64, K chunks of 16 double-buffered with cp.async, 4 warps of 32 x 32.
#include <math.h>

#include "pr_internal.cuh"

namespace pr {

constexpr int GM = 64, GN = 64, GK = 16;
constexpr int AST = GK + 4;    // smem row stride of K-fastest tiles (doubles): conflict-free frags
constexpr int BST = GN + 4;    // smem row stride of N-fastest B tiles
constexpr int G_THREADS = 128;

enum { EPI_NONE = 0, EPI_DIAG = 1, EPI_OFF = 2 };

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cpa16(void *smem, const void *gmem)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}

struct GemmArgs {
    const double *S;      // P x P
    int P;
    const double *X;  long ldx;    // vector b at X + b*ldx (P x P row-major)
    double *out;      long ldo;
    long B;
    const double *off; long ldoff; // EPI_OFF
    const double *lam;             // EPI_DIAG
    double dt;
    int msteps;
    long xrows;                    // BT: rows of the source matrix (bounds)
};

// out_b = (S * op(X_b))^T, op = identity (BT = false) or transpose (BT = true).
template <bool BT, int EPI>
__global__ void __launch_bounds__(G_THREADS) k_gemm_st(GemmArgs g)
{
    extern __shared__ __align__(16) double sm[];
    double *As = sm;                              // [2][GM * AST]
    double *Bs = sm + 2 * GM * AST;               // [2][GK * BST] or [2][GN * AST] (BT)
    const int P = g.P;
    const int TM = P / GM, TN = P / GN;
    const long blk = blockIdx.x;
    const int tm = (int)(blk % TM), tn = (int)((blk / TM) % TN);
    const long b = blk / ((long)TM * TN);
    const int m0 = tm * GM, n0 = tn * GN;
    const double *Xb = g.X + b * g.ldx;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int wm = (w & 1) * 32, wn = (w >> 1) * 32;
    const int gq = lane >> 2, tq = lane & 3;
    const int bstride = BT ? GN * AST : GK * BST;

    auto stage = [&](int kc, int buf) {
        const int k0 = kc * GK;
        double *a = As + buf * GM * AST;
        for (int i = tid; i < GM * (GK / 2); i += G_THREADS) {
            int row = i / (GK / 2), ch = i % (GK / 2);
            cpa16(a + row * AST + 2 * ch, g.S + (long)(m0 + row) * P + k0 + 2 * ch);
        }
        double *bb = Bs + buf * bstride;
        if (!BT) {
            for (int i = tid; i < GK * (GN / 2); i += G_THREADS) {
                int k = i / (GN / 2), ch = i % (GN / 2);
                cpa16(bb + k * BST + 2 * ch, Xb + (long)(k0 + k) * P + n0 + 2 * ch);
            }
        } else {
            for (int i = tid; i < GN * (GK / 2); i += G_THREADS) {
                int n = i / (GK / 2), ch = i % (GK / 2);
                cpa16(bb + n * AST + 2 * ch, Xb + (long)(n0 + n) * P + k0 + 2 * ch);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int nk = P / GK;
    stage(0, 0);
    for (int kc = 0; kc < nk; ++kc) {
        if (kc + 1 < nk) {
            stage(kc + 1, (kc + 1) & 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const double *a = As + (kc & 1) * GM * AST;
        const double *bb = Bs + (kc & 1) * bstride;
#pragma unroll
        for (int kk = 0; kk < GK / 4; ++kk) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = a[(wm + i * 8 + gq) * AST + kk * 4 + tq];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                bf[j] = BT ? bb[(wn + j * 8 + gq) * AST + kk * 4 + tq]
                           : bb[(kk * 4 + tq) * BST + wn + j * 8 + gq];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncthreads();
    }

    // epilogue: stage C^T (n-major) in smem, then coalesced row writes of out_b
    double *Cs = sm;                              // GN x (GM + 1)
    constexpr int CST = GM + 1;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int m = wm + i * 8 + gq;
            const int n = wn + j * 8 + 2 * tq;
            Cs[n * CST + m] = acc[i][j][0];
            Cs[(n + 1) * CST + m] = acc[i][j][1];
        }
    __syncthreads();
    double *ob = g.out + b * g.ldo;
    const double *offb = (EPI == EPI_OFF) ? g.off + b * g.ldoff : nullptr;
    for (int i = tid; i < GN * GM; i += G_THREADS) {
        const int n = i / GM, mm = i % GM;
        double x = Cs[n * CST + mm];
        const long pos = (long)(n0 + n) * P + m0 + mm;
        if (EPI == EPI_DIAG) {
            // m implicit-Euler steps in the eigenbasis: x <- D x, one step at a time
            const double D = 1.0 / (1.0 + g.dt * (g.lam[n0 + n] + g.lam[m0 + mm]));
            for (int s = 0; s < g.msteps; ++s) x *= D;
        }
        if (EPI == EPI_OFF) x += offb[pos];
        ob[pos] = x;
    }
}

template <bool BT, int EPI>
static cudaError_t launch_gemm_t(const GemmArgs &g, cudaStream_t s)
{
    const long tiles = (long)(g.P / GM) * (g.P / GN) * g.B;
    if (tiles == 0) return cudaSuccess;
    const size_t main = (size_t)2 * GM * AST + (size_t)2 * (BT ? GN * AST : GK * BST);
    const size_t epi = (size_t)GN * (GM + 1);
    const size_t smem = (main > epi ? main : epi) * sizeof(double);
    auto kern = k_gemm_st<BT, EPI>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (tiles > 0x7fffffffL) return cudaErrorInvalidValue;
    note_launch();
    kern<<<(unsigned)tiles, G_THREADS, smem, s>>>(g);
    return cudaGetLastError();
}

static cudaError_t launch_gemm(const GemmArgs &g, int epi, cudaStream_t s)
{
    switch (epi) {
    case EPI_DIAG: return launch_gemm_t<false, EPI_DIAG>(g, s);
    case EPI_OFF: return launch_gemm_t<false, EPI_OFF>(g, s);
    default: return launch_gemm_t<false, EPI_NONE>(g, s);
    }
}

// ----------------------------------------------------------------- setup
__global__ void k_sep2d_init(int P, double *S, double *lam)
{
    long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < (long)P * P) {
        long i = idx / P, j = idx % P;
        long r = (i * j) % (2L * P);     // exact argument reduction of i j pi / P
        S[idx] = sqrt(2.0 / P) * sinpi((double)r / P);
    }
    if (idx < P) {
        // lam_i = (4/h^2) sin^2(i pi / (2P)), h = 1/P
        double sv = sinpi((double)idx / (2.0 * P));
        lam[idx] = 4.0 * (double)P * (double)P * sv * sv;
    }
}

// ghat[(b*nsl + t)*P + a] = sum_i S[a][i] * g[(b*nsteps + g0 + t)*P + i], t < nsl
__global__ void k_src_hat(const double *S, int P, const double *gsrc, int nsteps, int g0, int nsl,
                          int nb, double *ghat)
{
    long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    long tot = (long)nb * nsl * P;
    if (idx >= tot) return;
    const int a = (int)(idx % P);
    const long bt = idx / P;
    const int bb = (int)(bt / nsl), t = (int)(bt % nsl);
    const double *gv = gsrc + ((long)bb * nsteps + g0 + t) * P;
    const double *Sa = S + (long)a * P;
    double s = 0.0;
    for (int i = 0; i < P; ++i) s = fma(Sa[i], gv[i], s);
    ghat[idx] = s;
}

// Offsets in the eigenbasis from a zero state: for vector v (interval
// q = q0 + v / vpi), x^_ac = 0; for j = 1..m: x^ <- D (x^ + dt sum_b gxh[a] gyh[c]).
__global__ void k_affine_hat(int P, int m, int q0, int vpi, int nb, int nsl, int g0,
                             const double *gxh, const double *gyh, const double *lam, double dt,
                             double *out, long ldo, long B)
{
    const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long per = (long)P * P;
    if (idx >= per * B) return;
    const long v = idx / per;
    const long e = idx % per;
    const int a = (int)(e / P), c = (int)(e % P);
    const int q = q0 + (int)(v / vpi);
    const double D = 1.0 / (1.0 + dt * (lam[a] + lam[c]));
    double x = 0.0;
    for (int j = 1; j <= m; ++j) {
        const int t = q * m + j - 1 - g0;       // local time index of step g = q m + j
        double f = 0.0;
        for (int bb = 0; bb < nb; ++bb)
            f = fma(gxh[((long)bb * nsl + t) * P + a], gyh[((long)bb * nsl + t) * P + c], f);
        x = D * fma(dt, f, x);
    }
    out[v * ldo + e] = (a == 0 || c == 0) ? 0.0 : x;
}

// ------------------------------------------------------------------ driver
static pr_status run_sep2d_impl(const Sep2dArgs &a, cudaStream_t s, int *passes);

// Timed wrapper: the fine solves of one call (all its GEMM passes and
// epilogues) are one "stepper launch" for pr_counters; flops = 2 P^3 per
// vector per GEMM pass.
pr_status run_sep2d(const Sep2dArgs &a, cudaStream_t s)
{
    const bool prof = profiling();
    if (prof) stepper_timed_begin(s);
    int passes = 0;
    pr_status st = run_sep2d_impl(a, s, &passes);
    if (prof) {
        const double P = a.op->P;
        const double n2 = (double)a.op->n * a.op->n;
        stepper_timed_end(s, n2 * (double)a.B * a.m, 2.0 * P * P * P * (double)a.B * passes);
    }
    return st;
}

static pr_status run_sep2d_impl(const Sep2dArgs &a, cudaStream_t s, int *passes)
{
    const Op &op = *a.op;
    const int P = op.P;
    const long per = (long)P * P;
    const long B = a.B;
    double *T = (double *)ws_alloc((size_t)B * per * sizeof(double), s);
    if (!T) { set_error("out of device memory"); return PR_EOOM; }
    struct Free { void *p; cudaStream_t s; ~Free() { ws_free(p, s); } } fT{T, s};
    GemmArgs g{};
    g.S = op.S;
    g.P = P;
    g.B = B;
    g.lam = op.lam;
    g.dt = op.dt;
    g.msteps = a.m;
    const bool affine = (a.mode == PR_AFFINE) && a.f && a.f->kind == PR_SRC_BUMP2D;
    if (affine && a.in && a.off) {
        set_error("PR_AFFINE with both an input and an offset is not supported in 2D");
        return PR_EINVAL;
    }
    double *bvec = nullptr;
    struct Free2 { void *p; cudaStream_t s; ~Free2() { ws_free(p, s); } } fb{nullptr, s};
    if (affine) {
        // b = F 0: eigenbasis offsets, then S b^ S (+ offset when there is no input)
        const int nint = (int)((B + a.vpi - 1) / a.vpi);
        const int g0 = a.q0 * a.m;
        const int nsl = nint * a.m;
        const int nb = a.f->nterms;
        double *gh = (double *)ws_alloc((size_t)2 * nb * nsl * P * sizeof(double), s);
        if (!gh) { set_error("out of device memory"); return PR_EOOM; }
        struct Free3 { void *p; cudaStream_t s; ~Free3() { ws_free(p, s); } } fg{gh, s};
        double *gxh = gh, *gyh = gh + (size_t)nb * nsl * P;
        long tot = (long)nb * nsl * P;
        note_launch();
        k_src_hat<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(op.S, P, a.f->gx, a.f->nsteps, g0, nsl, nb, gxh);
        note_launch();
        k_src_hat<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(op.S, P, a.f->gy, a.f->nsteps, g0, nsl, nb, gyh);
        PR_CHECK_LAUNCH("k_src_hat");
        bvec = a.in ? (double *)ws_alloc((size_t)B * per * sizeof(double), s) : a.out;
        if (!bvec) { set_error("out of device memory"); return PR_EOOM; }
        if (a.in) fb.p = bvec;
        const long ldb = a.in ? per : a.ld_out;
        long tot2 = per * B;
        note_launch();
        k_affine_hat<<<(unsigned)((tot2 + 255) / 256), 256, 0, s>>>(P, a.m, a.q0, a.vpi, nb, nsl, g0, gxh, gyh,
                                                                    op.lam, op.dt, bvec, ldb, B);
        PR_CHECK_LAUNCH("k_affine_hat");
        g.X = bvec; g.ldx = ldb; g.out = T; g.ldo = per;
        PR_CUDA(launch_gemm(g, EPI_NONE, s));                   // T = (S b^)^T
        *passes += 2;
        g.X = T; g.ldx = per; g.out = bvec; g.ldo = ldb;
        if (!a.in && a.off) {
            g.off = a.off; g.ldoff = a.ld_off;
            PR_CUDA(launch_gemm(g, EPI_OFF, s));                // b = S b^ S + offset
        } else {
            PR_CUDA(launch_gemm(g, EPI_NONE, s));               // b = S b^ S
        }
        if (!a.in) return PR_OK;
    }
    if (!a.in) {
        // linear map of a zero input (+ offset)
        if (a.off) PR_CUDA(launch_copy_vectors(a.off, 1, a.ld_off, a.out, 1, a.ld_out, per, (int)B, s));
        else PR_CUDA(cudaMemset2DAsync(a.out, a.ld_out * sizeof(double), 0, per * sizeof(double), B, s));
        return PR_OK;
    }
    // LINEAR / ADJOINT (A symmetric, time-independent: F'^* = F'), + offset
    g.X = a.in; g.ldx = a.ld_in; g.out = T; g.ldo = per;
    *passes += 4;
    PR_CUDA(launch_gemm(g, EPI_NONE, s));                       // T  = (S X)^T
    g.X = T; g.ldx = per; g.out = a.out; g.ldo = a.ld_out;
    PR_CUDA(launch_gemm(g, EPI_DIAG, s));                       // X^ = S X S, m diagonal steps
    g.X = a.out; g.ldx = a.ld_out; g.out = T; g.ldo = per;
    PR_CUDA(launch_gemm(g, EPI_NONE, s));                       // T  = (S X^)^T
    g.X = T; g.ldx = per; g.out = a.out; g.ldo = a.ld_out;
    const double *off = a.off;
    long ldoff = a.ld_off;
    if (affine) { off = bvec; ldoff = per; }
    if (off) {
        g.off = off; g.ldoff = ldoff;
        PR_CUDA(launch_gemm(g, EPI_OFF, s));                    // out = S X^ S + offset
    } else {
        PR_CUDA(launch_gemm(g, EPI_NONE, s));
    }
    return PR_OK;
}

}  // namespace pr

extern "C" pr_status pr_op_create_sep2d(int n, double dt, pr_op *out)
{
    using namespace pr;
    PR_REQUIRE(out, PR_EINVAL, "out is NULL");
    *out = nullptr;
    PR_REQUIRE(n >= 2 && (n + 1) % 64 == 0, PR_EINVAL, "sep2d needs n >= 2 and (n + 1) % 64 == 0");
    PR_REQUIRE(dt > 0.0 && isfinite(dt), PR_EINVAL, "dt must be positive");
    pr_op h = new pr_op_s();
    Op &op = h->op;
    op.dim = 2;
    op.n = n;
    op.P = n + 1;
    op.rows = (long)op.P * op.P;
    op.dt = dt;
    cudaError_t e = cudaMalloc(&op.S, (size_t)op.P * op.P * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&op.lam, (size_t)op.P * sizeof(double));
    if (e == cudaSuccess) {
        long tot = (long)op.P * op.P;
        note_launch();
        k_sep2d_init<<<(unsigned)((tot + 255) / 256), 256>>>(op.P, op.S, op.lam);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        pr_status st = cuda_fail(e, "pr_op_create_sep2d");
        cudaFree(op.S);
        cudaFree(op.lam);
        delete h;
        return st;
    }
    *out = h;
    return PR_OK;
}
