// pr_internal.cuh -- shared internals of libpr (the CUDA path; no oracle code).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/pr.h"

namespace pr {

// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);
pr_status cuda_fail(cudaError_t e, const char *where);

#define PR_CUDA(call)                                         \
    do {                                                      \
        cudaError_t _e = (call);                              \
        if (_e != cudaSuccess) return ::pr::cuda_fail(_e, #call); \
    } while (0)

#define PR_CHECK_LAUNCH(where)                                \
    do {                                                      \
        cudaError_t _e = cudaGetLastError();                  \
        if (_e != cudaSuccess) return ::pr::cuda_fail(_e, where); \
    } while (0)

#define PR_REQUIRE(cond, code, msg)                           \
    do {                                                      \
        if (!(cond)) { ::pr::set_error(msg); return code; }   \
    } while (0)

// -------------------------------------------------------- device workspace
// Grow-only caching allocator: buffers returned by ws_free go back to a
// size-keyed free list and are reused (no cudaFree/cudaMalloc, hence no
// implicit device synchronisation, in repeated builds / Parareal runs).
// Stream-ordered: a block freed on stream s1 and reused on s2 makes s2 wait for
// an event recorded at the free (no host synchronisation).
void *ws_alloc(size_t bytes, cudaStream_t s);
void ws_free(void *p, cudaStream_t s);

// Diagnostic switches from the environment (PR_NO_PART, PR_NO_SRC_BASIS, PR_NO_XTY_RM,
// PR_NO_TRSM_DMMA, PR_NO_RINV_CM, PR_NO_EXPAND_MMA select the alternate
// kernels that tests/test_gpu_alt_paths.py exercises; PR_PART_H, PR_STEPPER_PD,
// PR_STEPPER_VPT force a launch shape; PR_PART_PROF, PR_QR_TRACE,
// PR_DEBUG_SYNC print diagnostics).  Read once per process and again on
// pr_reload_env(), never per launch.
struct Flags {
    bool no_part = false, no_xty_rm = false, no_trsm_dmma = false, no_rinv_cm = false,
         no_expand_mma = false, part_prof = false, qr_trace = false, debug_sync = false;
    bool part_vpt2 = false, no_src_basis = false;
    int part_h = 0, stepper_pd = 0, stepper_vpt = 0;
    int part_idle_ns = -1;       // PR_PART_IDLE_NS: interface-warp poll back-off (dev aid; -1 = default)
    bool part_nopersist = false; // PR_PART_NOPERSIST: one K1P cluster per vector group (no staging reuse)
    bool part_nodm = false;      // PR_PART_NODM: K1P TM variants solve the CTA-local interface system with the banded solver warps instead of the FP64 tensor-core product
    bool part_notmem = false;    // PR_PART_NOTMEM: K1P keeps {nl, w} in shared memory instead of tensor memory
    bool part_noiface = false;   // PR_PART_NOIFACE: K1P sweeps without the interface (timing aid; wrong results)
};
const Flags &flags();

// Number of SMs of the current device (cached).
int num_sms();

// Counters (pr_counters): every kernel launch of the library, and CUDA-event
// timing of the stepper launches when profiling is enabled.
void note_launch();
bool profiling();
void stepper_timed_begin(cudaStream_t s);
void stepper_timed_end(cudaStream_t s, double dof_steps, double flops);

// ---------------------------------------------------------------- operator
struct Coef {             // one row of a fused stepper pass (32 B, aligned)
    double a, b, c, d;
};

struct Op {
    int dim = 1;
    int n = 0;            // interior points per side
    long rows = 0;        // storage rows of one vector
    double dt = 0.0;
    // 1D: pass coefficients for I + dt A (fw) and (I + dt A)^T (tr).
    //   DN[i] = {ap_i, w_i, ga_i, 0}: down pass = UL back-substitution then LU forward
    //   UP[i] = {cp_i, wt_i, gc_i, 0}: up pass   = LU back-substitution then UL forward
    Coef *dn_fw = nullptr, *up_fw = nullptr, *dn_tr = nullptr, *up_tr = nullptr;
    // 1D partitioned stepper (k_part.cu, small batches): P = CL * W chunks of
    // L rows (rows >= n: identity padding).  rowc: (P*L) x 8 per-row
    // {w, nl, V2/d, W2/d, V, W, d, 1/d} (scaled form, k_part.cu); ctad: CL x PART_CTAD
    // per-CTA interface data.
    int part_P = 0, part_L = 0, part_CL = 0, part_K = 0;
    double *part_rowc_fw = nullptr, *part_ctad_fw = nullptr;
    double *part_rowc_tr = nullptr, *part_ctad_tr = nullptr;
    // time-dependent pencil (k_pencil.cu, pr_op_create_pencil): per-step factors
    // of L_g = M + dt A(t_g) (pen_nsteps x n Coef {w, ga, cp, gt}) and the mass
    // matrix M (3n: sub | diag | sup) or null (M = I)
    int pencil = 0, pen_nsteps = 0;
    Coef *pen_fac = nullptr;
    double *pen_m = nullptr;
    // weighted view (pr_op_create_weighted): propagation in the coordinates
    // u^ = C u of the mass-matrix inner product, M = C^T C (C upper bidiagonal:
    // wC = diag (n) | super (n)); shares every other array with its base op
    int weighted = 0;
    double *wC = nullptr;
    // 2D: P = n+1; S (P x P) sine matrix with zero row/col 0; lam[P] eigenvalues of T.
    int P = 0;
    double *S = nullptr;
    double *lam = nullptr;
};

// --------------------------------------------------------------- kernels
struct StepArgs {
    int n;
    long B;
    int m;
    const Coef *DN;
    const Coef *UP;
    const double *in;  long ld_in;     // null -> zero input
    double *out;       long ld_out;
    const double *off; long ld_off;    // null -> no offset
    int sketch;                        // 1 -> input is Omega (Philox)
    unsigned long long seed;
    int q0;                            // first interval
    int vpi;                           // vectors per interval
    // step numbering (time-dependent pencils only): step j (1-based) of this
    // launch is global step q*mstride + step0 + j (mstride 0: = m)
    int step0;
    int mstride;
    // source (PR_SRC_SEP1D) -- R == 0: none
    int R;
    const double *spaceT;              // (n x stepper_rs(R)) row-major, zero-padded transpose
    const double *time;                // (R x nsteps)
    const double *amp;                 // (S x R)
    int nsteps;
    int nsrc;
    double dt;
};

cudaError_t launch_factor_1d(int n, const double *subA, const double *supA, const double *rsA,
                             const double *diagA, double dt, int transpose, Coef *DN, Coef *UP,
                             int *bad, cudaStream_t s);
cudaError_t launch_stepper_1d(const StepArgs &a, cudaStream_t s);
// time-dependent pencil stepper (k_pencil.cu)
cudaError_t launch_pencil_factor(int n, int nsteps, const double *lsub, const double *ldiag,
                                 const double *lsup, const double *lrs, Coef *fac, int *bad,
                                 cudaStream_t s);
cudaError_t launch_stepper_pencil(const Op &op, int mode, const StepArgs &sa, cudaStream_t s);
// y = C x, C^T x, C^{-1} x, C^{-T} x for B vectors (op layout, row stride rs,
// vector stride vs; in == out allowed; in == null: zero input); C upper
// bidiagonal {diag, super} (k_pencil.cu)
enum { BIDIAG_C = 0, BIDIAG_CT = 1, BIDIAG_CINV = 2, BIDIAG_CTINV = 3 };
cudaError_t launch_bidiag(int mode, int n, const double *cdiag, const double *csup, long B, const double *in,
                          long irs, long ivs, double *out, long ors, long ovs, cudaStream_t s);

// partitioned stepper (k_part.cu): configuration for n (false: not supported),
// setup (ends: P x 8 scratch), selection and launch
constexpr int PART_KMAX = 32;                  // chunks per CTA
constexpr int PART_CLMAX = 16;                 // CTAs per cluster
constexpr int PART_CTAD = 5 * 2 * PART_KMAX + 14 * PART_KMAX + 4 * PART_CLMAX;
// dense inverse of a CTA's local interface matrix (M = 32 unknowns: K = 16 chunks),
// row-major, stored behind the CL x PART_CTAD interface data (k_part.cu, DM variant)
constexpr int PART_MINV = 32 * 32;
constexpr int PART_ROWC = 8;                   // doubles per row of the K1P row data
constexpr int PART_ENDS = 8;                   // doubles per chunk of the K1P end data
// P = CL * K chunks of L rows (K chunks per CTA)
bool part_config(int n, int &P, int &L, int &CL, int &K);
cudaError_t launch_part_setup(int n, int P, int L, int CL, int K, const double *subA, const double *supA,
                              const double *rsA, const double *diagA, double dt, int transpose, double *rowc,
                              double *ctad, double *ends, int *bad, int *noscale, cudaStream_t s);
bool part_preferred(const Op &op, long B, int m);
cudaError_t launch_stepper_part(const Op &op, const StepArgs &a, int transpose, cudaStream_t s);
// scale == 0: out = Omega; else out += scale * (independent N(0,1) field, counter word 3 = ctr3)
cudaError_t launch_sketch(int dim, int n, long rows, int q0, int nint, int l,
                          unsigned long long seed, double *out, long rs, long vs, cudaStream_t s,
                          double scale = 0.0, unsigned long long ctr3 = 0ULL);
cudaError_t launch_transpose(const double *in, int R, int n, double *out, int ldo, cudaStream_t s);
int stepper_rs(int R);   // source-term count padded to 1, 2, 4 or 8

// Tall-skinny cross products: for batch b, chunk t of rows,
//   part[((b*nchunk + t)*a + i)*c + j] = sum_{rows in chunk} X_b[row, i] * Y_b[row, j]
// with X_b[row, i] = X[b*xbs + row*xrs + i*xcs] (likewise Y).
struct XtY {
    const int *skip;                  // nullable: batch b skipped when skip[b] == 2 (QR done)
    const double *X; long xbs, xrs, xcs; int a;
    const double *Y; long ybs, yrs, ycs; int c;
    long rows;
    int nbatch;
    int nchunk;
    long chunk_rows;
    double *part;                     // (nbatch, nchunk, a, c + c2)
    const double *Y2 = nullptr;       // optional: columns [c, c + c2) from Y2 (Y's strides)
    int c2 = 0;
    int diff = 0;                     // 1: the right operand is Y2 - Y (c columns, c2 == 0)
};
cudaError_t launch_xty(const XtY &p, cudaStream_t s);
// partials of X^T (Y2 - Y) (pcols = 0) on the row-major DMMA path, else of X^T [Y | Y2] (pcols = c)
cudaError_t launch_xty_diff(XtY p, const double *Y2, int c, int &pcols, cudaStream_t s);
int xty_chunks(long rows, int nbatch);

// out[(b*a + i)*c + j] = scale_i(b) * sum_t part[...]  (fixed order over t)
cudaError_t launch_reduce_parts(const double *part, int nbatch, int nchunk, int a, int c,
                                const double *rowscale, long rowscale_bs, double *out,
                                cudaStream_t s);

// CholeskyQR control: per interval state machine + shifted Cholesky.
struct CholArgs {
    const double *part; int nchunk;   // Gram partials
    int nbatch; int l; long nrows;    // nrows: rows of the block (shift formula)
    int *state;                       // per batch: 0 shift phase, 1 one plain pass done, 2 done
    int *act;                         // per batch: 0 nothing, 1 apply R by substitution, 2 apply Rinv (GEMM)
    double *R;                        // per batch l x l (upper) for this pass
    double *Rtot;                     // per batch l x l accumulated product (nullable)
    int *active;                      // device counter of batches still active
    int *fail;                        // device flag: Cholesky broke down
    double *offI = nullptr;           // optional per-batch ||G - I||_F of this pass (debug)
    double *shift_dbg = nullptr;      // optional per-batch final shift / ||G||_F and attempts (debug)
    double *Rinv = nullptr;           // per batch l x l: R^{-1} written for unshifted passes (act = 2)
    int pass = 0, max_pass = 1 << 30; // this pass (1-based) and the cap: a batch still active after it fails
    int *passes = nullptr;            // device: max pass index in which some batch was still active
};
cudaError_t launch_chol(const CholArgs &a, cudaStream_t s);
cudaError_t launch_trsm(double *Q, long bs, long rs, long cs, long rows, int l, int nbatch,
                        const double *R, const int *act, cudaStream_t s);
// Q <- Q Rinv (upper triangular) for batches with act == 2, DMMA tiles
cudaError_t launch_rinv_apply(double *Q, long bs, long rs, long cs, long rows, int l, int nbatch,
                              const double *Rinv, const int *act, cudaStream_t s);

cudaError_t launch_jacobi(const double *Rtot, int nbatch, int l, double *Psi, double *sigma,
                          double *Phi, int *fail, cudaStream_t s);
// per batch b: X_b^T with A_b X_b = R_b^T (A, R, out: l x l row-major; R upper),
// Gaussian elimination with partial pivoting in shared memory; *fail on a
// zero pivot
cudaError_t launch_lu_solve_rt(const double *A, const double *R, int nbatch, int l, double *XT, int *fail,
                               cudaStream_t s);

// out_b[row, r] = sum_j X_b[row, j] * C_b[j, r]  (j < l, r < k); out is (nbatch, rows, k)
cudaError_t launch_lift(const double *X, long xbs, long xrs, long xcs, long rows, int l,
                        const double *Cm, int ldc, int k, int nbatch, double *out,
                        cudaStream_t s);

// sequential reduced sweep: e_j = C_j e_{j-1} + d_j, j = 0..N-1 (C_0 unused:
// e_{-1} = 0).  All (k x S) row-major per interval.
cudaError_t launch_sweep(const double *C, const double *d, int N, int k, int S, double *e,
                         cudaStream_t s);
// d_b = Sigma_b (q_b - p_b) from X^T Y partials with columns [p (pcols = S or 0) | q (S)]
cudaError_t launch_reduce_pq(const double *part, int nbatch, int nchunk, int k, int S, int pcols,
                             const double *sigma, long sbs, double *d, cudaStream_t s);

// expand: out[row, v] = base[row, v] + sum_r U_b[row, r] e_b[r, s]  for interval b,
// source s, vector v = b*S + s (vector offsets in the out/base arrays given by
// vbs), with optional partial squared norms of (new - old).
struct Expand {
    double *out; long ors, ovs;       // element (row, vec) at out[row*ors + vec*ovs]
    const double *base; long brs, bvs;  // nullable
    const double *U; long Ubs;        // U_b[row, r] at U[b*Ubs + row*k + r]
    const double *e;                  // (nbatch, k, S)
    int k, S, nbatch;
    long rows;
    int nchunk; long chunk_rows;
    double *normpart;                 // nullable: (nbatch*S, nchunk)
    // general strides (k_expand_mma only; 0 = the defaults above): U row stride,
    // e row / batch strides, per-batch element offset of out (default b*S*ovs)
    long Urs = 0, ers = 0, ebs = 0, obs = 0;
};
cudaError_t launch_expand(const Expand &a, cudaStream_t s);
// out[v] = sqrt(sum_t part[v*nchunk + t])
cudaError_t launch_norm_finish(const double *part, int nvec, int nchunk, double *out,
                               cudaStream_t s);
// plain squared-norm partials of vectors (op layout)
cudaError_t launch_vecnorm_parts(const double *X, long rs, long vs, long rows, int nvec,
                                 int nchunk, long chunk_rows, double *part, cudaStream_t s);
cudaError_t launch_eye(double *R, int nbatch, int l, cudaStream_t s);
cudaError_t launch_copy_vectors(const double *in, long irs, long ivs, double *out, long ors,
                                long ovs, long rows, int nvec, cudaStream_t s);

// ------------------------------------------------------------ communicator
// (pr_comm.cu)  All operations are stream-ordered on s; see include/pr.h.
struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() {}
    // rank r sends `bytes` from send to rank r+1's recv (rank 0's recv untouched)
    virtual pr_status shift_right(const void *send, void *recv, size_t bytes, cudaStream_t s) = 0;
    // recv = concatenation of every rank's `bytes` of send, in rank order
    virtual pr_status all_gather(const void *send, void *recv, size_t bytes, cudaStream_t s) = 0;
    // elementwise max over ranks of count doubles, in place
    virtual pr_status all_reduce_max(double *buf, int count, cudaStream_t s) = 0;
    // concatenation of counts[r] elements (elem bytes each) of every rank r
    pr_status all_gather_v(const void *send, void *recv, const long *counts, size_t elem, cudaStream_t s);
};
Comm *comm_of(pr_comm h);

// contiguous block partition of total units over world ranks: (start, count) of rank
inline void shard_of(long total, int rank, int world, long &start, long &count)
{
    const long base = total / world, rem = total % world;
    start = rank * base + (rank < rem ? rank : rem);
    count = base + (rank < rem ? 1 : 0);
}

// 2D separable stepper (k_sep2d.cu)
struct Sep2dArgs {
    const Op *op;
    int mode;            // PR_LINEAR / PR_ADJOINT / PR_AFFINE
    int q0, m, B, vpi;
    const pr_source *f;
    const double *in; long ld_in;
    double *out; long ld_out;
    const double *off; long ld_off;
};
pr_status run_sep2d(const Sep2dArgs &a, cudaStream_t s);

}  // namespace pr

// ------------------------------------------------------------- handles
struct pr_op_s {
    pr::Op op;
    bool view = false;     // a weighted view: owns only op.wC
};

struct pr_coarse_s {
    int N_total = 0, first = 0, nloc = 0, m = 0, k = 0, p = 0, l = 0;
    long rows = 0;
    int dim = 1;
    double *U = nullptr;       // (nloc, rows, k)
    double *V = nullptr;       // (nloc, rows, k)
    double *sigma = nullptr;   // (nloc, l)
    double *C = nullptr;       // (nloc, k, k): C_q = Sigma_q V_q^T U_{q-1} (q >= first+1)
    int *fail = nullptr;       // device flags [0]: qr, [1]: svd
    int qr_passes[2] = {0, 0};
    cudaStream_t stream = nullptr;   // stream of the last call that used the handle (destroy is ordered on it)
    pr_comm comm = nullptr;          // the communicator the handle was built with (not owned)
    int rank = 0, world = 1;
    double *de = nullptr;            // device [delta, eps]: max over ALL ranks' intervals
    double *C_all = nullptr;         // (N_total, k, k) sweep matrices of all intervals (== C at world 1)
};
