/* pr.h -- C ABI of the B200-native spectral-coarse-solver Parareal hot path.
 *
 * Gander, Ohlberger, Rave, "A Parareal Algorithm with Spectral Coarse Solver"
 * (arXiv 2508.08873).  Citations "P:n" are lines of the paper's LaTeX source
 * (reference/PAPER.md); "§" are its sections.
 *
 * The library computes, on one GPU, for the time intervals it owns:
 *   - the fine solver F_n (backward Euler), its linear part F_n',
 *     the adjoint F_n'^* and offsets b_n = F_n 0 (eq. F_n_affine,
 *     P:162-167)                                       -> pr_fine_propagate
 *   - the randomized SVD of F_n' (§2.1 steps 1-6) giving the
 *     spectral coarse solvers G_n' = U_n Sigma_n V_n^T (eq. spectral_G,
 *     P:186-195)                                       -> pr_build_coarse
 *   - the Parareal iteration (eq. def_Parareal) with the update
 *     norms of the a posteriori bound      -> pr_parareal
 *   - the a priori / a posteriori bounds -> pr_bounds
 *
 * Conventions (all functions):
 *   - Every call returns pr_status; PR_OK = 0.  No call aborts the process.
 *     pr_last_error() returns a thread-local message for the last failure.
 *   - Arguments are validated before any launch: a PR_EINVAL / PR_EDIM call
 *     writes nothing.  After PR_ENOCONV / PR_ECUDA outputs are undefined.
 *   - `double*` buffers are owned by the caller.  Unless stated "host", they
 *     are device pointers (e.g. torch CUDA tensors).  Handles (pr_op,
 *     pr_coarse) are owned by the library and freed only by *_destroy.
 *   - Work is enqueued asynchronously on the caller's `stream` (a
 *     cudaStream_t passed as void*; NULL = legacy default stream), except
 *     functions documented as synchronizing.
 *   - Interval indices are 0-based: q = n - 1 for the paper's interval n,
 *     covering (t_q, t_{q+1}] = (q*m*dt, (q+1)*m*dt].
 *   - Floating point is fp64 throughout.
 *
 * Vector storage ("op layout"), chosen by the operator:
 *   1D (pr_op_create_tridiag): `rows` = n.  A batch of B vectors is a
 *     row-major (n x ld) array with the vector index fastest: element (i, c)
 *     at U[i*ld + c], ld >= B.  (Coalesced across vectors for the stepper.)
 *   2D (pr_op_create_sep2d, n x n interior grid): `rows` = (n+1)^2.  Vector c
 *     is contiguous at U[c*ld + ix*(n+1) + iy], ld >= (n+1)^2, where ix, iy in
 *     0..n and index 0 is the (zero) Dirichlet ghost row/column; interior
 *     point (ix, iy) >= 1 sits at x = ix*h, y = iy*h, h = 1/(n+1).  Ghost
 *     entries of inputs must be 0; outputs keep them 0.
 */
#ifndef PR_H
#define PR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PR_OK = 0,
    PR_EINVAL = 1,     /* bad argument (null pointer, negative size, bad mode)   */
    PR_EDIM = 2,       /* dimension mismatch between arguments and handles        */
    PR_ESINGULAR = 3,  /* zero/negative pivot in an operator factorization        */
    PR_ENOCONV = 4,    /* CholeskyQR or Jacobi SVD did not converge               */
    PR_EUNAVAIL = 5,   /* quantity not available (e.g. eps needs p >= 1)          */
    PR_EOOM = 6,       /* device allocation failed                                */
    PR_ECUDA = 7,      /* CUDA runtime error (message in pr_last_error)           */
    PR_ENCCL = 8       /* NCCL missing or failed (message in pr_last_error)       */
} pr_status;

const char *pr_last_error(void);
int pr_version(void);

/* Re-read the PR_* diagnostic environment switches (DESIGN.md "Diagnostic
 * switches"; they select alternate kernels or print probes).  The library reads
 * them once, at its first call; a test that changes them calls this.  Host
 * only, never fails. */
pr_status pr_reload_env(void);

/* Instrumentation.  pr_profile(1) brackets every fine-propagation launch
 * (1D: the K1 stepper kernel; 2D: the K2 GEMM passes of one call) with CUDA
 * events on its stream.  pr_counters (host; synchronises on the recorded
 * events) returns the number of kernels the library has launched, and the
 * number, summed device time (ms), DOF-steps (n_dof * B * m) and tensor-core
 * flops (2D: 2 P^3 per vector per GEMM pass; 1D: 0) of the timed launches
 * since the last reset; reset != 0 clears them afterwards.  All output
 * pointers may be NULL. */
pr_status pr_profile(int enable);
pr_status pr_counters(int reset, long *kernel_launches, long *stepper_launches, double *stepper_ms,
                      double *stepper_dof_steps, double *stepper_flops);

/* The same timed fine-propagation launches split by the phase that issued
 * them (SURVEY §8(d) "Definitions": build fwd+adj, offsets b_n, Parareal
 * iterations): arrays of PR_NPHASES entries (host, nullable), indexed by
 * PR_PHASE_*.  reset != 0 clears the timed launches afterwards. */
enum { PR_PHASE_DIRECT = 0, PR_PHASE_BUILD = 1, PR_PHASE_OFFSETS = 2, PR_PHASE_ITERATION = 3, PR_NPHASES = 4 };
pr_status pr_phase_counters(int reset, long *launches, double *ms, double *dof_steps);

typedef struct pr_op_s *pr_op;
typedef struct pr_coarse_s *pr_coarse;
typedef struct pr_comm_s *pr_comm;

/* -------------------------------------------------------------- distribution
 * The path shards by time interval (the paper runs one MPI rank
 * per interval group): rank r of `world` owns the contiguous block
 * of intervals shard(N, r, world) = (first, n_local), first = r*floor(N/world)
 * + min(r, N % world).  Only interval-boundary data crosses ranks: one
 * boundary block per sweep to the right neighbour, the
 * k-dimensional reduced sweep data of all intervals (all-gather), and the
 * max-reductions of delta and eps (eq. bounds_delta_eps).  A
 * pr_comm carries them, stream-ordered on the caller's stream.
 *
 * pr_comm_nccl_unique_id: 128-byte NCCL id (host), made on rank 0 and handed to
 *   every rank by the caller (e.g. a torch.distributed broadcast).
 * pr_comm_create_nccl: one process per GPU (the current device); NCCL is loaded
 *   at run time (libnccl.so.2 already in the process, else the system's).
 *   Collective: every rank calls it.  Errors: EINVAL, ENCCL.
 * pr_comm_create_local: `world` virtual ranks in ONE process on the current
 *   GPU; out[r] (host array of world handles) is rank r.  Each rank must be
 *   driven by its own host thread (calls on different ranks meet at host
 *   barriers) with its own stream; data moves by device-to-device copies
 *   ordered with CUDA events.  For running the sharded schedule with more
 *   ranks than GPUs (tests).  Errors: EINVAL.
 * A communicator must outlive every handle built with it. */
pr_status pr_comm_nccl_unique_id(void *id);
pr_status pr_comm_create_nccl(int rank, int world, const void *id, pr_comm *out);
pr_status pr_comm_create_local(int world, pr_comm *out);
pr_status pr_comm_info(pr_comm c, int *rank, int *world);
pr_status pr_comm_destroy(pr_comm c);

/* ------------------------------------------------------------------ operator */

/* 1D operator: A = tridiag(sub, diag, sup) (host arrays of length n; sub[0]
 * and sup[n-1] ignored), semi-discretisation u_t = -A u + f.  The fine step is
 * (I + dt A) u_{j+1} = u_j + dt f(t_{j+1}).  rowsum / colsum
 * (host, length n, may be NULL) are the exact row / column sums of A: when
 * given, the LU and UL pivots of I + dt A are computed from them (DESIGN.md
 * reading R-ACC: relative accuracy independent of dt/h^2 for diagonally
 * dominant M-matrices); when NULL they are formed as sub+diag+sup.  The
 * factorizations (the whole-vector LU/UL pair and, for 64 <= n <= 16384, the
 * partitioned-stepper chunk LUs, spikes and interface factors, both built
 * from row sums) run once, in device kernels.  Synchronizing.
 * Errors: EINVAL (n < 2, dt <= 0, null arrays), ESINGULAR (pivot <= 0 or
 * non-finite), EOOM, ECUDA. */
pr_status pr_op_create_tridiag(int n, const double *sub, const double *diag, const double *sup,
                               const double *rowsum, const double *colsum, double dt,
                               pr_op *out);

/* Time-dependent 1D pencil: step g = 1..nsteps
 * (global, g = q*m + j) solves
 *     (M + dt A(t_g)) u_g = M u_{g-1} + dt l(t_g)
 * with its own tridiagonal left-hand side L_g = M + dt A(t_g): lsub / ldiag /
 * lsup are host arrays of nsteps x n (row-major by step; lsub[g*n] and
 * lsup[g*n + n-1] ignored).  Exp 2's conductivity kappa(x, t) =
 * 1 + 0.9 sin(7 pi t + 2 pi x) with Neumann boundary rows (eq.
 * ex2) gives L_g that differ per step, so the interval operators F_q' are not
 * normal; a non-symmetric A (advection) is allowed too.  lrowsum
 * (host, nsteps x n, may be NULL): exact row sums of L_g, for the R-ACC pivots
 * (requires L_g to be an M-matrix).  msub / mdiag / msup (host, length n,
 * all NULL for M = I): the mass matrix of linear finite elements.
 * l(t) enters through the PR_AFFINE source (the caller passes the assembled
 * load vectors as `space`).  The adjoint PR_ADJOINT is the Euclidean
 * transpose of the product, steps in reverse order:
 *     F_q'^T = (M^T L_{q,1}^{-T}) ... (M^T L_{q,m}^{-T})      (reading R-ADJ).
 * Fine propagation over intervals q with (q+1)*m > nsteps fails with EDIM.
 * All steps are factored once, on the device (k_pencil.cu).  Synchronizing.
 * Errors: EINVAL (n < 2, nsteps < 1, dt <= 0, NULL step arrays, partial M),
 * ESINGULAR (zero / non-finite pivot, or non-positive in row-sum form), EOOM,
 * ECUDA. */
pr_status pr_op_create_pencil(int n, int nsteps, const double *lsub, const double *ldiag,
                              const double *lsup, const double *lrowsum, const double *msub,
                              const double *mdiag, const double *msup, double dt, pr_op *out);

/* Weighted view of a pencil with a mass matrix: the
 * operator in the coordinates u^ = C u of the inner product (u, v)_M = u^T M v,
 * M = C^T C (Cholesky, C upper bidiagonal).  Its fine solver is
 * F^ = C F C^{-1}; the Euclidean SVD of F^' IS the generalized SVD of F'
 * with respect to (.,.)_M of eq. svd (sigma equal, psi = C^{-1} psi^,
 * phi = C^{-1} phi^), and F^'^T = C^{-T} F'^T C^T is F'^* = M^{-1} F'^T M in
 * these coordinates (reading R-WIP).  So pr_build_coarse / pr_parareal /
 * pr_bounds on the view run the paper's method in the M inner product
 * (Exp 1's L^2 choice): states, coarse factors and update norms are
 * in u^ coordinates (||u^|| = ||u||_M); map with pr_op_weight_apply.  The view
 * shares the base's device arrays: destroy it before the base.  Errors: EINVAL
 * (not a pencil with M), ESINGULAR (M not SPD), ECUDA. */
pr_status pr_op_create_weighted(pr_op base, pr_op *out);
enum { PR_TO_WEIGHTED = 0, PR_FROM_WEIGHTED = 1 };
/* Y = C X (PR_TO_WEIGHTED) or C^{-1} X (PR_FROM_WEIGHTED) for B vectors (1D
 * layout; X == Y allowed).  Asynchronous.  Errors: EINVAL, EDIM. */
pr_status pr_op_weight_apply(pr_op view, int direction, int B, const double *X, long ldx, double *Y, long ldy,
                             void *stream);

/* 2D operator: 5-point Laplacian on the unit square with homogeneous
 * Dirichlet conditions, n x n interior points, A = T (x) I + I (x) T,
 * T = tridiag(-1, 2, -1)/h^2.  Solved in the sine eigenbasis of T (DESIGN.md
 * "K2").  Synchronizing.  Errors: EINVAL (n < 2, (n+1) % 64 != 0, dt <= 0). */
pr_status pr_op_create_sep2d(int n, double dt, pr_op *out);

pr_status pr_op_destroy(pr_op op);

/* Storage rows of one vector (n in 1D, (n+1)^2 in 2D), spatial dimension, n. */
pr_status pr_op_info(pr_op op, long *rows, int *dim, int *n);

/* -------------------------------------------------------------------- source */
enum { PR_SRC_NONE = 0, PR_SRC_SEP1D = 1, PR_SRC_BUMP2D = 2 };

/* Host-sampled separable source term (device pointers):
 *   PR_SRC_SEP1D:  f_s(x_i, t_g) = sum_r amp[s*nterms + r] * space[r*n + i] * time[r*nsteps + g-1]
 *   PR_SRC_BUMP2D: f(x_ix, y_iy, t_g) = sum_b gx[(b*nsteps + g-1)*(n+1) + ix] * gy[(b*nsteps + g-1)*(n+1) + iy]
 *                  (index 0 of gx/gy is the ghost and must be 0)
 * g = q*m + j is the global step (1-based) of step j of interval q; the
 * source of step g is evaluated at t_g = g*dt (reading Z3). */
typedef struct {
    int kind;
    int nterms;          /* R (1D terms) or number of bumps (2D), 1..8            */
    int nsrc;            /* number of independent sources S (1D); 1 for 2D        */
    int nsteps;          /* length of the time axis (>= (last interval+1)*m)      */
    const double *space; /* 1D */
    const double *time;  /* 1D */
    const double *amp;   /* 1D */
    const double *gx;    /* 2D */
    const double *gy;    /* 2D */
} pr_source;

/* ---------------------------------------------------------- fine propagation */
enum { PR_LINEAR = 0, PR_ADJOINT = 1, PR_AFFINE = 2 };

/* m backward-Euler steps of interval q = first_interval + c / vecs_per_interval
 * applied to each of the B vectors c of U_in (op layout, stride ld_in):
 *   PR_LINEAR:  U_out = F_q' U_in                 (no source)
 *   PR_ADJOINT: U_out = F_q'^* U_in               (transposed steps, reverse order)
 *   PR_AFFINE:  U_out = F_q U_in = F_q' U_in + b_q (source f; vector c uses
 *               source c % f->nsrc; eq. F_n_affine)
 * U_in == NULL means a zero input (so PR_AFFINE gives b_q).  offset (nullable,
 * op layout, stride ld_off) is added to the result: F' u + b_q from a stored
 * b_q.  U_in may equal U_out (in place) when ld_in == ld_out.
 * Each step (I + dt A) x = r is solved exactly (up to rounding order): for a
 * 1D op with 64 <= n <= 16384 by the partition method over a thread-block
 * cluster with the state in registers (k_part.cu, reading R-PART),
 * otherwise by the fused LU/UL stepper; 2D ops in the sine eigenbasis.
 * Errors: EINVAL (mode, m < 0, B < 0, vecs_per_interval < 1, missing source
 * for PR_AFFINE with f->kind mismatched to the op), EDIM (ld too small). */
pr_status pr_fine_propagate(pr_op op, int mode, int first_interval, int m, int B,
                            int vecs_per_interval, const pr_source *f,
                            const double *U_in, long ld_in, double *U_out, long ld_out,
                            const double *offset, long ld_off, void *stream);

/* The Gaussian test vectors of rSVD step 1: Omega_q (rows x l)
 * for intervals q = first_interval .. first_interval + n_intervals - 1 into
 * out (op layout, vector (q - first_interval)*l + c, stride ld).  Philox4x64-10,
 * key (seed, 0), counter (i/4, c, q, 0), Box-Muller (reading R-RNG);
 * 2D numbers interior DOFs i = (ix-1)*n + (iy-1).  pr_build_coarse generates
 * the same values fused into its first stepper pass; this entry exists so the
 * generator can be checked on its own. */
pr_status pr_gaussian_sketch(pr_op op, int first_interval, int n_intervals, int l, uint64_t seed,
                             double *out, long ld, void *stream);

/* ------------------------------------------------------------ coarse solvers */

/* Randomized SVD of F_q' for q = first_interval .. first_interval
 * + n_local - 1 of N_total intervals, rank k, oversampling p (l = k + p <= 112,
 * l <= rows; 112 because the one-CTA Jacobi SVD of step 5 keeps two l x l
 * fp64 matrices in shared memory, 2 * 112^2 * 8 B = 196 KB of the 227 KB):
 *   1. Y = F_q' Omega_q, Omega as pr_gaussian_sketch
 *   2. W = orth(Y)      iterated shifted CholeskyQR (reading Z7)
 *   3. Z = F_q'^* W
 *   4. V R_Z = Z        (same orthonormalisation, R_Z accumulated)
 *   5. M = R_Z^T (= (F'^* w_i, v_j)), M = Psi Sigma Phi^T by one-sided Jacobi;
 *      psi_r = W Psi_r, phi_r = V Phi_r (swapped reading of P:293-294, Z5)
 *   6. keep r <= k.
 * comm (nullable): with a communicator, first_interval / n_local are ignored
 * and the rank's block shard(N_total, rank, world) is built; the handle keeps
 * comm (which must outlive it), receives U_{first-1} from the left neighbour
 * for its first sweep matrix, and holds delta / eps reduced over all ranks and
 * the sweep matrices C_q of all intervals (for pr_parareal).
 * Seeds depend only on (seed, q, column) and every reduction's chunking only
 * on N_total, so results are bit-identical for any sharding.  The handle also
 * holds the reduced sweep matrices C_q = Sigma_q V_q^T U_{q-1} (DESIGN.md
 * "reduced sweep").  Intervals are processed in chunks whose scratch fits
 * min(16 GiB, 40% of free memory), so scratch does not grow with n_local.
 * Asynchronous (no host synchronisation: the CholeskyQR pass loop is
 * controlled on the device, at most 24 passes); errors detected on the device
 * (no convergence) are reported by pr_coarse_info and pr_parareal.
 * opts (nullable = the paper's basic algorithm, both fields 0):
 *   power_iterations q (0..16): W = span{(F' F'^*)^q F' omega_i},
 *     evaluated as q rounds of orthonormalise / F'^* / orthonormalise / F'
 *     (same span; 2q more batched fine solves per interval);
 *   independent_adjoint (0/1): step 3 applies F'^* to an independent Gaussian
 *     set Psi (Philox counter word 3 = 2) instead of w_1..w_l, so the forward
 *     and adjoint solves are independent; G' then comes from the
 *     two-sided sketch F' ~ W C V^T, C = (Psi^T W)^{-1} R_Z^T (Z = F'^* Psi =
 *     V R_Z), whose SVD replaces step 5's M.  Less accurate (the paper says so).
 * Errors: EINVAL, EDIM (l > 112 or l > rows), EOOM, ENCCL. */
typedef struct {
    int power_iterations;
    int independent_adjoint;
} pr_rsvd_opts;
pr_status pr_build_coarse(pr_op op, int N_total, int first_interval, int n_local, int m,
                          int k, int p, uint64_t seed, const pr_rsvd_opts *opts, pr_comm comm,
                          void *stream, pr_coarse *out);

/* A posteriori estimate of the coarse error ||F_q' - G_q'|| for every local
 * interval (the failure-probability estimator behind an adaptive choice of p,
 * P:305-310; Halko, Martinsson & Tropp, Lemma 4.1):
 *   est_q = 10 sqrt(2/pi) max_{i<=r} ||(F_q' - G_q') omega_i||,
 * omega_i fresh N(0,1) probes (Philox counter word 3 = 3); est_q >= the true
 * norm with probability >= 1 - 10^{-r}.  r batched fine solves per interval.
 * est_host: host, n_local.  Synchronizing.  Errors: EINVAL, EDIM, EOOM. */
pr_status pr_coarse_estimate(pr_coarse G, pr_op op, int r, uint64_t seed, double *est_host, void *stream);

/* Adaptive oversampling: build with p = p0, estimate the coarse
 * error (pr_coarse_estimate, r probes), and rebuild with p doubled until the
 * largest estimate over ALL intervals (all ranks) is <= tol or p reaches
 * p_max; *p_used is the p of the returned handle.  Errors: as pr_build_coarse,
 * plus EINVAL (p0 < 1, p_max < p0, tol <= 0, r < 1). */
pr_status pr_build_coarse_adaptive(pr_op op, int N_total, int first_interval, int n_local, int m, int k,
                                   int p0, int p_max, double tol, int r, uint64_t seed,
                                   const pr_rsvd_opts *opts, pr_comm comm, void *stream, pr_coarse *out,
                                   int *p_used);

/* Synchronizes with the stream of the handle's last call.  k, l, n_local,
 * first_interval, m; delta = max_q sigma_{q,1} and eps = max_q sigma_{q,k+1}
 * over ALL intervals (all ranks when built with a communicator; eq.
 * bounds_delta_eps; eps uses the computed sigma_{k+1});
 * sigma_host (nullable, host, n_local*l) the local computed singular values;
 * qr_passes (nullable, host, 2) the CholeskyQR pass counts of steps 2 and 4
 * (max over the local intervals).  Returns PR_ENOCONV if a QR or SVD failed to
 * converge on the device, and PR_EUNAVAIL for eps when p == 0 (eps = NaN). */
pr_status pr_coarse_info(pr_coarse G, int *k, int *l, int *n_local, int *first_interval, int *m,
                         double *delta, double *eps, double *sigma_host, int *qr_passes);

/* Device views of the factors: U and V are (n_local, rows, k) row-major
 * (U[(q*rows + i)*k + r]), sigma is (n_local, l).  Owned by the handle. */
pr_status pr_coarse_factors(pr_coarse G, const double **U, const double **V, const double **sigma);

/* Y = G_q' X = U_q Sigma_q V_q^T X for nvec probe vectors (op layout). */
pr_status pr_coarse_apply(pr_coarse G, int q_local, int nvec, const double *X, long ldx,
                          double *Y, long ldy, void *stream);

pr_status pr_coarse_destroy(pr_coarse G);

/* ----------------------------------------------------------------- Parareal */

/* Parareal (eq. def_Parareal) with nsrc independent sources
 * sharing G' (Remark affine_g_n), G_n = G_n' + b_n:
 *   b_q = F_q 0                                    (PR_AFFINE from zero)
 *   u^0_0 = u0, u^0_{q+1} = G_{q+1} u^0_q           (initialisation)
 *   u^{k+1}_{q+1} = F_{q+1} u^k_q + G'_{q+1} u^{k+1}_q - G'_{q+1} u^k_q
 * for K_iter iterations.  The fine solves of an iteration run as one batched
 * stepper launch (F' u + b_q); the sequential part runs in the reduced
 * coordinates e_q = C_q e_{q-1} + (q_q - p_q) of dimension k (DESIGN.md
 * "reduced sweep"; exact algebra, no approximation).
 * G either covers all intervals (built without a communicator) or is one
 * rank's shard (built with one): then this is a collective call of all ranks,
 * each computing its own intervals q0 .. q0+nq-1 (q0 = first_interval,
 * nq = n_local of pr_coarse_info), with one boundary block per half-iteration
 * sent to the right neighbour and the k x nsrc sweep data all-gathered.  The
 * result is bit-identical to the unsharded run.
 *   u0       device, nsrc vectors (op layout, stride ld_u0); read on rank 0
 *            only (may be NULL elsewhere)
 *   U_out    device, (nq+1)*nsrc vectors, vector i*nsrc + s = u^K_{q0+i} of
 *            source s (op layout, stride ld_out); block 0 is u_{q0} (u0 on
 *            rank 0); also the iteration state.
 *   upd_host host, nullable, K_iter x (N+1) x nsrc: ||u^k_j - u^{k-1}_j||,
 *            k = 1..K, all boundaries j (gathered from every rank)
 *   bnorm_host host, nullable, (N+1) x nsrc: ||b_j|| with b_0 := u0
 *   hist     device, nullable: if given, u^k (the (nq+1)*nsrc local vectors,
 *            same layout as U_out) is stored at hist + k*hist_stride, k = 0..K.
 * Synchronizing (at the end, to fill the host arrays).  Returns PR_ENOCONV
 * (outputs undefined) if the rSVD of G failed on the device.
 * Errors: EINVAL, EDIM (G not covering all intervals without a communicator,
 * source/op mismatch), ENOCONV, EOOM, ENCCL. */
pr_status pr_parareal(pr_coarse G, pr_op op, int nsrc, const double *u0, long ld_u0,
                      const pr_source *f, int K_iter, double *U_out, long ld_out,
                      double *upd_host, double *bnorm_host, double *hist, long hist_stride,
                      void *stream);

/* pr_parareal with the a posteriori stopping rule: iterate until the bound of
 * eq. apost_bound,
 *     max_{n, s} eps * sum_{m=1}^{n-1} delta^{n-m-1} ||u^k_m - u^{k-1}_m||,
 * with delta, eps of the coarse handle (eq. bounds_delta_eps, eps from the
 * computed sigma_{k+1}), is <= tol, or K_max iterations; *k_done
 * receives the number of iterations run (the arrays are filled for those).
 * One device-to-host read of the update norms per iteration.  Errors: as
 * pr_parareal, plus EINVAL (tol <= 0, k_done NULL) and EUNAVAIL (p == 0). */
pr_status pr_parareal_tol(pr_coarse G, pr_op op, int nsrc, const double *u0, long ld_u0,
                          const pr_source *f, int K_max, double tol, double *U_out, long ld_out,
                          double *upd_host, double *bnorm_host, double *hist, long hist_stride,
                          int *k_done, void *stream);

/* --------------------------------------------------------------- reporting
 * (SURVEY 8(f) row 3.)  Arrays of boundary blocks as in pr_parareal: block j
 * (nsrc vectors, op layout) belongs to t_j, j = 0..N. */

/* The sequential fine solution u_0 = u0, u_{q+1} = F_{q+1} u_q, q < N
 * (P:136-139): N dependent batched launches.  U_out: (N+1)*nsrc vectors. */
pr_status pr_sequential(pr_op op, int nsrc, const double *u0, long ld_u0, const pr_source *f, int N,
                        int m, double *U_out, long ld_out, void *stream);

/* The l2-in-space, max-in-time error of a Parareal iterate (the
 * numerator of eq. def_efficiency): u^k(t) on [t_{q-1}, t_q) is the fine
 * trajectory F_q started from u^k_{q-1} (and t = T the end of interval N's;
 * reading R-TRAJ), compared with the fine trajectory from u_{q-1}.  Evaluated
 * exactly as the LINEAR propagation of e_{q-1} = u^k_{q-1} - u_{q-1} (the
 * source cancels, eq. F_n_affine), m one-step launches with a norm after each.
 * U, Uref: (N+1)*nsrc vectors (same ld).  err_host (nsrc): max over t;
 * ivl_host (nullable, N*nsrc): the max over interval q+1 at [q*nsrc + s].
 * Synchronizing.  Errors: EINVAL, EDIM. */
pr_status pr_trajectory_error(pr_op op, int nsrc, int N, int m, const double *U, long ldU,
                              const double *Uref, long ldR, double *err_host, double *ivl_host,
                              void *stream);

/* Efficiency of the a posteriori estimator, eq. def_efficiency:
 *   eta^k = traj_err[k] / max_{1 <= n < N} eps sum_{m=1}^{n-1} delta^{n-m-1} upd_k[m]
 * for k = 1..K (host arrays, one source: upd as pr_parareal's K x (N+1),
 * traj_err K+1 values for k = 0..K, eta K values).  Host only. */
pr_status pr_efficiency(double delta, double eps, int N, int K, const double *upd,
                        const double *traj_err, double *eta);

/* Classical Parareal (eq. def_Parareal) with a coarse PROPAGATOR instead of
 * the spectral G (the baselines of P:157-158 and P:209-215, the dashed lines
 * of the paper's figures): G_{q+1} v = one backward-Euler step of `coarse`
 * (time step Delta T: its step q+1, source fc sampled at t_{q+1}), or G = 0
 * when coarse == NULL (u^0_q = 0 for q >= 1).  F_{q+1} = m steps of
 * op with source f.  The coarse sweep is sequential (N launches per
 * iteration).  upd_host (nullable, host, K x (N+1) x nsrc); hist as
 * pr_parareal.  Synchronizing.  Errors: EINVAL, EDIM. */
pr_status pr_parareal_classical(pr_op coarse, const pr_source *fc, pr_op op, int nsrc, const double *u0,
                                long ld_u0, const pr_source *f, int N, int m, int K_iter, double *U_out,
                                long ld_out, double *upd_host, double *hist, long hist_stride, void *stream);

/* ------------------------------------------------- distributed building blocks
 * Stages of pr_parareal on the intervals a handle owns (first .. first+n_local-1),
 * for an interval-sharded Parareal over several GPUs.  Arrays
 * hold "blocks" of nsrc vectors (op layout, stride ld): block i of an
 * input-side array belongs to boundary first+i (u_q, Fu_q), block i of an
 * output-side array to boundary first+i+1.  All device pointers, asynchronous. */

/* C_q = Sigma_q V_q^T U_{q-1} for the local q; for q = first, U_{first-1} is
 * U_prev (rows x k row-major, e.g. the left neighbour's last U block; NULL ->
 * C_first = 0, correct for first == 0).  pr_build_coarse already computes the
 * C_q that need no neighbour. */
pr_status pr_coarse_sweep_matrices(pr_coarse G, const double *U_prev, void *stream);

/* Device copies of the handle's data (each pointer nullable): U, V as
 * (n_local, rows, k), sigma (n_local, l), C (n_local, k, k). */
pr_status pr_coarse_export(pr_coarse G, double *U, double *V, double *sigma, double *C, void *stream);

/* Device copies of U_q and V_q (rows x k each, nullable) of local interval q_local. */
pr_status pr_coarse_export_interval(pr_coarse G, int q_local, double *U_q, double *V_q, void *stream);

/* d_i = Sigma_q V_q^T (Y2_i - Y1_i), q = first + i, i < n_local: d is
 * (n_local, k, nsrc).  Y1 == NULL means zero (initialisation). */
pr_status pr_coarse_project(pr_coarse G, int nsrc, const double *Y1, const double *Y2, long ld,
                            double *d, void *stream);

/* e_j = C_j e_{j-1} + d_j, j = 0..N-1, e_{-1} = 0 (C_0 ignored): the sequential
 * coarse sweep in reduced coordinates; C (N, k, k), d and e (N, k, nsrc). */
pr_status pr_reduced_sweep(const double *C, const double *d, int N, int k, int nsrc, double *e,
                           void *stream);

/* out_i = Fu_i + U_q e_i (q = first + i; Fu, out output-side blocks), and, if
 * upd != NULL, upd[i*nsrc + s] = ||out_i,s(new) - out_i,s(old)||. */
pr_status pr_coarse_expand(pr_coarse G, int nsrc, const double *Fu, const double *e, double *out,
                           long ld, double *upd, void *stream);

/* --------------------------------------------------------------------- bounds */

/* Host only.  delta, eps (eq. bounds_delta_eps), bnorm[m] = ||b_m|| (b_0 =
 * u0), m = 0..N; upd[(k-1)*(N+1) + n] = ||u^k_n - u^{k-1}_n||, k = 1..K.
 * Outputs (host, nullable):
 *   apriori[k*(N+1) + n], k = 0..K: eq. error_bound_initial (k = 0) and
 *                                   eq. error_bound_eps_delta2 (k >= 1)
 *   apost[(k-1)*(N+1) + n], k = 1..K: eq. apost_bound
 *   apost_sup[k-1]: eq. apost_bound_sup (NaN if delta >= 1)
 * Binomials are evaluated in log space.  Errors: EINVAL. */
pr_status pr_bounds(double delta, double eps, int N, int K, const double *bnorm,
                    const double *upd, double *apriori, double *apost, double *apost_sup);

#ifdef __cplusplus
}
#endif
#endif /* PR_H */
