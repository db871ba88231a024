// pr_api.cu -- the C ABI of include/pr.h: validation, handles, workspace and
// the host-side orchestration of the kernels (no numerical work on the host
// except the O(N^2) scalar bound formulas of pr_bounds).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <unordered_map>

#include "pr_internal.cuh"

namespace pr {

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

pr_status cuda_fail(cudaError_t e, const char *where)
{
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error %d (%s) at %s", (int)e, cudaGetErrorString(e), where);
    g_err = buf;
    if (e == cudaErrorMemoryAllocation) return PR_EOOM;
    return PR_ECUDA;
}

// --------------------------------------------------------------- workspace
// Stream-ordered caching pool.  A freed block remembers the stream it was last
// used on and an event recorded there at free time; reusing it on the same
// stream needs nothing (stream order), reusing it on another stream first makes
// that stream wait for the event (no host synchronisation in either case).
// Free lists are per device.
struct WsBlock {
    size_t bytes;
    int dev;
    cudaStream_t last;
    cudaEvent_t ev;
};
static std::mutex g_ws_mu;
static std::multimap<std::pair<int, size_t>, void *> g_ws_free;   // (device, bytes) -> block
static std::unordered_map<void *, WsBlock> g_ws_blk;

static int cur_device()
{
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

void *ws_alloc(size_t bytes, cudaStream_t s)
{
    if (bytes == 0) bytes = 256;
    bytes = (bytes + 255) & ~(size_t)255;
    const int dev = cur_device();
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto it = g_ws_free.lower_bound({dev, bytes});
    if (it != g_ws_free.end() && it->first.first == dev && it->first.second <= 2 * bytes + (64 << 20)) {
        void *p = it->second;
        g_ws_free.erase(it);
        WsBlock &b = g_ws_blk[p];
        if (b.last != s && b.ev) cudaStreamWaitEvent(s, b.ev, 0);
        b.last = s;
        return p;
    }
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        // release this device's cached blocks (cudaFree synchronises) and retry once
        for (auto i = g_ws_free.begin(); i != g_ws_free.end();) {
            if (i->first.first != dev) { ++i; continue; }
            auto b = g_ws_blk.find(i->second);
            if (b != g_ws_blk.end()) {
                if (b->second.ev) cudaEventDestroy(b->second.ev);
                g_ws_blk.erase(b);
            }
            cudaFree(i->second);
            i = g_ws_free.erase(i);
        }
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
    }
    g_ws_blk[p] = WsBlock{bytes, dev, s, nullptr};
    return p;
}

void ws_free(void *p, cudaStream_t s)
{
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto it = g_ws_blk.find(p);
    if (it == g_ws_blk.end()) return;
    WsBlock &b = it->second;
    if (!b.ev) cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming);
    if (b.ev) cudaEventRecord(b.ev, s);
    b.last = s;
    g_ws_free.emplace(std::make_pair(b.dev, b.bytes), p);
}

// ------------------------------------------------------------------- flags
static Flags g_flags;
static std::atomic<int> g_flags_gen{-1};
static std::mutex g_flags_mu;

static void read_flags()
{
    auto on = [](const char *n) { const char *e = getenv(n); return e && *e && *e != '0'; };
    auto num = [](const char *n) { const char *e = getenv(n); return e ? atoi(e) : 0; };
    Flags f;
    f.no_part = on("PR_NO_PART");
    f.no_xty_rm = on("PR_NO_XTY_RM");
    f.no_trsm_dmma = on("PR_NO_TRSM_DMMA");
    f.no_rinv_cm = on("PR_NO_RINV_CM");
    f.no_expand_mma = on("PR_NO_EXPAND_MMA");
    f.part_prof = on("PR_PART_PROF");
    f.qr_trace = on("PR_QR_TRACE");
    f.debug_sync = on("PR_DEBUG_SYNC");
    f.part_vpt2 = on("PR_PART_VPT2");
    f.no_src_basis = on("PR_NO_SRC_BASIS");
    f.part_h = num("PR_PART_H");
    f.stepper_pd = num("PR_STEPPER_PD");
    f.stepper_vpt = num("PR_STEPPER_VPT");
    if (getenv("PR_PART_IDLE_NS")) f.part_idle_ns = num("PR_PART_IDLE_NS");
    f.part_noiface = on("PR_PART_NOIFACE");
    f.part_notmem = on("PR_PART_NOTMEM");
    f.part_nodm = on("PR_PART_NODM");
    f.part_nopersist = on("PR_PART_NOPERSIST");
    g_flags = f;
}

const Flags &flags()
{
    if (g_flags_gen.load(std::memory_order_acquire) < 0) {
        std::lock_guard<std::mutex> lk(g_flags_mu);
        if (g_flags_gen.load() < 0) { read_flags(); g_flags_gen.store(0, std::memory_order_release); }
    }
    return g_flags;
}

// ---------------------------------------------------------------- counters
static std::atomic<long> g_launches{0};
static std::atomic<int> g_prof{0};
struct TimedLaunch {
    cudaEvent_t a, b;
    double dof_steps, flops;
    int phase;
};
static std::mutex g_prof_mu;
static std::vector<TimedLaunch> g_timed;
static thread_local cudaEvent_t g_pending_begin = nullptr;
static thread_local int g_phase = PR_PHASE_DIRECT;

// phase of the fine-propagation launches issued by this thread (pr_phase_counters)
struct PhaseScope {
    int saved;
    explicit PhaseScope(int p) : saved(g_phase) { g_phase = p; }
    ~PhaseScope() { g_phase = saved; }
};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
bool profiling() { return g_prof.load(std::memory_order_relaxed) != 0; }

void stepper_timed_begin(cudaStream_t s)
{
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) { g_pending_begin = nullptr; return; }
    cudaEventRecord(e, s);
    g_pending_begin = e;
}

void stepper_timed_end(cudaStream_t s, double dof_steps, double flops)
{
    if (!g_pending_begin) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_timed.push_back({g_pending_begin, e, dof_steps, flops, g_phase});
    g_pending_begin = nullptr;
}

int num_sms()
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
        cudaGetLastError();
        sms = 148;
    }
    return sms;
}

// RAII set of workspace buffers of one stream, released in stream order at scope exit.
struct Scratch {
    cudaStream_t s;
    std::vector<void *> bufs;
    explicit Scratch(cudaStream_t st) : s(st) {}
    ~Scratch() { for (void *p : bufs) ws_free(p, s); }
    template <class T>
    T *get(size_t count)
    {
        void *p = ws_alloc(count * sizeof(T), s);
        if (p) bufs.push_back(p);
        return (T *)p;
    }
};

#define PR_ALLOC(ptr, T, count, S)                                   \
    do {                                                             \
        ptr = (S).get<T>(count);                                     \
        if (!ptr) { ::pr::set_error("out of device memory"); return PR_EOOM; } \
    } while (0)

// Strides of vector v / row i in the op layout with leading dimension ld.
struct Lay {
    long rs, vs;
};
static inline Lay lay(const Op &op, long ld) { return op.dim == 1 ? Lay{ld, 1} : Lay{1, ld}; }

// PR_DEBUG_SYNC=1: synchronise and log after every orchestration stage.
static bool debug_sync() { return flags().debug_sync; }

static void stage(const char *what, cudaStream_t s)
{
    if (!debug_sync()) return;
    cudaError_t e = cudaStreamSynchronize(s);
    fprintf(stderr, "[pr] %s: %s\n", what, cudaGetErrorString(e));
    fflush(stderr);
}

// -------------------------------------------------------------- QR driver
// Iterated shifted CholeskyQR of nb blocks Q_b (rows x l), in place.  The
// pass loop is controlled on the device: every pass up to the cap is enqueued
// without a host check, a block that is done (state 2) makes every kernel of
// the later passes return at once, the pass count lands in passes_dev, and a
// block still active after the cap raises *fail (reported by pr_coarse_info).
// So pr_build_coarse never waits for the device.  nchunk_total: the Gram
// row-chunking depends on the global interval count only, so a shard computes
// bit-identical bases.
constexpr int QR_MAX_PASSES = 24;

static pr_status cholqr(const Op &op, double *Q, long ld, int nb, int l, double *Rtot, int *fail,
                        int *passes_dev, int nchunk, cudaStream_t s)
{
    Scratch S(s);
    Lay L = lay(op, ld);
    const long rows = op.rows;
    const long xbs = (op.dim == 1) ? (long)l : (long)l * ld;
    long chunk_rows = (rows + nchunk - 1) / nchunk;
    double *part, *R;
    int *state, *act;
    PR_ALLOC(part, double, (size_t)nb * nchunk * l * l, S);
    PR_ALLOC(R, double, (size_t)nb * l * l, S);
    double *Rinv;
    PR_ALLOC(Rinv, double, (size_t)nb * l * l, S);
    PR_ALLOC(state, int, nb, S);
    PR_ALLOC(act, int, nb, S);
    PR_CUDA(cudaMemsetAsync(state, 0, nb * sizeof(int), s));
    PR_CUDA(cudaMemsetAsync(passes_dev, 0, sizeof(int), s));
    if (Rtot) PR_CUDA(launch_eye(Rtot, nb, l, s));
    for (int pass = 1; pass <= QR_MAX_PASSES; ++pass) {
        XtY x{state, Q, xbs, L.rs, L.vs, l, Q, xbs, L.rs, L.vs, l, rows, nb, nchunk, chunk_rows, part};
        PR_CUDA(launch_xty(x, s));
        stage("qr gram", s);
        CholArgs c{part, nchunk, nb, l, rows, state, act, R, Rtot, nullptr, fail};
        c.Rinv = Rinv;
        c.pass = pass;
        c.max_pass = QR_MAX_PASSES;
        c.passes = passes_dev;
        double *offI = nullptr;
        if (debug_sync()) {
            offI = S.get<double>(3 * nb);
            if (offI) PR_CUDA(cudaMemsetAsync(offI, 0, 3 * nb * sizeof(double), s));
            c.offI = offI;
            c.shift_dbg = offI + nb;
        }
        PR_CUDA(launch_chol(c, s));
        stage("qr chol", s);
        if (offI) {
            std::vector<double> h(3 * nb);
            std::vector<int> hs(nb);
            PR_CUDA(cudaMemcpy(h.data(), offI, 3 * nb * sizeof(double), cudaMemcpyDeviceToHost));
            double smax = 0, amax = 0;
            for (int i = 0; i < nb; ++i) { smax = std::max(smax, h[nb + 2 * i]); amax = std::max(amax, h[nb + 2 * i + 1]); }
            fprintf(stderr, "[pr]   shift/||G||_F max %.3e, Cholesky retries max %.0f\n", smax, amax);
            PR_CUDA(cudaMemcpy(hs.data(), state, nb * sizeof(int), cudaMemcpyDeviceToHost));
            double mn = 1e300, mx = 0;
            int cnt[3] = {0, 0, 0};
            for (int i = 0; i < nb; ++i) { mn = std::min(mn, h[i]); mx = std::max(mx, h[i]); cnt[hs[i]]++; }
            fprintf(stderr, "[pr] qr pass %d: ||G-I||_F min %.3e max %.3e; states after: shift %d plain1 %d done %d\n",
                    pass, mn, mx, cnt[0], cnt[1], cnt[2]);
            if (cnt[2] == nb) break;
        }
        PR_CUDA(launch_trsm(Q, xbs, L.rs, L.vs, rows, l, nb, R, act, s));
        PR_CUDA(launch_rinv_apply(Q, xbs, L.rs, L.vs, rows, l, nb, Rinv, act, s));
        stage("qr apply", s);
    }
    return PR_OK;
}

// out += off for B vectors of a 1D batch (row strides ld_off / ld_out)
__global__ void k_vadd(const double *off, long ld_off, long rows, long B, double *out, long ld_out)
{
    const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * B) return;
    const long i = idx / B, v = idx % B;
    out[i * ld_out + v] += off[i * ld_off + v];
}

// out = x - y (op-layout vector blocks)
__global__ void k_vdiff(const double *x, const double *y, long rs, long vs, long rows, int nvec, double *out)
{
    const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * nvec) return;
    const long v = idx % nvec, i = idx / nvec;
    const long o = i * rs + v * vs;
    out[o] = x[o] - y[o];
}

// mx[c] = max(mx[c], nrm[c]) for c < cnt (c >= lo only)
__global__ void k_runmax(double *mx, const double *nrm, int lo, int cnt)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < cnt && c >= lo) mx[c] = fmax(mx[c], nrm[c]);
}

// One fine-propagation launch (1D or 2D), shared by the ABI and the drivers.
static pr_status propagate(const Op &op, int mode, int q0, int m, int B, int vpi,
                           const pr_source *f, const double *in, long ld_in, double *out,
                           long ld_out, const double *off, long ld_off, int sketch,
                           unsigned long long seed, cudaStream_t s, unsigned long long ctr3 = 0ULL,
                           int step0 = 0, int mstride = 0)
{
    if (B == 0) return PR_OK;
    if (op.weighted) {
        // F^ = C F C^{-1} (LINEAR / AFFINE: the source term maps with C too) and
        // its Euclidean adjoint C^{-T} F'^T C^T, in place in `out` (R-WIP)
        Op base = op;
        base.weighted = 0;
        const double *cd = op.wC, *ce = op.wC + op.n;
        if (sketch) {
            PR_CUDA(launch_sketch(1, op.n, op.rows, q0, B / vpi, vpi, seed, out, ld_out, 1, s, 0.0, ctr3));
            in = out;
            ld_in = ld_out;
        }
        PR_CUDA(launch_bidiag(mode == PR_ADJOINT ? BIDIAG_CT : BIDIAG_CINV, op.n, cd, ce, B, in, ld_in, 1, out,
                              ld_out, 1, s));
        pr_status st = propagate(base, mode, q0, m, B, vpi, f, out, ld_out, out, ld_out, nullptr, 0, 0, 0, s, 0ULL,
                                 step0, mstride);
        if (st != PR_OK) return st;
        PR_CUDA(launch_bidiag(mode == PR_ADJOINT ? BIDIAG_CTINV : BIDIAG_C, op.n, cd, ce, B, out, ld_out, 1, out,
                              ld_out, 1, s));
        if (off) {
            note_launch();
            k_vadd<<<(unsigned)((op.rows * (long)B + 255) / 256), 256, 0, s>>>(off, ld_off, op.rows, B, out, ld_out);
            PR_CHECK_LAUNCH("k_vadd");
        }
        return PR_OK;
    }
    if (op.dim == 2) {
        Sep2dArgs a{&op, mode, q0, m, B, vpi, f, in, ld_in, out, ld_out, off, ld_off};
        if (sketch) {
            PR_CUDA(cudaMemset2DAsync(out, ld_out * sizeof(double), 0, op.rows * sizeof(double), B, s));
            PR_CUDA(launch_sketch(2, op.n, op.rows, q0, B / vpi, vpi, seed, out, 1, ld_out, s, 0.0, ctr3));
            a.in = out;
            a.ld_in = ld_out;
        }
        return run_sep2d(a, s);
    }
    Scratch S(s);
    if (sketch) {
        // Omega materialised by the fully parallel generator, then stepped in place
        // (a thread-serial Philox inside the stepper's first pass costs more than
        // the extra write + read)
        PR_CUDA(launch_sketch(1, op.n, op.rows, q0, B / vpi, vpi, seed, out, ld_out, 1, s, 0.0, ctr3));
        in = out;
        ld_in = ld_out;
        sketch = 0;
    }
    StepArgs a{};
    a.n = op.n;
    a.B = B;
    a.m = m;
    a.DN = (mode == PR_ADJOINT) ? op.dn_tr : op.dn_fw;
    a.UP = (mode == PR_ADJOINT) ? op.up_tr : op.up_fw;
    a.in = in; a.ld_in = ld_in;
    a.out = out; a.ld_out = ld_out;
    a.off = off; a.ld_off = ld_off;
    a.sketch = sketch;
    a.seed = seed;
    a.q0 = q0;
    a.vpi = vpi;
    a.step0 = step0;
    a.mstride = mstride;
    a.R = 0;
    a.dt = op.dt;
    if (mode == PR_AFFINE && f && f->kind == PR_SRC_SEP1D && f->nterms > 0) {
        double *spT;
        const int rsp = stepper_rs(f->nterms);
        PR_ALLOC(spT, double, (size_t)op.n * rsp, S);
        PR_CUDA(launch_transpose(f->space, f->nterms, op.n, spT, rsp, s));
        a.R = f->nterms;
        a.spaceT = spT;
        a.time = f->time;
        a.amp = f->amp;
        a.nsteps = f->nsteps;
        a.nsrc = f->nsrc;
    }
    if (op.pencil) {
        const long ms = mstride > 0 ? mstride : m;
        PR_REQUIRE((long)(q0 + (B + vpi - 1) / vpi - 1) * ms + step0 + m <= op.pen_nsteps, PR_EDIM,
                   "intervals beyond the time-dependent operator's step count");
        PR_CUDA(launch_stepper_pencil(op, mode, a, s));
    } else if (part_preferred(op, B, m)) {
        PR_CUDA(launch_stepper_part(op, a, mode == PR_ADJOINT, s));
    } else {
        PR_CUDA(launch_stepper_1d(a, s));
    }
    return PR_OK;
}

}  // namespace pr

using namespace pr;

// =================================================================== ABI
extern "C" {

const char *pr_last_error(void) { return g_err.c_str(); }

pr_status pr_reload_env(void)
{
    std::lock_guard<std::mutex> lk(g_flags_mu);
    read_flags();
    g_flags_gen.store(1, std::memory_order_release);
    return PR_OK;
}
int pr_version(void) { return 1; }

pr_status pr_profile(int enable)
{
    g_prof.store(enable ? 1 : 0);
    return PR_OK;
}

pr_status pr_counters(int reset, long *kernel_launches, long *stepper_launches, double *stepper_ms,
                      double *stepper_dof_steps, double *stepper_flops)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    double ms = 0.0, dof = 0.0, fl = 0.0;
    long n = 0;
    for (auto &t : g_timed) {
        float f = 0.f;
        cudaEventSynchronize(t.b);
        if (cudaEventElapsedTime(&f, t.a, t.b) == cudaSuccess) { ms += f; dof += t.dof_steps; fl += t.flops; ++n; }
    }
    if (stepper_flops) *stepper_flops = fl;
    if (kernel_launches) *kernel_launches = g_launches.load();
    if (stepper_launches) *stepper_launches = n;
    if (stepper_ms) *stepper_ms = ms;
    if (stepper_dof_steps) *stepper_dof_steps = dof;
    if (reset) {
        for (auto &t : g_timed) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
        g_timed.clear();
        g_launches.store(0);
    }
    return PR_OK;
}

pr_status pr_phase_counters(int reset, long *launches, double *ms, double *dof_steps)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    long n[PR_NPHASES] = {0};
    double t[PR_NPHASES] = {0.0}, d[PR_NPHASES] = {0.0};
    for (auto &x : g_timed) {
        float f = 0.f;
        cudaEventSynchronize(x.b);
        if (cudaEventElapsedTime(&f, x.a, x.b) == cudaSuccess && x.phase >= 0 && x.phase < PR_NPHASES) {
            n[x.phase] += 1;
            t[x.phase] += f;
            d[x.phase] += x.dof_steps;
        }
    }
    for (int i = 0; i < PR_NPHASES; ++i) {
        if (launches) launches[i] = n[i];
        if (ms) ms[i] = t[i];
        if (dof_steps) dof_steps[i] = d[i];
    }
    if (reset) {
        for (auto &x : g_timed) { cudaEventDestroy(x.a); cudaEventDestroy(x.b); }
        g_timed.clear();
        g_launches.store(0);
    }
    return PR_OK;
}

pr_status pr_op_create_tridiag(int n, const double *sub, const double *diag, const double *sup,
                               const double *rowsum, const double *colsum, double dt, pr_op *out)
{
    PR_REQUIRE(out, PR_EINVAL, "out is NULL");
    PR_REQUIRE(n >= 2 && sub && diag && sup, PR_EINVAL, "n < 2 or NULL operator arrays");
    PR_REQUIRE(dt > 0.0 && isfinite(dt), PR_EINVAL, "dt must be positive");
    PR_REQUIRE((rowsum == nullptr) == (colsum == nullptr), PR_EINVAL,
               "give both rowsum and colsum or neither");
    *out = nullptr;
    pr_op h = new pr_op_s();
    Op &op = h->op;
    op.dim = 1;
    op.n = n;
    op.rows = n;
    op.dt = dt;
    double *d_in = nullptr;
    int *d_bad = nullptr;
    const size_t nb = (size_t)n * sizeof(double);
    auto fail = [&](pr_status st) {
        cudaFree(d_in);
        cudaFree(d_bad);
        cudaFree(op.dn_fw); cudaFree(op.up_fw); cudaFree(op.dn_tr); cudaFree(op.up_tr);
        cudaFree(op.part_rowc_fw); cudaFree(op.part_ctad_fw); cudaFree(op.part_rowc_tr); cudaFree(op.part_ctad_tr);
        delete h;
        return st;
    };
    cudaError_t e = cudaMalloc(&d_in, 5 * nb);
    if (e == cudaSuccess) e = cudaMalloc(&d_bad, 2 * sizeof(int));   // {bad pivot, not scalable}
    if (e == cudaSuccess) e = cudaMalloc(&op.dn_fw, n * sizeof(Coef));
    if (e == cudaSuccess) e = cudaMalloc(&op.up_fw, n * sizeof(Coef));
    if (e == cudaSuccess) e = cudaMalloc(&op.dn_tr, n * sizeof(Coef));
    if (e == cudaSuccess) e = cudaMalloc(&op.up_tr, n * sizeof(Coef));
    if (e != cudaSuccess) return fail(cuda_fail(e, "pr_op_create_tridiag alloc"));
    double *dsub = d_in, *ddiag = d_in + n, *dsup = d_in + 2 * n, *drs = d_in + 3 * n, *dcs = d_in + 4 * n;
    e = cudaMemcpy(dsub, sub, nb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(ddiag, diag, nb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dsup, sup, nb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && rowsum) e = cudaMemcpy(drs, rowsum, nb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && colsum) e = cudaMemcpy(dcs, colsum, nb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(d_bad, 0, 2 * sizeof(int));
    if (e == cudaSuccess)
        e = launch_factor_1d(n, dsub, dsup, rowsum ? drs : nullptr, ddiag, dt, 0, op.dn_fw, op.up_fw, d_bad, 0);
    if (e == cudaSuccess)
        e = launch_factor_1d(n, dsub, dsup, colsum ? dcs : nullptr, ddiag, dt, 1, op.dn_tr, op.up_tr, d_bad, 0);
    // partitioned-stepper factors (small batches), both orientations
    int pP = 0, pL = 0, pCL = 0, pK = 0;
    double *d_ends = nullptr;
    if (e == cudaSuccess && part_config(n, pP, pL, pCL, pK)) {
        op.part_P = pP; op.part_L = pL; op.part_CL = pCL; op.part_K = pK;
        const size_t rb = (size_t)pP * pL * PART_ROWC * sizeof(double), cb = (size_t)pCL * (PART_CTAD + PART_MINV) * sizeof(double);
        e = cudaMalloc(&op.part_rowc_fw, rb);
        if (e == cudaSuccess) e = cudaMalloc(&op.part_rowc_tr, rb);
        if (e == cudaSuccess) e = cudaMalloc(&op.part_ctad_fw, cb);
        if (e == cudaSuccess) e = cudaMalloc(&op.part_ctad_tr, cb);
        if (e == cudaSuccess) e = cudaMalloc(&d_ends, (size_t)PART_ENDS * pP * sizeof(double));
        if (e == cudaSuccess)
            e = launch_part_setup(n, pP, pL, pCL, pK, dsub, dsup, rowsum ? drs : nullptr, ddiag, dt, 0,
                                  op.part_rowc_fw, op.part_ctad_fw, d_ends, d_bad, d_bad + 1, 0);
        if (e == cudaSuccess)
            e = launch_part_setup(n, pP, pL, pCL, pK, dsub, dsup, colsum ? dcs : nullptr, ddiag, dt, 1,
                                  op.part_rowc_tr, op.part_ctad_tr, d_ends, d_bad, d_bad + 1, 0);
    }
    int bad[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(bad, d_bad, 2 * sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(d_ends);
    if (e == cudaSuccess && bad[1] && op.part_P) {
        // the chunk-local scaling of the partitioned stepper does not exist for
        // this operator (decoupled rows or extreme coupling ratios, k_part.cu):
        // every fine solve uses the streaming stepper K1
        cudaFree(op.part_rowc_fw); cudaFree(op.part_ctad_fw); cudaFree(op.part_rowc_tr); cudaFree(op.part_ctad_tr);
        op.part_rowc_fw = op.part_ctad_fw = op.part_rowc_tr = op.part_ctad_tr = nullptr;
        op.part_P = op.part_L = op.part_CL = op.part_K = 0;
    }
    if (e != cudaSuccess) return fail(cuda_fail(e, "pr_op_create_tridiag factor"));
    if (bad[0]) {
        set_error("non-positive or non-finite pivot in the factorisation of I + dt A");
        return fail(PR_ESINGULAR);
    }
    cudaFree(d_in);
    cudaFree(d_bad);
    *out = h;
    return PR_OK;
}

pr_status pr_op_create_pencil(int n, int nsteps, const double *lsub, const double *ldiag,
                              const double *lsup, const double *lrowsum, const double *msub,
                              const double *mdiag, const double *msup, double dt, pr_op *out)
{
    PR_REQUIRE(out, PR_EINVAL, "out is NULL");
    PR_REQUIRE(n >= 2 && nsteps >= 1 && lsub && ldiag && lsup, PR_EINVAL,
               "n < 2, nsteps < 1 or NULL step matrices");
    PR_REQUIRE(dt > 0.0 && isfinite(dt), PR_EINVAL, "dt must be positive");
    PR_REQUIRE((msub == nullptr) == (mdiag == nullptr) && (mdiag == nullptr) == (msup == nullptr),
               PR_EINVAL, "give all three mass-matrix arrays or none");
    *out = nullptr;
    pr_op h = new pr_op_s();
    Op &op = h->op;
    op.dim = 1;
    op.n = n;
    op.rows = n;
    op.dt = dt;
    op.pencil = 1;
    op.pen_nsteps = nsteps;
    const size_t sn = (size_t)nsteps * n;
    double *d_in = nullptr;
    int *d_bad = nullptr;
    auto fail = [&](pr_status st) {
        cudaFree(d_in);
        cudaFree(d_bad);
        cudaFree(op.pen_fac);
        cudaFree(op.pen_m);
        delete h;
        return st;
    };
    cudaError_t e = cudaMalloc(&d_in, (lrowsum ? 4 : 3) * sn * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&d_bad, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&op.pen_fac, sn * sizeof(Coef));
    if (e == cudaSuccess && mdiag) e = cudaMalloc(&op.pen_m, 3 * (size_t)n * sizeof(double));
    if (e != cudaSuccess) return fail(cuda_fail(e, "pr_op_create_pencil alloc"));
    double *da = d_in, *db = d_in + sn, *dc = d_in + 2 * sn, *drs = lrowsum ? d_in + 3 * sn : nullptr;
    e = cudaMemcpy(da, lsub, sn * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(db, ldiag, sn * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dc, lsup, sn * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && drs) e = cudaMemcpy(drs, lrowsum, sn * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && mdiag) {
        e = cudaMemcpy(op.pen_m, msub, n * sizeof(double), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(op.pen_m + n, mdiag, n * sizeof(double), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(op.pen_m + 2 * n, msup, n * sizeof(double), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaMemset(d_bad, 0, sizeof(int));
    if (e == cudaSuccess) e = launch_pencil_factor(n, nsteps, da, db, dc, drs, op.pen_fac, d_bad, 0);
    int bad = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(cuda_fail(e, "pr_op_create_pencil factor"));
    if (bad) {
        set_error("zero, negative (row-sum form) or non-finite pivot in a step matrix M + dt A(t_g)");
        return fail(PR_ESINGULAR);
    }
    cudaFree(d_in);
    cudaFree(d_bad);
    *out = h;
    return PR_OK;
}

pr_status pr_op_destroy(pr_op h)
{
    if (!h) return PR_OK;
    Op &op = h->op;
    if (h->view) {
        cudaFree(op.wC);
        delete h;
        return PR_OK;
    }
    cudaFree(op.dn_fw); cudaFree(op.up_fw); cudaFree(op.dn_tr); cudaFree(op.up_tr);
    cudaFree(op.part_rowc_fw); cudaFree(op.part_ctad_fw); cudaFree(op.part_rowc_tr); cudaFree(op.part_ctad_tr);
    cudaFree(op.S); cudaFree(op.lam);
    cudaFree(op.pen_fac); cudaFree(op.pen_m);
    delete h;
    return PR_OK;
}

pr_status pr_op_create_weighted(pr_op base, pr_op *out)
{
    PR_REQUIRE(base && out, PR_EINVAL, "NULL argument");
    const Op &b = base->op;
    PR_REQUIRE(b.pencil && b.pen_m && !b.weighted, PR_EINVAL,
               "a weighted view needs a pencil operator with a mass matrix");
    const int n = b.n;
    std::vector<double> m(3 * (size_t)n), c(2 * (size_t)n);
    PR_CUDA(cudaMemcpy(m.data(), b.pen_m, m.size() * sizeof(double), cudaMemcpyDeviceToHost));
    const double *ms = m.data(), *md = m.data() + n, *mp = m.data() + 2 * n;
    // M = C^T C, C upper bidiagonal (Cholesky of the SPD tridiagonal mass matrix)
    for (int i = 0; i < n; ++i) {
        const double e = (i > 0) ? c[n + i - 1] : 0.0;
        const double d2 = md[i] - e * e;
        PR_REQUIRE(d2 > 0.0 && isfinite(d2), PR_ESINGULAR, "mass matrix not positive definite");
        c[i] = sqrt(d2);
        c[n + i] = (i + 1 < n) ? mp[i] / c[i] : 0.0;
        (void)ms;
    }
    pr_op h = new pr_op_s();
    h->op = b;                   // shares the base's factor arrays
    h->view = true;
    h->op.weighted = 1;
    h->op.wC = nullptr;
    cudaError_t e = cudaMalloc(&h->op.wC, c.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(h->op.wC, c.data(), c.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(h->op.wC);
        delete h;
        return cuda_fail(e, "pr_op_create_weighted");
    }
    *out = h;
    return PR_OK;
}

pr_status pr_op_weight_apply(pr_op view, int direction, int B, const double *X, long ldx, double *Y, long ldy,
                             void *stream)
{
    PR_REQUIRE(view && Y && (X || B == 0), PR_EINVAL, "NULL argument");
    const Op &op = view->op;
    PR_REQUIRE(op.weighted, PR_EINVAL, "not a weighted view");
    PR_REQUIRE(direction == PR_TO_WEIGHTED || direction == PR_FROM_WEIGHTED, PR_EINVAL, "bad direction");
    PR_REQUIRE(B >= 0 && ldx >= B && ldy >= B, PR_EDIM, "leading dimension too small");
    PR_CUDA(launch_bidiag(direction == PR_TO_WEIGHTED ? BIDIAG_C : BIDIAG_CINV, op.n, op.wC, op.wC + op.n, B, X,
                          ldx, 1, Y, ldy, 1, (cudaStream_t)stream));
    return PR_OK;
}

pr_status pr_op_info(pr_op h, long *rows, int *dim, int *n)
{
    PR_REQUIRE(h, PR_EINVAL, "op is NULL");
    if (rows) *rows = h->op.rows;
    if (dim) *dim = h->op.dim;
    if (n) *n = h->op.n;
    return PR_OK;
}

static pr_status check_source(const Op &op, const pr_source *f, int q0, int m, int nint)
{
    PR_REQUIRE(f, PR_EINVAL, "PR_AFFINE needs a source (kind PR_SRC_NONE for none)");
    if (f->kind == PR_SRC_NONE) return PR_OK;
    PR_REQUIRE(f->nterms >= 1 && f->nterms <= 8, PR_EINVAL, "source nterms must be 1..8");
    PR_REQUIRE((long)f->nsteps >= (long)(q0 + nint) * m, PR_EDIM, "source time axis too short");
    if (op.dim == 1) {
        PR_REQUIRE(f->kind == PR_SRC_SEP1D, PR_EDIM, "1D operator needs a PR_SRC_SEP1D source");
        PR_REQUIRE(f->nsrc >= 1 && f->space && f->time && f->amp, PR_EINVAL, "incomplete 1D source");
    } else {
        PR_REQUIRE(f->kind == PR_SRC_BUMP2D, PR_EDIM, "2D operator needs a PR_SRC_BUMP2D source");
        PR_REQUIRE(f->gx && f->gy, PR_EINVAL, "incomplete 2D source");
    }
    return PR_OK;
}

pr_status pr_fine_propagate(pr_op h, int mode, int first_interval, int m, int B,
                            int vecs_per_interval, const pr_source *f, const double *U_in,
                            long ld_in, double *U_out, long ld_out, const double *offset,
                            long ld_off, void *stream)
{
    PR_REQUIRE(h && U_out, PR_EINVAL, "NULL op or output");
    const Op &op = h->op;
    PR_REQUIRE(mode == PR_LINEAR || mode == PR_ADJOINT || mode == PR_AFFINE, PR_EINVAL, "bad mode");
    PR_REQUIRE(m >= 0 && B >= 0 && vecs_per_interval >= 1 && first_interval >= 0, PR_EINVAL,
               "negative size or vecs_per_interval < 1");
    long minld = (op.dim == 1) ? B : op.rows;
    PR_REQUIRE(ld_out >= minld && (!U_in || ld_in >= minld) && (!offset || ld_off >= minld), PR_EDIM,
               "leading dimension too small");
    if (mode == PR_AFFINE) {
        int nint = (B + vecs_per_interval - 1) / vecs_per_interval;
        pr_status st = check_source(op, f, first_interval, m, nint);
        if (st != PR_OK) return st;
        if (op.dim == 1 && f->kind == PR_SRC_SEP1D)
            PR_REQUIRE(vecs_per_interval % f->nsrc == 0, PR_EDIM,
                       "vecs_per_interval must be a multiple of nsrc");
    }
    return propagate(op, mode, first_interval, m, B, vecs_per_interval,
                     mode == PR_AFFINE ? f : nullptr, U_in, ld_in, U_out, ld_out, offset, ld_off,
                     0, 0, (cudaStream_t)stream);
}

pr_status pr_gaussian_sketch(pr_op h, int first_interval, int n_intervals, int l, uint64_t seed,
                             double *out, long ld, void *stream)
{
    PR_REQUIRE(h && out, PR_EINVAL, "NULL op or output");
    const Op &op = h->op;
    PR_REQUIRE(first_interval >= 0 && n_intervals >= 0 && l >= 1, PR_EINVAL, "bad sizes");
    long nvec = (long)n_intervals * l;
    PR_REQUIRE(ld >= (op.dim == 1 ? nvec : op.rows), PR_EDIM, "leading dimension too small");
    cudaStream_t s = (cudaStream_t)stream;
    Lay L = lay(op, ld);
    if (op.dim == 2 && nvec > 0)
        PR_CUDA(cudaMemset2DAsync(out, ld * sizeof(double), 0, op.rows * sizeof(double), nvec, s));
    PR_CUDA(launch_sketch(op.dim, op.n, op.rows, first_interval, n_intervals, l, seed, out, L.rs,
                          L.vs, s));
    return PR_OK;
}

// ------------------------------------------------------------ build
// pass counts of this chunk's two QRs -> running max in out[0..1]
__global__ void k_imax2(const int *in, int *out)
{
    if (threadIdx.x < 2) out[threadIdx.x] = max(out[threadIdx.x], in[threadIdx.x]);
}

// [delta, eps] of the local intervals: max_q sigma_{q,1}, max_q sigma_{q,k+1}
// (eq. bounds_delta_eps; eps from the computed sigma_{k+1},
// P:1231-1232; 0 when p == 0)
__global__ void k_delta_eps(const double *sigma, int nloc, int l, int k, int p, double *de)
{
    __shared__ double red[2][256];
    double d = 0.0, e = 0.0;
    for (int q = threadIdx.x; q < nloc; q += blockDim.x) {
        d = fmax(d, sigma[(long)q * l]);
        if (p > 0) e = fmax(e, sigma[(long)q * l + k]);
    }
    red[0][threadIdx.x] = d;
    red[1][threadIdx.x] = e;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            red[0][threadIdx.x] = fmax(red[0][threadIdx.x], red[0][threadIdx.x + w]);
            red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) { de[0] = red[0][0]; de[1] = red[1][0]; }
}

// Scratch of one build chunk: Y, Z (and the 2D stepper's temporary) per interval.
static size_t build_bytes_per_interval(const Op &op, int l)
{
    const size_t blk = (size_t)op.rows * l * sizeof(double);
    return (op.dim == 1 ? 2 : 3) * blk + (size_t)3 * l * l * sizeof(double);
}

// Intervals per build chunk: all of them if their scratch fits the budget
// (min(16 GiB, 40% of the free device memory)), else as many as fit (>= 1).
// Results do not depend on the chunking (per-interval seeds, per-vector
// stepper arithmetic, Gram chunking fixed by N_total).
static int build_chunk(const Op &op, int l, int nl)
{
    size_t fr = 0, tot = 0;
    size_t budget = (size_t)16 << 30;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) budget = std::min(budget, (size_t)(0.4 * (double)fr));
    else cudaGetLastError();
    const size_t per = build_bytes_per_interval(op, l);
    long c = (long)(budget / std::max<size_t>(per, 1));
    if (c < 1) c = 1;
    if (c > nl) c = nl;
    return (int)c;
}

pr_status pr_build_coarse(pr_op h, int N_total, int first_interval, int n_local, int m, int k,
                          int p, uint64_t seed, const pr_rsvd_opts *opts, pr_comm comm, void *stream,
                          pr_coarse *out)
{
    PR_REQUIRE(h && out, PR_EINVAL, "NULL op or out");
    const int qpow = opts ? opts->power_iterations : 0;
    const int indep = opts ? opts->independent_adjoint : 0;
    PR_REQUIRE(qpow >= 0 && qpow <= 16 && (indep == 0 || indep == 1), PR_EINVAL,
               "power_iterations must be 0..16 and independent_adjoint 0 or 1");
    const Op &op = h->op;
    Comm *cm = comm_of(comm);
    if (cm) {   // the canonical block partition of the intervals over the ranks
        long f0, nl0;
        shard_of(N_total, cm->rank, cm->world, f0, nl0);
        first_interval = (int)f0;
        n_local = (int)nl0;
    }
    PR_REQUIRE(N_total >= 1 && n_local >= 1 && first_interval >= 0 &&
                   first_interval + n_local <= N_total && m >= 1 && k >= 1 && p >= 0,
               PR_EINVAL, "bad interval range or rank (with a communicator: N >= world)");
    const int l = k + p;
    PR_REQUIRE(l <= 112 && l <= op.rows, PR_EDIM, "l = k + p must be <= 112 and <= rows");
    cudaStream_t s = (cudaStream_t)stream;
    *out = nullptr;
    pr_coarse G = new pr_coarse_s();
    G->N_total = N_total; G->first = first_interval; G->nloc = n_local; G->m = m;
    G->k = k; G->p = p; G->l = l; G->rows = op.rows; G->dim = op.dim;
    G->stream = s;
    G->comm = comm;
    G->rank = cm ? cm->rank : 0;
    G->world = cm ? cm->world : 1;
    const long rows = op.rows;
    const int nl = n_local;
    G->U = (double *)ws_alloc((size_t)nl * rows * k * sizeof(double), s);
    G->V = (double *)ws_alloc((size_t)nl * rows * k * sizeof(double), s);
    G->sigma = (double *)ws_alloc((size_t)nl * l * sizeof(double), s);
    G->C = (double *)ws_alloc((size_t)nl * k * k * sizeof(double), s);
    G->fail = (int *)ws_alloc(4 * sizeof(int), s);             // qr fail, svd fail, passes Y, passes Z
    G->de = (double *)ws_alloc(2 * sizeof(double), s);
    G->C_all = (G->world > 1) ? (double *)ws_alloc((size_t)N_total * k * k * sizeof(double), s) : G->C;
    if (!G->U || !G->V || !G->sigma || !G->C || !G->fail || !G->de || !G->C_all) {
        pr_coarse_destroy(G);
        set_error("out of device memory");
        return PR_EOOM;
    }
    auto bail = [&](pr_status st) { pr_coarse_destroy(G); return st; };
    cudaError_t e = cudaMemsetAsync(G->fail, 0, 4 * sizeof(int), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(G->C, 0, (size_t)nl * k * k * sizeof(double), s);
    if (e != cudaSuccess) return bail(cuda_fail(e, "build init"));
    const int nchunk = xty_chunks(rows, N_total);      // global: shard-independent arithmetic
    const long cr = (rows + nchunk - 1) / nchunk;
    PhaseScope phase(PR_PHASE_BUILD);
    {
        Scratch S(s);
        const int nc = build_chunk(op, l, nl);
        const long Bmax = (long)nc * l;
        const long ld = (op.dim == 1) ? ((Bmax + 1) & ~1L) : rows;   // even ld: 16-B rows
        double *Y = S.get<double>((size_t)rows * (op.dim == 1 ? ld : Bmax));
        double *Z = S.get<double>((size_t)rows * (op.dim == 1 ? ld : Bmax));
        double *Rtot = S.get<double>((size_t)nc * l * l);
        double *Psi = S.get<double>((size_t)nc * l * l);
        double *Phi = S.get<double>((size_t)nc * l * l);
        int *pass_tmp = S.get<int>(2);
        if (!Y || !Z || !Rtot || !Psi || !Phi || !pass_tmp) { set_error("out of device memory"); return bail(PR_EOOM); }
        for (int c0 = 0; c0 < nl; c0 += nc) {
            const int cn = std::min(nc, nl - c0);            // intervals of this chunk
            const int q0 = first_interval + c0;
            const long B = (long)cn * l;
            pr_status st;
            // step 1: Y = F' Omega (Omega generated from (seed, q, column))
            st = propagate(op, PR_LINEAR, q0, m, (int)B, l, nullptr, nullptr, ld, Y, ld, nullptr, 0, 1, seed, s);
            if (st != PR_OK) return bail(st);
            stage("build step 1", s);
            // power iterations: W = span{(F' F'^*)^q F' omega}, with
            // re-orthonormalisation between the applications (same span, stable)
            for (int it = 0; it < qpow; ++it) {
                st = cholqr(op, Y, ld, cn, l, nullptr, G->fail, pass_tmp, nchunk, s);
                if (st == PR_OK)
                    st = propagate(op, PR_ADJOINT, q0, m, (int)B, l, nullptr, Y, ld, Z, ld, nullptr, 0, 0, 0, s);
                if (st == PR_OK) st = cholqr(op, Z, ld, cn, l, nullptr, G->fail, pass_tmp, nchunk, s);
                if (st == PR_OK)
                    st = propagate(op, PR_LINEAR, q0, m, (int)B, l, nullptr, Z, ld, Y, ld, nullptr, 0, 0, 0, s);
                if (st != PR_OK) return bail(st);
            }
            // step 2: W = orth(Y)
            st = cholqr(op, Y, ld, cn, l, nullptr, G->fail, pass_tmp, nchunk, s);
            if (st != PR_OK) return bail(st);
            stage("build step 2", s);
            // step 3: Z = F'^* W -- or, with independent_adjoint,
            // Z = F'^* Psi on an independent Gaussian set (Philox stream 2),
            // which needs no result of steps 1-2
            if (indep)
                st = propagate(op, PR_ADJOINT, q0, m, (int)B, l, nullptr, nullptr, ld, Z, ld, nullptr, 0, 1, seed, s,
                               2ULL);
            else
                st = propagate(op, PR_ADJOINT, q0, m, (int)B, l, nullptr, Y, ld, Z, ld, nullptr, 0, 0, 0, s);
            if (st != PR_OK) return bail(st);
            stage("build step 3", s);
            // Rounding-level regularisation of Z (reading R-QRF): the
            // stepper damps its own rounding errors, so F'^* W has singular values
            // far below u ||F'|| in the directions W does not resolve; lifting them
            // to ~u with ||delta_c|| ~ 2^-52 (within the floating-point error of
            // evaluating F'^* w_c, ||w_c|| = 1) saves the shifted CholeskyQR passes
            // that would only amplify noise.  G changes by O(u sigma_1).
            {
                // columns of W have norm 1; those of Psi ~ sqrt(ndof)
                const double ndof = (op.dim == 1) ? (double)op.n : (double)op.n * op.n;
                const double scale = indep ? ldexp(1.0, -52) : ldexp(1.0, -52) / sqrt(ndof);
                PR_CUDA(launch_sketch(op.dim, op.n, op.rows, q0, cn, l, seed, Z, (op.dim == 1) ? ld : 1,
                                      (op.dim == 1) ? 1 : ld, s, scale, 1ULL));
            }
            // step 4: V R_Z = Z
            st = cholqr(op, Z, ld, cn, l, Rtot, G->fail, pass_tmp + 1, nchunk, s);
            if (st != PR_OK) return bail(st);
            stage("build step 4", s);
            // pass counts: max over chunks
            note_launch();
            k_imax2<<<1, 32, 0, s>>>(pass_tmp, G->fail + 2);
            // step 5: M = R_Z^T = Psi Sigma Phi^T  (M_ij = (F'^* w_i, v_j))
            const double *Mt = Rtot;            // k_jacobi takes M^T (row-major)
            if (indep) {
                // single-view two-sided sketch: F' ~ W C V^T with Psi^T W C = Z^T V
                // = R_Z^T, i.e. C = (Psi^T W)^{-1} R_Z^T; M := C (Martinsson & Tropp's
                // reconstruction from the independent adjoint sketch)
                double *Psi_b = S.get<double>((size_t)rows * (op.dim == 1 ? ld : Bmax));
                double *A = S.get<double>((size_t)cn * l * l);
                double *part = S.get<double>((size_t)cn * nchunk * l * l);
                double *Ct = S.get<double>((size_t)cn * l * l);
                if (!Psi_b || !A || !part || !Ct) { set_error("out of device memory"); return bail(PR_EOOM); }
                Lay L = lay(op, ld);
                const long xbs = (op.dim == 1) ? (long)l : (long)l * ld;
                if (op.dim == 2)
                    PR_CUDA(cudaMemset2DAsync(Psi_b, ld * sizeof(double), 0, rows * sizeof(double), B, s));
                PR_CUDA(launch_sketch(op.dim, op.n, op.rows, q0, cn, l, seed, Psi_b, L.rs, L.vs, s, 0.0, 2ULL));
                XtY x{nullptr, Psi_b, xbs, L.rs, L.vs, l, Y, xbs, L.rs, L.vs, l, rows, cn, nchunk, cr, part};
                PR_CUDA(launch_xty(x, s));
                PR_CUDA(launch_reduce_parts(part, cn, nchunk, l, l, nullptr, 0, A, s));
                // Ct = C^T from A C = R_Z^T (pivoted LU, one CTA per interval)
                PR_CUDA(launch_lu_solve_rt(A, Rtot, cn, l, Ct, G->fail + 1, s));
                Mt = Ct;
            }
            e = launch_jacobi(Mt, cn, l, Psi, G->sigma + (long)c0 * l, Phi, G->fail + 1, s);
            if (e != cudaSuccess) return bail(cuda_fail(e, "jacobi"));
            stage("build step 5 (jacobi)", s);
            // steps 5-6: psi = W Psi_k, phi = V Phi_k
            Lay L = lay(op, ld);
            const long xbs = (op.dim == 1) ? (long)l : (long)l * ld;
            e = launch_lift(Y, xbs, L.rs, L.vs, rows, l, Psi, l, k, cn, G->U + (long)c0 * rows * k, s);
            if (e == cudaSuccess) e = launch_lift(Z, xbs, L.rs, L.vs, rows, l, Phi, l, k, cn, G->V + (long)c0 * rows * k, s);
            if (e != cudaSuccess) return bail(cuda_fail(e, "lift"));
            stage("build lift", s);
        }
        // reduced sweep matrices C_q = Sigma_q V_q^T U_{q-1}, local q >= first + 1
        if (nl >= 2) {
            int nb = nl - 1;
            double *part = S.get<double>((size_t)nb * nchunk * k * k);
            if (!part) { set_error("out of device memory"); return bail(PR_EOOM); }
            XtY x{nullptr, G->V + rows * k, rows * k, k, 1, k, G->U, rows * k, k, 1, k, rows, nb,
                  nchunk, cr, part};
            e = launch_xty(x, s);
            if (e == cudaSuccess)
                e = launch_reduce_parts(part, nb, nchunk, k, k, G->sigma + l, l, G->C + (long)k * k, s);
            if (e != cudaSuccess) return bail(cuda_fail(e, "sweep matrices"));
        }
        note_launch();
        k_delta_eps<<<1, 256, 0, s>>>(G->sigma, nl, l, k, p, G->de);
        PR_CHECK_LAUNCH("k_delta_eps");
        if (cm && cm->world > 1) {
            // C_first needs the left neighbour's last U block (one boundary hop)
            double *Uprev = S.get<double>((size_t)rows * k);
            if (!Uprev) { set_error("out of device memory"); return bail(PR_EOOM); }
            pr_status st = cm->shift_right(G->U + (long)(nl - 1) * rows * k, Uprev,
                                          (size_t)rows * k * sizeof(double), s);
            if (st != PR_OK) return bail(st);
            if (cm->rank > 0) {
                double *part = S.get<double>((size_t)nchunk * k * k);
                if (!part) { set_error("out of device memory"); return bail(PR_EOOM); }
                XtY x{nullptr, G->V, 0, k, 1, k, Uprev, 0, k, 1, k, rows, 1, nchunk, cr, part};
                e = launch_xty(x, s);
                if (e == cudaSuccess) e = launch_reduce_parts(part, 1, nchunk, k, k, G->sigma, 0, G->C, s);
                if (e != cudaSuccess) return bail(cuda_fail(e, "sweep matrix C_first"));
            }
            // global delta, eps and every interval's sweep matrix (for the
            // redundant k-dimensional sweep of pr_parareal)
            st = cm->all_reduce_max(G->de, 2, s);
            if (st != PR_OK) return bail(st);
            std::vector<long> cnt(cm->world);
            for (int r = 0; r < cm->world; ++r) {
                long f0, n0;
                shard_of(N_total, r, cm->world, f0, n0);
                cnt[r] = n0 * k * k;
            }
            st = cm->all_gather_v(G->C, G->C_all, cnt.data(), sizeof(double), s);
            if (st != PR_OK) return bail(st);
        }
    }
    *out = G;
    return PR_OK;
}

pr_status pr_build_coarse_adaptive(pr_op h, int N_total, int first_interval, int n_local, int m, int k,
                                   int p0, int p_max, double tol, int r, uint64_t seed,
                                   const pr_rsvd_opts *opts, pr_comm comm, void *stream, pr_coarse *out,
                                   int *p_used)
{
    PR_REQUIRE(h && out && p_used, PR_EINVAL, "NULL argument");
    PR_REQUIRE(p0 >= 1 && p_max >= p0 && tol > 0.0 && r >= 1, PR_EINVAL, "need 1 <= p0 <= p_max, tol > 0, r >= 1");
    *out = nullptr;
    int p = p0;
    for (;;) {
        pr_coarse G = nullptr;
        pr_status st = pr_build_coarse(h, N_total, first_interval, n_local, m, k, p, seed, opts, comm, stream, &G);
        if (st != PR_OK) return st;
        std::vector<double> est(G->nloc);
        st = pr_coarse_estimate(G, h, r, seed, est.data(), stream);
        if (st != PR_OK) { pr_coarse_destroy(G); return st; }
        double mx = 0.0;
        for (double e : est) mx = std::max(mx, e);
        if (comm) {                      // the same decision on every rank
            cudaStream_t s = (cudaStream_t)stream;
            Scratch Sd(s);
            double *dg = Sd.get<double>(1);
            if (!dg) { pr_coarse_destroy(G); set_error("out of device memory"); return PR_EOOM; }
            cudaError_t e = cudaMemcpyAsync(dg, &mx, sizeof(double), cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) st = comm_of(comm)->all_reduce_max(dg, 1, s);
            if (e == cudaSuccess && st == PR_OK) e = cudaMemcpyAsync(&mx, dg, sizeof(double), cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) { pr_coarse_destroy(G); return cuda_fail(e, "adaptive p reduction"); }
            if (st != PR_OK) { pr_coarse_destroy(G); return st; }
        }
        if (mx <= tol || p >= p_max) {
            *out = G;
            *p_used = p;
            return PR_OK;
        }
        pr_coarse_destroy(G);
        p = std::min(2 * p, p_max);
    }
}

pr_status pr_coarse_info(pr_coarse G, int *k, int *l, int *n_local, int *first_interval, int *m,
                         double *delta, double *eps, double *sigma_host, int *qr_passes)
{
    PR_REQUIRE(G, PR_EINVAL, "NULL handle");
    PR_CUDA(cudaStreamSynchronize(G->stream));
    if (k) *k = G->k;
    if (l) *l = G->l;
    if (n_local) *n_local = G->nloc;
    if (first_interval) *first_interval = G->first;
    if (m) *m = G->m;
    if (sigma_host)
        PR_CUDA(cudaMemcpy(sigma_host, G->sigma, (size_t)G->nloc * G->l * sizeof(double), cudaMemcpyDeviceToHost));
    int fl[4] = {0, 0, 0, 0};
    double de[2] = {0.0, 0.0};
    PR_CUDA(cudaMemcpy(fl, G->fail, sizeof fl, cudaMemcpyDeviceToHost));
    PR_CUDA(cudaMemcpy(de, G->de, sizeof de, cudaMemcpyDeviceToHost));
    if (qr_passes) { qr_passes[0] = fl[2]; qr_passes[1] = fl[3]; }
    if (delta) *delta = de[0];
    if (eps) *eps = (G->p > 0) ? de[1] : NAN;
    if (fl[0]) { set_error("CholeskyQR broke down or did not converge on the device"); return PR_ENOCONV; }
    if (fl[1]) { set_error("Jacobi SVD did not converge in 60 sweeps"); return PR_ENOCONV; }
    if (G->p == 0 && eps) { set_error("eps needs p >= 1"); return PR_EUNAVAIL; }
    return PR_OK;
}

pr_status pr_coarse_factors(pr_coarse G, const double **U, const double **V, const double **sigma)
{
    PR_REQUIRE(G, PR_EINVAL, "NULL handle");
    if (U) *U = G->U;
    if (V) *V = G->V;
    if (sigma) *sigma = G->sigma;
    return PR_OK;
}

// Y = G_q' X for nvec vectors with general strides (the body of pr_coarse_apply)
static pr_status coarse_apply(pr_coarse G, int q_local, int nvec, const double *X, Lay Lx, double *Y, Lay Ly,
                              cudaStream_t s)
{
    const long rows = G->rows;
    const int k = G->k;
    Scratch S(s);
    int nchunk = xty_chunks(rows, 1);
    long cr = (rows + nchunk - 1) / nchunk;
    double *part, *ev;
    PR_ALLOC(part, double, (size_t)nchunk * k * nvec, S);
    PR_ALLOC(ev, double, (size_t)k * nvec, S);
    const double *Vq = G->V + (long)q_local * rows * k;
    const double *Uq = G->U + (long)q_local * rows * k;
    XtY x{nullptr, Vq, 0, k, 1, k, X, 0, Lx.rs, Lx.vs, nvec, rows, 1, nchunk, cr, part};
    PR_CUDA(launch_xty(x, s));
    PR_CUDA(launch_reduce_parts(part, 1, nchunk, k, nvec, G->sigma + (long)q_local * G->l, 0, ev, s));
    Expand ex{Y, Ly.rs, Ly.vs, nullptr, 0, 0, Uq, 0, ev, k, nvec, 1, rows, nchunk, cr, nullptr};
    PR_CUDA(launch_expand(ex, s));
    return PR_OK;
}

pr_status pr_coarse_apply(pr_coarse G, int q_local, int nvec, const double *X, long ldx, double *Y,
                          long ldy, void *stream)
{
    PR_REQUIRE(G && X && Y, PR_EINVAL, "NULL argument");
    PR_REQUIRE(q_local >= 0 && q_local < G->nloc && nvec >= 1 && nvec <= 128, PR_EINVAL,
               "bad interval or nvec (1..128)");
    const long rows = G->rows;
    long minld = (G->dim == 1) ? nvec : rows;
    PR_REQUIRE(ldx >= minld && ldy >= minld, PR_EDIM, "leading dimension too small");
    cudaStream_t s = (cudaStream_t)stream;
    G->stream = s;
    Lay Lx = (G->dim == 1) ? Lay{ldx, 1} : Lay{1, ldx};
    Lay Ly = (G->dim == 1) ? Lay{ldy, 1} : Lay{1, ldy};
    return coarse_apply(G, q_local, nvec, X, Lx, Y, Ly, s);
}

pr_status pr_coarse_estimate(pr_coarse G, pr_op h, int r, uint64_t seed, double *est_host, void *stream)
{
    PR_REQUIRE(G && h && est_host, PR_EINVAL, "NULL argument");
    const Op &op = h->op;
    PR_REQUIRE(G->rows == op.rows && G->dim == op.dim, PR_EDIM, "coarse handle / operator mismatch");
    PR_REQUIRE(r >= 1 && r <= 64, PR_EINVAL, "r must be 1..64");
    cudaStream_t s = (cudaStream_t)stream;
    G->stream = s;
    Scratch S(s);
    const int nq = G->nloc, q0 = G->first;
    const long rows = op.rows;
    const long B = (long)nq * r;
    const long ld = (op.dim == 1) ? ((B + 1) & ~1L) : rows;
    Lay L = lay(op, ld);
    const size_t arr = (op.dim == 1) ? (size_t)rows * ld : (size_t)B * ld;
    double *Om, *Y, *Z, *npart, *nrm;
    PR_ALLOC(Om, double, arr, S);
    PR_ALLOC(Y, double, arr, S);
    PR_ALLOC(Z, double, arr, S);
    const int nchunk = xty_chunks(rows, nq);
    const long cr = (rows + nchunk - 1) / nchunk;
    PR_ALLOC(npart, double, (size_t)B * nchunk, S);
    PR_ALLOC(nrm, double, (size_t)B, S);
    if (op.dim == 2) PR_CUDA(cudaMemsetAsync(Om, 0, arr * sizeof(double), s));
    // fresh Gaussian probes (Philox counter word 3 = 3), F' and G' applied to them
    PR_CUDA(launch_sketch(op.dim, op.n, rows, q0, nq, r, seed, Om, L.rs, L.vs, s, 0.0, 3ULL));
    pr_status st = propagate(op, PR_LINEAR, q0, G->m, (int)B, r, nullptr, Om, ld, Y, ld, nullptr, 0, 0, 0, s);
    if (st != PR_OK) return st;
    for (int q = 0; q < nq; ++q) {
        const long off = (long)q * r * L.vs;
        if ((st = coarse_apply(G, q, r, Om + off, L, Z + off, L, s)) != PR_OK) return st;
    }
    note_launch();
    k_vdiff<<<(unsigned)((rows * B + 255) / 256), 256, 0, s>>>(Y, Z, L.rs, L.vs, rows, (int)B, Y);
    PR_CHECK_LAUNCH("k_vdiff");
    PR_CUDA(launch_vecnorm_parts(Y, L.rs, L.vs, rows, (int)B, nchunk, cr, npart, s));
    PR_CUDA(launch_norm_finish(npart, (int)B, nchunk, nrm, s));
    std::vector<double> h_n(B);
    PR_CUDA(cudaMemcpyAsync(h_n.data(), nrm, B * sizeof(double), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    // Halko, Martinsson & Tropp, Lemma 4.1: ||B|| <= 10 sqrt(2/pi) max_i ||B omega_i||
    // with probability >= 1 - 10^{-r}
    const double c = 10.0 * sqrt(2.0 / M_PI);
    for (int q = 0; q < nq; ++q) {
        double mx = 0.0;
        for (int i = 0; i < r; ++i) mx = std::max(mx, h_n[(size_t)q * r + i]);
        est_host[q] = c * mx;
    }
    return PR_OK;
}

pr_status pr_coarse_destroy(pr_coarse G)
{
    if (!G) return PR_OK;
    cudaStream_t s = G->stream;   // ordered after the last call that used the handle
    ws_free(G->U, s); ws_free(G->V, s); ws_free(G->sigma, s); ws_free(G->C, s); ws_free(G->fail, s);
    ws_free(G->de, s);
    if (G->C_all != G->C) ws_free(G->C_all, s);
    delete G;
    return PR_OK;
}

// ---------------------------------------------------- offsets by source basis
// b_{q,s} = F_q(0) for source s = sum_r amp[s, r] b^{(r)}_q, where b^{(r)}_q is
// F_q(0) for the single separable term time[r, .] * space[r, .] (F_q(0) is
// linear in the source; reading R-SRC).  S sources of R <= 8 terms
// then cost N*R offset fine solves instead of N*S.
__global__ void k_eye(double *E, int R)
{
    const int t = threadIdx.x;
    if (t < R * R) E[t] = (t / R == t % R) ? 1.0 : 0.0;
}

// out[i*ld + q*S + s] = sum_r amp[s*R + r] * basis[i*ldb + q*R + r]
__global__ void k_combine_offsets(const double *basis, long ldb, int R, const double *amp, int S, int nq,
                                  long rows, double *out, long ld)
{
    // a thread owns column c = (q, s) (grid.x * block over the nq * S columns:
    // coalesced stores) and walks the rows i = blockIdx.y, + gridDim.y, ...;
    // its R amplitudes stay in registers (R <= 8), the basis values of a row
    // are the same address for the S threads of an interval
    const int per = nq * S;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < per; c += gridDim.x * blockDim.x) {
        const int q = c / S, sI = c - q * S;
        const double *av = amp + (long)sI * R;
        if (R <= 8) {
            double ar[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) ar[r] = (r < R) ? av[r] : 0.0;
            for (long i = blockIdx.y; i < rows; i += gridDim.y) {
                const double *bv = basis + i * ldb + (long)q * R;
                double acc = 0.0;
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    if (r < R) acc = fma(ar[r], bv[r], acc);
                out[i * ld + c] = acc;
            }
        } else {
            for (long i = blockIdx.y; i < rows; i += gridDim.y) {
                const double *bv = basis + i * ldb + (long)q * R;
                double acc = 0.0;
                for (int r = 0; r < R; ++r) acc = fma(av[r], bv[r], acc);
                out[i * ld + c] = acc;
            }
        }
    }
}

// ---------------------------------------------------------------- Parareal
// One schedule for one GPU and for an interval-sharded run (the handle's
// communicator): rank r owns intervals q0 .. q0+nq-1 and the boundary blocks
// 0..nq of every array (block i = boundary q0+i; block 0 is the halo = the
// left neighbour's last block, u0 on rank 0).  Per iteration only the last
// block of Fu and of u moves right, and the k x S reduced sweep
// data of every interval is all-gathered so each rank runs the (cheap,
// k-dimensional) sequential sweep over all N intervals itself (DESIGN.md
// section 9).  With world = 1 every exchange is a no-op.
static pr_status parareal_core(pr_coarse G, pr_op h, int nsrc, const double *u0, long ld_u0,
                               const pr_source *f, int K_iter, double *U_out, long ld_out, double *upd_host,
                               double *bnorm_host, double *hist, long hist_stride, void *stream, double tol,
                               int *k_done)
{
    PR_REQUIRE(G && h && U_out, PR_EINVAL, "NULL argument");
    const Op &op = h->op;
    Comm *cm = comm_of(G->comm);
    const int world = G->world, rank = G->rank;
    PR_REQUIRE(world > 1 || (G->first == 0 && G->nloc == G->N_total), PR_EDIM,
               "pr_parareal needs a coarse handle covering all intervals, or one built with a communicator");
    PR_REQUIRE(rank > 0 || u0, PR_EINVAL, "u0 is NULL on rank 0");
    PR_REQUIRE(G->rows == op.rows && G->dim == op.dim, PR_EDIM, "coarse handle / operator mismatch");
    PR_REQUIRE(nsrc >= 1 && nsrc <= 128 && K_iter >= 0, PR_EINVAL, "nsrc must be 1..128, K_iter >= 0");
    const int N = G->N_total, nq = G->nloc, q0 = G->first, k = G->k, m = G->m, S = nsrc;
    const long rows = op.rows;
    const long nvec = (long)(nq + 1) * S;             // local boundary blocks 0..nq
    long minld = (op.dim == 1) ? nvec : rows;
    PR_REQUIRE(ld_out >= minld, PR_EDIM, "ld_out too small");
    PR_REQUIRE(!u0 || ld_u0 >= (op.dim == 1 ? S : rows), PR_EDIM, "ld_u0 too small");
    {
        pr_status st = check_source(op, f, q0, m, nq);
        if (st != PR_OK) return st;
        if (op.dim == 1 && f->kind == PR_SRC_SEP1D)
            PR_REQUIRE(f->nsrc == S, PR_EDIM, "source nsrc must equal nsrc");
    }
    cudaStream_t s = (cudaStream_t)stream;
    G->stream = s;
    Scratch Sc(s);
    const long ld = ld_out;          // Fu and b share U_out's layout
    Lay L = lay(op, ld);
    const size_t arr = (op.dim == 1) ? (size_t)rows * ld : (size_t)nvec * ld;
    double *Fu, *bb, *qv, *dall, *ev, *part, *npart, *upd, *bn;
    PR_ALLOC(Fu, double, arr, Sc);
    PR_ALLOC(bb, double, arr, Sc);
    const size_t red_loc = (size_t)nq * k * S, red = (size_t)N * k * S;
    PR_ALLOC(qv, double, red_loc, Sc);
    dall = qv;
    if (world > 1) PR_ALLOC(dall, double, red, Sc);
    PR_ALLOC(ev, double, red, Sc);
    const int nchunk = xty_chunks(rows, N);            // global: shard-independent arithmetic
    const long cr = (rows + nchunk - 1) / nchunk;
    PR_ALLOC(part, double, (size_t)nq * nchunk * k * 2 * S, Sc);
    PR_ALLOC(npart, double, (size_t)nvec * nchunk, Sc);
    PR_ALLOC(upd, double, (size_t)(K_iter > 0 ? K_iter : 1) * nq * S, Sc);
    PR_ALLOC(bn, double, (size_t)nvec, Sc);
    const long blk = (op.dim == 1) ? (long)S : (long)S * ld;   // element offset of one block
    double *hsend = nullptr, *hrecv = nullptr;                   // 1D halo staging (rows x S)
    if (world > 1 && op.dim == 1) {
        PR_ALLOC(hsend, double, (size_t)rows * S, Sc);
        PR_ALLOC(hrecv, double, (size_t)rows * S, Sc);
    }
    // block 0 of a := block nq of the left neighbour's a (rank 0 keeps its own)
    auto halo = [&](double *a) -> pr_status {
        if (world == 1) return PR_OK;
        if (op.dim == 2)
            return cm->shift_right(a + (long)nq * blk, a, (size_t)S * ld * sizeof(double), s);
        PR_CUDA(launch_copy_vectors(a + (long)nq * blk, L.rs, L.vs, hsend, S, 1, rows, S, s));
        pr_status st = cm->shift_right(hsend, hrecv, (size_t)rows * S * sizeof(double), s);
        if (st != PR_OK) return st;
        if (rank > 0) PR_CUDA(launch_copy_vectors(hrecv, S, 1, a, L.rs, L.vs, rows, S, s));
        return PR_OK;
    };
    auto gather_red = [&]() -> pr_status {              // d of all intervals, in order
        if (world == 1) return PR_OK;
        std::vector<long> cnt(world);
        for (int r = 0; r < world; ++r) {
            long f0, n0;
            shard_of(N, r, world, f0, n0);
            cnt[r] = n0 * k * S;
        }
        return cm->all_gather_v(qv, dall, cnt.data(), sizeof(double), s);
    };

    // u^k_0 = u0 in the state and in block 0 of Fu (Fu_0 := u0) on rank 0
    if (rank == 0) {
        Lay L0 = lay(op, ld_u0);
        PR_CUDA(launch_copy_vectors(u0, L0.rs, L0.vs, U_out, L.rs, L.vs, rows, S, s));
        PR_CUDA(launch_copy_vectors(u0, L0.rs, L0.vs, Fu, L.rs, L.vs, rows, S, s));
        PR_CUDA(launch_copy_vectors(u0, L0.rs, L0.vs, bb, L.rs, L.vs, rows, S, s));   // ||b_0|| := ||u0||
    } else if (op.dim == 1) {
        PR_CUDA(cudaMemset2DAsync(bb, ld * sizeof(double), 0, S * sizeof(double), rows, s));
    }
    if (op.dim == 2 && rank > 0) PR_CUDA(cudaMemsetAsync(bb, 0, (size_t)S * ld * sizeof(double), s));
    // offsets b_q = F_q 0 into blocks 1..nq of bb
    {
        PhaseScope phase(PR_PHASE_OFFSETS);
        pr_status st;
        if (op.dim == 1 && f->kind == PR_SRC_SEP1D && f->nterms < S && !flags().no_src_basis) {
            const int R = f->nterms;
            const long ldb = ((long)nq * R + 1) & ~1L;
            double *eye, *basis;
            PR_ALLOC(eye, double, (size_t)R * R, Sc);
            PR_ALLOC(basis, double, (size_t)rows * ldb, Sc);
            note_launch();
            k_eye<<<1, 64, 0, s>>>(eye, R);
            PR_CHECK_LAUNCH("k_eye");
            pr_source fb = *f;
            fb.nsrc = R;
            fb.amp = eye;
            st = propagate(op, PR_AFFINE, q0, m, nq * R, R, &fb, nullptr, ldb, basis, ldb, nullptr, 0, 0, 0, s);
            if (st != PR_OK) return st;
            const long per = (long)nq * S;
            dim3 cgrid((unsigned)std::min<long>((per + 255) / 256, 1024), (unsigned)std::min<long>(rows, 128));
            note_launch();
            k_combine_offsets<<<cgrid, 256, 0, s>>>(basis, ldb, R, f->amp, S, nq, rows, bb + blk, ld);
            PR_CHECK_LAUNCH("k_combine_offsets");
        } else {
            st = propagate(op, PR_AFFINE, q0, m, nq * S, S, f, nullptr, ld, bb + blk, ld, nullptr, 0, 0, 0, s);
            if (st != PR_OK) return st;
        }
    }
    PR_CUDA(launch_vecnorm_parts(bb, L.rs, L.vs, rows, (int)nvec, nchunk, cr, npart, s));
    PR_CUDA(launch_norm_finish(npart, (int)nvec, nchunk, bn, s));
    // Fu blocks 1..nq := b (initialisation uses G_q u = G'_q u + b_q)
    PR_CUDA(launch_copy_vectors(bb + blk, L.rs, L.vs, Fu + blk, L.rs, L.vs, rows, nq * S, s));
    pr_status st;
    if ((st = halo(Fu)) != PR_OK) return st;

    const double *sig = G->sigma;
    // d_q = Sigma_q V_q^T (Fu[block q] - u[block q])   (one pass over V_q)
    auto project = [&](bool with_p) -> pr_status {
        XtY x{nullptr, G->V, rows * k, k, 1, k, with_p ? U_out : Fu, blk, L.rs, L.vs, S, rows, nq,
              nchunk, cr, part};
        int pcols = 0;
        if (with_p) PR_CUDA(launch_xty_diff(x, Fu, S, pcols, s));
        else PR_CUDA(launch_xty(x, s));
        PR_CUDA(launch_reduce_pq(part, nq, nchunk, k, S, pcols, sig, G->l, qv, s));
        return gather_red();
    };
    auto expand = [&](bool norms) -> pr_status {
        Expand ex{U_out + blk, L.rs, L.vs, Fu + blk, L.rs, L.vs, G->U, rows * k, ev + (size_t)q0 * k * S, k, S,
                  nq, rows, nchunk, cr, norms ? npart : nullptr};
        PR_CUDA(launch_expand(ex, s));
        return PR_OK;
    };
    // ---- initialisation: u^0_{q+1} = G_q u^0_q (p = 0)
    if ((st = project(false)) != PR_OK) return st;
    PR_CUDA(launch_sweep(G->C_all, dall, N, k, S, ev, s));
    if ((st = expand(false)) != PR_OK) return st;
    if ((st = halo(U_out)) != PR_OK) return st;
    stage("parareal init", s);
    if (hist) PR_CUDA(launch_copy_vectors(U_out, L.rs, L.vs, hist, L.rs, L.vs, rows, (int)nvec, s));
    // ---- iterations (tol > 0: stop at the first k whose a posteriori bound
    // max_n eps sum_{m<n} delta^{n-m-1} ||u^k_m - u^{k-1}_m|| (eq. apost_bound) <= tol)
    double de[2] = {0.0, 0.0};
    if (tol > 0.0) {
        PR_CUDA(cudaMemcpyAsync(de, G->de, sizeof de, cudaMemcpyDeviceToHost, s));
        PR_CUDA(cudaStreamSynchronize(s));
    }
    std::vector<long> sf0(world), sn0(world);
    for (int r = 0; r < world; ++r) shard_of(N, r, world, sf0[r], sn0[r]);
    int K_run = K_iter;
    for (int it = 1; it <= K_iter; ++it) {
        // fine solves of all local intervals in one launch: Fu_{q+1} = F_q' u_q + b_q
        PhaseScope phase(PR_PHASE_ITERATION);
        st = propagate(op, PR_LINEAR, q0, m, nq * S, S, nullptr, U_out, ld, Fu + blk, ld, bb + blk,
                       ld, 0, 0, s);
        if (st != PR_OK) return st;
        if ((st = halo(Fu)) != PR_OK) return st;
        stage("parareal fine", s);
        if ((st = project(true)) != PR_OK) return st;
        stage("parareal project", s);
        PR_CUDA(launch_sweep(G->C_all, dall, N, k, S, ev, s));
        stage("parareal sweep", s);
        if ((st = expand(true)) != PR_OK) return st;
        PR_CUDA(launch_norm_finish(npart, nq * S, nchunk, upd + (size_t)(it - 1) * nq * S, s));
        if ((st = halo(U_out)) != PR_OK) return st;
        stage("parareal expand", s);
        if (hist)
            PR_CUDA(launch_copy_vectors(U_out, L.rs, L.vs, hist + (size_t)it * hist_stride, L.rs, L.vs, rows,
                                        (int)nvec, s));
        if (tol > 0.0) {
            double *ua = upd + (size_t)(it - 1) * nq * S;
            if (world > 1) {
                double *uall;
                PR_ALLOC(uall, double, (size_t)N * S, Sc);
                std::vector<long> cnt(world);
                for (int r = 0; r < world; ++r) cnt[r] = sn0[r] * S;
                if ((st = cm->all_gather_v(ua, uall, cnt.data(), sizeof(double), s)) != PR_OK) return st;
                ua = uall;
            }
            std::vector<double> hu1((size_t)N * S);      // boundary j = 1..N at index j-1
            PR_CUDA(cudaMemcpyAsync(hu1.data(), ua, hu1.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
            PR_CUDA(cudaStreamSynchronize(s));
            double bound = 0.0;
            for (int sI = 0; sI < S; ++sI)
                for (int n = 1; n <= N; ++n) {
                    double acc = 0.0;
                    for (int mm = 1; mm <= n - 1; ++mm) acc += pow(de[0], n - mm - 1) * hu1[(size_t)(mm - 1) * S + sI];
                    bound = std::max(bound, de[1] * acc);
                }
            if (bound <= tol) {
                K_run = it;
                break;
            }
        }
    }
    if (k_done) *k_done = K_run;
    K_iter = K_run;
    // ---- host outputs: update norms and ||b_j|| of ALL boundaries
    std::vector<long> f0(world), n0(world);
    for (int r = 0; r < world; ++r) shard_of(N, r, world, f0[r], n0[r]);
    std::vector<double> hu, hb((size_t)(N + 1) * S);
    if (upd_host && K_iter > 0) {
        double *uall = upd;
        if (world > 1) {
            PR_ALLOC(uall, double, (size_t)K_iter * N * S, Sc);
            std::vector<long> cnt(world);
            for (int r = 0; r < world; ++r) cnt[r] = (long)K_iter * n0[r] * S;
            if ((st = cm->all_gather_v(upd, uall, cnt.data(), sizeof(double), s)) != PR_OK) return st;
        }
        hu.resize((size_t)K_iter * N * S);
        PR_CUDA(cudaMemcpyAsync(hu.data(), uall, hu.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    if (bnorm_host) {
        double *ball = bn;
        if (world > 1) {
            PR_ALLOC(ball, double, (size_t)(N + 1) * S, Sc);
            std::vector<long> cnt(world);
            for (int r = 0; r < world; ++r) cnt[r] = (n0[r] + (r == 0 ? 1 : 0)) * S;
            if ((st = cm->all_gather_v(rank == 0 ? bn : bn + S, ball, cnt.data(), sizeof(double), s)) != PR_OK)
                return st;
        }
        PR_CUDA(cudaMemcpyAsync(hb.data(), ball, hb.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    int fl[2] = {0, 0};
    PR_CUDA(cudaMemcpyAsync(fl, G->fail, sizeof fl, cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    if (upd_host && K_iter > 0) {
        // gathered as [rank][it][i][s] -> upd_host[it][boundary][s], boundary 0 = 0
        size_t off = 0;
        for (int r = 0; r < world; ++r) {
            for (int it = 0; it < K_iter; ++it)
                for (long i = 0; i < n0[r]; ++i)
                    for (int sI = 0; sI < S; ++sI)
                        upd_host[((size_t)it * (N + 1) + f0[r] + i + 1) * S + sI] = hu[off++];
        }
        for (int it = 0; it < K_iter; ++it)
            for (int sI = 0; sI < S; ++sI) upd_host[(size_t)it * (N + 1) * S + sI] = 0.0;
    }
    if (bnorm_host) memcpy(bnorm_host, hb.data(), hb.size() * sizeof(double));
    if (fl[0] || fl[1]) {
        set_error("the coarse handle's rSVD failed on the device (see pr_coarse_info); outputs undefined");
        return PR_ENOCONV;
    }
    return PR_OK;
}

pr_status pr_parareal(pr_coarse G, pr_op h, int nsrc, const double *u0, long ld_u0,
                      const pr_source *f, int K_iter, double *U_out, long ld_out, double *upd_host,
                      double *bnorm_host, double *hist, long hist_stride, void *stream)
{
    return parareal_core(G, h, nsrc, u0, ld_u0, f, K_iter, U_out, ld_out, upd_host, bnorm_host, hist,
                         hist_stride, stream, 0.0, nullptr);
}

pr_status pr_parareal_tol(pr_coarse G, pr_op h, int nsrc, const double *u0, long ld_u0,
                          const pr_source *f, int K_max, double tol, double *U_out, long ld_out,
                          double *upd_host, double *bnorm_host, double *hist, long hist_stride,
                          int *k_done, void *stream)
{
    PR_REQUIRE(tol > 0.0 && k_done, PR_EINVAL, "pr_parareal_tol needs tol > 0 and k_done");
    PR_REQUIRE(G && G->p > 0, PR_EUNAVAIL, "the a posteriori bound needs eps (p >= 1)");
    return parareal_core(G, h, nsrc, u0, ld_u0, f, K_max, U_out, ld_out, upd_host, bnorm_host, hist,
                         hist_stride, stream, tol, k_done);
}

// ------------------------------------------------------ distributed stages
pr_status pr_coarse_sweep_matrices(pr_coarse G, const double *U_prev, void *stream)
{
    PR_REQUIRE(G, PR_EINVAL, "NULL handle");
    cudaStream_t s = (cudaStream_t)stream;
    G->stream = s;
    const long rows = G->rows;
    const int k = G->k;
    Scratch S(s);
    if (!U_prev) {
        PR_CUDA(cudaMemsetAsync(G->C, 0, (size_t)k * k * sizeof(double), s));
        return PR_OK;
    }
    int nchunk = xty_chunks(rows, G->N_total);
    long cr = (rows + nchunk - 1) / nchunk;
    double *part;
    PR_ALLOC(part, double, (size_t)nchunk * k * k, S);
    XtY x{nullptr, G->V, 0, k, 1, k, U_prev, 0, k, 1, k, rows, 1, nchunk, cr, part};
    PR_CUDA(launch_xty(x, s));
    PR_CUDA(launch_reduce_parts(part, 1, nchunk, k, k, G->sigma, 0, G->C, s));
    return PR_OK;
}

pr_status pr_coarse_export(pr_coarse G, double *U, double *V, double *sigma, double *C, void *stream)
{
    PR_REQUIRE(G, PR_EINVAL, "NULL handle");
    cudaStream_t s = (cudaStream_t)stream;
    G->stream = s;
    const size_t f = (size_t)G->nloc * G->rows * G->k * sizeof(double);
    if (U) PR_CUDA(cudaMemcpyAsync(U, G->U, f, cudaMemcpyDeviceToDevice, s));
    if (V) PR_CUDA(cudaMemcpyAsync(V, G->V, f, cudaMemcpyDeviceToDevice, s));
    if (sigma) PR_CUDA(cudaMemcpyAsync(sigma, G->sigma, (size_t)G->nloc * G->l * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (C) PR_CUDA(cudaMemcpyAsync(C, G->C, (size_t)G->nloc * G->k * G->k * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return PR_OK;
}

pr_status pr_coarse_export_interval(pr_coarse G, int q_local, double *U_q, double *V_q, void *stream)
{
    PR_REQUIRE(G && q_local >= 0 && q_local < G->nloc, PR_EINVAL, "bad handle or interval");
    cudaStream_t s = (cudaStream_t)stream;
    G->stream = s;
    const size_t f = (size_t)G->rows * G->k;
    if (U_q) PR_CUDA(cudaMemcpyAsync(U_q, G->U + q_local * f, f * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (V_q) PR_CUDA(cudaMemcpyAsync(V_q, G->V + q_local * f, f * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return PR_OK;
}

pr_status pr_coarse_project(pr_coarse G, int nsrc, const double *Y1, const double *Y2, long ld,
                            double *d, void *stream)
{
    PR_REQUIRE(G && Y2 && d, PR_EINVAL, "NULL argument");
    PR_REQUIRE(nsrc >= 1 && nsrc <= 128, PR_EINVAL, "nsrc must be 1..128");
    const long rows = G->rows;
    const int k = G->k, N = G->nloc, S = nsrc;
    PR_REQUIRE(ld >= (G->dim == 1 ? (long)N * S : rows), PR_EDIM, "ld too small");
    cudaStream_t s = (cudaStream_t)stream;
    G->stream = s;
    Scratch Sc(s);
    const Lay L = (G->dim == 1) ? Lay{ld, 1} : Lay{1, ld};
    const long blk = (G->dim == 1) ? (long)S : (long)S * ld;
    const int nchunk = xty_chunks(rows, G->N_total);
    const long cr = (rows + nchunk - 1) / nchunk;
    double *part;
    PR_ALLOC(part, double, (size_t)N * nchunk * k * 2 * S, Sc);
    XtY x{nullptr, G->V, rows * k, k, 1, k, Y1 ? Y1 : Y2, blk, L.rs, L.vs, S, rows, N, nchunk, cr, part};
    int pcols = 0;
    if (Y1) PR_CUDA(launch_xty_diff(x, Y2, S, pcols, s));
    else PR_CUDA(launch_xty(x, s));
    PR_CUDA(launch_reduce_pq(part, N, nchunk, k, S, pcols, G->sigma, G->l, d, s));
    return PR_OK;
}

pr_status pr_reduced_sweep(const double *C, const double *d, int N, int k, int nsrc, double *e,
                           void *stream)
{
    PR_REQUIRE(C && d && e && N >= 1 && k >= 1 && nsrc >= 1, PR_EINVAL, "bad sweep arguments");
    PR_CUDA(launch_sweep(C, d, N, k, nsrc, e, (cudaStream_t)stream));
    return PR_OK;
}

pr_status pr_coarse_expand(pr_coarse G, int nsrc, const double *Fu, const double *e, double *out,
                           long ld, double *upd, void *stream)
{
    PR_REQUIRE(G && Fu && e && out, PR_EINVAL, "NULL argument");
    PR_REQUIRE(nsrc >= 1 && nsrc <= 128, PR_EINVAL, "nsrc must be 1..128");
    const long rows = G->rows;
    const int k = G->k, N = G->nloc, S = nsrc;
    PR_REQUIRE(ld >= (G->dim == 1 ? (long)N * S : rows), PR_EDIM, "ld too small");
    cudaStream_t s = (cudaStream_t)stream;
    G->stream = s;
    Scratch Sc(s);
    const Lay L = (G->dim == 1) ? Lay{ld, 1} : Lay{1, ld};
    const int nchunk = xty_chunks(rows, G->N_total);
    const long cr = (rows + nchunk - 1) / nchunk;
    double *npart = nullptr;
    if (upd) PR_ALLOC(npart, double, (size_t)N * S * nchunk, Sc);
    Expand ex{out, L.rs, L.vs, Fu, L.rs, L.vs, G->U, rows * k, e, k, S, N, rows, nchunk, cr, npart};
    PR_CUDA(launch_expand(ex, s));
    if (upd) PR_CUDA(launch_norm_finish(npart, N * S, nchunk, upd, s));
    return PR_OK;
}

// ------------------------------------------------------------------ bounds
static double log_binom(int n, int k)
{
    return lgamma((double)n + 1.0) - lgamma((double)k + 1.0) - lgamma((double)(n - k) + 1.0);
}

pr_status pr_bounds(double delta, double eps, int N, int K, const double *bnorm, const double *upd,
                    double *apriori, double *apost, double *apost_sup)
{
    PR_REQUIRE(N >= 1 && K >= 0 && delta >= 0 && eps >= 0, PR_EINVAL, "bad bound arguments");
    PR_REQUIRE(!apriori || bnorm, PR_EINVAL, "apriori needs bnorm");
    PR_REQUIRE((!apost && !apost_sup) || upd, PR_EINVAL, "a posteriori bounds need upd");
    const int W = N + 1;
    if (apriori) {
        for (int n = 0; n <= N; ++n) {
            // eq. error_bound_initial
            double s = 0.0;
            for (int mm = 0; mm < n; ++mm)
                s += std::min(2.0 * delta, (n - mm) * eps) * pow(delta, n - mm - 1) * bnorm[mm];
            apriori[n] = s;
        }
        for (int k = 1; k <= K; ++k)
            for (int n = 0; n <= N; ++n) {
                // eq. error_bound_eps_delta2, log space
                double s = 0.0;
                if (eps > 0.0)
                    for (int mm = 0; mm <= n - k - 1; ++mm) {
                        if (!(bnorm[mm] > 0.0)) continue;
                        double lg = log(2.0) + k * log(eps) + log_binom(n - mm, k) +
                                    (n - mm - k) * (delta > 0 ? log(delta) : -INFINITY) + log(bnorm[mm]);
                        if (n - mm - k == 0) lg = log(2.0) + k * log(eps) + log_binom(n - mm, k) + log(bnorm[mm]);
                        s += exp(lg);
                    }
                apriori[(size_t)k * W + n] = s;
            }
    }
    for (int k = 1; k <= K; ++k) {
        const double *u = upd + (size_t)(k - 1) * W;
        if (apost)
            for (int n = 0; n <= N; ++n) {
                double s = 0.0;   // eq. apost_bound
                for (int mm = 1; mm <= n - 1; ++mm) s += pow(delta, n - mm - 1) * u[mm];
                apost[(size_t)(k - 1) * W + n] = eps * s;
            }
        if (apost_sup) {
            double mx = 0.0;
            for (int n = 1; n <= N; ++n) mx = std::max(mx, u[n]);
            apost_sup[k - 1] = (delta < 1.0) ? eps / (1.0 - delta) * mx : NAN;   // eq. apost_bound_sup
        }
    }
    return PR_OK;
}

// ============================================================ reporting
// (the sequential fine reference, the max-over-time error
// of the paper's figures, the estimator efficiency eta^k, and the classical
// Parareal baselines G = 0 and G = one coarse backward-Euler step.)

pr_status pr_sequential(pr_op h, int nsrc, const double *u0, long ld_u0, const pr_source *f, int N, int m,
                        double *U_out, long ld_out, void *stream)
{
    PR_REQUIRE(h && u0 && U_out, PR_EINVAL, "NULL argument");
    const Op &op = h->op;
    PR_REQUIRE(nsrc >= 1 && N >= 1 && m >= 0, PR_EINVAL, "bad sizes");
    const long rows = op.rows;
    const long nvec = (long)(N + 1) * nsrc;
    PR_REQUIRE(ld_out >= ((op.dim == 1) ? nvec : rows), PR_EDIM, "ld_out too small");
    PR_REQUIRE(ld_u0 >= ((op.dim == 1) ? nsrc : rows), PR_EDIM, "ld_u0 too small");
    {
        pr_status st = check_source(op, f, 0, m, N);
        if (st != PR_OK) return st;
        if (op.dim == 1 && f->kind == PR_SRC_SEP1D)
            PR_REQUIRE(f->nsrc == nsrc, PR_EDIM, "source nsrc must equal nsrc");
    }
    cudaStream_t s = (cudaStream_t)stream;
    Lay L = lay(op, ld_out), L0 = lay(op, ld_u0);
    const long blk = (op.dim == 1) ? (long)nsrc : (long)nsrc * ld_out;
    PR_CUDA(launch_copy_vectors(u0, L0.rs, L0.vs, U_out, L.rs, L.vs, rows, nsrc, s));
    for (int q = 0; q < N; ++q) {       // u_{q+1} = F_{q+1} u_q
        pr_status st = propagate(op, PR_AFFINE, q, m, nsrc, nsrc, f, U_out + q * blk, ld_out,
                                 U_out + (q + 1) * blk, ld_out, nullptr, 0, 0, 0, s);
        if (st != PR_OK) return st;
    }
    return PR_OK;
}

pr_status pr_trajectory_error(pr_op h, int nsrc, int N, int m, const double *U, long ldU,
                              const double *Uref, long ldR, double *err_host, double *ivl_host,
                              void *stream)
{
    PR_REQUIRE(h && U && Uref && err_host, PR_EINVAL, "NULL argument");
    const Op &op = h->op;
    PR_REQUIRE(nsrc >= 1 && N >= 1 && m >= 1, PR_EINVAL, "bad sizes");
    PR_REQUIRE(ldU == ldR, PR_EDIM, "U and Uref must share the leading dimension");
    const long rows = op.rows;
    const int B = N * nsrc;              // error vectors at the starts of intervals 1..N
    PR_REQUIRE(ldU >= ((op.dim == 1) ? (long)(N + 1) * nsrc : rows), PR_EDIM, "ld too small");
    cudaStream_t s = (cudaStream_t)stream;
    Scratch Sc(s);
    const long ld = ldU;
    Lay L = lay(op, ld);
    const size_t arr = (op.dim == 1) ? (size_t)rows * ld : (size_t)B * ld;
    double *E, *mx, *nrm, *npart;
    PR_ALLOC(E, double, arr, Sc);
    PR_ALLOC(mx, double, (size_t)B, Sc);
    PR_ALLOC(nrm, double, (size_t)B, Sc);
    const int nchunk = xty_chunks(rows, N);
    const long cr = (rows + nchunk - 1) / nchunk;
    PR_ALLOC(npart, double, (size_t)B * nchunk, Sc);
    // e_{q-1} = u^k_{q-1} - u_{q-1}: the source cancels, so the trajectory error
    // inside interval q is the LINEAR propagation of e_{q-1} (eq. F_n_affine)
    note_launch();
    k_vdiff<<<(unsigned)((rows * B + 255) / 256), 256, 0, s>>>(U, Uref, L.rs, L.vs, rows, B, E);
    PR_CHECK_LAUNCH("k_vdiff");
    PR_CUDA(launch_vecnorm_parts(E, L.rs, L.vs, rows, B, nchunk, cr, npart, s));
    PR_CUDA(launch_norm_finish(npart, B, nchunk, mx, s));
    for (int j = 1; j <= m; ++j) {
        pr_status st = propagate(op, PR_LINEAR, 0, 1, B, nsrc, nullptr, E, ld, E, ld, nullptr, 0, 0, 0, s,
                                 0ULL, j - 1, m);
        if (st != PR_OK) return st;
        PR_CUDA(launch_vecnorm_parts(E, L.rs, L.vs, rows, B, nchunk, cr, npart, s));
        PR_CUDA(launch_norm_finish(npart, B, nchunk, nrm, s));
        // t in [t_{q-1}, t_q) for every interval; t = T (j = m) for the last one (R-TRAJ)
        const int lo = (j < m) ? 0 : (N - 1) * nsrc;
        note_launch();
        k_runmax<<<(B + 127) / 128, 128, 0, s>>>(mx, nrm, lo, B);
        PR_CHECK_LAUNCH("k_runmax");
    }
    std::vector<double> hm(B);
    PR_CUDA(cudaMemcpyAsync(hm.data(), mx, B * sizeof(double), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    for (int sI = 0; sI < nsrc; ++sI) {
        double e = 0.0;
        for (int q = 0; q < N; ++q) e = std::max(e, hm[(size_t)q * nsrc + sI]);
        err_host[sI] = e;
    }
    if (ivl_host) memcpy(ivl_host, hm.data(), B * sizeof(double));
    return PR_OK;
}

pr_status pr_efficiency(double delta, double eps, int N, int K, const double *upd, const double *traj_err,
                        double *eta)
{
    PR_REQUIRE(N >= 2 && K >= 1 && upd && traj_err && eta, PR_EINVAL, "bad arguments");
    const int W = N + 1;
    for (int k = 1; k <= K; ++k) {
        const double *u = upd + (size_t)(k - 1) * W;
        double den = 0.0;              // eq. def_efficiency: max over 1 <= n < N (as printed, Z21)
        for (int n = 1; n < N; ++n) {
            double acc = 0.0;
            for (int mm = 1; mm <= n - 1; ++mm) acc += pow(delta, n - mm - 1) * u[mm];
            den = std::max(den, eps * acc);
        }
        eta[k - 1] = traj_err[k] / den;
    }
    return PR_OK;
}

pr_status pr_parareal_classical(pr_op coarse, const pr_source *fc, pr_op h, int nsrc, const double *u0,
                                long ld_u0, const pr_source *f, int N, int m, int K_iter, double *U_out,
                                long ld_out, double *upd_host, double *hist, long hist_stride, void *stream)
{
    PR_REQUIRE(h && u0 && U_out, PR_EINVAL, "NULL argument");
    const Op &op = h->op;
    PR_REQUIRE(nsrc >= 1 && N >= 1 && m >= 0 && K_iter >= 0, PR_EINVAL, "bad sizes");
    const long rows = op.rows;
    const int S = nsrc;
    const long nvec = (long)(N + 1) * S;
    PR_REQUIRE(ld_out >= ((op.dim == 1) ? nvec : rows), PR_EDIM, "ld_out too small");
    PR_REQUIRE(ld_u0 >= ((op.dim == 1) ? S : rows), PR_EDIM, "ld_u0 too small");
    if (coarse) {
        PR_REQUIRE(coarse->op.rows == rows && coarse->op.dim == op.dim, PR_EDIM, "coarse / fine operator mismatch");
        pr_status st = check_source(coarse->op, fc, 0, 1, N);
        if (st != PR_OK) return st;
    }
    {
        pr_status st = check_source(op, f, 0, m, N);
        if (st != PR_OK) return st;
    }
    cudaStream_t s = (cudaStream_t)stream;
    Scratch Sc(s);
    const long ld = ld_out;
    Lay L = lay(op, ld), L0 = lay(op, ld_u0);
    const size_t arr = (op.dim == 1) ? (size_t)rows * ld : (size_t)nvec * ld;
    const long blk = (op.dim == 1) ? (long)S : (long)S * ld;
    double *Fu, *Gu, *Uold, *npart, *upd;
    PR_ALLOC(Fu, double, arr, Sc);
    PR_ALLOC(Gu, double, arr, Sc);
    PR_ALLOC(Uold, double, arr, Sc);
    const int nchunk = xty_chunks(rows, N);
    const long cr = (rows + nchunk - 1) / nchunk;
    PR_ALLOC(npart, double, (size_t)nvec * nchunk, Sc);
    PR_ALLOC(upd, double, (size_t)(K_iter > 0 ? K_iter : 1) * nvec, Sc);
    pr_status st;
    // G_{q+1} x (+ off): one backward-Euler step of the coarse operator over
    // interval q+1 (its step q+1, time step Delta T), or 0
    auto Gstep = [&](int q, int nb, const double *in, double *out, const double *off) -> pr_status {
        if (coarse)
            return propagate(coarse->op, PR_AFFINE, q, 1, nb * S, S, fc, in, ld, out, ld, off, ld, 0, 0, s);
        if (off) PR_CUDA(launch_copy_vectors(off, L.rs, L.vs, out, L.rs, L.vs, rows, nb * S, s));
        else if (op.dim == 1) PR_CUDA(cudaMemset2DAsync(out, ld * sizeof(double), 0, nb * S * sizeof(double), rows, s));
        else PR_CUDA(cudaMemsetAsync(out, 0, (size_t)nb * S * ld * sizeof(double), s));
        return PR_OK;
    };
    // initialisation u^0_0 = u0, u^0_{q+1} = G_{q+1} u^0_q
    PR_CUDA(launch_copy_vectors(u0, L0.rs, L0.vs, U_out, L.rs, L.vs, rows, S, s));
    for (int q = 0; q < N; ++q)
        if ((st = Gstep(q, 1, U_out + q * blk, U_out + (q + 1) * blk, nullptr)) != PR_OK) return st;
    if (hist) PR_CUDA(launch_copy_vectors(U_out, L.rs, L.vs, hist, L.rs, L.vs, rows, (int)nvec, s));
    for (int it = 1; it <= K_iter; ++it) {
        PR_CUDA(launch_copy_vectors(U_out, L.rs, L.vs, Uold, L.rs, L.vs, rows, (int)nvec, s));
        // F_{q+1} u^k_q and G_{q+1} u^k_q for all q (parallel)
        if ((st = propagate(op, PR_AFFINE, 0, m, N * S, S, f, Uold, ld, Fu + blk, ld, nullptr, 0, 0, 0, s)) != PR_OK)
            return st;
        if ((st = Gstep(0, N, Uold, Gu + blk, nullptr)) != PR_OK) return st;
        // c_{q+1} = F u^k_q - G u^k_q into Fu
        note_launch();
        k_vdiff<<<(unsigned)((rows * N * S + 255) / 256), 256, 0, s>>>(Fu + blk, Gu + blk, L.rs, L.vs, rows,
                                                                         N * S, Fu + blk);
        PR_CHECK_LAUNCH("k_vdiff");
        // sequential sweep u^{k+1}_{q+1} = G_{q+1} u^{k+1}_q + c_{q+1} (eq. def_Parareal)
        for (int q = 0; q < N; ++q)
            if ((st = Gstep(q, 1, U_out + q * blk, U_out + (q + 1) * blk, Fu + (q + 1) * blk)) != PR_OK) return st;
        // update norms ||u^{k+1}_j - u^k_j||, all boundaries
        note_launch();
        k_vdiff<<<(unsigned)((rows * nvec + 255) / 256), 256, 0, s>>>(U_out, Uold, L.rs, L.vs, rows, (int)nvec, Gu);
        PR_CHECK_LAUNCH("k_vdiff");
        PR_CUDA(launch_vecnorm_parts(Gu, L.rs, L.vs, rows, (int)nvec, nchunk, cr, npart, s));
        PR_CUDA(launch_norm_finish(npart, (int)nvec, nchunk, upd + (size_t)(it - 1) * nvec, s));
        if (hist)
            PR_CUDA(launch_copy_vectors(U_out, L.rs, L.vs, hist + (size_t)it * hist_stride, L.rs, L.vs, rows,
                                        (int)nvec, s));
    }
    if (upd_host && K_iter > 0)
        PR_CUDA(cudaMemcpyAsync(upd_host, upd, (size_t)K_iter * nvec * sizeof(double), cudaMemcpyDeviceToHost, s));
    PR_CUDA(cudaStreamSynchronize(s));
    return PR_OK;
}

}  // extern "C"
