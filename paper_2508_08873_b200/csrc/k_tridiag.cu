// k_tridiag.cu -- K1: batched 1D backward-Euler stepper (the hot loop of
// rSVD steps 1 and 3 and of every Parareal fine solve), its one-time
// factorisation, and the fused Gaussian sketch generator (K3).
//
// Paper: fine solver = backward Euler; rSVD step 1 draws
// Gaussian omega_i and computes F_n' omega_i; step 3 applies the
// adjoint; F_n v = F_n' v + b_n.
//
// Layout: B vectors interleaved, element (row i, vector c) at U[i*ld + c].
// A warp owns 32*VPT consecutive vectors; every row it touches is one
// contiguous 256*VPT-byte segment.  Each thread runs the whole m-step solve
// of its own VPT vectors: no inter-thread dependency at all.
//
// Pass fusion: odd steps use I + dt A = L U (down: forward
// elimination, up: back substitution), even steps use I + dt A = U~ L~ (up,
// then down).  The up sweep that finishes step s is fused with the up sweep
// that starts step s+1 (and likewise down), so m steps take m+1 streaming
// passes over the state instead of 2m: 16 B of HBM traffic per DOF-step.
//
// Memory pipeline: each thread streams its own column through a per-warp
// shared-memory ring with cp.async (PD groups of 32 rows in flight); the
// per-row coefficients are loaded one group ahead distributed over the 32
// lanes and broadcast with shuffles.
#include "pr_internal.cuh"

namespace pr {

// ------------------------------------------------------------ factorisation
// One thread computes the LU pivots top-down, another the UL pivots
// bottom-up, both from row sums (reading R-ACC):
//   LU: r_0 = s_0, r_i = s_i - a_i r_{i-1} / den_{i-1},  den_i = r_i - c_i
//   UL: r_{n-1} = s_{n-1}, r_i = s_i - c_i r_{i+1} / den~_{i+1}, den~_i = r_i - a_i
// a_i = (I+dtA)[i,i-1], c_i = (I+dtA)[i,i+1], s_i = 1 + dt * rowsum(A)_i.
__global__ void k_factor(int n, const double *__restrict__ subA, const double *__restrict__ supA,
                         const double *__restrict__ rsA, const double *__restrict__ diagA,
                         double dt, int transpose, Coef *DN, Coef *UP, int *bad)
{
    auto a_of = [&](int i) -> double {
        if (i <= 0) return 0.0;
        return dt * (transpose ? supA[i - 1] : subA[i]);
    };
    auto c_of = [&](int i) -> double {
        if (i >= n - 1) return 0.0;
        return dt * (transpose ? subA[i + 1] : supA[i]);
    };
    auto s_of = [&](int i) -> double {
        if (rsA) return 1.0 + dt * rsA[i];
        // no exact sums given: form them from the stencil entries of this orientation
        double d = 1.0 + dt * diagA[i];
        return a_of(i) + d + c_of(i);
    };
    if (threadIdx.x == 0) {                   // LU, top-down
        double r = 0.0, den = 1.0;
        for (int i = 0; i < n; ++i) {
            double ai = a_of(i), ci = c_of(i);
            r = (i == 0) ? s_of(0) : s_of(i) - ai * (r / den);
            den = r - ci;
            if (!(den > 0.0) || !isfinite(den)) atomicExch(bad, 1);
            double w = 1.0 / den;
            DN[i].b = w;
            DN[i].c = w * ai;                 // ga_i
            UP[i].a = w * ci;                 // cp_i
            DN[i].d = 0.0;
            UP[i].d = 0.0;
        }
    } else if (threadIdx.x == 1) {            // UL, bottom-up
        double r = 0.0, den = 1.0;
        for (int i = n - 1; i >= 0; --i) {
            double ai = a_of(i), ci = c_of(i);
            r = (i == n - 1) ? s_of(n - 1) : s_of(i) - ci * (r / den);
            den = r - ai;
            if (!(den > 0.0) || !isfinite(den)) atomicExch(bad, 1);
            double w = 1.0 / den;
            UP[i].b = w;                      // wt_i
            UP[i].c = w * ci;                 // gc_i
            DN[i].a = w * ai;                 // ap_i
        }
    }
}

cudaError_t launch_factor_1d(int n, const double *subA, const double *supA, const double *rsA,
                                  const double *diagA, double dt, int transpose, Coef *DN,
                                  Coef *UP, int *bad, cudaStream_t s)
{
    k_factor<<<1, 32, 0, s>>>(n, subA, supA, rsA, diagA, dt, transpose, DN, UP, bad);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- Philox
__device__ __forceinline__ void philox4x64_10(unsigned long long c[4], unsigned long long k0,
                                              unsigned long long k1)
{
    const unsigned long long M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    const unsigned long long W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += W0; k1 += W1; }
        unsigned long long hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
        unsigned long long hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
        unsigned long long n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
}

// Four N(0,1) values for rows 4*blk .. 4*blk+3 of column col of interval q.
__device__ __forceinline__ void gauss4(unsigned long long seed, unsigned long long blk, int col,
                                       int q, double z[4])
{
    unsigned long long c[4] = {blk, (unsigned long long)col, (unsigned long long)q, 0ULL};
    philox4x64_10(c, seed, 0ULL);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double u1 = ((double)(c[2 * h] >> 11) + 1.0) * 0x1.0p-53;
        double u2 = (double)(c[2 * h + 1] >> 11) * 0x1.0p-53;
        double r = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        z[2 * h] = r * cs;
        z[2 * h + 1] = r * sn;
    }
}

__global__ void k_sketch(int dim, int n, long rows, int q0, int nint, int l,
                         unsigned long long seed, double *out, long rs, long vs)
{
    // one thread = 4 consecutive interior DOFs of one column
    long ndof = (dim == 1) ? n : (long)n * n;
    long nb = (ndof + 3) / 4;
    long tid = (long)blockIdx.x * blockDim.x + threadIdx.x;
    long total = nb * (long)nint * l;
    if (tid >= total) return;
    long blk = tid % nb;
    long v = tid / nb;                // vector within the output
    int q = q0 + (int)(v / l);
    int col = (int)(v % l);
    double z[4];
    gauss4(seed, (unsigned long long)blk, col, q, z);
    for (int h = 0; h < 4; ++h) {
        long dof = blk * 4 + h;
        if (dof >= ndof) break;
        long row = dof;
        if (dim == 2) {
            long ix = dof / n, iy = dof % n;
            row = (ix + 1) * (n + 1) + (iy + 1);
        }
        out[row * rs + v * vs] = z[h];
    }
    (void)rows;
}

cudaError_t launch_sketch(int dim, int n, long rows, int q0, int nint, int l,
                          unsigned long long seed, double *out, long rs, long vs, cudaStream_t s)
{
    long ndof = (dim == 1) ? n : (long)n * n;
    long total = ((ndof + 3) / 4) * (long)nint * l;
    if (total == 0) return cudaSuccess;
    int th = 256;
    long bl = (total + th - 1) / th;
    k_sketch<<<(unsigned)bl, th, 0, s>>>(dim, n, rows, q0, nint, l, seed, out, rs, vs);
    return cudaGetLastError();
}

__global__ void k_transpose(const double *in, int R, int n, double *out)
{
    long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long)R * n) return;
    int r = (int)(t / n), i = (int)(t % n);
    out[(long)i * R + r] = in[t];
}

cudaError_t launch_transpose(const double *in, int R, int n, double *out, cudaStream_t s)
{
    long total = (long)R * n;
    k_transpose<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(in, R, n, out);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- stepper
constexpr int GR = 32;   // rows per group (one coefficient row per lane)
constexpr int PD = 2;    // groups in flight ahead of the one being computed
constexpr int RING = PD + 1;
constexpr int SWARPS = 1;  // warps per CTA (small CTAs: every warp resident, fine balance)

template <int VPT>
struct VecT;
template <>
struct VecT<1> { using T = double; };
template <>
struct VecT<2> { using T = double2; };

__device__ __forceinline__ void cp_async_8(void *smem, const void *gmem)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_16(void *smem, const void *gmem)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int VPT>
__device__ __forceinline__ void cp_async_vec(double *smem, const double *gmem)
{
    if (VPT == 1) cp_async_8(smem, gmem);
    else cp_async_16(smem, gmem);
}

// Stepper kernel.  AFF: source terms present (R in 1..8).
template <int VPT, bool AFF>
__global__ void __launch_bounds__(32 * SWARPS) k_stepper(StepArgs a)
{
    extern __shared__ __align__(16) double smem_dyn[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const long c0 = ((long)blockIdx.x * blockDim.x + threadIdx.x) * VPT;  // first vector
    const bool valid = c0 < a.B;    // B is a multiple of VPT when VPT > 1
    const bool have_off = a.off != nullptr;
    double *ring = smem_dyn + (size_t)warp * RING * GR * 32 * VPT;
    double *ringo = have_off ? smem_dyn + (size_t)(SWARPS + warp) * RING * GR * 32 * VPT : nullptr;

    const int n = a.n;
    const int ngroups = (n + GR - 1) / GR;
    const int m = a.m;
    const int P = (m > 0) ? m + 1 : 1;

    // per-vector interval / column / source
    int qv[VPT], colv[VPT], srcv[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        long c = c0 + v;
        qv[v] = a.q0 + (int)(c / a.vpi);
        colv[v] = (int)(c % a.vpi);
        srcv[v] = AFF ? (int)(c % a.nsrc) : 0;
    }

    for (int p = 1; p <= P; ++p) {
        const bool down = (p & 1);
        const bool finish = (p >= 2);
        const bool start = (p <= m);
        const bool last = (p == P);
        const bool from_in = (p == 1);
        const bool do_load = !from_in || (a.in != nullptr && !a.sketch);
        const bool gen = from_in && a.sketch;
        const double *src = from_in ? a.in : a.out;
        const long lds = from_in ? a.ld_in : a.ld_out;
        const bool load_off = last && have_off;
        const Coef *coefs = down ? a.DN : a.UP;

        // source coefficients alpha_r = dt * amp[s, r] * time[r, g-1] of step p
        double alpha[AFF ? 8 : 1][VPT];
        if (AFF) {
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int v = 0; v < VPT; ++v) {
                    double al = 0.0;
                    if (start && r < a.R && valid) {
                        long g1 = (long)qv[v] * m + p - 1;       // g - 1
                        al = a.dt * a.amp[(long)srcv[v] * a.R + r] * a.time[(long)r * a.nsteps + g1];
                    }
                    alpha[r][v] = al;
                }
        }

        auto row_of = [&](int g, int r) -> int {
            int t = g * GR + r;
            return down ? t : n - 1 - t;
        };
        auto issue = [&](int g) {
            if (g < ngroups && valid) {
                int slot0 = (g % RING) * GR;
#pragma unroll 4
                for (int r = 0; r < GR; ++r) {
                    int i = row_of(g, r);
                    if (i >= 0 && i < n) {
                        if (do_load)
                            cp_async_vec<VPT>(ring + ((size_t)(slot0 + r) * 32 + lane) * VPT,
                                              src + (long)i * lds + c0);
                        if (load_off)
                            cp_async_vec<VPT>(ringo + ((size_t)(slot0 + r) * 32 + lane) * VPT,
                                              a.off + (long)i * a.ld_off + c0);
                    }
                }
            }
            cp_async_commit();
        };

        // prologue
#pragma unroll
        for (int g = 0; g < PD; ++g) issue(g);
        Coef cnext;
        double snext[AFF ? 8 : 1];
        {
            int i = row_of(0, lane);
            bool ok = (i >= 0 && i < n);
            cnext = ok ? coefs[i] : Coef{0, 0, 0, 0};
            if (AFF) {
#pragma unroll
                for (int r = 0; r < 8; ++r) snext[r] = (ok && r < a.R) ? a.spaceT[(long)i * a.R + r] : 0.0;
            }
        }

        double xprev[VPT], yprev[VPT];
#pragma unroll
        for (int v = 0; v < VPT; ++v) { xprev[v] = 0.0; yprev[v] = 0.0; }
        double z4[VPT][4];

        for (int g = 0; g < ngroups; ++g) {
            issue(g + PD);
            Coef ccur = cnext;
            double scur[AFF ? 8 : 1];
            if (AFF) {
#pragma unroll
                for (int r = 0; r < 8; ++r) scur[r] = snext[r];
            }
            if (g + 1 < ngroups) {
                int i = row_of(g + 1, lane);
                bool ok = (i >= 0 && i < n);
                cnext = ok ? coefs[i] : Coef{0, 0, 0, 0};
                if (AFF) {
#pragma unroll
                    for (int r = 0; r < 8; ++r) snext[r] = (ok && r < a.R) ? a.spaceT[(long)i * a.R + r] : 0.0;
                }
            }
            cp_async_wait<PD>();
            const int slot0 = (g % RING) * GR;
#pragma unroll
            for (int r = 0; r < GR; ++r) {
                const int i = row_of(g, r);
                const bool rowok = (i >= 0 && i < n);   // warp-uniform
                const double ca = __shfl_sync(0xffffffffu, ccur.a, r);
                const double cb = __shfl_sync(0xffffffffu, ccur.b, r);
                const double cc = __shfl_sync(0xffffffffu, ccur.c, r);
                double fsrc[VPT];
#pragma unroll
                for (int v = 0; v < VPT; ++v) fsrc[v] = 0.0;
                if (AFF && start) {
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        double sp = __shfl_sync(0xffffffffu, scur[t], r);
#pragma unroll
                        for (int v = 0; v < VPT; ++v) fsrc[v] = fma(alpha[t][v], sp, fsrc[v]);
                    }
                }
                if (gen && (r & 3) == 0 && valid) {
#pragma unroll
                    for (int v = 0; v < VPT; ++v)
                        gauss4(a.seed, (unsigned long long)(i >> 2), colv[v], qv[v], z4[v]);
                }
                if (rowok && valid) {
                    double val[VPT];
                    if (do_load) {
                        const double *sp = ring + ((size_t)(slot0 + r) * 32 + lane) * VPT;
#pragma unroll
                        for (int v = 0; v < VPT; ++v) val[v] = sp[v];
                    } else if (gen) {
#pragma unroll
                        for (int v = 0; v < VPT; ++v) val[v] = z4[v][r & 3];
                    } else {
#pragma unroll
                        for (int v = 0; v < VPT; ++v) val[v] = 0.0;
                    }
                    double res[VPT];
#pragma unroll
                    for (int v = 0; v < VPT; ++v) {
                        // finish the previous step: back substitution
                        double x = finish ? fma(-ca, xprev[v], val[v]) : val[v];
                        xprev[v] = x;
                        if (start) {
                            double rr = x + fsrc[v];
                            double y = fma(cb, rr, -cc * yprev[v]);
                            yprev[v] = y;
                            res[v] = y;
                        } else {
                            res[v] = x;
                        }
                    }
                    if (last && have_off) {
                        const double *so = ringo + ((size_t)(slot0 + r) * 32 + lane) * VPT;
#pragma unroll
                        for (int v = 0; v < VPT; ++v) res[v] += so[v];
                    }
                    double *dst = a.out + (long)i * a.ld_out + c0;
                    if (VPT == 1) {
                        dst[0] = res[0];
                    } else {
                        *reinterpret_cast<double2 *>(dst) = make_double2(res[0], res[VPT - 1]);
                    }
                }
            }
        }
        cp_async_wait<0>();
        __syncwarp();
    }
}

template <int VPT, bool AFF>
static cudaError_t launch_stepper_t(const StepArgs &a, cudaStream_t s)
{
    const int threads = 32 * SWARPS;
    long nthreads = (a.B + VPT - 1) / VPT;
    long blocks = (nthreads + threads - 1) / threads;
    if (blocks == 0) return cudaSuccess;
    size_t ring_bytes = (size_t)SWARPS * RING * GR * 32 * VPT * sizeof(double);
    size_t smem = ring_bytes * (a.off ? 2 : 1);
    auto kern = k_stepper<VPT, AFF>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)blocks, threads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_stepper_1d(const StepArgs &a, cudaStream_t s)
{
    // two vectors per thread (16 B accesses) when every base and stride allows it
    auto al16 = [](const void *p) { return ((uintptr_t)p & 15) == 0; };
    bool v2 = (a.B % 2 == 0) && (a.ld_out % 2 == 0) && al16(a.out) &&
              (a.in == nullptr || a.sketch || ((a.ld_in % 2 == 0) && al16(a.in))) &&
              (a.off == nullptr || ((a.ld_off % 2 == 0) && al16(a.off)));
    bool aff = a.R > 0;
    if (v2) return aff ? launch_stepper_t<2, true>(a, s) : launch_stepper_t<2, false>(a, s);
    return aff ? launch_stepper_t<1, true>(a, s) : launch_stepper_t<1, false>(a, s);
}

}  // namespace pr
