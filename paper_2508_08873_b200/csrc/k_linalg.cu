// k_linalg.cu -- dense kernels of the randomized SVD and of the Parareal
// correction (CUDA path; no oracle code).
//
//   K4 xty / reduce_parts : tall-skinny X^T Y per interval, split over row
//                           chunks, fixed-order reduction (deterministic)
//   K5 chol / trsm        : iterated shifted CholeskyQR (rSVD steps 2 and 4,
//                           P:269-275; reading Z7)
//   K6 jacobi             : one-sided Jacobi SVD of M = R_Z^T, one CTA per
//                           interval (step 5)
//   K7 lift               : U = W Psi_k, V = V Phi_k (steps 5-6)
//   K8/K9 sweep, expand   : reduced Parareal correction (eq. def_Parareal,
//                           P:144-151) and update norms
#include <float.h>
#include <stdlib.h>

#include "pr_internal.cuh"

namespace pr {

// ------------------------------------------------------------------ X^T Y
constexpr int XT_THREADS = 256;
constexpr int XT_TR = 32;       // rows per smem tile

cudaError_t launch_xty_fma(const XtY &p, cudaStream_t s);

int xty_chunks(long rows, int nbatch)
{
    // enough CTAs to fill the machine four times (the DMMA kernels run one or
    // two CTAs per SM; more, shorter CTAs shrink the last-wave tail), at least
    // 64 rows per chunk; among up to three times that many chunks the count whose
    // grid (chunks x nbatch CTAs, two per SM) leaves the emptiest last wave
    // fullest (C4: 8 chunks x 256 intervals = 6.92 waves instead of 3 x 256 = 2.59)
    long want = (4L * num_sms() + nbatch - 1) / nbatch;
    long maxc = (rows + 63) / 64;
    if (maxc > 256) maxc = 256;
    if (want < 1) want = 1;
    if (want >= maxc) return (int)(maxc < 1 ? 1 : maxc);
    long hi = 3 * want < maxc ? 3 * want : maxc;
    const long slots = 2L * num_sms();
    long best = want;
    double best_eff = 0.0;
    for (long c = want; c <= hi; ++c) {
        const long total = c * nbatch;
        const double eff = (double)total / (double)(((total + slots - 1) / slots) * slots);
        if (eff > best_eff + 0.02) { best_eff = eff; best = c; }
    }
    return (int)best;
}

template <int BPT>
__global__ void __launch_bounds__(XT_THREADS) k_xty(XtY p)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y, t = blockIdx.x;
    if (p.skip && p.skip[b] == 2) return;
    const int A4 = (p.a + 3) & ~3, C4 = (p.c + p.c2 + 3) & ~3;
    double *Xs = sm;                     // [XT_TR][A4]
    double *Ys = sm + XT_TR * A4;        // [XT_TR][C4]
    const int ctot = p.c + p.c2;
    const bool same = (p.X == p.Y) && (p.xbs == p.ybs) && (p.xrs == p.yrs) && (p.xcs == p.ycs) &&
                      (p.a == p.c) && p.c2 == 0;
    if (same) Ys = Xs;
    const int nbi = A4 / 4, nbj = C4 / 4;
    const int nblk = nbi * nbj;
    double acc[BPT][16];
#pragma unroll
    for (int q = 0; q < BPT; ++q)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[q][e] = 0.0;

    const long r0 = (long)t * p.chunk_rows;
    long r1 = r0 + p.chunk_rows;
    if (r1 > p.rows) r1 = p.rows;
    const double *Xb = p.X + (long)b * p.xbs;
    const double *Yb = p.Y + (long)b * p.ybs;
    const double *Y2b = p.Y2 ? p.Y2 + (long)b * p.ybs : nullptr;

    for (long rt = r0; rt < r1; rt += XT_TR) {
        __syncthreads();
        // cooperative coalesced tile loads (zero-filled beyond rows / columns)
        auto load = [&](const double *Bp, long rs, long cs, int ncol, int C, double *dst) {
            const int tot = XT_TR * C;
            for (int idx = threadIdx.x; idx < tot; idx += XT_THREADS) {
                int r, j;
                if (cs == 1) { r = idx / C; j = idx % C; }
                else { j = idx / XT_TR; r = idx % XT_TR; }
                long row = rt + r;
                double v = 0.0;
                if (row < r1 && j < ncol) v = Bp[row * rs + (long)j * cs];
                dst[r * C + j] = v;
            }
        };
        load(Xb, p.xrs, p.xcs, p.a, A4, Xs);
        if (!same) {
            if (!Y2b) {
                load(Yb, p.yrs, p.ycs, p.c, C4, Ys);
            } else {
                // columns [0, c) from Y, [c, c + c2) from Y2 (same strides)
                const int tot = XT_TR * C4;
                for (int idx = threadIdx.x; idx < tot; idx += XT_THREADS) {
                    int r, j;
                    if (p.ycs == 1) { r = idx / C4; j = idx % C4; }
                    else { j = idx / XT_TR; r = idx % XT_TR; }
                    long row = rt + r;
                    double v = 0.0;
                    if (row < r1 && j < ctot) {
                        const double *src = (j < p.c) ? Yb : Y2b;
                        int jj = (j < p.c) ? j : j - p.c;
                        v = src[row * p.yrs + (long)jj * p.ycs];
                    }
                    Ys[r * C4 + j] = v;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < BPT; ++q) {
            int blk = threadIdx.x + q * XT_THREADS;
            if (blk < nblk) {
                int bi = blk / nbj, bj = blk % nbj;
#pragma unroll 4
                for (int r = 0; r < XT_TR; ++r) {
                    const double2 *xp = reinterpret_cast<const double2 *>(Xs + r * A4 + 4 * bi);
                    const double2 *yp = reinterpret_cast<const double2 *>(Ys + r * C4 + 4 * bj);
                    double2 x01 = xp[0], x23 = xp[1], y01 = yp[0], y23 = yp[1];
                    double x[4] = {x01.x, x01.y, x23.x, x23.y};
                    double y[4] = {y01.x, y01.y, y23.x, y23.y};
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[q][u * 4 + v] = fma(x[u], y[v], acc[q][u * 4 + v]);
                }
            }
        }
    }
    double *out = p.part + ((long)b * p.nchunk + t) * p.a * ctot;
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        int blk = threadIdx.x + q * XT_THREADS;
        if (blk < nblk) {
            int bi = blk / nbj, bj = blk % nbj;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    int i = 4 * bi + u, j = 4 * bj + v;
                    if (i < p.a && j < ctot) out[(long)i * ctot + j] = acc[q][u * 4 + v];
                }
        }
    }
}

// ---- X^T Y on FP64 tensor cores (DMMA m8n8k4).  A CTA accumulates the whole
// a x c output over its row chunk: rows are the K dimension, streamed through
// a 2-stage cp.async ring of XM_TR rows.  Warp w owns output tile-columns
// w, w+8 (8 columns each) and every tile-row.  CM selects the shared layout:
// false = row-major tiles (1D layout: a row's columns contiguous in HBM),
// true = column-major tiles (2D layout: a column's rows contiguous).  Row
// strides are 4 (mod 16) doubles, which makes the fragment loads conflict-free.
constexpr int XM_TR = 32;
constexpr int XM_THREADS = 256;

__device__ __forceinline__ void dmma_f64(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cpa8_zfill(double *smem, const double *gmem, bool valid)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}

__host__ __device__ inline int xm_stride(int w) { return ((w + 15) / 16) * 16 + 4; }

// Warp layout: NGR = 16 / NQ groups of MS warps; warp (group wn, member ms)
// owns tile-columns wn, wn + NGR, ... (NQ of them) and a contiguous 1/MS share
// of the tile-rows (at most MTM).
template <bool CM, int MTM, int NQ, int MS>
__global__ void __launch_bounds__(512 / NQ * MS) k_xty_mma(XtY p)
{
    constexpr int NGR = 16 / NQ, NWARP = NGR * MS, NTH = 32 * NWARP;
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y, t = blockIdx.x;
    if (p.skip && p.skip[b] == 2) return;
    const int ctot = p.c + p.c2;
    const int MT = (p.a + 7) / 8, NT = (ctot + 7) / 8;
    // stage sizes (doubles)
    const int SXr = xm_stride(p.a), SYr = xm_stride(ctot);   // row-major strides
    const int SC = XM_TR + 4;                                  // column-major stride
    const int xsz = CM ? MT * 8 * SC : XM_TR * SXr;
    const int ysz = CM ? NT * 8 * SC : XM_TR * SYr;
    double *Xs = sm, *Ys = sm + 2 * xsz;
    const long r0 = (long)t * p.chunk_rows;
    long r1 = r0 + p.chunk_rows;
    if (r1 > p.rows) r1 = p.rows;
    const double *Xb = p.X + (long)b * p.xbs;
    const double *Yb = p.Y + (long)b * p.ybs;
    const double *Y2b = p.Y2 ? p.Y2 + (long)b * p.ybs : nullptr;
    // a Gram matrix (Y == X) stages its operand once
    const bool same = (p.X == p.Y) && (p.xbs == p.ybs) && (p.xrs == p.yrs) && (p.xcs == p.ycs) && (p.a == p.c) &&
                      p.c2 == 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int wn = w / MS, ms = w % MS;
    const int mtm = (MT + MS - 1) / MS, m0 = ms * mtm;      // this warp's tile-rows m0 + i, i < mtm

    // column-major tiles (2D layout): rows of a column are contiguous, so the
    // tile is staged in 16-byte pieces (2 rows) when the strides allow it
    const bool v16 = CM && (p.xcs % 2 == 0) && (p.ycs % 2 == 0) && (p.xbs % 2 == 0) && (p.ybs % 2 == 0) &&
                     (r0 % 2 == 0) && ((uintptr_t)p.X % 16 == 0) && ((uintptr_t)p.Y % 16 == 0) &&
                     (p.Y2 == nullptr || (uintptr_t)p.Y2 % 16 == 0);
    auto stage = [&](long rt, int buf) {
        double *xs = Xs + buf * xsz, *ys = Ys + buf * ysz;
        const int ax = MT * 8, cy = NT * 8;
        if (v16) {
            constexpr int HR = XM_TR / 2;
            for (int e = threadIdx.x; e < HR * ax; e += NTH) {
                const int i = e / HR, r = 2 * (e % HR);
                const long row = rt + r;
                const int nb = (i < p.a) ? (row + 1 < r1 ? 16 : (row < r1 ? 8 : 0)) : 0;
                const double *src = nb ? Xb + row + (long)i * p.xcs : Xb;
                unsigned sd = (unsigned)__cvta_generic_to_shared(xs + i * SC + r);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sd), "l"(src), "r"(nb) : "memory");
            }
            for (int e = threadIdx.x; e < (same ? 0 : HR * cy); e += NTH) {
                const int j = e / HR, r = 2 * (e % HR);
                const long row = rt + r;
                const int nb = (j < ctot) ? (row + 1 < r1 ? 16 : (row < r1 ? 8 : 0)) : 0;
                const double *src = Yb;
                if (nb) src = (j < p.c) ? Yb + row + (long)j * p.ycs : Y2b + row + (long)(j - p.c) * p.ycs;
                unsigned sd = (unsigned)__cvta_generic_to_shared(ys + j * SC + r);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sd), "l"(src), "r"(nb) : "memory");
            }
        } else {
        for (int e = threadIdx.x; e < XM_TR * ax; e += NTH) {
            int r, i;
            if (CM) { i = e / XM_TR; r = e % XM_TR; } else { r = e / ax; i = e % ax; }
            const long row = rt + r;
            const bool ok = row < r1 && i < p.a;
            cpa8_zfill(xs + (CM ? i * SC + r : r * SXr + i), ok ? Xb + row * p.xrs + (long)i * p.xcs : Xb, ok);
        }
        for (int e = threadIdx.x; e < (same ? 0 : XM_TR * cy); e += NTH) {
            int r, j;
            if (CM) { j = e / XM_TR; r = e % XM_TR; } else { r = e / cy; j = e % cy; }
            const long row = rt + r;
            const bool ok = row < r1 && j < ctot;
            const double *src = Yb;
            if (ok) src = (j < p.c) ? Yb + row * p.yrs + (long)j * p.ycs
                                    : Y2b + row * p.yrs + (long)(j - p.c) * p.ycs;
            cpa8_zfill(ys + (CM ? j * SC + r : r * SYr + j), src, ok);
        }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    double acc[NQ][MTM][2];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int i = 0; i < MTM; ++i) acc[q][i][0] = acc[q][i][1] = 0.0;

    const int ntiles = (int)((r1 - r0 + XM_TR - 1) / XM_TR);
    if (ntiles > 0) stage(r0, 0);
    for (int it = 0; it < ntiles; ++it) {
        if (it + 1 < ntiles) {
            stage(r0 + (long)(it + 1) * XM_TR, (it + 1) & 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const double *xs = Xs + (it & 1) * xsz, *ys = same ? xs : Ys + (it & 1) * ysz;
#pragma unroll
        for (int ks = 0; ks < XM_TR / 4; ++ks) {
            const int k = ks * 4 + tq;
            double af[MTM];
#pragma unroll
            for (int i = 0; i < MTM; ++i) {
                const int mi = m0 + i;
                af[i] = (i < mtm && mi < MT) ? (CM ? xs[(mi * 8 + gq) * SC + k] : xs[k * SXr + mi * 8 + gq]) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int nj = wn + NGR * q;
                if (nj < NT) {
                    const double bf = CM ? ys[(nj * 8 + gq) * SC + k] : ys[k * SYr + nj * 8 + gq];
#pragma unroll
                    for (int i = 0; i < MTM; ++i)
                        if (i < mtm && m0 + i < MT) dmma_f64(acc[q][i][0], acc[q][i][1], af[i], bf);
                }
            }
        }
        __syncthreads();
    }
    double *out = p.part + ((long)b * p.nchunk + t) * p.a * ctot;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int nj = wn + NGR * q;
        if (nj >= NT) continue;
#pragma unroll
        for (int ii = 0; ii < MTM; ++ii) {
            const int mi = m0 + ii;
            if (ii >= mtm || mi >= MT) continue;
            const int i = mi * 8 + gq, j = nj * 8 + 2 * tq;
            if (i < p.a) {
                if (j < ctot) out[(long)i * ctot + j] = acc[q][ii][0];
                if (j + 1 < ctot) out[(long)i * ctot + j + 1] = acc[q][ii][1];
            }
        }
    }
}

// ---- X^T Y on FP64 tensor cores for the 1D row-major layout (a row's a resp.
// c values contiguous and 16-byte aligned): rows stream through a 2-stage ring
// of 16-byte cp.async copies (XR_TR rows per stage); warp w owns output
// tile-columns w and w + 8 and every tile-row.  diff: the right operand is
// Y2 - Y (the Parareal projection V^T (F u - u)), formed on the fly.
constexpr int XR_TR = 32;

__device__ __forceinline__ void cpa16_zfill(double *smem, const double *gmem, bool valid)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}

template <bool DIFF>
__global__ void __launch_bounds__(XM_THREADS) k_xty_rm(XtY p)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y, t = blockIdx.x;
    if (p.skip && p.skip[b] == 2) return;
    const int ctot = DIFF ? p.c : p.c + p.c2;
    const int MT = (p.a + 7) / 8, NT = (ctot + 7) / 8;
    const int SX = xm_stride(p.a), SY = xm_stride(ctot);
    const int xsz = XR_TR * SX, ysz = XR_TR * SY;
    const int nY = DIFF ? 2 : 1;
    double *Xs = sm, *Ys = sm + 2 * xsz;                 // Ys: [stage][nY][XR_TR][SY]
    const long r0 = (long)t * p.chunk_rows;
    long r1 = r0 + p.chunk_rows;
    if (r1 > p.rows) r1 = p.rows;
    const double *Xb = p.X + (long)b * p.xbs;
    const double *Yb = p.Y + (long)b * p.ybs;
    const double *Y2b = p.Y2 ? p.Y2 + (long)b * p.ybs : nullptr;
    // a Gram matrix (Y == X) stages its operand once
    const bool same = !DIFF && (p.X == p.Y) && (p.xbs == p.ybs) && (p.xrs == p.yrs) && (p.a == p.c) && p.c2 == 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int ax2 = (p.a + 1) / 2, cy2 = (ctot + 1) / 2;   // 16-byte pieces per row (a, c even)

    auto stage = [&](long rt, int buf) {
        double *xs = Xs + buf * xsz, *ys = Ys + buf * nY * ysz;
        for (int e = threadIdx.x; e < XR_TR * ax2; e += XM_THREADS) {
            const int r = e / ax2, i = 2 * (e % ax2);
            const long row = rt + r;
            const bool ok = row < r1;
            cpa16_zfill(xs + r * SX + i, ok ? Xb + row * p.xrs + i : Xb, ok);
        }
        for (int e = threadIdx.x; e < (same ? 0 : XR_TR * cy2); e += XM_THREADS) {
            const int r = e / cy2, j = 2 * (e % cy2);
            const long row = rt + r;
            const bool ok = row < r1;
            if (DIFF) {
                cpa16_zfill(ys + r * SY + j, ok ? Yb + row * p.yrs + j : Yb, ok);
                cpa16_zfill(ys + ysz + r * SY + j, ok ? Y2b + row * p.yrs + j : Y2b, ok);
            } else {
                const double *src = Yb;
                if (ok) src = (j < p.c) ? Yb + row * p.yrs + j : Y2b + row * p.yrs + (j - p.c);
                cpa16_zfill(ys + r * SY + j, src, ok);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    double acc[2][8][2];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[q][i][0] = acc[q][i][1] = 0.0;

    const int ntiles = (int)((r1 - r0 + XR_TR - 1) / XR_TR);
    if (ntiles > 0) stage(r0, 0);
    for (int it = 0; it < ntiles; ++it) {
        if (it + 1 < ntiles) {
            stage(r0 + (long)(it + 1) * XR_TR, (it + 1) & 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const double *xs = Xs + (it & 1) * xsz, *ys = same ? xs : Ys + (it & 1) * nY * ysz;
#pragma unroll
        for (int ks = 0; ks < XR_TR / 4; ++ks) {
            const int k = ks * 4 + tq;
            double af[8];
#pragma unroll
            for (int mi = 0; mi < 8; ++mi) af[mi] = (mi < MT) ? xs[k * SX + mi * 8 + gq] : 0.0;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int nj = w + 8 * q;
                if (nj < NT) {
                    double bf = ys[k * SY + nj * 8 + gq];
                    if (DIFF) bf = ys[ysz + k * SY + nj * 8 + gq] - bf;
#pragma unroll
                    for (int mi = 0; mi < 8; ++mi)
                        if (mi < MT) dmma_f64(acc[q][mi][0], acc[q][mi][1], af[mi], bf);
                }
            }
        }
        __syncthreads();
    }
    double *out = p.part + ((long)b * p.nchunk + t) * p.a * ctot;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int nj = w + 8 * q;
        if (nj >= NT) continue;
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) {
            if (mi >= MT) continue;
            const int i = mi * 8 + gq, j = nj * 8 + 2 * tq;
            if (i < p.a) {
                if (j < ctot) out[(long)i * ctot + j] = acc[q][mi][0];
                if (j + 1 < ctot) out[(long)i * ctot + j + 1] = acc[q][mi][1];
            }
        }
    }
}

// ---- skinny X^T Y (few right-hand columns, e.g. the Parareal projections with
// one source): warp lanes run over the a columns of a row of X (row-major, one
// coalesced load per row), the <= 8 values of Y's row are warp broadcasts; each
// warp accumulates its rows, the 8 warps are summed in fixed order at the end.
constexpr int XS_WARPS = 8;

template <int CT>
__global__ void __launch_bounds__(32 * XS_WARPS) k_xty_skinny(XtY p)
{
    __shared__ double red[XS_WARPS][128 * CT];
    const int b = blockIdx.y, t = blockIdx.x;
    if (p.skip && p.skip[b] == 2) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ctot = p.c + p.c2;
    const long r0 = (long)t * p.chunk_rows;
    long r1 = r0 + p.chunk_rows;
    if (r1 > p.rows) r1 = p.rows;
    const double *Xb = p.X + (long)b * p.xbs;
    const double *Yb = p.Y + (long)b * p.ybs;
    const double *Y2b = p.Y2 ? p.Y2 + (long)b * p.ybs : nullptr;
    constexpr int AJ = 4;                    // a <= 128: lane owns columns lane + 32 j
    double acc[AJ][CT];
#pragma unroll
    for (int j = 0; j < AJ; ++j)
#pragma unroll
        for (int c = 0; c < CT; ++c) acc[j][c] = 0.0;
    for (long row = r0 + w; row < r1; row += XS_WARPS) {
        double y[CT];
#pragma unroll
        for (int c = 0; c < CT; ++c) {
            y[c] = 0.0;
            if (c < ctot) {
                const double *src = (c < p.c) ? Yb + row * p.yrs + (long)c * p.ycs
                                              : Y2b + row * p.yrs + (long)(c - p.c) * p.ycs;
                y[c] = __ldg(src);
            }
        }
        const double *xr = Xb + row * p.xrs;
#pragma unroll
        for (int j = 0; j < AJ; ++j) {
            const int i = lane + 32 * j;
            const double xv = (i < p.a) ? xr[i] : 0.0;
#pragma unroll
            for (int c = 0; c < CT; ++c) acc[j][c] = fma(xv, y[c], acc[j][c]);
        }
    }
#pragma unroll
    for (int j = 0; j < AJ; ++j)
#pragma unroll
        for (int c = 0; c < CT; ++c) red[w][(lane + 32 * j) * CT + c] = acc[j][c];
    __syncthreads();
    double *out = p.part + ((long)b * p.nchunk + t) * p.a * ctot;
    for (int e = threadIdx.x; e < p.a * ctot; e += 32 * XS_WARPS) {
        const int i = e / ctot, c = e % ctot;
        double sum = 0.0;
        for (int ww = 0; ww < XS_WARPS; ++ww) sum += red[ww][i * CT + c];
        out[e] = sum;
    }
}

// row-major 1D operands that the 16-byte staging of k_xty_rm can take
static bool xty_rm_ok(const XtY &p, int ctot)
{
    auto al16 = [](const void *q) { return ((uintptr_t)q & 15) == 0; };
    if (flags().no_xty_rm) return false;
    if (p.xcs != 1 || p.ycs != 1 || p.a > 64 || ctot > 128 || p.a % 2 || ctot % 2) return false;
    if (p.diff ? (p.c % 2) : (p.c % 2 || p.c2 % 2)) return false;
    if (p.xrs % 2 || p.yrs % 2 || p.xbs % 2 || p.ybs % 2) return false;
    return al16(p.X) && al16(p.Y) && (!p.Y2 || al16(p.Y2));
}

cudaError_t launch_xty(const XtY &p, cudaStream_t s)
{
    const int ctot = p.diff ? p.c : p.c + p.c2;
    if (p.diff || ctot > 4) {
        if (xty_rm_ok(p, ctot)) {
            const int SX = xm_stride(p.a), SY = xm_stride(ctot);
            const size_t smem = (size_t)2 * XR_TR * (SX + (p.diff ? 2 : 1) * SY) * sizeof(double);
            dim3 grid(p.nchunk, p.nbatch);
            cudaError_t e;
            if (p.diff) {
                e = cudaFuncSetAttribute(k_xty_rm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
                note_launch();
                k_xty_rm<true><<<grid, XM_THREADS, smem, s>>>(p);
            } else {
                e = cudaFuncSetAttribute(k_xty_rm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
                note_launch();
                k_xty_rm<false><<<grid, XM_THREADS, smem, s>>>(p);
            }
            return cudaGetLastError();
        }
        if (p.diff) return cudaErrorInvalidValue;    // callers fall back to the [Y | Y2] form
    }
    if (ctot <= 4 && p.a <= 128 && p.xcs == 1) {
        dim3 grid(p.nchunk, p.nbatch);
        note_launch();
        if (ctot <= 2) k_xty_skinny<2><<<grid, 32 * XS_WARPS, 0, s>>>(p);
        else k_xty_skinny<4><<<grid, 32 * XS_WARPS, 0, s>>>(p);
        return cudaGetLastError();
    }
    // DMMA path for the 2D (column-contiguous) layout (the 1D row-major layout
    // takes k_xty_rm above when its strides allow 16-byte staging)
    if (p.a <= 128 && ctot <= 128 && p.xrs == 1 && p.yrs == 1 && p.xcs != 1 && p.ycs != 1) {
        const bool cm = (p.xcs != 1);
        const int MT = (p.a + 7) / 8, NT = (ctot + 7) / 8;
        const int xsz = cm ? MT * 8 * (XM_TR + 4) : XM_TR * xm_stride(p.a);
        const int ysz = cm ? NT * 8 * (XM_TR + 4) : XM_TR * xm_stride(ctot);
        const size_t smem = (size_t)2 * (xsz + ysz) * sizeof(double);
        dim3 grid(p.nchunk, p.nbatch);
        cudaError_t e;
        auto go = [&](auto kern, int threads) -> cudaError_t {
            cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e2 != cudaSuccess) return e2;
            note_launch();
            kern<<<grid, threads, smem, s>>>(p);
            return cudaSuccess;
        };
        // MT <= 8 (a <= 64): 8 warps with 2 tile-columns each and half the
        // accumulators (two CTAs per SM)
        // MT <= 16, NT <= 16 otherwise: 16 warps as 8 groups of 2 (each warp two
        // tile-columns and half the tile-rows: every warp busy for a = c = 74)
        if (cm) e = (MT <= 8) ? go(k_xty_mma<true, 8, 2, 1>, 256) : go(k_xty_mma<true, 8, 2, 2>, 512);
        else e = (MT <= 8) ? go(k_xty_mma<false, 8, 2, 1>, 256) : go(k_xty_mma<false, 8, 2, 2>, 512);
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
    }
    return launch_xty_fma(p, s);
}

cudaError_t launch_xty_diff(XtY p, const double *Y2, int c, int &pcols, cudaStream_t s)
{
    p.Y2 = Y2;
    p.c = c;
    p.c2 = 0;
    p.diff = 1;
    if (xty_rm_ok(p, c)) {
        pcols = 0;
        return launch_xty(p, s);
    }
    p.diff = 0;
    p.c2 = c;
    pcols = c;
    return launch_xty(p, s);
}

cudaError_t launch_xty_fma(const XtY &p, cudaStream_t s)
{
    const int A4 = (p.a + 3) & ~3, C4 = (p.c + p.c2 + 3) & ~3;
    const int nblk = (A4 / 4) * (C4 / 4);
    const int bpt = (nblk + XT_THREADS - 1) / XT_THREADS;
    size_t smem = (size_t)XT_TR * (A4 + C4) * sizeof(double);
    dim3 grid(p.nchunk, p.nbatch);
    cudaError_t e;
#define XT_LAUNCH(K)                                                                        \
    e = cudaFuncSetAttribute(k_xty<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                         \
    note_launch();                                                                          \
    k_xty<K><<<grid, XT_THREADS, smem, s>>>(p);
    if (bpt <= 1) { XT_LAUNCH(1) }
    else if (bpt <= 2) { XT_LAUNCH(2) }
    else if (bpt <= 4) { XT_LAUNCH(4) }
    else return cudaErrorInvalidValue;
#undef XT_LAUNCH
    return cudaGetLastError();
}

__global__ void k_reduce_parts(const double *part, int nbatch, int nchunk, int a, int c,
                               const double *rowscale, long rsbs, double *out)
{
    long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    long per = (long)a * c;
    if (idx >= per * nbatch) return;
    int b = (int)(idx / per);
    long e = idx % per;
    int i = (int)(e / c);
    const double *pp = part + (long)b * nchunk * per + e;
    double sum = 0.0;
    for (int t = 0; t < nchunk; ++t) sum += pp[(long)t * per];
    if (rowscale) sum *= rowscale[(long)b * rsbs + i];
    out[idx] = sum;
}

cudaError_t launch_reduce_parts(const double *part, int nbatch, int nchunk, int a, int c,
                                const double *rowscale, long rowscale_bs, double *out,
                                cudaStream_t s)
{
    long tot = (long)a * c * nbatch;
    if (tot == 0) return cudaSuccess;
    note_launch();
    k_reduce_parts<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(part, nbatch, nchunk, a, c,
                                                                 rowscale, rowscale_bs, out);
    return cudaGetLastError();
}

// ---------------------------------------------------------- CholeskyQR control
// One CTA per interval.  Shifted CholeskyQR (Fukaya et al. 2020):
//   G = Q^T Q, s = 11 (rows*l + l(l+1)) u ||G||_F, R^T R = G + s I, Q <- Q R^{-1};
// repeated while ||G - I||_F >= 1/2, then unshifted passes: one if it starts
// from ||G - I||_F < 1/8, else two (CholeskyQR2).
constexpr int CH_THREADS = 256;

__global__ void __launch_bounds__(CH_THREADS) k_chol(CholArgs a)
{
    extern __shared__ __align__(16) double G[];   // l x l
    __shared__ double red[CH_THREADS];
    __shared__ int sflag;
    const int b = blockIdx.x;
    const int l = a.l;
    const int st = a.state[b];
    if (st == 2) {
        if (threadIdx.x == 0) a.act[b] = 0;
        return;
    }
    if (a.passes && threadIdx.x == 0) atomicMax(a.passes, a.pass);   // last pass that did work
    const long per = (long)l * l;
    auto load_G = [&]() {
        for (int e = threadIdx.x; e < l * l; e += CH_THREADS) {
            const double *pp = a.part + (long)b * a.nchunk * per + e;
            double s = 0.0;
            for (int t = 0; t < a.nchunk; ++t) s += pp[(long)t * per];
            G[e] = s;
        }
        __syncthreads();
    };
    load_G();
    // ||G||_F and ||G - I||_F (fixed-order tree reduction)
    double f1 = 0.0, f2 = 0.0;
    for (int e = threadIdx.x; e < l * l; e += CH_THREADS) {
        double g = G[e];
        f1 += g * g;
        double d = g - ((e / l == e % l) ? 1.0 : 0.0);
        f2 += d * d;
    }
    red[threadIdx.x] = f1;
    __syncthreads();
    for (int w = CH_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    const double normG = sqrt(red[0]);
    __syncthreads();
    red[threadIdx.x] = f2;
    __syncthreads();
    for (int w = CH_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    const double offI = sqrt(red[0]);
    if (a.offI && threadIdx.x == 0) a.offI[b] = offI;
    __syncthreads();

    const bool plain = (st == 1) || (offI < 0.5);
    // Shift: 64 l u ||G||_F.  Much smaller than the worst-case bound of Fukaya
    // et al. (11 (rows l + l(l+1)) u ||G||_2), so the small singular values grow
    // by ~1/sqrt(64 l u) per pass instead of ~1/sqrt(11 rows l u) (fewer
    // passes); a breakdown is caught below and retried with a 100x larger
    // shift, and Q = Y R^{-1} by substitution keeps Y = Q R backward stable for
    // any successful R.
    double shift = plain ? 0.0 : 64.0 * l * (DBL_EPSILON * 0.5) * normG;
    if (!(normG > 0.0)) shift = 1.0;   // zero block: any SPD shift; Q stays zero
    int attempt = 0;
    for (;;) {
        if (shift > 0.0) {
            for (int i = threadIdx.x; i < l; i += CH_THREADS) G[i * l + i] += shift;
        }
        if (threadIdx.x == 0) sflag = 0;
        __syncthreads();
        // right-looking Cholesky on the upper triangle: G = R^T R
        for (int j = 0; j < l; ++j) {
            if (threadIdx.x == 0) {
                double d = G[j * l + j];
                if (!(d > 0.0) || !isfinite(d)) { sflag = 1; d = 1.0; }
                G[j * l + j] = sqrt(d);
            }
            __syncthreads();
            const double piv = G[j * l + j];
            for (int k = j + 1 + threadIdx.x; k < l; k += CH_THREADS) G[j * l + k] /= piv;
            __syncthreads();
            const int rem = l - j - 1;
            for (int e = threadIdx.x; e < rem * rem; e += CH_THREADS) {
                int i = j + 1 + e / rem, k = j + 1 + e % rem;
                if (k >= i) G[i * l + k] -= G[j * l + i] * G[j * l + k];
            }
            __syncthreads();
        }
        if (!sflag) break;
        // breakdown: reload and retry with a larger shift
        __syncthreads();
        if (++attempt > 30) {
            if (threadIdx.x == 0) atomicExch(a.fail, 1);
            break;
        }
        load_G();
        shift = (shift > 0.0 ? shift * 100.0 : DBL_EPSILON * (normG > 0 ? normG : 1.0));
    }
    if (a.shift_dbg && threadIdx.x == 0) {
        a.shift_dbg[2 * b] = (normG > 0.0) ? shift / normG : shift;
        a.shift_dbg[2 * b + 1] = attempt;
    }
    // write R (upper, zero below)
    double *Rb = a.R + (long)b * per;
    for (int e = threadIdx.x; e < l * l; e += CH_THREADS) {
        int i = e / l, k = e % l;
        Rb[e] = (k >= i) ? G[e] : 0.0;
    }
    // Rtot <- R * Rtot  (row i of the product needs rows >= i of the old Rtot)
    if (a.Rtot) {
        double *Tb = a.Rtot + (long)b * per;
        __syncthreads();
        for (int i = 0; i < l; ++i) {
            // each thread owns column k: it reads rows >= i of its own column, then
            // overwrites row i of that column -- no cross-thread hazard
            for (int k = threadIdx.x; k < l; k += CH_THREADS) {
                double s = 0.0;
                for (int j = i; j < l; ++j) s += G[i * l + j] * Tb[(long)j * l + k];
                Tb[(long)i * l + k] = s;
            }
        }
    }
    // Unshifted passes: ||G - I|| < 1/2 gives cond(R) <= sqrt(3), so applying
    // an explicit R^{-1} is as stable as substitution and runs as a GEMM on the
    // tensor cores.  Column j of R^{-1} by back substitution (one thread each).
    const bool use_inv = plain && a.Rinv;
    if (use_inv) {
        double *Xb = a.Rinv + (long)b * per;
        __syncthreads();
        for (int j = threadIdx.x; j < l; j += CH_THREADS) {
            for (int i = l - 1; i > j; --i) Xb[(long)i * l + j] = 0.0;
            for (int i = j; i >= 0; --i) {
                double t = (i == j) ? 1.0 : 0.0;
                for (int k = i + 1; k <= j; ++k) t -= G[i * l + k] * Xb[(long)k * l + j];
                Xb[(long)i * l + j] = t / G[i * l + i];
            }
        }
    }
    if (threadIdx.x == 0) {
        // An unshifted pass from ||G - I||_F = d leaves an orthogonality error of
        // O(l u (1 + d) / (1 - d)): for d < 1/8 this pass is the last one (no
        // second CholeskyQR2 pass, no verification Gram); else one more follows.
        int ns = plain ? ((st == 1 || offI < 0.125) ? 2 : 1) : 0;
        a.state[b] = ns;
        a.act[b] = use_inv ? 2 : 1;
        if (ns != 2 && a.active) atomicAdd(a.active, 1);
        if (ns != 2 && a.pass >= a.max_pass) atomicExch(a.fail, 1);   // not orthonormal within the cap
    }
}

cudaError_t launch_chol(const CholArgs &a, cudaStream_t s)
{
    size_t smem = (size_t)a.l * a.l * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    note_launch();
    k_chol<<<a.nbatch, CH_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

// Q <- Q R^{-1} row by row: q R = y by right-looking substitution in column
// blocks of TB = 32.  For block B the 32 unknowns live in registers: first the
// contributions of all earlier blocks, y_j2 -= q_j R_j,j2 (q_j read back from
// the row's shared-memory copy), then the in-block solve
//   q_j = y_j / R_jj,  y_j2 -= q_j R_j,j2  (j2 > j, fully unrolled).
// All updates of a column are independent FMAs; R rows are warp broadcasts.
// A CTA loads R once and sweeps a chunk of TS_CHUNK rows in tiles of one row
// per thread (R is l^2 doubles: reloading it per small tile dominated).
constexpr int TB = 32;
constexpr long TS_CHUNK = 2048;

__global__ void __launch_bounds__(128) k_trsm(double *Q, long bs, long rs, long cs, long rows, int l,
                                              const double *R, const int *act)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y;
    if (act[b] != 1) return;
    const int nt = blockDim.x;
    const int LP = (l + TB - 1) / TB * TB;   // padded width
    double *Rs = sm;                          // LP x LP, diag = 1/R_jj, zero padded
    double *Ys = sm + (size_t)LP * LP;        // nt x (LP + 1)
    const int ld = LP + 1;
    const double *Rb = R + (long)b * l * l;
    for (int e = threadIdx.x; e < LP * LP; e += nt) {
        const int i = e / LP, j = e % LP;
        double v = 0.0;
        if (i < l && j < l) v = (i == j) ? 1.0 / Rb[(long)i * l + j] : Rb[(long)i * l + j];
        else if (i == j) v = 1.0;
        Rs[e] = v;
    }
    double *Qb = Q + (long)b * bs;
    const long c0 = (long)blockIdx.x * TS_CHUNK;
    const long c1 = min(rows, c0 + TS_CHUNK);
    double *yr = Ys + threadIdx.x * ld;
    for (long r0 = c0; r0 < c1; r0 += nt) {
        __syncthreads();
        for (int e = threadIdx.x; e < nt * LP; e += nt) {
            int r, j;
            if (cs == 1) { r = e / LP; j = e % LP; } else { j = e / nt; r = e % nt; }
            const long row = r0 + r;
            Ys[r * ld + j] = (row < c1 && j < l) ? Qb[row * rs + (long)j * cs] : 0.0;
        }
        __syncthreads();
        for (int B = 0; B < LP; B += TB) {
            double y[TB];
#pragma unroll
            for (int t = 0; t < TB; ++t) y[t] = yr[B + t];
            for (int j = 0; j < B; ++j) {                 // earlier blocks
                const double qj = -yr[j];
                const double *Rj = Rs + (size_t)j * LP + B;
#pragma unroll
                for (int t = 0; t < TB; ++t) y[t] = fma(qj, Rj[t], y[t]);
            }
#pragma unroll
            for (int t = 0; t < TB; ++t) {                // in-block solve
                const double *Rj = Rs + (size_t)(B + t) * LP + B;
                y[t] *= Rj[t];
                const double qj = -y[t];
#pragma unroll
                for (int t2 = t + 1; t2 < TB; ++t2) y[t2] = fma(qj, Rj[t2], y[t2]);
            }
#pragma unroll
            for (int t = 0; t < TB; ++t) yr[B + t] = y[t];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nt * LP; e += nt) {
            int r, j;
            if (cs == 1) { r = e / LP; j = e % LP; } else { j = e / nt; r = e % nt; }
            const long row = r0 + r;
            if (row < c1 && j < l) Qb[row * rs + (long)j * cs] = Ys[r * ld + j];
        }
    }
}

// Blocked substitution on the FP64 tensor cores: Q <- Q R^{-1} for the shifted
// passes (act == 1), row-wise backward stable like k_trsm.  A warp owns 16 rows
// of a 64-row tile; per 16-column block B it first subtracts the solved
// columns, Y[:, B] -= X[:, <B] R[<B, B] (DMMA, warp-local), then its lanes 0..15
// solve the 16 x 16 triangular block of their row by substitution.
constexpr int TK_TB = 16;
constexpr int TK_ROWS = 64;                // rows per tile (4 warps x 16)

__global__ void __launch_bounds__(128) k_trsm_dmma(double *Q, long bs, long rs, long cs, long rows, int l,
                                                   const double *R, const int *act)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y;
    if (act[b] != 1) return;
    const int LP = (l + TK_TB - 1) / TK_TB * TK_TB;
    const int ST = LP + 4;                    // stride = 4 (mod 16): conflict-free fragments
    double *Rs = sm;                          // LP x ST: -R off the diagonal, 1/R_jj on it, identity padding
    double *Ys = sm + (size_t)LP * ST;        // TK_ROWS x ST
    const double *Rb = R + (long)b * l * l;
    for (int e = threadIdx.x; e < LP * LP; e += 128) {
        const int i = e / LP, j = e % LP;
        double v = 0.0;
        if (i < l && j < l) v = (i == j) ? 1.0 / Rb[(long)i * l + j] : -Rb[(long)i * l + j];
        else if (i == j) v = 1.0;
        Rs[i * ST + j] = v;
    }
    double *Qb = Q + (long)b * bs;
    const long c0 = (long)blockIdx.x * TS_CHUNK;
    const long c1 = min(rows, c0 + TS_CHUNK);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const bool cmaj = (cs != 1);
    for (long r0 = c0; r0 < c1; r0 += TK_ROWS) {
        __syncthreads();
        for (int e = threadIdx.x; e < TK_ROWS * LP; e += 128) {
            int r, j;
            if (cmaj) { j = e / TK_ROWS; r = e % TK_ROWS; } else { r = e / LP; j = e % LP; }
            const long row = r0 + r;
            Ys[r * ST + j] = (row < c1 && j < l) ? Qb[row * rs + (long)j * cs] : 0.0;
        }
        __syncthreads();
        double *yw = Ys + (size_t)(w * 16) * ST;       // this warp's 16 rows
        for (int B = 0; B < LP; B += TK_TB) {
            if (B > 0) {
                double acc[2][2][2];
#pragma unroll
                for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                    for (int nj = 0; nj < 2; ++nj) {
                        const double2 c = *reinterpret_cast<const double2 *>(yw + (mi * 8 + gq) * ST + B + nj * 8 + 2 * tq);
                        acc[mi][nj][0] = c.x;
                        acc[mi][nj][1] = c.y;
                    }
                for (int k0 = 0; k0 < B; k0 += 4) {
                    double af[2], bf[2];
#pragma unroll
                    for (int mi = 0; mi < 2; ++mi) af[mi] = yw[(mi * 8 + gq) * ST + k0 + tq];
#pragma unroll
                    for (int nj = 0; nj < 2; ++nj) bf[nj] = Rs[(k0 + tq) * ST + B + nj * 8 + gq];
#pragma unroll
                    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                        for (int nj = 0; nj < 2; ++nj) dmma_f64(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf[nj]);
                }
#pragma unroll
                for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                    for (int nj = 0; nj < 2; ++nj)
                        *reinterpret_cast<double2 *>(yw + (mi * 8 + gq) * ST + B + nj * 8 + 2 * tq) =
                            make_double2(acc[mi][nj][0], acc[mi][nj][1]);
            }
            __syncwarp();
            if (lane < 16) {                       // in-block substitution, one row per lane
                double *yr = yw + lane * ST + B;
                double x[TK_TB];
#pragma unroll
                for (int t = 0; t < TK_TB; ++t) {
                    double y = yr[t];
#pragma unroll
                    for (int u = 0; u < t; ++u) y = fma(x[u], Rs[(B + u) * ST + B + t], y);   // Rs = -R
                    x[t] = y * Rs[(B + t) * ST + B + t];
                }
#pragma unroll
                for (int t = 0; t < TK_TB; ++t) yr[t] = x[t];
            }
            __syncwarp();
        }
        __syncthreads();
        for (int e = threadIdx.x; e < TK_ROWS * LP; e += 128) {
            int r, j;
            if (cmaj) { j = e / TK_ROWS; r = e % TK_ROWS; } else { r = e / LP; j = e % LP; }
            const long row = r0 + r;
            if (row < c1 && j < l) Qb[row * rs + (long)j * cs] = Ys[r * ST + j];
        }
    }
}

cudaError_t launch_trsm(double *Q, long bs, long rs, long cs, long rows, int l, int nbatch,
                        const double *R, const int *act, cudaStream_t s)
{
    if (l <= 128 && !flags().no_trsm_dmma) {
        const int LPd = (l + TK_TB - 1) / TK_TB * TK_TB;
        const size_t smem = ((size_t)LPd + TK_ROWS) * (LPd + 4) * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(k_trsm_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        dim3 grid((unsigned)((rows + TS_CHUNK - 1) / TS_CHUNK), nbatch);
        note_launch();
        k_trsm_dmma<<<grid, 128, smem, s>>>(Q, bs, rs, cs, rows, l, R, act);
        return cudaGetLastError();
    }
    const int LP = (l + TB - 1) / TB * TB;
    const int nt = (LP <= 96) ? 128 : 64;
    size_t smem = ((size_t)LP * LP + (size_t)nt * (LP + 1)) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((rows + TS_CHUNK - 1) / TS_CHUNK), nbatch);
    note_launch();
    k_trsm<<<grid, nt, smem, s>>>(Q, bs, rs, cs, rows, l, R, act);
    return cudaGetLastError();
}

// ---- Q <- Q Rinv on FP64 tensor cores (unshifted CholeskyQR passes).  A CTA
// loads Rinv once and sweeps TS_CHUNK rows in tiles of 64; warp w computes rows
// 16w .. 16w+15 of the tile times Rinv (m8n8k4 DMMA), in place.
constexpr int RA_ROWS = 64;

template <bool CM>
__global__ void __launch_bounds__(128) k_rinv_apply(double *Q, long bs, long rs, long cs, long rows,
                                                    int l, const double *Rinv, const int *act)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y;
    if (act[b] != 2) return;
    const int LP = (l + 15) / 16 * 16;
    const int ST = LP + 4;                    // stride = 4 (mod 16): conflict-free fragments
    double *Rs = sm;                          // LP x ST
    double *Ys = sm + (size_t)LP * ST;        // RA_ROWS x ST
    const double *Rb = Rinv + (long)b * l * l;
    for (int e = threadIdx.x; e < LP * LP; e += 128) {
        const int i = e / LP, j = e % LP;
        Rs[i * ST + j] = (i < l && j < l) ? Rb[(long)i * l + j] : 0.0;
    }
    double *Qb = Q + (long)b * bs;
    const long c0 = (long)blockIdx.x * TS_CHUNK;
    const long c1 = min(rows, c0 + TS_CHUNK);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int NT = LP / 8;                    // <= 16 output column tiles
    for (long r0 = c0; r0 < c1; r0 += RA_ROWS) {
        __syncthreads();
        for (int e = threadIdx.x; e < RA_ROWS * LP; e += 128) {
            int r, j;
            if (CM) { j = e / RA_ROWS; r = e % RA_ROWS; } else { r = e / LP; j = e % LP; }
            const long row = r0 + r;
            Ys[r * ST + j] = (row < c1 && j < l) ? Qb[row * rs + (long)j * cs] : 0.0;
        }
        __syncthreads();
        double acc[2][16][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < 16; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
        for (int k0 = 0; k0 < LP; k0 += 4) {
            double af[2];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) af[mi] = Ys[(w * 16 + mi * 8 + gq) * ST + k0 + tq];
#pragma unroll
            for (int nj = 0; nj < 16; ++nj) {
                if (nj < NT) {
                    const double bf = Rs[(k0 + tq) * ST + nj * 8 + gq];
#pragma unroll
                    for (int mi = 0; mi < 2; ++mi) dmma_f64(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf);
                }
            }
        }
        __syncwarp();      // this warp's rows of Ys are only read by this warp
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < 16; ++nj) {
                if (nj < NT) {
                    const int r = w * 16 + mi * 8 + gq, j = nj * 8 + 2 * tq;
                    Ys[r * ST + j] = acc[mi][nj][0];
                    Ys[r * ST + j + 1] = acc[mi][nj][1];
                }
            }
        __syncthreads();
        for (int e = threadIdx.x; e < RA_ROWS * LP; e += 128) {
            int r, j;
            if (CM) { j = e / RA_ROWS; r = e % RA_ROWS; } else { r = e / LP; j = e % LP; }
            const long row = r0 + r;
            if (row < c1 && j < l) Qb[row * rs + (long)j * cs] = Ys[r * ST + j];
        }
    }
}

// 2D layout variant (a column's rows contiguous): the 64-row tiles are staged
// column-major through a 2-stage ring of 16-byte cp.async copies (the next tile
// loads while the tensor cores work on the current one), and the result goes
// back through the same shared buffer as 16-byte column stores.
constexpr int RC_S = RA_ROWS + 4;          // column stride of a staged tile

__global__ void __launch_bounds__(128) k_rinv_apply_cm(double *Q, long bs, long cs, long rows, int l,
                                                       const double *Rinv, const int *act)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y;
    if (act[b] != 2) return;
    const int LP = (l + 15) / 16 * 16;
    const int ST = LP + 4;
    double *Rs = sm;                          // LP x ST (row-major R^{-1})
    double *Ys = sm + (size_t)LP * ST;        // [2][LP][RC_S] column-major tiles
    const double *Rb = Rinv + (long)b * l * l;
    for (int e = threadIdx.x; e < LP * LP; e += 128) {
        const int i = e / LP, j = e % LP;
        Rs[i * ST + j] = (i < l && j < l) ? Rb[(long)i * l + j] : 0.0;
    }
    double *Qb = Q + (long)b * bs;
    const long c0 = (long)blockIdx.x * TS_CHUNK;
    const long c1 = min(rows, c0 + TS_CHUNK);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int NT = LP / 8;
    constexpr int HR = RA_ROWS / 2;
    auto stage = [&](long r0, int buf) {
        double *ys = Ys + (size_t)buf * LP * RC_S;
        for (int e = threadIdx.x; e < LP * HR; e += 128) {
            const int j = e / HR, r = 2 * (e % HR);
            const long row = r0 + r;
            const int nb = (j < l) ? (row + 1 < c1 ? 16 : (row < c1 ? 8 : 0)) : 0;
            const double *src = nb ? Qb + row + (long)j * cs : Qb;
            unsigned sd = (unsigned)__cvta_generic_to_shared(ys + j * RC_S + r);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sd), "l"(src), "r"(nb) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    const int ntiles = (int)((c1 - c0 + RA_ROWS - 1) / RA_ROWS);
    if (ntiles > 0) stage(c0, 0);
    for (int it = 0; it < ntiles; ++it) {
        const long r0 = c0 + (long)it * RA_ROWS;
        if (it + 1 < ntiles) {
            stage(r0 + RA_ROWS, (it + 1) & 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        double *ys = Ys + (size_t)(it & 1) * LP * RC_S;
        double acc[2][16][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < 16; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
        for (int k0 = 0; k0 < LP; k0 += 4) {
            double af[2];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) af[mi] = ys[(k0 + tq) * RC_S + w * 16 + mi * 8 + gq];
#pragma unroll
            for (int nj = 0; nj < 16; ++nj) {
                if (nj < NT) {
                    const double bf = Rs[(k0 + tq) * ST + nj * 8 + gq];
#pragma unroll
                    for (int mi = 0; mi < 2; ++mi) dmma_f64(acc[mi][nj][0], acc[mi][nj][1], af[mi], bf);
                }
            }
        }
        __syncthreads();                      // every warp has read the tile
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < 16; ++nj) {
                if (nj < NT) {
                    const int r = w * 16 + mi * 8 + gq, j = nj * 8 + 2 * tq;
                    ys[j * RC_S + r] = acc[mi][nj][0];
                    ys[(j + 1) * RC_S + r] = acc[mi][nj][1];
                }
            }
        __syncthreads();
        for (int e = threadIdx.x; e < l * HR; e += 128) {
            const int j = e / HR, r = 2 * (e % HR);
            const long row = r0 + r;
            if (row + 1 < c1) {
                *reinterpret_cast<double2 *>(Qb + row + (long)j * cs) = *reinterpret_cast<const double2 *>(ys + j * RC_S + r);
            } else if (row < c1) {
                Qb[row + (long)j * cs] = ys[j * RC_S + r];
            }
        }
        __syncthreads();                      // the buffer is refilled two tiles later
    }
}

cudaError_t launch_rinv_apply(double *Q, long bs, long rs, long cs, long rows, int l, int nbatch,
                              const double *Rinv, const int *act, cudaStream_t s)
{
    if (l > 128) return cudaErrorInvalidValue;
    const int LP = (l + 15) / 16 * 16;
    const size_t smem = ((size_t)LP + RA_ROWS) * (LP + 4) * sizeof(double);
    const bool cm = (cs != 1);
    dim3 grid((unsigned)((rows + TS_CHUNK - 1) / TS_CHUNK), nbatch);
    cudaError_t e;
    if (cm && rs == 1 && cs % 2 == 0 && bs % 2 == 0 && ((uintptr_t)Q & 15) == 0 && !flags().no_rinv_cm) {
        const size_t smem2 = ((size_t)LP * (LP + 4) + (size_t)2 * LP * RC_S) * sizeof(double);
        e = cudaFuncSetAttribute(k_rinv_apply_cm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        if (e != cudaSuccess) return e;
        note_launch();
        k_rinv_apply_cm<<<grid, 128, smem2, s>>>(Q, bs, cs, rows, l, Rinv, act);
    } else if (cm) {
        e = cudaFuncSetAttribute(k_rinv_apply<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        note_launch();
        k_rinv_apply<true><<<grid, 128, smem, s>>>(Q, bs, rs, cs, rows, l, Rinv, act);
    } else {
        e = cudaFuncSetAttribute(k_rinv_apply<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        note_launch();
        k_rinv_apply<false><<<grid, 128, smem, s>>>(Q, bs, rs, cs, rows, l, Rinv, act);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------ Jacobi SVD
// One-sided (Hestenes) Jacobi on the columns of A = M = R_Z^T, parallel
// round-robin ordering (circle method), one warp per column pair.
constexpr int JW = 8;   // warps per CTA

__global__ void __launch_bounds__(32 * JW) k_jacobi(const double *Rtot, int l, double *Psi,
                                                     double *sigma, double *Phi, int *fail)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.x;
    const int L = (l + 1) & ~1;             // even number of columns (zero pad)
    double *A = sm;                          // column-major: A[col*l + row]
    double *V = sm + (size_t)L * l;          // column-major: V[col*L + row]
    double *sig = V + (size_t)L * L;         // L
    __shared__ int rotated;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double *Tb = Rtot + (long)b * l * l;
    // A[:, j] = M[:, j] = R_Z[j, :]^T
    for (int e = threadIdx.x; e < L * l; e += 32 * JW) {
        int j = e / l, i = e % l;
        A[e] = (j < l) ? Tb[(long)j * l + i] : 0.0;
    }
    for (int e = threadIdx.x; e < L * L; e += 32 * JW) V[e] = ((e / L) == (e % L)) ? 1.0 : 0.0;
    __syncthreads();
    const double tol = (double)l * DBL_EPSILON;
    int sweep = 0;
    for (; sweep < 60; ++sweep) {
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int rnd = 0; rnd < L - 1; ++rnd) {
            for (int k = warp; k < L / 2; k += JW) {
                int p, q;
                if (k == 0) { p = rnd; q = L - 1; }
                else { p = (rnd + k) % (L - 1); q = (rnd - k + (L - 1)) % (L - 1); }
                if (p > q) { int t = p; p = q; q = t; }
                double *ap = A + (size_t)p * l, *aq = A + (size_t)q * l;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = lane; i < l; i += 32) {
                    double x = ap[i], y = aq[i];
                    al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
                    double zeta = (be - al) / (2.0 * ga);
                    double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    double c = 1.0 / sqrt(1.0 + t * t);
                    double s = c * t;
                    for (int i = lane; i < l; i += 32) {
                        double x = ap[i], y = aq[i];
                        ap[i] = c * x - s * y;
                        aq[i] = s * x + c * y;
                    }
                    double *vp = V + (size_t)p * L, *vq = V + (size_t)q * L;
                    for (int i = lane; i < L; i += 32) {
                        double x = vp[i], y = vq[i];
                        vp[i] = c * x - s * y;
                        vq[i] = s * x + c * y;
                    }
                    if (lane == 0) rotated = 1;
                }
            }
            __syncthreads();
        }
        if (!rotated) break;
        __syncthreads();
    }
    if (sweep >= 60 && threadIdx.x == 0) atomicExch(fail, 1);
    // singular values = column norms
    for (int j = warp; j < L; j += JW) {
        double s = 0.0;
        for (int i = lane; i < l; i += 32) s = fma(A[(size_t)j * l + i], A[(size_t)j * l + i], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sig[j] = sqrt(s);
    }
    __syncthreads();
    // sort descending (rank by counting; ties by index), sign convention, write
    for (int j = warp; j < l; j += JW) {
        double sj = sig[j];
        int rank = 0;
        for (int t = 0; t < L; ++t) {
            double st = sig[t];
            if (st > sj || (st == sj && t < j)) ++rank;
        }
        // largest-|.| entry of the right vector positive (reading Z10)
        const double *vj = V + (size_t)j * L;
        double best = -1.0, sgnv = 1.0;
        int bi = 0;
        for (int i = 0; i < l; ++i) {
            double av = fabs(vj[i]);
            if (av > best) { best = av; bi = i; }
        }
        sgnv = (vj[bi] < 0.0) ? -1.0 : 1.0;
        (void)bi;
        double inv = (sj > 0.0) ? 1.0 / sj : 0.0;
        for (int i = lane; i < l; i += 32) {
            Psi[((long)b * l + i) * l + rank] = sgnv * A[(size_t)j * l + i] * inv;
            Phi[((long)b * l + i) * l + rank] = sgnv * vj[i];
        }
        if (lane == 0) sigma[(long)b * l + rank] = sj;
    }
}

cudaError_t launch_jacobi(const double *Rtot, int nbatch, int l, double *Psi, double *sigma,
                          double *Phi, int *fail, cudaStream_t s)
{
    int L = (l + 1) & ~1;
    size_t smem = ((size_t)L * l + (size_t)L * L + L) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    note_launch();
    k_jacobi<<<nbatch, 32 * JW, smem, s>>>(Rtot, l, Psi, sigma, Phi, fail);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ lift
constexpr int LF_ROWS = 32;
constexpr int LF_THREADS = 256;

__global__ void __launch_bounds__(LF_THREADS) k_lift(const double *X, long xbs, long xrs, long xcs,
                                                     long rows, int l, const double *Cm, int ldc,
                                                     int k, double *out)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y;
    double *Cs = sm;                 // l x k
    double *Xs = sm + l * k;         // LF_ROWS x (l+1)
    const int ld = l + 1;
    const double *Cb = Cm + (long)b * l * ldc;
    for (int e = threadIdx.x; e < l * k; e += LF_THREADS) Cs[e] = Cb[(long)(e / k) * ldc + e % k];
    const long r0 = (long)blockIdx.x * LF_ROWS;
    const double *Xb = X + (long)b * xbs;
    for (int e = threadIdx.x; e < LF_ROWS * l; e += LF_THREADS) {
        int r, j;
        if (xcs == 1) { r = e / l; j = e % l; } else { j = e / LF_ROWS; r = e % LF_ROWS; }
        long row = r0 + r;
        Xs[r * ld + j] = (row < rows) ? Xb[row * xrs + (long)j * xcs] : 0.0;
    }
    __syncthreads();
    double *ob = out + (long)b * rows * k;
    for (int e = threadIdx.x; e < LF_ROWS * k; e += LF_THREADS) {
        int r = e / k, c = e % k;
        long row = r0 + r;
        if (row >= rows) continue;
        double s = 0.0;
        for (int j = 0; j < l; ++j) s = fma(Xs[r * ld + j], Cs[j * k + c], s);
        ob[row * k + c] = s;
    }
}

constexpr int EM_TR = 32;   // rows per stage of k_expand_mma
template <bool ACM, int KSM>
__global__ void __launch_bounds__(256, 2) k_expand_mma(Expand a);

cudaError_t launch_lift(const double *X, long xbs, long xrs, long xcs, long rows, int l,
                        const double *Cm, int ldc, int k, int nbatch, double *out, cudaStream_t s)
{
    // 1D layout (a row's l values contiguous): out_b = X_b C_b on the DMMA expand kernel
    if (xcs == 1 && l <= 64 && l % 2 == 0 && xrs % 2 == 0 && xbs % 2 == 0 && k % 8 == 0 && k <= 64 &&
        ((uintptr_t)X & 15) == 0 && ((uintptr_t)out & 15) == 0 && !flags().no_expand_mma) {
        const int nchunk = xty_chunks(rows, nbatch);
        Expand ex{out, k, 1, nullptr, 0, 0, X, xbs, Cm, l, k, nbatch, rows, nchunk, (rows + nchunk - 1) / nchunk,
                  nullptr};
        ex.Urs = xrs;
        ex.ers = ldc;
        ex.ebs = (long)l * ldc;
        ex.obs = rows * k;
        return launch_expand(ex, s);
    }
    // 2D layout (a column's rows contiguous): same product with column-major staging
    if (xrs == 1 && l <= 80 && xcs % 2 == 0 && xbs % 2 == 0 && k % 8 == 0 && k <= 64 &&
        ((uintptr_t)X & 15) == 0 && ((uintptr_t)out & 15) == 0 && !flags().no_expand_mma) {
        const int nchunk = xty_chunks(rows, nbatch);
        Expand ex{out, k, 1, nullptr, 0, 0, X, xbs, Cm, l, k, nbatch, rows, nchunk, (rows + nchunk - 1) / nchunk,
                  nullptr};
        ex.Urs = xcs;
        ex.ers = ldc;
        ex.ebs = (long)l * ldc;
        ex.obs = rows * k;
        const int KS = (l + 3) / 4;
        const size_t smem = (size_t)2 * 4 * KS * (EM_TR + 4) * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(k_expand_mma<true, 20>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        dim3 grid(nchunk, nbatch);
        note_launch();
        k_expand_mma<true, 20><<<grid, 256, smem, s>>>(ex);
        return cudaGetLastError();
    }
    size_t smem = ((size_t)l * k + (size_t)LF_ROWS * (l + 1)) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_lift, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((rows + LF_ROWS - 1) / LF_ROWS), nbatch);
    note_launch();
    k_lift<<<grid, LF_THREADS, smem, s>>>(X, xbs, xrs, xcs, rows, l, Cm, ldc, k, out);
    return cudaGetLastError();
}

cudaError_t launch_sweep_seq(const double *C, const double *d, int N, int k, int S, double *e,
                             cudaStream_t s);

// ----------------------------------------------------------------- sweep
// e_j = C_j e_{j-1} + d_j, e_{-1} = 0: the only sequential part of a Parareal
// iteration, in k-dimensional reduced coordinates.  C_{j+1} and d_{j+1} are
// prefetched with cp.async while step j is computed.
constexpr int SW_THREADS = 1024;

__device__ __forceinline__ void sw_cp8(double *dst, const double *src)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}

__global__ void __launch_bounds__(SW_THREADS) k_sweep(const double *C, const double *d, int N, int k,
                                                      int S, double *e)
{
    extern __shared__ __align__(16) double sm[];
    const int kS = k * S, kk = k * k;
    double *eb[2] = {sm, sm + kS};
    double *Cb[2] = {sm + 2 * kS, sm + 2 * kS + kk};
    double *db[2] = {sm + 2 * kS + 2 * kk, sm + 3 * kS + 2 * kk};
    for (int i = threadIdx.x; i < kS; i += SW_THREADS) eb[0][i] = 0.0;
    auto fetch = [&](int j, int buf) {
        if (j < N) {
            const double *Cj = C + (long)j * kk;
            const double *dj = d + (long)j * kS;
            for (int i = threadIdx.x; i < kk; i += SW_THREADS) sw_cp8(Cb[buf] + i, Cj + i);
            for (int i = threadIdx.x; i < kS; i += SW_THREADS) sw_cp8(db[buf] + i, dj + i);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    fetch(0, 0);
    int cur = 0;
    for (int j = 0; j < N; ++j) {
        fetch(j + 1, (j + 1) & 1);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();
        const double *Cs = Cb[j & 1];
        const double *ds = db[j & 1];
        const double *eo = eb[cur];
        double *en = eb[cur ^ 1];
        for (int o = threadIdx.x; o < kS; o += SW_THREADS) {
            const int r = o / S, s = o % S;
            double acc = ds[o];
            if (j > 0)
                for (int t = 0; t < k; ++t) acc = fma(Cs[r * k + t], eo[t * S + s], acc);
            en[o] = acc;
            e[(long)j * kS + o] = acc;
        }
        cur ^= 1;
        __syncthreads();
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// ---- blocked sweep: blocks of SWB consecutive intervals.
//  A (one CTA per block): zero-start local solution f and transfer Phi = C_last..C_first
//  B (one CTA): E_b = Phi_b E_{b-1} + f_b over the NB block ends (sequential, short)
//  C (one CTA per block): e_j = C_j e_{j-1} + d_j from e_{first-1} = E_{b-1}
// Exact algebra; only the association of the block-boundary products differs
// from the sequential recurrence.
constexpr int SWB = 16;

// y (r x S) = M (r x r) x (r x S) + add  (shared-memory operands, block-wide)
__device__ __forceinline__ void sw_gemm(const double *M, const double *x, const double *add,
                                        double *y, int r, int S)
{
    for (int o = threadIdx.x; o < r * S; o += blockDim.x) {
        const int i = o / S, c = o % S;
        double acc = add ? add[o] : 0.0;
        for (int t = 0; t < r; ++t) acc = fma(M[i * r + t], x[t * S + c], acc);
        y[o] = acc;
    }
}

__global__ void __launch_bounds__(1024) k_sweep_A(const double *C, const double *d, int N, int k, int S,
                                                  double *fend, double *Phi)
{
    extern __shared__ __align__(16) double sm[];
    const int kS = k * S, kk = k * k;
    double *f0 = sm, *f1 = sm + kS, *Cs = sm + 2 * kS, *P0 = Cs + kk, *P1 = P0 + kk;
    const int b = blockIdx.x;
    const int j0 = b * SWB, j1 = min(N, j0 + SWB);
    for (int i = threadIdx.x; i < kS; i += blockDim.x) f0[i] = 0.0;
    for (int i = threadIdx.x; i < kk; i += blockDim.x) P0[i] = (i / k == i % k) ? 1.0 : 0.0;
    __syncthreads();
    for (int j = j0; j < j1; ++j) {
        if (j == 0) {                       // e_{-1} = 0: f = d_0, Phi irrelevant (block 0)
            for (int i = threadIdx.x; i < kS; i += blockDim.x) f1[i] = d[i];
            for (int i = threadIdx.x; i < kk; i += blockDim.x) P1[i] = 0.0;
        } else {
            for (int i = threadIdx.x; i < kk; i += blockDim.x) Cs[i] = C[(long)j * kk + i];
            __syncthreads();
            sw_gemm(Cs, f0, d + (long)j * kS, f1, k, S);
            sw_gemm(Cs, P0, nullptr, P1, k, k);
        }
        __syncthreads();
        double *t = f0; f0 = f1; f1 = t;
        t = P0; P0 = P1; P1 = t;
    }
    for (int i = threadIdx.x; i < kS; i += blockDim.x) fend[(long)b * kS + i] = f0[i];
    for (int i = threadIdx.x; i < kk; i += blockDim.x) Phi[(long)b * kk + i] = P0[i];
}

__global__ void __launch_bounds__(1024) k_sweep_B(const double *fend, const double *Phi, int NB, int k,
                                                  int S, double *E)
{
    extern __shared__ __align__(16) double sm[];
    const int kS = k * S, kk = k * k;
    double *e0 = sm, *e1 = sm + kS, *Ps = sm + 2 * kS;
    for (int i = threadIdx.x; i < kS; i += blockDim.x) e0[i] = 0.0;
    __syncthreads();
    for (int b = 0; b < NB; ++b) {
        for (int i = threadIdx.x; i < kk; i += blockDim.x) Ps[i] = Phi[(long)b * kk + i];
        __syncthreads();
        sw_gemm(Ps, e0, fend + (long)b * kS, e1, k, S);
        __syncthreads();
        for (int i = threadIdx.x; i < kS; i += blockDim.x) E[(long)b * kS + i] = e1[i];
        double *t = e0; e0 = e1; e1 = t;
    }
}

__global__ void __launch_bounds__(1024) k_sweep_C(const double *C, const double *d, const double *E,
                                                  int N, int k, int S, double *e)
{
    extern __shared__ __align__(16) double sm[];
    const int kS = k * S, kk = k * k;
    double *e0 = sm, *e1 = sm + kS, *Cs = sm + 2 * kS;
    const int b = blockIdx.x;
    const int j0 = b * SWB, j1 = min(N, j0 + SWB);
    for (int i = threadIdx.x; i < kS; i += blockDim.x) e0[i] = (b > 0) ? E[(long)(b - 1) * kS + i] : 0.0;
    __syncthreads();
    for (int j = j0; j < j1; ++j) {
        if (j == 0) {
            for (int i = threadIdx.x; i < kS; i += blockDim.x) e1[i] = d[i];
        } else {
            for (int i = threadIdx.x; i < kk; i += blockDim.x) Cs[i] = C[(long)j * kk + i];
            __syncthreads();
            sw_gemm(Cs, e0, d + (long)j * kS, e1, k, S);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kS; i += blockDim.x) e[(long)j * kS + i] = e1[i];
        double *t = e0; e0 = e1; e1 = t;
    }
}

cudaError_t launch_sweep(const double *C, const double *d, int N, int k, int S, double *e,
                         cudaStream_t s)
{
    const int NB = (N + SWB - 1) / SWB;
    const size_t kS = (size_t)k * S, kk = (size_t)k * k;
    const size_t smA = (2 * kS + 3 * kk) * sizeof(double);
    if (NB >= 4 && smA <= 200 * 1024) {
        double *tmp = (double *)ws_alloc((size_t)NB * (2 * kS + kk) * sizeof(double), s);
        if (tmp) {
            double *fend = tmp, *E = tmp + NB * kS, *Phi = tmp + 2 * NB * kS;
            const size_t smB = (2 * kS + kk) * sizeof(double);
            cudaError_t er;
            er = cudaFuncSetAttribute(k_sweep_A, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA);
            if (er == cudaSuccess) er = cudaFuncSetAttribute(k_sweep_B, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB);
            if (er == cudaSuccess) er = cudaFuncSetAttribute(k_sweep_C, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB);
            if (er != cudaSuccess) { ws_free(tmp, s); return er; }
            const int th = (kS > 512 || kk > 512) ? 1024 : 256;
            note_launch();
            k_sweep_A<<<NB, th, smA, s>>>(C, d, N, k, S, fend, Phi);
            note_launch();
            k_sweep_B<<<1, th, smB, s>>>(fend, Phi, NB, k, S, E);
            note_launch();
            k_sweep_C<<<NB, th, smB, s>>>(C, d, E, N, k, S, e);
            er = cudaGetLastError();
            ws_free(tmp, s);                 // stream-ordered reuse
            return er;
        }
    }
    return launch_sweep_seq(C, d, N, k, S, e, s);
}

cudaError_t launch_sweep_seq(const double *C, const double *d, int N, int k, int S, double *e,
                             cudaStream_t s)
{
    size_t smem = ((size_t)4 * k * S + (size_t)2 * k * k) * sizeof(double);
    cudaError_t er = cudaFuncSetAttribute(k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (er != cudaSuccess) return er;
    note_launch();
    k_sweep<<<1, SW_THREADS, smem, s>>>(C, d, N, k, S, e);
    return cudaGetLastError();
}

// d[b][i][s] = sigma_b[i] * (sum_t part[b][t][i][S + s] - sum_t part[b][t][i][s])
// from the partials of [p | q] = V_b^T [Y1_b | Y2_b]  (Y1 absent: pcols = 0).
__global__ void k_reduce_pq(const double *part, int nbatch, int nchunk, int k, int S, int pcols,
                            const double *sigma, long sbs, double *d)
{
    long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long per = (long)k * S;
    if (idx >= per * nbatch) return;
    const int b = (int)(idx / per);
    const long e = idx % per;
    const int i = (int)(e / S), s = (int)(e % S);
    const int c = pcols + S;
    const double *pp = part + (long)b * nchunk * k * c + (long)i * c;
    double q = 0.0, p = 0.0;
    for (int t = 0; t < nchunk; ++t) {
        const double *row = pp + (long)t * k * c;
        q += row[pcols + s];
        if (pcols) p += row[s];
    }
    d[idx] = sigma[(long)b * sbs + i] * (q - p);
}

cudaError_t launch_reduce_pq(const double *part, int nbatch, int nchunk, int k, int S, int pcols,
                             const double *sigma, long sbs, double *d, cudaStream_t s)
{
    long tot = (long)k * S * nbatch;
    if (tot == 0) return cudaSuccess;
    note_launch();
    k_reduce_pq<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(part, nbatch, nchunk, k, S, pcols,
                                                              sigma, sbs, d);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- expand
// out[row, v] = base[row, v] + sum_r U_b[row, r] e_b[r, s], v = b*S + s.
// U tile (EX_TR rows) staged in smem; each thread owns 4 sources of one row
// per step; optional per-(b, s) partial ||new - old||^2 in fixed order.
constexpr int EX_THREADS = 256;
constexpr int EX_TR = 64;

__global__ void __launch_bounds__(EX_THREADS) k_expand(Expand a)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y, t = blockIdx.x;
    const int k = a.k, S = a.S;
    const int S4 = (S + 3) & ~3;
    const int NS4 = S4 / 4;
    const int RPP = EX_THREADS / NS4;
    const int kp = k + 1;
    double *es = sm;                         // k x S4
    double *Us = sm + (size_t)k * S4;        // EX_TR x (k+1)
    double *red = Us + (size_t)EX_TR * kp;   // RPP x NS4 x 4
    const double *eb = a.e + (long)b * k * S;
    for (int i = threadIdx.x; i < k * S4; i += EX_THREADS) {
        int r = i / S4, s = i % S4;
        es[i] = (s < S) ? eb[(long)r * S + s] : 0.0;
    }
    const int ts = threadIdx.x % NS4, tr = threadIdx.x / NS4;
    const bool act = tr < RPP;
    const long r0 = (long)t * a.chunk_rows;
    long r1 = r0 + a.chunk_rows;
    if (r1 > a.rows) r1 = a.rows;
    const double *__restrict__ Ub = a.U + (long)b * a.Ubs;
    const double *__restrict__ base = a.base;
    double *__restrict__ out = a.out;
    const bool norms = a.normpart != nullptr;
    // vectors handled by this thread: v = b*S + 4 ts + j, j < nj
    const int nj = max(0, min(4, S - 4 * ts));
    const long v0 = (long)b * S + 4 * ts;
    double nrm[4] = {0.0, 0.0, 0.0, 0.0};
    constexpr int RU = 4;                    // rows per thread in flight
    for (long rt = r0; rt < r1; rt += EX_TR) {
        const int nr = (int)min((long)EX_TR, r1 - rt);
        __syncthreads();
        const double *ut = Ub + rt * k;
        for (int i = threadIdx.x; i < nr * k; i += EX_THREADS) Us[(i / k) * kp + i % k] = ut[i];
        __syncthreads();
        if (!act) continue;
        for (int rl0 = tr; rl0 < nr; rl0 += RPP * RU) {
            // issue every global load of RU rows first (memory-level parallelism)
            double bv[RU][4], ov[RU][4];
#pragma unroll
            for (int q = 0; q < RU; ++q) {
                const int rl = rl0 + q * RPP;
                const long row = rt + rl;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const bool ok = (rl < nr) && (j < nj);
                    bv[q][j] = (ok && base) ? base[row * a.brs + (v0 + j) * a.bvs] : 0.0;
                    ov[q][j] = (ok && norms) ? out[row * a.ors + (v0 + j) * a.ovs] : 0.0;
                }
            }
#pragma unroll
            for (int q = 0; q < RU; ++q) {
                const int rl = rl0 + q * RPP;
                if (rl >= nr) break;
                const long row = rt + rl;
                double acc[4] = {bv[q][0], bv[q][1], bv[q][2], bv[q][3]};
                const double *ur = Us + rl * kp;
#pragma unroll 4
                for (int r = 0; r < k; ++r) {
                    const double u = ur[r];
                    const double2 e01 = *reinterpret_cast<const double2 *>(es + r * S4 + 4 * ts);
                    const double2 e23 = *reinterpret_cast<const double2 *>(es + r * S4 + 4 * ts + 2);
                    acc[0] = fma(u, e01.x, acc[0]);
                    acc[1] = fma(u, e01.y, acc[1]);
                    acc[2] = fma(u, e23.x, acc[2]);
                    acc[3] = fma(u, e23.y, acc[3]);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j < nj) {
                        if (norms) {
                            const double dlt = acc[j] - ov[q][j];
                            nrm[j] = fma(dlt, dlt, nrm[j]);
                        }
                        out[row * a.ors + (v0 + j) * a.ovs] = acc[j];
                    }
                }
            }
        }
    }
    if (norms) {
        __syncthreads();
        if (act)
#pragma unroll
            for (int j = 0; j < 4; ++j) red[(tr * NS4 + ts) * 4 + j] = nrm[j];
        __syncthreads();
        if (tr == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int s = 4 * ts + j;
                if (s >= S) break;
                double sum = 0.0;
                for (int y = 0; y < RPP; ++y) sum += red[(y * NS4 + ts) * 4 + j];
                a.normpart[((long)b * S + s) * a.nchunk + t] = sum;
            }
        }
    }
}

// Wide variant (S >= 16): CTA tile 64 rows x 64 sources, each thread 4 x 4
// outputs; U tile stored transposed so 4 rows are one 32-B smem read.
constexpr int EW_ROWS = 64;
constexpr int EW_SRC = 64;

__global__ void __launch_bounds__(256) k_expand_wide(Expand a)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y, t = blockIdx.x;
    const int k = a.k, S = a.S;
    const int UST = EW_ROWS + 2;              // Ut[r][row], row stride (16-B aligned)
    double *Ut = sm;                          // k x UST
    double *Es = sm + (size_t)k * UST;        // k x EW_SRC (one source tile)
    double *red = Es + (size_t)k * EW_SRC;    // 16 x 64
    const int tr = threadIdx.x / 16, ts = threadIdx.x % 16;
    const long r0 = (long)t * a.chunk_rows;
    long r1 = r0 + a.chunk_rows;
    if (r1 > a.rows) r1 = a.rows;
    const double *__restrict__ Ub = a.U + (long)b * a.Ubs;
    const double *__restrict__ base = a.base;
    double *__restrict__ out = a.out;
    const bool norms = a.normpart != nullptr;
    const double *eb = a.e + (long)b * k * S;
    for (int sb = 0; sb < S; sb += EW_SRC) {                  // source tiles
        const int ns = min(EW_SRC, S - sb);
        __syncthreads();
        for (int i = threadIdx.x; i < k * EW_SRC; i += 256) {
            const int r = i / EW_SRC, c = i % EW_SRC;
            Es[i] = (c < ns) ? eb[(long)r * S + sb + c] : 0.0;
        }
        double nrm[4] = {0.0, 0.0, 0.0, 0.0};
        const int s0 = 4 * ts;
        const int nj = max(0, min(4, ns - s0));
        const long v0 = (long)b * S + sb + s0;
        for (long rt = r0; rt < r1; rt += EW_ROWS) {
            const int nr = (int)min((long)EW_ROWS, r1 - rt);
            __syncthreads();
            const double *ut = Ub + rt * k;
            for (int i = threadIdx.x; i < nr * k; i += 256) {
                const int row = i / k, r = i % k;
                Ut[r * UST + row] = ut[i];
            }
            for (int i = threadIdx.x; i < (EW_ROWS - nr) * k; i += 256) {
                const int row = nr + i / k, r = i % k;
                Ut[r * UST + row] = 0.0;
            }
            // global loads of base / old values first (memory-level parallelism)
            double bv[4][4], ov[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int rl = 4 * tr + q;
                const long row = rt + rl;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const bool ok = (rl < nr) && (j < nj);
                    bv[q][j] = (ok && base) ? base[row * a.brs + (v0 + j) * a.bvs] : 0.0;
                    ov[q][j] = (ok && norms) ? out[row * a.ors + (v0 + j) * a.ovs] : 0.0;
                }
            }
            __syncthreads();
            double acc[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[q][j] = bv[q][j];
#pragma unroll 4
            for (int r = 0; r < k; ++r) {
                const double2 u01 = *reinterpret_cast<const double2 *>(Ut + r * UST + 4 * tr);
                const double2 u23 = *reinterpret_cast<const double2 *>(Ut + r * UST + 4 * tr + 2);
                const double2 e01 = *reinterpret_cast<const double2 *>(Es + r * EW_SRC + s0);
                const double2 e23 = *reinterpret_cast<const double2 *>(Es + r * EW_SRC + s0 + 2);
                const double uu[4] = {u01.x, u01.y, u23.x, u23.y};
                const double ee[4] = {e01.x, e01.y, e23.x, e23.y};
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[q][j] = fma(uu[q], ee[j], acc[q][j]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int rl = 4 * tr + q;
                if (rl >= nr) break;
                const long row = rt + rl;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j < nj) {
                        if (norms) {
                            const double dl = acc[q][j] - ov[q][j];
                            nrm[j] = fma(dl, dl, nrm[j]);
                        }
                        out[row * a.ors + (v0 + j) * a.ovs] = acc[q][j];
                    }
                }
            }
        }
        if (norms) {
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 4; ++j) red[tr * EW_SRC + s0 + j] = nrm[j];
            __syncthreads();
            if (tr == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j >= nj) break;
                    double sum = 0.0;
                    for (int y = 0; y < 16; ++y) sum += red[y * EW_SRC + s0 + j];
                    a.normpart[((long)b * S + sb + s0 + j) * a.nchunk + t] = sum;
                }
            }
        }
    }
}

// DMMA variant for the 1D layout (sources contiguous in a row, S % 8 == 0,
// S <= 64, k <= 64): out_b = base_b + U_b e_b as an (rows x k) x (k x S) product
// on the FP64 tensor cores.  e_b's B fragments stay in registers for the whole
// chunk (warp w: source tile w); the U rows, the base rows and (for the norm
// partials) the old rows of each 32-row stage stream through a 2-stage ring of
// 16-byte cp.async copies, so HBM requests stay in flight while the tensor
// cores work on the previous stage.  Norm partials as in k_expand_wide.
__host__ __device__ inline int em_sy(int S) { return S + 4; }   // conflict-light row stride

// ACM: U_b column-major (U_b[row, i] at U[b*Ubs + i*Urs + row], the 2D layout),
// staged column-major in shared memory
template <bool ACM, int KSM>
__global__ void __launch_bounds__(256, 2) k_expand_mma(Expand a)
{
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y, t = blockIdx.x;
    const int k = a.k, S = a.S;
    const int KS = (k + 3) / 4, NT = S / 8;
    const int SU = xm_stride(k), SY = em_sy(S), SC = EM_TR + 4;
    const bool norms = a.normpart != nullptr;
    const bool hasb = a.base != nullptr;
    const int ustage = ACM ? 4 * KS * SC : EM_TR * SU, ystage = EM_TR * SY;
    const int stage_sz = ustage + (hasb ? ystage : 0) + (norms ? ystage : 0);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const long r0 = (long)t * a.chunk_rows;
    long r1 = r0 + a.chunk_rows;
    if (r1 > a.rows) r1 = a.rows;
    const double *Ub = a.U + (long)b * a.Ubs;
    const long urs = a.Urs ? a.Urs : k, ers = a.ers ? a.ers : S;
    const double *eb = a.e + (long)b * (a.ebs ? a.ebs : (long)k * S);
    const long col0 = (long)b * (a.obs ? a.obs : S);
    // B fragments: B[kk][n] = e_b[kk, n], kk = 4 ks + tq, n = 8 w + gq (warp w: source tile w)
    const bool act = w < NT;
    double bf[KSM];
#pragma unroll
    for (int ks = 0; ks < KSM; ++ks) {
        const int kk = 4 * ks + tq;
        bf[ks] = (act && ks < KS && kk < k) ? eb[(long)kk * ers + w * 8 + gq] : 0.0;
    }
    const int k2 = k / 2, s2 = S / 2;
    auto stage = [&](long rt, int buf) {
        double *us = sm + buf * stage_sz;
        double *bs = us + ustage;
        double *os = bs + (hasb ? ystage : 0);
        if (ACM) {
            constexpr int HR = EM_TR / 2;
            for (int e = threadIdx.x; e < HR * k; e += 256) {
                const int i = e / HR, r = 2 * (e % HR);
                const long row = rt + r;
                const int nb = row + 1 < r1 ? 16 : (row < r1 ? 8 : 0);
                const double *src = nb ? Ub + (long)i * urs + row : Ub;
                unsigned sd = (unsigned)__cvta_generic_to_shared(us + i * SC + r);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sd), "l"(src), "r"(nb) : "memory");
            }
        } else {
            for (int e = threadIdx.x; e < EM_TR * k2; e += 256) {
                const int r = e / k2, i = 2 * (e % k2);
                const long row = rt + r;
                const bool ok = row < r1;
                cpa16_zfill(us + r * SU + i, ok ? Ub + row * urs + i : Ub, ok);
            }
        }
        if (hasb)
            for (int e = threadIdx.x; e < EM_TR * s2; e += 256) {
                const int r = e / s2, j = 2 * (e % s2);
                const long row = rt + r;
                const bool ok = row < r1;
                cpa16_zfill(bs + r * SY + j, ok ? a.base + row * a.brs + col0 + j : a.base, ok);
            }
        if (norms)
            for (int e = threadIdx.x; e < EM_TR * s2; e += 256) {
                const int r = e / s2, j = 2 * (e % s2);
                const long row = rt + r;
                const bool ok = row < r1;
                cpa16_zfill(os + r * SY + j, ok ? a.out + row * a.ors + col0 + j : a.out, ok);
            }
        for (int e = threadIdx.x; e < EM_TR * (4 * KS - k); e += 256) {   // k-step padding
            const int r = e / (4 * KS - k), i = k + e % (4 * KS - k);
            us[ACM ? i * SC + r : r * SU + i] = 0.0;
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    double nrm[2] = {0.0, 0.0};
    const int ntiles = (int)((r1 - r0 + EM_TR - 1) / EM_TR);
    if (ntiles > 0) stage(r0, 0);
    for (int it = 0; it < ntiles; ++it) {
        if (it + 1 < ntiles) {
            stage(r0 + (long)(it + 1) * EM_TR, (it + 1) & 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const double *us = sm + (it & 1) * stage_sz;
        const double *bs = us + ustage;
        const double *os = bs + (hasb ? ystage : 0);
        const long rt = r0 + (long)it * EM_TR;
        // the stage's 4 m-tiles run as independent accumulator chains over k
        constexpr int MTS = EM_TR / 8;
        if (act) {
            double acc[MTS][2];
#pragma unroll
            for (int mi = 0; mi < MTS; ++mi) {
                double2 bv = make_double2(0.0, 0.0);
                if (hasb) bv = *reinterpret_cast<const double2 *>(bs + (mi * 8 + gq) * SY + w * 8 + 2 * tq);
                acc[mi][0] = bv.x;
                acc[mi][1] = bv.y;
            }
#pragma unroll
            for (int ks = 0; ks < KSM; ++ks) {
                if (ks < KS) {
#pragma unroll
                    for (int mi = 0; mi < MTS; ++mi)
                        dmma_f64(acc[mi][0], acc[mi][1],
                                 ACM ? us[(4 * ks + tq) * SC + mi * 8 + gq] : us[(mi * 8 + gq) * SU + 4 * ks + tq],
                                 bf[ks]);
                }
            }
#pragma unroll
            for (int mi = 0; mi < MTS; ++mi) {
                const int rl = mi * 8 + gq;
                const long row = rt + rl;
                if (row < r1) {
                    const long col = col0 + w * 8 + 2 * tq;
                    *reinterpret_cast<double2 *>(a.out + row * a.ors + col) = make_double2(acc[mi][0], acc[mi][1]);
                    if (norms) {
                        const double2 ov = *reinterpret_cast<const double2 *>(os + rl * SY + w * 8 + 2 * tq);
                        const double d0 = acc[mi][0] - ov.x, d1 = acc[mi][1] - ov.y;
                        nrm[0] = fma(d0, d0, nrm[0]);
                        nrm[1] = fma(d1, d1, nrm[1]);
                    }
                }
            }
        }
        __syncthreads();
    }
    if (norms && act) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            double v = nrm[c];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (gq == 0) a.normpart[((long)b * S + w * 8 + 2 * tq + c) * a.nchunk + t] = v;
        }
    }
}

// Narrow variant (S < 16): one row per thread, the row of U_b read straight
// from global memory (contiguous k doubles, 16-B loads), e_b broadcast from
// shared memory, four independent partial sums per output.
__global__ void __launch_bounds__(256) k_expand_narrow(Expand a)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[256];
    const int b = blockIdx.y, t = blockIdx.x;
    const int k = a.k, S = a.S;
    double *es = sm;   // k x S
    const double *eb = a.e + (long)b * k * S;
    for (int i = threadIdx.x; i < k * S; i += 256) es[i] = eb[i];
    __syncthreads();
    const long r0 = (long)t * a.chunk_rows;
    long r1 = r0 + a.chunk_rows;
    if (r1 > a.rows) r1 = a.rows;
    const double *__restrict__ Ub = a.U + (long)b * a.Ubs;
    const bool norms = a.normpart != nullptr;
    const bool vec = (k % 2 == 0);
    for (int s = 0; s < S; ++s) {
        const long v = (long)b * S + s;
        double nrm = 0.0;
        for (long row = r0 + threadIdx.x; row < r1; row += 256) {
            const double *ur = Ub + row * k;
            double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
            int r = 0;
            if (vec) {
                for (; r + 3 < k; r += 4) {
                    const double2 u01 = *reinterpret_cast<const double2 *>(ur + r);
                    const double2 u23 = *reinterpret_cast<const double2 *>(ur + r + 2);
                    c0 = fma(u01.x, es[r * S + s], c0);
                    c1 = fma(u01.y, es[(r + 1) * S + s], c1);
                    c2 = fma(u23.x, es[(r + 2) * S + s], c2);
                    c3 = fma(u23.y, es[(r + 3) * S + s], c3);
                }
            }
            for (; r < k; ++r) c0 = fma(ur[r], es[r * S + s], c0);
            double val = (c0 + c1) + (c2 + c3);
            if (a.base) val += a.base[row * a.brs + v * a.bvs];
            double *o = a.out + row * a.ors + v * a.ovs;
            if (norms) {
                const double dl = val - *o;
                nrm = fma(dl, dl, nrm);
            }
            *o = val;
        }
        if (norms) {
            red[threadIdx.x] = nrm;
            __syncthreads();
            for (int w = 128; w > 0; w >>= 1) {
                if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
                __syncthreads();
            }
            if (threadIdx.x == 0) a.normpart[v * a.nchunk + t] = red[0];
            __syncthreads();
        }
    }
}

cudaError_t launch_expand(const Expand &a, cudaStream_t s)
{
    const bool general = a.Urs || a.ers || a.ebs || a.obs;     // only k_expand_mma takes these
    if (!general && a.S < 16 && ((uintptr_t)a.U & 15) == 0 && a.k % 2 == 0) {
        size_t smem = (size_t)a.k * a.S * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(k_expand_narrow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        dim3 grid(a.nchunk, a.nbatch);
        note_launch();
        k_expand_narrow<<<grid, 256, smem, s>>>(a);
        return cudaGetLastError();
    }
    {
        auto al16 = [](const void *q) { return ((uintptr_t)q & 15) == 0; };
        if (!flags().no_expand_mma && a.ovs == 1 && (a.base == nullptr || a.bvs == 1) && a.S % 8 == 0 &&
            a.S <= 64 && a.k <= 64 && a.k % 2 == 0 && a.ors % 2 == 0 && (a.base == nullptr || a.brs % 2 == 0) &&
            a.Ubs % 2 == 0 && a.Urs % 2 == 0 && a.obs % 2 == 0 && al16(a.out) && al16(a.U) &&
            (a.base == nullptr || al16(a.base))) {
            const size_t smem = (size_t)2 * EM_TR *
                                (xm_stride(a.k) + (a.base ? em_sy(a.S) : 0) + (a.normpart ? em_sy(a.S) : 0)) *
                                sizeof(double);
            cudaError_t e = cudaFuncSetAttribute(k_expand_mma<false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
            dim3 grid(a.nchunk, a.nbatch);
            note_launch();
            k_expand_mma<false, 16><<<grid, 256, smem, s>>>(a);
            return cudaGetLastError();
        }
    }
    if (general) return cudaErrorInvalidValue;
    if (a.S >= 16 && a.k <= 128) {
        size_t smem = ((size_t)a.k * (EW_ROWS + 2) + (size_t)a.k * EW_SRC + 16 * EW_SRC) * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(k_expand_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        dim3 grid(a.nchunk, a.nbatch);
        note_launch();
        k_expand_wide<<<grid, 256, smem, s>>>(a);
        return cudaGetLastError();
    }
    if (a.S > 128 || a.k > 128) return cudaErrorInvalidValue;
    const int S4 = (a.S + 3) & ~3;
    const int NS4 = S4 / 4;
    const int RPP = EX_THREADS / NS4;
    size_t smem = ((size_t)a.k * S4 + (size_t)EX_TR * (a.k + 1) + (size_t)RPP * NS4 * 4) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_expand, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(a.nchunk, a.nbatch);
    note_launch();
    k_expand<<<grid, EX_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

__global__ void k_norm_finish(const double *part, int nvec, int nchunk, double *out)
{
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nvec) return;
    double s = 0.0;
    for (int t = 0; t < nchunk; ++t) s += part[(long)v * nchunk + t];
    out[v] = sqrt(s);
}

cudaError_t launch_norm_finish(const double *part, int nvec, int nchunk, double *out, cudaStream_t s)
{
    if (nvec == 0) return cudaSuccess;
    note_launch();
    k_norm_finish<<<(nvec + 127) / 128, 128, 0, s>>>(part, nvec, nchunk, out);
    return cudaGetLastError();
}

__global__ void k_vecnorm_parts(const double *X, long rs, long vs, long rows, int nvec, int nchunk,
                                long chunk_rows, double *part)
{
    __shared__ double red[256];
    const int v = blockIdx.y, t = blockIdx.x;
    const long r0 = (long)t * chunk_rows;
    long r1 = r0 + chunk_rows;
    if (r1 > rows) r1 = rows;
    double s = 0.0;
    for (long r = r0 + threadIdx.x; r < r1; r += 256) {
        double x = X[r * rs + (long)v * vs];
        s = fma(x, x, s);
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[(long)v * nchunk + t] = red[0];
}

cudaError_t launch_vecnorm_parts(const double *X, long rs, long vs, long rows, int nvec, int nchunk,
                                 long chunk_rows, double *part, cudaStream_t s)
{
    if (nvec == 0) return cudaSuccess;
    dim3 grid(nchunk, nvec);
    note_launch();
    k_vecnorm_parts<<<grid, 256, 0, s>>>(X, rs, vs, rows, nvec, nchunk, chunk_rows, part);
    return cudaGetLastError();
}

__global__ void k_copy_vectors(const double *in, long irs, long ivs, double *out, long ors, long ovs,
                               long rows, int nvec)
{
    long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    long tot = rows * nvec;
    if (idx >= tot) return;
    long r, v;
    if (ivs == 1 || ovs == 1) { r = idx / nvec; v = idx % nvec; }   // vector index fastest
    else { v = idx / rows; r = idx % rows; }
    out[r * ors + v * ovs] = in[r * irs + v * ivs];
}

cudaError_t launch_copy_vectors(const double *in, long irs, long ivs, double *out, long ors, long ovs,
                                long rows, int nvec, cudaStream_t s)
{
    long tot = rows * nvec;
    if (tot == 0) return cudaSuccess;
    note_launch();
    k_copy_vectors<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(in, irs, ivs, out, ors, ovs, rows, nvec);
    return cudaGetLastError();
}

__global__ void k_eye(double *R, int nbatch, int l)
{
    long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    long per = (long)l * l;
    if (idx >= per * nbatch) return;
    long e = idx % per;
    R[idx] = (e / l == e % l) ? 1.0 : 0.0;
}

cudaError_t launch_eye(double *R, int nbatch, int l, cudaStream_t s)
{
    long tot = (long)l * l * nbatch;
    if (tot == 0) return cudaSuccess;
    note_launch();
    k_eye<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(R, nbatch, l);
    return cudaGetLastError();
}

}  // namespace pr

namespace pr {

// ----------------------------------------------- small pivoted LU solve
// One CTA per batch: A X = R^T (l x l, row-major in global memory), written as
// X^T.  A in shared memory is eliminated column by column with partial
// pivoting (row swaps applied to the right-hand side too), then the l
// right-hand sides are back-substituted one per thread.
constexpr int LU_THREADS = 256;

__global__ void __launch_bounds__(LU_THREADS) k_lu_solve_rt(const double *Ag, const double *Rg, int l, double *XT,
                                                            int *fail)
{
    extern __shared__ __align__(16) double sm[];
    double *A = sm;                  // l x l
    double *Bm = sm + (size_t)l * l; // l x l right-hand sides, Bm[i*l + c]
    __shared__ int piv;
    __shared__ double pv[LU_THREADS];
    __shared__ int pi[LU_THREADS];
    const int b = blockIdx.x;
    const long per = (long)l * l;
    for (int e = threadIdx.x; e < l * l; e += LU_THREADS) {
        A[e] = Ag[b * per + e];
        const int i = e / l, c = e % l;
        Bm[e] = Rg[b * per + (long)c * l + i];        // R^T
    }
    __syncthreads();
    for (int j = 0; j < l; ++j) {
        // pivot: max |A[i][j]|, i >= j (fixed-order tree reduction)
        double best = -1.0;
        int bi = j;
        for (int i = j + threadIdx.x; i < l; i += LU_THREADS) {
            const double v = fabs(A[i * l + j]);
            if (v > best) { best = v; bi = i; }
        }
        pv[threadIdx.x] = best;
        pi[threadIdx.x] = bi;
        __syncthreads();
        for (int w = LU_THREADS / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) {
                const double o = pv[threadIdx.x + w];
                const int oi = pi[threadIdx.x + w];
                if (o > pv[threadIdx.x] || (o == pv[threadIdx.x] && oi < pi[threadIdx.x])) {
                    pv[threadIdx.x] = o;
                    pi[threadIdx.x] = oi;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            piv = pi[0];
            if (!(pv[0] > 0.0) || !isfinite(pv[0])) atomicExch(fail, 1);
        }
        __syncthreads();
        const int r = piv;
        if (r != j) {
            for (int c = threadIdx.x; c < l; c += LU_THREADS) {
                double t = A[j * l + c]; A[j * l + c] = A[r * l + c]; A[r * l + c] = t;
                t = Bm[j * l + c]; Bm[j * l + c] = Bm[r * l + c]; Bm[r * l + c] = t;
            }
        }
        __syncthreads();
        const double d = A[j * l + j];
        const double inv = (d != 0.0) ? 1.0 / d : 0.0;
        // eliminate rows below j (multipliers stored in A's column j)
        for (int i = j + 1 + threadIdx.x; i < l; i += LU_THREADS) A[i * l + j] *= inv;
        __syncthreads();
        const int rem = l - j - 1;
        for (int e = threadIdx.x; e < rem * l; e += LU_THREADS) {
            const int i = j + 1 + e / l, c = e % l;
            const double mlt = A[i * l + j];
            if (c > j) A[i * l + c] -= mlt * A[j * l + c];
            Bm[i * l + c] -= mlt * Bm[j * l + c];
        }
        __syncthreads();
    }
    // back substitution, one right-hand side per thread: U x = y
    for (int c = threadIdx.x; c < l; c += LU_THREADS) {
        for (int i = l - 1; i >= 0; --i) {
            double t = Bm[i * l + c];
            for (int k2 = i + 1; k2 < l; ++k2) t -= A[i * l + k2] * Bm[k2 * l + c];
            Bm[i * l + c] = t / A[i * l + i];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < l * l; e += LU_THREADS) {
        const int i = e / l, c = e % l;
        XT[b * per + (long)c * l + i] = Bm[e];        // X^T
    }
}

cudaError_t launch_lu_solve_rt(const double *A, const double *R, int nbatch, int l, double *XT, int *fail,
                               cudaStream_t s)
{
    const size_t smem = (size_t)2 * l * l * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_lu_solve_rt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    note_launch();
    k_lu_solve_rt<<<nbatch, LU_THREADS, smem, s>>>(A, R, l, XT, fail);
    return cudaGetLastError();
}

}  // namespace pr
