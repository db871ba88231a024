// Microbenchmark: tensor memory (TMEM) as a per-thread coefficient store.
//  (1) throughput of tcgen05.ld.32x32b.xN (N 32-bit columns per lane) with 8
//      warps per SM (two per TMEM lane quadrant), alone and with a concurrent
//      stream of shared-memory loads;
//  (2) the K1P chunk sweep (ub_sweep.cu, VPT 1, L 64, H 2, W 8) with the two LU
//      coefficients per row {nl, w} read from TMEM instead of shared memory
//      (the spike coefficients {V2~, W2~} stay in shared memory).
// One CTA per SM on every SM; prints SM cycles.
#include <cstdio>

__device__ __forceinline__ unsigned tmem_alloc_all(unsigned *slot)
{
    // one warp allocates all 512 columns; the base address goes through shared memory
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     :: "r"((unsigned)__cvta_generic_to_shared(slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    return *slot;
}

__device__ __forceinline__ void tmem_free_all(unsigned base)
{
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base) : "memory");
}

__device__ __forceinline__ void tm_ld8(unsigned addr, unsigned (&r)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr) : "memory");
}
__device__ __forceinline__ void tm_wait8(unsigned (&r)[8])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
                 :: "memory");
}
__device__ __forceinline__ void tm_ld16(unsigned addr, unsigned (&r)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(addr) : "memory");
}
__device__ __forceinline__ void tm_wait16(unsigned (&r)[16])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
                 :: "memory");
}
__device__ __forceinline__ void tm_st8(unsigned addr, const unsigned (&r)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// (1) raw throughput: each warp issues `iters` x (UN loads then one wait); LDS > 0 adds that
// many independent 8-byte shared loads per tcgen05.ld
template <int X, int LDS>
__global__ void __launch_bounds__(256, 1) k_tp(double *out, long long *t, int iters)
{
    __shared__ unsigned slot;
    __shared__ __align__(16) double sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1.0 + i;
    const unsigned base = tmem_alloc_all(&slot);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned my = base + ((unsigned)(32 * (w & 3)) << 16) + (unsigned)((w >> 2) * 256);
    unsigned z[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    for (int c = 0; c < 256; c += 8) tm_st8(my + c, z);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    __syncthreads();
    unsigned acc = 0;
    unsigned long long accl = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned col = (unsigned)(((it * 4 + u) * X) & 255);
            if (X == 8) {
                unsigned r[8];
                tm_ld8(my + col, r);
                tm_wait8(r);
                acc ^= r[0] ^ r[7];
            } else {
                unsigned r[16];
                tm_ld16(my + col, r);
                tm_wait16(r);
                acc ^= r[0] ^ r[15];
            }
#pragma unroll
            for (int l = 0; l < LDS; ++l) {
                unsigned long long x;
                const unsigned a = (unsigned)__cvta_generic_to_shared(sm + (((it * 4 + u) * LDS + l) * 2 + (lane >> 4)) % 2048);
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x) : "r"(a));
                accl ^= x;
            }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = (double)acc + (double)accl;
    tmem_free_all(base);
}

// (2) the sweep; TM = 1: {nl, w} from TMEM in blocks of 4 rows (x8), double buffered
template <int TM>
__global__ void __launch_bounds__(320, 1) k_sweep(const double *g, double *out, long long *t, int m)
{
    constexpr int L = 64, H = 2, W = 8, K = W * H, RSTR = 4 * L + 4;
    extern __shared__ __align__(16) double sm[];
    __shared__ unsigned slot;
    for (int i = threadIdx.x; i < K * RSTR; i += blockDim.x) sm[i] = g[i % 4096];
    const unsigned base = tmem_alloc_all(&slot);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w >= W) {
        tmem_free_all(base);
        return;
    }
    const int u = w * H + lane / (32 / H);
    const double2 *cd = reinterpret_cast<const double2 *>(sm + u * RSTR);
    const double *nl = sm + u * RSTR + 2 * L;
    const double *wv = nl + L;
    const unsigned my = base + ((unsigned)(32 * (w & 3)) << 16) + (unsigned)((w >> 2) * 256);
    if (TM) {   // columns 0..127: nl rows 0..63; 128..255: w rows 0..63
        for (int b = 0; b < 32; ++b) {
            unsigned r[8];
            for (int e = 0; e < 4; ++e) {
                const double v = (b < 16) ? nl[b * 4 + e] : wv[(b - 16) * 4 + e];
                r[2 * e] = (unsigned)__double2loint(v);
                r[2 * e + 1] = (unsigned)__double2hiint(v);
            }
            tm_st8(my + b * 8, r);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    double S[L];
#pragma unroll
    for (int i = 0; i < L; ++i) S[i] = g[(i * 7 + lane) & 4095];
    double ca = g[0], cc = g[1];
    long long t0 = clock64();
    for (int j = 0; j < m; ++j) {
        asm volatile("" ::: "memory");
        double zp = 0.0;
        if (TM) {
            unsigned buf[2][8];
            tm_ld8(my, buf[0]);
#pragma unroll
            for (int b = 0; b < 16; ++b) {
                tm_wait8(buf[b & 1]);
                tm_ld8(my + (b + 1) * 8, buf[(b + 1) & 1]);     // b = 15: first block of w (rows 0..3), unused order fixed below
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = b * 4 + e;
                    const double2 q2 = cd[i];
                    const double nli = __hiloint2double((int)buf[b & 1][2 * e + 1], (int)buf[b & 1][2 * e]);
                    double x = fma(q2.x, ca, fma(q2.y, cc, S[i]));
                    zp = (i == 0) ? x : fma(nli, zp, x);
                    S[i] = zp;
                }
            }
            tm_wait8(buf[0]);                                   // drain (block 16 in buf[0])
            double gn = 0.0;
            tm_ld8(my + 128 + 15 * 8, buf[0]);
#pragma unroll
            for (int b = 15; b >= 0; --b) {
                const int s = (15 - b) & 1;
                tm_wait8(buf[s]);
                if (b > 0) tm_ld8(my + 128 + (b - 1) * 8, buf[s ^ 1]);
#pragma unroll
                for (int e = 3; e >= 0; --e) {
                    const int i = b * 4 + e;
                    const double wi = __hiloint2double((int)buf[s][2 * e + 1], (int)buf[s][2 * e]);
                    gn = (i == L - 1) ? wi * S[i] : fma(wi, S[i], gn);
                    S[i] = gn;
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < L; ++i) {
                const double2 q2 = cd[i];
                const double nli = nl[i];
                double x = fma(q2.x, ca, fma(q2.y, cc, S[i]));
                zp = (i == 0) ? x : fma(nli, zp, x);
                S[i] = zp;
            }
            double gn = 0.0;
#pragma unroll
            for (int i = L - 1; i >= 0; --i) {
                const double wi = wv[i];
                gn = (i == L - 1) ? wi * S[i] : fma(wi, S[i], gn);
                S[i] = gn;
            }
        }
        ca = S[0] * 1e-3;
        cc = S[L - 1] * 1e-3;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) s += S[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    tmem_free_all(base);
}

// (3) as (2) but 12 warps: the 8 compute warps raise their register budget to 232 with
// setmaxnreg (warps 8..11 drop to 40), {nl, w} from TMEM and the spike coefficients prefetched
// one block (4 rows) ahead; SPLIT: the up sweep (a running sum of w_i z_i) as two interleaved
// half chains plus a carry fix-up
__device__ __forceinline__ void tm_ld8n(unsigned addr, unsigned (&r)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
}
__device__ __forceinline__ void tm_wait8n(unsigned (&r)[8])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]));
}

template <int SPLIT, int REGS>
__global__ void __launch_bounds__(384, 1) k_sweep2(const double *g, double *out, long long *t, int m)
{
    constexpr int L = 64, H = 2, W = 8, K = W * H, RSTR = 4 * L + 4;
    extern __shared__ __align__(16) double sm[];
    __shared__ unsigned slot;
    for (int i = threadIdx.x; i < K * RSTR; i += blockDim.x) sm[i] = g[i % 4096];
    const unsigned base = tmem_alloc_all(&slot);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w >= W) {
        if (REGS) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
        tmem_free_all(base);
        return;
    }
    if (REGS) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    const int u = w * H + lane / (32 / H);
    const double2 *cd = reinterpret_cast<const double2 *>(sm + u * RSTR);
    const double *nl = sm + u * RSTR + 2 * L;
    const double *wv = nl + L;
    const unsigned my = base + ((unsigned)(32 * (w & 3)) << 16) + (unsigned)((w >> 2) * 256);
    for (int b = 0; b < 32; ++b) {
        unsigned r[8];
        for (int e = 0; e < 4; ++e) {
            const double v = (b < 16) ? nl[b * 4 + e] : wv[(b - 16) * 4 + e];
            r[2 * e] = (unsigned)__double2loint(v);
            r[2 * e + 1] = (unsigned)__double2hiint(v);
        }
        tm_st8(my + b * 8, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    double S[L];
#pragma unroll
    for (int i = 0; i < L; ++i) S[i] = g[(i * 7 + lane) & 4095];
    double ca = g[0], cc = g[1];
    long long t0 = clock64();
    for (int j = 0; j < m; ++j) {
        asm volatile("" ::: "memory");
        double zp = 0.0;
        unsigned buf[2][8];
        double2 qn[2][4];
        tm_ld8n(my, buf[0]);
#pragma unroll
        for (int e = 0; e < 4; ++e) qn[0][e] = cd[e];
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            tm_wait8n(buf[b & 1]);
            tm_ld8n(b < 15 ? my + (b + 1) * 8 : my + 128 + 15 * 8, buf[(b + 1) & 1]);
            if (b < 15) {
#pragma unroll
                for (int e = 0; e < 4; ++e) qn[(b + 1) & 1][e] = cd[(b + 1) * 4 + e];
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = b * 4 + e;
                const double2 q2 = qn[b & 1][e];
                const double nli = __hiloint2double((int)buf[b & 1][2 * e + 1], (int)buf[b & 1][2 * e]);
                double x = fma(q2.x, ca, fma(q2.y, cc, S[i]));
                zp = (i == 0) ? x : fma(nli, zp, x);
                S[i] = zp;
            }
        }
        if (SPLIT) {
            // rows 63..32 (chain A) and 31..0 (chain B, from zero), then B += carry
            double ga = 0.0, gb = 0.0;
            unsigned bufb[8];
#pragma unroll
            for (int b = 15; b >= 8; --b) {
                const int s = (15 - b) & 1;
                tm_wait8n(buf[s]);                       // block b (rows 4b..4b+3), chain A
                tm_ld8n(my + 128 + (b - 8) * 8, bufb);   // block b-8, chain B
                tm_wait8n(bufb);
                if (b > 8) tm_ld8n(my + 128 + (b - 1) * 8, buf[s ^ 1]);
#pragma unroll
                for (int e = 3; e >= 0; --e) {
                    const int ia = b * 4 + e, ib = (b - 8) * 4 + e;
                    const double wa = __hiloint2double((int)buf[s][2 * e + 1], (int)buf[s][2 * e]);
                    const double wb = __hiloint2double((int)bufb[2 * e + 1], (int)bufb[2 * e]);
                    ga = (ia == L - 1) ? wa * S[ia] : fma(wa, S[ia], ga);
                    gb = (ib == L / 2 - 1) ? wb * S[ib] : fma(wb, S[ib], gb);
                    S[ia] = ga;
                    S[ib] = gb;
                }
            }
#pragma unroll
            for (int i = 0; i < L / 2; ++i) S[i] += ga;
        } else {
            double gn = 0.0;
#pragma unroll
            for (int b = 15; b >= 0; --b) {
                const int s = (15 - b) & 1;
                tm_wait8n(buf[s]);
                if (b > 0) tm_ld8n(my + 128 + (b - 1) * 8, buf[s ^ 1]);
#pragma unroll
                for (int e = 3; e >= 0; --e) {
                    const int i = b * 4 + e;
                    const double wi = __hiloint2double((int)buf[s][2 * e + 1], (int)buf[s][2 * e]);
                    gn = (i == L - 1) ? wi * S[i] : fma(wi, S[i], gn);
                    S[i] = gn;
                }
            }
        }
        ca = S[0] * 1e-3;
        cc = S[L - 1] * 1e-3;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) s += S[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    tmem_free_all(base);
}

// (4) the DFMA structure alone: coefficients are four loop-invariant registers (no LDS, no TMEM)
template <int W, int SPLIT>
__global__ void __launch_bounds__(384, 1) k_sweep3(const double *g, double *out, long long *t, int m)
{
    constexpr int L = 64;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w >= W) return;
    double S[L];
#pragma unroll
    for (int i = 0; i < L; ++i) S[i] = g[(i * 7 + lane) & 4095];
    double ca = g[0], cc = g[1];
    const double q2x = g[5], q2y = g[6], nli = g[7], wi = g[8];
    long long t0 = clock64();
    for (int j = 0; j < m; ++j) {
        asm volatile("" ::: "memory");
        double zp = 0.0;
#pragma unroll
        for (int i = 0; i < L; ++i) {
            double x = fma(q2x, ca, fma(q2y, cc, S[i]));
            zp = (i == 0) ? x : fma(nli, zp, x);
            S[i] = zp;
        }
        if (SPLIT) {
            double ga = 0.0, gb = 0.0;
#pragma unroll
            for (int i = L / 2 - 1; i >= 0; --i) {
                ga = fma(wi, S[i + L / 2], ga);
                gb = fma(wi, S[i], gb);
                S[i + L / 2] = ga;
                S[i] = gb;
            }
#pragma unroll
            for (int i = 0; i < L / 2; ++i) S[i] += ga;
        } else {
            double gn = 0.0;
#pragma unroll
            for (int i = L - 1; i >= 0; --i) {
                gn = fma(wi, S[i], gn);
                S[i] = gn;
            }
        }
        ca = S[0] * 1e-3;
        cc = S[L - 1] * 1e-3;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) s += S[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int W, int SPLIT>
void run_sweep3(const double *g, double *o, long long *t, long long *h)
{
    const int m = 256, nsm = 148;
    for (int r = 0; r < 2; ++r) k_sweep3<W, SPLIT><<<nsm, 384>>>(g, o, t, m);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, t, 8 * nsm, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("sweep3 (DFMA structure only, coefficients in registers) %d compute warps split-up %d: %.0f cycles/step %s\n", W,
           SPLIT, mx / m, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int SPLIT, int REGS>
void run_sweep2(const double *g, double *o, long long *t, long long *h)
{
    const int m = 256, nsm = 148;
    const size_t smem = (size_t)16 * (4 * 64 + 4) * 8;
    cudaFuncSetAttribute(k_sweep2<SPLIT, REGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int r = 0; r < 2; ++r) k_sweep2<SPLIT, REGS><<<nsm, 384, smem>>>(g, o, t, m);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, t, 8 * nsm, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("sweep2 (12 warps, TMEM {nl, w}, spikes prefetched) setmaxnreg %d split-up %d: %.0f cycles/step %s\n", REGS, SPLIT,
           mx / m, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

static double maxof(long long *t, long long *h, int nsm)
{
    cudaMemcpy(h, t, 8 * nsm, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    return mx;
}

template <int X, int LDS>
void run_tp(double *o, long long *t, long long *h)
{
    const int iters = 2048, nsm = 148;
    for (int r = 0; r < 2; ++r) k_tp<X, LDS><<<nsm, 256>>>(o, t, iters);
    cudaError_t e = cudaDeviceSynchronize();
    const double cyc = maxof(t, h, nsm) / (iters * 4.0);
    printf("tcgen05.ld.32x32b.x%-2d + %d LDS.64 (8 warps/SM, ld+wait back to back): %.1f cycles per warp iteration, "
           "%.1f B/cycle/SM of TMEM reads %s\n", X, LDS, cyc, 8.0 * 32 * X * 4 / cyc,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int TM>
void run_sweep(const double *g, double *o, long long *t, long long *h)
{
    const int m = 256, nsm = 148;
    const size_t smem = (size_t)16 * (4 * 64 + 4) * 8;
    cudaFuncSetAttribute(k_sweep<TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int r = 0; r < 2; ++r) k_sweep<TM><<<nsm, 320, smem>>>(g, o, t, m);
    cudaError_t e = cudaDeviceSynchronize();
    const double cyc = maxof(t, h, nsm) / m;
    printf("sweep VPT 1 L 64 H 2 W 8, {nl, w} from %s: %.0f cycles/step (FMA-issue bound 1024) %s\n",
           TM ? "TMEM" : "shared memory", cyc, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main()
{
    double *g, *o;
    long long *t, h[512];
    cudaMalloc(&g, 4096 * 8);
    double hg[4096];
    for (int i = 0; i < 4096; ++i) hg[i] = 0.01 + 1e-4 * (i % 97);
    cudaMemcpy(g, hg, sizeof(hg), cudaMemcpyHostToDevice);
    cudaMalloc(&o, 1024 * 8 * 148);
    cudaMalloc(&t, 8 * 148);
    run_tp<8, 0>(o, t, h);
    run_tp<16, 0>(o, t, h);
    run_tp<8, 2>(o, t, h);
    run_tp<8, 4>(o, t, h);
    run_tp<16, 8>(o, t, h);
    run_sweep<0>(g, o, t, h);
    run_sweep<1>(g, o, t, h);
    run_sweep2<0, 0>(g, o, t, h);
    run_sweep2<0, 1>(g, o, t, h);
    run_sweep2<1, 1>(g, o, t, h);
    run_sweep3<4, 0>(g, o, t, h);
    run_sweep3<8, 0>(g, o, t, h);
    run_sweep3<8, 1>(g, o, t, h);
    run_sweep3<12, 0>(g, o, t, h);
    return 0;
}
