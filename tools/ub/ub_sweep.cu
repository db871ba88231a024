// Microbenchmark: the K1P chunk sweep in isolation (no interface exchange).
// Each lane keeps VPT vectors x L rows of state in registers; per step the
// down sweep  x = S + ca V2 + cc W2 ; z = x + nl z'  and the up sweep
// S = w z + S' read the coefficients from shared memory (H chunks per warp,
// 32/H lanes per chunk).  Prints SM cycles per step per CTA with W compute
// warps per CTA, one CTA per SM on every SM.
#include <cstdio>

template <int VPT, int L, int H, int W, int MODE>
__global__ void __launch_bounds__(32 * (W + 2), 1) k(const double *g, double *out, long long *t, int m)
{
    extern __shared__ __align__(16) double sm[];
    constexpr int K = W * H;
    constexpr int RSTR = 4 * L + 4;
    for (int i = threadIdx.x; i < K * RSTR; i += blockDim.x) sm[i] = g[i % 4096];
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int u = w * H + lane / (32 / H);
    const double2 *cd = reinterpret_cast<const double2 *>(sm + u * RSTR);
    const double *nl = sm + u * RSTR + 2 * L;
    const double *wv = nl + L;
    double S[VPT][L];
#pragma unroll
    for (int v = 0; v < VPT; ++v)
#pragma unroll
        for (int i = 0; i < L; ++i) S[v][i] = g[(i * 7 + lane + v) & 4095];
    double ca[VPT], cc[VPT];
    for (int v = 0; v < VPT; ++v) { ca[v] = g[v]; cc[v] = g[v + 1]; }
    __syncthreads();
    long long t0 = clock64();
    for (int j = 0; j < m; ++j) {
        asm volatile("" ::: "memory");   // the kernel's mbarrier waits: no hoisting of coefficient loads
        if (MODE == 1) {            // correction as its own pass
#pragma unroll
            for (int i = 0; i < L; ++i) {
                const double2 q2 = cd[i];
#pragma unroll
                for (int v = 0; v < VPT; ++v) S[v][i] = fma(q2.x, ca[v], fma(q2.y, cc[v], S[v][i]));
            }
        }
        double zp[VPT];
#pragma unroll
        for (int i = 0; i < L; ++i) {
            double2 q2 = make_double2(0.0, 0.0);
            if (MODE == 0) q2 = cd[i];
            const double nli = nl[i];
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                double x = S[v][i];
                if (MODE == 0) x = fma(q2.x, ca[v], fma(q2.y, cc[v], x));
                zp[v] = (i == 0) ? x : fma(nli, zp[v], x);
                S[v][i] = zp[v];
            }
        }
        double gn[VPT];
#pragma unroll
        for (int i = L - 1; i >= 0; --i) {
            const double wi = wv[i];
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                gn[v] = (i == L - 1) ? wi * S[v][i] : fma(wi, S[v][i], gn[v]);
                S[v][i] = gn[v];
            }
        }
#pragma unroll
        for (int v = 0; v < VPT; ++v) { ca[v] = S[v][0] * 1e-3; cc[v] = S[v][L - 1] * 1e-3; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
    double s = 0.0;
#pragma unroll
    for (int v = 0; v < VPT; ++v)
#pragma unroll
        for (int i = 0; i < L; ++i) s += S[v][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int VPT, int L, int H, int W, int MODE>
void run(const double *g, double *o, long long *t, long long *h)
{
    const int m = 256, nsm = 148;
    constexpr int K = W * H;
    const size_t smem = (size_t)K * (4 * L + 4) * 8;
    cudaFuncSetAttribute(k<VPT, L, H, W, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int r = 0; r < 2; ++r) k<VPT, L, H, W, MODE><<<nsm, 32 * W, smem>>>(g, o, t, m);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, t, 8 * nsm, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    const double dof = 32.0 * W * VPT * L;     // DOF-steps per CTA-step
    printf("VPT %d L %2d H %d W %2d mode %d: %7.0f cycles/step  %.2f DOF-steps/cycle/SM  (FMA-issue bound %.0f) %s\n",
           VPT, L, H, W, MODE, mx / m, dof / (mx / m), dof * 4 / 64.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
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
    run<1, 64, 2, 8, 0>(g, o, t, h);
    run<1, 64, 2, 8, 1>(g, o, t, h);
    run<2, 32, 4, 8, 0>(g, o, t, h);
    run<2, 32, 4, 8, 1>(g, o, t, h);
    run<1, 32, 2, 16, 0>(g, o, t, h);
    run<1, 64, 2, 4, 0>(g, o, t, h);
    run<2, 32, 4, 4, 0>(g, o, t, h);
    run<1, 64, 1, 8, 0>(g, o, t, h);
    run<4, 16, 8, 8, 0>(g, o, t, h);
    return 0;
}
