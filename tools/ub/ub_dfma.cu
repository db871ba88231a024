#include <cstdio>
__global__ void k(double *out, long long *t, int n, double a)
{
    __shared__ double st[4 * 1024];
    double x = threadIdx.x * 1e-3, y[8];
    for (int i = 0; i < 8; ++i) y[i] = x + i;
    for (int i = threadIdx.x; i < 4 * 1024; i += 32) st[i] = i * 1e-6;
    __syncwarp();
    long long t0 = clock64();
    // (a) dependent chain
#pragma unroll 16
    for (int i = 0; i < n; ++i) x = fma(x, a, 1.0);
    long long t1 = clock64();
    // (b) 8 independent chains
    for (int i = 0; i < n / 8; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) y[u] = fma(y[u], a, 1.0);
    }
    long long t2 = clock64();
    // (c) up-sweep shape: chain with smem operand loads + stores
    double g = 0.0;
    for (int b = 0; b < 512 / 8; ++b) {
        double yy[8], pp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { yy[u] = st[(b * 8 + u) * 8 + (threadIdx.x & 7)]; pp[u] = a; }
#pragma unroll
        for (int u = 0; u < 8; ++u) { g = fma(pp[u], g, yy[u]); yy[u] = g; }
#pragma unroll
        for (int u = 0; u < 8; ++u) st[(b * 8 + u) * 8 + (threadIdx.x & 7)] = yy[u];
    }
    long long t3 = clock64();
    // (d) chain of DADD
    double z = x;
#pragma unroll 16
    for (int i = 0; i < n; ++i) z = z * a;
    long long t4 = clock64();
    if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; }
    double s = x + g + z;
    for (int i = 0; i < 8; ++i) s += y[i];
    out[threadIdx.x] = s;
}
int main()
{
    double *o; long long *t, h[4];
    cudaMalloc(&o, 32 * 8); cudaMalloc(&t, 32);
    int n = 4096;
    for (int r = 0; r < 3; ++r) k<<<1, 32>>>(o, t, n, 0.999);
    cudaMemcpy(h, t, 32, cudaMemcpyDeviceToHost);
    printf("dep DFMA chain: %.2f cyc/op\n", (double)h[0] / n);
    printf("8 indep chains: %.2f cyc/op (per warp instr)\n", (double)h[1] / n);
    printf("up-sweep shape: %.2f cyc/row\n", (double)h[2] / 512);
    printf("dep DMUL chain: %.2f cyc/op\n", (double)h[3] / n);
    k<<<148 * 4, 32>>>(o, t, n, 0.999);
    cudaDeviceSynchronize();
    return 0;
}
