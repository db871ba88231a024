#include <cstdio>
__global__ void k(double *out, long long *t, int n, double a)
{
    double y[8];
    for (int i = 0; i < 8; ++i) y[i] = threadIdx.x * 1e-3 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n / 8; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) y[u] = fma(y[u], a, 1.0);
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) t[threadIdx.x >> 5] = t1 - t0;
    double s = 0;
    for (int i = 0; i < 8; ++i) s += y[i];
    out[threadIdx.x] = s;
}
int main()
{
    double *o; long long *t, h[32];
    cudaMalloc(&o, 1024 * 8); cudaMalloc(&t, 32 * 8);
    int n = 8192;
    for (int warps = 1; warps <= 16; warps *= 2) {
        for (int r = 0; r < 3; ++r) k<<<1, 32 * warps>>>(o, t, n, 0.999);
        cudaMemcpy(h, t, warps * 8, cudaMemcpyDeviceToHost);
        printf("warps/CTA %2d: %.2f cycles per DFMA warp-instr per warp\n", warps, (double)h[0] / n);
    }
    return 0;
}
