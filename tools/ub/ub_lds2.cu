// Microbenchmark: SM throughput of warp-wide shared loads (LDS.64 / LDS.128)
// when each group of 32/G lanes reads one address (G = 1, 2, 4, 8 distinct
// addresses, records 4128 B apart as in K1P's per-chunk regions).
#include <cstdio>
template <int VEC, int G>
__global__ void k(const double *g, double *out, long long *t, int iters)
{
    __shared__ __align__(16) double sm[6144];
    for (int i = threadIdx.x; i < 6144; i += blockDim.x) sm[i] = g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int grp = lane / (32 / G);
    const int base = grp * 516 % 4096;
    double acc[8];
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int off = (it & 31) * 4;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (VEC == 2) {
                double2 v = *reinterpret_cast<const double2 *>(sm + base + off + u * 256);
                acc[u] += v.x + v.y;
            } else {
                acc[u] += sm[base + off + u * 256];
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) t[0] = t1 - t0;
    double s = 0;
    for (int u = 0; u < 8; ++u) s += acc[u];
    out[threadIdx.x] = s;
}
template <int VEC, int G>
void run(const double *g, double *o, long long *t)
{
    const int iters = 2048;
    long long h;
    for (int r = 0; r < 2; ++r) k<VEC, G><<<1, 256>>>(g, o, t, iters);
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("LDS.%d, %d distinct address(es) per warp: %.2f SM cycles per warp-instruction (8 warps)\n",
           VEC * 64, G, (double)h / (iters * 8.0 * 8.0));
}
int main()
{
    double *g, *o; long long *t;
    cudaMalloc(&g, 6144 * 8); cudaMemset(g, 0, 6144 * 8);
    cudaMalloc(&o, 256 * 8); cudaMalloc(&t, 8);
    run<1, 1>(g, o, t); run<1, 2>(g, o, t); run<1, 4>(g, o, t); run<1, 8>(g, o, t);
    run<2, 1>(g, o, t); run<2, 2>(g, o, t); run<2, 4>(g, o, t); run<2, 8>(g, o, t);
    return 0;
}
