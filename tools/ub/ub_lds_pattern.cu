// Microbenchmark: shared-memory wavefronts of warp-wide LDS.128 / LDS.64 loads
// for the access patterns of the K1P coefficient stream (one address per
// half-warp).  Prints cycles per load instruction per SM with 8 warps.
#include <cstdio>
template <int MODE>
__global__ void k(const double *g, double *out, long long *t, int iters)
{
    __shared__ __align__(16) double sm[6144];
    for (int i = threadIdx.x; i < 6144; i += blockDim.x) sm[i] = g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, h = lane >> 4;
    // base offset (doubles) of this half-warp's 16-B record
    int base;
    if (MODE == 0) base = 0;                       // every lane the same address
    else if (MODE == 1) base = h * 516;            // halves 4128 B apart (K1P regions)
    else if (MODE == 2) base = h * 2;              // halves adjacent 16 B in one line
    else base = (lane & 7) * 2 + w * 0;            // 8 distinct addresses (one line)
    double2 acc[8];
    for (int u = 0; u < 8; ++u) acc[u] = make_double2(0.0, 0.0);
    double acc1 = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int off = (it & 63) * 4;             // walk rows (stride 32 B per row, like a double4 record)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double2 v = *reinterpret_cast<const double2 *>(sm + base + off + u * 640);
            acc[u].x += v.x; acc[u].y += v.y;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
    for (int u = 0; u < 8; ++u) acc1 += acc[u].x + acc[u].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc1;
}
int main()
{
    double *g, *o; long long *t, h[1];
    cudaMalloc(&g, 16384 * 8); cudaMemset(g, 0, 16384 * 8);
    cudaMalloc(&o, 256 * 8 * 148); cudaMalloc(&t, 8 * 148);
    const int iters = 4096;
    const char *names[4] = {"broadcast (1 address)", "2 addresses, 4128 B apart", "2 addresses, adjacent 16 B",
                            "8 addresses in one 128-B line"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int r = 0; r < 2; ++r) {
            if (mode == 0) k<0><<<1, 256>>>(g, o, t, iters);
            if (mode == 1) k<1><<<1, 256>>>(g, o, t, iters);
            if (mode == 2) k<2><<<1, 256>>>(g, o, t, iters);
            if (mode == 3) k<3><<<1, 256>>>(g, o, t, iters);
        }
        cudaMemcpy(h, t, 8, cudaMemcpyDeviceToHost);
        printf("LDS.128 %-32s: %.2f cycles per warp-instruction (8 warps)\n", names[mode],
               (double)h[0] / (iters * 8.0 * 8.0));
    }
    return 0;
}
