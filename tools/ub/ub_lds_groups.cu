// Microbenchmark: cycles per warp-wide shared load when the warp's lanes split
// into G groups (32/G consecutive lanes each) that each read ONE record, the G
// records either adjacent (one contiguous G*VEC*8-byte span) or 4128 B apart.
// This is the coefficient stream of K1P (a chunk's lanes read the same row
// record).  8 warps per CTA, one CTA per SM on every SM; prints SM cycles per
// warp-instruction (1.0 = one wavefront per instruction at full LSU rate).
#include <cstdio>
template <int VEC, int G, bool ADJ>
__global__ void k(const double *g, double *out, long long *t, int iters)
{
    __shared__ __align__(16) double sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int grp = lane / (32 / G);
    // record of this group: adjacent records (stride VEC doubles) or 4128 B apart
    const int base = ADJ ? grp * VEC : grp * 516;
    unsigned acc[8];
    for (int u = 0; u < 8; ++u) acc[u] = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int off = (it & 15) * 8 * VEC;   // walk rows: G records per row, row stride 8 records
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double *p = sm + ((base + off + u * 256) & 4095);
            // volatile asm keeps the full load width; consumers are cheap
            // 32-bit logic ops on the low words
            const unsigned a = (unsigned)__cvta_generic_to_shared(p);
            if (VEC == 2) {
                unsigned long long x, y;
                asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a));
                acc[u] ^= (unsigned)x ^ (unsigned)y;
            } else {
                unsigned long long x;
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x) : "r"(a));
                acc[u] ^= (unsigned)x;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
    double s = 0.0;
    for (int u = 0; u < 8; ++u) s += (double)acc[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int VEC, int G, bool ADJ>
void run(const char *name, const double *g, double *o, long long *t, long long *h, int nsm)
{
    const int iters = 4096;
    for (int r = 0; r < 2; ++r) k<VEC, G, ADJ><<<nsm, 256>>>(g, o, t, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, t, 8 * nsm, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("LDS.%d  %d group(s) %-9s: %.2f SM cycles per warp-instruction (8 warps/SM)\n", VEC * 64, G,
           ADJ ? "adjacent" : "apart", mx / (iters * 8.0 * 8.0));
}

int main()
{
    double *g, *o;
    long long *t, h[512];
    int nsm = 148;
    cudaMalloc(&g, 8192 * 8);
    cudaMemset(g, 0, 8192 * 8);
    cudaMalloc(&o, 256 * 8 * nsm);
    cudaMalloc(&t, 8 * nsm);
    run<2, 1, true>("", g, o, t, h, nsm);
    run<2, 2, true>("", g, o, t, h, nsm);
    run<2, 2, false>("", g, o, t, h, nsm);
    run<2, 4, true>("", g, o, t, h, nsm);
    run<2, 4, false>("", g, o, t, h, nsm);
    run<2, 8, true>("", g, o, t, h, nsm);
    run<1, 1, true>("", g, o, t, h, nsm);
    run<1, 2, true>("", g, o, t, h, nsm);
    run<1, 2, false>("", g, o, t, h, nsm);
    run<1, 4, true>("", g, o, t, h, nsm);
    run<1, 8, true>("", g, o, t, h, nsm);
    return 0;
}
