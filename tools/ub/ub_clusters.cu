// Microbenchmark: (1) how many thread-block clusters of each size are co-resident
// with one 384-thread / 221 KB CTA per SM (cudaOccupancyMaxActiveClusters), and
// which SMs a 7 x 16 grid leaves idle; (2) the latency of a flag + payload
// exchange between two CTAs through global memory (release store / acquire
// poll, L2), the alternative to DSMEM st.async for CTAs outside a hardware cluster.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(384, 1) k_where(unsigned *smid)
{
    extern __shared__ double sm[];
    if (threadIdx.x == 0) {
        unsigned s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        smid[blockIdx.x] = s;
        sm[0] = s;
    }
    // keep the CTA alive long enough for the whole grid to be resident together
    long long t0 = clock64();
    while (clock64() - t0 < 2000000) { }
}

__device__ __forceinline__ void st_release(unsigned *p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ping-pong: CTA 0 writes payload + flag, CTA 1 polls, reads the payload, answers
__global__ void k_pingpong(unsigned *flag, double *payload, int iters, long long *cycles, double *sink)
{
    const int me = blockIdx.x;
    double acc = 0.0;
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if ((i & 1) == me) {          // my turn to send
            payload[me * 32 + threadIdx.x] = (double)i;
            __syncwarp();
            if (threadIdx.x == 0) st_release(flag + me * 32, (unsigned)i);
        } else {                      // wait for the peer's message i
            if (threadIdx.x == 0) while (ld_acquire(flag + (1 - me) * 32) < (unsigned)i) { }
            __syncwarp();
            acc += __ldcg(payload + (1 - me) * 32 + threadIdx.x);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[me] = t1 - t0;
    sink[me * 32 + threadIdx.x] = acc;
}

int main()
{
    const size_t smem = 221 * 1024;
    cudaFuncSetAttribute(k_where, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_where, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cl : {1, 2, 4, 6, 8, 10, 12, 14, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl * 16);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k_where, &cfg);
        printf("cluster size %2d: max active clusters %3d (%3d SMs) %s\n", cl, nc, nc * cl,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    // which SMs does a 7 x 16 launch use
    unsigned *smid;
    cudaMallocManaged(&smid, 256 * sizeof(unsigned));
    for (int cl : {16, 8, 4}) {
        int ncl = (cl == 16) ? 7 : (cl == 8 ? 18 : 37);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl * ncl);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        for (int i = 0; i < 256; ++i) smid[i] = 9999;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_where, smid);
        cudaDeviceSynchronize();
        printf("grid %d x %d (%s): smid per cluster\n", ncl, cl, cudaGetErrorString(e));
        bool used[256] = {};
        for (int c = 0; c < ncl; ++c) {
            printf("  cluster %2d:", c);
            for (int i = 0; i < cl; ++i) { printf(" %3u", smid[c * cl + i]); if (smid[c * cl + i] < 256) used[smid[c * cl + i]] = true; }
            printf("\n");
        }
        printf("  idle SMs:");
        for (int i = 0; i < 148; ++i) if (!used[i]) printf(" %d", i);
        printf("\n");
    }
    // global-memory ping-pong
    unsigned *flag;
    double *payload, *sink;
    long long *cyc;
    cudaMalloc(&flag, 64 * sizeof(unsigned));
    cudaMemset(flag, 0, 64 * sizeof(unsigned));
    cudaMalloc(&payload, 64 * sizeof(double));
    cudaMalloc(&sink, 64 * sizeof(double));
    cudaMallocManaged(&cyc, 2 * sizeof(long long));
    const int iters = 20000;
    k_pingpong<<<2, 32>>>(flag, payload, iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    printf("global ping-pong (%s): %.0f cycles per one-way message (payload store + release flag -> acquire poll + payload load)\n",
           cudaGetErrorString(e), (double)cyc[0] / iters);
    return 0;
}
