// Measured FP64 ceilings of this B200 (roofline denominators for the FP64
// kernels; MEASURED_PEAKS.json has none):
//   DFMA: every SM, 16 warps, 8 independent FMA chains per thread
//   DMMA: mma.sync m8n8k4 f64 back to back, independent accumulators
// Prints JSON.  CUDA events, best of 5 after a warm-up.
#include <cstdio>
__global__ void k_dfma(double *out, int n, double a)
{
    double y[8];
    for (int i = 0; i < 8; ++i) y[i] = threadIdx.x * 1e-3 + i;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) y[u] = fma(y[u], a, 1e-3);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += y[i];
    if (s == 12345.678) out[0] = s;
}
__global__ void k_dmma(double *out, int n)
{
    double acc[8][2];
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[u][0]), "+d"(acc[u][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[0] = s;
}
int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *o;
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int n = 1 << 14, thr = 512, blocks = sms * 2;
    float best_f = 1e30f, best_m = 1e30f, ms;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, thr>>>(o, n, 0.9999);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best_f) best_f = ms;
        cudaEventRecord(e0);
        k_dmma<<<blocks, thr>>>(o, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best_m) best_m = ms;
    }
    const double thr_total = (double)blocks * thr;
    const double dfma_flops = thr_total * n * 8 * 2.0;
    const double dmma_flops = (thr_total / 32.0) * n * 8 * (8.0 * 8 * 4 * 2);   // m8n8k4 per warp
    printf("{\"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_m8n8k4_tflops\": %.3f}\n", sms,
           dfma_flops / (best_f * 1e-3) / 1e12, dmma_flops / (best_m * 1e-3) / 1e12);
    return 0;
}
