// FP64 peak of the whole B200, measured: independent DFMA / DADD chains on every SM, timed with
// CUDA events.  Prints one JSON line (profiles/fp64_peak.json): DFMA flop/s (FMA = 2 flops) and
// DADD op/s -- the FP64 denominators of the roofline (ops counted unfused, one per
// dmul / dadd, so the issue-rate bound is the DADD figure) -- plus the dependent-chain latencies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>

template <int OP>  // 0 = DFMA, 1 = DADD
__global__ void __launch_bounds__(256) thr(double *out, double a, double b, int iters)
{
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = a + j + threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = OP == 0 ? fma(x[j], b, a) : __dadd_rn(x[j], b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains alive
}
__global__ void chain(double *out, long long *cyc, double a, double b, int iters, int op)
{
    double x = a + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (op == 0) x = __dadd_rn(x, b);
        else if (op == 1) x = __dmul_rn(x, b);
        else x = fma(x, b, a);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *o; long long *c;
    cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 1 << 16);
    double lat[3];
    for (int op = 0; op < 3; ++op) {
        long long h = 0;
        for (int r = 0; r < 2; ++r) chain<<<1, 1>>>(o, c, 1.0, 1.0000001, 4096, op);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        lat[op] = h / 4096.0;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    double best[2] = {0, 0};
    for (int op = 0; op < 2; ++op)
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            if (op == 0) thr<0><<<blocks, threads>>>(o, 1.0, 0.999999, iters);
            else thr<1><<<blocks, threads>>>(o, 1.0, 1e-30, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = (double)blocks * threads * iters * 8;
            const double rate = ops / (ms * 1e-3);
            if (rate > best[op]) best[op] = rate;
        }
    printf("{\"dfma_tflops\": %.2f, \"dadd_tops\": %.2f, \"dfma_per_sm_per_clk\": %.2f, \"sms\": %d, "
           "\"clock_mhz_attr\": %d, \"latency_cycles\": {\"dadd\": %.1f, \"dmul\": %.1f, \"dfma\": %.1f}, "
           "\"how\": \"%d blocks x %d threads x 8 independent chains x %d iters, best of 5, CUDA events\"}\n",
           2 * best[0] / 1e12, best[1] / 1e12, best[0] / (sms * (clk * 1e3)), sms, clk / 1000, lat[0], lat[1], lat[2],
           blocks, threads, iters);
    return 0;
}
