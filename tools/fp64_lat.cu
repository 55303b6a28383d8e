// Microbenchmark: dependent-chain latency and throughput of DADD / DMUL / DFMA on one SM.
#include <cstdio>
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
__global__ void thr(double *out, long long *cyc, double a, double b, int iters)
{
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
        x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main()
{
    double *o; long long *c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 1 << 16);
    long long h;
    const char *nm[3] = {"DADD", "DMUL", "DFMA"};
    for (int op = 0; op < 3; ++op) {
        chain<<<1, 1>>>(o, c, 1.0, 1.0000001, 4096, op);
        chain<<<1, 1>>>(o, c, 1.0, 1.0000001, 4096, op);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%s dependent latency: %.1f cycles\n", nm[op], h / 4096.0);
    }
    for (int warps = 1; warps <= 32; warps *= 2) {
        thr<<<1, 32 * warps>>>(o, c, 1.0, 0.999999, 4096);
        thr<<<1, 32 * warps>>>(o, c, 1.0, 0.999999, 4096);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("warps %2d: 8 indep DFMA chains/thread: %.2f cycles per warp-DFMA per SM (%.1f lane-flop/cycle)\n", warps,
               h / (4096.0 * 8 * warps), 2.0 * 32 * 4096 * 8 * warps / h);
    }
    return 0;
}
