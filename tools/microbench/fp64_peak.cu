// FP64 issue-rate microbenchmark for the roofline's arithmetic ceiling:
// independent DFMA / DMUL / DADD chains (ILP 8 per thread), full occupancy.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void kern(double* out, double a, double b, int iters) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = __fma_rn(x[i], a, b);
            if (OP == 1) x[i] = __dmul_rn(x[i], a);
            if (OP == 2) x[i] = __dadd_rn(x[i], b);
            if (OP == 3) x[i] = (i & 1) ? __dmul_rn(x[i], a) : __dadd_rn(x[i], b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"DFMA", "DMUL", "DADD", "DMUL+DADD"};
    for (int threads : {256, 512, 1024}) {
        for (int op = 0; op < 4; ++op) {
            const int blocks = nsm * (2048 / threads), iters = 4096;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (op == 0) kern<0><<<blocks, threads>>>(out, 0.999, 1e-9, iters);
                if (op == 1) kern<1><<<blocks, threads>>>(out, 0.999, 1e-9, iters);
                if (op == 2) kern<2><<<blocks, threads>>>(out, 0.999, 1e-9, iters);
                if (op == 3) kern<3><<<blocks, threads>>>(out, 0.999, 1e-9, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = (double)blocks * threads * iters * 8;
            int clk = 0;
            cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            printf("%-10s threads/blk %4d: %.2f T instr-lanes/s = %.1f per SM per clk (@%.0f MHz max)\n",
                   names[op], threads, ops / ms / 1e9, ops / (ms * 1e-3) / nsm / (clk * 1e3),
                   clk / 1e3);
        }
    }
    return 0;
}
