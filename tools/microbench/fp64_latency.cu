// FP64 throughput vs (warps per SM, independent chains per thread): how much
// parallelism the FP64 pipe needs to stay busy (DADD chains).
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void kern(double* out, double b, int iters) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __dadd_rn(x[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

template <int ILP>
void run(double* out, int nsm, int warps_per_sm) {
    const int threads = 32 * warps_per_sm, blocks = nsm, iters = 8192;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        kern<ILP><<<blocks, threads>>>(out, 1e-9, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    const double ops = (double)blocks * threads * iters * ILP;
    const double per_clk = ops / (ms * 1e-3) / nsm / 1.965e9;
    printf("warps/SM %2d ILP %d: %5.1f DADD lanes/clk/SM (%.0f%% of 62)\n", warps_per_sm, ILP,
           per_clk, per_clk / 62 * 100);
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 16, 32}) {
        run<1>(out, nsm, w);
        run<2>(out, nsm, w);
        run<4>(out, nsm, w);
        run<8>(out, nsm, w);
    }
    return 0;
}
