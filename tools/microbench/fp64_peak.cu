// fp64_peak.cu — FP64 (and FP32 FMA) pipe ceilings of this B200 (the arithmetic roofline the
// stencil kernels are checked against; MEASURED_PEAKS.json has no FP64 entry).
//
//   throughput: DFMA / DMUL / DADD (and FFMA) with 8 independent chains per thread,
//               148 x {4..32} warps, CUDA events, best of 5
//   latency:    one dependent DADD / DFMA chain in one thread, clock64
//
// Build + run:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
//               ./fp64_peak > profiles/fp_peaks.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

template <int OP, typename T>
__device__ __forceinline__ T op(T a, T b, T c) {
    if constexpr (OP == 3) return __fmaf_rn(a, b, c);
    else if constexpr (OP == 0) return __fma_rn(a, b, c);
    else if constexpr (OP == 1) return __dmul_rn(a, b);
    else return __dadd_rn(a, c);
}

template <int OP, typename T = double>
__global__ void tput(double* out, T b, T c) {
    T x[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) x[i] = op<OP>(x[i], b, c);
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += x[i];
    if (s == T(-1)) out[0] = (double)s;  // keep the chains live
}

template <int OP>
__global__ void latency(double* out, long long* cycles, double b, double c) {
    double x = out[1];
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) x = op<OP>(x, b, c);
    const long long t1 = clock64();
    out[0] = x;
    cycles[0] = t1 - t0;
}

template <int OP, typename T = double>
double run_tput(double* d, int warps_per_sm, int nsm) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 32 * (warps_per_sm > 32 ? 32 : warps_per_sm);
    const int blocks = nsm * (warps_per_sm * 32 / threads);
    tput<OP, T><<<blocks, threads>>>(d, T(0.999999), T(1e-9));  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        tput<OP, T><<<blocks, threads>>>(d, T(0.999999), T(1e-9));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double ops = (double)blocks * threads * CHAINS * ITERS;
    return ops / (best * 1e-3);
}

template <int OP>
double run_latency(double* d, long long* cyc) {
    latency<OP><<<1, 1>>>(d, cyc, 0.999999, 1e-9);
    latency<OP><<<1, 1>>>(d, cyc, 0.999999, 1e-9);
    long long h;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    return (double)h / ITERS;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    double* d;
    long long* cyc;
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    cudaMalloc(&cyc, 8);
    const int nsm = p.multiProcessorCount;
    const char* names[4] = {"dfma", "dmul", "dadd", "ffma"};
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_mhz_attr\": %.0f, \"chains_per_thread\": %d,\n",
           p.name, nsm, clk_khz / 1e3, CHAINS);
    printf(" \"throughput_ops_per_s\": {");
    for (int o = 0; o < 4; ++o) {
        printf("%s\"%s\": {", o ? ", " : "", names[o]);
        const int ws[4] = {4, 8, 16, 32};
        for (int i = 0; i < 4; ++i) {
            double v = o == 0 ? run_tput<0>(d, ws[i], nsm)
                     : o == 1 ? run_tput<1>(d, ws[i], nsm)
                     : o == 2 ? run_tput<2>(d, ws[i], nsm)
                              : run_tput<3, float>(d, ws[i], nsm);
            printf("%s\"%d_warps_per_sm\": %.4e", i ? ", " : "", ws[i], v);
        }
        printf("}");
    }
    printf("},\n \"latency_cycles\": {\"dfma\": %.2f, \"dmul\": %.2f, \"dadd\": %.2f}}\n",
           run_latency<0>(d, cyc), run_latency<1>(d, cyc), run_latency<2>(d, cyc));
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
