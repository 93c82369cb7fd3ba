// stream1d.cu — 1-D sweeps (Heat-1D, Star-1D5P: any radius) with K time steps
// fused per HBM pass.
//
// Each CTA owns a segment of kSeg points; it loads the segment plus r*K halo
// points per side into shared memory once, advances K levels there
// (ping-pong buffers, one __syncthreads per level; level l is computed on the
// segment widened by r*(K-l), the overlapped-tiling cone), and stores the
// segment.  Cells outside the interior keep their level-0 value at every
// level (Dirichlet halo, proj/include/tessera/grid.hpp:14-18); interior cells
// sum the taps in canonical order from acc = 0 exactly as apply_box does
// (proj/include/tessera/naive.hpp:69-82), so EXACT mode is bitwise naive_run.
#include "common.cuh"

namespace tsr {

namespace {

constexpr int kThreads = 256;
constexpr int kSeg = kThreads * 8;  // output points per CTA
constexpr int kMaxK = 16;
constexpr int kMaxTaps1 = 9;        // radius <= 4

template <typename T>
struct S1Args {
    int64_t n;       // interior points
    int64_t h;       // halo width
    int64_t origin;  // element index of interior point 0
    int64_t lo, hi;  // output points [lo, hi)
    T* mirror;       // LaunchCtx::mirror (fused halo exchange), or nullptr
    int64_t mshift;
    int r, ntaps;
    int off[kMaxTaps1];
    T w[kMaxTaps1];
};

template <typename T, bool EXACT>
__global__ void __launch_bounds__(kThreads) stream1d_kernel(const T* __restrict__ in,
                                                           T* __restrict__ out,
                                                           const __grid_constant__ S1Args<T> a,
                                                           int K) {
    extern __shared__ __align__(16) unsigned char smem1[];
    const int tid = threadIdx.x;
    const int64_t seg_lo = a.lo + (int64_t)blockIdx.x * kSeg;
    const int64_t seg_hi = min(seg_lo + kSeg, a.hi);
    const int rk = a.r * K;
    const int64_t base = seg_lo - rk;  // interior index of buffer slot 0
    const int L = (int)(seg_hi - seg_lo) + 2 * rk;
    const int cap = kSeg + 2 * a.r * kMaxK;
    T* src = reinterpret_cast<T*>(smem1);
    T* dst = src + cap;

    // the dependency cone, clipped to the allocation (halo included)
    for (int j = tid; j < L; j += kThreads) {
        const int64_t p = base + j;
        src[j] = (p >= -a.h && p < a.n + a.h) ? in[a.origin + p] : T(0);
    }
    __syncthreads();
    for (int l = 1; l <= K; ++l) {
        const int64_t lo = max(seg_lo - (int64_t)a.r * (K - l), (int64_t)0);
        const int64_t hi = min(seg_hi + (int64_t)a.r * (K - l), a.n);
        for (int j = tid; j < L; j += kThreads) {
            const int64_t p = base + j;
            T v = src[j];  // outside the interior: the level-0 (halo) value
            if (p >= lo && p < hi) {
                v = first<EXACT>(a.w[0], src[j + a.off[0]]);
                for (int t = 1; t < a.ntaps; ++t) v = madd<EXACT>(v, a.w[t], src[j + a.off[t]]);
            }
            dst[j] = v;
        }
        __syncthreads();
        T* tmp = src;
        src = dst;
        dst = tmp;
    }
    for (int j = rk + tid; j < rk + (int)(seg_hi - seg_lo); j += kThreads) {
        const int64_t idx = a.origin + base + j;
        out[idx] = src[j];
        if (a.mirror) a.mirror[idx + a.mshift] = src[j];
    }
}

bool supports(const Geo& g, const TapSet& t, int* max_fused, int* default_fused) {
    if (t.dims != 1 || t.ntaps > kMaxTaps1 || t.ntaps != 2 * t.radius + 1) return false;
    *max_fused = kMaxK;
    *default_fused = 8;
    return true;
}

template <typename T>
Status launch(const LaunchCtx& c, const void* in, void* out, int k) {
    const Geo& g = *c.g;
    S1Args<T> a;
    a.n = g.n[2];
    a.h = g.h[2];
    a.origin = g.origin;
    a.lo = c.range_lo();
    a.hi = c.range_hi();
    if (a.hi <= a.lo) return Status::Ok();
    a.mirror = static_cast<T*>(c.mirror);
    a.mshift = c.mirror_shift;
    a.r = c.taps->radius;
    a.ntaps = c.taps->ntaps;
    for (int q = 0; q < a.ntaps; ++q) {
        a.off[q] = c.taps->off[q][2];
        a.w[q] = static_cast<T>(c.taps->w[q]);
    }
    const int smem = 2 * (kSeg + 2 * a.r * kMaxK) * (int)sizeof(T);
    const unsigned blocks = (unsigned)((a.hi - a.lo + kSeg - 1) / kSeg);
    if (c.exact) {
        TSR_CUDA_TRY(cudaFuncSetAttribute(stream1d_kernel<T, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        stream1d_kernel<T, true><<<blocks, kThreads, smem, c.stream>>>(
            static_cast<const T*>(in), static_cast<T*>(out), a, k);
    } else {
        TSR_CUDA_TRY(cudaFuncSetAttribute(stream1d_kernel<T, false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        stream1d_kernel<T, false><<<blocks, kThreads, smem, c.stream>>>(
            static_cast<const T*>(in), static_cast<T*>(out), a, k);
    }
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

Status run(const LaunchCtx& c, const void* in, void* out, int k) {
    if (k < 1 || k > kMaxK) return Status::Err(TSR_EUNSUPPORTED, "stream1d fuses 1..16 steps");
    if (c.g->dtype == TSR_F64) return launch<double>(c, in, out, k);
    return launch<float>(c, in, out, k);
}

}  // namespace

extern const Engine kStream1dEngine = {"stream1d_smem", supports, run};

}  // namespace tsr
