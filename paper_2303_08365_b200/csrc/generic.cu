// generic.cu — the parity-anchor sweep: one thread per interior point, any
// dimensionality, shape, radius and tap count.
//
// It restates apply_box (proj/include/tessera/naive.hpp:41-84) on the device
// layout: acc = 0, then acc += w[t] * in[p + delta[t]] over the canonical tap
// order, weights cast to T.  Tuned engines are checked against it and it is
// the engine for kernels no tuned engine serves (radius-2 box, 1-D, ...).
#include "common.cuh"

namespace tsr {

namespace {

template <typename T, int MAXT>
struct GenericArgs {
    int64_t n[3];  // box extents (normalised)
    int64_t base;  // element index of box corner
    int64_t pitch0, pitch1;
    T* mirror;  // LaunchCtx::mirror (fused halo exchange), or nullptr
    int64_t mshift;
    int ntaps;
    int32_t delta[MAXT];
    T w[MAXT];
};

template <typename T, int MAXT, bool EXACT>
__global__ void __launch_bounds__(256) generic_sweep_kernel(const T* __restrict__ in,
                                                            T* __restrict__ out,
                                                            const __grid_constant__ GenericArgs<T, MAXT> a) {
    const int64_t n12 = a.n[1] * a.n[2];
    const int64_t npts = a.n[0] * n12;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = p / n12;
        const int64_t r = p - i * n12;
        const int64_t j = r / a.n[2];
        const int64_t k = r - j * a.n[2];
        const int64_t idx = a.base + i * a.pitch0 + j * a.pitch1 + k;
        T acc = first<EXACT>(a.w[0], in[idx + a.delta[0]]);
#pragma unroll 4
        for (int t = 1; t < a.ntaps; ++t) acc = madd<EXACT>(acc, a.w[t], in[idx + a.delta[t]]);
        out[idx] = acc;
        if (a.mirror) a.mirror[idx + a.mshift] = acc;
    }
}

template <typename T, int MAXT>
Status launch(const LaunchCtx& c, const void* in, void* out, const int64_t lo[3],
              const int64_t hi[3]) {
    GenericArgs<T, MAXT> a;
    const Geo& g = *c.g;
    for (int d = 0; d < 3; ++d) a.n[d] = hi[d] - lo[d];
    a.base = g.origin + lo[0] * g.pitch[0] + lo[1] * g.pitch[1] + lo[2];
    a.pitch0 = g.pitch[0];
    a.pitch1 = g.pitch[1];
    a.mirror = static_cast<T*>(c.mirror);
    a.mshift = c.mirror_shift;
    a.ntaps = c.taps->ntaps;
    for (int t = 0; t < a.ntaps; ++t) {
        const int* o = c.taps->off[t];
        a.delta[t] = static_cast<int32_t>(o[0] * g.pitch[0] + o[1] * g.pitch[1] + o[2]);
        a.w[t] = static_cast<T>(c.taps->w[t]);
    }
    const int64_t npts = a.n[0] * a.n[1] * a.n[2];
    if (npts <= 0) return Status::Ok();
    int blocks = static_cast<int>(std::min<int64_t>((npts + 255) / 256, 148 * 32));
    if (c.exact)
        generic_sweep_kernel<T, MAXT, true><<<blocks, 256, 0, c.stream>>>(
            static_cast<const T*>(in), static_cast<T*>(out), a);
    else
        generic_sweep_kernel<T, MAXT, false><<<blocks, 256, 0, c.stream>>>(
            static_cast<const T*>(in), static_cast<T*>(out), a);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

template <typename T>
Status launch_t(const LaunchCtx& c, const void* in, void* out, const int64_t lo[3],
                const int64_t hi[3]) {
    const int nt = c.taps->ntaps;
    if (nt <= 32) return launch<T, 32>(c, in, out, lo, hi);
    if (nt <= 128) return launch<T, 128>(c, in, out, lo, hi);
    if (nt <= 512) return launch<T, 512>(c, in, out, lo, hi);
    return launch<T, kMaxTaps>(c, in, out, lo, hi);
}

// Halo shell copy: one warp per padded row.  Rows that lie in the a0/a1 halo
// are copied whole; interior rows copy only their a2 halo cells.
template <typename T>
__global__ void halo_copy_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t n0,
                                 int64_t n1, int64_t n2, int64_t h0, int64_t h1, int64_t h2,
                                 int64_t pitch0, int64_t pitch1, int64_t off2) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t rows1 = n1 + 2 * h1;
    const int64_t rows = (n0 + 2 * h0) * rows1;
    for (int64_t r = warp; r < rows; r += nwarps) {
        const int64_t r0 = r / rows1, r1 = r - r0 * rows1;
        const int64_t row = r0 * pitch0 + r1 * pitch1 + off2 - h2;
        const bool halo_row = r0 < h0 || r0 >= n0 + h0 || r1 < h1 || r1 >= n1 + h1;
        if (halo_row) {
            for (int64_t x = lane; x < n2 + 2 * h2; x += 32) dst[row + x] = src[row + x];
        } else {
            for (int64_t x = lane; x < 2 * h2; x += 32) {
                const int64_t e = x < h2 ? x : n2 + x;
                dst[row + e] = src[row + e];
            }
        }
    }
}

// One warp per segment of up to kSeg elements of a padded row (a 1-D grid
// is one row of 10^7 elements: one warp per row would copy it alone);
// `src`/`dst` rows start at r0*p0 + r1*p1 + off.
constexpr int64_t kSeg = 2048;
template <typename T>
__global__ void relayout_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t rows1,
                                int64_t rows, int64_t width, int64_t sp0, int64_t sp1,
                                int64_t soff, int64_t dp0, int64_t dp1, int64_t doff) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t segs = (width + kSeg - 1) / kSeg;
    for (int64_t w = warp; w < rows * segs; w += nwarps) {
        const int64_t r = w / segs, x0 = (w - r * segs) * kSeg;
        const int64_t r0 = r / rows1, r1 = r - r0 * rows1;
        const T* s = src + r0 * sp0 + r1 * sp1 + soff;
        T* d = dst + r0 * dp0 + r1 * dp1 + doff;
        const int64_t x1 = min(width, x0 + kSeg);
        for (int64_t x = x0 + lane; x < x1; x += 32) d[x] = s[x];
    }
}

template <typename T>
void relayout_t(const Geo& g, const void* src, void* dst, bool h2d, cudaStream_t s) {
    const int64_t rows1 = g.n[1] + 2 * g.h[1], rows = g.rows_padded();
    const int64_t width = g.n[2] + 2 * g.h[2];
    const int64_t items = rows * ((width + kSeg - 1) / kSeg);
    const int blocks = static_cast<int>(std::min<int64_t>((items * 32 + 255) / 256, 148 * 16));
    const int64_t hp0 = g.hpitch[0], hp1 = g.hpitch[1], dp0 = g.pitch[0], dp1 = g.pitch[1];
    const int64_t doff = g.off2 - g.h[2];
    if (h2d)
        relayout_kernel<T><<<blocks, 256, 0, s>>>(static_cast<const T*>(src), static_cast<T*>(dst),
                                                  rows1, rows, width, hp0, hp1, 0, dp0, dp1, doff);
    else
        relayout_kernel<T><<<blocks, 256, 0, s>>>(static_cast<const T*>(src), static_cast<T*>(dst),
                                                  rows1, rows, width, dp0, dp1, doff, hp0, hp1, 0);
}

}  // namespace

Status generic_sweep(const LaunchCtx& c, const void* in, void* out, const int64_t lo[3],
                     const int64_t hi[3]) {
    if (c.g->dtype == TSR_F64) return launch_t<double>(c, in, out, lo, hi);
    return launch_t<float>(c, in, out, lo, hi);
}

Status halo_copy(const Geo& g, const void* src, void* dst, cudaStream_t s) {
    const int64_t rows = g.rows_padded();
    const int blocks = static_cast<int>(std::min<int64_t>((rows * 32 + 255) / 256, 148 * 16));
    if (g.dtype == TSR_F64)
        halo_copy_kernel<double><<<blocks, 256, 0, s>>>(
            static_cast<const double*>(src), static_cast<double*>(dst), g.n[0], g.n[1], g.n[2],
            g.h[0], g.h[1], g.h[2], g.pitch[0], g.pitch[1], g.off2);
    else
        halo_copy_kernel<float><<<blocks, 256, 0, s>>>(
            static_cast<const float*>(src), static_cast<float*>(dst), g.n[0], g.n[1], g.n[2],
            g.h[0], g.h[1], g.h[2], g.pitch[0], g.pitch[1], g.off2);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

Status relayout(const Geo& g, const void* src, void* dst, bool host_to_device, cudaStream_t s) {
    if (g.dtype == TSR_F64)
        relayout_t<double>(g, src, dst, host_to_device, s);
    else
        relayout_t<float>(g, src, dst, host_to_device, s);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

}  // namespace tsr
