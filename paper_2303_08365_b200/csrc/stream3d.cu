// stream3d.cu — 3-D radius-1 star (7-point) sweep, 2.5-D streaming.
//
// One thread owns an (a1, a2) column and walks a chunk of a0 planes, keeping
// the column's previous / current / next values in registers (the register
// tier of the paper's pattern mapping); the four in-plane neighbours come
// through L1/L2.  Taps are accumulated in the oracle's canonical order:
// (-1,0,0) (0,-1,0) (0,0,-1) (0,0,0) (0,0,1) (0,1,0) (1,0,0)
// (proj/src/kernel.cpp:19-43 orders them; naive.hpp:76-78 sums them).
#include "common.cuh"

namespace tsr {

namespace {

constexpr int kBX = 32;  // threads along a2 (contiguous)
constexpr int kBY = 8;   // threads along a1

template <typename T>
struct Star3Args {
    int64_t n0, n1, n2;
    int64_t pitch0, pitch1;
    int64_t origin;
    int64_t chunk;  // a0 planes per CTA
    int64_t lo0, hi0;  // output planes [lo0, hi0) of a0
    T* mirror;  // LaunchCtx::mirror (fused halo exchange), or nullptr
    int64_t mshift;
    T w[7];
};

template <typename T, bool EXACT>
__global__ void __launch_bounds__(kBX* kBY) star3d_r1_kernel(const T* __restrict__ in,
                                                            T* __restrict__ out,
                                                            const __grid_constant__ Star3Args<T> a) {
    const int64_t k = blockIdx.x * (int64_t)kBX + threadIdx.x;
    const int64_t j = blockIdx.y * (int64_t)kBY + threadIdx.y;
    const int64_t i0 = a.lo0 + blockIdx.z * a.chunk;
    const int64_t i1 = min(i0 + a.chunk, a.hi0);
    if (k >= a.n2 || j >= a.n1) return;
    int64_t p = a.origin + i0 * a.pitch0 + j * a.pitch1 + k;
    const int64_t P0 = a.pitch0, P1 = a.pitch1;
    T prev = __ldg(in + p - P0);
    T cur = __ldg(in + p);
    for (int64_t i = i0; i < i1; ++i) {
        const T next = __ldg(in + p + P0);
        T acc = first<EXACT>(a.w[0], prev);
        acc = madd<EXACT>(acc, a.w[1], __ldg(in + p - P1));
        acc = madd<EXACT>(acc, a.w[2], __ldg(in + p - 1));
        acc = madd<EXACT>(acc, a.w[3], cur);
        acc = madd<EXACT>(acc, a.w[4], __ldg(in + p + 1));
        acc = madd<EXACT>(acc, a.w[5], __ldg(in + p + P1));
        acc = madd<EXACT>(acc, a.w[6], next);
        out[p] = acc;
        if (a.mirror) a.mirror[p + a.mshift] = acc;
        prev = cur;
        cur = next;
        p += P0;
    }
}

bool supports(const Geo& g, const TapSet& t, int* max_fused, int* default_fused) {
    if (t.dims != 3 || t.shape != TSR_STAR || t.radius != 1 || t.ntaps != 7) return false;
    *max_fused = 1;
    *default_fused = 1;
    return true;
}

template <typename T>
Status launch(const LaunchCtx& c, const void* in, void* out) {
    const Geo& g = *c.g;
    Star3Args<T> a;
    a.n0 = g.n[0];
    a.n1 = g.n[1];
    a.n2 = g.n[2];
    a.pitch0 = g.pitch[0];
    a.pitch1 = g.pitch[1];
    a.origin = g.origin;
    a.mirror = static_cast<T*>(c.mirror);
    a.mshift = c.mirror_shift;
    for (int t = 0; t < 7; ++t) a.w[t] = static_cast<T>(c.taps->w[t]);
    const int64_t gx = (g.n[2] + kBX - 1) / kBX, gy = (g.n[1] + kBY - 1) / kBY;
    // Enough CTAs for ~8 resident per SM, but chunks of >= 32 planes.
    int64_t nz = std::max<int64_t>(1, (148 * 8 + gx * gy - 1) / (gx * gy));
    a.lo0 = c.range_lo();
    a.hi0 = c.range_hi();
    if (a.hi0 <= a.lo0) return Status::Ok();
    const int64_t span = a.hi0 - a.lo0;
    a.chunk = std::max<int64_t>(32, (span + nz - 1) / nz);
    nz = (span + a.chunk - 1) / a.chunk;
    dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>(nz));
    dim3 block(kBX, kBY);
    if (c.exact)
        star3d_r1_kernel<T, true><<<grid, block, 0, c.stream>>>(static_cast<const T*>(in),
                                                                 static_cast<T*>(out), a);
    else
        star3d_r1_kernel<T, false><<<grid, block, 0, c.stream>>>(static_cast<const T*>(in),
                                                                  static_cast<T*>(out), a);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

Status run(const LaunchCtx& c, const void* in, void* out, int k) {
    if (k != 1) return Status::Err(TSR_EUNSUPPORTED, "star3d_r1 fuses one step per pass");
    if (c.g->dtype == TSR_F64) return launch<double>(c, in, out);
    return launch<float>(c, in, out);
}

}  // namespace

extern const Engine kStar3dR1Engine = {"star3d_r1_stream", supports, run};

}  // namespace tsr
