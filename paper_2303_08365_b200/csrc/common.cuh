// common.cuh — shared geometry, tap tables and arithmetic modes for the
// B200 sweep engines.
//
// Every grid is normalised to three axes (a0, a1, a2) with a2 contiguous:
// a 1-D grid of extent n becomes (1, 1, n), a 2-D grid (n0, n1) becomes
// (1, n0, n1).  Tap offsets are shifted the same way, so one set of kernels
// serves the reference's 1-, 2- and 3-D BasicGrid<T>
// (proj/include/tessera/grid.hpp:26-132).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <type_traits>

#include "../../include/tessera_b200.h"

namespace tsr {

constexpr int kMaxTaps = 1024;

// Normalised geometry plus the device (pitched) layout of one buffer.
struct Geo {
    int dims = 0;        // the grid's own dimensionality (1..3)
    int dtype = TSR_F64;
    int esize = 8;       // bytes per element
    int64_t n[3]{};      // interior extents, normalised
    int64_t h[3]{};      // halo widths, normalised
    int64_t pitch[3]{};  // device element strides, pitch[2] == 1
    int64_t off2 = 0;    // element offset of interior a2 == 0 inside a row
    int64_t origin = 0;  // element offset of interior (0,0,0)
    int64_t elements = 0;
    // host (reference) layout strides, grid.hpp:46-49
    int64_t hpitch[3]{};
    int64_t horigin = 0;
    int64_t host_elements = 0;

    int64_t interior() const { return n[0] * n[1] * n[2]; }
    int64_t rows_padded() const { return (n[0] + 2 * h[0]) * (n[1] + 2 * h[1]); }
};

// Tap table normalised to three axes, canonical order preserved.
struct TapSet {
    int dims = 0;
    int shape = TSR_STAR;
    int radius = 0;
    int ntaps = 0;
    int off[kMaxTaps][3];
    double w[kMaxTaps];
};

// Status + message, set by the host helpers; the C-ABI turns it into
// tsr_last_error().
struct Status {
    int code = TSR_OK;
    std::string msg;
    bool ok() const { return code == TSR_OK; }
    static Status Ok() { return {}; }
    static Status Err(int c, std::string m) { return {c, std::move(m)}; }
};

Status make_geo(const tsr_grid& g, Geo& out);
Status make_taps(const tsr_kernel& k, TapSet& out);
Status check_layout(const Geo& g, const tsr_layout* l);

#define TSR_CUDA_TRY(expr)                                                              \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return ::tsr::Status::Err(TSR_ECUDA, std::string(#expr) + ": " +            \
                                                     cudaGetErrorString(_e));           \
    } while (0)

// ---------------------------------------------------------------------------
// Arithmetic modes.  EXACT reproduces `acc += w * x` of apply_box compiled
// with -ffp-contract=off (proj/CMakeLists.txt:35-38, naive.hpp:76-78): a
// separately rounded multiply and add, never contracted.  FAST is one FMA per
// tap in the same order.
// ---------------------------------------------------------------------------
template <bool EXACT>
__device__ __forceinline__ double madd(double acc, double w, double x) {
    if constexpr (EXACT) {
        return __dadd_rn(acc, __dmul_rn(w, x));
    } else {
        return __fma_rn(w, x, acc);
    }
}

template <bool EXACT>
__device__ __forceinline__ float madd(float acc, float w, float x) {
    if constexpr (EXACT) {
        return __fadd_rn(acc, __fmul_rn(w, x));
    } else {
        return __fmaf_rn(w, x, acc);
    }
}

// First tap: apply_box starts from acc = T(0) (naive.hpp:75), so the first
// sum is 0 + w*x, which maps -0 to +0.  Kept explicit for bitwise parity.
template <bool EXACT, typename T>
__device__ __forceinline__ T first(T w, T x) {
    return madd<EXACT>(T(0), w, x);
}

// Leading tap without the "0 +": the reference's accumulator starts at +0 and
// can never become -0 (x + y is -0 only if both are -0), so a sum started
// from the first product differs from it at most in the sign of a zero
// result — in intermediate fused levels too, because a signed zero addend
// never changes a nonzero sum.  Engines that use lead() apply fix_zero() to
// every value they store, restoring the reference bit pattern exactly.
__device__ __forceinline__ double lead(double w, double x) { return __dmul_rn(w, x); }
__device__ __forceinline__ float lead(float w, float x) { return __fmul_rn(w, x); }
template <bool EXACT, typename T>
__device__ __forceinline__ T fix_zero(T v) {
    if constexpr (EXACT) return v + T(0);
    else return v;
}

// N consecutive outputs of one row: vector stores (16 B, or N elements when
// shorter) wherever a whole vector is inside the output tile, scalar
// predicated stores at its ragged edge.  `o` must be vector aligned: device rows start interior column 0 on a
// 128-B boundary and every engine's column offsets are vector multiples.
template <typename T, int N>
__device__ __forceinline__ void store_row(T* o, const T (&v)[N], const bool (&ok)[N]) {
    constexpr int NV = (16 / (int)sizeof(T)) < N ? 16 / (int)sizeof(T) : N;  // vector width
    static_assert(N % NV == 0, "row length must be a multiple of the vector");
#pragma unroll
    for (int c = 0; c < N; c += NV) {
        bool all = true, any = false;
#pragma unroll
        for (int u = 0; u < NV; ++u) all &= ok[c + u], any |= ok[c + u];
        if (!any) continue;  // lanes outside the output tile skip the scalar path too
        if (all) {
            if constexpr (sizeof(T) == 8 && NV == 2) {
                *reinterpret_cast<double2*>(o + c) = make_double2(v[c], v[c + 1]);
            } else if constexpr (sizeof(T) == 4 && NV == 4) {
                *reinterpret_cast<float4*>(o + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
            } else if constexpr (sizeof(T) == 4 && NV == 2) {
                *reinterpret_cast<float2*>(o + c) = make_float2(v[c], v[c + 1]);
            } else {
#pragma unroll
                for (int u = 0; u < NV; ++u) o[c + u] = v[c + u];
            }
        } else {
#pragma unroll
            for (int u = 0; u < NV; ++u)
                if (ok[c + u]) o[c + u] = v[c + u];
        }
    }
}

// Correctly rounded multiply / add, never contracted into an FMA.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// True when every tap carries the same weight (the reference's box kernels:
// 1/9, 1/25, 1/27): engines then share one rounded product per input value.
inline bool uniform_weights(const TapSet& t) {
    for (int i = 1; i < t.ntaps; ++i)
        if (t.w[i] != t.w[0]) return false;
    return true;
}

// Compile-time loop: f(std::integral_constant<int, i>) for i in [0, N).
template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N>(f);
    }
}

// ---------------------------------------------------------------------------
// Engine entry points (each in its own translation unit).
// ---------------------------------------------------------------------------
struct LaunchCtx {
    const Geo* g;
    const TapSet* taps;
    bool exact;
    cudaStream_t stream;
    // Output planes [lo0, hi0) along the grid's own axis 0 (normalised axis
    // 3 - dims): the slab axis of a multi-GPU partition.  A fused pass still
    // reads every input plane its dependency cone needs; only the stores are
    // restricted, so interior and seam planes can be launched separately.
    int64_t lo0 = 0;
    int64_t hi0 = INT64_MAX;
    // Fused halo exchange: every value stored to `out` is also stored to
    // `mirror` at the same element index + mirror_shift (a neighbour slab's
    // ghost planes in peer memory, same layout).  nullptr = no mirror.
    void* mirror = nullptr;
    int64_t mirror_shift = 0;

    int64_t range_lo() const { return lo0; }
    int64_t range_hi() const { return std::min<int64_t>(hi0, g->n[3 - g->dims]); }
};

// One sweep over the normalised box [lo, hi) from `in` to `out` (apply_box).
Status generic_sweep(const LaunchCtx& c, const void* in, void* out, const int64_t lo[3],
                     const int64_t hi[3]);

// Tuned engines.  `supports` reports whether an engine serves the kernel and
// the largest fused step count it accepts; `run` advances `k` steps from `in`
// to `out` in one pass over HBM (in != out).
struct Engine {
    const char* name;
    bool (*supports)(const Geo&, const TapSet&, int* max_fused, int* default_fused);
    Status (*run)(const LaunchCtx&, const void* in, void* out, int k);
    // Optional: the default fused depth in FAST mode when it differs from
    // the EXACT one (nullptr = same as supports()'s default_fused).
    int (*fast_default)(const Geo&, const TapSet&) = nullptr;
    // Optional: the largest fused depth in FAST mode when it differs.
    int (*fast_max)(const Geo&, const TapSet&) = nullptr;
};
const Engine* find_engine(const Geo& g, const TapSet& t, int* max_fused, int* default_fused);

Status halo_copy(const Geo& g, const void* src, void* dst, cudaStream_t s);
// Whole padded grid (interior + halo) between the host layout (grid.hpp:46-49,
// contiguous rows of n2+2h2) and the pitched device layout, device to device:
// lets tsr_run move a grid over PCIe as one contiguous copy.
Status relayout(const Geo& g, const void* src, void* dst, bool host_to_device, cudaStream_t s);

}  // namespace tsr
