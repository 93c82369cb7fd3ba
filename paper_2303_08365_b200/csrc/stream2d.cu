// stream2d.cu — 2-D star (r = 1, 2) and box (r = 1, 2) sweeps with K time
// steps fused per HBM pass.
//
// Register-level tetrominoes (north_star tier 1) + temporal blocking (tier 2):
// every warp owns a strip of 32*V columns and streams down the rows.  Each
// lane keeps, for every fused level l = 0..K-1, the last 2R+1 rows of its V
// columns in registers; level l+1 of row x is computed as soon as level l of
// row x+R exists, so one pass over HBM advances K time steps.  Column
// neighbours come from the adjacent lanes through warp shuffles.  Strips
// overlap by R*K columns per side (overlapped tiling): edge lanes compute
// values that are never stored.
//
// Dirichlet semantics under fusion (proj/include/tessera/grid.hpp:14-18): a
// cell outside the interior keeps its level-0 (halo) value at every level,
// so a fused pass reads exactly what K separate apply_box sweeps would.
// Interior cells sum the taps in canonical lexicographic order (dr, dc),
// identical per point to apply_box (proj/include/tessera/naive.hpp:69-82),
// so EXACT mode is bitwise equal to naive_run for any K.
#include "common.cuh"

namespace tsr {

namespace {

constexpr int kWarpsPerBlock = 4;

template <typename T>
struct S2Args {
    int64_t rows, cols;      // interior extents (normalised a1, a2)
    int64_t hrow;            // halo rows (a1)
    int64_t pitch;           // row pitch (elements)
    int64_t origin;          // element index of interior (0,0)
    int64_t col_lo, col_hi;  // allocated column range relative to interior col 0
    int64_t chunk;           // output rows per warp
    int64_t row_lo, row_hi;  // output rows [row_lo, row_hi) (the grid's axis 0)
    int64_t nstrips;
    int64_t wout;            // output columns per strip
    int64_t hl;              // left margin of the strip (>= R*K, vector aligned)
    int64_t total_warps;
    T* mirror;  // LaunchCtx::mirror (fused halo exchange), or nullptr
    int64_t mshift;
    T w[25];
};

template <int R, bool BOX>
__host__ __device__ constexpr bool has_tap(int dr, int dc) {
    return BOX || dr == 0 || dc == 0;
}

template <typename T, int V>
struct Vec;
template <>
struct Vec<double, 2> {
    using type = double2;
};
template <>
struct Vec<float, 4> {
    using type = float4;
};
template <>
struct Vec<double, 4> {
    using type = double4;
};

// Level-0 rows are staged through a per-warp shared-memory ring filled by
// cp.async (16 B per lane per row, zero-filled outside the allocation), kDepth
// rows ahead of use, so DRAM latency hides behind kDepth row steps instead of
// the 2R+1 a register prefetch can afford.
constexpr int kDepth = 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool ok) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(gmem),
                 "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One lane's V outputs of a row: a vector store when the whole run is in the
// output strip, predicated scalars otherwise.
template <typename T, int V>
__device__ __forceinline__ void store_vals(T* dst, const T (&res)[V], const bool (&cout)[V],
                                           bool all_out) {
    if (all_out) {
        if constexpr (sizeof(T) * V == 16) {
            typename Vec<T, V>::type o;
            T* os = reinterpret_cast<T*>(&o);
#pragma unroll
            for (int v = 0; v < V; ++v) os[v] = res[v];
            *reinterpret_cast<typename Vec<T, V>::type*>(dst) = o;
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v) dst[v] = res[v];
        }
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (cout[v]) dst[v] = res[v];
    }
}

// Fills the R halo columns on each side of a row from the neighbouring lanes.
template <typename T, int V, int R>
__device__ __forceinline__ void exchange(T (&row)[V + 2 * R]) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        row[r] = __shfl_up_sync(0xffffffffu, row[V + r], 1);          // left: lane-1's tail
        row[V + R + r] = __shfl_down_sync(0xffffffffu, row[R + r], 1);  // right: lane+1's head
    }
}

// SEP: horizontal 3-sums of one window row (its V values at [1, V+1), the
// outer neighbours from the adjacent lanes), consecutive pairs shared.
template <typename T, int V>
__device__ __forceinline__ void hsum(const T (&row)[V + 2], T (&h)[V]) {
    const T left = __shfl_up_sync(0xffffffffu, row[V], 1);
    const T right = __shfl_down_sync(0xffffffffu, row[1], 1);
#pragma unroll
    for (int v = 0; v < V; v += 2) {
        const T m = row[1 + v] + row[2 + v];
        h[v] = (v == 0 ? left : row[v]) + m;
        h[v + 1] = m + (v + 2 == V ? right : row[3 + v]);
    }
}

// MODE: 0 = FAST (FMA per tap), 1 = EXACT (multiply, then add, per tap),
// 2 = Q (exact, for kernels whose taps all carry one weight w, e.g. the
// reference's Box-2D9P / Box-2D25P): the level windows hold q = w*v, the
// product every tap of every output reading v computes — rounded once, shared
// by all of them, so each update is a chain of adds and the next level's q is
// one multiply per produced value.  Bitwise equal to EXACT.
template <typename T, int R, bool BOX, int K, int V, int MODE>
__global__ void __launch_bounds__(32 * kWarpsPerBlock) stream2d_kernel(
    const T* __restrict__ in, T* __restrict__ out, const __grid_constant__ S2Args<T> a) {
    constexpr bool EXACT = MODE == 1 || MODE == 2;
    constexpr bool QS = MODE == 2;
    // MODE 3 = SEP (FAST, uniform-weight 9-point box): the windows hold each
    // row's raw values and its horizontal 3-sums h; an update is
    // w * ((h[x-1] + h[x]) + h[x+1]): 2 adds + 1 multiply, plus 1.5 adds per
    // produced value for its h, instead of 9 adds (Q) — within 1e-12.
    constexpr bool SEP = MODE == 3;
    static_assert(!SEP || (BOX && R == 1), "SEP serves the 9-point box");
    constexpr int P = 2 * R + 1;  // ring depth per level
    constexpr int W = V + 2 * R;  // values per ring row incl. lane halo
    const int lane = threadIdx.x & 31;
    const int64_t gw = blockIdx.x * (int64_t)kWarpsPerBlock + (threadIdx.x >> 5);
    if (gw >= a.total_warps) return;
    const int64_t strip = gw % a.nstrips;
    const int64_t chunk = gw / a.nstrips;
    const int64_t rb = a.row_lo + chunk * a.chunk;
    const int64_t re = min(rb + a.chunk, a.row_hi);
    const int64_t ob = strip * a.wout;                 // first output column
    const int64_t oe = min(ob + a.wout, a.cols);       // output column end
    const int64_t c0 = ob - a.hl + (int64_t)lane * V;  // this lane's first column
    const bool col_alloc = c0 >= a.col_lo && c0 + V <= a.col_hi;

    // Per-value column masks (constant down the strip).
    bool cint[V], cout[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        cint[v] = c0 + v >= 0 && c0 + v < a.cols;
        cout[v] = c0 + v >= ob && c0 + v < oe;
    }
    bool all_out = true;
#pragma unroll
    for (int v = 0; v < V; ++v) all_out &= cout[v];

    T win[K][P][W];  // ring of rows per level (level K is stored, not kept)
    T hwin[SEP ? K : 1][P][V];  // SEP: horizontal 3-sums of the window rows
    // staging ring of level-0 rows: kDepth + 1 slots, row t in slot
    // (t - t_start) % (kDepth + 1); a slot is refilled one step after it was
    // read, so a lane never overwrites data it has not consumed
    __shared__ __align__(16) uint4 stage[kWarpsPerBlock][kDepth + 1][32];
    uint4* my_stage = &stage[threadIdx.x >> 5][0][lane];

    // Level l produces row t - l*S at step t.  S = R (EXACT/FAST): level l
    // reads the row level l-1 produced in the same step.  S = R+1 (Q mode,
    // whose updates are pure add chains and latency-bound): every row a
    // level reads was produced in an earlier step, so the K levels of a step
    // are independent chains (levels run in descending order, level 0 last).
    constexpr bool SKEW = (QS || SEP) && R == 1;  // (the 25-point box measured slower skewed)
    constexpr int S = SKEW ? R + 1 : R;
    const int64_t t_start = rb - (int64_t)K * R;  // first level-0 row of the cone
    const int64_t t_end = re + (int64_t)K * S;    // exclusive: level K stores row re-1
    const int64_t cone_end = re + (int64_t)K * R; // level-0 rows [t_start, cone_end)
    const T* base_in = in + a.origin + c0;
    T* base_out = out + a.origin + c0;
    // output row of the current step (level K produces row x = t - K*S),
    // advanced by one row per step: no 64-bit row multiply per store
    T* orow = base_out + (t_start - (int64_t)K * S) * a.pitch;

    // Fetchable level-0 rows: allocated ([-hrow, rows+hrow)) and inside the
    // cone (< cone_end), for lanes whose columns are allocated; one unsigned
    // compare per fetch.  Rows advance by one per step: incremental pointer
    // and ring slots.
    const int64_t ok_lo = -a.hrow;
    const uint64_t ok_span = col_alloc ? (uint64_t)(min(a.rows + a.hrow, cone_end) - ok_lo) : 0;
    int64_t fr = t_start;  // next row to fetch
    const T* fsrc = base_in + t_start * a.pitch;
    int rd = 0, wr = 0;    // staging slots to read / fill next
    auto fetch = [&]() {
        const bool ok = (uint64_t)(fr - ok_lo) < ok_span;
        cp_async16(my_stage + wr * 32, ok ? (const void*)fsrc : (const void*)in, ok);
        cp_async_commit();
        wr = wr == kDepth ? 0 : wr + 1;
        ++fr;
        fsrc += a.pitch;
    };
    for (int s = 0; s < kDepth; ++s) fetch();

    bool mine = true;
#pragma unroll
    for (int v = 0; v < V; ++v) mine &= cint[v];
    const bool warp_int = __all_sync(0xffffffffu, mine);  // no boundary column in the strip

    // Level 0 takes row t from the staging ring into window slot ph.
    auto level0 = [&](auto PHc) {
        constexpr int ph = decltype(PHc)::value;
        cp_async_wait<kDepth - 1>();  // row t (the oldest pending group) has landed
        const uint4 raw = my_stage[rd * 32];
        rd = rd == kDepth ? 0 : rd + 1;
        const T* rv = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int v = 0; v < V; ++v) win[0][ph][R + v] = QS ? mul_rn(a.w[0], rv[v]) : rv[v];
        fetch();  // row t + kDepth, into the slot row t-1 vacated
        if constexpr (SEP) hsum<T, V>(win[0][ph], hwin[0][ph]);
        else if constexpr (BOX) exchange<T, V, R>(win[0][ph]);
    };

    // One row step: level 0 takes row t, level l produces row t - l*S.
    // SEL = false is the select-free instantiation for steps where every
    // produced row and every column of the warp is interior.
    auto step = [&](auto PHc, auto SELc, int64_t t) {
        constexpr int ph = decltype(PHc)::value;
        constexpr bool SEL = decltype(SELc)::value;
        if constexpr (!SKEW) level0(PHc);
#pragma unroll
        for (int li = 0; li < K; ++li) {
            const int l = SKEW ? K - li : 1 + li;
            const int64_t x = t - (int64_t)l * S;
            const int sx = ((ph - l * S) % P + P) % P;  // slot of row x (static)
            // Star taps read lane-halo columns of the centre row only:
            // exchange it at use, so the halos of the other rows never
            // occupy registers.  Box rows carry halos from production.
            if constexpr (!BOX) exchange<T, V, R>(win[l - 1][sx]);
            T res[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if constexpr (SEP) {
                    const int sm = (sx + P - 1) % P, sp = (sx + 1) % P;
                    T nv = mul_rn(a.w[0], (hwin[l - 1][sm][v] + hwin[l - 1][sx][v]) + hwin[l - 1][sp][v]);
                    if constexpr (SEL) {
                        const bool rint = x >= 0 && x < a.rows;
                        if (l < K) nv = (rint && cint[v]) ? nv : win[l - 1][sx][R + v];
                    }
                    res[v] = nv;
                    continue;
                }
                T acc = T(0);
                int tap = 0;
#pragma unroll
                for (int dr = -R; dr <= R; ++dr) {
                    const int sr = ((sx + dr) % P + P) % P;
#pragma unroll
                    for (int dc = -R; dc <= R; ++dc) {
                        if (has_tap<R, BOX>(dr, dc)) {
                            const T xv = win[l - 1][sr][R + v + dc];
                            if constexpr (QS)
                                acc = tap == 0 ? xv : add_rn(acc, xv);
                            else
                                acc = tap == 0 ? lead(a.w[0], xv) : madd<EXACT>(acc, a.w[tap], xv);
                            ++tap;
                        }
                    }
                }
                // level K only stores interior cells: no Dirichlet select
                T nv = acc;
                if (l < K && QS) nv = mul_rn(a.w[0], acc);  // the next level's q
                if constexpr (SEL) {
                    const bool rint = x >= 0 && x < a.rows;
                    if (l < K) nv = (rint && cint[v]) ? nv : win[l - 1][sx][R + v];
                }
                res[v] = nv;
            }
            if (l < K) {
#pragma unroll
                for (int v = 0; v < V; ++v) win[l][sx][R + v] = res[v];
                if constexpr (SEP) hsum<T, V>(win[l][sx], hwin[l][sx]);
                else if constexpr (BOX) exchange<T, V, R>(win[l][sx]);
            } else if (x >= rb && x < re) {
#pragma unroll
                for (int v = 0; v < V; ++v) res[v] = fix_zero<EXACT>(res[v]);
                T* dst = orow;
                store_vals<T, V>(dst, res, cout, all_out);
                if (a.mirror) store_vals<T, V>(a.mirror + (dst - out) + a.mshift, res, cout, all_out);
            }
        }
        if constexpr (SKEW) level0(PHc);  // row t replaces row t-P, which level 1 has just read
        orow += a.pitch;
    };

    for (int64_t tb = t_start; tb < t_end; tb += P) {
        static_for<0, P>([&](auto PHc) {
            const int64_t t = tb + decltype(PHc)::value;
            if (t < t_end) {
                if (warp_int && t - (int64_t)K * S >= 0 && t - S < a.rows)
                    step(PHc, std::false_type{}, t);
                else
                    step(PHc, std::true_type{}, t);
            }
        });
    }
}

struct Shape {
    int R;
    bool box;
};

bool classify(const TapSet& t, Shape* s) {
    if (t.dims != 2) return false;
    if (t.shape == TSR_STAR && (t.radius == 1 || t.radius == 2)) {
        *s = {t.radius, false};
        return true;
    }
    if (t.shape == TSR_BOX && (t.radius == 1 || t.radius == 2)) {
        *s = {t.radius, true};
        return true;
    }
    return false;
}

constexpr int kMaxK = 8;
constexpr int kMaxKBox2 = 2;  // 25-point box: five 6-wide rows per level in registers (k=3 spills)

// Default fused depths from a k sweep over 4096^2, 9600^2 and 16384^2 fp64
// (tools/probe_2d_k.py): k = 4 for the 5-point star and the 9-point box
// (EXACT / Q mode: 919 at 16384^2 against 753-839 for k = 5..8), k = 3 for the
// radius-2 star (its windows are 5 rows deep: 489 / 608 GS/s exact / fast at
// 16384^2 against 468 / 584 at k = 4), k = 1 for the 25-point box (10000^2:
// 309 against 243 GS/s at k = 2, tools/probe/box25.py), and k = 5 for the
// 9-point box in FAST (separable sums, fewer registers per level: 1156
// against 1076 at 9600^2).
bool supports(const Geo& g, const TapSet& t, int* max_fused, int* default_fused) {
    Shape s;
    if (!classify(t, &s)) return false;
    const bool box2 = s.box && s.R == 2;
    *max_fused = box2 ? kMaxKBox2 : kMaxK;
    *default_fused = box2 ? 1 : (!s.box && s.R == 2) ? 3 : 4;
    return true;
}

int fast_default(const Geo& g, const TapSet& t) {
    Shape s;
    int maxk = 1, defk = 1;
    if (!supports(g, t, &maxk, &defk)) return 1;
    classify(t, &s);
    return s.box && s.R == 1 && uniform_weights(t) ? 5 : defk;
}

template <typename T, int R, bool BOX, int K, int V>
Status launch_k(const LaunchCtx& c, const void* in, void* out) {
    const Geo& g = *c.g;
    S2Args<T> a;
    a.rows = g.n[1];
    a.cols = g.n[2];
    a.hrow = g.h[1];
    a.pitch = g.pitch[1];
    a.origin = g.origin;
    a.mirror = static_cast<T*>(c.mirror);
    a.mshift = c.mirror_shift;
    a.col_lo = -g.off2;
    a.col_hi = g.pitch[1] - g.off2;
    constexpr int vec = 16 / sizeof(T);
    a.hl = ((int64_t)R * K + vec - 1) / vec * vec;
    a.wout = (32 * V - a.hl - (int64_t)R * K) / vec * vec;
    if (a.wout <= 0) return Status::Err(TSR_EUNSUPPORTED, "stream2d: strip too narrow for K");
    a.nstrips = (a.cols + a.wout - 1) / a.wout;
    // Aim for ~16 resident warps per SM, chunks of >= 16*K*R rows.
    const int64_t target = 148 * 24;
    int64_t nchunks = std::max<int64_t>(1, target / a.nstrips);
    a.row_lo = c.range_lo();
    a.row_hi = c.range_hi();
    if (a.row_hi <= a.row_lo) return Status::Ok();
    const int64_t span = a.row_hi - a.row_lo;
    // chunks of >= 16*K*R rows keep the 2*K*R-row wavefront fill small; a
    // grid too small to give every SM a few warps that way (latency-bound)
    // goes down to 2*K*R-row chunks
    int64_t min_chunk = 16 * K * R;
    if (a.nstrips * ((span + min_chunk - 1) / min_chunk) < 148 * 8) min_chunk = 2 * K * R;
    a.chunk = std::max<int64_t>(min_chunk, (span + nchunks - 1) / nchunks);
    nchunks = (span + a.chunk - 1) / a.chunk;
    a.total_warps = nchunks * a.nstrips;
    for (int t = 0; t < c.taps->ntaps; ++t) a.w[t] = static_cast<T>(c.taps->w[t]);
    const unsigned blocks =
        static_cast<unsigned>((a.total_warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
    if constexpr (BOX) {
        if (uniform_weights(*c.taps)) {  // Q mode (exact), separable sums in FAST (R = 1)
            if constexpr (R == 1) {
                if (!c.exact) {
                    stream2d_kernel<T, R, BOX, K, V, 3>
                        <<<blocks, 32 * kWarpsPerBlock, 0, c.stream>>>(
                            static_cast<const T*>(in), static_cast<T*>(out), a);
                    TSR_CUDA_TRY(cudaGetLastError());
                    return Status::Ok();
                }
            }
            stream2d_kernel<T, R, BOX, K, V, 2><<<blocks, 32 * kWarpsPerBlock, 0, c.stream>>>(
                static_cast<const T*>(in), static_cast<T*>(out), a);
            TSR_CUDA_TRY(cudaGetLastError());
            return Status::Ok();
        }
    }
    if (c.exact)
        stream2d_kernel<T, R, BOX, K, V, 1><<<blocks, 32 * kWarpsPerBlock, 0, c.stream>>>(
            static_cast<const T*>(in), static_cast<T*>(out), a);
    else
        stream2d_kernel<T, R, BOX, K, V, 0><<<blocks, 32 * kWarpsPerBlock, 0, c.stream>>>(
            static_cast<const T*>(in), static_cast<T*>(out), a);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

template <typename T, int R, bool BOX>
Status launch_shape(const LaunchCtx& c, const void* in, void* out, int k) {
    constexpr int V = 16 / sizeof(T);  // one 16-byte vector per lane per row
    switch (k) {
        case 1: return launch_k<T, R, BOX, 1, V>(c, in, out);
        case 2: return launch_k<T, R, BOX, 2, V>(c, in, out);
        case 3: return launch_k<T, R, BOX, 3, V>(c, in, out);
        case 4: return launch_k<T, R, BOX, 4, V>(c, in, out);
        case 5: return launch_k<T, R, BOX, 5, V>(c, in, out);
        case 6: return launch_k<T, R, BOX, 6, V>(c, in, out);
        case 7: return launch_k<T, R, BOX, 7, V>(c, in, out);
        case 8: return launch_k<T, R, BOX, 8, V>(c, in, out);
        default: return Status::Err(TSR_EUNSUPPORTED, "stream2d: fused steps must be 1..8");
    }
}

template <typename T>
Status launch_t(const LaunchCtx& c, const void* in, void* out, int k) {
    Shape s;
    classify(*c.taps, &s);
    if (s.box && s.R == 2) {
        constexpr int V = 16 / sizeof(T);
        switch (k) {
            case 1: return launch_k<T, 2, true, 1, V>(c, in, out);
            case 2: return launch_k<T, 2, true, 2, V>(c, in, out);
            default: return Status::Err(TSR_EUNSUPPORTED, "stream2d: 25-point box fuses 1..2");
        }
    }
    if (s.box) return launch_shape<T, 1, true>(c, in, out, k);
    if (s.R == 1) return launch_shape<T, 1, false>(c, in, out, k);
    return launch_shape<T, 2, false>(c, in, out, k);
}

Status run(const LaunchCtx& c, const void* in, void* out, int k) {
    if (c.g->dtype == TSR_F64) return launch_t<double>(c, in, out, k);
    return launch_t<float>(c, in, out, k);
}

}  // namespace

extern const Engine kStream2dEngine = {"stream2d_regtile", supports, run, fast_default};

}  // namespace tsr
