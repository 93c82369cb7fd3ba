// box3d.cu — 3-D radius-1 box (27-point) sweep, 2.5-D streaming with
// per-plane partial sums.
//
// The oracle sums the 27 taps in lexicographic (di, dj, dk) order
// (proj/src/kernel.cpp:19-43, naive.hpp:76-78): all nine taps of plane p-1,
// then plane p, then plane p+1.  So output plane p's accumulator can be
// advanced plane by plane as a0 streams past: when plane q sits in shared
// memory, every thread reads its (4+2) x (4+2) neighbourhood once and
//   * finishes the accumulator of output q-1 (taps di=+1) and stores it,
//   * continues output q (taps di=0),
//   * starts output q+1 (taps di=-1),
// each accumulator seeing its taps in exactly the oracle's order.  One plane
// read serves three outputs: 2.25 shared-memory loads per output instead of
// 27.  Planes arrive by TMA (cp.async.bulk.tensor.3d) into a 4-stage
// mbarrier ring.  FAST mode is one FMA per tap; EXACT a separately rounded
// multiply and add (bitwise naive_run).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tma.cuh"

namespace tsr {

namespace {

constexpr int OX = 64;  // output tile width  (a2)
constexpr int OY = 32;  // output tile height (a1)
constexpr int VX = 4;   // outputs per thread along a2
constexpr int VY = 4;   // outputs per thread along a1
constexpr int NLX = OX / VX;   // 16
constexpr int NLY = OY / VY;   // 8
constexpr int NT = NLX * NLY;  // 128 threads
constexpr int STAGES = 4;
constexpr int BY = OY + 2;

template <typename T>
constexpr int PAD = 16 / (int)sizeof(T);  // 16-B aligned box start / rows
template <typename T>
constexpr int BXW = OX + 3 * PAD<T>;  // k=2 box: one spare vector so rows 4 apart
                                      // (the two half-warps) fall in other banks
template <typename T>
constexpr int slot_bytes() {
    return (BXW<T> * BY * (int)sizeof(T) + 127) / 128 * 128;
}
// The K = 1 kernel uses a wider tile: the TMA box of a 64-column fp32 tile
// touches 10 DRAM sectors per row for 8 useful ones (the 1-cell halo plus the
// 16-B aligned start add a sector each side), 128 columns make it 18 for 16.
// fp64 keeps 64 columns (512 B rows, 4 CTAs per SM).
template <typename T>
constexpr int OX1 = sizeof(T) == 4 ? 128 : 64;
template <typename T>
constexpr int NT1 = OX1<T> / VX * NLY;  // 256 / 128 threads
template <typename T>
constexpr int BXW1 = OX1<T> + 2 * PAD<T>;
template <typename T>
constexpr int slot1_bytes() {
    return (BXW1<T> * BY * (int)sizeof(T) + 127) / 128 * 128;
}
template <typename T>
constexpr int smem_bytes() {
    return STAGES * slot1_bytes<T>() + STAGES * 8;
}

template <typename T>
struct BoxArgs {
    int n0, n1, n2;
    int tiles_x, tiles_y, chunk;
    int lo0, hi0;  // output planes [lo0, hi0) of a0
    int h0, h1, off2;
    long long pitch0, pitch1, origin;
    T* mirror;  // LaunchCtx::mirror (fused halo exchange), or nullptr
    long long mshift;
    T w[27];
};

template <typename T, int V>
struct VecT;
template <>
struct VecT<float, 4> {
    using type = float4;
};
template <>
struct VecT<double, 2> {
    using type = double2;
};

// One row of a thread's (VX + 2)-wide neighbourhood: its VX cells by vector
// loads, the two outer cells from the neighbouring lanes by shuffle (W lanes
// span one row of the region), and only the row's first / last lane takes
// the region edge cell from shared memory — a broadcast load every lane
// issues (one address per row), so no 16-B-strided scalar loads and no bank
// conflicts.  `row` points at the thread's first cell, x its region column.
template <typename T, int W>
__device__ __forceinline__ void load_row(const T* row, int x, int lx, T (&nbr)[VX + 2]) {
    using V4 = typename VecT<T, 16 / sizeof(T)>::type;
    constexpr int NV = 16 / sizeof(T);
#pragma unroll
    for (int v = 0; v < VX; v += NV) {
        const V4 vv = *reinterpret_cast<const V4*>(row + v);
        const T* e = reinterpret_cast<const T*>(&vv);
#pragma unroll
        for (int u = 0; u < NV; ++u) nbr[1 + v + u] = e[u];
    }
    const T left = __shfl_up_sync(0xffffffffu, nbr[VX], 1, W);
    const T right = __shfl_down_sync(0xffffffffu, nbr[1], 1, W);
    const T* row0 = row - x;  // region column 0 of this row
    const T el = row0[-1], er = row0[W * VX];
    nbr[0] = lx == 0 ? el : left;
    nbr[VX + 1] = lx == W - 1 ? er : right;
}

// Nine taps of one plane offset applied to the neighbourhood nb (rows y-1..y+VY,
// cols x-1..x+VX) for every output of the thread's 4x4 tile.
// Q: nb holds q = w*v (uniform-weight kernel, see stream2d.cu): every tap is
// an add of the shared rounded product, bitwise the EXACT sum.
template <bool EXACT, bool START, typename T, bool Q = false>
__device__ __forceinline__ void apply9(const T* __restrict__ w, const T (&nb)[VY + 2][VX + 2],
                                       T (&acc)[VY][VX]) {
#pragma unroll
    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
        for (int cx = 0; cx < VX; ++cx) {
            T s = acc[cy][cx];
#pragma unroll
            for (int dj = 0; dj < 3; ++dj)
#pragma unroll
                for (int dk = 0; dk < 3; ++dk) {
                    const T v = nb[cy + dj][cx + dk];
                    if (START && dj == 0 && dk == 0)
                        s = Q ? add_rn(T(0), v) : first<EXACT>(w[0], v);
                    else
                        s = Q ? add_rn(s, v) : madd<EXACT>(s, w[dj * 3 + dk], v);
                }
            acc[cy][cx] = s;
        }
}

// SEP (FAST mode, uniform weights): the 27-point box sum factorises into
// row sums along a2, then column sums along a1 (this function: the 2-D
// 9-point sum of one plane for every output of the thread's 4x4 tile, 5
// adds per output with the shared pair sums), then the three plane sums
// along a0, times the one weight: 8 operations per output instead of 27
// (Q) or 27 FMAs (FAST), within the 1e-5 fp32 / 1e-12 fp64 tolerance of the
// oracle's order (only the rounding of the reassociated sum differs).
template <typename T>
__device__ __forceinline__ void plane_sum9(const T (&nb)[VY + 2][VX + 2], T (&s)[VY][VX]) {
    static_assert(VX == 4, "pair sums assume four outputs per row");
    T r[VY + 2][VX];
#pragma unroll
    for (int q = 0; q < VY + 2; ++q) {
        const T p0 = nb[q][1] + nb[q][2], p2 = nb[q][3] + nb[q][4];
        r[q][0] = nb[q][0] + p0;
        r[q][1] = p0 + nb[q][3];
        r[q][2] = nb[q][2] + p2;
        r[q][3] = p2 + nb[q][5];
    }
#pragma unroll
    for (int cx = 0; cx < VX; ++cx) {
#pragma unroll
        for (int cy = 0; cy < VY; cy += 2) {
            const T m = r[cy + 1][cx] + r[cy + 2][cx];  // shared by rows cy and cy+1
            s[cy][cx] = r[cy][cx] + m;
            s[cy + 1][cx] = m + r[cy + 3][cx];
        }
    }
}

// MODE: 0 FAST, 1 EXACT, 2 Q (uniform weights: shared products, exact),
// 3 SEP (uniform weights, FAST: separable sums)
template <typename T, int MODE>
__global__ void __launch_bounds__(NT1<T>) box3d_kernel(T* __restrict__ out,
                                                   const __grid_constant__ CUtensorMap tmap,
                                                   const __grid_constant__ BoxArgs<T> a) {
    constexpr bool EXACT = MODE == 1 || MODE == 2, Q = MODE == 2, SEP = MODE == 3;
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int SLOT = slot1_bytes<T>() / (int)sizeof(T);
    constexpr int BX = BXW1<T>, PL = PAD<T>;
    constexpr int NLX1 = OX1<T> / VX;
    T* ring = reinterpret_cast<T*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + STAGES * slot1_bytes<T>());

    const int tid = threadIdx.x;
    const int lx = tid % NLX1, ly = tid / NLX1;
    const int tile = blockIdx.x;
    const int bx = tile % a.tiles_x;
    const int by = (tile / a.tiles_x) % a.tiles_y;
    const int bz = tile / (a.tiles_x * a.tiles_y);
    const int gx = bx * OX1<T>, gy = by * OY;  // interior coords of the tile origin
    const int i0 = a.lo0 + bz * a.chunk;
    const int i1 = min(i0 + a.chunk, a.hi0);
    // planes i0-1 .. i1 feed outputs i0 .. i1-1
    const int t_begin = i0 - 1, niter = i1 - i0 + 2;
    const int x = VX * lx, y = VY * ly;

    bool ok[VY][VX];
#pragma unroll
    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
        for (int cx = 0; cx < VX; ++cx)
            ok[cy][cx] = gy + y + cy < a.n1 && gx + x + cx < a.n2;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmap);
    }
    __syncthreads();
    constexpr unsigned kBoxBytes = BX * BY * sizeof(T);
    const int c0 = a.off2 + gx - PL, c1 = a.h1 + gy - 1;
    if (tid == 0)
        for (int s = 0; s < STAGES && s < niter; ++s) {
            mbar_expect_tx(&bar[s], kBoxBytes);
            tma_load_3d(ring + s * SLOT, &tmap, &bar[s], c0, c1, a.h0 + t_begin + s);
        }

    T accA[VY][VX], accB[VY][VX];  // outputs q+1 (started) and q (in progress)
#pragma unroll
    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
        for (int cx = 0; cx < VX; ++cx) accA[cy][cx] = accB[cy][cx] = T(0);

    using V4 = typename VecT<T, 16 / sizeof(T)>::type;
    constexpr int NV = 16 / sizeof(T);
    // output plane q-1 of step it, advanced by one plane per step (no 64-bit
    // plane multiply per store)
    T* orow = out + (a.origin + (long long)(t_begin - 1) * a.pitch0 +
                     (long long)(gy + y) * a.pitch1 + (gx + x));
    for (int it = 0; it < niter; ++it) {
        const int q = t_begin + it;  // plane in shared memory
        const int slot = it % STAGES;
        mbar_wait(&bar[slot], (it / STAGES) & 1);
        const T* P = ring + slot * SLOT;
        // (direct edge loads here: the shuffled rows of load_row measured 4%
        // slower in this single-level, HBM-bound kernel)
        T nb[VY + 2][VX + 2];
#pragma unroll
        for (int r = 0; r < VY + 2; ++r) {
            const T* row = P + (y + r) * BX + PL + x;  // region col x <-> ring col x+PL
            nb[r][0] = row[-1];
#pragma unroll
            for (int v = 0; v < VX; v += NV) {
                const V4 vv = *reinterpret_cast<const V4*>(row + v);
                const T* e = reinterpret_cast<const T*>(&vv);
#pragma unroll
                for (int u = 0; u < NV; ++u) nb[r][1 + v + u] = e[u];
            }
            nb[r][VX + 1] = row[VX];
        }
        if constexpr (Q) {
#pragma unroll
            for (int r = 0; r < VY + 2; ++r)
#pragma unroll
                for (int c = 0; c < VX + 2; ++c) nb[r][c] = mul_rn(a.w[0], nb[r][c]);
        }
        __syncthreads();  // every thread has its neighbourhood: slot may be refilled
        if (tid == 0 && it + STAGES < niter) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[slot], kBoxBytes);
            tma_load_3d(ring + slot * SLOT, &tmap, &bar[slot], c0, c1,
                        a.h0 + t_begin + it + STAGES);
        }
        T ps[VY][VX];  // SEP: this plane's 9-point sums
        if constexpr (SEP) {
            plane_sum9(nb, ps);
#pragma unroll
            for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                for (int cx = 0; cx < VX; ++cx) accB[cy][cx] = mul_rn(a.w[0], accB[cy][cx] + ps[cy][cx]);
        } else {
            // finish output q-1 (di = +1 taps)
            apply9<EXACT, false, T, Q>(a.w + 18, nb, accB);
        }
        const int po = q - 1;
        if (it >= 2 && po < i1) {
            T* o = orow;  // plane po
#pragma unroll
            for (int cy = 0; cy < VY; ++cy) {
                store_row<T, VX>(o + cy * a.pitch1, accB[cy], ok[cy]);
                if (a.mirror)
                    store_row<T, VX>(a.mirror + (o - out) + a.mshift + cy * a.pitch1, accB[cy], ok[cy]);
            }
        }
        orow += a.pitch0;
        // output q continues (di = 0), output q+1 starts (di = -1)
        if constexpr (SEP) {
#pragma unroll
            for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                for (int cx = 0; cx < VX; ++cx) {
                    accB[cy][cx] = accA[cy][cx] + ps[cy][cx];
                    accA[cy][cx] = ps[cy][cx];
                }
        } else {
            apply9<EXACT, false, T, Q>(a.w + 9, nb, accA);
#pragma unroll
            for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                for (int cx = 0; cx < VX; ++cx) accB[cy][cx] = accA[cy][cx];
            apply9<EXACT, true, T, Q>(a.w, nb, accA);
        }
    }
}

// ---------------------------------------------------------------------------
// K = 2: two time steps per HBM pass.  Level 1 is computed with the same
// plane-partial sums on the whole 64 x 32 tile (the level-0 box carries one
// extra cell of halo), written to a triple-buffered SMEM plane, and level 2
// runs the plane-partial sums over those SMEM planes for the inner 62 x 30
// cells.  One __syncthreads per plane: after the level-1 plane is published.
// Dirichlet: level-1 cells outside the interior keep their level-0 value, so
// level 2 reads exactly what a second apply_box sweep would.
constexpr int L1X = OX, L1Y = OY;  // level-1 region = the 64 x 32 tile
constexpr int BH = L1Y + 2;        // SMEM level-1 plane rows incl. 1-row border
constexpr int NB = 2;              // level-1 plane buffers
// Vector alignment: the region's left margin is one 16-B vector (so TMA box
// starts stay 16-B aligned) and SMEM rows put region column x at x + PAD.
template <typename T>
constexpr int HX2 = PAD<T>;                                          // left margin
template <typename T>
constexpr int TX2 = (L1X - HX2<T> - 1) / PAD<T> * PAD<T>;            // output width
constexpr int TY2 = L1Y - 2;                                         // output height
template <typename T>
constexpr int BWP = L1X + 3 * PAD<T>;  // SMEM row pitch (+1 vector: conflict-free edges)

template <typename T>
constexpr int b_bytes() {
    return (BWP<T> * BH * (int)sizeof(T) + 127) / 128 * 128;
}
template <typename T>
constexpr int smem2_bytes() {
    return STAGES * slot_bytes<T>() + NB * b_bytes<T>() + STAGES * 8;
}

template <typename T, int MODE>
__global__ void __launch_bounds__(NT) box3d_tb2_kernel(T* __restrict__ out,
                                                      const __grid_constant__ CUtensorMap tmap,
                                                      const __grid_constant__ BoxArgs<T> a) {
    constexpr bool EXACT = MODE != 0, Q = MODE == 2;
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int SLOT = slot_bytes<T>() / (int)sizeof(T);
    constexpr int BE = b_bytes<T>() / (int)sizeof(T);
    constexpr int BX = BXW<T>, PL = PAD<T>;
    T* ring = reinterpret_cast<T*>(smem);
    T* buf = reinterpret_cast<T*>(smem + STAGES * slot_bytes<T>());
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + STAGES * slot_bytes<T>() + NB * b_bytes<T>());

    const int tid = threadIdx.x;
    const int lx = tid % NLX, ly = tid / NLX;
    const int tile = blockIdx.x;
    const int bx = tile % a.tiles_x;
    const int by = (tile / a.tiles_x) % a.tiles_y;
    const int bz = tile / (a.tiles_x * a.tiles_y);
    constexpr int HX = HX2<T>, TX = TX2<T>, BW = BWP<T>;
    const int gx = bx * TX - HX, gy = by * TY2 - 1;  // global coords of L1 cell (0, 0)
    const int i0 = a.lo0 + bz * a.chunk;
    const int i1 = min(i0 + a.chunk, a.hi0);
    // level-0 planes i0-2 .. i1+1 feed level-2 outputs i0 .. i1-1
    const int t_begin = i0 - 2, niter = i1 - i0 + 4;
    const int x = VX * lx, y = VY * ly;

    bool cint[VY][VX], cout[VY][VX];
#pragma unroll
    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
        for (int cx = 0; cx < VX; ++cx) {
            const int ga1 = gy + y + cy, ga2 = gx + x + cx;
            cint[cy][cx] = ga1 >= 0 && ga1 < a.n1 && ga2 >= 0 && ga2 < a.n2;
            cout[cy][cx] = cint[cy][cx] && y + cy >= 1 && y + cy < L1Y - 1 && x + cx >= HX &&
                           x + cx < HX + TX;
        }
    bool mine = true;
#pragma unroll
    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
        for (int cx = 0; cx < VX; ++cx) mine &= cint[cy][cx];
    const bool warp_int = __all_sync(0xffffffffu, mine);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmap);
    }
    __syncthreads();
    constexpr unsigned kBoxBytes = BX * BY * sizeof(T);
    // level-0 box: L1 region plus one cell, 16-B aligned start
    const int c0 = a.off2 + gx - PL, c1 = a.h1 + gy - 1;
    if (tid == 0)
        for (int s = 0; s < STAGES && s < niter; ++s) {
            mbar_expect_tx(&bar[s], kBoxBytes);
            tma_load_3d(ring + s * SLOT, &tmap, &bar[s], c0, c1, a.h0 + t_begin + s);
        }

    T a1A[VY][VX], a1B[VY][VX];  // level 1: outputs q+1 (started), q (in progress)
    T a2A[VY][VX], a2B[VY][VX];  // level 2: outputs q (started), q-1 (in progress)
    T keep0[VY][VX];             // level-0 centre of plane q-1 (frozen level-1 cells)
#pragma unroll
    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
        for (int cx = 0; cx < VX; ++cx)
            a1A[cy][cx] = a1B[cy][cx] = a2A[cy][cx] = a2B[cy][cx] = keep0[cy][cx] = T(0);

    using V4 = typename VecT<T, 16 / sizeof(T)>::type;
    constexpr int NV = 16 / sizeof(T);
    auto read_nb = [&](const T* rowbase, int pitch, T(&nb)[VY + 2][VX + 2]) {
#pragma unroll
        for (int r = 0; r < VY + 2; ++r) load_row<T, NLX>(rowbase + (y + r) * pitch, x, lx, nb[r]);
    };

    // output plane q-2 of step it, advanced by one plane per step
    T* orow2 = out + (a.origin + (long long)(t_begin - 2) * a.pitch0 +
                      (long long)(gy + y) * a.pitch1 + (gx + x));
    for (int it = 0; it < niter; ++it, orow2 += a.pitch0) {
        const int q = t_begin + it;  // level-0 plane in the ring
        const int slot = it % STAGES;
        mbar_wait(&bar[slot], (it / STAGES) & 1);
        const bool sel = !(warp_int && q - 2 >= 0 && q < a.n0);  // planes q-2..q
        T nb[VY + 2][VX + 2];
        read_nb(ring + slot * SLOT + PL + x, BX, nb);
        if constexpr (Q) {  // level 0 -> q; level-1 planes are published as q
#pragma unroll
            for (int r = 0; r < VY + 2; ++r)
#pragma unroll
                for (int c = 0; c < VX + 2; ++c) nb[r][c] = mul_rn(a.w[0], nb[r][c]);
        }
        // level 1: finish q-1, continue q, start q+1
        apply9<EXACT, false, T, Q>(a.w + 18, nb, a1B);
        T l1[VY][VX];
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int cx = 0; cx < VX; ++cx) l1[cy][cx] = Q ? mul_rn(a.w[0], a1B[cy][cx]) : a1B[cy][cx];
        if (sel) {  // warp-uniform: boundary warps and a0-boundary planes only
            const bool pint = q - 1 >= 0 && q - 1 < a.n0;
#pragma unroll
            for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                for (int cx = 0; cx < VX; ++cx)
                    if (!(pint && cint[cy][cx])) l1[cy][cx] = keep0[cy][cx];
        }
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int cx = 0; cx < VX; ++cx) keep0[cy][cx] = nb[cy + 1][cx + 1];
        apply9<EXACT, false, T, Q>(a.w + 9, nb, a1A);
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int cx = 0; cx < VX; ++cx) a1B[cy][cx] = a1A[cy][cx];
        apply9<EXACT, true, T, Q>(a.w, nb, a1A);
        // publish level-1 plane q-1: cell (y, x) at row y+1, column x+PAD
        T* B = buf + (((q - 1) % NB + NB) % NB) * BE;
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int v = 0; v < VX; v += NV) {
                V4 vv;
                T* e = reinterpret_cast<T*>(&vv);
#pragma unroll
                for (int u = 0; u < NV; ++u) e[u] = l1[cy][v + u];
                *reinterpret_cast<V4*>(B + (y + cy + 1) * BW + x + PL + v) = vv;
            }
        __syncthreads();
        // every thread has read plane q: its slot takes plane q + STAGES
        if (tid == 0 && it + STAGES < niter) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[slot], kBoxBytes);
            tma_load_3d(ring + slot * SLOT, &tmap, &bar[slot], c0, c1,
                        a.h0 + t_begin + it + STAGES);
        }
        // level 2 on level-1 plane q-1: finish q-2, continue q-1, start q
        T nb2[VY + 2][VX + 2];
        read_nb(B + PL + x, BW, nb2);  // buffer rows y..y+VY+1 = region rows y-1..y+VY
        apply9<EXACT, false, T, Q>(a.w + 18, nb2, a2B);
        const int po = q - 2;
        if (it >= 4 && po < i1) {
            // stored cells are interior (cout implies cint): no Dirichlet select
            T* o = orow2;
#pragma unroll
            for (int cy = 0; cy < VY; ++cy) {
                T v[VX];
#pragma unroll
                for (int cx = 0; cx < VX; ++cx) v[cx] = fix_zero<EXACT>(a2B[cy][cx]);
                store_row<T, VX>(o + cy * a.pitch1, v, cout[cy]);
                if (a.mirror) store_row<T, VX>(a.mirror + (o - out) + a.mshift + cy * a.pitch1, v, cout[cy]);
            }
        }
        apply9<EXACT, false, T, Q>(a.w + 9, nb2, a2A);
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int cx = 0; cx < VX; ++cx) a2B[cy][cx] = a2A[cy][cx];
        apply9<EXACT, true, T, Q>(a.w, nb2, a2A);
    }
}

// ---------------------------------------------------------------------------
// k = KL levels in SEP mode (FAST, uniform weights), one __syncthreads per
// plane: level l consumes the level-(l-1) plane published in the PREVIOUS
// plane step (a lag of two planes per level, as tb3d's skew), so every read
// of a step sees data published before its barrier.  Level 1 reads the TMA
// ring; level l > 1 reads a two-slot SMEM plane of level l-1 (written at
// step s, read at s+1, rewritten at s+2 after the barrier).  Each level
// keeps the two open accumulators of the plane-sum recurrence (finish
// p-1, continue p, start p+1 per consumed plane) and the previous consumed
// centre for its Dirichlet cells.  Output plane of step it: q - (2KL - 1).
template <int KL, typename T>
constexpr int HXK = (KL - 1 + PAD<T> - 1) / PAD<T> * PAD<T>;  // left margin (>= KL-1, aligned)
template <int KL, typename T>
constexpr int TXK = (L1X - HXK<KL, T> - (KL - 1)) / PAD<T> * PAD<T>;  // output width
template <int KL>
constexpr int TYK = L1Y - 2 * (KL - 1);  // output height
template <int KL, typename T>
constexpr int smemk_bytes() {
    return STAGES * slot_bytes<T>() + (KL - 1) * NB * b_bytes<T>() + STAGES * 8;
}

template <typename T, int KL>
__global__ void __launch_bounds__(NT) box3d_tbk_sep_kernel(T* __restrict__ out,
                                                          const __grid_constant__ CUtensorMap tmap,
                                                          const __grid_constant__ BoxArgs<T> a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int SLOT = slot_bytes<T>() / (int)sizeof(T);
    constexpr int BE = b_bytes<T>() / (int)sizeof(T);
    constexpr int BX = BXW<T>, PL = PAD<T>, BW = BWP<T>;
    constexpr int HX = HXK<KL, T>, TX = TXK<KL, T>, TY = TYK<KL>;
    T* ring = reinterpret_cast<T*>(smem);
    T* buf = reinterpret_cast<T*>(smem + STAGES * slot_bytes<T>());
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + STAGES * slot_bytes<T>() +
                                                (KL - 1) * NB * b_bytes<T>());

    const int tid = threadIdx.x;
    const int lx = tid % NLX, ly = tid / NLX;
    const int tile = blockIdx.x;
    const int bx = tile % a.tiles_x;
    const int by = (tile / a.tiles_x) % a.tiles_y;
    const int bz = tile / (a.tiles_x * a.tiles_y);
    const int gx = bx * TX - HX, gy = by * TY - (KL - 1);  // global coords of region cell (0, 0)
    const int i0 = a.lo0 + bz * a.chunk;
    const int i1 = min(i0 + a.chunk, a.hi0);
    constexpr int LAG = 2 * KL - 1;  // output plane = ring plane - LAG
    const int t_begin = i0 - KL, niter = i1 - i0 + LAG + KL;
    const int x = VX * lx, y = VY * ly;

    bool cint[VY][VX], cout[VY][VX];
#pragma unroll
    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
        for (int cx = 0; cx < VX; ++cx) {
            const int ga1 = gy + y + cy, ga2 = gx + x + cx;
            cint[cy][cx] = ga1 >= 0 && ga1 < a.n1 && ga2 >= 0 && ga2 < a.n2;
            cout[cy][cx] = cint[cy][cx] && y + cy >= KL - 1 && y + cy < L1Y - (KL - 1) &&
                           x + cx >= HX && x + cx < HX + TX;
        }
    bool mine = true;
#pragma unroll
    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
        for (int cx = 0; cx < VX; ++cx) mine &= cint[cy][cx];
    const bool warp_int = __all_sync(0xffffffffu, mine);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmap);
    }
    __syncthreads();
    constexpr unsigned kBoxBytes = BX * BY * sizeof(T);
    const int c0 = a.off2 + gx - PL, c1 = a.h1 + gy - 1;
    // level-0 planes of the dependency cone are [i0-KL, i1+KL); the drain
    // steps re-load the last one, so a launch never reads outside its cone
    // (a slab's interior range runs while its ghost planes are written)
    const int last_plane = a.h0 + i1 + KL - 1;
    if (tid == 0)
        for (int s = 0; s < STAGES && s < niter; ++s) {
            mbar_expect_tx(&bar[s], kBoxBytes);
            tma_load_3d(ring + s * SLOT, &tmap, &bar[s], c0, c1, min(a.h0 + t_begin + s, last_plane));
        }

    T accA[KL][VY][VX], accB[KL][VY][VX];  // per level: outputs p+1 (started), p (open)
    T keep0[VY][VX];  // level-0 centre of the previous ring plane (Dirichlet cells of level 1)
#pragma unroll
    for (int l = 0; l < KL; ++l)
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int cx = 0; cx < VX; ++cx) accA[l][cy][cx] = accB[l][cy][cx] = T(0);
#pragma unroll
    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
        for (int cx = 0; cx < VX; ++cx) keep0[cy][cx] = T(0);
    const T w = a.w[0];
    using V4 = typename VecT<T, 16 / sizeof(T)>::type;
    constexpr int NV = 16 / sizeof(T);

    T* orow = out + (a.origin + (long long)(t_begin - LAG) * a.pitch0 +
                     (long long)(gy + y) * a.pitch1 + (gx + x));
    for (int it = 0; it < niter; ++it, orow += a.pitch0) {
        const int q = t_begin + it;  // level-0 plane in the ring
        const int slot = it % STAGES;
        mbar_wait(&bar[slot], (it / STAGES) & 1);
        // level l consumes the level-(l-1) plane c_l = q - 2(l-1) and
        // finishes output plane c_l - 1; levels in descending order so each
        // reads its source buffer before the level below republishes
#pragma unroll
        for (int l = KL; l >= 1; --l) {
            const int c = q - 2 * (l - 1);  // consumed level-(l-1) plane
            T nb[VY + 2][VX + 2];
            if (l == 1) {
#pragma unroll
                for (int r = 0; r < VY + 2; ++r)
                    load_row<T, NLX>(ring + slot * SLOT + PL + x + (y + r) * BX, x, lx, nb[r]);
            } else {
                const T* B = buf + ((l - 2) * NB + ((c % NB) + NB) % NB) * BE;
#pragma unroll
                for (int r = 0; r < VY + 2; ++r)
                    load_row<T, NLX>(B + PL + x + (y + r) * BW, x, lx, nb[r]);
            }
            T ps[VY][VX];
            plane_sum9(nb, ps);
            T v[VY][VX];  // level-l plane c-1
#pragma unroll
            for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                for (int cx = 0; cx < VX; ++cx) {
                    v[cy][cx] = mul_rn(w, accB[l - 1][cy][cx] + ps[cy][cx]);
                    accB[l - 1][cy][cx] = accA[l - 1][cy][cx] + ps[cy][cx];
                    accA[l - 1][cy][cx] = ps[cy][cx];
                }
            const int p = c - 1;
            if (l < KL) {
                // Dirichlet: cells outside the interior keep their level-0 value
                // (value of level l-1 at plane p: for l = 1 the previous ring
                // plane's centre kept in registers; for l > 1 the level-(l-1)
                // plane p still in its SMEM slot — level l-1 overwrites it only
                // later in this step)
                if (!(warp_int && p >= 0 && p < a.n0)) {  // warp-uniform
                    const bool pint = p >= 0 && p < a.n0;
                    T kv[VY][VX];
                    if (l == 1) {
#pragma unroll
                        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                            for (int cx = 0; cx < VX; ++cx) kv[cy][cx] = keep0[cy][cx];
                    } else {
                        const T* Bp = buf + ((l - 2) * NB + ((p % NB) + NB) % NB) * BE;
#pragma unroll
                        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                            for (int cx = 0; cx < VX; ++cx)
                                kv[cy][cx] = Bp[(y + cy + 1) * BW + x + PL + cx];
                    }
#pragma unroll
                    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                        for (int cx = 0; cx < VX; ++cx)
                            if (!(pint && cint[cy][cx])) v[cy][cx] = kv[cy][cx];
                }
                if (l == 1 && (!warp_int || c - 1 < 0 || c + 1 >= a.n0)) {  // next plane may select
#pragma unroll
                    for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                        for (int cx = 0; cx < VX; ++cx) keep0[cy][cx] = nb[cy + 1][cx + 1];
                }
                T* B = buf + ((l - 1) * NB + ((p % NB) + NB) % NB) * BE;
#pragma unroll
                for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                    for (int vv = 0; vv < VX; vv += NV) {
                        V4 o;
                        T* e = reinterpret_cast<T*>(&o);
#pragma unroll
                        for (int u = 0; u < NV; ++u) e[u] = v[cy][vv + u];
                        *reinterpret_cast<V4*>(B + (y + cy + 1) * BW + x + PL + vv) = o;
                    }
            } else if (p >= i0 && p < i1) {  // p = q - LAG
#pragma unroll
                for (int cy = 0; cy < VY; ++cy) {
                    store_row<T, VX>(orow + cy * a.pitch1, v[cy], cout[cy]);
                    if (a.mirror)
                        store_row<T, VX>(a.mirror + (orow - out) + a.mshift + cy * a.pitch1, v[cy],
                                         cout[cy]);
                }
            }
        }
        __syncthreads();  // level planes published; ring slot of plane q free
        if (tid == 0 && it + STAGES < niter) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[slot], kBoxBytes);
            tma_load_3d(ring + slot * SLOT, &tmap, &bar[slot], c0, c1,
                        min(a.h0 + t_begin + it + STAGES, last_plane));
        }
    }
}

bool supports(const Geo& g, const TapSet& t, int* max_fused, int* default_fused) {
    if (t.dims != 3 || t.shape != TSR_BOX || t.radius != 1 || t.ntaps != 27) return false;
    if (g.n[0] + 2 * g.h[0] > (1 << 30) || g.n[1] + 2 * g.h[1] > (1 << 30)) return false;
    *max_fused = 2;
    *default_fused = 1;  // EXACT: k=2 is FP-issue-bound at the same rate
    return true;
}

// FAST with uniform weights runs the separable sums: fp32 in tbbox.cu
// (register windows of plane sums, k = 3 default: C4 1238 GS/s, against
// 1068 at k = 2 and 714 for EXACT's Q mode), fp64 in the k-level
// shared-memory pipeline above (k = 2: 199 / 250 registers at k = 3 / 4).
int fast_default(const Geo& g, const TapSet& t) {
    if (!uniform_weights(t)) return 1;
    return g.dtype == TSR_F32 ? 3 : 2;
}
int fast_max(const Geo&, const TapSet& t) { return uniform_weights(t) ? 4 : 2; }

template <typename T, int MODE>
Status launch(const LaunchCtx& c, const void* in, void* out) {
    const Geo& g = *c.g;
    CUtensorMap map;
    Status s = make_tmap_3d<T>(g, in, BXW1<T>, BY, &map);
    if (!s.ok()) return s;
    BoxArgs<T> a;
    a.n0 = (int)g.n[0];
    a.n1 = (int)g.n[1];
    a.n2 = (int)g.n[2];
    a.tiles_x = (int)((g.n[2] + OX1<T> - 1) / OX1<T>);
    a.tiles_y = (int)((g.n[1] + OY - 1) / OY);
    a.h0 = (int)g.h[0];
    a.h1 = (int)g.h[1];
    a.off2 = (int)g.off2;
    a.pitch0 = g.pitch[0];
    a.pitch1 = g.pitch[1];
    a.origin = g.origin;
    a.mirror = static_cast<T*>(c.mirror);
    a.mshift = c.mirror_shift;
    for (int q = 0; q < 27; ++q) a.w[q] = static_cast<T>(c.taps->w[q]);
    constexpr int bytes = smem_bytes<T>();
    int per_sm = 1, nsm = 148;
    s = occupancy(box3d_kernel<T, MODE>, NT1<T>, bytes, &per_sm, &nsm);
    if (!s.ok()) return s;
    const long long tiles = (long long)a.tiles_x * a.tiles_y;
    a.lo0 = (int)c.range_lo();
    a.hi0 = (int)c.range_hi();
    if (a.hi0 <= a.lo0) return Status::Ok();
    const int64_t span = a.hi0 - a.lo0;
    a.chunk = pick_chunk(span, tiles, (long long)nsm * per_sm, 2, 32);
    const long long nchunks = (span + a.chunk - 1) / a.chunk;
    box3d_kernel<T, MODE><<<(unsigned)(tiles * nchunks), NT1<T>, bytes, c.stream>>>(
        static_cast<T*>(out), map, a);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

template <typename T, int MODE>
Status launch2(const LaunchCtx& c, const void* in, void* out) {
    const Geo& g = *c.g;
    CUtensorMap map;
    Status s = make_tmap_3d<T>(g, in, BXW<T>, BY, &map);
    if (!s.ok()) return s;
    BoxArgs<T> a;
    a.n0 = (int)g.n[0];
    a.n1 = (int)g.n[1];
    a.n2 = (int)g.n[2];
    a.tiles_x = (int)((g.n[2] + TX2<T> - 1) / TX2<T>);
    a.tiles_y = (int)((g.n[1] + TY2 - 1) / TY2);
    a.h0 = (int)g.h[0];
    a.h1 = (int)g.h[1];
    a.off2 = (int)g.off2;
    a.pitch0 = g.pitch[0];
    a.pitch1 = g.pitch[1];
    a.origin = g.origin;
    a.mirror = static_cast<T*>(c.mirror);
    a.mshift = c.mirror_shift;
    for (int q = 0; q < 27; ++q) a.w[q] = static_cast<T>(c.taps->w[q]);
    constexpr int bytes = smem2_bytes<T>();
    int per_sm = 1, nsm = 148;
    s = occupancy(box3d_tb2_kernel<T, MODE>, NT, bytes, &per_sm, &nsm);
    if (!s.ok()) return s;
    const long long tiles = (long long)a.tiles_x * a.tiles_y;
    a.lo0 = (int)c.range_lo();
    a.hi0 = (int)c.range_hi();
    if (a.hi0 <= a.lo0) return Status::Ok();
    const int64_t span = a.hi0 - a.lo0;
    a.chunk = pick_chunk(span, tiles, (long long)nsm * per_sm, 4, 32);
    const long long nchunks = (span + a.chunk - 1) / a.chunk;
    box3d_tb2_kernel<T, MODE><<<(unsigned)(tiles * nchunks), NT, bytes, c.stream>>>(
        static_cast<T*>(out), map, a);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

template <typename T, int KL>
Status launchk(const LaunchCtx& c, const void* in, void* out) {
    const Geo& g = *c.g;
    CUtensorMap map;
    Status s = make_tmap_3d<T>(g, in, BXW<T>, BY, &map);
    if (!s.ok()) return s;
    BoxArgs<T> a;
    a.n0 = (int)g.n[0];
    a.n1 = (int)g.n[1];
    a.n2 = (int)g.n[2];
    a.tiles_x = (int)((g.n[2] + TXK<KL, T> - 1) / TXK<KL, T>);
    a.tiles_y = (int)((g.n[1] + TYK<KL> - 1) / TYK<KL>);
    a.h0 = (int)g.h[0];
    a.h1 = (int)g.h[1];
    a.off2 = (int)g.off2;
    a.pitch0 = g.pitch[0];
    a.pitch1 = g.pitch[1];
    a.origin = g.origin;
    a.mirror = static_cast<T*>(c.mirror);
    a.mshift = c.mirror_shift;
    for (int q = 0; q < 27; ++q) a.w[q] = static_cast<T>(c.taps->w[q]);
    constexpr int bytes = smemk_bytes<KL, T>();
    int per_sm = 1, nsm = 148;
    s = occupancy(box3d_tbk_sep_kernel<T, KL>, NT, bytes, &per_sm, &nsm);
    if (!s.ok()) return s;
    const long long tiles = (long long)a.tiles_x * a.tiles_y;
    a.lo0 = (int)c.range_lo();
    a.hi0 = (int)c.range_hi();
    if (a.hi0 <= a.lo0) return Status::Ok();
    const int64_t span = a.hi0 - a.lo0;
    a.chunk = pick_chunk(span, tiles, (long long)nsm * per_sm, 3 * KL, 32);
    const long long nchunks = (span + a.chunk - 1) / a.chunk;
    box3d_tbk_sep_kernel<T, KL><<<(unsigned)(tiles * nchunks), NT, bytes, c.stream>>>(
        static_cast<T*>(out), map, a);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

Status tbbox_run_dispatch(const LaunchCtx& c, const void* in, void* out, int k);

template <typename T>
Status run_t(const LaunchCtx& c, const void* in, void* out, int k) {
    // uniform weights: Q in EXACT mode (bitwise), separable sums in FAST
    const int mode = uniform_weights(*c.taps) ? (c.exact ? 2 : 3) : c.exact ? 1 : 0;
    // (k = 1: the one-level plane-sum kernel below streams faster than tbbox's k = 1)
    if (mode == 3 && sizeof(T) == 4 && k >= 2) return tbbox_run_dispatch(c, in, out, k);
    if (mode == 3 && k >= 2) {  // SEP: the k-level skewed pipeline
        if (k == 3) return launchk<T, 3>(c, in, out);
        if (k == 4) return launchk<T, 4>(c, in, out);
        return launchk<T, 2>(c, in, out);
    }
    if (k == 2) {
        switch (mode) {
            case 0: return launch2<T, 0>(c, in, out);
            case 1: return launch2<T, 1>(c, in, out);
            default: return launch2<T, 2>(c, in, out);
        }
    }
    if (k != 1) return Status::Err(TSR_EUNSUPPORTED, "box3d fuses one or two steps per pass");
    switch (mode) {
        case 0: return launch<T, 0>(c, in, out);
        case 1: return launch<T, 1>(c, in, out);
        case 2: return launch<T, 2>(c, in, out);
        default: return launch<T, 3>(c, in, out);
    }
}

Status run(const LaunchCtx& c, const void* in, void* out, int k) {
    if (c.g->dtype == TSR_F64) return run_t<double>(c, in, out, k);
    return run_t<float>(c, in, out, k);
}

}  // namespace

Status tbbox_run(const LaunchCtx& c, const void* in, void* out, int k);

namespace {
Status tbbox_run_dispatch(const LaunchCtx& c, const void* in, void* out, int k) {
    return tbbox_run(c, in, out, k);
}
}  // namespace

extern const Engine kBox3dEngine = {"box3d_r1_planesum", supports, run, fast_default, fast_max};

}  // namespace tsr
