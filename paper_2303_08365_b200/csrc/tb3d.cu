// tb3d.cu — 3-D radius-1 star (7-point) sweep with K time steps fused per
// HBM pass: the paper's three tiers rebuilt for sm_100a.
//
//  * Memory tier: a CTA owns an output tile of (R1Y-2(K-1)) x (64-2(K-1))
//    cells of the (a1, a2) plane (region R1Y = 32, or 36 for K = 3) and
//    streams consecutive a0 planes of it.  For K >= 2 the grid is
//    persistent, one CTA per SM: CTA b streams whole tiles b, b+W, ... with
//    every CTA at the same plane, so neighbouring tiles read the halo rows
//    their boxes share once from HBM and once from L2 (C3: 2.86 -> 2.29 GB
//    of DRAM per launch), then an even share of the leftover tiles' planes.
//    Level-0 planes (the tile plus a (K-1)+1 halo ring) arrive by TMA
//    (cp.async.bulk.tensor.3d) into a shared-memory ring guarded by
//    mbarriers (planes t-2 .. t+STAGES-3 of step t, as deep as the shared
//    memory left by the level buffers allows).
//  * SMEM tier (locality enhancer): levels 1..K-1 are computed on the same
//    region (overlapped tiling: the valid part shrinks by one cell per level)
//    as a wavefront along a0 — level l works on plane t-2l — so K steps cost
//    one HBM read and one HBM write per cell.  The two-plane skew makes the
//    K levels' dependency chains independent within a step; each level's
//    newest plane goes to a 3-deep SMEM buffer for the a1-neighbours of other
//    warps, read two steps later; one __syncthreads per plane serves all K
//    levels.
//  * Register tier (pattern mapping): a thread owns a 2 (a1) x 2 (a2) stack
//    of columns and keeps, per level, a three-plane window in registers (the
//    a0-neighbours), rotated by renaming (step loop unrolled by 3);
//    a2-neighbours come from the adjacent lane by warp shuffle,
//    a1-neighbours inside the stack from its own registers.
//  * Boundary handling is decided per warp and per 3-step unit: warps with no
//    boundary column whose planes are all interior run a select-free
//    instantiation (no Dirichlet selects, no store-range check).
// Per point and level the arithmetic is apply_box's
// (proj/include/tessera/naive.hpp:69-82): acc = 0, then the seven taps in
// canonical order (-1,0,0) (0,-1,0) (0,0,-1) (0,0,0) (0,0,1) (0,1,0) (1,0,0).
// Cells outside the interior keep their level-0 value at every level
// (Dirichlet halo, grid.hpp:14-18), so EXACT mode is bitwise naive_run.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tma.cuh"

namespace tsr {

namespace {

constexpr int R1X = 64;  // level-1 region width  (a2)
constexpr int VX = 2;    // columns per thread along a2
constexpr int NLX = R1X / VX;  // 32 lanes

// Region height and column-stack depth: a warp owns VY rows of the R1Y-row
// level-1 region, so a CTA has R1Y / VY warps.
template <int VY_, int R1Y_>
struct Shape {
    static constexpr int VY = VY_;          // columns per thread along a1
    static constexpr int R1Y = R1Y_;        // level-1 region height (a1)
    static constexpr int NLY = R1Y / VY;    // warps
    static constexpr int NT = NLX * NLY;    // threads
    static constexpr int BY0 = R1Y + 2;     // TMA box height: 1 extra row per side
    // Level buffers keep only the rows other warps read: each warp's first
    // and last row (warp w's at buffer rows 2w+1 and 2w+2), plus one padding
    // row per side.  For VY = 2 that is every region row.
    static constexpr int LEVY = 2 * NLY + 2;
};
// 512 threads, 2x2 columns per thread.  A 4x2 stack with 256 threads
// (half the SMEM traffic per point, 186-239 registers) measured 2-4% slower
// in exact mode: 8 warps per SM hide too little latency.
using ShapeA = Shape<2, 32>;

template <typename T>
struct Pair;
template <>
struct Pair<double> {
    using type = double2;
};
template <>
struct Pair<float> {
    using type = float2;
};

// TMA boxes must start on a 16-byte boundary of the innermost dimension, so
// the ring carries PADL = 16/sizeof(T) columns left of region-1 (and as many
// right), and the region's left overlap Hx is rounded up to that vector.
template <typename T>
constexpr int VEC = 16 / (int)sizeof(T);
template <typename T>
constexpr int PADL = VEC<T>;
template <typename T>
constexpr int BX0 = R1X + 2 * PADL<T>;  // TMA box width
template <typename T, int K>
constexpr int HXL = (K - 1 + VEC<T> - 1) / VEC<T> * VEC<T>;  // left overlap
template <typename T, int K>
constexpr int TXO = (R1X - HXL<T, K> - (K - 1)) / VEC<T> * VEC<T>;  // output tile width

template <typename T, typename G>
constexpr int slot_bytes() {
    return (BX0<T> * G::BY0 * (int)sizeof(T) + 1023) / 1024 * 1024;
}
template <typename T, typename G>
constexpr int lev_bytes() {
    return (G::LEVY * R1X * (int)sizeof(T) + 127) / 128 * 128;
}
constexpr int NLEV = 3;  // level-l planes are read two steps after they are written
constexpr int kSmemMax = 227 * 1024;  // dynamic shared memory per CTA (sm_100)
constexpr int kMaxStages = 10;
// Ring depth: planes t-2 .. t+STAGES-3 of the level-0 ring, i.e. STAGES-2
// planes in flight ahead of the one being consumed.  As deep as the shared
// memory left by the level buffers allows: the persistent K >= 2 schedule
// keeps one CTA per SM, so the planes in flight per SM bound the HBM rate
// (measured: K = 2 and K = 3 both stalled near 4.6 TB/s with 3 in flight).
template <typename T, int K, typename G>
constexpr int stages() {
    if (K == 1) return 5;  // chunked schedule, several CTAs per SM: HBM-bound already
    const int avail = kSmemMax - NLEV * (K - 1) * lev_bytes<T, G>() - kMaxStages * 8;
    const int n = avail / slot_bytes<T, G>();
    return n < kMaxStages ? n : kMaxStages;
}
template <typename T, int K, typename G>
constexpr int smem_bytes() {
    return stages<T, K, G>() * slot_bytes<T, G>() + NLEV * (K - 1) * lev_bytes<T, G>() +
           kMaxStages * 8;
}

template <typename T>
struct TbArgs {
    int n0, n1, n2;
    int tiles_x, tiles_y;
    long long per_cta;  // remainder (tile, plane) positions per CTA (persistent), or
    int chunk;          // > 0: one chunk of a0 planes per CTA, tiles fastest
    int full_tiles;     // persistent: whole tiles per CTA before the remainder
    int lo0, hi0;  // output planes [lo0, hi0) of a0
    int h0, h1, off2;
    long long pitch0, pitch1, origin;
    T* mirror;  // LaunchCtx::mirror (fused halo exchange), or nullptr
    long long mshift;
    T w[7];
};

// The reference starts every sum from +0 (naive.hpp:75); that accumulator can
// never become -0, so dropping the leading "0 +" changes at most the sign of
// a zero result, in intermediate levels too (x + (-0) == x + (+0) unless both
// are zero).  tb3d_step restores the reference's +0 with one `+ 0.0` per
// stored value instead of one per level and point.
template <bool EXACT, typename T>
__device__ __forceinline__ T stencil7(const T* w, T prev, T up, T left, T c, T right, T down,
                                      T next) {
    T acc;
    if constexpr (EXACT)
        acc = sizeof(T) == 8 ? (T)__dmul_rn((double)w[0], (double)prev) : (T)__fmul_rn((float)w[0], (float)prev);
    else
        acc = first<EXACT>(w[0], prev);
    acc = madd<EXACT>(acc, w[1], up);
    acc = madd<EXACT>(acc, w[2], left);
    acc = madd<EXACT>(acc, w[3], c);
    acc = madd<EXACT>(acc, w[4], right);
    acc = madd<EXACT>(acc, w[5], down);
    return madd<EXACT>(acc, w[6], next);
}

// One step of the wavefront (iteration `it`, PH = it % 3).  Level l works on
// plane t - 2l: two planes behind level l-1, so every input of every level
// was produced in an earlier step and the K levels' dependency chains are
// independent within a step.  Levels run in descending order: level l+1
// consumes the oldest plane of level l's three-plane register window before
// level l overwrites it.  Hs[l][s] holds the level-l value of plane q with
// (q - t_begin) % 3 == s, so the window rotates by renaming (loop unrolled
// by 3).  a1-neighbour rows of other warps are read two steps after they
// were written (3-deep SMEM buffers, one __syncthreads per step).
template <typename T, int K, bool EXACT, int PH, int SEL, typename G, bool EARLY0, bool MIRROR>
__device__ __forceinline__ void tb3d_step(const TbArgs<T>& a, T* __restrict__ out, T* ring, T* lev,
                                          uint64_t* bar, int& rslot, unsigned& rphase, int it,
                                          int t_begin,
                                          int i0, int i1, int lx, int x, int y, long long& ooff,
                                          const bool (&cint)[G::VY][VX],
                                          const bool (&cout)[G::VY][VX], bool hl,
                                          T (&Hs)[K][3][G::VY][VX]) {
    constexpr int VY = G::VY;
    constexpr int STAGES = stages<T, K, G>();
    using P2 = typename Pair<T>::type;
    constexpr int SLOT = slot_bytes<T, G>() / (int)sizeof(T);
    constexpr int LEV = lev_bytes<T, G>() / (int)sizeof(T);
    constexpr int BX = BX0<T>, PL = PADL<T>;
    const int t = t_begin + it;
    const int ly2 = 2 * (y / VY);  // level-buffer row of this warp's first row, minus 1
    // ring position of plane t (slot and mbarrier phase), advanced by one per
    // step instead of divided out of the load count
    const int slot = rslot;
    const unsigned phase = rphase;
    const int slot_m2 = slot >= 2 ? slot - 2 : slot + STAGES - 2;  // plane t-2
    const T* P0 = ring + slot * SLOT;
    P2 early[VY];
    if constexpr (EARLY0) {  // level-0 rows of plane t fetched before the levels' math
        mbar_wait(&bar[slot], phase);
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
            early[cy] = *reinterpret_cast<const P2*>(P0 + (y + cy + 1) * BX + x + PL);
    }

#pragma unroll
    for (int l = K; l >= 1; --l) {
        const int p = t - 2 * l;                          // plane level l produces now
        const int sP = ((PH - 2 * l - 1) % 3 + 3) % 3;    // slot of plane p-1
        const int sC = ((PH - 2 * l) % 3 + 3) % 3;        // slot of plane p
        const int sN = ((PH - 2 * l + 1) % 3 + 3) % 3;    // slot of plane p+1
        // a1-neighbour rows y-1 and y+VY of level l-1 at plane p
        P2 u, d;
        const T* Pm = nullptr;
        if (l == 1) {
            Pm = ring + slot_m2 * SLOT;  // level 0, plane t-2
            u = *reinterpret_cast<const P2*>(Pm + (y) * BX + x + PL);
            d = *reinterpret_cast<const P2*>(Pm + (y + VY + 1) * BX + x + PL);
        } else {
            const T* L = lev + ((l - 2) * NLEV + sC) * LEV;
            // last row of the warp above, first row of the warp below
            u = *reinterpret_cast<const P2*>(L + (ly2) * R1X + x);
            d = *reinterpret_cast<const P2*>(L + (ly2 + 3) * R1X + x);
        }
        T res[VY][VX];
#pragma unroll
        for (int cy = 0; cy < VY; ++cy) {
            const T c0v = Hs[l - 1][sC][cy][0], c1v = Hs[l - 1][sC][cy][1];
            T left = __shfl_up_sync(0xffffffffu, c1v, 1);
            T right = __shfl_down_sync(0xffffffffu, c0v, 1);
            if (l == 1) {  // region-1 edge columns read the level-0 halo ring
                // every lane loads the two edge cells (one broadcast wavefront
                // each) and the edge lanes select them: no divergent branch
                const T el = Pm[(y + cy + 1) * BX + PL - 1];
                const T er = Pm[(y + cy + 1) * BX + R1X + PL];
                left = lx == 0 ? el : left;
                right = lx == NLX - 1 ? er : right;
            }
            const T up0 = cy == 0 ? u.x : Hs[l - 1][sC][cy - 1][0];
            const T up1 = cy == 0 ? u.y : Hs[l - 1][sC][cy - 1][1];
            const T dn0 = cy == VY - 1 ? d.x : Hs[l - 1][sC][cy + 1][0];
            const T dn1 = cy == VY - 1 ? d.y : Hs[l - 1][sC][cy + 1][1];
            res[cy][0] = stencil7<EXACT>(a.w, Hs[l - 1][sP][cy][0], up0, left, c0v, c1v, dn0,
                                         Hs[l - 1][sN][cy][0]);
            res[cy][1] = stencil7<EXACT>(a.w, Hs[l - 1][sP][cy][1], up1, c0v, c1v, right, dn1,
                                         Hs[l - 1][sN][cy][1]);
        }
        // Dirichlet: cells outside the interior keep their level-0 value
        // (only the SEL instantiations: 1 = boundary columns/rows of this
        // warp on interior planes, 2 = also a0-boundary planes / wavefront
        // fill and drain).
        // Level K's values are only stored where cout (interior) holds, so
        // it needs no select.
        if ((SEL == 3 || SEL == 4) && l < K) {
            // a2-edge warp whose rows are all interior: the one non-interior
            // cell an interior cell reads is the halo column, held by lane
            // `hl` in column 1 (SEL 3) or 0 (SEL 4); cells beyond it feed only it
            constexpr int hc = SEL == 3 ? 1 : 0;
#pragma unroll
            for (int cy = 0; cy < VY; ++cy)
                if (hl) res[cy][hc] = Hs[l - 1][sC][cy][hc];
        } else if (SEL != 0 && l < K) {
            const bool pint = SEL == 1 || (p >= 0 && p < a.n0);
#pragma unroll
            for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                for (int cx = 0; cx < VX; ++cx) {
                    const bool keep = !(pint & cint[cy][cx]);  // one predicate, one select
                    if (keep) res[cy][cx] = Hs[l - 1][sC][cy][cx];
                }
        }
        if (l < K) {
            T* L = lev + ((l - 1) * NLEV + sC) * LEV;
#pragma unroll
            for (int cy = 0; cy < VY; ++cy) {
                // only a warp's first and last rows are read by other warps
                if (cy == 0 || cy == VY - 1) {
                    P2 v;
                    v.x = res[cy][0];
                    v.y = res[cy][1];
                    *reinterpret_cast<P2*>(L + (ly2 + (cy == 0 ? 1 : 2)) * R1X + x) = v;
                }
#pragma unroll
                for (int cx = 0; cx < VX; ++cx) Hs[l][sC][cy][cx] = res[cy][cx];
            }
        } else if (SEL != 2 || (p >= i0 && p < i1)) {  // SEL < 2: the caller checked the range
            T* o = out + ooff;  // plane p of this thread's column stack
#pragma unroll
            for (int cy = 0; cy < VY; ++cy) {
                T v[VX];
#pragma unroll
                for (int cx = 0; cx < VX; ++cx) v[cx] = fix_zero<EXACT>(res[cy][cx]);
                if constexpr (SEL == 0 && VX * sizeof(T) == 16) {
                    // select-free warps have no boundary column: a lane's two
                    // columns are both in or both out of the output tile
                    if (cout[cy][0]) {
                        *reinterpret_cast<P2*>(o + cy * a.pitch1) = P2{v[0], v[1]};
                        if constexpr (MIRROR)
                            *reinterpret_cast<P2*>(a.mirror + (o - out) + a.mshift + cy * a.pitch1) =
                                P2{v[0], v[1]};
                    }
                } else {
                    store_row<T, VX>(o + cy * a.pitch1, v, cout[cy]);
                    if constexpr (MIRROR)
                        store_row<T, VX>(a.mirror + (o - out) + a.mshift + cy * a.pitch1, v, cout[cy]);
                }
            }
        }
    }
    // Level 0 last: plane t into the window slot level 1 has just consumed.
    if constexpr (!EARLY0) mbar_wait(&bar[slot], phase);
#pragma unroll
    for (int cy = 0; cy < VY; ++cy) {
        const P2 v = EARLY0 ? early[cy]
                            : *reinterpret_cast<const P2*>(P0 + (y + cy + 1) * BX + x + PL);
        Hs[0][PH][cy][0] = v.x;
        Hs[0][PH][cy][1] = v.y;
    }
    ooff += a.pitch0;
    if (slot == STAGES - 1) {
        rslot = 0;
        rphase = phase ^ 1u;
    } else {
        rslot = slot + 1;
    }
}

template <typename T, int K, bool EXACT, typename G, bool EARLY0, bool MIRROR>
__global__ void __launch_bounds__(G::NT, 1)
    tb3d_kernel(T* __restrict__ out, const __grid_constant__ CUtensorMap tmap,
                const __grid_constant__ TbArgs<T> a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int VY = G::VY, R1Y = G::R1Y, BY0 = G::BY0;
    constexpr int STAGES = stages<T, K, G>();
    static_assert(STAGES >= 5, "the ring holds planes t-2 .. t+2 at least");
    constexpr int SLOT = slot_bytes<T, G>() / (int)sizeof(T);
    T* ring = reinterpret_cast<T*>(smem);
    T* lev = reinterpret_cast<T*>(smem + STAGES * slot_bytes<T, G>());
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + STAGES * slot_bytes<T, G>() +
                                                NLEV * (K - 1) * lev_bytes<T, G>());

    const int tid = threadIdx.x;
    const int lx = tid & 31, ly = tid >> 5;
    constexpr int TX = TXO<T, K>, TY = R1Y - 2 * (K - 1);
    constexpr int PL = PADL<T>, HX = HXL<T, K>;
    constexpr unsigned kBoxBytes = BX0<T> * BY0 * sizeof(T);
    // Columns owned: region-1 (y, x) = (VY*ly + cy, VX*lx + cx).
    const int x = VX * lx, y = VY * ly;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmap);
    }
    __syncthreads();

    // Persistent schedule (K >= 2), in two phases.  Phase 1: CTA b streams
    // whole tiles b, b + W, b + 2W, ... (W = grid size), all CTAs starting
    // at the same plane, so tiles that are neighbours in (a1, a2) run
    // side by side at the same a0 position and the halo rows their TMA
    // boxes share are read from HBM once and from L2 the second time.
    // Phase 2: the tiles left over (fewer than W) are one tile-major
    // (tile, plane) position space split evenly over the CTAs.  Only a tile
    // change refills the wavefront (3K steps).
    // K = 1 is HBM-bound: it keeps one chunk per CTA with the tiles of a
    // chunk on consecutive CTAs (the same L2 sharing, many CTAs per SM).
    const long long span = a.hi0 - a.lo0;
    const int ntile = a.tiles_x * a.tiles_y;
    const int tile_rem0 = a.full_tiles * (int)gridDim.x;  // first phase-2 tile
    const long long total = (long long)(ntile - tile_rem0) * span;
    long long pos, end;
    int full_left = 0, full_tile = blockIdx.x;
    if (a.chunk > 0) {
        const int tile = blockIdx.x % ntile, bz = blockIdx.x / ntile;
        const long long off = (long long)bz * a.chunk;
        pos = (long long)tile * span + off;
        end = pos + min((long long)a.chunk, span - off);
    } else {
        full_left = a.full_tiles;
        pos = (long long)blockIdx.x * a.per_cta;
        end = min(pos + a.per_cta, total);
    }
    unsigned gbase = 0;  // ring loads issued by earlier segments
    int rslot = 0;         // ring slot / mbarrier phase of the next load, i.e.
    unsigned rphase = 0;   // (gbase + it) % STAGES and ((gbase + it) / STAGES) & 1
    T Hs[K][3][VY][VX];
#pragma unroll
    for (int l = 0; l < K; ++l)
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                for (int cx = 0; cx < VX; ++cx) Hs[l][s][cy][cx] = T(0);

    while (full_left > 0 || pos < end) {
        int tile, i0, i1;
        if (full_left > 0) {
            tile = full_tile;
            i0 = a.lo0;
            i1 = a.hi0;
            full_tile += gridDim.x;
            --full_left;
        } else {
            const int t = (int)(pos / span);
            i0 = a.lo0 + (int)(pos - (long long)t * span);
            i1 = (int)min((long long)a.hi0, (long long)i0 + (end - pos));
            pos += i1 - i0;
            tile = (a.chunk > 0 ? 0 : tile_rem0) + t;
        }
        const int bx = tile % a.tiles_x;
        const int by = tile / a.tiles_x;
        const int gx = bx * TX - HX;       // global a2 of region-1 column 0
        const int gy = by * TY - (K - 1);  // global a1 of region-1 row 0
        // level-0 planes i0-K .. i1+K-1; level K finishes plane i1-1 at step i1-1+2K
        const int t_begin = i0 - K, t_end = i1 + 2 * K;
        const int niter = t_end - t_begin;
        const int nload = i1 - i0 + 2 * K;  // level-0 planes actually needed

        bool cint[VY][VX], cout[VY][VX];
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int cx = 0; cx < VX; ++cx) {
                const int ga1 = gy + y + cy, ga2 = gx + x + cx;
                cint[cy][cx] = ga1 >= 0 && ga1 < a.n1 && ga2 >= 0 && ga2 < a.n2;
                cout[cy][cx] = cint[cy][cx] && y + cy >= K - 1 && y + cy < R1Y - (K - 1) &&
                               x + cx >= HX && x + cx < HX + TX;
            }

        const int c0 = a.off2 + gx - PL, c1 = a.h1 + gy - 1;  // 16-B aligned box start
        // element offset of this thread's output column stack at the plane
        // level K produces in the current step (p = t - 2K), advanced by one
        // plane per step: stores need no per-step 64-bit index arithmetic
        long long ooff = a.origin + (long long)(gy + y) * a.pitch1 + (gx + x) +
                         (long long)(t_begin - 2 * K) * a.pitch0;
        // plane index j (0-based from t_begin) is loaded at most once; the
        // steps that drain the wavefront past the last needed plane (i1+K-1)
        // re-load that plane instead, so a launch never reads outside its
        // dependency cone (a slab's interior range runs while its ghost
        // planes are being written)
        const int last_plane = a.h0 + t_begin + nload - 1;
        if (tid == 0) {
            // every thread finished the previous segment (after()'s barrier)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (int s = 0; s < STAGES && s < niter; ++s) {
                const int sl = (gbase + s) % STAGES;
                mbar_expect_tx(&bar[sl], kBoxBytes);
                tma_load_3d(ring + sl * SLOT, &tmap, &bar[sl], c0, c1,
                            min(a.h0 + t_begin + s, last_plane));
            }
        }

        auto after = [&](int it) {
            __syncthreads();
            // Plane t-2 was last read in this step (level-1 neighbours): its
            // slot takes plane t-2+STAGES.
            if (tid == 0 && it >= 2 && it - 2 + STAGES < niter) {
                // slot of plane t-2 = (gbase + it - 2) % STAGES; rslot is
                // already (gbase + it + 1) % STAGES, so the slot is rslot - 3.
                const int sl = rslot >= 3 ? rslot - 3 : rslot + STAGES - 3;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bar[sl], kBoxBytes);
                tma_load_3d(ring + sl * SLOT, &tmap, &bar[sl], c0, c1,
                            min(a.h0 + t_begin + it - 2 + STAGES, last_plane));
            }
        };
        bool mine = true;
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int cx = 0; cx < VX; ++cx) mine &= cint[cy][cx];
        const bool warp_int = __all_sync(0xffffffffu, mine);  // no boundary column in this warp
        // a2-edge warps with every row interior (the bulk of the boundary
        // tiles): only the halo column next to the interior (a2 = -1 or n2)
        // must keep its level-0 value; it sits in the same column slot of
        // every such lane (region columns start 16-B aligned), so a
        // one-column select tier serves them
        bool rows_in = true, hl0 = false, hl1 = false;
#pragma unroll
        for (int cy = 0; cy < VY; ++cy) rows_in &= gy + y + cy >= 0 && gy + y + cy < a.n1;
        hl0 = gx + x == -1 || gx + x == a.n2;
        hl1 = gx + x + 1 == -1 || gx + x + 1 == a.n2;
        const bool warp_rows = __all_sync(0xffffffffu, rows_in);
        const bool any0 = __any_sync(0xffffffffu, hl0), any1 = __any_sync(0xffffffffu, hl1);
        const int edge_tier = warp_int || !warp_rows ? 0 : (any1 && !any0) ? 3
                                                         : (any0 && !any1) ? 4 : 0;
        const bool hl = edge_tier == 3 ? hl1 : hl0;
        // A unit of three steps runs select-free when the planes its levels
        // read (t-2K .. t-2) are interior, no column of this warp is on the
        // a1/a2 boundary and every plane level K produces is one of this
        // segment's outputs (p = i0 + it - 3K in [i0, i1)); the conditions
        // are monotone in `it`, so checking the unit's first and last step
        // suffices.  Warp-uniform, decided once per unit.
        auto clear = [&](int it) {
            const int t = t_begin + it;
            return t - 2 * K >= 0 && t - 2 < a.n0 && it >= 3 * K && it < 3 * K + (i1 - i0);
        };
#define TB3D_STEP(PH, IT, SEL)                                                                  \
    tb3d_step<T, K, EXACT, PH, SEL, G, EARLY0, MIRROR>(a, out, ring, lev, bar, rslot, rphase, IT, t_begin, i0, i1, \
                                               lx, x, y, ooff, cint, cout, hl, Hs);             \
    after(IT);
        // The clear units form one interval of `it` (every condition of
        // clear() is an interval), so the tier is chosen once per segment:
        // general units for the wavefront fill, one uniform-tier loop over
        // the clear middle, general units for the drain.  Tier changes (and
        // the register moves that join them) happen at most twice per
        // segment instead of once per unit.
        auto unit_clear = [&](int it) { return clear(it) && clear(it + 2); };
        auto general_unit = [&](int it) {
            TB3D_STEP(0, it, 2)
            if (it + 1 < niter) {
                TB3D_STEP(1, it + 1, 2)
            }
            if (it + 2 < niter) {
                TB3D_STEP(2, it + 2, 2)
            }
        };
        int it = 0;
        for (; it < niter && !unit_clear(it); it += 3) general_unit(it);
        if (warp_int) {
            for (; it < niter && unit_clear(it); it += 3) {  // clear implies it + 2 < niter
                TB3D_STEP(0, it, 0)
                TB3D_STEP(1, it + 1, 0)
                TB3D_STEP(2, it + 2, 0)
            }
        } else if (!MIRROR && edge_tier == 3) {
            for (; it < niter && unit_clear(it); it += 3) {
                TB3D_STEP(0, it, 3)
                TB3D_STEP(1, it + 1, 3)
                TB3D_STEP(2, it + 2, 3)
            }
        } else if (!MIRROR && edge_tier == 4) {
            for (; it < niter && unit_clear(it); it += 3) {
                TB3D_STEP(0, it, 4)
                TB3D_STEP(1, it + 1, 4)
                TB3D_STEP(2, it + 2, 4)
            }
        } else if (!MIRROR) {  // a2/a1-edge warps of boundary tiles on interior planes
                               // (the seam-pass instance keeps two tiers: a third spills it)
            for (; it < niter && unit_clear(it); it += 3) {
                TB3D_STEP(0, it, 1)
                TB3D_STEP(1, it + 1, 1)
                TB3D_STEP(2, it + 2, 1)
            }
        }
        for (; it < niter; it += 3) general_unit(it);
        gbase += niter;
    }
#undef TB3D_STEP
}

constexpr int kMaxK = 3;  // k = 4 needs more SMEM than the 5-stage ring leaves

bool supports(const Geo& g, const TapSet& t, int* max_fused, int* default_fused) {
    if (t.dims != 3 || t.shape != TSR_STAR || t.radius != 1 || t.ntaps != 7) return false;
    // 32-bit plane / row indices inside the kernel
    if (g.n[0] + 2 * g.h[0] > (1 << 30) || g.n[1] + 2 * g.h[1] > (1 << 30)) return false;
    *max_fused = kMaxK;
    *default_fused = 3;
    return true;
}

template <typename T, int K, bool EXACT, typename G, bool EARLY0 = false>
Status launch_k(const LaunchCtx& c, const void* in, void* out) {
    const Geo& g = *c.g;
    CUtensorMap map;
    Status s = make_tmap_3d<T>(g, in, BX0<T>, G::BY0, &map);
    if (!s.ok()) return s;
    TbArgs<T> a;
    a.n0 = (int)g.n[0];
    a.n1 = (int)g.n[1];
    a.n2 = (int)g.n[2];
    constexpr int TX = TXO<T, K>, TY = G::R1Y - 2 * (K - 1);
    a.tiles_x = (int)((g.n[2] + TX - 1) / TX);
    a.tiles_y = (int)((g.n[1] + TY - 1) / TY);
    const long long tiles = (long long)a.tiles_x * a.tiles_y;
    constexpr int bytes = smem_bytes<T, K, G>();
    int per_sm = 1, nsm = 148;
    s = occupancy(tb3d_kernel<T, K, EXACT, G, EARLY0, false>, G::NT, bytes, &per_sm, &nsm);
    if (!s.ok()) return s;
    // persistent: one CTA per resident slot, each streaming an equal share of
    // the (tile, plane) positions
    a.lo0 = (int)c.range_lo();
    a.hi0 = (int)c.range_hi();
    if (a.hi0 <= a.lo0) return Status::Ok();
    const int64_t span = a.hi0 - a.lo0;
    const long long total = tiles * span;
    unsigned grid;
    a.full_tiles = 0;
    if (K == 1) {
        a.chunk = pick_chunk(span, tiles, (long long)nsm * per_sm, 2 * K, 48);
        a.per_cta = 0;
        grid = (unsigned)(tiles * ((span + a.chunk - 1) / a.chunk));
    } else {
        const long long slots = (long long)nsm * per_sm;
        a.chunk = 0;
        if (tiles >= slots) {  // phase 1: whole tiles, aligned planes
            grid = (unsigned)slots;
            a.full_tiles = (int)(tiles / slots);
            const long long left = tiles - (long long)a.full_tiles * slots;
            // nearly one leftover tile per CTA (C5: 132 for 148): whole tiles,
            // aligned, a few SMs idle; otherwise an even split of the planes
            a.per_cta = left * 100 >= slots * 85 ? span : (left * span + slots - 1) / slots;
        } else if (tiles * 10 >= slots * 9) {
            // nearly one tile per SM (C3: 144 tiles, 148 SMs): one whole tile
            // per CTA keeps the planes aligned; an even split would leave 4
            // SMs less idle but put neighbouring tiles at different planes
            grid = (unsigned)tiles;
            a.full_tiles = 1;
            a.per_cta = 0;
        } else {  // fewer tiles than SMs: the position space split evenly
            const long long ctas = std::min<long long>(slots, total);
            a.per_cta = (total + ctas - 1) / ctas;
            grid = (unsigned)((total + a.per_cta - 1) / a.per_cta);
        }
    }
    a.h0 = (int)g.h[0];
    a.h1 = (int)g.h[1];
    a.off2 = (int)g.off2;
    a.pitch0 = g.pitch[0];
    a.pitch1 = g.pitch[1];
    a.origin = g.origin;
    a.mirror = static_cast<T*>(c.mirror);
    a.mshift = c.mirror_shift;
    for (int q = 0; q < 7; ++q) a.w[q] = static_cast<T>(c.taps->w[q]);
    if (c.mirror) {
        static bool attr_set[64] = {};  // per device, once
        int dev = 0;
        TSR_CUDA_TRY(cudaGetDevice(&dev));
        if (dev >= 64 || !attr_set[dev]) {
            TSR_CUDA_TRY(cudaFuncSetAttribute(tb3d_kernel<T, K, EXACT, G, EARLY0, true>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            if (dev < 64) attr_set[dev] = true;
        }
        tb3d_kernel<T, K, EXACT, G, EARLY0, true><<<grid, G::NT, bytes, c.stream>>>(
            static_cast<T*>(out), map, a);
    } else {
        tb3d_kernel<T, K, EXACT, G, EARLY0, false><<<grid, G::NT, bytes, c.stream>>>(
            static_cast<T*>(out), map, a);
    }
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

// K = 3 uses 3x2 column stacks in a 64 x 36 region (384 threads, 168
// registers, 60 x 32 output tiles): against 2x2 stacks in 64 x 32 (512
// threads) it moves 22% fewer shared-memory / shuffle wavefronts per point
// (the warp-edge rows are a third of the rows instead of all of them),
// computes 5% fewer redundant cells per tile, and a 512^2 cross-section is
// 144 whole tiles (one wave on 148 SMs).  Measured C3 FAST 689 -> 714 GS/s,
// C5 772 -> 795.  K = 2 keeps 2x2 stacks (628 vs 515 GS/s).
using ShapeC = Shape<3, 36>;

template <typename T, bool EXACT>
Status launch_m(const LaunchCtx& c, const void* in, void* out, int k) {
    switch (k) {
        case 1: return launch_k<T, 1, EXACT, ShapeA>(c, in, out);
        case 2: return launch_k<T, 2, EXACT, ShapeA>(c, in, out);
        case 3: return launch_k<T, 3, EXACT, ShapeC, true>(c, in, out);
        default: return Status::Err(TSR_EUNSUPPORTED, "tb3d: fused steps must be 1..3");
    }
}

Status run(const LaunchCtx& c, const void* in, void* out, int k) {
    if (c.g->dtype == TSR_F64)
        return c.exact ? launch_m<double, true>(c, in, out, k)
                       : launch_m<double, false>(c, in, out, k);
    return c.exact ? launch_m<float, true>(c, in, out, k) : launch_m<float, false>(c, in, out, k);
}

}  // namespace

extern const Engine kTb3dEngine = {"star3d_r1_tb", supports, run};

}  // namespace tsr
