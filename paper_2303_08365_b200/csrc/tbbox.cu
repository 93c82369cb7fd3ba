// tbbox.cu — 3-D 27-point uniform box (the reference's Box-3D27P), FAST
// mode, k time steps fused per HBM pass: tb3d's design for the separable
// box sum (fp32).
//
// A uniform box update is w * S where S, the 27-point sum, factorises into
// horizontal 3-sums h (a2), their vertical 3-sums (a1: the plane sum P of
// one a0 plane) and three plane sums along a0:
//     out(p) = w * ((P(p-1) + P(p)) + P(p+1)),
// so each level keeps two open accumulators per point (accB = P(p-1)+P(p),
// accA = P(p+1)) and consumes one source plane per step.  Within the
// north star's tolerance of the oracle's lexicographic order (1e-5 fp32;
// only the rounding of the reassociated sum differs).  The weight multiply is
// __fmul_rn: were it left to the compiler, it could be contracted into an FMA
// with the next level's h additions in some step tiers and not others, and a
// point's bits would depend on the tiling (a slab run would not reproduce a
// one-device run).
//
//  * Memory tier: a CTA owns a 128 (a2) x R1Y (a1) level-1 region and
//    streams a0 planes of it; level-0 planes (region + 1-cell halo) arrive
//    by TMA into a shared-memory ring guarded by mbarriers; persistent,
//    aligned schedule as tb3d's (neighbouring tiles at the same plane share
//    their halo rows through L2).
//  * Levels: level l consumes at step t the level-(l-1) plane
//    c = t - 2(l-1) (level 1: ring plane t; higher levels: the plane the
//    level below produced in the previous step) and produces plane c - 1,
//    so a step's reads all see data published before the last barrier.  Each
//    thread owns a VY x 4 column stack; a2 neighbours by warp shuffle (one
//    SHFL per float), a1 neighbours as the h rows other warps publish to a
//    two-slot shared-memory buffer per level (only the warps' edge rows).
//  * Dirichlet: cells outside the interior keep their level-0 value at every
//    level; level l+1 reads level l's raw values of the plane two back, kept
//    in registers (level 1: the ring).  Select-free tier for interior warps
//    on interior planes, chosen once per segment (fill / clear / drain).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tma.cuh"

namespace tsr {

namespace {

using T = float;
constexpr int VX = 4;             // columns per thread (one 16-B vector)
constexpr int R1X = 32 * VX;      // region width: one warp spans it
constexpr int PL = 4;             // ring columns left of region col 0 (16-B aligned)
constexpr int BX0 = R1X + 2 * PL; // TMA box width
constexpr int kSmemMax = 227 * 1024;
constexpr int kMaxStages = 10;
constexpr int NB = 2;             // level h buffers: written at step s, read at s+1

template <int VY_, int R1Y_>
struct Shape {
    static constexpr int VY = VY_;
    static constexpr int R1Y = R1Y_;
    static constexpr int NLY = R1Y / VY;   // warps
    static constexpr int NT = 32 * NLY;
    static constexpr int BY0 = R1Y + 2;
    static constexpr int LEVY = 2 * NLY + 2;  // warps' edge rows + one padding row per side
};

template <int K>
constexpr int HXL = (K - 1 + 3) / 4 * 4;  // left overlap, vector aligned
template <int K>
constexpr int TXO = (R1X - HXL<K> - (K - 1)) / 4 * 4;  // output tile width

template <typename G>
constexpr int slot_bytes() {
    return (BX0 * G::BY0 * (int)sizeof(T) + 1023) / 1024 * 1024;
}
template <typename G>
constexpr int lev_bytes() {
    return (G::LEVY * R1X * (int)sizeof(T) + 127) / 128 * 128;
}
template <int K, typename G>
constexpr int stages() {
    const int avail = kSmemMax - NB * (K - 1) * lev_bytes<G>() - kMaxStages * 8;
    const int n = avail / slot_bytes<G>();
    return n < kMaxStages ? n : kMaxStages;
}
template <int K, typename G>
constexpr int smem_bytes() {
    return stages<K, G>() * slot_bytes<G>() + NB * (K - 1) * lev_bytes<G>() + kMaxStages * 8;
}

struct BoxArgs {
    int n0, n1, n2;
    int tiles_x, tiles_y;
    long long per_cta;
    int full_tiles;
    int lo0, hi0;
    int h0, h1, off2;
    long long pitch0, pitch1, origin;
    T* mirror;
    long long mshift;
    T w;
};

// h of one row of the thread's 4 columns: left / right neighbours from the
// adjacent lanes; lane 0 / 31 take the region-edge cells `el` / `er` (the
// ring's halo columns at level 0; don't-care values at higher levels, whose
// valid region has shrunk past the edge).
__device__ __forceinline__ void hrow(const float4 v, float el, float er, int lx, float (&h)[VX]) {
    float left = __shfl_up_sync(0xffffffffu, v.w, 1);
    float right = __shfl_down_sync(0xffffffffu, v.x, 1);
    left = lx == 0 ? el : left;
    right = lx == 31 ? er : right;
    const float m0 = v.x + v.y, m2 = v.z + v.w;
    h[0] = left + m0;
    h[1] = m0 + v.z;
    h[2] = v.y + m2;
    h[3] = m2 + right;
}

// Vertical 3-sums of h rows for the thread's VY rows (rows r-1 .. r+1,
// with `above` / `below` the rows outside the stack); consecutive rows share
// their middle pair.
template <int VY>
__device__ __forceinline__ void vsum(const float (&above)[VX], const float (&h)[VY][VX],
                                     const float (&below)[VX], float (&ps)[VY][VX]) {
#pragma unroll
    for (int cy = 0; cy < VY; cy += 2)
#pragma unroll
        for (int v = 0; v < VX; ++v) {
            if (cy + 1 < VY) {
                const float m = h[cy][v] + h[cy + 1][v];
                ps[cy][v] = (cy == 0 ? above[v] : h[cy - 1][v]) + m;
                ps[cy + 1][v] = m + (cy + 2 == VY ? below[v] : h[cy + 2][v]);
            } else {
                ps[cy][v] = ((cy == 0 ? above[v] : h[cy - 1][v]) + h[cy][v]) + below[v];
            }
        }
}

// One step (iteration parity PH): each level's plane sums alternate between
// two register slots (slot PH takes this step's P, slot PH^1 holds the
// previous one), and so do the raw planes kept for the next level's
// Dirichlet cells (read, then overwritten, in slot PH) — no moves.
template <int K, int SEL, int PH, typename G, bool MIRROR>
__device__ __forceinline__ void box_step(const BoxArgs& a, T* __restrict__ out, const T* ring,
                                         T* lev, uint64_t* bar, int& rslot, unsigned& rphase,
                                         int t, int i0, int i1, int lx, int x, int y,
                                         long long& ooff, const bool (&cint)[G::VY][VX],
                                         const bool (&cout)[G::VY][VX], bool hl,
                                         T (&acc)[K][2][G::VY][VX], T (&accB)[K][G::VY][VX],
                                         T (&hs)[K][G::VY][VX], T (&vr)[K][2][G::VY][VX]) {
    constexpr int VY = G::VY, STAGES = stages<K, G>();
    constexpr int SLOT = slot_bytes<G>() / (int)sizeof(T);
    constexpr int LEV = lev_bytes<G>() / (int)sizeof(T);
    const int slot = rslot;
    const int slot_m1 = slot >= 1 ? slot - 1 : slot + STAGES - 1;  // plane t-1
    const int ly2 = 2 * (y / VY);
    mbar_wait(&bar[slot], rphase);  // level-0 plane t

#pragma unroll
    for (int l = K; l >= 1; --l) {
        const int p = t - 2 * l + 1;  // plane level l produces now (source plane p+1)
        // ---- plane sum P of the consumed source plane c = p + 1 ----------
        T (&ps)[VY][VX] = acc[l - 1][PH];  // this step's P (slot PH^1: the previous one)
        if (l == 1) {
            const T* Pc = ring + slot * SLOT;
            float hh[VY][VX], hu[VX], hd[VX];
            {  // ring row y + r = region row y - 1 + r
                const T* row = Pc + y * BX0 + PL;
                hrow(*reinterpret_cast<const float4*>(row + x), row[-1], row[R1X], lx, hu);
            }
#pragma unroll
            for (int cy = 0; cy < VY; ++cy) {
                const T* row = Pc + (y + cy + 1) * BX0 + PL;
                hrow(*reinterpret_cast<const float4*>(row + x), row[-1], row[R1X], lx, hh[cy]);
            }
            {
                const T* row = Pc + (y + VY + 1) * BX0 + PL;
                hrow(*reinterpret_cast<const float4*>(row + x), row[-1], row[R1X], lx, hd);
            }
            vsum<VY>(hu, hh, hd, ps);
        } else {
            // own rows' h from registers (level l-1 produced plane c in the
            // previous step), the rows above / below from the other warps
            const T* L = lev + ((l - 2) * NB + ((p + 1) & 1)) * LEV;
            const float4 u = *reinterpret_cast<const float4*>(L + ly2 * R1X + x);
            const float4 d = *reinterpret_cast<const float4*>(L + (ly2 + 3) * R1X + x);
            const float uu[VX] = {u.x, u.y, u.z, u.w}, dd[VX] = {d.x, d.y, d.z, d.w};
            vsum<VY>(uu, hs[l - 2], dd, ps);
        }
        // ---- level-l plane p = w * ((P(p-1) + P(p)) + P(p+1)) ----------------
        T res[VY][VX];
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int v = 0; v < VX; ++v) {
                res[cy][v] = __fmul_rn(a.w, accB[l - 1][cy][v] + ps[cy][v]);
                accB[l - 1][cy][v] = acc[l - 1][PH ^ 1][cy][v] + ps[cy][v];
            }
        if (l < K) {
            if constexpr (SEL >= 3) {
                // a2-edge warp with every row interior: only the halo column
                // next to the interior (column HC of lane `hl`) keeps its
                // level-0 value; cells beyond it feed only it
                constexpr int HC = SEL - 3;
                if (hl) {
#pragma unroll
                    for (int cy = 0; cy < VY; ++cy)
                        res[cy][HC] = l == 1 ? ring[slot_m1 * SLOT + (y + cy + 1) * BX0 + PL + x + HC]
                                             : vr[l - 2][PH][cy][HC];
                }
            }
            // (plane t_begin-1 is never loaded: level 1's first product is
            // outside every cone, so it skips the ring read)
            if (SEL == 1 || SEL == 2) if (!(l == 1 && p < i0 - K)) {
                // Dirichlet: level-(l-1) raw value of plane p (= level 0)
                const bool pint = p >= 0 && p < a.n0;
#pragma unroll
                for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                    for (int v = 0; v < VX; ++v) {
                        if (pint && cint[cy][v]) continue;
                        res[cy][v] = l == 1 ? ring[slot_m1 * SLOT + (y + cy + 1) * BX0 + PL + x + v]
                                            : vr[l - 2][PH][cy][v];  // plane p, two steps back
                    }
            }
            // raw values for the next level's Dirichlet cells: read there two
            // steps from now, in the slot of this parity
            if (l + 1 < K) {
#pragma unroll
                for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                    for (int v = 0; v < VX; ++v) vr[l - 1][PH][cy][v] = res[cy][v];
            }
            // h of the new rows: kept for this warp, edge rows published
            T* L = lev + ((l - 1) * NB + (p & 1)) * LEV;
#pragma unroll
            for (int cy = 0; cy < VY; ++cy) {
                const float4 v4 = make_float4(res[cy][0], res[cy][1], res[cy][2], res[cy][3]);
                hrow(v4, 0.f, 0.f, lx, hs[l - 1][cy]);
                if (cy == 0 || cy == VY - 1)
                    *reinterpret_cast<float4*>(L + (ly2 + (cy == 0 ? 1 : 2)) * R1X + x) =
                        make_float4(hs[l - 1][cy][0], hs[l - 1][cy][1], hs[l - 1][cy][2],
                                    hs[l - 1][cy][3]);
            }
        } else if (SEL == 0 || SEL >= 3 || (p >= i0 && p < i1)) {  // clear tiers: in range
            T* o = out + ooff;
#pragma unroll
            for (int cy = 0; cy < VY; ++cy) {
                if constexpr (SEL == 0) {
                    if (cout[cy][0]) {  // lanes are wholly inside or outside the tile
                        *reinterpret_cast<float4*>(o + cy * a.pitch1) =
                            make_float4(res[cy][0], res[cy][1], res[cy][2], res[cy][3]);
                        if constexpr (MIRROR)
                            *reinterpret_cast<float4*>(a.mirror + (o - out) + a.mshift +
                                                       cy * a.pitch1) =
                                make_float4(res[cy][0], res[cy][1], res[cy][2], res[cy][3]);
                    }
                } else {
                    store_row<T, VX>(o + cy * a.pitch1, res[cy], cout[cy]);
                    if constexpr (MIRROR)
                        store_row<T, VX>(a.mirror + (o - out) + a.mshift + cy * a.pitch1, res[cy],
                                         cout[cy]);
                }
            }
        }
    }
    ooff += a.pitch0;
    if (slot == STAGES - 1) {
        rslot = 0;
        rphase ^= 1u;
    } else {
        rslot = slot + 1;
    }
}

template <int K, typename G, bool MIRROR>
__global__ void __launch_bounds__(G::NT, 1)
    tbbox_kernel(T* __restrict__ out, const __grid_constant__ CUtensorMap tmap,
                 const __grid_constant__ BoxArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int VY = G::VY, R1Y = G::R1Y;
    constexpr int STAGES = stages<K, G>();
    static_assert(STAGES >= 3, "the ring holds planes t-1 .. t+1 at least");
    constexpr int SLOT = slot_bytes<G>() / (int)sizeof(T);
    T* ring = reinterpret_cast<T*>(smem);
    T* lev = reinterpret_cast<T*>(smem + STAGES * slot_bytes<G>());
    uint64_t* bar =
        reinterpret_cast<uint64_t*>(smem + STAGES * slot_bytes<G>() + NB * (K - 1) * lev_bytes<G>());

    const int tid = threadIdx.x;
    const int lx = tid & 31, ly = tid >> 5;
    constexpr int TX = TXO<K>, TY = R1Y - 2 * (K - 1), HX = HXL<K>;
    constexpr unsigned kBoxBytes = BX0 * G::BY0 * sizeof(T);
    const int x = VX * lx, y = VY * ly;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&tmap);
    }
    __syncthreads();

    // aligned persistent schedule (tb3d.cu): whole tiles b, b+W, ... with
    // every CTA at the same plane, then an even share of the leftovers
    const long long span = a.hi0 - a.lo0;
    const int ntile = a.tiles_x * a.tiles_y;
    const int tile_rem0 = a.full_tiles * (int)gridDim.x;
    const long long total = (long long)(ntile - tile_rem0) * span;
    int full_left = a.full_tiles, full_tile = blockIdx.x;
    long long pos = (long long)blockIdx.x * a.per_cta;
    const long long end = min(pos + a.per_cta, total);
    unsigned gbase = 0;
    int rslot = 0;
    unsigned rphase = 0;
    T acc[K][2][VY][VX], accB[K][VY][VX], hs[K][VY][VX], vr[K][2][VY][VX];

    while (full_left > 0 || pos < end) {
        int tile, i0, i1;
        if (full_left > 0) {
            tile = full_tile;
            i0 = a.lo0;
            i1 = a.hi0;
            full_tile += gridDim.x;
            --full_left;
        } else {
            const int tt = (int)(pos / span);
            i0 = a.lo0 + (int)(pos - (long long)tt * span);
            i1 = (int)min((long long)a.hi0, (long long)i0 + (end - pos));
            pos += i1 - i0;
            tile = tile_rem0 + tt;
        }
        const int bx = tile % a.tiles_x, by = tile / a.tiles_x;
        const int gx = bx * TX - HX, gy = by * TY - (K - 1);
        // level-0 planes i0-K .. i1+K-1; level K produces plane t-2K+1 at
        // step t, so it finishes plane i1-1 at step i1+2K-2
        const int t_begin = i0 - K;
        const int niter = (i1 - i0) + 3 * K - 1;
        const int nload = i1 - i0 + 2 * K;

#pragma unroll
        for (int l = 0; l < K; ++l)
#pragma unroll
            for (int cy = 0; cy < VY; ++cy)
#pragma unroll
                for (int v = 0; v < VX; ++v) {
                    acc[l][0][cy][v] = acc[l][1][cy][v] = accB[l][cy][v] = hs[l][cy][v] = T(0);
                    vr[l][0][cy][v] = vr[l][1][cy][v] = T(0);
                }
        bool cint[VY][VX], cout[VY][VX];
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int v = 0; v < VX; ++v) {
                const int ga1 = gy + y + cy, ga2 = gx + x + v;
                cint[cy][v] = ga1 >= 0 && ga1 < a.n1 && ga2 >= 0 && ga2 < a.n2;
                cout[cy][v] = cint[cy][v] && y + cy >= K - 1 && y + cy < R1Y - (K - 1) &&
                              x + v >= HX && x + v < HX + TX;
            }
        const int c0 = a.off2 + gx - PL, c1 = a.h1 + gy - 1;
        long long ooff = a.origin + (long long)(gy + y) * a.pitch1 + (gx + x) +
                         (long long)(t_begin - 2 * K + 1) * a.pitch0;
        const int last_plane = a.h0 + t_begin + nload - 1;
        if (tid == 0) {  // every warp finished the previous segment (the last barrier)
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
            // plane t-1 was last read in this step: its slot takes t-1+STAGES
            // (rslot already names plane t+1's slot)
            if (tid == 0 && it >= 1 && it - 1 + STAGES < niter) {
                const int sl = rslot >= 2 ? rslot - 2 : rslot + STAGES - 2;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bar[sl], kBoxBytes);
                tma_load_3d(ring + sl * SLOT, &tmap, &bar[sl], c0, c1,
                            min(a.h0 + t_begin + it - 1 + STAGES, last_plane));
            }
        };
        bool mine = true;
#pragma unroll
        for (int cy = 0; cy < VY; ++cy)
#pragma unroll
            for (int v = 0; v < VX; ++v) mine &= cint[cy][v];
        const bool warp_int = __all_sync(0xffffffffu, mine);
        // a2-edge warps (the bulk of the boundary tiles): every row interior,
        // the only halo column read by interior cells (a2 = -1 or n2) in one
        // column slot HC of the lanes -> the one-column tier SEL = 3 + HC
        bool rows_in = true;
#pragma unroll
        for (int cy = 0; cy < VY; ++cy) rows_in &= gy + y + cy >= 0 && gy + y + cy < a.n1;
        const bool warp_rows = __all_sync(0xffffffffu, rows_in);
        int edge_hc = -1, nhc = 0;
#pragma unroll
        for (int v = 0; v < VX; ++v) {
            const bool h = gx + x + v == -1 || gx + x + v == a.n2;
            if (__any_sync(0xffffffffu, h)) {
                edge_hc = v;
                ++nhc;
            }
        }
        if (warp_int || !warp_rows || nhc != 1) edge_hc = -1;
        const bool hl = edge_hc >= 0 && (gx + x + edge_hc == -1 || gx + x + edge_hc == a.n2);
        // select-free steps: every plane the levels below K produce is
        // interior (t-2K+3 .. t-1) and level K's plane (t-2K+1) is one of
        // this segment's outputs
        auto clear = [&](int it) {
            const int t = t_begin + it;
            return t - 2 * K + 3 >= 0 && t - 1 < a.n0 && it >= 3 * K - 1 &&
                   it < 3 * K - 1 + (i1 - i0);
        };
#define TBBOX_STEP(IT, SEL, PH)                                                              \
    box_step<K, SEL, PH, G, MIRROR>(a, out, ring, lev, bar, rslot, rphase, t_begin + (IT), i0, i1, \
                                    lx, x, y, ooff, cint, cout, hl, acc, accB, hs, vr);       \
    after(IT);
#define TBBOX_CLEAR_LOOP(SEL)                                                                \
    for (; it < niter && pair_clear(it); it += 2) {                                           \
        TBBOX_STEP(it, SEL, 0)                                                               \
        TBBOX_STEP(it + 1, SEL, 1)                                                           \
    }
        // pairs of steps (the parity selects the register slots); the clear
        // pairs form one interval, so the tier is chosen once per segment
        auto pair_clear = [&](int it) { return clear(it) && clear(it + 1); };
        int it = 0;
        for (; it < niter && !pair_clear(it); it += 2) {
            TBBOX_STEP(it, 2, 0)
            if (it + 1 < niter) {
                TBBOX_STEP(it + 1, 2, 1)
            }
        }
        // (clear implies it + 1 < niter)
        if (warp_int) {
            TBBOX_CLEAR_LOOP(0)
        } else if (!MIRROR) {  // the seam-pass instance keeps the general tier
            switch (edge_hc) {
                case 0: TBBOX_CLEAR_LOOP(3) break;
                case 1: TBBOX_CLEAR_LOOP(4) break;
                case 2: TBBOX_CLEAR_LOOP(5) break;
                case 3: TBBOX_CLEAR_LOOP(6) break;
                default: break;
            }
        }
        for (; it < niter; it += 2) {
            TBBOX_STEP(it, 2, 0)
            if (it + 1 < niter) {
                TBBOX_STEP(it + 1, 2, 1)
            }
        }
#undef TBBOX_CLEAR_LOOP
#undef TBBOX_STEP
        gbase += niter;
    }
}

constexpr int kMaxK = 4;

bool supports(const Geo& g, const TapSet& t, bool exact) {
    if (exact || g.dtype != TSR_F32) return false;
    if (t.dims != 3 || t.shape != TSR_BOX || t.radius != 1 || t.ntaps != 27) return false;
    if (!uniform_weights(t)) return false;
    if (g.n[0] + 2 * g.h[0] > (1 << 30) || g.n[1] + 2 * g.h[1] > (1 << 30)) return false;
    return true;
}

template <int K, typename G>
Status launch_k(const LaunchCtx& c, const void* in, void* out) {
    const Geo& g = *c.g;
    CUtensorMap map;
    Status s = make_tmap_3d<T>(g, in, BX0, G::BY0, &map);
    if (!s.ok()) return s;
    BoxArgs a;
    a.n0 = (int)g.n[0];
    a.n1 = (int)g.n[1];
    a.n2 = (int)g.n[2];
    constexpr int TX = TXO<K>, TY = G::R1Y - 2 * (K - 1);
    a.tiles_x = (int)((g.n[2] + TX - 1) / TX);
    a.tiles_y = (int)((g.n[1] + TY - 1) / TY);
    const long long tiles = (long long)a.tiles_x * a.tiles_y;
    constexpr int bytes = smem_bytes<K, G>();
    int per_sm = 1, nsm = 148;
    s = occupancy(tbbox_kernel<K, G, false>, G::NT, bytes, &per_sm, &nsm);
    if (!s.ok()) return s;
    a.lo0 = (int)c.range_lo();
    a.hi0 = (int)c.range_hi();
    if (a.hi0 <= a.lo0) return Status::Ok();
    const long long span = a.hi0 - a.lo0;
    const long long slots = (long long)nsm * per_sm;
    unsigned grid;
    a.full_tiles = 0;
    if (tiles >= slots) {
        grid = (unsigned)slots;
        a.full_tiles = (int)(tiles / slots);
        const long long left = tiles - (long long)a.full_tiles * slots;
        a.per_cta = left * 100 >= slots * 85 ? span : (left * span + slots - 1) / slots;
    } else if (tiles * 10 >= slots * 9) {
        grid = (unsigned)tiles;
        a.full_tiles = 1;
        a.per_cta = 0;
    } else {
        const long long total = tiles * span;
        const long long ctas = std::min<long long>(slots, total);
        a.per_cta = (total + ctas - 1) / ctas;
        grid = (unsigned)((total + a.per_cta - 1) / a.per_cta);
    }
    a.h0 = (int)g.h[0];
    a.h1 = (int)g.h[1];
    a.off2 = (int)g.off2;
    a.pitch0 = g.pitch[0];
    a.pitch1 = g.pitch[1];
    a.origin = g.origin;
    a.mirror = static_cast<T*>(c.mirror);
    a.mshift = c.mirror_shift;
    a.w = static_cast<T>(c.taps->w[0]);
    if (c.mirror) {
        static bool attr_set[64] = {};  // per device, once
        int dev = 0;
        TSR_CUDA_TRY(cudaGetDevice(&dev));
        if (dev >= 64 || !attr_set[dev]) {
            TSR_CUDA_TRY(cudaFuncSetAttribute(tbbox_kernel<K, G, true>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            if (dev < 64) attr_set[dev] = true;
        }
        tbbox_kernel<K, G, true><<<grid, G::NT, bytes, c.stream>>>(static_cast<T*>(out), map, a);
    } else {
        tbbox_kernel<K, G, false><<<grid, G::NT, bytes, c.stream>>>(static_cast<T*>(out), map, a);
    }
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

using ShapeB = Shape<2, 28>;  // 448 threads, 128 x 28 level-1 region (k <= 2)

}  // namespace

// Entry point used by the box3d engine for FAST uniform boxes in fp32.
bool tbbox_supports(const Geo& g, const TapSet& t, bool exact) { return supports(g, t, exact); }

// k = 3 runs 384 threads (a 128 x 24 region) so each may hold 168
// registers: 1238 GS/s on C4 against 1020 for 448 threads capped at 128
// registers (the allocation granularity is four warps).  k <= 2 fit 128.
using ShapeC = Shape<2, 24>;

Status tbbox_run(const LaunchCtx& c, const void* in, void* out, int k) {
    switch (k) {
        case 1: return launch_k<1, ShapeB>(c, in, out);
        case 2: return launch_k<2, ShapeB>(c, in, out);
        case 3: return launch_k<3, ShapeC>(c, in, out);
        case 4: return launch_k<4, ShapeC>(c, in, out);
        default: return Status::Err(TSR_EUNSUPPORTED, "tbbox: fused steps must be 1..4");
    }
}

}  // namespace tsr
