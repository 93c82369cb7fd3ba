/*
 * oracle.c — CPU restatement of the reference stencil sweep.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_2303_08365_b200/) may link, load or call this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * use it, and only as the checker.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function here
 * bitwise against (a) the reference library compiled from
 * /root/reference/proj/src by oracle/Makefile into oracle/_ref/, and (b) the
 * golden fixtures under tests/golden/ (one of which, star2d9p_64x64_t12.ttrs,
 * is written by the reference's own gen_golden tool).
 *
 * Compiled with -ffp-contract=off, exactly like the reference
 * (proj/CMakeLists.txt:35-38), so the sums below are never fused into FMAs.
 *
 * Layout (proj/include/tessera/grid.hpp:26-58): row-major, axis 0 outermost,
 * last axis contiguous, every axis padded by its halo on both sides;
 * stride[dims-1] = 1, stride[a] = stride[a+1] * (extent[a+1] + 2*halo[a+1]).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ---------------------------------------------------------------------- */
/* std::mt19937_64, restated (the reference seeds inputs with it:           */
/* proj/include/tessera/random.hpp:13-24).  Parameters are the C++11        */
/* standard's: w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9 u=29               */
/* d=0x5555555555555555 s=17 b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000  */
/* l=43 f=6364136223846793005.                                               */
/* ---------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156

typedef struct {
    uint64_t mt[MT_N];
    int idx;
} orc_mt64;

static void mt64_seed(orc_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = MT_N;
}

static uint64_t mt64_next(orc_mt64* s) {
    if (s->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) |
                               (s->mt[(i + 1) % MT_N] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + MT_M) % MT_N] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* First `count` raw outputs of mt19937_64(seed); used to pin the generator. */
void orc_mt64_stream(uint64_t seed, int64_t count, uint64_t* out) {
    orc_mt64 s;
    mt64_seed(&s, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = mt64_next(&s);
}

/* ---------------------------------------------------------------------- */
/* Grid geometry helpers                                                    */
/* ---------------------------------------------------------------------- */
typedef struct {
    int dims;
    int64_t ext[3];
    int64_t halo[3];
    int64_t stride[3];
} geom;

static void make_geom(geom* g, int dims, const int64_t* ext, const int64_t* halo) {
    g->dims = dims;
    for (int a = 0; a < 3; ++a) {
        g->ext[a] = a < dims ? ext[a] : 1;
        g->halo[a] = a < dims ? halo[a] : 0;
        g->stride[a] = 0;
    }
    g->stride[dims - 1] = 1;
    for (int a = dims - 2; a >= 0; --a)
        g->stride[a] = g->stride[a + 1] * (g->ext[a + 1] + 2 * g->halo[a + 1]);
}

/* grid.hpp:73-78 */
static int64_t flat(const geom* g, int64_t i, int64_t j, int64_t k) {
    int64_t f = (i + g->halo[0]) * g->stride[0];
    if (g->dims > 1) f += (j + g->halo[1]) * g->stride[1];
    if (g->dims > 2) f += (k + g->halo[2]) * g->stride[2];
    return f;
}

/* ---------------------------------------------------------------------- */
/* fill_random (random.hpp:20-24): interior only, for_each_interior order  */
/* i -> j -> k, value = (T)(lo + (hi - lo) * ((rng() >> 11) * 2^-53)),     */
/* written to both buffers; halo untouched.                                 */
/* ---------------------------------------------------------------------- */
#define DEFINE_FILL(T, SUFFIX)                                                                  \
    void orc_fill_random_##SUFFIX(int dims, const int64_t* ext, const int64_t* halo,            \
                                  uint64_t seed, double lo, double hi, T* buf0, T* buf1) {      \
        geom g;                                                                                 \
        make_geom(&g, dims, ext, halo);                                                         \
        orc_mt64 s;                                                                             \
        mt64_seed(&s, seed);                                                                    \
        for (int64_t i = 0; i < g.ext[0]; ++i)                                                  \
            for (int64_t j = 0; j < g.ext[1]; ++j)                                              \
                for (int64_t k = 0; k < g.ext[2]; ++k) {                                        \
                    const double u = (double)(mt64_next(&s) >> 11) * 0x1.0p-53;                 \
                    const T v = (T)(lo + (hi - lo) * u);                                        \
                    const int64_t f = flat(&g, i, j, k);                                        \
                    buf0[f] = v;                                                                \
                    buf1[f] = v;                                                                \
                }                                                                               \
    }
DEFINE_FILL(double, f64)
DEFINE_FILL(float, f32)

/* ---------------------------------------------------------------------- */
/* apply_box (naive.hpp:41-84): one Jacobi sweep over box [lo, hi) clipped */
/* to the interior; reads `in`, writes `out`.  acc starts at 0 and adds   */
/* w[t]*in[p+delta[t]] in the given (canonical lexicographic) tap order,  */
/* weights cast to T first.  Returns the number of point updates.          */
/* Rows (i, j) are independent, so large boxes are split over host threads */
/* (ORC_THREADS, default all cores); every point's sum is computed exactly */
/* as in the serial loop, so the result is bit-identical.                  */
/* ---------------------------------------------------------------------- */
#define MAX_TAPS 4096

static int orc_threads(int64_t points) {
    if (points < (1 << 20)) return 1;
    const char* e = getenv("ORC_THREADS");
    long n = e ? strtol(e, NULL, 10) : sysconf(_SC_NPROCESSORS_ONLN);
    if (n < 1) n = 1;
    if (n > 256) n = 256;
    return (int)n;
}

#define DEFINE_APPLY(T, SUFFIX)                                                                   \
    typedef struct {                                                                              \
        const geom* g;                                                                            \
        const int64_t *lo, *hi, *delta;                                                           \
        const T* w;                                                                               \
        int ntaps;                                                                                \
        const T* in;                                                                              \
        T* out;                                                                                   \
        int64_t r0, r1; /* flattened (i, j) rows */                                               \
    } rows_##SUFFIX;                                                                              \
    static void* apply_rows_##SUFFIX(void* p) {                                                   \
        const rows_##SUFFIX* a = (const rows_##SUFFIX*)p;                                         \
        const int64_t nj = a->hi[1] - a->lo[1];                                                   \
        const int64_t n = a->hi[2] - a->lo[2];                                                    \
        for (int64_t r = a->r0; r < a->r1; ++r) {                                                 \
            const int64_t i = a->lo[0] + r / nj, j = a->lo[1] + r % nj;                           \
            const int64_t base = flat(a->g, i, j, a->lo[2]);                                      \
            const T* irow = a->in + base;                                                         \
            T* orow = a->out + base;                                                              \
            for (int64_t c = 0; c < n; ++c) {                                                     \
                T acc = (T)0;                                                                     \
                for (int t = 0; t < a->ntaps; ++t) acc += a->w[t] * irow[c + a->delta[t]];        \
                orow[c] = acc;                                                                    \
            }                                                                                     \
        }                                                                                         \
        return NULL;                                                                              \
    }                                                                                             \
    int64_t orc_apply_box_##SUFFIX(int dims, const int64_t* ext, const int64_t* halo, int ntaps,   \
                                   const int32_t* offsets, const double* weights,                 \
                                   const int64_t* box_lo, const int64_t* box_hi, const T* in,     \
                                   T* out) {                                                      \
        if (ntaps < 0 || ntaps > MAX_TAPS) return -1;                                             \
        geom g;                                                                                   \
        make_geom(&g, dims, ext, halo);                                                           \
        int64_t lo[3], hi[3];                                                                     \
        for (int a = 0; a < 3; ++a) {                                                             \
            if (a < dims) {                                                                       \
                lo[a] = box_lo[a] > 0 ? box_lo[a] : 0;                                            \
                hi[a] = box_hi[a] < g.ext[a] ? box_hi[a] : g.ext[a];                              \
                if (lo[a] >= hi[a]) return 0;                                                     \
            } else {                                                                              \
                lo[a] = 0;                                                                        \
                hi[a] = 1;                                                                        \
            }                                                                                     \
        }                                                                                         \
        int64_t delta[MAX_TAPS];                                                                  \
        T w[MAX_TAPS];                                                                            \
        for (int t = 0; t < ntaps; ++t) {                                                         \
            int64_t d = 0;                                                                        \
            for (int a = 0; a < dims; ++a) d += (int64_t)offsets[3 * t + a] * g.stride[a];        \
            delta[t] = d;                                                                         \
            w[t] = (T)weights[t];                                                                 \
        }                                                                                         \
        const int64_t rows = (hi[0] - lo[0]) * (hi[1] - lo[1]);                                   \
        const int nt = orc_threads(rows * (hi[2] - lo[2]));                                       \
        rows_##SUFFIX job[256];                                                                   \
        pthread_t th[256];                                                                        \
        for (int q = 0; q < nt; ++q) {                                                            \
            rows_##SUFFIX a = {&g, lo, hi, delta, w, ntaps, in, out, rows * q / nt,               \
                               rows * (q + 1) / nt};                                              \
            job[q] = a;                                                                           \
        }                                                                                         \
        int live[256] = {0};                                                                      \
        for (int q = 1; q < nt; ++q)                                                              \
            live[q] = pthread_create(&th[q], NULL, apply_rows_##SUFFIX, &job[q]) == 0;            \
        for (int q = 0; q < nt; ++q) /* this thread's share, and any that did not start */        \
            if (!live[q]) apply_rows_##SUFFIX(&job[q]);                                            \
        for (int q = 1; q < nt; ++q)                                                              \
            if (live[q]) pthread_join(th[q], NULL);                                               \
        return rows * (hi[2] - lo[2]);                                                            \
    }
DEFINE_APPLY(double, f64)
DEFINE_APPLY(float, f32)

/* naive_run (naive.hpp:89-100): `steps` full-interior sweeps, alternating  */
/* buffers starting from read parity `parity`.  Returns the final parity.   */
#define DEFINE_RUN(T, SUFFIX)                                                                     \
    int orc_naive_run_##SUFFIX(int dims, const int64_t* ext, const int64_t* halo, int ntaps,       \
                               const int32_t* offsets, const double* weights, T* buf0, T* buf1,   \
                               int parity, int64_t steps) {                                       \
        if (steps < 0) return -1;                                                                 \
        const int64_t lo[3] = {0, 0, 0};                                                          \
        const int64_t hi[3] = {ext[0], dims > 1 ? ext[1] : 1, dims > 2 ? ext[2] : 1};             \
        T* buf[2] = {buf0, buf1};                                                                 \
        for (int64_t s = 0; s < steps; ++s) {                                                     \
            orc_apply_box_##SUFFIX(dims, ext, halo, ntaps, offsets, weights, lo, hi, buf[parity],  \
                                   buf[1 - parity]);                                              \
            parity ^= 1;                                                                          \
        }                                                                                         \
        return parity;                                                                            \
    }
DEFINE_RUN(double, f64)
DEFINE_RUN(float, f32)

/* ---------------------------------------------------------------------- */
/* Metrics (proj/src/metrics.cpp:22-39) on the read buffers of two grids of */
/* identical geometry: max|a-b| / max(1, max|ref|) over the interior.      */
/* Also max-abs and L2-relative, which the reference lacks.                */
/* ---------------------------------------------------------------------- */
#define DEFINE_DEV(T, SUFFIX)                                                                     \
    void orc_deviation_##SUFFIX(int dims, const int64_t* ext, const int64_t* halo, const T* a,     \
                                const T* ref, double* out3) {                                     \
        geom g;                                                                                   \
        make_geom(&g, dims, ext, halo);                                                           \
        double mref = 0.0, dev = 0.0, se = 0.0, sr = 0.0;                                         \
        for (int64_t i = 0; i < g.ext[0]; ++i)                                                    \
            for (int64_t j = 0; j < g.ext[1]; ++j)                                                \
                for (int64_t k = 0; k < g.ext[2]; ++k) {                                          \
                    const int64_t f = flat(&g, i, j, k);                                          \
                    const double r = (double)ref[f], x = (double)a[f];                            \
                    const double d = fabs(x - r);                                                 \
                    if (fabs(r) > mref) mref = fabs(r);                                           \
                    if (d > dev || d != d) dev = d != d ? INFINITY : (d > dev ? d : dev);         \
                    se += (x - r) * (x - r);                                                      \
                    sr += r * r;                                                                  \
                }                                                                                 \
        out3[0] = dev / (mref > 1.0 ? mref : 1.0); /* max_rel_deviation */                        \
        out3[1] = dev;                             /* max abs error */                            \
        out3[2] = sr > 0.0 ? sqrt(se / sr) : sqrt(se); /* L2-relative */                          \
    }
DEFINE_DEV(double, f64)
DEFINE_DEV(float, f32)
