/*
 * tessera_b200.h — C-ABI of the B200-native Jacobi stencil sweep.
 *
 * This is the drop-in boundary for the reference's sweep loop.  The reference
 * (arXiv 2303.08365 artifact, namespace tessera) runs every time step through
 * apply_box (proj/include/tessera/naive.hpp:41-84), driven by
 *   naive_run       (proj/include/tessera/naive.hpp:96-100)      -> tsr_run, k = 1
 *   run_tessellated (proj/src/tiling.cpp:137-184)                -> tsr_run, k = plan.tb
 *   run_heterogeneous's HaloWorker rounds (proj/src/scheduler.cpp:371-406)
 *                                                                -> tsr_advance per slab
 * and seeds inputs with fill_random (proj/include/tessera/random.hpp:20-24)
 * -> tsr_fill_random.  The reference's pybind11 seam that a maintainer would
 * re-point is proj/bindings/module.cpp:164-202; its C++ seam is execute_path
 * (proj/src/bench.cpp:153-190).  INTEGRATION.md shows both bindings.
 *
 * Only plain C types cross this boundary.  Host buffers use the reference's
 * own BasicGrid<T> layout (proj/include/tessera/grid.hpp:46-49): row-major,
 * axis 0 outermost, every axis padded by its halo, last axis contiguous.
 * Device buffers use the pitched layout reported by tsr_layout_of().
 *
 * Every entry point returns TSR_OK (0) or an error code; tsr_last_error()
 * returns the calling thread's last message.  Error codes follow the
 * reference's exception classes: TSR_EINVAL <-> std::invalid_argument.
 */
#ifndef TESSERA_B200_H
#define TESSERA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSR_ABI_VERSION 1

enum tsr_status {
    TSR_OK = 0,
    TSR_EINVAL = 1,      /* invalid argument (reference: std::invalid_argument) */
    TSR_ECUDA = 2,       /* CUDA runtime / launch error (std::runtime_error)      */
    TSR_ENCCL = 3,       /* reserved for the collective layer                     */
    TSR_ENOMEM = 4,      /* device or pinned-host allocation failed               */
    TSR_EUNSUPPORTED = 5 /* valid request this build cannot serve                 */
};

enum tsr_dtype { TSR_F64 = 0, TSR_F32 = 1 };
enum tsr_shape { TSR_STAR = 0, TSR_BOX = 1 }; /* KernelShape, kernel.hpp:17 */
enum tsr_mode {
    TSR_EXACT = 0, /* no FMA, oracle tap order: bitwise equal to naive_run   */
    TSR_FAST = 1   /* FMA in oracle tap order: within 1e-12 / 1e-5 of it      */
};
enum tsr_engine {
    TSR_ENGINE_AUTO = 0,    /* tuned engine when one exists for the kernel   */
    TSR_ENGINE_GENERIC = 1, /* one thread per point, any dims/shape/radius   */
    TSR_ENGINE_TUNED = 2    /* require a tuned engine (TSR_EUNSUPPORTED if none) */
};

/* StencilKernel (kernel.hpp:26-51): taps in canonical lexicographic order. */
typedef struct tsr_kernel {
    int32_t dims;           /* 1..3                                          */
    int32_t shape;          /* tsr_shape                                     */
    int32_t radius;         /* >= 1                                          */
    int32_t ntaps;          /* lattice size for (dims, shape, radius)        */
    const int32_t* offsets; /* ntaps x 3 ints, components >= dims are zero   */
    const double* weights;  /* ntaps fp64 weights (cast to the grid type)    */
} tsr_kernel;

/* BasicGrid<T> geometry (grid.hpp:29-52). */
typedef struct tsr_grid {
    int32_t dims;      /* 1..3                                               */
    int32_t dtype;     /* tsr_dtype                                          */
    int64_t extent[3]; /* interior extent per axis (unused axes ignored)     */
    int64_t halo[3];   /* halo width per axis (>= kernel radius)             */
} tsr_grid;

/* Device layout of one buffer (both buffers share it). */
typedef struct tsr_layout {
    int64_t pitch[3];  /* element stride per grid axis                       */
    int64_t origin;    /* element offset of interior cell (0,0,0)            */
    int64_t elements;  /* elements to allocate per buffer                    */
} tsr_layout;

typedef struct tsr_opts {
    int32_t fused_steps; /* k: time steps fused per HBM pass (0 = auto)      */
    int32_t mode;        /* tsr_mode                                         */
    int32_t engine;      /* tsr_engine                                       */
    int32_t device;      /* CUDA ordinal for tsr_run (-1 = current device)   */
} tsr_opts;

typedef struct tsr_stats {
    double device_ms;        /* CUDA-event time of the sweep launches        */
    int64_t point_updates;   /* interior points x steps (TessellateStats)    */
    int64_t rounds;          /* fused rounds of k steps                      */
    int64_t trailing_steps;  /* steps run outside full k-step rounds         */
    int64_t kernel_launches; /* sweep kernels launched                       */
    int64_t h2d_bytes;       /* host->device bytes moved (tsr_run)           */
    int64_t d2h_bytes;       /* device->host bytes moved (tsr_run)           */
    int32_t fused_steps;     /* k actually used                              */
    int32_t engine;          /* tsr_engine actually used (1 or 2)            */
} tsr_stats;

/* ---- library ---------------------------------------------------------- */
int tsr_abi_version(void);
const char* tsr_last_error(void);
/* Frees the device buffers tsr_run caches between calls. */
int tsr_release_cache(void);

/* ---- host-side helpers (no GPU) ------------------------------------- */
/* Validates a kernel against the exact (dims, shape, radius) lattice and the
 * canonical order, as make_kernel does (proj/src/kernel.cpp:78-116). */
int tsr_check_kernel(const tsr_kernel* k);
/* fill_random (random.hpp:20-24): std::mt19937_64(seed), interior only, both
 * buffers, value (T)(lo + (hi-lo) * ((rng()>>11) * 2^-53)). */
int tsr_fill_random(const tsr_grid* g, void* buf0, void* buf1, uint64_t seed, double lo,
                    double hi);
int tsr_layout_of(const tsr_grid* g, tsr_layout* out);

/* ---- one-call host-buffer path: naive_run / run_tessellated drop-in ---
 * Advances the grid `steps` time steps on the GPU.  buf0/buf1 are the two
 * host buffers of a BasicGrid<T>, `parity` its read buffer.  On return the
 * buffers are exactly as naive_run leaves them: buffer(parity ^ (steps&1))
 * holds step T, the other buffer holds step T-1, halo cells untouched.  The
 * caller flips its parity `steps` times.  Requires the halo cells of both
 * buffers to be equal (every reference constructor guarantees it).  Pinned
 * host buffers make the copies run at full PCIe rate. */
int tsr_run(const tsr_kernel* k, const tsr_grid* g, void* buf0, void* buf1, int32_t parity,
            int64_t steps, const tsr_opts* opts, tsr_stats* stats);

/* ---- device-resident path (buffers in the tsr_layout_of layout) ----- */
/* `stream` is a cudaStream_t (NULL = legacy default stream). */
int tsr_upload(const tsr_grid* g, const tsr_layout* l, const void* host, void* dev,
               void* stream);
int tsr_download(const tsr_grid* g, const tsr_layout* l, const void* dev, void* host,
                 int32_t interior_only, void* stream);
/* Copies the halo shell of `src` into `dst` (device buffers). */
int tsr_copy_halo(const tsr_grid* g, const tsr_layout* l, const void* src, void* dst,
                  void* stream);
/* Advances `steps` time steps on device buffers dev[0]/dev[1]; *cur names the
 * buffer holding the current step and is updated.  keep_previous != 0 makes
 * the other buffer hold step T-1 on return (naive_run's post-condition);
 * otherwise its interior is scratch.  Launches are asynchronous on `stream`;
 * stats->device_ms is left 0. */
int tsr_advance(const tsr_kernel* k, const tsr_grid* g, const tsr_layout* l, void* dev0,
                void* dev1, int32_t* cur, int64_t steps, int32_t keep_previous,
                const tsr_opts* opts, void* stream, tsr_stats* stats);
/* One fused pass of `steps` (1..k of tsr_query_plan) time steps from `in` to
 * `out` that stores only the planes [lo, hi) of the grid's axis 0 (interior
 * coordinates); every other cell of `out` is left untouched.  Inputs are read
 * from all planes of `in` the dependency cone needs (r*steps planes beyond
 * the range, halo included).  This is HaloWorker::step_range
 * (proj/src/scheduler.cpp:352-356) for a slab decomposition: the interior
 * planes of a slab are launched while its ghost planes are still in flight
 * and the seam planes after they land. */
int tsr_sweep_range(const tsr_kernel* k, const tsr_grid* g, const tsr_layout* l, const void* in,
                    void* out, int64_t lo, int64_t hi, int32_t steps, const tsr_opts* opts,
                    void* stream);
/* tsr_sweep_range whose stores are also written to `mirror` (a buffer in the
 * same layout, normally a neighbour slab's buffer mapped by tsr_ipc_open) at
 * axis-0 plane p + mirror_planes: the seam pass of a slab round delivers its
 * planes straight into the neighbour's ghost planes over NVLink, replacing
 * SlabChannel's per-round message (proj/src/scheduler.cpp:142-194, 371-406).
 * mirror == NULL is tsr_sweep_range. */
int tsr_sweep_range_mirror(const tsr_kernel* k, const tsr_grid* g, const tsr_layout* l,
                           const void* in, void* out, int64_t lo, int64_t hi, int32_t steps,
                           const tsr_opts* opts, void* mirror, int64_t mirror_planes,
                           void* stream);

/* ---- peer-memory transport (one process per GPU) ---------------------- */
/* CUDA IPC handle of the allocation that contains `ptr` (any device pointer,
 * e.g. a torch tensor's data) and ptr's byte offset inside it. */
typedef struct tsr_ipc_handle {
    unsigned char bytes[64];
} tsr_ipc_handle;
int tsr_ipc_export(const void* ptr, tsr_ipc_handle* handle, int64_t* offset);
/* Maps another process's allocation (peer access enabled lazily); *base is
 * the allocation's base in this process.  tsr_ipc_close unmaps it. */
int tsr_ipc_open(const tsr_ipc_handle* handle, void** base);
int tsr_ipc_close(void* base);
/* Stream-ordered round flags: tsr_peer_signal stores `value` to a 32-bit
 * word (local or peer-mapped) with system-scope release once all earlier
 * work on `stream` is complete; tsr_peer_wait holds back later work on
 * `stream` until the word reaches `value` (wrap-around compare). */
int tsr_peer_signal(void* flag, uint32_t value, void* stream);
int tsr_peer_wait(const void* flag, uint32_t value, void* stream);
/* Round-counting forms for graph-captured rounds (no per-round arguments):
 * `counter` (local) holds the rounds this rank has completed.
 * tsr_peer_round_wait holds `stream` until each non-NULL local flag word
 * (rounds completed by the lo / hi neighbour) reaches *counter;
 * tsr_peer_round_signal increments *counter and stores it, system-scope
 * release, into each non-NULL peer-mapped flag word. */
int tsr_peer_round_wait(const void* flag_lo, const void* flag_hi, const void* counter,
                        void* stream);
int tsr_peer_round_signal(void* peer_lo, void* peer_hi, void* counter, void* stream);

/* Reports the engine (tsr_engine) and fused step count k tsr_advance /
 * tsr_run would use for this kernel, grid and opts (no device work). */
int tsr_query_plan(const tsr_kernel* k, const tsr_grid* g, const tsr_opts* opts,
                   int32_t* engine, int32_t* fused_steps);
/* One sweep of the box [lo, hi) (interior coordinates, clipped) from `in` to
 * `out`: apply_box (naive.hpp:41-84) on device buffers. */
int tsr_apply_box(const tsr_kernel* k, const tsr_grid* g, const tsr_layout* l, const void* in,
                  void* out, const int64_t* lo, const int64_t* hi, const tsr_opts* opts,
                  void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TESSERA_B200_H */
