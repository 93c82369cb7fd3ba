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

#define TSR_ABI_VERSION 3

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
    int32_t ngpus;       /* tsr_run: slabs / GPUs (0 or 1 = one device); >1
                            runs tsr_run_multi with an equal split over
                            devices 0..ngpus-1 (PartitionPlan, scheduler.hpp:49-64) */
    int32_t split_axis;  /* slab axis; only 0 (the reference's split_axis)  */
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
    /* slab runs (CommLog, scheduler.hpp:75-89); zero on one device          */
    int64_t bytes_exchanged;        /* halo bytes delivered to neighbours    */
    int64_t messages;               /* per-round seam deliveries             */
    int64_t ghost_recompute_points; /* HaloWorker::tally_ghost's count       */
    int32_t ngpus;                  /* slabs the run used                    */
    int32_t transport;              /* tsr_transport actually used          */
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
/* The same after discarding the first `skip` draws: a slab whose interior is
 * planes [p, p + n) of a global grid gets the global stream's values with
 * skip = p * (interior cells per plane). */
int tsr_fill_random_at(const tsr_grid* g, void* buf0, void* buf1, uint64_t seed, double lo,
                       double hi, uint64_t skip);
/* The thermal case study's initial plate (proj/src/case_study.cpp:193-207):
 * ambient everywhere, interior cell (i, j) = ambient + (peak - ambient) *
 * exp(-((i-c0)^2 + (j-c0)^2) / (2 sigma^2)), c0 = (n-1)/2 per axis, computed
 * in double (std::exp) and cast to the grid type; both buffers; 2-D only. */
int tsr_fill_plate(const tsr_grid* g, void* buf0, void* buf1, double ambient, double peak,
                   double sigma);
int tsr_layout_of(const tsr_grid* g, tsr_layout* out);

/* ---- one-call host-buffer path: naive_run / run_tessellated drop-in ---
 * Advances the grid `steps` time steps on the GPU.  buf0/buf1 are the two
 * host buffers of a BasicGrid<T>, `parity` its read buffer.  On return the
 * buffers are exactly as naive_run leaves them: buffer(parity ^ (steps&1))
 * holds step T, the other buffer holds step T-1, halo cells untouched.  The
 * caller flips its parity `steps` times.  When the halo cells of the two
 * buffers are equal (every reference constructor guarantees it) one buffer
 * is uploaded and the steps are fused; when they differ, both buffers are
 * uploaded and every step is its own sweep reading its read buffer's halo,
 * as naive_run does (stats->fused_steps = 1).  Pinned host buffers make the
 * copies run at full PCIe rate. */
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

/* ---- memory-level tetrominoes: slab decomposition over GPUs ---------
 * The reference splits axis 0 between two workers with a deep halo of
 * r*tb rows and one exchange per direction per tb-step round
 * (run_heterogeneous, proj/src/scheduler.cpp:441-563; PartitionPlan,
 * proj/include/tessera/scheduler.hpp:49-64).  Here one host thread drives
 * `ngpus` slabs, one per GPU (several may share a device), each holding its
 * owned planes plus r*k ghost planes per seam.  A round of n <= k fused
 * steps per slab is: seam passes (the r*k boundary planes, storing each
 * output row locally AND into the neighbour's next-buffer ghost planes over
 * NVLink peer memory, TSR_XPORT_MIRROR) on one stream, concurrently with the
 * interior pass on a second stream; ordering across slabs is by CUDA events
 * (a slab's seam pass of round n waits for its neighbours' of round n-1).
 * TSR_XPORT_COPY stores locally and moves the planes with
 * cudaMemcpyPeerAsync (the path when peer access is unavailable). */
enum tsr_transport { TSR_XPORT_AUTO = 0, TSR_XPORT_MIRROR = 1, TSR_XPORT_COPY = 2 };

typedef struct tsr_partition {
    int32_t ngpus;              /* slabs (>= 1)                                */
    int32_t split_axis;         /* must be 0                                   */
    const int32_t* devices;     /* ngpus CUDA ordinals; NULL = i mod count     */
    const int64_t* boundaries;  /* ngpus-1 ascending axis-0 boundaries (slab i
                                   owns [b[i-1], b[i])); NULL = equal split    */
    int32_t transport;          /* tsr_transport                               */
    int32_t flags;              /* TSR_PART_POISON: NaN in every slab's
                                   seam-side halo planes (beyond the ghosts)
                                   after each upload, proving they are never
                                   read (run_heterogeneous_instrumented,
                                   scheduler.hpp:115-124)                     */
} tsr_partition;
#define TSR_PART_POISON 1

typedef struct tsr_multi tsr_multi; /* opaque slab set */

typedef struct tsr_slab_info {
    int32_t device;
    int32_t cur;           /* buffer holding the current step                */
    int64_t own_lo, own_hi;/* owned global interior planes [lo, hi)          */
    int64_t ghost_lo, ghost_hi; /* ghost planes below / above the owned ones */
    tsr_grid grid;         /* the local slab's geometry                      */
    tsr_layout layout;     /* its device layout                              */
    void* buf[2];          /* device buffers                                 */
} tsr_slab_info;

/* One halo delivery (CommRecord, scheduler.hpp:75-81). */
typedef struct tsr_comm_record {
    int64_t round;
    int32_t from_slab, to_slab;
    int64_t bytes;         /* depth * interior cross-section * sizeof(T)     */
    double seam_ms;        /* device time of the sender's seam passes        */
    /* Timeline of the sender's round on its device, ms after the first
     * logged round of that slab: seam passes [seam_t0, seam_t1) on the seam
     * stream, interior pass [interior_t0, interior_t1) on the second stream
     * (equal when the slab has no interior planes). */
    double seam_t0_ms, seam_t1_ms, interior_t0_ms, interior_t1_ms;
} tsr_comm_record;

/* Validates the partition (each slab >= r*k planes, the reference's
 * "subdomain smaller than the halo depth"), enables peer access and
 * allocates the slabs.  No data is uploaded yet. */
int tsr_multi_create(const tsr_kernel* k, const tsr_grid* g, const tsr_partition* part,
                     const tsr_opts* opts, tsr_multi** out);
int tsr_multi_destroy(tsr_multi* m);
/* Uploads a whole global host buffer (the reference's layout; its halo is
 * the Dirichlet boundary) into every slab, ghosts included. */
int tsr_multi_upload(tsr_multi* m, const void* host);
/* fill_random(seed, lo, hi) of the GLOBAL grid (random.hpp:20-24: one
 * std::mt19937_64 stream over the global interior, halo zero), streamed
 * straight into the slabs through a bounded pinned staging buffer. */
int tsr_multi_fill_random(tsr_multi* m, uint64_t seed, double lo, double hi);
/* Advances `steps` time steps (ceil(steps/k) rounds, plus a final one-step
 * round when keep_previous != 0 so the other buffers hold step T-1).
 * Synchronous; stats->device_ms is the max over slabs of the CUDA-event time
 * from a common start (all devices idle) to each slab's last launch. */
int tsr_multi_advance(tsr_multi* m, int64_t steps, int32_t keep_previous, tsr_stats* stats);
/* Owned planes of the current buffers -> host_cur, of the other buffers ->
 * host_prev (NULL = skip); host buffers in the reference's global layout,
 * other cells untouched. */
int tsr_multi_download(tsr_multi* m, void* host_cur, void* host_prev);
int tsr_multi_slab_info(const tsr_multi* m, int32_t slab, tsr_slab_info* out);
/* Per-round deliveries of the rounds since the last call (records kept only
 * after tsr_multi_set_logging(m, 1)).  *count = records available; at most
 * `cap` are copied. */
int tsr_multi_set_logging(tsr_multi* m, int32_t on);
int tsr_multi_comm_log(tsr_multi* m, tsr_comm_record* out, int64_t cap, int64_t* count);
/* A 64-bit position-mixed checksum of every owned global interior plane
 * (slab axis) of the current (which = 0) or other (which = 1) buffers:
 * out[p] for p in [0, n0).  Equal planes give equal sums; used to compare a
 * slab run with a one-device run of the same global grid without moving it. */
int tsr_multi_plane_checksums(tsr_multi* m, int32_t which, uint64_t* out);
/* The same checksum over planes [lo, hi) of one device buffer. */
int tsr_plane_checksums(const tsr_grid* g, const tsr_layout* l, const void* dev, int64_t lo,
                        int64_t hi, uint64_t* out, void* stream);

/* One-call host-buffer slab run: tsr_run over `part` (NULL = opts->ngpus
 * equal slabs).  keep_previous != 0: buffers end as naive_run leaves them
 * (step T and T-1); 0: only buffer(parity ^ (steps&1)) is written, as
 * run_heterogeneous leaves a grid (it scatters the workers' rows into the
 * read buffer only, scheduler.cpp:555-557). */
int tsr_run_multi(const tsr_kernel* k, const tsr_grid* g, void* buf0, void* buf1,
                  int32_t parity, int64_t steps, const tsr_partition* part,
                  int32_t keep_previous, const tsr_opts* opts, tsr_stats* stats);

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
