// peer.cu — the memory tier's peer-memory transport: CUDA IPC mappings of a
// neighbour slab's buffers and stream-ordered round flags.
//
// The reference moves a halo slab per round through SlabChannel
// (proj/src/scheduler.cpp:142-194, one mutex-guarded copy per message).  Here
// the seam sweep itself stores its output planes into the neighbour's ghost
// planes over NVLink (LaunchCtx::mirror, every engine's store path), so the
// exchange costs no extra pass and no collective; these helpers provide the
// mappings and the per-round ordering:
//   round n on rank r:  interior sweep  ||  wait(flags from both neighbours >= n-1)
//                       seam sweeps (mirror -> neighbours' next-buffer ghosts)
//                       signal(neighbours' flags = n)
// A neighbour finishing round n-1 has (a) filled my current ghosts and (b)
// finished reading the buffer my round-n seams write into, so one wait per
// round covers both the RAW and the WAR hazard.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "common.cuh"

namespace tsr {

namespace {

// A neighbour that never signals (a dead rank, a mapping that does not reach
// the peer) must fail the stream loudly instead of hanging the device: spins
// give up after kSpinTimeoutNs of wall time and trap (a sticky launch error
// the host sees at its next synchronisation).
constexpr unsigned long long kSpinTimeoutNs = 120ull * 1000 * 1000 * 1000;

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void spin_until(const unsigned* flag, unsigned value) {
    const unsigned long long t0 = global_ns();
    for (;;) {
        unsigned v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (static_cast<int>(v - value) >= 0) return;
        __nanosleep(200);
        if (global_ns() - t0 > kSpinTimeoutNs) {
            printf("tessera_b200: peer flag %p stuck at %u (waiting for %u); trapping\n",
                   flag, v, value);
            __trap();
        }
    }
}

__global__ void signal_kernel(unsigned* flag, unsigned value) {
    // every store of earlier work on this stream is complete at kernel
    // boundaries; the fence orders them before the flag for the peer
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

__global__ void wait_kernel(const unsigned* flag, unsigned value) { spin_until(flag, value); }

// Round-counting variants (no per-round kernel arguments, so a round can be
// captured once into a CUDA graph and replayed): `counter` holds the rounds
// this rank has completed.
__global__ void round_wait_kernel(const unsigned* flag_lo, const unsigned* flag_hi,
                                  const unsigned* counter) {
    unsigned want;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(want) : "l"(counter) : "memory");
    for (const unsigned* f : {flag_lo, flag_hi})
        if (f) spin_until(f, want);
}

__global__ void round_signal_kernel(unsigned* peer_lo, unsigned* peer_hi, unsigned* counter) {
    __threadfence_system();
    const unsigned done = *counter + 1;
    *counter = done;
    for (unsigned* f : {peer_lo, peer_hi})
        if (f) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(done) : "memory");
}

using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

GetRangeFn get_range() {
    static GetRangeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<GetRangeFn>(p);
        return static_cast<GetRangeFn>(nullptr);
    }();
    return fn;
}

}  // namespace

Status peer_signal(void* flag, unsigned value, cudaStream_t s) {
    signal_kernel<<<1, 1, 0, s>>>(static_cast<unsigned*>(flag), value);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

Status peer_wait(const void* flag, unsigned value, cudaStream_t s) {
    wait_kernel<<<1, 1, 0, s>>>(static_cast<const unsigned*>(flag), value);
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

Status peer_round_wait(const void* flag_lo, const void* flag_hi, const void* counter,
                       cudaStream_t s) {
    round_wait_kernel<<<1, 1, 0, s>>>(static_cast<const unsigned*>(flag_lo),
                                      static_cast<const unsigned*>(flag_hi),
                                      static_cast<const unsigned*>(counter));
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

Status peer_round_signal(void* peer_lo, void* peer_hi, void* counter, cudaStream_t s) {
    round_signal_kernel<<<1, 1, 0, s>>>(static_cast<unsigned*>(peer_lo),
                                        static_cast<unsigned*>(peer_hi),
                                        static_cast<unsigned*>(counter));
    TSR_CUDA_TRY(cudaGetLastError());
    return Status::Ok();
}

Status ipc_export(const void* ptr, unsigned char* handle, int64_t* offset) {
    auto fn = get_range();
    if (!fn) return Status::Err(TSR_ECUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        return Status::Err(TSR_EINVAL, "pointer is not a device allocation");
    cudaIpcMemHandle_t h;
    TSR_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, sizeof(h));
    *offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(ptr) - base);
    return Status::Ok();
}

Status ipc_open(const unsigned char* handle, void** base) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    TSR_CUDA_TRY(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
    return Status::Ok();
}

Status ipc_close(void* base) {
    TSR_CUDA_TRY(cudaIpcCloseMemHandle(base));
    return Status::Ok();
}

}  // namespace tsr
