// tma.cuh — TMA tensor maps, mbarriers and launch sizing shared by the
// plane-streaming 3-D engines (tb3d.cu, box3d.cu).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace tsr {

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned addr = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// One box of a 3-D tensor map into shared memory, completion signalled on
// `bar` as transaction bytes.  The innermost coordinate must be 16-B aligned.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
        "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();

// Tensor map over a whole device buffer in the pitched layout of `g`:
// dims (row pitch, a1 rows incl. halo, a0 planes incl. halo); out-of-range
// boxes are zero-filled.
template <typename T>
Status make_tmap_3d(const Geo& g, const void* base, int box_w, int box_h, CUtensorMap* m) {
    auto enc = tmap_encoder();
    if (!enc) return Status::Err(TSR_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {(cuuint64_t)g.pitch[1], (cuuint64_t)(g.n[1] + 2 * g.h[1]),
                          (cuuint64_t)(g.n[0] + 2 * g.h[0])};
    cuuint64_t strides[2] = {(cuuint64_t)(g.pitch[1] * sizeof(T)),
                             (cuuint64_t)(g.pitch[0] * sizeof(T))};
    cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return Status::Err(TSR_ECUDA, "cuTensorMapEncodeTiled failed");
    return Status::Ok();
}

// Resident CTAs per SM for `kernel` (after raising its dynamic smem limit)
// and the SM count of the current device.
// Cached per kernel (function address) and device: the first call sets the
// shared-memory limit and queries the driver; the slab runtime launches
// several sweeps per round from one host thread, so per-launch driver
// queries would be host time on every round.
bool occupancy_cached(const void* fn, int dev, int threads, int smem, int* per_sm, int* nsm);
void occupancy_store(const void* fn, int dev, int threads, int smem, int per_sm, int nsm);

template <typename K>
Status occupancy(K kernel, int threads, int smem, int* per_sm, int* nsm) {
    int dev = 0;
    TSR_CUDA_TRY(cudaGetDevice(&dev));
    const void* fn = reinterpret_cast<const void*>(kernel);
    if (occupancy_cached(fn, dev, threads, smem, per_sm, nsm)) return Status::Ok();
    TSR_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    TSR_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kernel, threads, smem));
    TSR_CUDA_TRY(cudaDeviceGetAttribute(nsm, cudaDevAttrMultiProcessorCount, dev));
    if (*per_sm < 1) return Status::Err(TSR_ECUDA, "kernel cannot be resident on an SM");
    occupancy_store(fn, dev, threads, smem, *per_sm, *nsm);
    return Status::Ok();
}

// a0 chunk length minimising waves * (chunk + overlap) over CTA slots.
int pick_chunk(int64_t n0, int64_t tiles, int64_t slots, int overlap, int min_chunk);

}  // namespace tsr
