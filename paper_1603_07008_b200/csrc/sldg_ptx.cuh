// sldg_ptx.cuh -- mbarrier / bulk-copy / tensor-TMA wrappers for sm_100a shared by the TMA
// kernels (sldg_sweep_tma.cu, sldg_fused.cu).  The PTX spellings are the ISA's.
#pragma once
#include <cuda.h>  // CUtensorMap (types only)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

namespace sldg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef SLDG_MBAR_HINT_NS
#define SLDG_MBAR_HINT_NS 1000000u  // suspend-time hint of mbarrier waits (ns); 0: plain try_wait spin
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    if (SLDG_MBAR_HINT_NS == 0) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            "@!p bra WAIT_%=;\n"
            "}\n" ::"r"(smem_u32(bar)),
            "r"(parity)
            : "memory");
    } else {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
            "@!p bra WAIT_%=;\n"
            "}\n" ::"r"(smem_u32(bar)),
            "r"(parity), "r"(SLDG_MBAR_HINT_NS)  // suspend-time hint (ns): sleep until the phase completes
            : "memory");
    }
}
// 1D bulk copy global -> shared (fallback for rows that wrap around a periodic line)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// 5D tensor box global -> shared (dense, row-major box in shared memory)
__device__ __forceinline__ void tma_5d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3, int c4,
                                       uint64_t* bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
        "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tm)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)tm) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Programmatic dependent launch (PDL): a kernel launched with the programmatic-serialization
// attribute may start while its predecessor in the stream finishes; pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible (no-op without PDL), pdl_trigger()
// lets the successor launch once every CTA of this grid has triggered or exited.  The sweep kernels
// trigger at the start of their LAST tile (all their CTAs are resident by then, so a successor's
// waiting CTAs can never hold an SM one of ours still needs); the weight build at its start.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// launch with the PDL attribute (SLDG_PDL=0 disables it: plain stream order)
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     Args&&... args)
{
    static const bool on = !(getenv("SLDG_PDL") && atoi(getenv("SLDG_PDL")) == 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = on ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// 5D tile tensor map (sldg_sweep_tma.cu): dims / strides in elements (strides[0] = 1 implied),
// box in elements; false if the driver's encoder is unavailable or rejects the shape
bool make_tmap5(CUtensorMap* tm, bool f64, void* base, const int64_t* dims, const int64_t* strides, const int* box);
// SM count and opt-in shared memory per block of the current device (queried once)
void tma_device_info(int* num_sms, int* smem_optin);

}  // namespace sldg
