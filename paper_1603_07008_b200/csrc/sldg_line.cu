// sldg_line.cu -- 1D sweeps (D == 1) for any precision layout: the paper's own workload (one
// periodic line of N cells, o = k Legendre coefficients per cell, the first d = nd of them in
// fp64, P:391-456 SS III-A, Tables II-VI).  Same update as every sweep (R1-R6):
//     c'_{i,j} = sum_l A_jl c_{(i-i*-1) mod N, l} + sum_l B_jl c_{(i-i*) mod N, l}.
//
//   line_tma_kernel<k, d>   N % 4 == 0 and N >= 1024: warp-specialised persistent kernel.  A tile
//                           is a segment of Wt consecutive targets; the producer bulk-copies
//                           every slot's source window [t0-i*-1, t0+Wt-i*) (aligned to 16 bytes,
//                           two pieces when it wraps around the periodic line) into the stage;
//                           consumers read their two sources per slot from shared memory.
//   line_simple_kernel<k>   any N, any nd (C1-sized lines): one thread per target cell.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "sldg_internal.h"

namespace sldg {

namespace {

__device__ __forceinline__ uint32_t l_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void l_mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(l_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void l_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(l_smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void l_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(l_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void l_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra LWAIT_%=;\n"
        "}\n" ::"r"(l_smem_u32(bar)),
        "r"(parity), "r"(1000000u)  // suspend-time hint (ns)
        : "memory");
}
__device__ __forceinline__ void l_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     l_smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(l_smem_u32(bar))
                 : "memory");
}

// pointer to slot q of cell i of a 1D grid (general nd layout, pad = 0, one layer)
__device__ __forceinline__ const char* l_slot(const Arrays& a, const Layout& L, int q, int64_t i)
{
    if (q < L.nd) return (const char*)dslot(a, 0, L.nd, q, L.L, i);
    return (const char*)fslot(a, 0, L.K, L.nd, q, L.L, i);
}

}  // namespace

struct LinePlan {
    int Wt;           // targets per tile
    int slot_elems;   // elements reserved per slot in a stage (Wt + 16)
    int stage_bytes;
    int stages;
};

// ============================================================================================
template <int KK>
__global__ void __launch_bounds__(256) line_simple_kernel(Layout lay, Sweep sw, Arrays src, Arrays dst)
{
    const int64_t N = lay.n[0];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int64_t s = __ldg(&sw.smod[0]);
    const int cp = __ldg(&sw.copy[0]);
    const double* __restrict__ w = sw.ab;
    int64_t iB = i - s;
    if (iB < 0) iB += N;
    int64_t iA = iB - 1;
    if (iA < 0) iA += N;
    double a[KK], b[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        if (j < lay.nd) {
            a[j] = *(const double*)l_slot(src, lay, j, iA);
            b[j] = *(const double*)l_slot(src, lay, j, iB);
        } else {
            a[j] = (double)*(const float*)l_slot(src, lay, j, iA);
            b[j] = (double)*(const float*)l_slot(src, lay, j, iB);
        }
    }
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        double o = 0.0;
#pragma unroll
        for (int l = 0; l < KK; ++l) o = fma(__ldg(&w[j * KK + l]), a[l], o);
#pragma unroll
        for (int l = 0; l < KK; ++l) o = fma(__ldg(&w[KK * KK + j * KK + l]), b[l], o);
        if (cp) o = b[j];  // alpha == 0: exact copy (R4)
        if (j < lay.nd) *(double*)l_slot(dst, lay, j, i) = o;
        else *(float*)l_slot(dst, lay, j, i) = __double2float_rn(o);
    }
}

// ============================================================================================
// Consumer side of line_tma_kernel for one stage.  A thread owns 4 consecutive targets
// i0..i0+3 of the tile: their sources are the 5 consecutive window cells i0..i0+4 (target r reads
// A from cell r and B from cell r+1), so every source is read from shared memory and promoted
// once, and the 4 outputs of a slot leave as one 16-byte (fp32) or two 16-byte (fp64) stores.
// OFF = (w0 mod 4) is the window's offset inside its 16-byte-aligned copy; it is the same for
// every tile of a launch (t0 is a multiple of 256), so it is a template parameter and all
// register indexing below is static.
template <int KK, int NDJ, int OFF>
__device__ __forceinline__ void line_consume_stage(const unsigned char* st, int slot_elems, int nt, int64_t N,
                                                   int64_t t0, const double (&wr)[2 * KK * KK], int cp,
                                                   const Arrays& dst)
{
    constexpr int NT = kTmaConsumerWarps * 32;
    for (int u = threadIdx.x; 4 * u < nt; u += NT) {
        double v[KK][5];
        if (cp) {  // alpha == 0: target r is source r+1, copied bit for bit (R4)
            int soff = 0;
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                if (j < NDJ) {
                    const double2* p = (const double2*)(st + soff) + 2 * u;
                    const double2 a = p[0], b = p[1], c = p[2];
                    const double e[6] = {a.x, a.y, b.x, b.y, c.x, c.y};
                    double2* q = (double2*)dslot(dst, 0, NDJ, j, N, t0 + 4 * u);
                    __stcs(q, make_double2(e[(OFF & 1) + 1], e[(OFF & 1) + 2]));
                    __stcs(q + 1, make_double2(e[(OFF & 1) + 3], e[(OFF & 1) + 4]));
                    soff += slot_elems * 8;
                } else {
                    const float4* p = (const float4*)(st + soff) + u;
                    const float4 a = p[0], b = p[1];
                    const float e[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                    __stcs((float4*)fslot(dst, 0, KK, NDJ, j, N, t0 + 4 * u),
                           make_float4(e[OFF + 1], e[OFF + 2], e[OFF + 3], e[OFF + 4]));
                    soff += slot_elems * 4;
                }
            }
            continue;
        }
        int soff = 0;
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            if (j < NDJ) {
                const double2* p = (const double2*)(st + soff) + 2 * u;
                const double2 a = p[0], b = p[1], c = p[2];
                const double e[6] = {a.x, a.y, b.x, b.y, c.x, c.y};
#pragma unroll
                for (int r = 0; r < 5; ++r) v[j][r] = e[(OFF & 1) + r];
                soff += slot_elems * 8;
            } else {
                const float4* p = (const float4*)(st + soff) + u;
                const float4 a = p[0], b = p[1];
                const float e[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
                for (int r = 0; r < 5; ++r) v[j][r] = (double)e[OFF + r];
                soff += slot_elems * 4;
            }
        }
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            double o[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                double oa = 0.0, ob = 0.0;
#pragma unroll
                for (int l = 0; l < KK; ++l) {
                    oa = fma(wr[j * KK + l], v[l][r], oa);
                    ob = fma(wr[KK * KK + j * KK + l], v[l][r + 1], ob);
                }
                o[r] = oa + ob;
            }
            if (j < NDJ) {
                double2* q = (double2*)dslot(dst, 0, NDJ, j, N, t0 + 4 * u);
                __stcs(q, make_double2(o[0], o[1]));
                __stcs(q + 1, make_double2(o[2], o[3]));
            } else {
                __stcs((float4*)fslot(dst, 0, KK, NDJ, j, N, t0 + 4 * u),
                       make_float4(__double2float_rn(o[0]), __double2float_rn(o[1]), __double2float_rn(o[2]),
                                   __double2float_rn(o[3])));
            }
        }
    }
}

template <int KK, int NDJ>
__global__ void __launch_bounds__(kTmaThreads, 1) line_tma_kernel(Layout lay, Sweep sw, Arrays src, Arrays dst,
                                                                   LinePlan lp)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int S = lp.stages;
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = full + S;
    unsigned char* stage0 = smem + 256;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NC = kTmaConsumerWarps;
    const bool producer = (warp == NC);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            l_mbar_init(&full[s], 1);
            l_mbar_init(&empty[s], NC);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int64_t N = lay.n[0];
    const int Wt = lp.Wt;
    const int64_t ntiles = (N + Wt - 1) / Wt;
    const int64_t s = __ldg(&sw.smod[0]);
    const int cp = __ldg(&sw.copy[0]);
    double wr[2 * KK * KK];
#pragma unroll
    for (int i = 0; i < 2 * KK * KK; ++i) wr[i] = __ldg(&sw.ab[i]);
    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int64_t t0 = tile * Wt;
        const int nt = (int)((N - t0) < Wt ? (N - t0) : Wt);
        int64_t w0 = (t0 - s - 1) % N;  // first source cell of the window (the A-source of t0)
        if (w0 < 0) w0 += N;
        const int st_i = it % S;
        const uint32_t ph = (it / S) & 1;
        unsigned char* st = stage0 + (size_t)st_i * lp.stage_bytes;
        if (producer) {
            if (lane == 0) {
                l_wait(&empty[st_i], ph ^ 1);
                uint32_t bytes = 0;
#pragma unroll
                for (int j = 0; j < KK; ++j) {
                    const int es = (j < NDJ) ? 8 : 4, al = 16 / es;
                    const int64_t a0 = w0 - (w0 % al);
                    const int64_t len = ((w0 - a0) + nt + 1 + al - 1) / al * al;
                    bytes += (uint32_t)(len * es);
                }
                l_expect_tx(&full[st_i], bytes);
                int soff = 0;
#pragma unroll
                for (int j = 0; j < KK; ++j) {
                    const int es = (j < NDJ) ? 8 : 4, al = 16 / es;
                    const int64_t a0 = w0 - (w0 % al);
                    const int64_t len = ((w0 - a0) + nt + 1 + al - 1) / al * al;
                    if (a0 + len <= N) {
                        l_bulk(st + soff, l_slot(src, lay, j, a0), (uint32_t)(len * es), &full[st_i]);
                    } else {  // the window wraps around the periodic line: two pieces
                        const int64_t n1 = N - a0;
                        l_bulk(st + soff, l_slot(src, lay, j, a0), (uint32_t)(n1 * es), &full[st_i]);
                        l_bulk(st + soff + n1 * es, l_slot(src, lay, j, 0), (uint32_t)((len - n1) * es), &full[st_i]);
                    }
                    soff += lp.slot_elems * es;
                }
            }
            __syncwarp();
        } else {
            l_wait(&full[st_i], ph);
            // window start inside each slot's 16-byte-aligned copy: (t0 - s - 1) mod 4, equal for all tiles
            switch ((int)(w0 & 3)) {
                case 0: line_consume_stage<KK, NDJ, 0>(st, lp.slot_elems, nt, N, t0, wr, cp, dst); break;
                case 1: line_consume_stage<KK, NDJ, 1>(st, lp.slot_elems, nt, N, t0, wr, cp, dst); break;
                case 2: line_consume_stage<KK, NDJ, 2>(st, lp.slot_elems, nt, N, t0, wr, cp, dst); break;
                default: line_consume_stage<KK, NDJ, 3>(st, lp.slot_elems, nt, N, t0, wr, cp, dst); break;
            }
            __syncwarp();
            if (lane == 0) l_arrive(&empty[st_i]);
        }
    }
}

// ============================================================================================
static int g_sms = 0, g_optin = 0;

static bool line_plan(const Layout& lay, LinePlan* lp)
{
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&g_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    const int64_t N = lay.n[0];
    if (lay.D != 1 || lay.k > 4 || N % 4 != 0 || N < 1024) return false;
    const int64_t budget = std::min<int64_t>(g_optin, 200 * 1024) - 256;
    const int bpc = 8 * lay.nd + 4 * (lay.k - lay.nd);
    int64_t Wt = (budget / 3 / bpc - 16) / 256 * 256;
    Wt = std::min<int64_t>(Wt, (N - 16) / 256 * 256);
    // keep >= 2 tiles per SM when the line allows it
    while (Wt > 256 && (N + Wt - 1) / Wt < 2 * g_sms) Wt -= 256;
    if (Wt < 256) return false;
    lp->Wt = (int)Wt;
    lp->slot_elems = (int)Wt + 16;
    lp->stage_bytes = (int)(((int64_t)lp->slot_elems * bpc + 127) / 128 * 128);
    lp->stages = (int)std::min<int64_t>(8, budget / lp->stage_bytes);
    return lp->stages >= 2;
}

template <int KK, int NDJ>
static cudaError_t launch_line_tma(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst,
                                   const LinePlan& lp, cudaStream_t s)
{
    auto kern = line_tma_kernel<KK, NDJ>;
    ensure_max_smem((const void*)kern);  // full opt-in carveout (per device)
    const size_t smem = 256 + (size_t)lp.stages * lp.stage_bytes;
    const int64_t ntiles = (lay.n[0] + lp.Wt - 1) / lp.Wt;
    const int64_t grid = std::min<int64_t>(ntiles, g_sms);
    kern<<<(unsigned)grid, kTmaThreads, smem, s>>>(lay, sw, src, dst, lp);
    return cudaGetLastError();
}

template <int KK>
static cudaError_t launch_line_k(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst,
                                 cudaStream_t s, const char** name)
{
    LinePlan lp;
    if constexpr (KK <= 4) {
        if (line_plan(lay, &lp)) {
            *name = "line_tma_kernel";
            switch (lay.nd) {
                case 0: return launch_line_tma<KK, 0>(lay, sw, src, dst, lp, s);
                case 1: return launch_line_tma<KK, (KK >= 1 ? 1 : 0)>(lay, sw, src, dst, lp, s);
                case 2: return launch_line_tma<KK, (KK >= 2 ? 2 : 0)>(lay, sw, src, dst, lp, s);
                case 3: return launch_line_tma<KK, (KK >= 3 ? 3 : 0)>(lay, sw, src, dst, lp, s);
                case 4: return launch_line_tma<KK, (KK >= 4 ? 4 : 0)>(lay, sw, src, dst, lp, s);
            }
            return cudaErrorInvalidValue;
        }
    }
    *name = "line_simple_kernel";
    const int64_t N = lay.n[0];
    line_simple_kernel<KK><<<(unsigned)((N + 255) / 256), 256, 0, s>>>(lay, sw, src, dst);
    return cudaGetLastError();
}

cudaError_t launch_line(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst, cudaStream_t s,
                        const char** name)
{
    const char* dummy;
    if (!name) name = &dummy;
    switch (lay.k) {
        case 1: return launch_line_k<1>(lay, sw, src, dst, s, name);
        case 2: return launch_line_k<2>(lay, sw, src, dst, s, name);
        case 3: return launch_line_k<3>(lay, sw, src, dst, s, name);
        case 4: return launch_line_k<4>(lay, sw, src, dst, s, name);
        case 5: return launch_line_k<5>(lay, sw, src, dst, s, name);
        case 6: return launch_line_k<6>(lay, sw, src, dst, s, name);
        case 7: return launch_line_k<7>(lay, sw, src, dst, s, name);
        case 8: return launch_line_k<8>(lay, sw, src, dst, s, name);
    }
    return cudaErrorInvalidValue;
}

const char* line_kernel_name(const Layout& lay)
{
    LinePlan lp;
    return line_plan(lay, &lp) ? "line_tma_kernel" : "line_simple_kernel";
}

}  // namespace sldg
