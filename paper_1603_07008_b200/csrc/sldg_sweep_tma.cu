// sldg_sweep_tma.cu -- TMA-staged SLDG sweep kernels for sm_100a.
//
// Same arithmetic as sldg_sweep.cu (readings R1-R6), different data movement:
// a warp-specialised persistent kernel.  One producer warp streams the source rows of each
// (tile, coupled group) into a ring of shared-memory stages with bulk asynchronous copies
// (cp.async.bulk global->shared, completion counted on an mbarrier, SASS UBLKCP); the consumer
// warps wait on the stage's "full" barrier, read their two source cells per target from
// shared memory, do the fp64 contraction and write the outputs with coalesced streaming stores,
// then release the stage on its "empty" barrier.  Bytes in flight are set by the number of
// stages (~200 KB per SM), not by registers, which is what an HBM-bound stream needs.
//
//   sweep_strided_tma  d >= 1: tile = W consecutive i_0 columns x T targets along d of one
//                      perpendicular line set; per coupled group a stage holds the k slots'
//                      rows [t0 - i*max - 1, t0 + T - 1 - i*min] (the union over the tile's
//                      per-lane shifts), so per-lane CFL fields still read each row once.
//                      Rows that are contiguous in HBM are merged into one copy.
//   sweep_d0_tma       d = 0: tile = R whole lines (the line is periodic, so the stage holds
//                      every source cell and the modulo indexing is done in shared memory);
//                      a stage holds GC coupled groups (all of them when they fit).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "sldg_internal.h"

namespace sldg {

// ---- PTX helpers ----------------------------------------------------------------------
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// bulk copy global -> shared, completion signalled as transaction bytes on `bar`;
// evict-first L2 policy: every source byte is read once per sweep.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <int PREC>
__device__ __forceinline__ int64_t toff_m(const Layout& L, int64_t layerp, int64_t inner)
{
    return (PREC == SLDG_FP64) ? layerp * (int64_t)L.K * L.L + inner : layerp * L.L + inner;
}
template <int PREC>
__device__ __forceinline__ int64_t toff_f(const Layout& L, int64_t layerp, int64_t inner)
{
    return (PREC == SLDG_FP64) ? 0 : layerp * (int64_t)(L.K - 1) * L.L + inner;
}
__device__ __forceinline__ int64_t tfield_index(const Sweep& sw, const int64_t* idx, int D)
{
    int64_t f = 0;
#pragma unroll
    for (int e = 0; e < kMaxDim; ++e)
        if (e < D) f += idx[e] * sw.fstride[e];
    return f;
}
__device__ __forceinline__ int64_t pmod(int64_t x, int64_t n)
{
    int64_t r = x % n;
    return r < 0 ? r + n : r;
}

// global element pointer of slot q at (padded layer, inner) -- as a byte pointer
template <int PREC>
__device__ __forceinline__ const char* slot_ptr(const Arrays& a, const Layout& L, int q, int64_t layerp, int64_t inner)
{
    if (PREC == SLDG_FP64) return (const char*)(a.s64 + toff_m<PREC>(L, layerp, inner) + (int64_t)q * L.L);
    if (q == 0) return (const char*)(a.mass + toff_m<PREC>(L, layerp, inner));
    return (const char*)(a.pl + toff_f<PREC>(L, layerp, inner) + (int64_t)(q - 1) * L.L);
}

template <int PREC>
__device__ __forceinline__ int esz(bool massg, int j)
{
    return (PREC == SLDG_FP64 || (massg && j == 0)) ? 8 : 4;
}

// ============================================================================================
// strided sweep (d >= 1)
// ============================================================================================
template <int KK, int PREC>
__global__ void __launch_bounds__(kTmaThreads) sweep_strided_tma(Layout lay, Sweep sw, Arrays src, Arrays dst,
                                                                  int64_t lb, int64_t le, TmaPlan pl)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int S = pl.stages;
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = full + S;
    unsigned char* stage0 = smem + 256;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NC = kTmaConsumerWarps;
    const bool producer = (warp == NC);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC);
        }
        fence_barrier_init();
    }
    __syncthreads();

    const int D = lay.D, d = sw.dim;
    const bool outer = (d == D - 1);
    const int W = pl.W, T = pl.T, Rmax = pl.Rmax;
    const int64_t n0 = lay.n[0];
    const int64_t nb0 = n0 / W;
    const int64_t nlay = le - lb;
    const int64_t nline = outer ? nlay : sw.nd;
    const int64_t nseg = (nline + T - 1) / T;
    int64_t nperp = 1;
    for (int e = 1; e < D - 1; ++e)
        if (e != d) nperp *= lay.n[e];
    const int64_t ntiles = nseg * nb0 * nperp * (outer ? 1 : nlay);
    int kd = 1;
    for (int e = 0; e < d; ++e) kd *= KK;
    const int G = lay.K / KK;
    const int64_t L = lay.L;
    const uint64_t pol = policy_evict_first();

    // consumer thread -> column c, part of the targets
    const int NT = NC * 32;
    const int P = NT / W;
    const int tid = threadIdx.x;
    const int c = tid % W, part = tid / W;

    uint32_t it = 0;  // stage-use counter, identical in every warp
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int64_t rem = tile;
        const int64_t seg = rem % nseg;
        rem /= nseg;
        const int64_t cb = rem % nb0;
        rem /= nb0;
        int64_t idx[kMaxDim];
#pragma unroll
        for (int e = 0; e < kMaxDim; ++e) idx[e] = 0;
        for (int e = 1; e < D - 1; ++e)
            if (e != d) {
                idx[e] = rem % lay.n[e];
                rem /= lay.n[e];
            }
        int64_t layer = 0;
        if (!outer) {
            layer = lb + rem;
            idx[D - 1] = lay.first_layer + layer;
        }
        int64_t inner_base = 0;  // inner offset of column 0 of the tile at line coordinate 0
        for (int e = 1; e < D - 1; ++e)
            if (e != d) inner_base += idx[e] * lay.S[e];
        inner_base += cb * W;
        const int64_t t0 = seg * T;  // first target (local index along the line)
        const int64_t nt = (nline - t0) < T ? (nline - t0) : T;
        // global line coordinate of target index 0 (outer: global layer; inner: i_d)
        const int64_t tg0 = outer ? lay.first_layer + lb : 0;

        // shift range over the tile's W columns (computed redundantly by every warp)
        int64_t imin = INT64_MAX, imax = INT64_MIN;
        for (int cc = lane; cc < W; cc += 32) {
            int64_t id2[kMaxDim];
#pragma unroll
            for (int e = 0; e < kMaxDim; ++e) id2[e] = idx[e];
            id2[0] = cb * W + cc;
            id2[d] = 0;
            int64_t s = __ldg(&sw.shift[tfield_index(sw, id2, D)]);
            imin = s < imin ? s : imin;
            imax = s > imax ? s : imax;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            int64_t a = __shfl_xor_sync(0xffffffffu, imin, o), b = __shfl_xor_sync(0xffffffffu, imax, o);
            imin = a < imin ? a : imin;
            imax = b > imax ? b : imax;
        }
        const int64_t span = imax - imin;
        const int64_t teff = (Rmax - 1 - span) < nt ? (Rmax - 1 - span) : nt;
        if (teff < 1) {
            // ---- slow path (shift spread too wide for the stage): direct global loads ----
            if (!producer) {
                for (int col = tid; col < W; col += NT) {
                    int64_t id2[kMaxDim];
#pragma unroll
                    for (int e = 0; e < kMaxDim; ++e) id2[e] = idx[e];
                    id2[0] = cb * W + col;
                    id2[d] = 0;
                    const int64_t f = tfield_index(sw, id2, D);
                    const int64_t s = __ldg(&sw.shift[f]);
                    const int cpf = __ldg(&sw.copy[f]);
                    const double* w = sw.ab + f * (2 * KK * KK);
                    for (int g = 0; g < G; ++g) {
                        int qbase = 0, gg = g, kp = 1;
                        for (int e = 0; e < D; ++e) {
                            if (e != d) {
                                qbase += (gg % KK) * kp;
                                gg /= KK;
                            }
                            kp *= KK;
                        }
                        for (int64_t tt = t0; tt < t0 + nt; ++tt) {
                            const int64_t xB = tg0 + tt - s;
                            double va[KK], vb[KK];
                            for (int half = 0; half < 2; ++half) {
                                int64_t x = xB - 1 + half;
                                int64_t lp, in;
                                if (outer) {
                                    lp = sw.wrap ? lay.pad + pmod(x, sw.nd) : x - lay.first_layer + lay.pad;
                                    in = inner_base + col;
                                } else {
                                    lp = lay.pad + layer;
                                    in = inner_base + col + pmod(x, sw.nd) * lay.S[d];
                                }
#pragma unroll
                                for (int j = 0; j < KK; ++j) {
                                    const int q = qbase + j * kd;
                                    const char* p = slot_ptr<PREC>(src, lay, q, lp, in);
                                    double v = (PREC == SLDG_FP64 || q == 0) ? *(const double*)p : (double)*(const float*)p;
                                    if (half) vb[j] = v;
                                    else va[j] = v;
                                }
                            }
                            int64_t lp, in;
                            if (outer) {
                                lp = lay.pad + lb + tt;
                                in = inner_base + col;
                            } else {
                                lp = lay.pad + layer;
                                in = inner_base + col + tt * lay.S[d];
                            }
#pragma unroll
                            for (int j = 0; j < KK; ++j) {
                                double o = 0.0;
                                if (cpf) {
                                    o = vb[j];
                                } else {
#pragma unroll
                                    for (int l = 0; l < KK; ++l) o = fma(w[j * KK + l], va[l], o);
#pragma unroll
                                    for (int l = 0; l < KK; ++l) o = fma(w[KK * KK + j * KK + l], vb[l], o);
                                }
                                const int q = qbase + j * kd;
                                char* p = (char*)slot_ptr<PREC>(dst, lay, q, lp, in);
                                if (PREC == SLDG_FP64 || q == 0) *(double*)p = o;
                                else *(float*)p = __double2float_rn(o);
                            }
                        }
                    }
                }
            }
            continue;
        }

        // consumer: per-column line data (weights in registers)
        int64_t my_s = 0;
        int my_cp = 0;
        double wr[2 * KK * KK];
        if (!producer && c < W) {
            int64_t id2[kMaxDim];
#pragma unroll
            for (int e = 0; e < kMaxDim; ++e) id2[e] = idx[e];
            id2[0] = cb * W + c;
            id2[d] = 0;
            const int64_t f = tfield_index(sw, id2, D);
            my_s = __ldg(&sw.shift[f]);
            my_cp = __ldg(&sw.copy[f]);
#pragma unroll
            for (int i = 0; i < 2 * KK * KK; ++i) wr[i] = __ldg(&sw.ab[f * (2 * KK * KK) + i]);
        }

        for (int64_t sub = 0; sub < nt; sub += teff) {
            const int64_t te = (nt - sub) < teff ? (nt - sub) : teff;
            const int64_t rows = te + 1 + span;
            const int64_t rowbase = tg0 + t0 + sub - imax - 1;  // global line coordinate of row 0
            for (int g = 0; g < G; ++g) {
                const int s = it % S;
                const uint32_t ph = (it / S) & 1;
                ++it;
                const bool massg = (PREC == SLDG_MIXED) && g == 0;
                int qbase = 0;
                {
                    int gg = g, kp = 1;
                    for (int e = 0; e < D; ++e) {
                        if (e != d) {
                            qbase += (gg % KK) * kp;
                            gg /= KK;
                        }
                        kp *= KK;
                    }
                }
                unsigned char* st = stage0 + (size_t)s * pl.stage_bytes;
                if (producer) {
                    if (lane == 0) mbar_wait(&empty[s], ph ^ 1);
                    __syncwarp();
                    uint32_t bytes = 0;
#pragma unroll
                    for (int j = 0; j < KK; ++j) bytes += (uint32_t)(rows * W * esz<PREC>(massg, j));
                    if (lane == 0) mbar_expect_tx(&full[s], bytes);
                    __syncwarp();
                    // one copy per (slot, run of contiguous rows); lanes share the rows
                    int soff = 0;
#pragma unroll
                    for (int j = 0; j < KK; ++j) {
                        const int q = qbase + j * kd;
                        const int es = esz<PREC>(massg, j);
                        const uint32_t rowb = (uint32_t)(W * es);
                        for (int64_t r = lane; r < rows; r += 32) {
                            const int64_t x = rowbase + r;
                            int64_t lp, in;
                            if (outer) {
                                lp = sw.wrap ? lay.pad + pmod(x, sw.nd) : x - lay.first_layer + lay.pad;
                                in = inner_base;
                            } else {
                                lp = lay.pad + layer;
                                in = inner_base + pmod(x, sw.nd) * lay.S[d];
                            }
                            bulk_g2s(st + soff + r * rowb, slot_ptr<PREC>(src, lay, q, lp, in), rowb, &full[s], pol);
                        }
                        soff += Rmax * W * es;
                    }
                } else {
                    mbar_wait(&full[s], ph);
                    // this thread: column c, targets [lo, hi) of the sub-chunk
                    const int64_t tp = (te + P - 1) / P;
                    const int64_t lo = part * tp, hi = (lo + tp) < te ? (lo + tp) : te;
                    if (lo < hi) {
                        // slot j base in the stage
                        const unsigned char* sb[KK];
                        {
                            int soff = 0;
#pragma unroll
                            for (int j = 0; j < KK; ++j) {
                                sb[j] = st + soff;
                                soff += Rmax * W * esz<PREC>(massg, j);
                            }
                        }
                        auto rd = [&](int j, int64_t r) -> double {
                            if (esz<PREC>(massg, j) == 8) return ((const double*)sb[j])[r * W + c];
                            return (double)((const float*)sb[j])[r * W + c];
                        };
                        // row of the B-source of target lo: (tg - s) - rowbase
                        int64_t rB = (tg0 + t0 + sub + lo - my_s) - rowbase;
                        double va[KK], vb[KK];
#pragma unroll
                        for (int j = 0; j < KK; ++j) va[j] = rd(j, rB - 1);
                        for (int64_t tt = lo; tt < hi; ++tt, ++rB) {
#pragma unroll
                            for (int j = 0; j < KK; ++j) vb[j] = rd(j, rB);
                            const int64_t tl = t0 + sub + tt;  // local target index
                            int64_t lp, in;
                            if (outer) {
                                lp = lay.pad + lb + tl;
                                in = inner_base + c;
                            } else {
                                lp = lay.pad + layer;
                                in = inner_base + c + tl * lay.S[d];
                            }
#pragma unroll
                            for (int j = 0; j < KK; ++j) {
                                double o;
                                if (my_cp) {
                                    o = vb[j];
                                } else {
                                    o = 0.0;
#pragma unroll
                                    for (int l = 0; l < KK; ++l) o = fma(wr[j * KK + l], va[l], o);
#pragma unroll
                                    for (int l = 0; l < KK; ++l) o = fma(wr[KK * KK + j * KK + l], vb[l], o);
                                }
                                const int q = qbase + j * kd;
                                if (PREC == SLDG_FP64) __stcs(dst.s64 + toff_m<PREC>(lay, lp, in) + (int64_t)q * L, o);
                                else if (massg && j == 0) __stcs(dst.mass + toff_m<PREC>(lay, lp, in), o);
                                else __stcs(dst.pl + toff_f<PREC>(lay, lp, in) + (int64_t)(q - 1) * L, __double2float_rn(o));
                            }
#pragma unroll
                            for (int j = 0; j < KK; ++j) va[j] = vb[j];
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                }
            }
        }
    }
}

// ============================================================================================
// contiguous sweep (d = 0): R whole lines x GC coupled groups per stage
// ============================================================================================
template <int KK, int PREC>
__global__ void __launch_bounds__(kTmaThreads) sweep_d0_tma(Layout lay, Sweep sw, Arrays src, Arrays dst, int64_t lb,
                                                             int64_t le, TmaPlan pl)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int S = pl.stages;
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = full + S;
    unsigned char* stage0 = smem + 256;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NC = kTmaConsumerWarps;
    const bool producer = (warp == NC);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC);
        }
        fence_barrier_init();
    }
    __syncthreads();

    const int D = lay.D;
    const int64_t n0 = lay.n[0];
    const int64_t L = lay.L;
    const int R = pl.R, GC = pl.GC;
    const int64_t lines_per_layer = L / n0;
    const int64_t nblk = lines_per_layer / R;
    const int64_t nlay = le - lb;
    const int64_t ntiles = nblk * nlay;
    const int G = lay.K / KK;
    const int NT = NC * 32;
    const uint64_t pol = policy_evict_first();

    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t blk = tile % nblk;
        const int64_t layer = lb + tile / nblk;
        const int64_t layerp = lay.pad + layer;
        const int64_t inner_base = blk * R * n0;  // first cell of the tile's first line
        for (int g0 = 0; g0 < G; g0 += GC) {
            const int gc = (G - g0) < GC ? (G - g0) : GC;
            const int s = it % S;
            const uint32_t ph = (it / S) & 1;
            ++it;
            unsigned char* st = stage0 + (size_t)s * pl.stage_bytes;
            if (producer) {
                if (lane == 0) mbar_wait(&empty[s], ph ^ 1);
                __syncwarp();
                const int nslot = gc * KK;
                uint32_t bytes = 0;
                for (int i = 0; i < nslot; ++i) {
                    const int q = g0 * KK + i;
                    bytes += (uint32_t)(R * n0 * ((PREC == SLDG_FP64 || q == 0) ? 8 : 4));
                }
                if (lane == 0) mbar_expect_tx(&full[s], bytes);
                __syncwarp();
                // slot i of the stage at offset soff(i): doubles first-slot-aware prefix sum
                for (int i = lane; i < nslot; i += 32) {
                    const int q = g0 * KK + i;
                    const int64_t soff = (PREC == SLDG_FP64) ? (int64_t)i * R * n0 * 8
                                                             : (int64_t)i * R * n0 * 4 + ((g0 == 0 && i > 0) ? (int64_t)R * n0 * 4 : 0);
                    const uint32_t b = (uint32_t)(R * n0 * ((PREC == SLDG_FP64 || q == 0) ? 8 : 4));
                    bulk_g2s(st + soff, slot_ptr<PREC>(src, lay, q, layerp, inner_base), b, &full[s], pol);
                }
            } else {
                mbar_wait(&full[s], ph);
                for (int64_t m = threadIdx.x; m < (int64_t)R * n0; m += NT) {
                    const int64_t r = m / n0, c = m - r * n0;
                    // the line's field entry / weights
                    int64_t f = 0;
                    if (sw.fmask) {
                        int64_t idx[kMaxDim];
                        int64_t rem2 = inner_base / n0 + r;  // line index within the layer
#pragma unroll
                        for (int e = 0; e < kMaxDim; ++e) idx[e] = 0;
                        for (int e = 1; e < D - 1; ++e) {
                            idx[e] = rem2 % lay.n[e];
                            rem2 /= lay.n[e];
                        }
                        if (D >= 2) idx[D - 1] = lay.first_layer + layer;
                        f = tfield_index(sw, idx, D);
                    }
                    const int64_t sm = __ldg(&sw.smod[f]);
                    const int cp = __ldg(&sw.copy[f]);
                    const double* __restrict__ w = sw.ab + f * (2 * KK * KK);
                    int64_t cB = c - sm;
                    if (cB < 0) cB += n0;
                    int64_t cA = cB - 1;
                    if (cA < 0) cA += n0;
                    const int64_t tin = inner_base + r * n0 + c;
                    for (int gi = 0; gi < gc; ++gi) {
                        const int g = g0 + gi;
                        const bool massg = (PREC == SLDG_MIXED) && g == 0;
                        double va[KK], vb[KK];
#pragma unroll
                        for (int j = 0; j < KK; ++j) {
                            const int i = gi * KK + j;
                            if (PREC == SLDG_FP64) {
                                const double* sp = (const double*)(st + (int64_t)i * R * n0 * 8) + r * n0;
                                va[j] = sp[cA];
                                vb[j] = sp[cB];
                            } else if (massg && j == 0) {
                                const double* sp = (const double*)st + r * n0;
                                va[j] = sp[cA];
                                vb[j] = sp[cB];
                            } else {
                                const float* sp = (const float*)(st + (int64_t)i * R * n0 * 4 +
                                                                 (g0 == 0 ? (int64_t)R * n0 * 4 : 0)) + r * n0;
                                va[j] = (double)sp[cA];
                                vb[j] = (double)sp[cB];
                            }
                        }
#pragma unroll
                        for (int j = 0; j < KK; ++j) {
                            double o;
                            if (cp) {
                                o = vb[j];
                            } else {
                                o = 0.0;
#pragma unroll
                                for (int l = 0; l < KK; ++l) o = fma(__ldg(&w[j * KK + l]), va[l], o);
#pragma unroll
                                for (int l = 0; l < KK; ++l) o = fma(__ldg(&w[KK * KK + j * KK + l]), vb[l], o);
                            }
                            const int q = g * KK + j;
                            if (PREC == SLDG_FP64) __stcs(dst.s64 + toff_m<PREC>(lay, layerp, tin) + (int64_t)q * L, o);
                            else if (q == 0) __stcs(dst.mass + toff_m<PREC>(lay, layerp, tin), o);
                            else __stcs(dst.pl + toff_f<PREC>(lay, layerp, tin) + (int64_t)(q - 1) * L, __double2float_rn(o));
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
        }
    }
}

// ============================================================================================
// planning + launch
// ============================================================================================
static int g_num_sms = 0;
static int g_smem_optin = 0;

static void query_device()
{
    if (g_num_sms) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&g_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
}

// Returns true and fills `pl` when the TMA path applies to this sweep.
bool tma_plan(const Layout& lay, const Sweep& sw, TmaPlan* pl)
{
    query_device();
    const int64_t n0 = lay.n[0];
    const int k = lay.k;
    const int64_t budget = std::min<int64_t>(g_smem_optin, 200 * 1024) - 256;
    const int bpc_max = (lay.prec == SLDG_FP64) ? 8 * k : 8 + 4 * (k - 1);  // bytes per row-column, mass group
    *pl = TmaPlan{};
    if (sw.dim == 0) {
        if (n0 % 4 != 0) return false;
        const int64_t lines = lay.L / n0;
        const int64_t line_bytes_group = n0 * bpc_max;  // one line, one coupled group (worst case)
        const int G = lay.K / k;
        // pick GC groups and R lines so a stage is <= budget/3 (>= 3 stages)
        int64_t target = budget / 3;
        if (line_bytes_group > target) return false;
        int GC = (int)std::min<int64_t>(G, target / line_bytes_group);
        int64_t R = 1;
        if (GC == G) {
            while (R * 2 <= lines && lines % (R * 2) == 0 && (R * 2) * line_bytes_group * G <= target) R *= 2;
        }
        pl->R = (int)R;
        pl->GC = GC;
        // exact stage bytes: the mass group dominates (first stage of a tile)
        const int64_t slot_f = R * n0 * ((lay.prec == SLDG_FP64) ? 8 : 4);
        pl->stage_bytes = (int)(GC * k * slot_f + ((lay.prec == SLDG_FP64) ? 0 : R * n0 * 4) + 127) / 128 * 128;
        pl->stages = (int)std::min<int64_t>(8, budget / pl->stage_bytes);
        if (pl->stages < 2) return false;
        return true;
    }
    // strided (line weights live in registers: k <= 4; larger k uses the register kernels)
    if (k > 4) return false;
    int W = 0;
    for (int w : {128, 64, 32})
        if (n0 % w == 0) {
            W = w;
            break;
        }
    if (W == 0) return false;
    const int T = (k <= 3) ? 16 : (k <= 5 ? 8 : 4);
    const int Rmax = T + 1 + 3;
    const int64_t stage = (int64_t)Rmax * W * bpc_max;
    const int stage_bytes = (int)((stage + 127) / 128 * 128);
    const int stages = (int)std::min<int64_t>(8, budget / stage_bytes);
    if (stages < 2) return false;
    pl->W = W;
    pl->T = T;
    pl->Rmax = Rmax;
    pl->stage_bytes = stage_bytes;
    pl->stages = stages;
    return true;
}

template <int KK, int PREC>
static cudaError_t launch_tma_k(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst, int64_t lb,
                                int64_t le, const TmaPlan& pl, cudaStream_t s)
{
    const size_t smem = 256 + (size_t)pl.stages * pl.stage_bytes;
    int64_t ntiles;
    if (sw.dim == 0) {
        ntiles = (lay.L / lay.n[0] / pl.R) * (le - lb);
        auto kern = sweep_d0_tma<KK, PREC>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = std::max<int>(1, (int)(228 * 1024 / (smem + 1024)));
        int64_t grid = std::min<int64_t>(ntiles, (int64_t)g_num_sms * per_sm);
        if (grid < 1) return cudaSuccess;
        kern<<<(unsigned)grid, kTmaThreads, smem, s>>>(lay, sw, src, dst, lb, le, pl);
    } else {
        const bool outer = (sw.dim == lay.D - 1);
        const int64_t nline = outer ? (le - lb) : sw.nd;
        int64_t nperp = 1;
        for (int e = 1; e < lay.D - 1; ++e)
            if (e != sw.dim) nperp *= lay.n[e];
        ntiles = ((nline + pl.T - 1) / pl.T) * (lay.n[0] / pl.W) * nperp * (outer ? 1 : (le - lb));
        auto kern = sweep_strided_tma<KK, PREC>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = std::max<int>(1, (int)(228 * 1024 / (smem + 1024)));
        int64_t grid = std::min<int64_t>(ntiles, (int64_t)g_num_sms * per_sm);
        if (grid < 1) return cudaSuccess;
        kern<<<(unsigned)grid, kTmaThreads, smem, s>>>(lay, sw, src, dst, lb, le, pl);
    }
    return cudaGetLastError();
}

template <int PREC>
static cudaError_t launch_tma_p(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst, int64_t lb,
                                int64_t le, const TmaPlan& pl, cudaStream_t s)
{
    switch (lay.k) {
        case 1: return launch_tma_k<1, PREC>(lay, sw, src, dst, lb, le, pl, s);
        case 2: return launch_tma_k<2, PREC>(lay, sw, src, dst, lb, le, pl, s);
        case 3: return launch_tma_k<3, PREC>(lay, sw, src, dst, lb, le, pl, s);
        case 4: return launch_tma_k<4, PREC>(lay, sw, src, dst, lb, le, pl, s);
        case 5: return launch_tma_k<5, PREC>(lay, sw, src, dst, lb, le, pl, s);
        case 6: return launch_tma_k<6, PREC>(lay, sw, src, dst, lb, le, pl, s);
        case 7: return launch_tma_k<7, PREC>(lay, sw, src, dst, lb, le, pl, s);
        case 8: return launch_tma_k<8, PREC>(lay, sw, src, dst, lb, le, pl, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_sweep_tma(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst, int64_t lb,
                             int64_t le, const TmaPlan& pl, cudaStream_t s)
{
    if (le <= lb) return cudaSuccess;
    if (lay.prec == SLDG_FP64) return launch_tma_p<SLDG_FP64>(lay, sw, src, dst, lb, le, pl, s);
    return launch_tma_p<SLDG_MIXED>(lay, sw, src, dst, lb, le, pl, s);
}

}  // namespace sldg
