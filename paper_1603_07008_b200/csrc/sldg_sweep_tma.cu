// sldg_sweep_tma.cu -- TMA-staged SLDG sweep kernels for sm_100a.
//
// Same arithmetic as sldg_sweep.cu (readings R1-R6), different data movement:
// a warp-specialised persistent kernel.  One producer thread streams the source rows of each
// (tile, coupled group) into a ring of shared-memory stages with tensor TMA (one
// cp.async.bulk.tensor box per coefficient slot per stage, SASS UTMALDG; completion counted on
// an mbarrier); the consumer warps wait on the stage's "full" barrier, read their two source
// cells per target from shared memory, do the fp64 contraction and write the outputs with
// coalesced streaming stores, then release the stage on its "empty" barrier.  Bytes in flight
// are set by the number of stages (~200 KB per SM), not by registers.
//
//   sweep_strided_tma  d >= 1: tile = W consecutive cells of the dims below d (the "lo" index,
//                      contiguous in HBM) x a run of targets along d; per coupled group a stage
//                      holds the k slots' rows [t0 - i*max - 1, t0 + te - 1 - i*min] (the union
//                      over the tile's per-lane shifts), so per-lane CFL fields still read each
//                      row once.  The rows of a stage are one run of consecutive source rows
//                      (two when they wrap around the periodic line), each run loaded as boxes
//                      of 2^h rows from a family of tensor maps (exact bytes, no over-fetch).
//   sweep_d0_tma       d = 0: tile = R whole lines (the line is periodic, so the stage holds
//                      every source cell and the modulo indexing is done in shared memory);
//                      a stage holds GC coupled groups as one TMA box (+ one for the mass).
// Consumers address HBM and shared memory by pointer increments set up once per stage; the
// coupled group that holds the fp64 mass slot is a separate template instance.
#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched from the driver at run time)
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "sldg_internal.h"
#include "sldg_ptx.cuh"

namespace sldg {

constexpr int kTmaHeights = 5;  // strided boxes of 1, 2, 4, 8, 16 rows (binary decomposition of a run)
struct TmapSet {
    CUtensorMap f[kTmaHeights];  // fp32 planes (mixed) or all slots (fp64)
    CUtensorMap m[kTmaHeights];  // fp64 mass slot (mixed)
};

#ifdef SLDG_STAMPS
// diagnostic builds (-DSLDG_STAMPS): per-CTA %globaltimer stamps of the strided kernel, printed by
// the launcher (start, first stage ready, consumers done, producer done)
__device__ unsigned long long g_stamp[8 * 1024];
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SLDG_STAMP(i) g_stamp[8 * blockIdx.x + (i)] = gtimer()
#else
#define SLDG_STAMP(i) ((void)0)
#endif

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

// byte pointer of slot q at (padded layer, inner)
template <int PREC>
__device__ __forceinline__ const char* slot_ptr(const Arrays& a, const Layout& L, int q, int64_t layerp, int64_t inner)
{
    if (PREC == SLDG_FP64) return (const char*)(a.s64 + toff_m<PREC>(L, layerp, inner) + (int64_t)q * L.L);
    if (q == 0) return (const char*)(a.mass + toff_m<PREC>(L, layerp, inner));
    return (const char*)(a.pl + toff_f<PREC>(L, layerp, inner) + (int64_t)(q - 1) * L.L);
}
template <int PREC>
__device__ __forceinline__ char* slot_ptr_w(const Arrays& a, const Layout& L, int q, int64_t layerp, int64_t inner)
{
    return const_cast<char*>(slot_ptr<PREC>(a, L, q, layerp, inner));
}
template <int PREC>
__host__ __device__ __forceinline__ int esz_rt(bool massg, int j)
{
    return (PREC == SLDG_FP64 || (massg && j == 0)) ? 8 : 4;
}
__device__ __forceinline__ void st_elem(char* p, int64_t i, double v, bool dbl)
{
    if (dbl) __stcs(((double*)p) + i, v);
    else __stcs(((float*)p) + i, __double2float_rn(v));
}

// Strided consumer: one stage (one coupled group), one column, `cnt` consecutive targets.
// sb[j]: stage slot j at row 0 of this column; sstride: elements between rows; rB0: row of the
// B-source of the first target; op[j]: output pointer of slot j at the first target; ostep:
// element step between consecutive targets (mass/fp64 array, fp32 planes).
template <int KK, int PREC, bool MASSG>
__device__ __forceinline__ void strided_consume(const unsigned char* const* sb, int sstride, int rB0, int cnt,
                                                char* const* op, int64_t ostep_m, int64_t ostep_f, int cp,
                                                const double* wr)
{
#define SLDG_DBL(j) ((PREC == SLDG_FP64) || (MASSG && (j) == 0))
    const unsigned char* rp[KK];  // row pointers (advance one row per target)
    char* wp[KK];                 // output pointers (advance one target per target)
    int64_t wstep[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        rp[j] = sb[j] + (int64_t)(rB0 - 1) * sstride * (SLDG_DBL(j) ? 8 : 4);
        wp[j] = op[j];
        wstep[j] = SLDG_DBL(j) ? ostep_m * 8 : ostep_f * 4;
    }
    const int rstep = sstride;  // elements
    if (cp) {  // alpha == 0: exact copy of the B-source, bit for bit (R4); rare, so a branch
        for (int u = 0; u < cnt; ++u) {
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                rp[j] += rstep * (SLDG_DBL(j) ? 8 : 4);
                if (SLDG_DBL(j)) __stcs((double*)wp[j], *(const double*)rp[j]);
                else __stcs((float*)wp[j], *(const float*)rp[j]);
                wp[j] += wstep[j];
            }
        }
        return;
    }
    // o_j(t) = sum_l A_jl a_l(t) + sum_l B_jl b_l(t) with a(t+1) = b(t): the A-part of target
    // t+1 is accumulated from the row just loaded for target t, so each output's dependent FMA
    // chain is k long instead of 2k (same operation order, hence the same rounding).
    double sA[KK], vb[KK];
    {
        double va[KK];
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            va[j] = SLDG_DBL(j) ? *(const double*)rp[j] : (double)*(const float*)rp[j];
            rp[j] += rstep * (SLDG_DBL(j) ? 8 : 4);
        }
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < KK; ++l) s = fma(wr[j * KK + l], va[l], s);
            sA[j] = s;
        }
    }
#pragma unroll 2
    for (int u = 0; u < cnt; ++u) {
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            vb[j] = SLDG_DBL(j) ? *(const double*)rp[j] : (double)*(const float*)rp[j];
            rp[j] += rstep * (SLDG_DBL(j) ? 8 : 4);
        }
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            double o = sA[j];
#pragma unroll
            for (int l = 0; l < KK; ++l) o = fma(wr[KK * KK + j * KK + l], vb[l], o);
            if (SLDG_DBL(j)) __stcs((double*)wp[j], o);
            else __stcs((float*)wp[j], __double2float_rn(o));
            wp[j] += wstep[j];
        }
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < KK; ++l) s = fma(wr[j * KK + l], vb[l], s);
            sA[j] = s;
        }
    }
#undef SLDG_DBL
}

// Split variant for k >= 5 (the 2k^2 weights of a whole line do not fit in registers next to the
// walk): SPL = 2 threads share a column, thread J0 / JN owns output slots [J0, J0 + JN) and their
// JN rows of A and B (wr[jj * KK + l] = A[J0 + jj][l], wr[JN * KK + jj * KK + l] = B[J0 + jj][l]);
// both read all k inputs of every row.  Same operation order per output as strided_consume.
template <int KK, int PREC, bool MASSG, int JN, int J0>
__device__ __forceinline__ void strided_consume_split(const unsigned char* const* sb, int sstride, int rB0, int cnt,
                                                      char* const* op, int64_t ostep_m, int64_t ostep_f, int cp,
                                                      const double* wr)
{
#define SLDG_DBL(j) ((PREC == SLDG_FP64) || (MASSG && (j) == 0))
    const unsigned char* rp[KK];
    char* wp[JN];
    int64_t wstep[JN];
#pragma unroll
    for (int j = 0; j < KK; ++j) rp[j] = sb[j] + (int64_t)(rB0 - 1) * sstride * (SLDG_DBL(j) ? 8 : 4);
#pragma unroll
    for (int jj = 0; jj < JN; ++jj) {
        const int j = J0 + jj;
        wp[jj] = (j < KK) ? op[j < KK ? j : 0] : nullptr;
        wstep[jj] = SLDG_DBL(j) ? ostep_m * 8 : ostep_f * 4;
    }
    const int rstep = sstride;
    if (cp) {
        for (int u = 0; u < cnt; ++u) {
#pragma unroll
            for (int j = 0; j < KK; ++j) rp[j] += rstep * (SLDG_DBL(j) ? 8 : 4);
#pragma unroll
            for (int jj = 0; jj < JN; ++jj) {
                const int j = J0 + jj;
                if (j >= KK) break;
                if (SLDG_DBL(j)) __stcs((double*)wp[jj], *(const double*)rp[j]);
                else __stcs((float*)wp[jj], *(const float*)rp[j]);
                wp[jj] += wstep[jj];
            }
        }
        return;
    }
    double sA[JN], vb[KK];
    {
        double va[KK];
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            va[j] = SLDG_DBL(j) ? *(const double*)rp[j] : (double)*(const float*)rp[j];
            rp[j] += rstep * (SLDG_DBL(j) ? 8 : 4);
        }
#pragma unroll
        for (int jj = 0; jj < JN; ++jj) {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < KK; ++l) s = fma(wr[jj * KK + l], va[l], s);
            sA[jj] = s;
        }
    }
#pragma unroll 2
    for (int u = 0; u < cnt; ++u) {
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            vb[j] = SLDG_DBL(j) ? *(const double*)rp[j] : (double)*(const float*)rp[j];
            rp[j] += rstep * (SLDG_DBL(j) ? 8 : 4);
        }
#pragma unroll
        for (int jj = 0; jj < JN; ++jj) {
            const int j = J0 + jj;
            if (j >= KK) break;
            double o = sA[jj];
#pragma unroll
            for (int l = 0; l < KK; ++l) o = fma(wr[JN * KK + jj * KK + l], vb[l], o);
            if (SLDG_DBL(j)) __stcs((double*)wp[jj], o);
            else __stcs((float*)wp[jj], __double2float_rn(o));
            wp[jj] += wstep[jj];
        }
#pragma unroll
        for (int jj = 0; jj < JN; ++jj) {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < KK; ++l) s = fma(wr[jj * KK + l], vb[l], s);
            sA[jj] = s;
        }
    }
#undef SLDG_DBL
}

// ============================================================================================
// strided sweep (d >= 1)
//   lo  = linear index over the dims below d (outer sweep: all dims below D-1), contiguous in
//         HBM; a tile covers W consecutive lo values (its "columns")
//   hi  = linear index over the dims strictly between d and D-1 (1 for the outer sweep)
//   tensor maps (5D, fp32 planes or fp64 slots / fp64 mass):
//         inner: {lo, i_d, hi, plane, layer}   outer: {lo, 1, 1, plane, layer}
// ============================================================================================
template <int KK, int PREC, int MINB, bool PSPAN>
__global__ void __launch_bounds__(kTmaThreads, MINB) sweep_strided_tma(Layout lay, Sweep sw, Arrays src, Arrays dst,
                                                                  int64_t lb, int64_t le, TmaPlan pl,
                                                                  const __grid_constant__ TmapSet tmaps)
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
        for (int h = 0; h < kTmaHeights; ++h) {
            prefetch_tmap(&tmaps.f[h]);
            if (PREC == SLDG_MIXED) prefetch_tmap(&tmaps.m[h]);
        }
    }
    __syncthreads();
    pdl_wait();  // the weights and the source array come from the preceding kernels
#ifdef SLDG_WARM_TMA
    // diagnostic: touch every tensor map with an L2 prefetch of one box before the span work
    if (threadIdx.x == kTmaConsumerWarps * 32) {
        for (int h = 0; h < kTmaHeights; ++h) {
            asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %1, %1, %1, %2}];" ::"l"(
                             (uint64_t)&tmaps.f[h]), "r"(0), "r"((int)lay.pad) : "memory");
            if (PREC == SLDG_MIXED)
                asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %1, %1, %1, %2}];" ::"l"(
                                 (uint64_t)&tmaps.m[h]), "r"(0), "r"((int)lay.pad) : "memory");
        }
    }
#endif
    if (threadIdx.x == 0) SLDG_STAMP(0);
#ifdef SLDG_STAMPS
    bool first_full = true;
#endif

    const int D = lay.D, d = sw.dim;
    const bool outer = (d == D - 1);
    const int W = pl.W, T = pl.T, Rmax = pl.Rmax, Tsub = pl.Tsub;
    int64_t M_lo = 1, M_hi = 1;
    for (int e = 0; e < (outer ? D - 1 : d); ++e) M_lo *= lay.n[e];
    if (!outer)
        for (int e = d + 1; e < D - 1; ++e) M_hi *= lay.n[e];
    const int64_t nb = M_lo / W;
    const int64_t nlay = le - lb;
    const int64_t nline = outer ? nlay : sw.nd;
    const int64_t nseg = (nline + T - 1) / T;
    const int64_t ntiles = nseg * nb * M_hi * (outer ? 1 : nlay);
    int kd = 1;
    for (int e = 0; e < d; ++e) kd *= KK;
    const int G = lay.K / KK;
    // default L2 priority: the last rows of a sub-chunk are read again by the next one
    const uint64_t pol = policy_evict_normal();
    // element step between consecutive targets along d (mass/fp64 array, fp32 planes)
    const int64_t tstep_m = outer ? (toff_m<PREC>(lay, 1, 0) - toff_m<PREC>(lay, 0, 0)) : M_lo;
    const int64_t tstep_f = outer ? (toff_f<PREC>(lay, 1, 0) - toff_f<PREC>(lay, 0, 0)) : M_lo;

    const int NT = NC * 32;
    // k >= 5: SPL = 2 threads per column, each with half of the output slots (W <= NT / 2)
    constexpr int SPL = (KK > 4) ? 2 : 1;
    constexpr int JN = (KK + SPL - 1) / SPL;
    const int P = NT / (W * SPL);
    const int tid = threadIdx.x;
    const int c = tid % W, part = tid / (W * SPL);
    const int jh = (SPL == 1) ? 0 : (tid / W) % SPL;

    // tile -> (segment along d, column block, hi, layer).  PSPAN: 32-bit index math with rolled
    // loops (compact code: in short sweeps such as C2's this runs often, and the inlined 64-bit
    // divisions made the kernel ~300 KB of SASS, instruction-cache bound); otherwise the 64-bit
    // form the long-tile instances were tuned with (their hot-loop codegen depends on it).
    auto decode = [&](int64_t tl, int64_t& cb, int64_t& hi, int64_t& layer, int64_t& t0) {
        if constexpr (PSPAN) {
            uint32_t rem = (uint32_t)tl;
            const uint32_t seg = rem % (uint32_t)nseg;
            rem /= (uint32_t)nseg;
            cb = rem % (uint32_t)nb;
            rem /= (uint32_t)nb;
            hi = rem % (uint32_t)M_hi;
            rem /= (uint32_t)M_hi;
            layer = outer ? 0 : lb + rem;
            t0 = (int64_t)seg * T;
        } else {
            int64_t rem = tl;
            const int64_t seg = rem % nseg;
            rem /= nseg;
            cb = rem % nb;
            rem /= nb;
            hi = rem % M_hi;
            rem /= M_hi;
            layer = outer ? 0 : lb + rem;
            t0 = seg * T;
        }
    };
    // field entry of column lo (all perpendicular indices from lo, hi, layer)
    auto findex = [&](int64_t lo64, int64_t hi64, int64_t layer) -> int64_t {
        const int elo = outer ? D - 1 : d;
        if constexpr (PSPAN) {
            uint32_t lo = (uint32_t)lo64, hi = (uint32_t)hi64;
            int64_t f = 0;
#pragma unroll 1
            for (int e = 0; e < elo; ++e) {
                const uint32_t ne = (uint32_t)lay.n[e], q = lo / ne;
                f += (int64_t)(lo - q * ne) * sw.fstride[e];
                lo = q;
            }
            if (!outer) {
#pragma unroll 1
                for (int e = d + 1; e < D - 1; ++e) {
                    const uint32_t ne = (uint32_t)lay.n[e], q = hi / ne;
                    f += (int64_t)(hi - q * ne) * sw.fstride[e];
                    hi = q;
                }
                f += (lay.first_layer + layer) * sw.fstride[D - 1];
            }
            return f;
        } else {
            int64_t lo = lo64, hi = hi64;
            int64_t idx[kMaxDim];
#pragma unroll
            for (int e = 0; e < kMaxDim; ++e) idx[e] = 0;
            for (int e = 0; e < elo; ++e) {
                idx[e] = lo % lay.n[e];
                lo /= lay.n[e];
            }
            if (!outer) {
                for (int e = d + 1; e < D - 1; ++e) {
                    idx[e] = hi % lay.n[e];
                    hi /= lay.n[e];
                }
                idx[D - 1] = lay.first_layer + layer;
            }
            return tfield_index(sw, idx, D);
        }
    };
    // The tile's shift span (min / max integer shift over its W columns).
    // PSPAN: computed by the producer warp alone, which loads the NEXT tile's column shifts while
    // the current tile streams (software prefetch, 1-CTA-per-SM instance) and publishes each
    // tile's span in a ring in shared memory before it arms the tile's first stage; consumers
    // read it after that stage's full barrier, so no consumer warp runs per-column index math.
    // Ring slot reuse is safe: slot (tile count % 8) is rewritten 8 tiles later, after the empty
    // barrier of a stage >= 8 - S >= 0 stages past this tile's first one (S <= 8).
    // Otherwise every warp computes the span itself from its own prefetch of the shifts.
    int64_t* span_ring = (int64_t*)(smem + 128);  // [8][2]: imin, imax
    constexpr bool PF = (MINB == 1);
    int64_t pf_sh[PF ? 8 : 1];
    auto prefetch = [&](int64_t tl) {
        int64_t cb, hi, layer, t0;
        decode(tl, cb, hi, layer, t0);
#pragma unroll
        for (int i = 0; i < (PF ? 8 : 1); ++i) {
            const int cc = lane + 32 * i;
            pf_sh[i] = (cc < W) ? __ldg(&sw.shift[findex(cb * W + cc, hi, layer)]) : 0;
        }
    };
    if (PF && (producer || !PSPAN) && (int64_t)blockIdx.x < ntiles) prefetch(blockIdx.x);

    uint32_t it = 0;  // stage-use counter, identical in every warp
    uint32_t tcount = 0;  // tiles of this CTA so far, identical in every warp
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
        if (tile + gridDim.x >= ntiles) pdl_trigger();  // this CTA's last tile
        int64_t cb, hi, layer, t0;
        decode(tile, cb, hi, layer, t0);
        const int nt = (int)((nline - t0) < T ? (nline - t0) : T);
        const int64_t tg0 = outer ? lay.first_layer + lb : 0;  // line coordinate of target index 0
        const int64_t inner_base = outer ? cb * W : cb * W + hi * M_lo * sw.nd;  // column 0, coordinate 0

        // this tile's consumer line data: column shift, copy flag, A/B in registers (PSPAN: issued
        // before the wait for the tile's first stage, so their latency overlaps its first copy)
        int64_t my_s = 0;
        int my_cp = 0;
        double wr[2 * JN * KK];
        if constexpr (PSPAN) {
            if (!producer) {
                const int64_t f = findex(cb * W + c, hi, layer);
                my_s = __ldg(&sw.shift[f]);
                my_cp = __ldg(&sw.copy[f]);
                if constexpr (SPL == 1) {
#pragma unroll
                    for (int i = 0; i < 2 * KK * KK; ++i) wr[i] = __ldg(&sw.ab[f * (2 * KK * KK) + i]);
                } else {
#pragma unroll
                    for (int jj = 0; jj < JN; ++jj) {
                        const int j = jh * JN + jj < KK ? jh * JN + jj : KK - 1;
#pragma unroll
                        for (int l = 0; l < KK; ++l) {
                            wr[jj * KK + l] = __ldg(&sw.ab[f * (2 * KK * KK) + j * KK + l]);
                            wr[JN * KK + jj * KK + l] = __ldg(&sw.ab[f * (2 * KK * KK) + KK * KK + j * KK + l]);
                        }
                    }
                }
            }
        }
        int64_t imin = INT64_MAX, imax = INT64_MIN;
        int64_t* ring = span_ring + 2 * (tcount & 7);
        if (producer || !PSPAN) {
            if (PF) {
#pragma unroll
                for (int i = 0; i < (PF ? 8 : 1); ++i) {
                    if (lane + 32 * i < W) {
                        imin = pf_sh[i] < imin ? pf_sh[i] : imin;
                        imax = pf_sh[i] > imax ? pf_sh[i] : imax;
                    }
                }
            } else {
#pragma unroll 1
                for (int cc = lane; cc < W; cc += 32) {
                    const int64_t sh = __ldg(&sw.shift[findex(cb * W + cc, hi, layer)]);
                    imin = sh < imin ? sh : imin;
                    imax = sh > imax ? sh : imax;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                int64_t a = __shfl_xor_sync(0xffffffffu, imin, o), b = __shfl_xor_sync(0xffffffffu, imax, o);
                imin = a < imin ? a : imin;
                imax = b > imax ? b : imax;
            }
            if (PF && tile + gridDim.x < ntiles) prefetch(tile + gridDim.x);
            // publish after the tile's first stage is free (see the ring comment above)
            if (PSPAN && lane == 0) {
                mbar_wait(&empty[it % S], ((it / S) & 1) ^ 1);
                ring[0] = imin;
                ring[1] = imax;
            }
        } else {
            mbar_wait(&full[it % S], (it / S) & 1);  // the tile's first stage: its span is published
            imin = ring[0];
            imax = ring[1];
        }
        const int64_t span = imax - imin;
        // sub-chunks of te targets: rows = te + 1 + span <= Rmax, balanced over the tile
        const int tmax = (int)(Rmax - 1 - span);
        (void)Tsub;
        if (tmax < 1) {
            // ---- shift spread too wide for a stage: direct global loads (rare) ----
            // PSPAN: the tile still takes one stage slot: the producer completes its full barrier
            // with a plain arrive (no bytes; it carried the span), the consumers release it
            const int s0 = it % S;
            if constexpr (PSPAN) {
                ++it;
                if (producer && lane == 0) mbar_arrive(&full[s0]);
                __syncwarp();
            }
            if (!producer) {
                for (int col = tid; col < W; col += NT) {
                    const int64_t f = findex(cb * W + col, hi, layer);
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
                                int64_t x = xB - 1 + half, lp, in;
                                int64_t xm = x % sw.nd;
                                if (xm < 0) xm += sw.nd;
                                if (outer) {
                                    lp = sw.wrap ? lay.pad + xm : x - lay.first_layer + lay.pad;
                                    in = inner_base + col;
                                } else {
                                    lp = lay.pad + layer;
                                    in = inner_base + col + xm * M_lo;
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
                            int64_t lp = outer ? lay.pad + lb + tt : lay.pad + layer;
                            int64_t in = outer ? inner_base + col : inner_base + col + tt * M_lo;
#pragma unroll
                            for (int j = 0; j < KK; ++j) {
                                double o = 0.0;
#pragma unroll
                                for (int l = 0; l < KK; ++l) o = fma(w[j * KK + l], va[l], o);
#pragma unroll
                                for (int l = 0; l < KK; ++l) o = fma(w[KK * KK + j * KK + l], vb[l], o);
                                o = cpf ? vb[j] : o;
                                const int q = qbase + j * kd;
                                st_elem(slot_ptr_w<PREC>(dst, lay, q, lp, in), 0, o, PREC == SLDG_FP64 || q == 0);
                            }
                        }
                    }
                }
                if constexpr (PSPAN) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s0]);
                }
            }
            continue;
        }
        const int nsub = (nt + tmax - 1) / tmax;
        const int tsz = (nt + nsub - 1) / nsub;
        if constexpr (!PSPAN) {
            if (!producer) {
                const int64_t f = findex(cb * W + c, hi, layer);
                my_s = __ldg(&sw.shift[f]);
                my_cp = __ldg(&sw.copy[f]);
                if constexpr (SPL == 1) {
#pragma unroll
                    for (int i = 0; i < 2 * KK * KK; ++i) wr[i] = __ldg(&sw.ab[f * (2 * KK * KK) + i]);
                } else {
#pragma unroll
                    for (int jj = 0; jj < JN; ++jj) {
                        const int j = jh * JN + jj < KK ? jh * JN + jj : KK - 1;
#pragma unroll
                        for (int l = 0; l < KK; ++l) {
                            wr[jj * KK + l] = __ldg(&sw.ab[f * (2 * KK * KK) + j * KK + l]);
                            wr[JN * KK + jj * KK + l] = __ldg(&sw.ab[f * (2 * KK * KK) + KK * KK + j * KK + l]);
                        }
                    }
                }
            }
        }

        // output position of target index 0 (padded layer, inner)
        const int64_t ob_lp = outer ? lay.pad + lb : lay.pad + layer;
        const int64_t ob_in = inner_base + c;

        for (int sub = 0; sub < nt; sub += tsz) {
            const int te = (nt - sub) < tsz ? (nt - sub) : tsz;
            const int rows = te + 1 + (int)span;
            const int64_t rowbase = tg0 + t0 + sub - imax - 1;  // line coordinate of stage row 0
            // this consumer thread's targets [lo, hi) of the sub-chunk
            const int tp = (te + P - 1) / P;
            const int lo_t = part * tp, hi_t = (lo_t + tp) < te ? (lo_t + tp) : te;
            const int rB0 = (int)((tg0 + t0 + sub + lo_t - my_s) - rowbase);
            const int64_t tl0 = t0 + sub + lo_t;  // local target index of lo_t
            // source row coordinate of stage row 0 in the tensor / memory
            int64_t x0;
            bool wraps = false;
            if (sw.wrap) {
                x0 = rowbase % sw.nd;
                if (x0 < 0) x0 += sw.nd;
                wraps = x0 + rows > sw.nd;
            } else {
                x0 = rowbase - lay.first_layer;  // local layer (halo rows live in the pad)
            }
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
                    if (lane == 0) {
#ifdef SLDG_STAMPS
                        if (it == 1) SLDG_STAMP(4);
#endif
                        mbar_wait(&empty[s], ph ^ 1);
                        uint32_t bytes = 0;
#pragma unroll
                        for (int j = 0; j < KK; ++j) bytes += (uint32_t)(rows * W * esz_rt<PREC>(massg, j));
                        mbar_expect_tx(&full[s], bytes);
                        // the stage rows as runs of consecutive source rows (a new run each time
                        // the rows wrap around the periodic line), each run as boxes of 2^h rows
                        int soff = 0;
#pragma unroll
                        for (int j = 0; j < KK; ++j) {
                            const int q = qbase + j * kd;
                            const bool mslot = (PREC == SLDG_MIXED) && q == 0;
                            const int es = esz_rt<PREC>(massg, j);
                            const int plane = (PREC == SLDG_FP64) ? q : (mslot ? 0 : q - 1);
                            const CUtensorMap* tms = mslot ? tmaps.m : tmaps.f;
                            int r = 0;        // next stage row
                            int64_t x = x0;   // its source row coordinate
                            while (r < rows) {
                                int left = rows - r;  // rows in this run
                                if (wraps && x + left > sw.nd) left = (int)(sw.nd - x);
                                for (int h = kTmaHeights - 1; h >= 0; --h) {
                                    while (left >= (1 << h)) {
                                        unsigned char* dstp = st + soff + (size_t)r * W * es;
                                        if (outer)
                                            tma_5d(dstp, &tms[h], (int)(cb * W), 0, 0, plane, (int)(x + lay.pad), &full[s], pol);
                                        else
                                            tma_5d(dstp, &tms[h], (int)(cb * W), (int)x, (int)hi, plane,
                                                   (int)(lay.pad + layer), &full[s], pol);
                                        r += 1 << h;
                                        x += 1 << h;
                                        left -= 1 << h;
                                    }
                                }
                                if (wraps && x >= sw.nd) x -= sw.nd;
                            }
                            soff += Rmax * W * es;
                        }
#ifdef SLDG_STAMPS
                        if (it == 1) SLDG_STAMP(5);
#endif
                    }
                    __syncwarp();
                } else {
#ifdef SLDG_STAMPS
                    if (first_full && threadIdx.x == 0) SLDG_STAMP(6);
#endif
                    mbar_wait(&full[s], ph);
#ifdef SLDG_STAMPS
                    if (first_full && threadIdx.x == 0) SLDG_STAMP(1);
                    first_full = false;
#endif
                    if (lo_t < hi_t) {
                        const unsigned char* sb[KK];
                        char* op[KK];
                        int soff = 0;
#pragma unroll
                        for (int j = 0; j < KK; ++j) {
                            const int es = esz_rt<PREC>(massg, j);
                            sb[j] = st + soff + c * es;
                            soff += Rmax * W * es;
                            const int q = qbase + j * kd;
                            op[j] = slot_ptr_w<PREC>(dst, lay, q, ob_lp, ob_in) +
                                    (int64_t)tl0 * (es == 8 ? tstep_m * 8 : tstep_f * 4);
                        }
                        if constexpr (SPL == 1) {
                            if (massg)
                                strided_consume<KK, PREC, true>(sb, W, rB0, hi_t - lo_t, op, tstep_m, tstep_f, my_cp, wr);
                            else
                                strided_consume<KK, PREC, false>(sb, W, rB0, hi_t - lo_t, op, tstep_m, tstep_f, my_cp, wr);
                        } else if (jh == 0) {
                            if (massg)
                                strided_consume_split<KK, PREC, true, JN, 0>(sb, W, rB0, hi_t - lo_t, op, tstep_m, tstep_f, my_cp, wr);
                            else
                                strided_consume_split<KK, PREC, false, JN, 0>(sb, W, rB0, hi_t - lo_t, op, tstep_m, tstep_f, my_cp, wr);
                        } else {
                            if (massg)
                                strided_consume_split<KK, PREC, true, JN, JN>(sb, W, rB0, hi_t - lo_t, op, tstep_m, tstep_f, my_cp, wr);
                            else
                                strided_consume_split<KK, PREC, false, JN, JN>(sb, W, rB0, hi_t - lo_t, op, tstep_m, tstep_f, my_cp, wr);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                }
            }
        }
    }
    if (threadIdx.x == 0) SLDG_STAMP(2);
    if (producer && lane == 0) SLDG_STAMP(3);
}

// ============================================================================================
// contiguous sweep (d = 0): R whole lines x GC coupled groups per stage.  Every consumer thread
// owns kD0Tpt = 4 consecutive target cells of ONE line of the tile (R = 4 NT / n0 lines when
// n0 <= 4 NT, else R = 1 and ceil(n0 / 4 NT) quads per thread), so its weights are loaded once
// per tile, and the 5 source cells of its 4 targets (target r: A from cell r, B from cell r+1)
// are read from shared memory and promoted once.  A layer's last tile may hold fewer than R
// lines: its box reaches past the layer (TMA fills zeros, never read) and the spare threads idle.
//   tensor maps (5D): {W, L / W, 1, plane, layer}, box {W, cs / W, 1, BP, 1},
//   cs = R n0 cells per stage row: one box = BP consecutive planes of the tile's cells.
// ============================================================================================
constexpr int kD0Tpt = 4;
// k <= kD0RegK: the line's 2k^2 weights live in registers for the whole tile; larger k reads
// them from the line record in shared memory, which then travels with EVERY stage of the tile
constexpr int kD0RegK = 4;

// weight load from the stage's line record: volatile, so the compiler re-reads it where it is
// used instead of hoisting all 2k^2 weights into registers for the whole stage (spills)
__device__ __forceinline__ double lds_f64(const double* p)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

// 4 outputs of one slot -> HBM (16-byte aligned: the quad starts at a multiple of 4 cells)
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d)
{
    __stcs((double2*)p, make_double2(a, b));
    __stcs((double2*)p + 1, make_double2(c, d));
}
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d)
{
    __stcs((float4*)p, make_float4(a, b, c, d));
}

// One coupled group for the thread's 4 targets.  sp: the group's first slot in the stage; slots
// are cs elements apart (CSC = compile-time cs when known, so the shared-memory loads use
// immediate offsets); col[0..4]: stage columns of the 5 source cells.  CP: alpha == 0, exact
// copy of the B-source bits.
template <int KK, int PREC, bool MASSG, bool CP, int CSC>
__device__ __forceinline__ void d0_group(const unsigned char*& sp, int cs_rt, const int* col, double*& om,
                                         float*& of, int64_t L, const double* wr)
{
#define SLDG_DBL(j) ((PREC == SLDG_FP64) || (MASSG && (j) == 0))
    const int cs = CSC ? CSC : cs_rt;
    if (CP) {
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            if (SLDG_DBL(j)) {
                const double* p = (const double*)sp;
                st4(om, p[col[1]], p[col[2]], p[col[3]], p[col[4]]);
                om += L;
                sp += cs * 8;
            } else {
                const float* p = (const float*)sp;
                st4(of, p[col[1]], p[col[2]], p[col[3]], p[col[4]]);
                of += L;
                sp += cs * 4;
            }
        }
        return;
    }
    double v[KK][kD0Tpt + 1];
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        if (SLDG_DBL(j)) {
            const double* p = (const double*)sp;
#pragma unroll
            for (int r = 0; r <= kD0Tpt; ++r) v[j][r] = p[col[r]];
            sp += cs * 8;
        } else {
            const float* p = (const float*)sp;
#pragma unroll
            for (int r = 0; r <= kD0Tpt; ++r) v[j][r] = (double)p[col[r]];
            sp += cs * 4;
        }
    }
    if constexpr (KK > kD0RegK) {
        // weights in shared memory (the stage's line record): each weight is read once and used
        // for the 4 targets; same operation order per target as below.  One output slot per
        // iteration (not unrolled: unrolled, the k = 6 body spilled ~230 registers)
#pragma unroll 1
        for (int j = 0; j < KK; ++j) {
            double oa[kD0Tpt], ob[kD0Tpt];
#pragma unroll
            for (int r = 0; r < kD0Tpt; ++r) oa[r] = ob[r] = 0.0;
#pragma unroll
            for (int l = 0; l < KK; ++l) {
                const double wa = lds_f64(&wr[j * KK + l]), wb = lds_f64(&wr[KK * KK + j * KK + l]);
#pragma unroll
                for (int r = 0; r < kD0Tpt; ++r) {
                    oa[r] = fma(wa, v[l][r], oa[r]);
                    ob[r] = fma(wb, v[l][r + 1], ob[r]);
                }
            }
            if (SLDG_DBL(j)) {
                st4(om, oa[0] + ob[0], oa[1] + ob[1], oa[2] + ob[2], oa[3] + ob[3]);
                om += L;
            } else {
                st4(of, __double2float_rn(oa[0] + ob[0]), __double2float_rn(oa[1] + ob[1]),
                    __double2float_rn(oa[2] + ob[2]), __double2float_rn(oa[3] + ob[3]));
                of += L;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < KK; ++j) {
            double o[kD0Tpt];
#pragma unroll
            for (int r = 0; r < kD0Tpt; ++r) {
                // A- and B-parts as two independent FMA chains (k deep instead of 2k), then one add
                double oa = 0.0, ob = 0.0;
#pragma unroll
                for (int l = 0; l < KK; ++l) {
                    oa = fma(wr[j * KK + l], v[l][r], oa);
                    ob = fma(wr[KK * KK + j * KK + l], v[l][r + 1], ob);
                }
                o[r] = oa + ob;
            }
            if (SLDG_DBL(j)) {
                st4(om, o[0], o[1], o[2], o[3]);
                om += L;
            } else {
                st4(of, __double2float_rn(o[0]), __double2float_rn(o[1]), __double2float_rn(o[2]),
                    __double2float_rn(o[3]));
                of += L;
            }
        }
    }
#undef SLDG_DBL
}

// all gc coupled groups of a stage for the thread's quad of target cells.
// Mixed: om = mass of the first cell, of = plane of slot q0 (or of slot 1 for the mass group);
// fp64: om = slot q0 of the first cell.
template <int KK, int PREC, bool MASSG, bool CP, int CSC>
__device__ __forceinline__ void d0_consume_t(const unsigned char* sbase, int gc, int cs, const int* col, double* om,
                                             float* of, int64_t L, const double* wr)
{
    const unsigned char* sp = sbase;
    int gi = 0;
    if (MASSG) {
        d0_group<KK, PREC, true, CP, CSC>(sp, cs, col, om, of, L, wr);
        gi = 1;
    }
#pragma unroll 1
    for (; gi < gc; ++gi) d0_group<KK, PREC, false, CP, CSC>(sp, cs, col, om, of, L, wr);
}

template <int KK, int PREC, bool MASSG>
__device__ __forceinline__ void d0_consume(const unsigned char* sbase, int gc, int cs, const int* col, double* om,
                                           float* of, int64_t L, int cp, const double* wr)
{
    if (cp) {
        d0_consume_t<KK, PREC, MASSG, true, 0>(sbase, gc, cs, col, om, of, L, wr);
    } else if (cs == 1024) {
        d0_consume_t<KK, PREC, MASSG, false, 1024>(sbase, gc, cs, col, om, of, L, wr);
    } else {
        d0_consume_t<KK, PREC, MASSG, false, 0>(sbase, gc, cs, col, om, of, L, wr);
    }
}

template <int KK, int PREC, int MINB>
__global__ void __launch_bounds__(kTmaThreads, MINB) sweep_d0_tma(Layout lay, Sweep sw, Arrays src, Arrays dst, int64_t lb,
                                                             int64_t le, TmaPlan pl,
                                                             const __grid_constant__ TmapSet tmaps)
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
        for (int h = 0; h < kTmaHeights; ++h) {
            prefetch_tmap(&tmaps.f[h]);
            if (PREC == SLDG_MIXED) prefetch_tmap(&tmaps.m[h]);
        }
    }
    __syncthreads();
    pdl_wait();  // the weights and the source array come from the preceding kernels

    const int D = lay.D;
    const int n0 = (int)lay.n[0];
    const int64_t L = lay.L;
    const int R = pl.R, GC = pl.GC;
    const int64_t lines_per_layer = L / n0;
    const int64_t nblk = (lines_per_layer + R - 1) / R;  // tiles per layer (the last may be partial)
    const int64_t nlay = le - lb;
    const int64_t ntiles = nblk * nlay;
    const int G = lay.K / KK;
    const int NQ = NC * 32 * kD0Tpt;  // cells covered by one pass of the consumer threads
    const int cell_stride = R * n0;    // elements of one slot in a stage
    const int box0 = pl.W;             // first box dim (cells)
    const int BP = GC * KK;            // planes per box
    const uint64_t pol = policy_evict_first();
    // this thread's line of the tile and first cell
    const int q4 = (int)threadIdx.x * kD0Tpt;
    const int my_r = (n0 <= NQ) ? q4 / n0 : 0;
    const int my_c0 = (n0 <= NQ) ? q4 % n0 : q4;
    const int nquad = (n0 <= NQ) ? 1 : (n0 + NQ - 1) / NQ;

    // Line data (A, B, i* mod n, copy flag) travels with the tile's first stage: the producer
    // bulk-copies the tile's packed line records (Weights::rec, 16(k^2+1) bytes each) into the
    // stage's record area, so no thread waits on a global load at a tile boundary and no
    // registers hold a prefetch.
    const int recw = 2 * KK * KK + 2;  // doubles per record
    const int rec_off = pl.stage_bytes - R * recw * 8;

    constexpr bool SMW = KK > kD0RegK;  // weights read from the stage's record (every stage)
    uint32_t it = 0;
    int64_t my_s = 0;
    int my_cp = 0;
    double wr[SMW ? 1 : 2 * KK * KK];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (tile + gridDim.x >= ntiles) pdl_trigger();  // this CTA's last tile
        const int64_t blk = tile % nblk;
        const int64_t layer = lb + tile / nblk;
        const int64_t layerp = lay.pad + layer;
        const int64_t inner_base = blk * R * (int64_t)n0;  // first cell of the tile's first line
        const int rv = (lines_per_layer - blk * R < R) ? (int)(lines_per_layer - blk * R) : R;  // lines in this tile
        const bool has_cell = !producer && my_r < rv;
        for (int g0 = 0; g0 < G; g0 += GC) {
            const int gc = (G - g0) < GC ? (G - g0) : GC;
            const int s = it % S;
            const uint32_t ph = (it / S) & 1;
            ++it;
            unsigned char* st = stage0 + (size_t)s * pl.stage_bytes;
            const bool massg = (PREC == SLDG_MIXED) && g0 == 0;
            if (producer) {
                if (lane == 0) {
                    mbar_wait(&empty[s], ph ^ 1);
                    const uint32_t es = (PREC == SLDG_FP64) ? 8u : 4u;
                    // the mass group: fp64 mass + the group's BP - 1 fp32 planes (tensor map 1)
                    uint32_t bytes = (uint32_t)cell_stride * (massg ? (BP - 1) * 4u + 8u : BP * es);
                    if (g0 == 0 || SMW) bytes += (uint32_t)((pl.rec1 ? 1 : rv) * recw * 8);
                    mbar_expect_tx(&full[s], bytes);
                    const int c1 = (int)(inner_base / box0);
                    if (massg) {
                        tma_5d(st, &tmaps.m[0], 0, c1, 0, 0, (int)layerp, &full[s], pol);
                        tma_5d(st + cell_stride * 8, &tmaps.f[1], 0, c1, 0, 0, (int)layerp, &full[s], pol);
                    } else {
                        const int plane0 = (PREC == SLDG_FP64) ? g0 * KK : g0 * KK - 1;
                        tma_5d(st, &tmaps.f[0], 0, c1, 0, plane0, (int)layerp, &full[s], pol);
                    }
                    if (g0 == 0 || SMW) {
                        for (int r = 0; r < (pl.rec1 ? 1 : rv); ++r) {  // the tile's line records
                            int64_t f = 0;
                            if (sw.fmask) {  // 32-bit index math: this thread feeds the whole CTA
                                int64_t idx[kMaxDim];
                                uint32_t rem2 = (uint32_t)(blk * R + r);  // line index within the layer
#pragma unroll
                                for (int e = 0; e < kMaxDim; ++e) idx[e] = 0;
                                for (int e = 1; e < D - 1; ++e) {
                                    const uint32_t ne = (uint32_t)lay.n[e];
                                    const uint32_t q = rem2 / ne;
                                    idx[e] = rem2 - q * ne;
                                    rem2 = q;
                                }
                                if (D >= 2) idx[D - 1] = lay.first_layer + layer;
                                f = tfield_index(sw, idx, D);
                            }
                            bulk_g2s(st + rec_off + r * recw * 8, sw.rec + f * recw, (uint32_t)(recw * 8), &full[s], pol);
                        }
                    }
                }
                __syncwarp();
            } else {
                mbar_wait(&full[s], ph);
                const double* rp = (const double*)(st + rec_off) + (pl.rec1 ? 0 : my_r) * recw;
                if (g0 == 0 && has_cell) {  // this tile's line data for my line
                    if (!SMW) {
#pragma unroll
                        for (int i = 0; i < 2 * KK * KK; ++i) wr[i] = rp[i];
                    }
                    my_s = __double_as_longlong(rp[2 * KK * KK]);
                    my_cp = (int)__double_as_longlong(rp[2 * KK * KK + 1]);
                }
                if (has_cell) {
                    for (int ci = 0; ci < nquad; ++ci) {
                        const int cc = my_c0 + ci * NQ;  // first target cell of the quad within the line
                        if (cc >= n0) break;
                        const int row0 = my_r * n0;
                        int col[kD0Tpt + 1];
                        int c = cc - (int)my_s - 1;  // A-source of target cc (i* mod n in [0, n0))
                        if (c < 0) c += n0;
#pragma unroll
                        for (int r = 0; r <= kD0Tpt; ++r) {
                            col[r] = row0 + c;
                            c = (c + 1 == n0) ? 0 : c + 1;
                        }
                        const int64_t tin = inner_base + row0 + cc;
                        const int q0 = g0 * KK;
                        double* om;
                        float* of = nullptr;
                        if (PREC == SLDG_FP64) {
                            om = dst.s64 + toff_m<PREC>(lay, layerp, tin) + (int64_t)q0 * L;
                        } else {
                            om = dst.mass + toff_m<PREC>(lay, layerp, tin);
                            of = dst.pl + toff_f<PREC>(lay, layerp, tin) + (massg ? 0 : (int64_t)(q0 - 1) * L);
                        }
                        const double* wsrc = SMW ? rp : wr;
                        if (massg)
                            d0_consume<KK, PREC, true>(st, gc, cell_stride, col, om, of, L, my_cp, wsrc);
                        else
                            d0_consume<KK, PREC, false>(st, gc, cell_stride, col, om, of, L, my_cp, wsrc);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
        }
    }
}

// ============================================================================================
// d = 0 for lines too long for two whole-line stages (fp64 k >= 4, mixed k >= 7 at n0 = 4096):
// tile = one WINDOW of cw = pl.T consecutive targets [a, a + cw) of one line (R = 1).  By
// P:259-272 target i reads cells i - i* - 1 and i - i*, so the window's sources are the cw + 1
// cells from ws = (a - i* - 1) mod n0 -- rounded down to a multiple of 4 cells (rofs) so every
// copy is 16-byte aligned -- loaded per plane as one 1D bulk copy, two where the periodic line
// wraps.  The producer reads i* mod n0 of the line (Weights::smod) at the tile's first stage;
// the consumers take it from the line record and compute the same rofs, and a target's source
// columns are then (target - a) + rofs + r: no modulo.  Stage layout as sweep_d0_tma (slot
// stride pl.Rmax cells, the line record at the end); the consumer code is the same d0_consume.
// ============================================================================================
template <int KK, int PREC>
__global__ void __launch_bounds__(kTmaThreads, 1) sweep_d0_win(Layout lay, Sweep sw, Arrays src, Arrays dst, int64_t lb,
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
    pdl_wait();  // the weights and the source array come from the preceding kernels

    const int D = lay.D;
    const int n0 = (int)lay.n[0];
    const int64_t L = lay.L;
    const int cw = pl.T;                       // targets per window
    const int cs = pl.Rmax;                    // stage slot stride (cells)
    const int nwin = (n0 + cw - 1) / cw;
    const int64_t lines_per_layer = L / n0;
    const int64_t nblk = lines_per_layer * nwin;
    const int64_t ntiles = nblk * (le - lb);
    const int G = lay.K / KK, GC = pl.GC;
    const int BP = GC * KK;
    const int NQ = NC * 32 * kD0Tpt;
    const uint64_t pol = policy_evict_first();
    const int recw = 2 * KK * KK + 2;
    const int rec_off = pl.stage_bytes - recw * 8;
    constexpr bool SMW = KK > kD0RegK;
    const int q4 = (int)threadIdx.x * kD0Tpt;
    uint32_t it = 0;
    int64_t my_s = 0;
    int my_cp = 0;
    double wr[SMW ? 1 : 2 * KK * KK];
    int64_t f = 0;            // producer: field entry of the tile's line
    int ws = 0, p1 = 0, p2 = 0;  // producer: window start (cells) and its two pieces
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (tile + gridDim.x >= ntiles) pdl_trigger();  // this CTA's last tile
        const int64_t blk = tile % nblk;
        const int64_t layer = lb + tile / nblk;
        const int64_t layerp = lay.pad + layer;
        const int64_t line = blk / nwin;
        const int a = (int)(blk - line * nwin) * cw;
        const int ct = (n0 - a < cw) ? n0 - a : cw;  // targets in this window (multiple of 4)
        const int64_t line_base = line * n0;
        for (int g0 = 0; g0 < G; g0 += GC) {
            const int gc = (G - g0) < GC ? (G - g0) : GC;
            const int s = it % S;
            const uint32_t ph = (it / S) & 1;
            ++it;
            unsigned char* st = stage0 + (size_t)s * pl.stage_bytes;
            const bool massg = (PREC == SLDG_MIXED) && g0 == 0;
            if (producer) {
                if (lane == 0) {
                    if (g0 == 0) {
                        f = 0;
                        if (sw.fmask) {
                            int64_t idx[kMaxDim];
                            int64_t rem = line;
#pragma unroll
                            for (int e = 0; e < kMaxDim; ++e) idx[e] = 0;
                            for (int e = 1; e < D - 1; ++e) {
                                idx[e] = rem % lay.n[e];
                                rem /= lay.n[e];
                            }
                            if (D >= 2) idx[D - 1] = lay.first_layer + layer;
                            f = tfield_index(sw, idx, D);
                        }
                        int w0 = a - (int)__ldg(&sw.smod[f]) - 1;  // A-source of target a, mod n0
                        if (w0 < 0) w0 += n0;
                        const int rofs = w0 & 3;
                        ws = w0 - rofs;
                        const int cnt = (ct + 1 + rofs + 3) & ~3;
                        p1 = (cnt < n0 - ws) ? cnt : n0 - ws;
                        p2 = cnt - p1;
                    }
                    mbar_wait(&empty[s], ph ^ 1);
                    const uint32_t es = (PREC == SLDG_FP64) ? 8u : 4u;
                    const uint32_t cb = (uint32_t)(p1 + p2);
                    uint32_t bytes = cb * (massg ? (BP - 1) * 4u + 8u : (uint32_t)gc * KK * es);
                    if (g0 == 0 || SMW) bytes += (uint32_t)(recw * 8);
                    mbar_expect_tx(&full[s], bytes);
                    unsigned char* dp = st;
                    for (int j = 0; j < gc * KK; ++j) {
                        const int q = g0 * KK + j;
                        const uint32_t ej = (PREC == SLDG_FP64 || (massg && j == 0)) ? 8u : 4u;
                        const char* sp = slot_ptr<PREC>(src, lay, q, layerp, line_base);
                        bulk_g2s(dp, sp + (size_t)ws * ej, (uint32_t)p1 * ej, &full[s], pol);
                        if (p2) bulk_g2s(dp + (size_t)p1 * ej, sp, (uint32_t)p2 * ej, &full[s], pol);
                        dp += (size_t)cs * ej;
                    }
                    if (g0 == 0 || SMW) bulk_g2s(st + rec_off, sw.rec + f * recw, (uint32_t)(recw * 8), &full[s], pol);
                }
                __syncwarp();
            } else {
                mbar_wait(&full[s], ph);
                const double* rp = (const double*)(st + rec_off);
                if (g0 == 0) {
                    if (!SMW) {
#pragma unroll
                        for (int i = 0; i < 2 * KK * KK; ++i) wr[i] = rp[i];
                    }
                    my_s = __double_as_longlong(rp[2 * KK * KK]);
                    my_cp = (int)__double_as_longlong(rp[2 * KK * KK + 1]);
                }
                int w0 = a - (int)my_s - 1;
                if (w0 < 0) w0 += n0;
                const int rofs = w0 & 3;
                for (int cc = q4; cc < ct; cc += NQ) {
                    int col[kD0Tpt + 1];
#pragma unroll
                    for (int r = 0; r <= kD0Tpt; ++r) col[r] = cc + rofs + r;
                    const int64_t tin = line_base + a + cc;
                    const int q0 = g0 * KK;
                    double* om;
                    float* of = nullptr;
                    if (PREC == SLDG_FP64) {
                        om = dst.s64 + toff_m<PREC>(lay, layerp, tin) + (int64_t)q0 * L;
                    } else {
                        om = dst.mass + toff_m<PREC>(lay, layerp, tin);
                        of = dst.pl + toff_f<PREC>(lay, layerp, tin) + (massg ? 0 : (int64_t)(q0 - 1) * L);
                    }
                    const double* wsrc = SMW ? rp : wr;
                    if (massg)
                        d0_consume<KK, PREC, true>(st, gc, cs, col, om, of, L, my_cp, wsrc);
                    else
                        d0_consume<KK, PREC, false>(st, gc, cs, col, om, of, L, my_cp, wsrc);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
        }
    }
}

// ============================================================================================
// planning, tensor maps, launch
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

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encoder()
{
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// 5D tile tensor map; dims/strides in elements (stride[0] = 1 implied), box in elements
static bool make_tmap(CUtensorMap* tm, bool f64, void* base, const int64_t* dims, const int64_t* strides,
                      const int* box)
{
    EncodeTiledFn enc = encoder();
    if (!enc) return false;
    const int es = f64 ? 8 : 4;
    cuuint64_t gd[5], gs[4];
    cuuint32_t bd[5], estr[5] = {1, 1, 1, 1, 1};
    for (int i = 0; i < 5; ++i) {
        gd[i] = (cuuint64_t)dims[i];
        bd[i] = (cuuint32_t)box[i];
    }
    for (int i = 0; i < 4; ++i) gs[i] = (cuuint64_t)strides[i + 1] * es;
    CUresult r = enc(tm, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, base, gd, gs, bd,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

void ensure_max_smem(const void* func)
{
    static std::mutex mu;
    static std::vector<std::pair<int, const void*>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    for (auto& d : done)
        if (d.first == dev && d.second == func) return;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    done.push_back({dev, func});
}

bool make_tmap5(CUtensorMap* tm, bool f64, void* base, const int64_t* dims, const int64_t* strides, const int* box)
{
    return make_tmap(tm, f64, base, dims, strides, box);
}

void tma_device_info(int* num_sms, int* smem_optin)
{
    query_device();
    *num_sms = g_num_sms;
    *smem_optin = g_smem_optin;
}

// Returns true and fills `pl` when the TMA path applies to this sweep.
static bool tma_plan_ctas(const Layout& lay, const Sweep& sw, TmaPlan* pl, int force_ctas);

bool tma_plan(const Layout& lay, const Sweep& sw, TmaPlan* pl)
{
    *pl = TmaPlan{};
    if (tma_plan_ctas(lay, sw, pl, 0)) return true;
    // a k <= 2 plan with 2 CTAs per SM halves the shared memory per CTA; a stage that no longer
    // fits twice (e.g. a 4096-cell line of the mass group) still fits with one CTA
    if (pl->ctas == 2 && !getenv("SLDG_TMA_CTAS")) return tma_plan_ctas(lay, sw, pl, 1);
    return false;
}

static bool tma_plan_ctas(const Layout& lay, const Sweep& sw, TmaPlan* pl, int force_ctas)
{
    query_device();
    if (!encoder()) return false;
    const int64_t n0 = lay.n[0];
    const int k = lay.k;
    // CTAs per SM (SLDG_TMA_CTAS=2: two CTAs, each with half the shared memory and <= 96
    // registers per thread -- twice the warps to hide latency, at the cost of spills)
    // Measured: k <= 2 fits 96 registers without hurtful spills and gains from the extra warps
    // (C4 64^4 k=2: 375 -> 467 GDoF/s); k = 3 loses (C5: 693 -> 643 GDoF/s).
    // Per sweep kind (C4 64^4 k = 2, profiles/round1/tuning.md): the d = 0 sweep and strided
    // sweeps over fewer than 256 cells below d gain from 2 CTAs (d0 3.8 vs 2.7 TB/s), strided
    // sweeps with full 256-column rows from 1 CTA with twice the stage (4.9 / 5.3 vs 4.5 / 4.8).
    int ctas = (k <= 2) ? 2 : 1;
    if (k <= 2 && sw.dim > 0) {
        int64_t mlo = 1;
        for (int e = 0; e < ((sw.dim == lay.D - 1) ? lay.D - 1 : sw.dim); ++e) mlo *= lay.n[e];
        if (mlo % 256 == 0) ctas = 1;
    }
    if (const char* e = getenv("SLDG_TMA_CTAS")) ctas = (atoi(e) == 2) ? 2 : 1;
    if (force_ctas) ctas = force_ctas;
    const int64_t budget = std::min<int64_t>(g_smem_optin, 200 * 1024) / ctas - 256 - (ctas - 1) * 1024;
    const int bpc_max = (lay.prec == SLDG_FP64) ? 8 * k : 8 + 4 * (k - 1);  // bytes per column, mass group
    const int NT = kTmaConsumerWarps * 32;
    *pl = TmaPlan{};
    pl->ctas = ctas;
    // strided: the line weights live in registers (k <= 4 one thread per column, k = 5, 6 two
    // threads per column with half the output slots each); k >= 7 uses the register kernels.
    // d = 0: k <= 4 in registers, 5..8 from the record in shared memory (kD0RegK)
    if (k > 8 || (k > 6 && sw.dim != 0)) return false;
    // fp64 k = 5, 6 strided: the split TMA kernel (round 2, C3 4096^2: 1.26 / 1.78 ms against the
    // register kernel's 2.08 / 4.89 ms; profiles/round2/d0win ab_*); SLDG_TMA_F64HI=0 selects the latter
    if (k > 4 && sw.dim != 0 && lay.prec == SLDG_FP64 && getenv("SLDG_TMA_F64HI") && atoi(getenv("SLDG_TMA_F64HI")) == 0)
        return false;
    if (n0 % 4 != 0) return false;
    const int64_t layers_alloc = lay.layers + 2 * lay.pad;
    if (lay.L > (int64_t)1 << 31 || layers_alloc > 65535) return false;
    if (sw.dim == 0) {
        // 4 consecutive targets per consumer thread (kD0Tpt): R lines of n0 cells per tile
        const int64_t NQ = (int64_t)NT * 4;
        const int64_t lines = lay.L / n0;
        int64_t R = (n0 <= NQ) ? std::min<int64_t>(NQ / n0, lines) : 1;
        // lines too long for two whole-line stages (or whose length is not a multiple of 16
        // cells): windows of cw targets (sweep_d0_win), one group per stage, the fewest windows
        // per line whose two stages fit the opt-in carveout
        auto try_win = [&]() -> bool {
            if (ctas != 1 || n0 < 64) return false;
            const int es = (lay.prec == SLDG_FP64) ? 8 : 4;
            const int64_t recb = (int64_t)(2 * k * k + 2) * 8;
            const int64_t budget_max = (int64_t)g_smem_optin - 256;
            for (int nwin = 2; nwin <= 64; nwin *= 2) {
                const int64_t cw = ((n0 + nwin - 1) / nwin + 3) / 4 * 4;
                const int64_t wcs = (cw + 8 + 15) / 16 * 16;  // cw + 1 sources + rofs <= 3, rounded to 4
                const int64_t sb = ((wcs * (k * es + ((lay.prec == SLDG_FP64) ? 0 : 4)) + 127) / 128 * 128 + recb + 127) /
                                   128 * 128;
                if (2 * sb > budget_max) continue;
                pl->R = 1;
                pl->GC = 1;
                pl->rec1 = 1;
                pl->T = (int)cw;
                pl->Rmax = (int)wcs;
                pl->stage_bytes = (int)sb;
                pl->stages = (int)std::min<int64_t>(8, std::max<int64_t>(2, budget / sb));
                if ((int64_t)pl->stages * sb > budget_max) pl->stages = 2;
                return true;
            }
            return false;
        };
        // windows also for long mixed k >= 6 lines (C3 k = 6: 1.23 vs 1.29 ms whole-line; slower for
        // k <= 5: 0.14 / 0.25 / 0.46 / 0.84 vs 0.125 / 0.22 / 0.43 / 0.82 ms, profiles/round2/d0win ab_*);
        // SLDG_D0_WIN=1 / 0 forces / forbids them where both apply
        {
            const char* e = getenv("SLDG_D0_WIN");
            const bool want_win = e ? atoi(e) == 1 : (k >= 6);
            if (n0 > NQ && want_win && try_win()) return true;
        }
        while (R > 1 && (R * n0) % 16 != 0) --R;  // stage slots stay 64-byte multiples
        if ((R * n0) % 16 != 0) return n0 > NQ ? try_win() : false;
        const int64_t cs = R * n0;
        const int64_t group_bytes = cs * bpc_max;  // one coupled group of the tile, worst case
        const int G = lay.K / k;
        int64_t d0div = (k <= 2) ? 2 : 3;  // stage <= budget / d0div (C4: 2 beats 3, 3.8 -> 4.1 TB/s; override SLDG_TMA_D0DIV)
        if (const char* e = getenv("SLDG_TMA_D0DIV")) d0div = atoi(e);
        const int64_t target = budget / d0div;
        if (group_bytes > std::max<int64_t>(budget, (int64_t)g_smem_optin / ctas - 256) / 2) return try_win();
        int gcmax = (int)std::max<int64_t>(1, std::min<int64_t>(G, target / group_bytes));
        const int nchunk = (G + gcmax - 1) / gcmax;
        const int GC = (G + nchunk - 1) / nchunk;  // balanced chunks
        if (GC * k > 256) return false;
        pl->R = (int)R;
        pl->GC = GC;
        // the R lines of a tile share their field entry when every masked dim among 1..D-2
        // changes only every (lines per step of that dim) % R == 0 lines: one record per tile
        {
            bool one = true;
            int64_t stride = 1;  // lines per step of dim e
            for (int e = 1; e < lay.D - 1; ++e) {
                if ((sw.fmask >> e & 1u) && stride % R != 0) one = false;
                stride *= lay.n[e];
            }
            pl->rec1 = one ? 1 : 0;
        }
        // first box dim: the largest power of two <= 256 dividing cs and L (tiles start at
        // multiples of cs, so at multiples of W)
        int W = 256;
        while (W > 16 && (cs % W != 0 || lay.L % W != 0)) W >>= 1;
        if (cs % W != 0 || lay.L % W != 0 || cs / W > 256) return false;
        pl->W = W;
        const int es = (lay.prec == SLDG_FP64) ? 8 : 4;
        // stage: GC*k planes, or for the mixed mass group the fp64 mass + GC*k - 1 fp32 planes
        // (max: GC*k*4 + 4 bytes per cell), + the tile's R packed line records at the end
        // (16-byte aligned: 16(k^2+1) bytes each; stage starts stay 128-byte aligned for the
        // tensor copies; records end the stage)
        if (lay.prec != SLDG_FP64 && GC * k < 2) return false;
        pl->stage_bytes = (int)(((cs * (GC * k * es + ((lay.prec == SLDG_FP64) ? 0 : 4)) + 127) / 128 * 128 +
                                 R * (2 * k * k + 2) * 8 + 127) / 128 * 128);
        pl->stages = (int)std::min<int64_t>(8, budget / pl->stage_bytes);
        // large stages (a long line of k >= 5): two of them may use the whole opt-in carveout
        const int64_t budget_max = (int64_t)g_smem_optin / ctas - 256 - (ctas - 1) * 1024;
        if (pl->stages < 2 && 2LL * pl->stage_bytes <= budget_max) pl->stages = 2;
        return pl->stages >= 2;
    }
    const bool outer = (sw.dim == lay.D - 1);
    int64_t M_lo = 1;
    for (int e = 0; e < (outer ? lay.D - 1 : sw.dim); ++e) M_lo *= lay.n[e];
    // sub-chunk Tsub targets; stage rows Rmax = Tsub + 1 + 3 (shift spans up to 3 cells)
    int W = 0, Tsub = 0;
    // Measured on B200 (tools/tune_tma.sh, profiles/round1/tuning.md): few LARGE stages beat many
    // small ones -- per-stage consumer overhead (barrier round trip, pointer setup, the A-part
    // prologue row) is amortised over more targets.  Default: 2 stages, Tsub as large as fits.
    int Tsub0 = 64;
    int Wmax = 256;
    int64_t sdiv = 2;  // stage <= budget / sdiv
    if (const char* e = getenv("SLDG_TMA_W")) Wmax = atoi(e);        // tuning overrides
    if (const char* e = getenv("SLDG_TMA_TSUB")) Tsub0 = atoi(e);
    if (const char* e = getenv("SLDG_TMA_SDIV")) sdiv = atoi(e);
    // Widest tile first.  A grid short of tiles (< 4 per SM at that width, e.g. C2's 1024-layer v
    // sweep) takes W = 64 instead: more column tiles AND a stage row 4x narrower, so Tsub reaches
    // its cap (measured on C2: 1.71 -> 2.04 TB/s; W = 32 is slower, profiles/round1/tuning.md).
    int64_t perp = outer ? 1 : lay.layers;  // tiles along the dims other than lo and d
    if (!outer)
        for (int e = sw.dim + 1; e < lay.D - 1; ++e) perp *= lay.n[e];
    const int64_t nline_p = outer ? lay.layers : sw.nd;
    for (int w : {256, 128, 64, 32}) {
        if (M_lo % w != 0 || w > Wmax) continue;
        if (k > 4 && w > NT / 2) continue;  // two threads per column (strided_consume_split)
        int ts = (int)std::min<int64_t>(Tsub0, budget / sdiv / ((int64_t)w * bpc_max) - 4);
        if (ts < 4) continue;
        W = w;
        Tsub = ts;
        break;
    }
    if (W > 64 && M_lo % 64 == 0 && !getenv("SLDG_TMA_W")) {
        const int64_t tiles = (M_lo / W) * perp * ((nline_p + Tsub - 1) / Tsub);
        const int ts64 = (int)std::min<int64_t>(Tsub0, budget / sdiv / (64LL * bpc_max) - 4);
        if (tiles < 4LL * g_num_sms * ctas && ts64 >= 4) {
            W = 64;
            Tsub = ts64;
        }
    }
    if (W == 0) return false;
    const int Rmax = Tsub + 4;
    const int64_t stage = (int64_t)Rmax * W * bpc_max;
    const int stage_bytes = (int)((stage + 127) / 128 * 128);
    const int stages = (int)std::min<int64_t>(8, budget / stage_bytes);
    if (stages < 2) return false;
    // tile length along d: whole lines (one line-data fetch per tile) unless that leaves fewer
    // than 4 tiles per SM, then the lines are cut into segments (multiples of Tsub)
    const int64_t nline = outer ? lay.layers : sw.nd;
    int64_t base = (M_lo / W) * (outer ? 1 : lay.layers);
    if (!outer)
        for (int e = sw.dim + 1; e < lay.D - 1; ++e) base *= lay.n[e];
    const int64_t want = 4LL * g_num_sms;
    int64_t nseg = std::max<int64_t>(1, (want + base - 1) / base);
    int64_t T = (nline + nseg - 1) / nseg;
    T = std::max<int64_t>(Tsub, (T + Tsub - 1) / Tsub * Tsub);
    pl->W = W;
    pl->T = (int)T;
    pl->Tsub = Tsub;
    // producer-computed tile spans (PSPAN) for short tiles: there the per-tile code runs often and
    // its compact form pays (2D strided sweeps k = 2..4 +7-20%, C4 dims 2/3 +4-6%); tiles of many
    // stages (C5: 27 groups x 7 sub-chunks) keep the other instance, whose hot loop the compiler
    // schedules 6 instructions shorter for k = 3 (C5 strided 4-7% faster); the 2-CTA instance
    // measured slower with it (C4 dim 1).  profiles/round1/tuning.md
    const int64_t stages_per_tile = (int64_t)(lay.K / k) * ((T + Tsub - 1) / Tsub);
    pl->pspan = (ctas == 1 && stages_per_tile <= 64) ? 1 : 0;
    if (const char* e = getenv("SLDG_TMA_PSPAN")) pl->pspan = atoi(e) ? 1 : 0;
    pl->Rmax = Rmax;
    pl->stage_bytes = stage_bytes;
    pl->stages = stages;
    return true;
}

// tensor maps of the source array for a sweep.  d0: one box shape (index 0).  Strided: box
// heights 2^h rows, h = 0..kTmaHeights-1 (index h).
static bool build_tmaps(const Layout& lay, const Sweep& sw, const Arrays& src, const TmaPlan& pl, TmapSet* ts)
{
    const bool f64 = lay.prec == SLDG_FP64;
    const int64_t P = f64 ? lay.K : lay.K - 1;  // planes in the fp32 (or fp64) array
    const int64_t layers_alloc = lay.layers + 2 * lay.pad;
    const int64_t L = lay.L;
    void* fbase = f64 ? (void*)src.s64 : (void*)src.pl;
    if (sw.dim == 0) {
        const int64_t b0 = pl.W, cs = (int64_t)pl.R * lay.n[0];
        const int64_t dm[5] = {b0, L / b0, 1, P, layers_alloc};
        const int64_t sm[5] = {1, b0, L, L, L * P};
        const int bx[5] = {(int)b0, (int)(cs / b0), 1, pl.GC * lay.k, 1};
        if (!make_tmap(&ts->f[0], f64, fbase, dm, sm, bx)) return false;
        if (!f64) {
            // the mass group's planes: slots 1 .. GC k - 1 (no spare plane in its stage)
            const int bx1[5] = {(int)b0, (int)(cs / b0), 1, pl.GC * lay.k - 1, 1};
            if (!make_tmap(&ts->f[1], f64, fbase, dm, sm, bx1)) return false;
            const int64_t dmm[5] = {b0, L / b0, 1, 1, layers_alloc};
            const int64_t smm[5] = {1, b0, L, L, L};
            const int bxm[5] = {(int)b0, (int)(cs / b0), 1, 1, 1};
            if (!make_tmap(&ts->m[0], true, src.mass, dmm, smm, bxm)) return false;
        }
        return true;
    }
    const bool outer = (sw.dim == lay.D - 1);
    int64_t M_lo = 1, M_hi = 1;
    for (int e = 0; e < (outer ? lay.D - 1 : sw.dim); ++e) M_lo *= lay.n[e];
    if (!outer)
        for (int e = sw.dim + 1; e < lay.D - 1; ++e) M_hi *= lay.n[e];
    const int64_t nd = outer ? 1 : sw.nd;
    for (int h = 0; h < kTmaHeights; ++h) {
        const int rowsb = 1 << h;
        const int64_t dm[5] = {M_lo, nd, M_hi, P, layers_alloc};
        const int64_t sm[5] = {1, M_lo, M_lo * nd, L, L * P};
        const int bx[5] = {pl.W, outer ? 1 : rowsb, 1, 1, outer ? rowsb : 1};
        if (!make_tmap(&ts->f[h], f64, fbase, dm, sm, bx)) return false;
        if (!f64) {
            const int64_t dmm[5] = {M_lo, nd, M_hi, 1, layers_alloc};
            const int64_t smm[5] = {1, M_lo, M_lo * nd, L, L};
            if (!make_tmap(&ts->m[h], true, src.mass, dmm, smm, bx)) return false;
        }
    }
    return true;
}

// Encoding 10 tensor maps costs tens of microseconds of host time per sweep, which matters for
// small grids; the maps only depend on the source buffer, the layout and the plan, so they are
// cached (two ping-pong buffers x D dims per grid; mutex-protected, handles may live on
// different threads).
// The key holds everything build_tmaps reads: the buffers, the device, the whole shape (two grids
// with equal L and n[dim] but a different split of L into the dims below / above dim encode
// different maps) and the plan.  sldg_destroy and the transpose path drop the entries of the
// buffers they free (tmap_cache_forget), so a new allocation at a recycled address never hits.
struct TmapCacheEntry {
    bool valid = false;
    const void* f = nullptr;
    const void* m = nullptr;
    int device = 0, prec = 0, D = 0, dim = 0, W = 0, T = 0, Rmax = 0, R = 0, GC = 0;
    int64_t n[kMaxDim] = {};
    int64_t L = 0, layers = 0, pad = 0, nd = 0, K = 0;
    TmapSet maps;
};
static std::mutex g_tmap_mu;
static TmapCacheEntry g_tmap_cache[32];
static int g_tmap_next = 0;

void tmap_cache_forget(const void* base, size_t bytes)
{
    if (!base) return;
    const char* lo = (const char*)base;
    const char* hi = lo + bytes;
    std::lock_guard<std::mutex> lock(g_tmap_mu);
    for (auto& e : g_tmap_cache) {
        const char* f = (const char*)e.f;
        const char* m = (const char*)e.m;
        if (e.valid && ((f >= lo && f < hi) || (m >= lo && m < hi))) e.valid = false;
    }
}

static bool same_shape(const TmapCacheEntry& e, const Layout& lay)
{
    if (e.D != lay.D || e.prec != lay.prec) return false;
    for (int i = 0; i < kMaxDim; ++i)
        if (e.n[i] != (i < lay.D ? lay.n[i] : 0)) return false;
    return true;
}

static bool cached_tmaps(const Layout& lay, const Sweep& sw, const Arrays& src, const TmaPlan& pl, TmapSet* out)
{
    const void* f = lay.prec == SLDG_FP64 ? (const void*)src.s64 : (const void*)src.pl;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_tmap_mu);
    for (auto& e : g_tmap_cache)
        if (e.valid && e.f == f && e.m == src.mass && e.device == dev && e.dim == sw.dim && e.W == pl.W &&
            e.T == pl.T && e.Rmax == pl.Rmax && e.R == pl.R && e.GC == pl.GC && e.L == lay.L &&
            e.layers == lay.layers && e.pad == lay.pad && e.nd == sw.nd && e.K == lay.K && same_shape(e, lay)) {
            *out = e.maps;
            return true;
        }
    TmapCacheEntry& e = g_tmap_cache[g_tmap_next];
    g_tmap_next = (g_tmap_next + 1) % 32;
    memset(&e.maps, 0, sizeof(e.maps));
    if (!build_tmaps(lay, sw, src, pl, &e.maps)) {
        e.valid = false;
        return false;
    }
    e.valid = true;
    e.f = f;
    e.m = src.mass;
    e.device = dev;
    e.prec = lay.prec;
    e.D = lay.D;
    for (int i = 0; i < kMaxDim; ++i) e.n[i] = (i < lay.D) ? lay.n[i] : 0;
    e.dim = sw.dim;
    e.W = pl.W;
    e.T = pl.T;
    e.Rmax = pl.Rmax;
    e.R = pl.R;
    e.GC = pl.GC;
    e.L = lay.L;
    e.layers = lay.layers;
    e.pad = lay.pad;
    e.nd = sw.nd;
    e.K = lay.K;
    *out = e.maps;
    return true;
}

template <int KK, int PREC>
static cudaError_t launch_tma_k(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst, int64_t lb,
                                int64_t le, const TmaPlan& pl, cudaStream_t s)
{
    const size_t smem = 256 + (size_t)pl.stages * pl.stage_bytes;
    if (sw.dim == 0 && pl.T > 0) {  // windowed d = 0 (no tensor maps: 1D bulk copies)
        const int64_t nwin = (lay.n[0] + pl.T - 1) / pl.T;
        const int64_t ntw = (lay.L / lay.n[0]) * nwin * (le - lb);
        auto kern = sweep_d0_win<KK, PREC>;
        ensure_max_smem((const void*)kern);
        int64_t grid = std::min<int64_t>(ntw, (int64_t)std::max(1, g_num_sms - sw.sm_reserve));
        if (grid < 1) return cudaSuccess;
        return launch_pdl(kern, dim3((unsigned)grid), dim3(kTmaThreads), smem, s, lay, sw, src, dst, lb, le, pl);
    }
    TmapSet tmaps;
    if (!cached_tmaps(lay, sw, src, pl, &tmaps)) return cudaErrorInvalidValue;
    int64_t ntiles;
    const int per_sm = pl.ctas;  // CTAs per SM the plan sized shared memory for
    if (sw.dim == 0) {
        ntiles = ((lay.L / lay.n[0] + pl.R - 1) / pl.R) * (le - lb);
        auto kern = (pl.ctas == 2) ? sweep_d0_tma<KK, PREC, 2> : sweep_d0_tma<KK, PREC, 1>;
        ensure_max_smem((const void*)kern);  // full opt-in carveout
        int64_t grid = std::min<int64_t>(ntiles, (int64_t)std::max(1, g_num_sms - sw.sm_reserve) * per_sm);
        if (grid < 1) return cudaSuccess;
        cudaError_t le0 = launch_pdl(kern, dim3((unsigned)grid), dim3(kTmaThreads), smem, s, lay, sw, src, dst, lb, le, pl,
                                     tmaps);
        if (le0 != cudaSuccess) return le0;
    } else if constexpr (KK <= 6) {
        const bool outer = (sw.dim == lay.D - 1);
        const int64_t nline = outer ? (le - lb) : sw.nd;
        int64_t M_lo = 1, M_hi = 1;
        for (int e = 0; e < (outer ? lay.D - 1 : sw.dim); ++e) M_lo *= lay.n[e];
        if (!outer)
            for (int e = sw.dim + 1; e < lay.D - 1; ++e) M_hi *= lay.n[e];
        ntiles = ((nline + pl.T - 1) / pl.T) * (M_lo / pl.W) * M_hi * (outer ? 1 : (le - lb));
        auto kern = (pl.ctas == 2) ? (pl.pspan ? sweep_strided_tma<KK, PREC, 2, true> : sweep_strided_tma<KK, PREC, 2, false>)
                                   : (pl.pspan ? sweep_strided_tma<KK, PREC, 1, true> : sweep_strided_tma<KK, PREC, 1, false>);
        ensure_max_smem((const void*)kern);  // full opt-in carveout
        int64_t grid = std::min<int64_t>(ntiles, (int64_t)std::max(1, g_num_sms - sw.sm_reserve) * per_sm);
        if (grid < 1) return cudaSuccess;
        cudaError_t le1 = launch_pdl(kern, dim3((unsigned)grid), dim3(kTmaThreads), smem, s, lay, sw, src, dst, lb, le, pl,
                                     tmaps);
        if (le1 != cudaSuccess) return le1;
#ifdef SLDG_STAMPS
        {
            std::vector<unsigned long long> h((size_t)8 * grid);
            cudaStreamSynchronize(s);
            cudaMemcpyFromSymbol(h.data(), g_stamp, h.size() * 8);
            unsigned long long t0 = ~0ull;
            for (int64_t b = 0; b < grid; ++b) t0 = std::min(t0, h[8 * b]);
            std::vector<double> st, ff, cd, pd, pe, pi, cw;
            for (int64_t b = 0; b < grid; ++b) {
                st.push_back((h[8 * b] - t0) * 1e-3);
                ff.push_back((h[8 * b + 1] - h[8 * b]) * 1e-3);
                cd.push_back((h[8 * b + 2] - t0) * 1e-3);
                pd.push_back((h[8 * b + 3] - t0) * 1e-3);
                pe.push_back((h[8 * b + 4] - h[8 * b]) * 1e-3);
                pi.push_back((h[8 * b + 5] - h[8 * b]) * 1e-3);
                cw.push_back((h[8 * b + 6] - h[8 * b]) * 1e-3);
            }
            auto q = [](std::vector<double> v, double f) {
                std::sort(v.begin(), v.end());
                return v[(size_t)(f * (v.size() - 1) + 0.5)];
            };
            fprintf(stderr,
                    "SLDG_STAMP strided dim=%d W=%d T=%d Tsub=%d stages=%d pspan=%d grid=%lld ntiles=%lld: start max %.1f "
                    "us; first stage after start p50 %.1f max %.1f; consumers done p0 %.1f p50 %.1f max %.1f; "
                    "producer done max %.1f us\n",
                    sw.dim, pl.W, pl.T, pl.Tsub, pl.stages, pl.pspan, (long long)grid, (long long)ntiles, q(st, 1.0),
                    q(ff, 0.5), q(ff, 1.0), q(cd, 0.0), q(cd, 0.5), q(cd, 1.0), q(pd, 1.0));
            fprintf(stderr, "SLDG_STAMP   first stage: producer at its empty wait p50 %.1f, TMAs issued p50 %.1f max %.1f, "
                            "consumers at their full wait p50 %.1f us after start\n",
                    q(pe, 0.5), q(pi, 0.5), q(pi, 1.0), q(cw, 0.5));
        }
#endif
    } else {
        return cudaErrorInvalidValue;  // strided k > 4: the plan never selects it
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
