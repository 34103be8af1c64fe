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
//                      Rows that are contiguous in HBM go in one copy.
//   sweep_d0_tma       d = 0: tile = R whole lines (the line is periodic, so the stage holds
//                      every source cell and the modulo indexing is done in shared memory);
//                      a stage holds GC coupled groups.
// Consumers address HBM and shared memory by pointer increments set up once per stage; the
// coupled group that holds the fp64 mass slot is a separate template instance.
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

// element type of slot j of a coupled group
template <int PREC, bool MASSG, int J>
struct ET {
    static constexpr bool dbl = (PREC == SLDG_FP64) || (MASSG && J == 0);
};
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
__device__ __forceinline__ double ld_smem(const unsigned char* p, int i, bool dbl)
{
    return dbl ? ((const double*)p)[i] : (double)((const float*)p)[i];
}

// Strided consumer: one stage (one coupled group), one column, targets [lo, hi) of the sub-chunk.
// sb[j]: stage slot j at row 0 of this column; sstride: elements between rows; rB0: row of the
// B-source of target lo; op[j]: output pointer of slot j at target lo; ostep: element step
// between consecutive targets in each array (mass/fp64 vs fp32 planes).
template <int KK, int PREC, bool MASSG>
__device__ __forceinline__ void strided_consume(const unsigned char* const* sb, int sstride, int rB0, int cnt,
                                                char* const* op, int64_t ostep_m, int64_t ostep_f, int cp,
                                                const double* wr)
{
    // element j is fp64 for the fp64 variant and for the mass slot of the mass group
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
    double va[KK], vb[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        va[j] = SLDG_DBL(j) ? *(const double*)rp[j] : (double)*(const float*)rp[j];
        rp[j] += rstep * (SLDG_DBL(j) ? 8 : 4);
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
            double o = 0.0;
#pragma unroll
            for (int l = 0; l < KK; ++l) o = fma(wr[j * KK + l], va[l], o);
#pragma unroll
            for (int l = 0; l < KK; ++l) o = fma(wr[KK * KK + j * KK + l], vb[l], o);
            o = cp ? vb[j] : o;  // alpha == 0: exact copy (R4)
            if (SLDG_DBL(j)) __stcs((double*)wp[j], o);
            else __stcs((float*)wp[j], __double2float_rn(o));
            wp[j] += wstep[j];
        }
#pragma unroll
        for (int j = 0; j < KK; ++j) va[j] = vb[j];
    }
#undef SLDG_DBL
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
    // element step between consecutive targets along d (mass/fp64 array, fp32 planes)
    const int64_t tstep_m = outer ? (toff_m<PREC>(lay, 1, 0) - toff_m<PREC>(lay, 0, 0)) : lay.S[d];
    const int64_t tstep_f = outer ? (toff_f<PREC>(lay, 1, 0) - toff_f<PREC>(lay, 0, 0)) : lay.S[d];
    // rows of one slot are contiguous in HBM when the line stride equals the tile width
    const bool rows_contig = !outer && lay.S[d] == W;

    const int NT = NC * 32;
    const int P = NT / W;
    const int tid = threadIdx.x;
    const int c = tid % W, part = tid / W;

    uint32_t it = 0;  // stage-use counter, identical in every warp
    // tile -> (segment along d, column block, perpendicular indices, layer)
    auto decode = [&](int64_t tl, int64_t* idx, int64_t& cb, int64_t& layer, int64_t& inner_base, int64_t& t0) {
        int64_t rem = tl;
        const int64_t seg = rem % nseg;
        rem /= nseg;
        cb = rem % nb0;
        rem /= nb0;
#pragma unroll
        for (int e = 0; e < kMaxDim; ++e) idx[e] = 0;
        for (int e = 1; e < D - 1; ++e)
            if (e != d) {
                idx[e] = rem % lay.n[e];
                rem /= lay.n[e];
            }
        layer = 0;
        if (!outer) {
            layer = lb + rem;
            idx[D - 1] = lay.first_layer + layer;
        }
        inner_base = cb * W;  // inner offset of the tile's column 0 at line coordinate 0
        for (int e = 1; e < D - 1; ++e)
            if (e != d) inner_base += idx[e] * lay.S[e];
        t0 = seg * T;
    };
    auto findex = [&](const int64_t* idx, int64_t col) {
        int64_t id2[kMaxDim];
#pragma unroll
        for (int e = 0; e < kMaxDim; ++e) id2[e] = idx[e];
        id2[0] = col;
        return tfield_index(sw, id2, D);
    };
    // The shifts of the NEXT tile's columns (for its shift span) are loaded while the current
    // tile streams (software prefetch).  Tiles are whole lines where possible (tma_plan), so the
    // per-tile consumer line data (A/B) is fetched once per ~k^{D-1} x n_d targets.
    int64_t pf_sh[4];
    auto prefetch = [&](int64_t tl) {
        int64_t idx[kMaxDim], cb, layer, inner_base, t0;
        decode(tl, idx, cb, layer, inner_base, t0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int cc = lane + 32 * i;
            pf_sh[i] = (cc < W) ? __ldg(&sw.shift[findex(idx, cb * W + cc)]) : 0;
        }
    };
    if ((int64_t)blockIdx.x < ntiles) prefetch(blockIdx.x);

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int64_t idx[kMaxDim], cb, layer, inner_base, t0;
        decode(tile, idx, cb, layer, inner_base, t0);
        const int nt = (int)((nline - t0) < T ? (nline - t0) : T);
        const int64_t tg0 = outer ? lay.first_layer + lb : 0;  // line coordinate of target index 0

        // shift range over the tile's W columns (every warp reduces its prefetched shifts)
        int64_t imin = INT64_MAX, imax = INT64_MIN;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (lane + 32 * i < W) {
                imin = pf_sh[i] < imin ? pf_sh[i] : imin;
                imax = pf_sh[i] > imax ? pf_sh[i] : imax;
            }
        }
        if (tile + gridDim.x < ntiles) prefetch(tile + gridDim.x);
        // this tile's consumer line data: column shift, copy flag, A/B in registers
        int64_t my_s = 0;
        int my_cp = 0;
        double wr[2 * KK * KK];
        if (!producer) {
            const int64_t f = findex(idx, cb * W + c);
            my_s = __ldg(&sw.shift[f]);
            my_cp = __ldg(&sw.copy[f]);
#pragma unroll
            for (int i = 0; i < 2 * KK * KK; ++i) wr[i] = __ldg(&sw.ab[f * (2 * KK * KK) + i]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            int64_t a = __shfl_xor_sync(0xffffffffu, imin, o), b = __shfl_xor_sync(0xffffffffu, imax, o);
            imin = a < imin ? a : imin;
            imax = b > imax ? b : imax;
        }
        const int64_t span = imax - imin;
        const int teff = (int)((Rmax - 1 - span) < nt ? (Rmax - 1 - span) : nt);
        if (teff < 1) {
            // ---- shift spread too wide for a stage: direct global loads (rare) ----
            if (!producer) {
                for (int col = tid; col < W; col += NT) {
                    int64_t id2[kMaxDim];
#pragma unroll
                    for (int e = 0; e < kMaxDim; ++e) id2[e] = idx[e];
                    id2[0] = cb * W + col;
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
                                int64_t x = xB - 1 + half, lp, in;
                                if (outer) {
                                    int64_t xm = x % sw.nd;
                                    if (xm < 0) xm += sw.nd;
                                    lp = sw.wrap ? lay.pad + xm : x - lay.first_layer + lay.pad;
                                    in = inner_base + col;
                                } else {
                                    int64_t xm = x % sw.nd;
                                    if (xm < 0) xm += sw.nd;
                                    lp = lay.pad + layer;
                                    in = inner_base + col + xm * lay.S[d];
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
                            int64_t in = outer ? inner_base + col : inner_base + col + tt * lay.S[d];
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
                                st_elem(slot_ptr_w<PREC>(dst, lay, q, lp, in), 0, o, PREC == SLDG_FP64 || q == 0);
                            }
                        }
                    }
                }
            }
            continue;
        }

        // output position of target index 0 (padded layer, inner)
        const int64_t ob_lp = outer ? lay.pad + lb : lay.pad + layer;
        const int64_t ob_in = inner_base + c;

        for (int sub = 0; sub < nt; sub += teff) {
            const int te = (nt - sub) < teff ? (nt - sub) : teff;
            const int rows = te + 1 + (int)span;
            const int64_t rowbase = tg0 + t0 + sub - imax - 1;  // line coordinate of stage row 0
            // this consumer thread's targets [lo, hi) of the sub-chunk
            const int tp = (te + P - 1) / P;
            const int lo = part * tp, hi = (lo + tp) < te ? (lo + tp) : te;
            const int rB0 = (int)((tg0 + t0 + sub + lo - my_s) - rowbase);
            const int64_t tl0 = t0 + sub + lo;  // local target index of `lo`
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
                    for (int j = 0; j < KK; ++j) bytes += (uint32_t)(rows * W * esz_rt<PREC>(massg, j));
                    if (lane == 0) mbar_expect_tx(&full[s], bytes);
                    __syncwarp();
                    int64_t x0 = rowbase % sw.nd;  // wrapped coordinate of row 0 (wrap mode)
                    if (x0 < 0) x0 += sw.nd;
                    const bool one_copy = rows_contig && sw.wrap && (x0 + rows <= sw.nd);
                    int soff = 0;
#pragma unroll
                    for (int j = 0; j < KK; ++j) {
                        const int q = qbase + j * kd;
                        const int es = esz_rt<PREC>(massg, j);
                        const uint32_t rowb = (uint32_t)(W * es);
                        if (one_copy) {
                            if (lane == j)
                                bulk_g2s(st + soff, slot_ptr<PREC>(src, lay, q, lay.pad + layer, inner_base + x0 * lay.S[d]),
                                         rowb * rows, &full[s], pol);
                        } else {
                            for (int r = lane; r < rows; r += 32) {
                                int64_t lp, in;
                                if (sw.wrap) {
                                    int64_t xm = x0 + r;
                                    while (xm >= sw.nd) xm -= sw.nd;
                                    lp = outer ? lay.pad + xm : lay.pad + layer;
                                    in = outer ? inner_base : inner_base + xm * lay.S[d];
                                } else {  // sharded layer dim: halo layers in the pad
                                    lp = rowbase + r - lay.first_layer + lay.pad;
                                    in = inner_base;
                                }
                                bulk_g2s(st + soff + r * rowb, slot_ptr<PREC>(src, lay, q, lp, in), rowb, &full[s], pol);
                            }
                        }
                        soff += Rmax * W * es;
                    }
                } else {
                    mbar_wait(&full[s], ph);
                    if (lo < hi) {
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
                        if (massg)
                            strided_consume<KK, PREC, true>(sb, W, rB0, hi - lo, op, tstep_m, tstep_f, my_cp, wr);
                        else
                            strided_consume<KK, PREC, false>(sb, W, rB0, hi - lo, op, tstep_m, tstep_f, my_cp, wr);
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                }
            }
        }
    }
}

// ============================================================================================
// contiguous sweep (d = 0): R whole lines x GC coupled groups per stage.  Every consumer thread
// owns cells of ONE line of the tile (R = NT / n0 lines of one cell per thread when n0 <= NT,
// else R = 1 and n0 / NT cells per thread), so its weights are loaded once per tile.
// ============================================================================================
// one coupled group: sources at columns cA, cB of the k stage slots starting at `sp`
// (slot stride cs elements), outputs to om (fp64 slot 0 of the mass group / fp64 variant) and
// of (fp32 planes), each advanced by one plane (L elements) per slot.
template <int KK, int PREC, bool MASSG>
__device__ __forceinline__ void d0_group(const unsigned char*& sp, int cs, int cA, int cB, double*& om, float*& of,
                                         int64_t L, int cp, const double* wr)
{
#define SLDG_DBL(j) ((PREC == SLDG_FP64) || (MASSG && (j) == 0))
    double va[KK], vb[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        if (SLDG_DBL(j)) {
            va[j] = ((const double*)sp)[cA];
            vb[j] = ((const double*)sp)[cB];
            sp += cs * 8;
        } else {
            va[j] = (double)((const float*)sp)[cA];
            vb[j] = (double)((const float*)sp)[cB];
            sp += cs * 4;
        }
    }
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        double o = 0.0;
#pragma unroll
        for (int l = 0; l < KK; ++l) o = fma(wr[j * KK + l], va[l], o);
#pragma unroll
        for (int l = 0; l < KK; ++l) o = fma(wr[KK * KK + j * KK + l], vb[l], o);
        o = cp ? vb[j] : o;  // alpha == 0: exact copy (R4)
        if (SLDG_DBL(j)) {
            __stcs(om, o);
            om += L;
        } else {
            __stcs(of, __double2float_rn(o));
            of += L;
        }
    }
#undef SLDG_DBL
}

// all gc coupled groups of a stage for one target cell.  Mixed: om = mass of the cell, of =
// plane of slot q0 (or q0+1 for the mass group); fp64: om = slot q0 of the cell.
template <int KK, int PREC, bool MASSG>
__device__ __forceinline__ void d0_consume(const unsigned char* sbase, int gc, int cs, int cA, int cB, double* om,
                                           float* of, int64_t L, int cp, const double* wr)
{
    const unsigned char* sp = sbase;
    int gi = 0;
    if (MASSG) {
        d0_group<KK, PREC, true>(sp, cs, cA, cB, om, of, L, cp, wr);
        gi = 1;
    }
#pragma unroll 1
    for (; gi < gc; ++gi) d0_group<KK, PREC, false>(sp, cs, cA, cB, om, of, L, cp, wr);
}

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
    const int n0 = (int)lay.n[0];
    const int64_t L = lay.L;
    const int R = pl.R, GC = pl.GC;
    const int64_t lines_per_layer = L / n0;
    const int64_t nblk = lines_per_layer / R;
    const int64_t nlay = le - lb;
    const int64_t ntiles = nblk * nlay;
    const int G = lay.K / KK;
    const int NT = NC * 32;
    const int cell_stride = R * n0;  // elements of one slot in a stage
    const uint64_t pol = policy_evict_first();
    // this thread's line of the tile and first cell
    const int my_r = (n0 <= NT) ? (int)threadIdx.x / n0 : 0;
    const int my_c0 = (n0 <= NT) ? (int)threadIdx.x % n0 : (int)threadIdx.x;
    const int ncell = (n0 <= NT) ? 1 : n0 / NT;
    const bool has_cell = !producer && my_r < R;

    // the line data (shift, copy flag, A/B) of the NEXT tile is loaded while the current one
    // streams (software prefetch), so tile boundaries do not stall the consumers
    int64_t pf_s = 0;
    int pf_cp = 0;
    double pf_w[2 * KK * KK];
    auto prefetch = [&](int64_t tl) {
        if (!has_cell) return;
        const int64_t blk = tl % nblk;
        const int64_t layer = lb + tl / nblk;
        int64_t f = 0;
        if (sw.fmask) {
            int64_t idx[kMaxDim];
            int64_t rem2 = blk * R + my_r;  // line index within the layer
#pragma unroll
            for (int e = 0; e < kMaxDim; ++e) idx[e] = 0;
            for (int e = 1; e < D - 1; ++e) {
                idx[e] = rem2 % lay.n[e];
                rem2 /= lay.n[e];
            }
            if (D >= 2) idx[D - 1] = lay.first_layer + layer;
            f = tfield_index(sw, idx, D);
        }
        pf_s = __ldg(&sw.smod[f]);
        pf_cp = __ldg(&sw.copy[f]);
#pragma unroll
        for (int i = 0; i < 2 * KK * KK; ++i) pf_w[i] = __ldg(&sw.ab[f * (2 * KK * KK) + i]);
    };
    if ((int64_t)blockIdx.x < ntiles) prefetch(blockIdx.x);

    uint32_t it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t blk = tile % nblk;
        const int64_t layer = lb + tile / nblk;
        const int64_t layerp = lay.pad + layer;
        const int64_t inner_base = blk * R * (int64_t)n0;  // first cell of the tile's first line
        const int64_t my_s = pf_s;
        const int my_cp = pf_cp;
        double wr[2 * KK * KK];
#pragma unroll
        for (int i = 0; i < 2 * KK * KK; ++i) wr[i] = pf_w[i];
        if (tile + gridDim.x < ntiles) prefetch(tile + gridDim.x);
        for (int g0 = 0; g0 < G; g0 += GC) {
            const int gc = (G - g0) < GC ? (G - g0) : GC;
            const int s = it % S;
            const uint32_t ph = (it / S) & 1;
            ++it;
            unsigned char* st = stage0 + (size_t)s * pl.stage_bytes;
            const bool massg = (PREC == SLDG_MIXED) && g0 == 0;
            if (producer) {
                if (lane == 0) mbar_wait(&empty[s], ph ^ 1);
                __syncwarp();
                const int nslot = gc * KK;
                const uint32_t bytes = (uint32_t)cell_stride * ((PREC == SLDG_FP64) ? 8u * nslot : 4u * nslot + (massg ? 4u : 0u));
                if (lane == 0) mbar_expect_tx(&full[s], bytes);
                __syncwarp();
                for (int i = lane; i < nslot; i += 32) {
                    const int q = g0 * KK + i;
                    const int64_t soff = (PREC == SLDG_FP64) ? (int64_t)i * cell_stride * 8
                                                             : (int64_t)i * cell_stride * 4 + ((massg && i > 0) ? (int64_t)cell_stride * 4 : 0);
                    const uint32_t b = (uint32_t)cell_stride * ((PREC == SLDG_FP64 || q == 0) ? 8u : 4u);
                    bulk_g2s(st + soff, slot_ptr<PREC>(src, lay, q, layerp, inner_base), b, &full[s], pol);
                }
            } else {
                mbar_wait(&full[s], ph);
                if (has_cell) {
                    for (int ci = 0; ci < ncell; ++ci) {
                        const int cc = my_c0 + ci * NT;  // column (target cell within the line)
                        int cB = cc - (int)my_s;
                        if (cB < 0) cB += n0;
                        int cA = cB - 1;
                        if (cA < 0) cA += n0;
                        const int row0 = my_r * n0;
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
                        if (massg)
                            d0_consume<KK, PREC, true>(st, gc, cell_stride, row0 + cA, row0 + cB, om, of, L, my_cp, wr);
                        else
                            d0_consume<KK, PREC, false>(st, gc, cell_stride, row0 + cA, row0 + cB, om, of, L, my_cp, wr);
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
    const int bpc_max = (lay.prec == SLDG_FP64) ? 8 * k : 8 + 4 * (k - 1);  // bytes per column, mass group
    const int NT = kTmaConsumerWarps * 32;
    *pl = TmaPlan{};
    if (k > 4) return false;  // line weights live in registers; larger k uses the register kernels
    if (sw.dim == 0) {
        if (n0 % 4 != 0) return false;
        int64_t R;
        if (n0 <= NT) {
            if (NT % n0 != 0) return false;
            R = NT / n0;
        } else {
            if (n0 % NT != 0) return false;
            R = 1;
        }
        const int64_t lines = lay.L / n0;
        if (lines % R != 0) return false;
        const int64_t group_bytes = R * n0 * bpc_max;  // one coupled group of the tile, worst case
        const int G = lay.K / k;
        const int64_t target = budget / 3;
        if (group_bytes > budget / 2) return false;
        int gcmax = (int)std::max<int64_t>(1, std::min<int64_t>(G, target / group_bytes));
        const int nchunk = (G + gcmax - 1) / gcmax;
        const int GC = (G + nchunk - 1) / nchunk;  // balanced chunks
        pl->R = (int)R;
        pl->GC = GC;
        const int64_t slot_f = R * n0 * ((lay.prec == SLDG_FP64) ? 8 : 4);
        pl->stage_bytes = (int)((GC * k * slot_f + ((lay.prec == SLDG_FP64) ? 0 : R * n0 * 4) + 127) / 128 * 128);
        pl->stages = (int)std::min<int64_t>(8, budget / pl->stage_bytes);
        return pl->stages >= 2;
    }
    int W = 0;
    for (int w : {128, 64, 32})
        if (n0 % w == 0) {
            W = w;
            break;
        }
    if (W == 0) return false;
    // sub-chunk: Tsub targets share a stage (rows = Tsub + 1 + shift span <= Rmax)
    const int Tsub = (k <= 3) ? 16 : 8;
    const int Rmax = Tsub + 1 + 3;
    const int64_t stage = (int64_t)Rmax * W * bpc_max;
    const int stage_bytes = (int)((stage + 127) / 128 * 128);
    const int stages = (int)std::min<int64_t>(8, budget / stage_bytes);
    if (stages < 2) return false;
    // tile length along d: whole lines (one line-data fetch per tile) unless that leaves fewer
    // than 4 tiles per SM, then the lines are cut into segments (multiples of Tsub)
    const bool outer = (sw.dim == lay.D - 1);
    const int64_t nline = outer ? lay.layers : sw.nd;
    int64_t base = (n0 / W) * (outer ? 1 : lay.layers);
    for (int e = 1; e < lay.D - 1; ++e)
        if (e != sw.dim) base *= lay.n[e];
    const int64_t want = 4LL * g_num_sms;
    int64_t nseg = std::max<int64_t>(1, (want + base - 1) / base);
    int64_t T = (nline + nseg - 1) / nseg;
    T = std::max<int64_t>(Tsub, (T + Tsub - 1) / Tsub * Tsub);
    pl->W = W;
    pl->T = (int)T;
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
    const int per_sm = std::max<int>(1, (int)(228 * 1024 / (smem + 1024)));
    if (sw.dim == 0) {
        ntiles = (lay.L / lay.n[0] / pl.R) * (le - lb);
        auto kern = sweep_d0_tma<KK, PREC>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
