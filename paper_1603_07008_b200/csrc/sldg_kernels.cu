// sldg_kernels.cu -- sm_100a kernels of the mixed-precision SLDG step (arXiv:1603.07008),
// everything except the sweeps themselves (those are in sldg_sweep.cu):
//   build_weights   a1 shift decomposition + a2 weight build (A, B per field entry)
//   mass            a9 deterministic fp64 reduction of the mass slot
//   set / get       host AoS fp64 <-> device split layout (RNE narrowing)
//   fills           synthetic inputs (counter-based random, separable Landau)
//   tr_block        pack / unpack of the transpose path of a sharded sweep
//
// Arithmetic is fp64 throughout (reading R6): fp32 slots are promoted exactly on load and
// rounded to nearest-even on store (__double2float_rn; no fast-math, no FTZ).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "sldg_basis.cuh"
#include "sldg_internal.h"
#include "sldg_ptx.cuh"

namespace sldg {

// slot q of a cell at (padded layer lp, inner) through the general nd layout (sldg_internal.h)
__device__ __forceinline__ double load_slot(const Layout& L, const Arrays& a, int q, int64_t lp, int64_t inner)
{
    if (q < L.nd) return *dslot(a, lp, L.nd, q, L.L, inner);
    return (double)*fslot(a, lp, L.K, L.nd, q, L.L, inner);
}
__device__ __forceinline__ void store_slot(const Layout& L, const Arrays& a, int q, int64_t lp, int64_t inner, double v)
{
    if (q < L.nd) *dslot(a, lp, L.nd, q, L.L, inner) = v;
    else *fslot(a, lp, L.K, L.nd, q, L.L, inner) = __double2float_rn(v);
}

// ============================================================================================
// a1 + a2: shift decomposition and weight build, one thread per field entry.
// A_jl = (2j+1)/2 int_{-1}^{2a-1} P_l(xi+2-2a) P_j(xi) dxi,  B_jl = (2j+1)/2 int_{2a-1}^{1}
// P_l(xi-2a) P_j(xi) dxi (P:259-268 SS II-A), each by a k-point Gauss-Legendre rule
// mapped to the sub-interval (exact for the degree <= 2k-2 integrand), mass row in closed
// form (reading R3), alpha == 0 -> A = 0, B = I and the exact-copy flag (reading R4).
// ============================================================================================

template <int KK>
__global__ void __launch_bounds__(32) build_weights_kernel(int64_t nd, const double* __restrict__ field, double shift,
                                     int64_t n_entries, int64_t* __restrict__ sh_raw,
                                     int64_t* __restrict__ sh_mod, int* __restrict__ cpy,
                                     double* __restrict__ ab, double* __restrict__ rec, int* __restrict__ err,
                                     const GaussTab gt, int64_t ilo, int64_t ihi)
{
    // PDL: let the sweep that reads these weights launch now; wait for the previous sweep (which
    // reads the table this kernel overwrites) before writing
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_entries) return;
    const double nu = field ? field[e] : shift;
    int64_t is = 0;
    double a = 0.0;
    if (!(fabs(nu) < 4.611686018427387904e18)) {  // non-finite or |nu| >= 2^62
        atomicExch(err, 1);
    } else {
        const double fl = floor(nu);
        a = nu - fl;
        is = (int64_t)fl;
        if (a >= 1.0) {  // tiny negative nu: alpha rounds to 1 (reading R2)
            is += 1;
            a = 0.0;
        }
        if (is < ilo || is > ihi) {  // outside the caller's bound: the halo may not cover it
            atomicExch(err, 1);
            is = 0;
            a = 0.0;
        }
    }
    int64_t m = is % nd;
    m = m < 0 ? m + nd : m;
    const int cp = (a == 0.0);
    // A, B in registers (alpha == 0: A = 0, B = I exactly, reading R4)
    double A[KK * KK], B[KK * KK];
    if (a != 0.0) {
        double xg[KK], wg[KK];
#pragma unroll
        for (int g = 0; g < KK; ++g) {
            xg[g] = gt.x[g];
            wg[g] = gt.w[g];
        }
        build_ab_regs<KK>(a, xg, wg, A, B);
    } else {
#pragma unroll
        for (int j = 0; j < KK * KK; ++j) {
            A[j] = 0.0;
            B[j] = ((j / KK) == (j % KK)) ? 1.0 : 0.0;
        }
    }
    sh_raw[e] = is;
    sh_mod[e] = m;
    cpy[e] = cp;
    double* pab = ab + e * 2 * KK * KK;
    // packed line record {A, B, i* mod n, copy} (16(k^2+1) bytes) for bulk copies into smem
    double* r = rec + e * (2 * KK * KK + 2);
#pragma unroll
    for (int j = 0; j < KK * KK; ++j) {
        pab[j] = A[j];
        pab[KK * KK + j] = B[j];
        r[j] = A[j];
        r[KK * KK + j] = B[j];
    }
    r[2 * KK * KK] = __longlong_as_double((long long)m);
    r[2 * KK * KK + 1] = __longlong_as_double((long long)cp);
}

const GaussTab& gauss_table(int k)
{
    static GaussTab tabs[kMaxK + 1];
    static bool done[kMaxK + 1] = {};
    if (!done[k]) {
        GaussTab t{};
        for (int i = 0; i < k; ++i) {  // Newton on P_k from the asymptotic guess of root i
            double z = cos(3.141592653589793238462643 * (i + 0.75) / (k + 0.5)), dp = 1.0;
            for (int it = 0; it < 100; ++it) {
                double p0 = 1.0, p1 = z;
                for (int m = 2; m <= k; ++m) {
                    const double p2 = ((2 * m - 1) * z * p1 - (m - 1) * p0) / m;
                    p0 = p1;
                    p1 = p2;
                }
                const double pn = (k == 1) ? z : p1, pm1 = (k == 1) ? 1.0 : p0;
                dp = k * (pm1 - z * pn) / (1.0 - z * z);
                const double dz = pn / dp;
                z -= dz;
                if (fabs(dz) < 1e-17) break;
            }
            double p0 = 1.0, p1 = z;  // derivative at the converged root
            for (int m = 2; m <= k; ++m) {
                const double p2 = ((2 * m - 1) * z * p1 - (m - 1) * p0) / m;
                p0 = p1;
                p1 = p2;
            }
            const double pn = (k == 1) ? z : p1, pm1 = (k == 1) ? 1.0 : p0;
            dp = k * (pm1 - z * pn) / (1.0 - z * z);
            t.x[k - 1 - i] = z;  // i = 0 is the largest root: ascending order
            t.w[k - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
        }
        if (k & 1) t.x[k / 2] = 0.0;
        tabs[k] = t;
        done[k] = true;
    }
    return tabs[k];
}

cudaError_t launch_weights(const Layout& lay, int64_t nd, const double* d_field, double shift,
                           int64_t n_entries, Weights& w, int* d_err, cudaStream_t s, int64_t ilo, int64_t ihi)
{
    // small blocks: one entry per thread is a serial fp64 build, so spread entries over SMs
    int threads = 32;
    int64_t blocks = (n_entries + threads - 1) / threads;
    const GaussTab& gt = gauss_table(lay.k);
    cudaError_t lerr = cudaSuccess;
#define SLDG_W(KK)                                                                                           \
    lerr = launch_pdl(build_weights_kernel<KK>, dim3((unsigned)blocks), dim3(threads), 0, s, nd, d_field, shift, n_entries, \
               w.shift, w.smod, w.copy, w.ab, w.rec, d_err, gt, ilo, ihi)
    switch (lay.k) {
        case 1: SLDG_W(1); break;
        case 2: SLDG_W(2); break;
        case 3: SLDG_W(3); break;
        case 4: SLDG_W(4); break;
        case 5: SLDG_W(5); break;
        case 6: SLDG_W(6); break;
        case 7: SLDG_W(7); break;
        case 8: SLDG_W(8); break;
        default: return cudaErrorInvalidValue;
    }
#undef SLDG_W
    if (lerr != cudaSuccess) return lerr;
    return cudaGetLastError();
}

// ============================================================================================
// a9: mass = sum of slot 0 over local cells, fixed-order two-pass reduction with Neumaier
// compensation per thread (deterministic for a fixed grid: kMassBlocks x 256 threads).
// ============================================================================================
__device__ __forceinline__ void neumaier_add(double& s, double& c, double x)
{
    double t = s + x;
    if (fabs(s) >= fabs(x)) c += (s - t) + x;
    else c += (x - t) + s;
    s = t;
}

__global__ void __launch_bounds__(256) mass_partials_kernel(Layout lay, Arrays a, double* __restrict__ partials)
{
    __shared__ double sh[256];
    double s = 0.0, c = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < lay.cells; e += stride) {
        int64_t layer = e / lay.L, inner = e - layer * lay.L;
        neumaier_add(s, c, load_slot(lay, a, 0, lay.pad + layer, inner));
    }
    sh[threadIdx.x] = s + c;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(1024) mass_final_kernel(const double* __restrict__ partials, int n,
                                                          double* __restrict__ out)
{
    __shared__ double sh[1024];
    sh[threadIdx.x] = threadIdx.x < n ? partials[threadIdx.x] : 0.0;
    __syncthreads();
    for (int off = 512; off > 0; off >>= 1) {
        if (threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

cudaError_t launch_mass_partials(const Layout& lay, const Arrays& a, double* d_partials, double* d_out,
                                 cudaStream_t s)
{
    mass_partials_kernel<<<kMassBlocks, 256, 0, s>>>(lay, a, d_partials);
    mass_final_kernel<<<1, 1024, 0, s>>>(d_partials, kMassBlocks, d_out);
    return cudaGetLastError();
}

// ============================================================================================
// set / get: host AoS fp64 [cell][q] chunk <-> device split layout.  RNE narrowing.
// ============================================================================================
__global__ void set_kernel(Layout lay, Arrays a, const double* __restrict__ srcv, int64_t first_cell,
                           int64_t n_elems)
{
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    int64_t cell = first_cell + e / lay.K;
    int q = (int)(e % lay.K);
    int64_t layer = cell / lay.L, inner = cell - layer * lay.L;
    store_slot(lay, a, q, lay.pad + layer, inner, srcv[e]);
}

__global__ void get_kernel(Layout lay, Arrays a, double* __restrict__ dstv, int64_t first_cell, int64_t n_elems)
{
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_elems) return;
    int64_t cell = first_cell + e / lay.K;
    int q = (int)(e % lay.K);
    int64_t layer = cell / lay.L, inner = cell - layer * lay.L;
    dstv[e] = load_slot(lay, a, q, lay.pad + layer, inner);
}

cudaError_t launch_set(const Layout& lay, const Arrays& a, const double* d_src, int64_t first_cell,
                       int64_t n_cells, cudaStream_t s)
{
    int64_t n = n_cells * lay.K;
    if (n == 0) return cudaSuccess;
    set_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lay, a, d_src, first_cell, n);
    return cudaGetLastError();
}

cudaError_t launch_get(const Layout& lay, const Arrays& a, double* d_dst, int64_t first_cell, int64_t n_cells,
                       cudaStream_t s)
{
    int64_t n = n_cells * lay.K;
    if (n == 0) return cudaSuccess;
    get_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lay, a, d_dst, first_cell, n);
    return cudaGetLastError();
}

// ============================================================================================
// Synthetic fills (inputs, not the method).
// ============================================================================================
__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void fill_random_kernel(Layout lay, Arrays a, uint64_t seed)
{
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= lay.cells * lay.K) return;
    int64_t cell = e / lay.K;
    int q = (int)(e - cell * lay.K);
    int64_t gcell = lay.first_layer * lay.L + cell;
    uint64_t z = seed * (1ull << 40) + (uint64_t)gcell * (uint64_t)lay.K + (uint64_t)q;
    uint64_t hsh = splitmix64_dev(z);
    double u = (double)(hsh >> 11) * 0x1.0p-53;
    double r = 2.0 * u - 1.0;
    double v;
    if (q == 0) {
        v = __dadd_rn(1.0, __dmul_rn(0.5, r));
    } else {
        int deg = 0, qq = q;
        for (int dd = 0; dd < lay.D; ++dd) {
            deg += qq % lay.k;
            qq /= lay.k;
        }
        // n0^deg as the correctly rounded double of the exact integer while it fits in 64 bits
        // (matches Python's float(n0**deg)); beyond that, exact double products (exact for
        // power-of-two n0, the only case where the integer exceeds 2^64 in the configs).
        uint64_t p = 1;
        double pd = 1.0;
        bool wide = false;
        for (int i = 0; i < deg; ++i) {
            if (!wide && p > UINT64_MAX / (uint64_t)lay.n[0]) {
                wide = true;
                pd = __ull2double_rn(p);
            }
            if (wide) pd = __dmul_rn(pd, (double)lay.n[0]);
            else p *= (uint64_t)lay.n[0];
        }
        v = __ddiv_rn(r, wide ? pd : __ull2double_rn(p));
    }
    int64_t layer = cell / lay.L, inner = cell - layer * lay.L;
    store_slot(lay, a, q, lay.pad + layer, inner, v);
}

cudaError_t launch_fill_random(const Layout& lay, const Arrays& a, uint64_t seed, cudaStream_t s)
{
    int64_t n = lay.cells * lay.K;
    if (n == 0) return cudaSuccess;
    fill_random_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lay, a, seed);
    return cudaGetLastError();
}

__global__ void fill_separable_kernel(Layout lay, Arrays a, int n_terms, const double* __restrict__ tab)
{
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= lay.cells * lay.K) return;
    int64_t cell = e / lay.K;
    int q = (int)(e - cell * lay.K);
    int64_t layer = cell / lay.L, inner = cell - layer * lay.L;
    int64_t idx[kMaxDim];
    int m[kMaxDim];
    int64_t rem = inner;
    int qq = q;
    int64_t off[kMaxDim], term_stride = 0;
    for (int d = 0; d < lay.D; ++d) {
        off[d] = term_stride;
        term_stride += lay.n[d] * lay.k;
        m[d] = qq % lay.k;
        qq /= lay.k;
        if (d < lay.D - 1 || lay.D == 1) {
            idx[d] = rem % lay.n[d];
            rem /= lay.n[d];
        }
    }
    if (lay.D >= 2) idx[lay.D - 1] = lay.first_layer + layer;
    double v = 0.0;
    for (int t = 0; t < n_terms; ++t) {
        double p = 1.0;
        for (int d = 0; d < lay.D; ++d) p *= tab[t * term_stride + off[d] + idx[d] * lay.k + m[d]];
        v += p;
    }
    store_slot(lay, a, q, lay.pad + layer, inner, v);
}

cudaError_t launch_fill_separable(const Layout& lay, const Arrays& a, int n_terms, const double* d_tables,
                                  cudaStream_t s)
{
    int64_t n = lay.cells * lay.K;
    if (n == 0) return cudaSuccess;
    fill_separable_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lay, a, n_terms, d_tables);
    return cudaGetLastError();
}

// min / max of floor(nu) over a device field (halo planning for sharded sweeps)
__global__ void field_range_kernel(const double* __restrict__ field, int64_t n, double shift, int64_t* out)
{
    __shared__ int64_t smin[256], smax[256];
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
        double nu = field ? field[e] : shift;
        if (!(fabs(nu) < 4.611686018427387904e18)) continue;
        double fl = floor(nu);
        int64_t is = (int64_t)fl;
        if (nu - fl >= 1.0) is += 1;
        lo = is < lo ? is : lo;
        hi = is > hi ? is : hi;
    }
    smin[threadIdx.x] = lo;
    smax[threadIdx.x] = hi;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            smin[threadIdx.x] = min(smin[threadIdx.x], smin[threadIdx.x + off]);
            smax[threadIdx.x] = max(smax[threadIdx.x], smax[threadIdx.x + off]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = smin[0];
        out[1] = smax[0];
    }
}

cudaError_t launch_field_range(const double* d_field, int64_t n, double shift, int64_t* d_out2, cudaStream_t s)
{
    field_range_kernel<<<1, 256, 0, s>>>(d_field, n, shift, d_out2);
    return cudaGetLastError();
}

// ---- transpose path of a sweep along the sharded dim (sldg_abi.cu transpose_sweep) ----------
// Message layout of one (layer range, inner range) block: fp64 part [layer][q < nd][len], then
// fp32 part [layer][q >= nd][len]; the inner range [first, first + len) of every plane of the
// padded layers pad .. pad + nl - 1.  pack: array -> block, unpack: block -> array.
template <bool PACK>
__global__ void tr_block_kernel(Layout lay, Arrays a, int64_t nl, int64_t first, int64_t len, double* bm,
                                float* bf)
{
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t lq = blockIdx.y + (int64_t)gridDim.y * blockIdx.z;  // layer * K + q
    if (j >= len || lq >= nl * lay.K) return;
    const int64_t l = lq / lay.K;
    const int q = (int)(lq - l * lay.K);
    const int64_t lp = lay.pad + l;
    if (q < lay.nd) {
        double* p = dslot(a, lp, lay.nd, q, lay.L, first + j);
        double* b = bm + (l * lay.nd + q) * len + j;
        if (PACK) *b = *p;
        else *p = *b;
    } else {
        float* p = fslot(a, lp, lay.K, lay.nd, q, lay.L, first + j);
        float* b = bf + (l * (lay.K - lay.nd) + (q - lay.nd)) * len + j;
        if (PACK) *b = *p;
        else *p = *b;
    }
}

cudaError_t launch_tr_block(const Layout& lay, const Arrays& a, int64_t nl, int64_t first, int64_t len, double* bm,
                            float* bf, bool pack, cudaStream_t s)
{
    if (nl <= 0 || len <= 0) return cudaSuccess;
    const int64_t rows = nl * lay.K;
    const unsigned gy = (unsigned)std::min<int64_t>(rows, 65535), gz = (unsigned)((rows + gy - 1) / gy);
    dim3 grid((unsigned)((len + 255) / 256), gy, gz);
    if (pack) tr_block_kernel<true><<<grid, 256, 0, s>>>(lay, a, nl, first, len, bm, bf);
    else tr_block_kernel<false><<<grid, 256, 0, s>>>(lay, a, nl, first, len, bm, bf);
    return cudaGetLastError();
}

// field entries of a slab grid: out[e'] = in[e] where e' indexes the masked dims with extents
// nT and e the same cell of the full extents nF, dim `sd` offset by `off`.
__global__ void field_slab_kernel(const double* in, int64_t n_out, uint32_t mask, Layout nT, Layout nF, int sd,
                                  int64_t off, double* out)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_out) return;
    int64_t rem = t, e = 0, stride = 1;
    for (int d = 0; d < nT.D; ++d) {
        if (!(mask >> d & 1u)) continue;
        int64_t i = rem % nT.n[d];
        rem /= nT.n[d];
        if (d == sd) i += off;
        e += i * stride;
        stride *= nF.n[d];
    }
    out[t] = in[e];
}

cudaError_t launch_field_slab(const double* in, int64_t n_out, uint32_t mask, const Layout& nT, const Layout& nF,
                              int sd, int64_t off, double* out, cudaStream_t s)
{
    if (n_out <= 0) return cudaSuccess;
    field_slab_kernel<<<(unsigned)((n_out + 255) / 256), 256, 0, s>>>(in, n_out, mask, nT, nF, sd, off, out);
    return cudaGetLastError();
}

}  // namespace sldg
