// sldg_vnodes.cu -- Gauss-node velocity treatment of x-sweeps (NEXT-3 of SURVEY 8(f); DESIGN.md
// 6d, reading V7; oracle/vnodes.py).
//
// An x-sweep along dim d whose CFL number varies with the velocity inside a v-cell of dim e:
// modal -> nodal in e at the k Gauss nodes (P:221-227 nodal basis), one SLDG line update per
// node with its own nu, nodal -> modal by Gauss quadrature.  All three
// steps are linear, so per v-cell j they fold into one operator per source offset o:
//   c'_{(m_e, m_d)}(i) = sum_o sum_{(l_e, l_d)} M_o[m_e m_d][l_e l_d] c_{(l_e, l_d)}(i - o)
//   M_o = sum_n Tinv[m_e][n] T[n][l_e] (A_n[m_d][l_d] [o == i*_n + 1] + B_n[m_d][l_d] [o == i*_n])
// with T[n][l] = P_l(xi_n), Tinv[m][n] = w_n (2m+1)/2 P_m(xi_n), (i*_n, A_n, B_n) the plain
// sweep's decomposition and shift matrices of node n.  Offsets span [min i*_n, max i*_n + 1]
// (2 cells when every node has the same integer part, 3 when the nodes straddle an integer).
//   vnode_weights_kernel   one CTA per v-cell: nodes, A_n/B_n, the M_o
//   vnode_sweep_kernel     one thread per target cell; for every coupled (m_e, m_d) block it
//                          loads the k^2 coefficients of each source cell and applies the M_o
// fp64 arithmetic, fp32 slots rounded to nearest-even on store (R6).  There is no exact-copy
// path: the modal -> nodal -> modal pair is the identity only up to rounding.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "sldg_basis.cuh"
#include "sldg_internal.h"

namespace sldg {

namespace {

// record of one v-cell: [omin (int64 bits), nofs (int64 bits), M[kVnMaxOfs][k^4]]
__host__ __device__ __forceinline__ int64_t vn_rec_words(int k) { return 2 + (int64_t)kVnMaxOfs * k * k * k * k; }

__global__ void vnode_weights_kernel(int k, const double* __restrict__ nodal, int64_t nv, double* __restrict__ rec,
                                     int* __restrict__ err, const GaussTab gt)
{
    const int64_t j = blockIdx.x;
    if (j >= nv) return;
    __shared__ double sT[kMaxK * kMaxK], sTi[kMaxK * kMaxK];
    __shared__ double sA[kMaxK * kMaxK * kMaxK], sB[kMaxK * kMaxK * kMaxK];  // [n][m][l]
    __shared__ int64_t sI[kMaxK];
    __shared__ int64_t s_omin;
    __shared__ int s_nofs, s_bad;
    double* r = rec + j * vn_rec_words(k);
    if (threadIdx.x == 0) {
        double P[kMaxK + 2];
        const double* xg = gt.x;
        const double* wg = gt.w;
        for (int n = 0; n < k; ++n) {
            dev_legendre(k - 1, xg[n], P);
            for (int m = 0; m < k; ++m) {
                sT[n * k + m] = P[m];
                sTi[m * k + n] = wg[n] * (0.5 * (2 * m + 1)) * P[m];
            }
        }
        int bad = 0;
        int64_t omin = INT64_MAX, omax = INT64_MIN;
        for (int n = 0; n < k; ++n) {
            const double nu = nodal[j * k + n];
            double* A = sA + n * k * k;
            double* B = sB + n * k * k;
            for (int q = 0; q < k * k; ++q) {
                A[q] = 0.0;
                B[q] = ((q / k) == (q % k)) ? 1.0 : 0.0;
            }
            int64_t is = 0;
            if (!(fabs(nu) < 4.611686018427387904e18)) {
                bad = 1;
            } else {
                const double fl = floor(nu);
                double a = nu - fl;
                is = (int64_t)fl;
                if (a >= 1.0) {  // reading R2 edge case
                    is += 1;
                    a = 0.0;
                }
                if (a != 0.0) build_ab(k, a, A, B, gt);
            }
            sI[n] = is;
            omin = is < omin ? is : omin;
            omax = (is + 1) > omax ? (is + 1) : omax;
        }
        if (bad || omax - omin + 1 > kVnMaxOfs) {
            bad = 1;
            omin = 0;
            omax = 0;  // leave the lines unchanged: identity at offset 0
        }
        s_bad = bad;
        s_omin = omin;
        s_nofs = (int)(omax - omin + 1);
        if (bad) atomicExch(err, 1);
        r[0] = __longlong_as_double((long long)omin);
        r[1] = __longlong_as_double((long long)(omax - omin + 1));
    }
    __syncthreads();
    const int k2 = k * k, k4 = k2 * k2;
    double* M = r + 2;
    for (int t = threadIdx.x; t < kVnMaxOfs * k4; t += blockDim.x) {
        const int o = t / k4, rem = t % k4;
        const int me = rem / (k * k2), md = (rem / k2) % k, le = (rem / k) % k, ld = rem % k;
        double v = 0.0;
        if (s_bad) {
            v = (o == 0 && me == le && md == ld) ? 1.0 : 0.0;
        } else if (o < s_nofs) {
            const int64_t off = s_omin + o;
            for (int n = 0; n < k; ++n) {
                double ab = 0.0;
                if (off == sI[n] + 1) ab += sA[(n * k + md) * k + ld];
                if (off == sI[n]) ab += sB[(n * k + md) * k + ld];
                v = fma(sTi[me * k + n] * sT[n * k + le], ab, v);
            }
        }
        M[t] = v;
    }
}

__device__ __forceinline__ double vn_load(const Layout& L, const Arrays& a, int q, int64_t lp, int64_t inner)
{
    if (q < L.nd) return *dslot(a, lp, L.nd, q, L.L, inner);
    return (double)*fslot(a, lp, L.K, L.nd, q, L.L, inner);
}
__device__ __forceinline__ void vn_store(const Layout& L, const Arrays& a, int q, int64_t lp, int64_t inner, double v)
{
    if (q < L.nd) *dslot(a, lp, L.nd, q, L.L, inner) = v;
    else *fslot(a, lp, L.K, L.nd, q, L.L, inner) = __double2float_rn(v);
}

// 4 CTAs/SM for k <= 3, 3 for k = 4: the sweep waits on load latency, so resident warps pay
// (profiles/round1/tuning.md, "Gauss-node x sweep")
template <int KK>
__global__ void __launch_bounds__(256, KK <= 3 ? 4 : 3) vnode_sweep_kernel(Layout lay, int d, int e, const double* __restrict__ rec,
                                                         Arrays src, Arrays dst)
{
    constexpr int K2 = KK * KK, K4 = K2 * K2;
    constexpr int RS = (K2 + 1) & ~1;  // shared-memory row stride (even: 16-byte row pairs)
    extern __shared__ __align__(16) double sM[];  // [kVnMaxOfs][K2][RS]
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = t < lay.cells;
    const int D = lay.D;
    const int64_t tt = valid ? t : blockIdx.x * (int64_t)blockDim.x;
    const int64_t layer = tt / lay.L, inner = tt - layer * lay.L;
    const int64_t lp = lay.pad + layer;
    // index along d and along e (global)
    auto idx_of = [&](int dd, int64_t lay_, int64_t in_) -> int64_t {
        if (dd == D - 1) return lay.first_layer + lay_;
        return (in_ / lay.S[dd]) % lay.n[dd];
    };
    const int64_t id = idx_of(d, layer, inner), j = idx_of(e, layer, inner);
    // the CTA's cells usually share their v-cell (C5: 256 consecutive cells along x1 or x2);
    // then its operators are staged in shared memory once and read as 16-byte broadcasts
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x;
    const int64_t l0 = t0 / lay.L;
    const int64_t j0 = idx_of(e, l0, t0 - l0 * lay.L);
    const bool uni = __syncthreads_and(!valid || j == j0);
    const double* r = rec + j * vn_rec_words(KK);
    const int64_t omin = (int64_t)__double_as_longlong(__ldg(&r[0]));
    const int nofs = (int)__double_as_longlong(__ldg(&r[1]));
    if (uni) {
        const double* M0 = rec + j0 * vn_rec_words(KK) + 2;
        for (int x = threadIdx.x; x < kVnMaxOfs * K4; x += blockDim.x) {  // transposed: [o][l][m]
            const int o = x / K4, rem = x - o * K4, m = rem / K2, l = rem - m * K2;
            sM[(o * K2 + l) * RS + m] = __ldg(&M0[x]);
        }
        if (RS != K2)
            for (int x = threadIdx.x; x < kVnMaxOfs * K2; x += blockDim.x) sM[x * RS + K2] = 0.0;
        __syncthreads();
    }
    if (!valid) return;
    const double* M = r + 2;
    // source positions per offset
    int64_t s_lp[kVnMaxOfs], s_in[kVnMaxOfs];
    const int64_t nd = lay.n[d];
#pragma unroll
    for (int o = 0; o < kVnMaxOfs; ++o) {
        int64_t sidx = (id - (omin + o)) % nd;
        if (sidx < 0) sidx += nd;
        if (d == D - 1) {
            s_lp[o] = lay.pad + (sidx - lay.first_layer);
            s_in[o] = inner;
        } else {
            s_lp[o] = lp;
            s_in[o] = inner + (sidx - id) * lay.S[d];
        }
    }
    int kd = 1, ke = 1;
    for (int x = 0; x < d; ++x) kd *= KK;
    for (int x = 0; x < e; ++x) ke *= KK;
    // element offsets of the block's k^2 slots from its first slot, in planes of L cells
    int64_t loff[K2];
#pragma unroll
    for (int le = 0; le < KK; ++le)
#pragma unroll
        for (int ld = 0; ld < KK; ++ld) loff[le * KK + ld] = (int64_t)(ld * kd + le * ke) * lay.L;
    // per source offset: slot-q pointers are fb[o] + q L (fp32 slots) and db[o] + q L (fp64 slots)
    const float* fb[kVnMaxOfs];
    const double* db[kVnMaxOfs];
    const int nd_ = lay.nd, nf_ = lay.K - lay.nd;
#pragma unroll
    for (int o = 0; o < kVnMaxOfs; ++o) {
        fb[o] = src.pl + (s_lp[o] * nf_ - nd_) * lay.L + s_in[o];
        db[o] = src.mass + s_lp[o] * nd_ * lay.L + s_in[o];
    }
    const int nblk = lay.K / K2;
    for (int b = 0; b < nblk; ++b) {
        // slot base of block b: the other dims' indices (all but d, e) from b
        int q0 = 0, bb = b, kp = 1;
        for (int x = 0; x < D; ++x) {
            if (x != d && x != e) {
                q0 += (bb % KK) * kp;
                bb /= KK;
            }
            kp *= KK;
        }
        const int64_t q0L = (int64_t)q0 * lay.L;
        // the block's slots are all fp32 unless it holds an fp64 slot (q < nd)
        const bool all_f = (q0 >= nd_);
        double out[K2];
#pragma unroll
        for (int m = 0; m < K2; ++m) out[m] = 0.0;
        for (int o = 0; o < nofs; ++o) {
            double v[RS];
            if (all_f) {
                const float* p = fb[o] + q0L;
#pragma unroll
                for (int i = 0; i < K2; ++i) v[i] = (double)p[loff[i]];
            } else {
#pragma unroll
                for (int le = 0; le < KK; ++le)
#pragma unroll
                    for (int ld = 0; ld < KK; ++ld)
                        v[le * KK + ld] = vn_load(lay, src, q0 + ld * kd + le * ke, s_lp[o], s_in[o]);
            }
            if (RS != K2) v[K2] = 0.0;
            if (uni) {
                // outer product over l: K2 independent accumulator chains (each out[m] still sums
                // over l = 0, 1, ... in order)
                const double* Mo = sM + o * K2 * RS;
#pragma unroll
                for (int l = 0; l < K2; ++l) {
#pragma unroll
                    for (int m = 0; m < RS; m += 2) {
                        const double2 mm = *(const double2*)&Mo[l * RS + m];
                        out[m] = fma(mm.x, v[l], out[m]);
                        if (m + 1 < K2) out[m + 1] = fma(mm.y, v[l], out[m + 1]);
                    }
                }
            } else {
                const double* Mo = M + o * K4;
#pragma unroll
                for (int m = 0; m < K2; ++m) {
                    double acc = out[m];
#pragma unroll
                    for (int l = 0; l < K2; ++l) acc = fma(__ldg(&Mo[m * K2 + l]), v[l], acc);
                    out[m] = acc;
                }
            }
        }
        if (all_f) {
            float* p = dst.pl + (lp * nf_ - nd_) * lay.L + inner + q0L;
#pragma unroll
            for (int me = 0; me < KK; ++me)
#pragma unroll
                for (int md = 0; md < KK; ++md) p[loff[me * KK + md]] = __double2float_rn(out[me * KK + md]);
        } else {
#pragma unroll
            for (int me = 0; me < KK; ++me)
#pragma unroll
                for (int md = 0; md < KK; ++md) vn_store(lay, dst, q0 + md * kd + me * ke, lp, inner, out[me * KK + md]);
        }
    }
}

// Round 2 (NEXT-3 speed): CPT consecutive cells per thread.  Taken when the CTA's 256 CPT cells
// share their v-cell (S_e a multiple of 256 CPT) and d is not the layer dim, so M_o always comes
// from shared memory and every 16-byte M read serves CPT cells (the one-cell kernel spends most
// of its issue slots and L1 bandwidth on those reads: profiles/round1/ncu_full_vnode_c5s.md).
// The source offset of cell c at offset o is one int32 delta (cells) from the cell itself; the
// offset loop is unrolled to kVnMaxOfs with guards, so deltas and accumulators stay in registers.
// Same operation order per output as vnode_sweep_kernel: results are bit-identical.
template <int KK, int CPT>
__global__ void __launch_bounds__(256, KK <= 3 ? 2 : 1) vnode_sweep_multi(Layout lay, int d, int e, const double* __restrict__ rec,
                                                            Arrays src, Arrays dst)
{
    constexpr int K2 = KK * KK, K4 = K2 * K2;
    constexpr int RS = (K2 + 1) & ~1;
    extern __shared__ __align__(16) double sM[];  // [kVnMaxOfs][K2][RS]
    const int D = lay.D;
    const int64_t cta0 = (int64_t)blockIdx.x * blockDim.x * CPT;
    const int64_t t0 = cta0 + (int64_t)threadIdx.x * CPT;
    auto idx_of = [&](int dd, int64_t lay_, int64_t in_) -> int64_t {
        if (dd == D - 1) return lay.first_layer + lay_;
        return (in_ / lay.S[dd]) % lay.n[dd];
    };
    const int64_t l0 = cta0 / lay.L;
    const int64_t j = idx_of(e, l0, cta0 - l0 * lay.L);  // the CTA's v-cell
    const double* r = rec + j * vn_rec_words(KK);
    const int64_t omin = (int64_t)__double_as_longlong(__ldg(&r[0]));
    const int nofs = (int)__double_as_longlong(__ldg(&r[1]));
    {
        const double* M0 = r + 2;
        for (int x = threadIdx.x; x < kVnMaxOfs * K4; x += blockDim.x) {  // transposed: [o][l][m]
            const int o = x / K4, rem = x - o * K4, m = rem / K2, l = rem - m * K2;
            sM[(o * K2 + l) * RS + m] = __ldg(&M0[x]);
        }
        if (RS != K2)
            for (int x = threadIdx.x; x < kVnMaxOfs * K2; x += blockDim.x) sM[x * RS + K2] = 0.0;
        __syncthreads();
    }
    if (t0 >= lay.cells) return;
    const int64_t layer = t0 / lay.L, inner = t0 - layer * lay.L;
    const int64_t lp = lay.pad + layer;
    const int64_t nd = lay.n[d];
    const int64_t id0 = idx_of(d, layer, inner);
    int dl[CPT][kVnMaxOfs];  // source cell of (cell c, offset o) relative to cell c
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const int64_t id = (d == 0) ? id0 + c : id0;  // n0 % CPT == 0: a thread's cells share a line along d > 0
#pragma unroll
        for (int o = 0; o < kVnMaxOfs; ++o) {
            int64_t sidx = (id - (omin + o)) % nd;
            if (sidx < 0) sidx += nd;
            dl[c][o] = (int)((sidx - id) * lay.S[d]);
        }
    }
    int kd = 1, ke = 1;
    for (int x = 0; x < d; ++x) kd *= KK;
    for (int x = 0; x < e; ++x) ke *= KK;
    const int64_t kdL = (int64_t)kd * lay.L, keL = (int64_t)ke * lay.L;
    const int nd_ = lay.nd, nf_ = lay.K - lay.nd;
    const float* fb = src.pl + (lp * nf_ - nd_) * lay.L + inner;
    float* fo = dst.pl + (lp * nf_ - nd_) * lay.L + inner;
    const int nblk = lay.K / K2;
    for (int b = 0; b < nblk; ++b) {
        int q0 = 0, bb = b, kp = 1;
        for (int x = 0; x < D; ++x) {
            if (x != d && x != e) {
                q0 += (bb % KK) * kp;
                bb /= KK;
            }
            kp *= KK;
        }
        const int64_t q0L = (int64_t)q0 * lay.L;
        const bool all_f = (q0 >= nd_);
        double out[CPT][K2];
#pragma unroll
        for (int c = 0; c < CPT; ++c)
#pragma unroll
            for (int m = 0; m < K2; ++m) out[c][m] = 0.0;
#pragma unroll
        for (int o = 0; o < kVnMaxOfs; ++o) {
            if (o >= nofs) break;
            double v[CPT][RS];
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                if (all_f) {
                    const float* p = fb + q0L + c + dl[c][o];
#pragma unroll
                    for (int le = 0; le < KK; ++le)
#pragma unroll
                        for (int ld = 0; ld < KK; ++ld) v[c][le * KK + ld] = (double)p[ld * kdL + le * keL];
                } else {
#pragma unroll
                    for (int le = 0; le < KK; ++le)
#pragma unroll
                        for (int ld = 0; ld < KK; ++ld)
                            v[c][le * KK + ld] = vn_load(lay, src, q0 + ld * kd + le * ke, lp, inner + c + dl[c][o]);
                }
                if (RS != K2) v[c][K2] = 0.0;
            }
            const double* Mo = sM + o * K2 * RS;
#pragma unroll
            for (int l = 0; l < K2; ++l) {  // outer product over l: CPT K2 independent chains
#pragma unroll
                for (int m = 0; m < RS; m += 2) {
                    const double2 mm = *(const double2*)&Mo[l * RS + m];
#pragma unroll
                    for (int c = 0; c < CPT; ++c) {
                        out[c][m] = fma(mm.x, v[c][l], out[c][m]);
                        if (m + 1 < K2) out[c][m + 1] = fma(mm.y, v[c][l], out[c][m + 1]);
                    }
                }
            }
        }
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            if (all_f) {
                float* p = fo + q0L + c;
#pragma unroll
                for (int me = 0; me < KK; ++me)
#pragma unroll
                    for (int md = 0; md < KK; ++md) p[md * kdL + me * keL] = __double2float_rn(out[c][me * KK + md]);
            } else {
#pragma unroll
                for (int me = 0; me < KK; ++me)
#pragma unroll
                    for (int md = 0; md < KK; ++md)
                        vn_store(lay, dst, q0 + md * kd + me * ke, lp, inner + c, out[c][me * KK + md]);
            }
        }
    }
}

}  // namespace

int64_t vnode_rec_words(int k) { return vn_rec_words(k); }

cudaError_t launch_vnode_weights(int k, const double* d_nodal, int64_t nv, double* d_rec, int* d_err, cudaStream_t s)
{
    vnode_weights_kernel<<<(unsigned)nv, 128, 0, s>>>(k, d_nodal, nv, d_rec, d_err, gauss_table(k));
    return cudaGetLastError();
}

cudaError_t launch_vnode_sweep(const Layout& lay, int d, int e, const double* d_rec, const Arrays& src,
                               const Arrays& dst, cudaStream_t s)
{
    const unsigned blocks = (unsigned)((lay.cells + 255) / 256);
    if (blocks == 0) return cudaSuccess;
    const int k2 = lay.k * lay.k;
    const size_t smem = (size_t)kVnMaxOfs * k2 * ((k2 + 1) & ~1) * sizeof(double);
    // CPT = 2 cells per thread where every CTA's 512 cells share their v-cell (SLDG_VN_MULTI=0: off)
    constexpr int CPT = 2;
    const char* em = getenv("SLDG_VN_MULTI");
    const bool multi = !(em && atoi(em) == 0) && lay.k <= 3 && d != lay.D - 1 && lay.n[0] % CPT == 0 &&
                       (int64_t)lay.K * lay.L < ((int64_t)1 << 31) &&
                       ((e == lay.D - 1) ? lay.L : lay.S[e]) % (256 * CPT) == 0;
    if (multi) {
        const unsigned mb = (unsigned)(lay.cells / (256 * CPT));
        switch (lay.k) {
            case 1: vnode_sweep_multi<1, CPT><<<mb, 256, smem, s>>>(lay, d, e, d_rec, src, dst); break;
            case 2: vnode_sweep_multi<2, CPT><<<mb, 256, smem, s>>>(lay, d, e, d_rec, src, dst); break;
            case 3: vnode_sweep_multi<3, CPT><<<mb, 256, smem, s>>>(lay, d, e, d_rec, src, dst); break;
            case 4: vnode_sweep_multi<4, CPT><<<mb, 256, smem, s>>>(lay, d, e, d_rec, src, dst); break;
            default: return cudaErrorInvalidValue;
        }
        return cudaGetLastError();
    }
    switch (lay.k) {
        case 1: vnode_sweep_kernel<1><<<blocks, 256, smem, s>>>(lay, d, e, d_rec, src, dst); break;
        case 2: vnode_sweep_kernel<2><<<blocks, 256, smem, s>>>(lay, d, e, d_rec, src, dst); break;
        case 3: vnode_sweep_kernel<3><<<blocks, 256, smem, s>>>(lay, d, e, d_rec, src, dst); break;
        case 4: vnode_sweep_kernel<4><<<blocks, 256, smem, s>>>(lay, d, e, d_rec, src, dst); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace sldg
