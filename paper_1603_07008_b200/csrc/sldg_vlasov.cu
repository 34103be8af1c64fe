// sldg_vlasov.cu -- the Vlasov-Poisson driver around the SLDG sweep (NEXT-2 of SURVEY 8(f);
// include/sldg.h "Vlasov-Poisson driver", readings V1-V6).
//
// Model: d_t f + v d_x f + E(x) d_v f = 0; Cheng-Knorr splitting into 1D advections
// whose CFL number depends on the field.  Field solver: S:267-334 (V2,
// V3) and a spectral reading for two space dims (V4).  Every step below runs on the grid's
// stream:
//   vp_x_field_kernel        nu of an x_c sweep per v_c cell                         (V5)
//   vp_density_partial_kernel / vp_density_final_kernel
//                            rho = (prod h_v) sum_{i_v} c_{(i_x,i_v),(m_x,0)}, a fixed-order
//                            two-pass sum (v split into kVSplit ranges)              (V2)
//   vp_poisson1d_kernel      one CTA: exact antiderivative per cell, cumulative interface
//                            constants, zero-mean gauge, centre values, energy       (V3)
//   vp_dft_* kernels         2D periodic Poisson on the cell means by direct DFTs in fp64
//                            (n1 n2 (n1 + n2) complex multiply-adds per transform) (V4)
//   vp_v_field_kernel        nu of a v_c sweep per x cell                            (V5)
// The sweeps are sldg_advect_device calls on the same grid.
#include <cuda_runtime.h>
#include <math.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "sldg_basis.cuh"
#include "sldg_internal.h"

using namespace sldg;

namespace {

constexpr int kVSplit = 16;  // v ranges of the first density pass (fixed => deterministic order)

__device__ __forceinline__ double vp_load(const Layout& L, const Arrays& a, int q, int64_t lp, int64_t inner)
{
    if (q < L.nd) return *dslot(a, lp, L.nd, q, L.L, inner);
    return (double)*fslot(a, lp, L.K, L.nd, q, L.L, inner);
}

// partial[(s * Kx + m) * Nx + ix] = sum over the s-th range of the local v cells
// (v cell = (local layer, iv_in): inner = ix + Nx * iv_in, iv_in < L / Nx)
__global__ void vp_density_partial_kernel(Layout lay, Arrays a, int64_t Nx, int Kx, double* partial)
{
    const int64_t ix = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int m = blockIdx.y, s = blockIdx.z;
    if (ix >= Nx) return;
    const int64_t nvin = lay.L / Nx;
    const int64_t nv = nvin * lay.layers;  // local v cells
    const int64_t b = nv * s / kVSplit, e = nv * (s + 1) / kVSplit;
    double acc = 0.0;
    int64_t layer = b / nvin, ivin = b - (b / nvin) * nvin;
    for (int64_t v = b; v < e; ++v) {
        acc += vp_load(lay, a, m, lay.pad + layer, ix + Nx * ivin);
        if (++ivin == nvin) {
            ivin = 0;
            ++layer;
        }
    }
    partial[((int64_t)s * Kx + m) * Nx + ix] = acc;
}

// rho[ix * Kx + m] = hv * sum_r sum_s partial_r[s][m][ix] (ranks, then ranges, in order)
__global__ void vp_density_final_kernel(const double* partial, int world, int64_t Nx, int Kx, double hv,
                                        double* rho)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= Nx * Kx) return;
    const int64_t ix = t % Nx;
    const int m = (int)(t / Nx);
    double acc = 0.0;
    for (int r = 0; r < world; ++r)
        for (int s = 0; s < kVSplit; ++s) acc += partial[(((int64_t)r * kVSplit + s) * Kx + m) * Nx + ix];
    rho[ix * Kx + m] = hv * acc;
}

// P_n(0): 1, 0, -1/2, 0, 3/8, ...
__device__ __forceinline__ double legendre_at0(int n)
{
    double p0 = 1.0, p1 = 0.0;
    if (n == 0) return 1.0;
    for (int j = 1; j < n; ++j) {  // (j+1) P_{j+1}(0) = -j P_{j-1}(0)
        const double p2 = -(double)j * p0 / (double)(j + 1);
        p0 = p1;
        p1 = p2;
    }
    return p1;
}

// V3 for one periodic line of n cells (one CTA, fixed-order reductions):
//   g_i = rho_i - rho_bar delta_m0; f_i = (h/2) int_{-1}^{xi} g_i (Legendre coefficients 0..k)
//   left_i = sum_{j<i} h g_j0; C0 = -mean_i(left_i + f_i0); e_i = f_i + (C0 + left_i) delta_n0
// e: n * (k+1) coefficients; ec: centre values; energy: 1/2 sum_i h sum_n e_in^2 / (2n+1).
__global__ void vp_poisson1d_kernel(const double* rho, int64_t n, int k, double h, double* work, double* e,
                                    double* ec, double* energy)
{
    __shared__ double sh[256];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t chunk = (n + nt - 1) / nt;
    const int64_t b = (tid * chunk < n) ? tid * chunk : n;
    const int64_t en = (b + chunk < n) ? b + chunk : n;
    // rho_bar: chunk sums, then thread 0 in order
    double s = 0.0;
    for (int64_t i = b; i < en; ++i) s += rho[i * k];
    sh[tid] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int j = 0; j < nt; ++j) t += sh[j];
        work[0] = t / (double)n;
    }
    __syncthreads();
    const double rb = work[0];
    const int K1 = k + 1;
    // antiderivative coefficients into e (before the constants)
    for (int64_t i = tid; i < n; i += nt) {
        double f[SLDG_MAX_K + 1];
        for (int m = 0; m <= k; ++m) f[m] = 0.0;
        const double g0 = rho[i * k] - rb;
        f[0] += g0;
        f[1] += g0;
        for (int m = 1; m < k; ++m) {
            const double gm = rho[i * k + m] / (double)(2 * m + 1);
            f[m + 1] += gm;
            f[m - 1] -= gm;
        }
        for (int m = 0; m <= k; ++m) e[i * K1 + m] = f[m] * (h / 2);
    }
    __syncthreads();
    // left_i: exclusive prefix sum of h g_j0 -- chunk totals, exclusive scan by thread 0, chunk pass
    s = 0.0;
    for (int64_t i = b; i < en; ++i) s += h * (rho[i * k] - rb);
    __syncthreads();
    sh[tid] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int j = 0; j < nt; ++j) {
            const double v = sh[j];
            sh[j] = t;
            t += v;
        }
    }
    __syncthreads();
    double left = sh[tid];
    double msum = 0.0;  // sum of left_i + f_i0 over the chunk
    for (int64_t i = b; i < en; ++i) {
        work[1 + i] = left;
        msum += left + e[i * K1];
        left += h * (rho[i * k] - rb);
    }
    __syncthreads();
    sh[tid] = msum;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int j = 0; j < nt; ++j) t += sh[j];
        work[0] = -t / (double)n;
    }
    __syncthreads();
    const double c0 = work[0];
    double en_acc = 0.0;
    for (int64_t i = b; i < en; ++i) {
        e[i * K1] += c0 + work[1 + i];
        double v = 0.0, w = 0.0;
        for (int m = 0; m <= k; ++m) {
            const double em = e[i * K1 + m];
            v += em * legendre_at0(m);
            w += em * em / (double)(2 * m + 1);
        }
        ec[i] = v;
        en_acc += h * w;
    }
    __syncthreads();
    sh[tid] = en_acc;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int j = 0; j < nt; ++j) t += sh[j];
        *energy = 0.5 * t;
    }
}

// e^{sign 2 pi i (a b mod n) / n}
__device__ __forceinline__ void twiddle(int64_t a, int64_t b, int64_t n, double sign, double* c, double* s)
{
    const int64_t r = (a * b) % n;
    double sv, cv;
    sincospi(2.0 * (double)r / (double)n, &sv, &cv);
    *c = cv;
    *s = sign * sv;
}

// signed angular frequency of index j on a periodic interval of n cells and length len
__device__ __forceinline__ double vp_freq(int64_t j, int64_t n, double len)
{
    const int64_t js = (j < (n + 1) / 2) ? j : j - n;  // numpy.fft.fftfreq ordering
    return 2.0 * M_PI * (double)js / len;
}

// F[t] = rho_mean(t) + 0i  (rho_mean = rho[t * Kx], the P_0 coefficient of x-cell t)
__global__ void vp_dft_load_kernel(const double* rho, int Kx, int64_t N, double2* F)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < N) F[t] = make_double2(rho[t * Kx], 0.0);
}

// one direct DFT pass along a dim of extent n and element stride `stride` of an N-element
// complex array: out[.. k ..] = sum_i in[.. i ..] e^{sign 2 pi i (k i mod n) / n}
__global__ void vp_dft_pass_kernel(const double2* in, double2* out, int64_t N, int64_t n, int64_t stride,
                                   double sign)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N) return;
    const int64_t kk = (t / stride) % n;
    const int64_t base = t - kk * stride;
    double re = 0.0, im = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double c, s;
        twiddle(kk, i, n, sign, &c, &s);
        const double2 a = in[base + i * stride];
        re += a.x * c - a.y * s;
        im += a.x * s + a.y * c;
    }
    out[t] = make_double2(re, im);
}

// Ehat_c = -i kappa_c phi_hat, phi_hat = F / |kappa|^2 (0 at kappa = 0); Nyquist modes of the
// derivative along c zeroed (V4).  dims / lengths of the dx x dims, dim 0 fastest.
struct VpDims {
    int dx;
    int64_t n[3];
    double len[3];
};
__global__ void vp_solve_kernel(const double2* F, int64_t N, VpDims g, int c, double2* E)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N) return;
    int64_t rem = t;
    double kk = 0.0, qc = 0.0;
    bool nyq = false;
    for (int a = 0; a < g.dx; ++a) {
        const int64_t j = rem % g.n[a];
        rem /= g.n[a];
        const double q = vp_freq(j, g.n[a], g.len[a]);
        kk += q * q;
        if (a == c) {
            qc = q;
            nyq = (g.n[a] % 2 == 0) && (j == g.n[a] / 2);
        }
    }
    const double d = nyq ? 0.0 : qc;
    double pr = 0.0, pi = 0.0;
    if (kk > 0.0) {
        pr = F[t].x / kk;
        pi = F[t].y / kk;
    }
    E[t] = make_double2(d * pi, -d * pr);  // -i d (pr + i pi)
}

// ec[t] = Re(A[t]) / N
__global__ void vp_real_scale_kernel(const double2* A, int64_t N, double* ec)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < N) ec[t] = A[t].x / (double)N;
}

// energy = 1/2 (prod h) sum_c sum (E_c^2), one CTA, fixed order
__global__ void vp_energy_nd_kernel(const double* ec, int64_t N, int dx, double hprod, double* energy)
{
    __shared__ double sh[256];
    const int tid = threadIdx.x, nt = blockDim.x;
    double s = 0.0;
    for (int64_t i = tid; i < N; i += nt)
        for (int c = 0; c < dx; ++c) s += ec[c * N + i] * ec[c * N + i];
    sh[tid] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int j = 0; j < nt; ++j) t += sh[j];
        *energy = 0.5 * hprod * t;
    }
}

// V5: nu[i] = (lo_v + (i + 1/2) h_v) * tau / h_x
__global__ void vp_x_field_kernel(int64_t nv, double lo_v, double h_v, double tau, double h_x, double* nu)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nv) nu[i] = (lo_v + ((double)i + 0.5) * h_v) * tau / h_x;
}

// V7 (NEXT-3): nu[i * k + n] = (lo_v + (i + 1/2) h_v + xi_n h_v / 2) * tau / h_x at the Gauss nodes
__global__ void vp_x_nodal_field_kernel(int64_t nv, int k, double lo_v, double h_v, double tau, double h_x,
                                        double* nu, const GaussTab gt)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nv * k) return;
    const int64_t i = t / k;
    const int n = (int)(t - i * k);
    nu[t] = (lo_v + ((double)i + 0.5) * h_v + gt.x[n] * h_v / 2) * tau / h_x;
}

// V5: nu[i_x] = E_c(i_x) * tau / h_v
__global__ void vp_v_field_kernel(const double* ec, int64_t N, double tau, double h_v, double* nu)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N) nu[i] = ec[i] * tau / h_v;
}

unsigned nblk(int64_t n, int bs = 256) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

struct sldg_vp_s {
    sldg_grid g = nullptr;
    int dx = 1, k = 1, Kx = 1;
    bool nodal = false;        // x sweeps by the Gauss-node velocity treatment (V7)
    int64_t nx[3] = {1, 1, 1}, Nx = 1;
    double hv = 1.0;           // prod_c h_vc
    double* d_partial = nullptr;   // [world][kVSplit][Kx][Nx]
    double* d_rho = nullptr;       // [Nx][Kx]
    double* d_work = nullptr;      // 1 + Nx (poisson1d scratch)
    double* d_ecoef = nullptr;     // dx = 1: [Nx][k+1]
    double* d_ec = nullptr;        // [dx][Nx] centre values
    double* d_energy = nullptr;
    double2* d_c[2] = {nullptr, nullptr};  // dx >= 2: DFT work [Nx] each
    double2* d_ctmp = nullptr;
    double* d_nux[3] = {nullptr, nullptr, nullptr};  // x_c sweep fields [n_vc] (nodal: [n_vc k])
    double* d_nuv[3] = {nullptr, nullptr, nullptr};  // v_c sweep fields [Nx]
    std::vector<void*> allocs;
};

namespace {

#define VCU(call)                                                                                  \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return set_error(e_ == cudaErrorMemoryAllocation ? SLDG_ENOMEM : SLDG_ECUDA,           \
                             std::string(#call) + ": " + cudaGetErrorString(e_));                  \
    } while (0)

sldg_status vp_alloc(sldg_vp vp, void** p, size_t bytes)
{
    VCU(cudaMalloc(p, std::max<size_t>(bytes, 8)));
    vp->allocs.push_back(*p);
    return SLDG_OK;
}

// density of the grid's current buffer into vp->d_rho (device), rank-ordered over ranks
sldg_status vp_density_dev(sldg_vp vp)
{
    sldg_grid g = vp->g;
    const Layout& L = g->lay;
    const Arrays& a = g->buf[g->cur];
    cudaStream_t s = g->stream;
    const int64_t part = (int64_t)kVSplit * vp->Kx * vp->Nx;
    const bool gather = g->world > 1 || g->nccl_self;
    double* mine = vp->d_partial + (g->world > 1 ? (int64_t)g->rank * part : 0);
    if (g->nccl_self) mine = vp->d_partial + part;  // gathered into slot 0 through NCCL (testing)
    vp_density_partial_kernel<<<dim3(nblk(vp->Nx), vp->Kx, kVSplit), 256, 0, s>>>(L, a, vp->Nx, vp->Kx, mine);
    VCU(cudaGetLastError());
    g->launches += 1;
    if (gather) {
        ncclResult_t r = ncclAllGather(mine, vp->d_partial, (size_t)part, ncclFloat64, (ncclComm_t)g->comm, s);
        if (r != ncclSuccess) return set_error(SLDG_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    }
    vp_density_final_kernel<<<nblk(vp->Nx * vp->Kx), 256, 0, s>>>(vp->d_partial, g->world, vp->Nx, vp->Kx, vp->hv,
                                                                  vp->d_rho);
    VCU(cudaGetLastError());
    g->launches += 1;
    return SLDG_OK;
}

// field from vp->d_rho into d_ec (centres), d_ecoef (dx = 1), d_energy
sldg_status vp_field_dev(sldg_vp vp)
{
    sldg_grid g = vp->g;
    cudaStream_t s = g->stream;
    if (vp->dx == 1) {
        const double h = g->h[0];
        vp_poisson1d_kernel<<<1, 256, 0, s>>>(vp->d_rho, vp->Nx, vp->k, h, vp->d_work, vp->d_ecoef, vp->d_ec,
                                              vp->d_energy);
        VCU(cudaGetLastError());
        g->launches += 1;
        return SLDG_OK;
    }
    const int64_t N = vp->Nx;
    VpDims gd{};
    gd.dx = vp->dx;
    double hprod = 1.0;
    for (int c = 0; c < vp->dx; ++c) {
        gd.n[c] = vp->nx[c];
        gd.len[c] = g->hi[c] - g->lo[c];
        hprod *= g->h[c];
    }
    // forward transform of the cell means, one pass per x dim (ping-pong d_c[0] <-> d_c[1])
    vp_dft_load_kernel<<<nblk(N), 256, 0, s>>>(vp->d_rho, vp->Kx, N, vp->d_c[0]);
    int cur = 0;
    int64_t stride = 1;
    for (int c = 0; c < vp->dx; ++c) {
        vp_dft_pass_kernel<<<nblk(N), 256, 0, s>>>(vp->d_c[cur], vp->d_c[1 - cur], N, vp->nx[c], stride, -1.0);
        cur = 1 - cur;
        stride *= vp->nx[c];
    }
    g->launches += 1 + vp->dx;
    // per component: solve into the spare buffer, inverse passes, real part
    const int F = cur;  // spectrum
    for (int c = 0; c < vp->dx; ++c) {
        double2* a = vp->d_c[1 - F];
        double2* b = vp->d_ctmp;
        vp_solve_kernel<<<nblk(N), 256, 0, s>>>(vp->d_c[F], N, gd, c, a);
        int64_t st2 = 1;
        for (int e = 0; e < vp->dx; ++e) {
            vp_dft_pass_kernel<<<nblk(N), 256, 0, s>>>(a, b, N, vp->nx[e], st2, 1.0);
            double2* t = a;
            a = b;
            b = t;
            st2 *= vp->nx[e];
        }
        vp_real_scale_kernel<<<nblk(N), 256, 0, s>>>(a, N, vp->d_ec + (int64_t)c * N);
        g->launches += 2 + vp->dx;
    }
    vp_energy_nd_kernel<<<1, 256, 0, s>>>(vp->d_ec, N, vp->dx, hprod, vp->d_energy);
    VCU(cudaGetLastError());
    g->launches += 1;
    return SLDG_OK;
}

sldg_status vp_x_sweeps(sldg_vp vp, double tau)
{
    sldg_grid g = vp->g;
    for (int c = 0; c < vp->dx; ++c) {
        const int dv = vp->dx + c;
        const int64_t nv = g->lay.n[dv];
        sldg_status st;
        if (vp->nodal) {
            vp_x_nodal_field_kernel<<<nblk(nv * vp->k), 256, 0, g->stream>>>(nv, vp->k, g->lo[dv], g->h[dv], tau,
                                                                             g->h[c], vp->d_nux[c],
                                                                             gauss_table(vp->k));
            VCU(cudaGetLastError());
            g->launches += 1;
            st = sldg_advect_vnodes_device(g, c, dv, vp->d_nux[c]);
        } else if (c == 0 && vp->dx >= 2) {
            // x1 and x2 together: their CFL numbers depend only on v1 / v2, so the pair runs in one
            // pass over HBM (sldg_advect_pair_device, bit-identical to the two sweeps)
            const int dv1 = vp->dx + 1;
            const int64_t nv1 = g->lay.n[dv1];
            vp_x_field_kernel<<<nblk(nv), 256, 0, g->stream>>>(nv, g->lo[dv], g->h[dv], tau, g->h[0], vp->d_nux[0]);
            VCU(cudaGetLastError());
            vp_x_field_kernel<<<nblk(nv1), 256, 0, g->stream>>>(nv1, g->lo[dv1], g->h[dv1], tau, g->h[1], vp->d_nux[1]);
            VCU(cudaGetLastError());
            g->launches += 2;
            st = sldg_advect_pair_device(g, 0.0, vp->d_nux[0], 1u << dv, 0.0, vp->d_nux[1], 1u << dv1);
            ++c;  // x2 done
        } else {
            vp_x_field_kernel<<<nblk(nv), 256, 0, g->stream>>>(nv, g->lo[dv], g->h[dv], tau, g->h[c], vp->d_nux[c]);
            VCU(cudaGetLastError());
            g->launches += 1;
            st = sldg_advect_device(g, c, 0.0, vp->d_nux[c], 1u << dv);
        }
        if (st != SLDG_OK) return st;
    }
    return SLDG_OK;
}

sldg_status copy_out(sldg_vp vp, double* host, const double* dev, size_t n)
{
    if (!host) return SLDG_OK;
    VCU(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, vp->g->stream));
    return SLDG_OK;
}

}  // namespace

extern "C" {

sldg_status sldg_vp_create(sldg_grid g, int dx, sldg_vp* out)
{
    if (!g || !out) return set_error(SLDG_EINVAL, "null argument");
    *out = nullptr;
    const Layout& L = g->lay;
    if (dx < 1 || dx > 3 || L.D != 2 * dx) return set_error(SLDG_EINVAL, "grid must be [x.., v..] with dx in {1, 2, 3}");
    if (L.prec == SLDG_GENERAL) return set_error(SLDG_EINVAL, "general precision layouts are 1D only");
    sldg_vp vp = new (std::nothrow) sldg_vp_s;
    if (!vp) return set_error(SLDG_ENOMEM, "host allocation");
    vp->g = g;
    vp->dx = dx;
    vp->k = L.k;
    vp->Kx = 1;
    for (int c = 0; c < dx; ++c) vp->Kx *= L.k;
    vp->Nx = 1;
    vp->hv = 1.0;
    for (int c = 0; c < dx; ++c) {
        vp->nx[c] = L.n[c];
        vp->Nx *= L.n[c];
        vp->hv *= g->h[dx + c];
    }
    const int64_t part = (int64_t)kVSplit * vp->Kx * vp->Nx;
    sldg_status st = SLDG_OK;
    auto A = [&](void** p, size_t b) {
        if (st == SLDG_OK) st = vp_alloc(vp, p, b);
    };
    A((void**)&vp->d_partial, (size_t)part * (std::max(1, g->world) + (g->nccl_self ? 1 : 0)) * sizeof(double));
    A((void**)&vp->d_rho, (size_t)vp->Nx * vp->Kx * sizeof(double));
    A((void**)&vp->d_work, (size_t)(vp->Nx + 1) * sizeof(double));
    A((void**)&vp->d_ecoef, (size_t)vp->Nx * (vp->k + 1) * sizeof(double));
    A((void**)&vp->d_ec, (size_t)dx * vp->Nx * sizeof(double));
    A((void**)&vp->d_energy, sizeof(double));
    if (dx >= 2) {
        for (int i = 0; i < 2; ++i) A((void**)&vp->d_c[i], (size_t)vp->Nx * sizeof(double2));
        A((void**)&vp->d_ctmp, (size_t)vp->Nx * sizeof(double2));
    }
    for (int c = 0; c < dx; ++c) {
        A((void**)&vp->d_nux[c], (size_t)L.n[dx + c] * L.k * sizeof(double));
        A((void**)&vp->d_nuv[c], (size_t)vp->Nx * sizeof(double));
    }
    if (st != SLDG_OK) {
        sldg_vp_destroy(vp);
        return st;
    }
    *out = vp;
    return SLDG_OK;
}

sldg_status sldg_vp_destroy(sldg_vp vp)
{
    if (!vp) return SLDG_OK;
    // no access to vp->g here: the grid may already be gone (the binding destroys drivers
    // first, but a C caller may not); cudaFree synchronises with outstanding device work
    cudaDeviceSynchronize();
    for (void* p : vp->allocs) cudaFree(p);
    delete vp;
    return SLDG_OK;
}

sldg_status sldg_vp_set_nodal(sldg_vp vp, int on)
{
    if (!vp) return set_error(SLDG_EINVAL, "null handle");
    if (on && vp->k > 4) return set_error(SLDG_ENOTSUP, "the Gauss-node sweep supports k <= 4");
    vp->nodal = (on != 0);
    return SLDG_OK;
}

sldg_status sldg_vp_density(sldg_vp vp, double* rho_out)
{
    if (!vp) return set_error(SLDG_EINVAL, "null handle");
    sldg_status st = vp_density_dev(vp);
    if (st != SLDG_OK) return st;
    st = copy_out(vp, rho_out, vp->d_rho, (size_t)vp->Nx * vp->Kx);
    if (st != SLDG_OK) return st;
    if (rho_out) VCU(cudaStreamSynchronize(vp->g->stream));
    return SLDG_OK;
}

sldg_status sldg_vp_field(sldg_vp vp, const double* rho, double* e_out, double* e_coef, double* energy)
{
    if (!vp) return set_error(SLDG_EINVAL, "null handle");
    if (e_coef && vp->dx != 1) return set_error(SLDG_EINVAL, "e_coef is for dx = 1 only");
    sldg_status st;
    if (rho) {
        const size_t n = (size_t)vp->Nx * vp->Kx;
        for (size_t i = 0; i < n; ++i)
            if (!isfinite(rho[i])) return set_error(SLDG_EINVAL, "non-finite density entry");
        VCU(cudaMemcpyAsync(vp->d_rho, rho, n * sizeof(double), cudaMemcpyHostToDevice, vp->g->stream));
        VCU(cudaStreamSynchronize(vp->g->stream));
    } else {
        st = vp_density_dev(vp);
        if (st != SLDG_OK) return st;
    }
    st = vp_field_dev(vp);
    if (st != SLDG_OK) return st;
    if ((st = copy_out(vp, e_out, vp->d_ec, (size_t)vp->dx * vp->Nx)) != SLDG_OK) return st;
    if ((st = copy_out(vp, e_coef, vp->d_ecoef, (size_t)vp->Nx * (vp->k + 1))) != SLDG_OK) return st;
    if ((st = copy_out(vp, energy, vp->d_energy, 1)) != SLDG_OK) return st;
    if (e_out || e_coef || energy) VCU(cudaStreamSynchronize(vp->g->stream));
    return SLDG_OK;
}

sldg_status sldg_vp_step(sldg_vp vp, double dt, double* energy_out)
{
    if (!vp) return set_error(SLDG_EINVAL, "null handle");
    if (!(dt > 0.0) || !isfinite(dt)) return set_error(SLDG_EINVAL, "dt must be finite and > 0");
    sldg_grid g = vp->g;
    sldg_status st = vp_x_sweeps(vp, dt / 2);
    if (st != SLDG_OK) return st;
    if ((st = vp_density_dev(vp)) != SLDG_OK) return st;
    if ((st = vp_field_dev(vp)) != SLDG_OK) return st;
    const uint32_t xmask = (1u << vp->dx) - 1u;
    for (int c = 0; c < vp->dx; ++c) {
        const int dv = vp->dx + c;
        vp_v_field_kernel<<<nblk(vp->Nx), 256, 0, g->stream>>>(vp->d_ec + (int64_t)c * vp->Nx, vp->Nx, dt, g->h[dv],
                                                               vp->d_nuv[c]);
        VCU(cudaGetLastError());
        g->launches += 1;
        st = sldg_advect_device(g, dv, 0.0, vp->d_nuv[c], xmask);
        if (st != SLDG_OK) return st;
    }
    if ((st = vp_x_sweeps(vp, dt / 2)) != SLDG_OK) return st;
    if (energy_out) {
        if ((st = copy_out(vp, energy_out, vp->d_energy, 1)) != SLDG_OK) return st;
        VCU(cudaStreamSynchronize(g->stream));
    }
    return SLDG_OK;
}

}  // extern "C"
