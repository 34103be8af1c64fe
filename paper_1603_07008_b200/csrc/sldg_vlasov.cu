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

// A[k1 + n1 i2] = sum_i1 rho_mean(i1, i2) e^{-2 pi i k1 i1 / n1}   (rho_mean = rho[(i1 + n1 i2) Kx])
__global__ void vp_dft_rows_kernel(const double* rho, int Kx, int64_t n1, int64_t n2, double2* A)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n1 * n2) return;
    const int64_t k1 = t % n1, i2 = t / n1;
    double re = 0.0, im = 0.0;
    for (int64_t i1 = 0; i1 < n1; ++i1) {
        double c, s;
        twiddle(k1, i1, n1, -1.0, &c, &s);
        const double r = rho[(i1 + n1 * i2) * Kx];
        re += r * c;
        im += r * s;
    }
    A[t] = make_double2(re, im);
}

// signed angular frequency of index j on a periodic interval of n cells and length len
__device__ __forceinline__ double vp_freq(int64_t j, int64_t n, double len)
{
    const int64_t js = (j < (n + 1) / 2) ? j : j - n;  // numpy.fft.fftfreq ordering
    return 2.0 * M_PI * (double)js / len;
}

// B = column DFT of A; then Ehat_c = -i kappa_c phi_hat, phi_hat = B / |kappa|^2 (0 at kappa = 0),
// with the Nyquist derivative modes zeroed (V4).  Out: E1hat, E2hat [k1 + n1 k2].
__global__ void vp_dft_cols_solve_kernel(const double2* A, int64_t n1, int64_t n2, double l1, double l2,
                                         double2* E1h, double2* E2h)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n1 * n2) return;
    const int64_t k1 = t % n1, k2 = t / n1;
    double re = 0.0, im = 0.0;
    for (int64_t i2 = 0; i2 < n2; ++i2) {
        double c, s;
        twiddle(k2, i2, n2, -1.0, &c, &s);
        const double2 a = A[k1 + n1 * i2];
        re += a.x * c - a.y * s;
        im += a.x * s + a.y * c;
    }
    const double q1 = vp_freq(k1, n1, l1), q2 = vp_freq(k2, n2, l2);
    const double kk = q1 * q1 + q2 * q2;
    double pr = 0.0, pi = 0.0;
    if (kk > 0.0) {
        pr = re / kk;
        pi = im / kk;
    }
    const double d1 = (n1 % 2 == 0 && k1 == n1 / 2) ? 0.0 : q1;
    const double d2 = (n2 % 2 == 0 && k2 == n2 / 2) ? 0.0 : q2;
    // -i d phi = (d pi, -d pr)
    E1h[t] = make_double2(d1 * pi, -d1 * pr);
    E2h[t] = make_double2(d2 * pi, -d2 * pr);
}

// T_c[k1 + n1 i2] = sum_k2 Ehat_c(k1, k2) e^{+2 pi i k2 i2 / n2}
__global__ void vp_idft_cols_kernel(const double2* E1h, const double2* E2h, int64_t n1, int64_t n2, double2* T1,
                                    double2* T2)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n1 * n2) return;
    const int64_t k1 = t % n1, i2 = t / n1;
    double r1 = 0.0, j1 = 0.0, r2 = 0.0, j2 = 0.0;
    for (int64_t k2 = 0; k2 < n2; ++k2) {
        double c, s;
        twiddle(k2, i2, n2, 1.0, &c, &s);
        const double2 a = E1h[k1 + n1 * k2], b = E2h[k1 + n1 * k2];
        r1 += a.x * c - a.y * s;
        j1 += a.x * s + a.y * c;
        r2 += b.x * c - b.y * s;
        j2 += b.x * s + b.y * c;
    }
    T1[t] = make_double2(r1, j1);
    T2[t] = make_double2(r2, j2);
}

// E_c(i1, i2) = Re sum_k1 T_c(k1, i2) e^{+2 pi i k1 i1 / n1} / (n1 n2) -> ec[c * N + i1 + n1 i2]
__global__ void vp_idft_rows_kernel(const double2* T1, const double2* T2, int64_t n1, int64_t n2, double* ec)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t N = n1 * n2;
    if (t >= N) return;
    const int64_t i1 = t % n1, i2 = t / n1;
    double r1 = 0.0, r2 = 0.0;
    for (int64_t k1 = 0; k1 < n1; ++k1) {
        double c, s;
        twiddle(k1, i1, n1, 1.0, &c, &s);
        const double2 a = T1[k1 + n1 * i2], b = T2[k1 + n1 * i2];
        r1 += a.x * c - a.y * s;
        r2 += b.x * c - b.y * s;
    }
    ec[t] = r1 / (double)N;
    ec[N + t] = r2 / (double)N;
}

// energy = 1/2 h1 h2 sum (E1^2 + E2^2), one CTA, fixed order
__global__ void vp_energy2d_kernel(const double* ec, int64_t N, double h1h2, double* energy)
{
    __shared__ double sh[256];
    const int tid = threadIdx.x, nt = blockDim.x;
    double s = 0.0;
    for (int64_t i = tid; i < N; i += nt) s += ec[i] * ec[i] + ec[N + i] * ec[N + i];
    sh[tid] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int j = 0; j < nt; ++j) t += sh[j];
        *energy = 0.5 * h1h2 * t;
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
                                        double* nu)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nv * k) return;
    double xg[kMaxK], wg[kMaxK];
    dev_gauss(k, xg, wg);
    const int64_t i = t / k;
    const int n = (int)(t - i * k);
    nu[t] = (lo_v + ((double)i + 0.5) * h_v + xg[n] * h_v / 2) * tau / h_x;
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
    int64_t nx[2] = {1, 1}, Nx = 1;
    double hv = 1.0;           // prod_c h_vc
    double* d_partial = nullptr;   // [world][kVSplit][Kx][Nx]
    double* d_rho = nullptr;       // [Nx][Kx]
    double* d_work = nullptr;      // 1 + Nx (poisson1d scratch)
    double* d_ecoef = nullptr;     // dx = 1: [Nx][k+1]
    double* d_ec = nullptr;        // [dx][Nx] centre values
    double* d_energy = nullptr;
    double2* d_c[4] = {nullptr, nullptr, nullptr, nullptr};  // dx = 2: DFT work [Nx] each
    double* d_nux[2] = {nullptr, nullptr};  // x_c sweep fields [n_vc]
    double* d_nuv[2] = {nullptr, nullptr};  // v_c sweep fields [Nx]
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
    const int64_t n1 = vp->nx[0], n2 = vp->nx[1], N = vp->Nx;
    const double l1 = g->hi[0] - g->lo[0], l2 = g->hi[1] - g->lo[1];
    vp_dft_rows_kernel<<<nblk(N), 256, 0, s>>>(vp->d_rho, vp->Kx, n1, n2, vp->d_c[0]);
    vp_dft_cols_solve_kernel<<<nblk(N), 256, 0, s>>>(vp->d_c[0], n1, n2, l1, l2, vp->d_c[1], vp->d_c[2]);
    vp_idft_cols_kernel<<<nblk(N), 256, 0, s>>>(vp->d_c[1], vp->d_c[2], n1, n2, vp->d_c[0], vp->d_c[3]);
    vp_idft_rows_kernel<<<nblk(N), 256, 0, s>>>(vp->d_c[0], vp->d_c[3], n1, n2, vp->d_ec);
    vp_energy2d_kernel<<<1, 256, 0, s>>>(vp->d_ec, N, g->h[0] * g->h[1], vp->d_energy);
    VCU(cudaGetLastError());
    g->launches += 5;
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
                                                                             g->h[c], vp->d_nux[c]);
            VCU(cudaGetLastError());
            g->launches += 1;
            st = sldg_advect_vnodes_device(g, c, dv, vp->d_nux[c]);
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
    if ((dx != 1 && dx != 2) || L.D != 2 * dx) return set_error(SLDG_EINVAL, "grid must be [x.., v..] with dx in {1, 2}");
    if (L.prec == SLDG_GENERAL) return set_error(SLDG_EINVAL, "general precision layouts are 1D only");
    sldg_vp vp = new (std::nothrow) sldg_vp_s;
    if (!vp) return set_error(SLDG_ENOMEM, "host allocation");
    vp->g = g;
    vp->dx = dx;
    vp->k = L.k;
    vp->Kx = (dx == 1) ? L.k : L.k * L.k;
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
    if (dx == 2)
        for (int i = 0; i < 4; ++i) A((void**)&vp->d_c[i], (size_t)vp->Nx * sizeof(double2));
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
    if (vp->g) cudaStreamSynchronize(vp->g->stream);
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
