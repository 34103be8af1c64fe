// sldg_basis.cuh -- device-side Legendre / Gauss-Legendre / shift-matrix helpers shared by the
// weight-build kernels of the plain sweep (sldg_kernels.cu) and of the Gauss-node velocity
// sweep (sldg_vnodes.cu).  Inline so that every translation unit has its own copy (no -rdc).
//
// build_ab: A_jl = (2j+1)/2 int_{-1}^{2a-1} P_l(xi+2-2a) P_j(xi) dxi, B_jl = (2j+1)/2
// int_{2a-1}^{1} P_l(xi-2a) P_j(xi) dxi (P:259-268 SS II-A), each by a k-point
// Gauss-Legendre rule mapped to the sub-interval (exact for the degree <= 2k-2 integrand), mass
// row in closed form (reading R3).  The Gauss nodes/weights come from the host (GaussTab,
// sldg_kernels.cu gauss_table) as a kernel parameter.
#pragma once
#include <math.h>

#include "sldg_internal.h"

namespace sldg {

__device__ __forceinline__ void dev_legendre(int pmax, double x, double* P)
{
    P[0] = 1.0;
    if (pmax > 0) P[1] = x;
#pragma unroll
    for (int n = 2; n <= pmax; ++n) P[n] = ((2 * n - 1) * x * P[n - 1] - (n - 1) * P[n - 2]) / n;
}

// KK compile-time: the Legendre values and both accumulators live in registers (a runtime k
// put them in local memory and made every += a dependent global read-modify-write of A / B).
template <int KK>
__device__ __forceinline__ void build_ab_regs(double a, const double* xg, const double* wg, double* Al, double* Bl)
{
    double Pj[KK + 2], Pl[KK + 2];
#pragma unroll
    for (int j = 0; j < KK * KK; ++j) {
        Al[j] = 0.0;
        Bl[j] = 0.0;
    }
#pragma unroll
    for (int g = 0; g < KK; ++g) {
        // A: xi in [-1, 2a-1] -> xi = (a - 1) + a t ; integrand P_l(xi + 2 - 2a) P_j(xi)
        double xi = (a - 1.0) + a * xg[g];
        dev_legendre(KK - 1, xi, Pj);
        dev_legendre(KK - 1, xi + 2.0 - 2.0 * a, Pl);
#pragma unroll
        for (int j = 0; j < KK; ++j)
#pragma unroll
            for (int l = 0; l < KK; ++l) Al[j * KK + l] += wg[g] * (Pj[j] * Pl[l]);
        // B: xi in [2a-1, 1] -> xi = a + (1 - a) t ; integrand P_l(xi - 2a) P_j(xi)
        xi = a + (1.0 - a) * xg[g];
        dev_legendre(KK - 1, xi, Pj);
        dev_legendre(KK - 1, xi - 2.0 * a, Pl);
#pragma unroll
        for (int j = 0; j < KK; ++j)
#pragma unroll
            for (int l = 0; l < KK; ++l) Bl[j * KK + l] += wg[g] * (Pj[j] * Pl[l]);
    }
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        const double sa = 0.5 * (2 * j + 1) * a, sb = 0.5 * (2 * j + 1) * (1.0 - a);
#pragma unroll
        for (int l = 0; l < KK; ++l) {
            Al[j * KK + l] *= sa;
            Bl[j * KK + l] *= sb;
        }
    }
    // mass row, closed form (reading R3): int_x^1 P_l = -(P_{l+1}(x) - P_{l-1}(x))/(2l+1)
    {
        double P[KK + 2];
        dev_legendre(KK, 1.0 - 2.0 * a, P);
#pragma unroll
        for (int l = 1; l < KK; ++l) {
            const double v = -(P[l + 1] - P[l - 1]) / (2.0 * (2 * l + 1));
            Al[l] = v;
            Bl[l] = -v;
        }
        if (a <= 0.5) {
            Bl[0] = 1.0 - a;
            Al[0] = 1.0 - Bl[0];
        } else {
            Al[0] = a;
            Bl[0] = 1.0 - a;
        }
    }
}

template <int KK>
__device__ __forceinline__ void build_ab_t(double a, double* A, double* B, const GaussTab& gt)
{
    double xg[KK], wg[KK], Al[KK * KK], Bl[KK * KK];
#pragma unroll
    for (int g = 0; g < KK; ++g) {
        xg[g] = gt.x[g];
        wg[g] = gt.w[g];
    }
    build_ab_regs<KK>(a, xg, wg, Al, Bl);
#pragma unroll
    for (int j = 0; j < KK * KK; ++j) {
        A[j] = Al[j];
        B[j] = Bl[j];
    }
}

__device__ __forceinline__ void build_ab(int k, double a, double* A, double* B, const GaussTab& gt)
{
    switch (k) {
        case 1: build_ab_t<1>(a, A, B, gt); break;
        case 2: build_ab_t<2>(a, A, B, gt); break;
        case 3: build_ab_t<3>(a, A, B, gt); break;
        case 4: build_ab_t<4>(a, A, B, gt); break;
        case 5: build_ab_t<5>(a, A, B, gt); break;
        case 6: build_ab_t<6>(a, A, B, gt); break;
        case 7: build_ab_t<7>(a, A, B, gt); break;
        default: build_ab_t<8>(a, A, B, gt); break;
    }
}

}  // namespace sldg
