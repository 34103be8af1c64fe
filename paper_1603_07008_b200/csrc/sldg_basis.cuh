// sldg_basis.cuh -- device-side Legendre / Gauss-Legendre / shift-matrix helpers shared by the
// weight-build kernels of the plain sweep (sldg_kernels.cu) and of the Gauss-node velocity
// sweep (sldg_vnodes.cu).  Inline so that every translation unit has its own copy (no -rdc).
//
// build_ab: A_jl = (2j+1)/2 int_{-1}^{2a-1} P_l(xi+2-2a) P_j(xi) dxi, B_jl = (2j+1)/2
// int_{2a-1}^{1} P_l(xi-2a) P_j(xi) dxi (P:259-268 SS II-A), each by a k-point
// Gauss-Legendre rule mapped to the sub-interval (exact for the degree <= 2k-2 integrand), mass
// row in closed form (reading R3).
#pragma once
#include <math.h>

#include "sldg_internal.h"

namespace sldg {

__device__ __forceinline__ void dev_legendre(int pmax, double x, double* P)
{
    P[0] = 1.0;
    if (pmax > 0) P[1] = x;
    for (int n = 2; n <= pmax; ++n) P[n] = ((2 * n - 1) * x * P[n - 1] - (n - 1) * P[n - 2]) / n;
}

// Gauss-Legendre nodes/weights on [-1,1] by Newton on P_n (roots symmetric; compute the
// non-negative half and mirror).
__device__ __forceinline__ void dev_gauss(int n, double* x, double* w)
{
    const double kPi = 3.141592653589793238462643;
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double z = cos(kPi * (i + 0.75) / (n + 0.5));
        double pn = 0.0, dpn = 1.0;
        for (int it = 0; it < 60; ++it) {
            double p0 = 1.0, p1 = z;
            for (int m = 2; m <= n; ++m) {
                double p2 = ((2 * m - 1) * z * p1 - (m - 1) * p0) / m;
                p0 = p1;
                p1 = p2;
            }
            pn = (n == 1) ? z : p1;
            double pm1 = (n == 1) ? 1.0 : p0;
            dpn = n * (pm1 - z * pn) / (1.0 - z * z);
            double dz = pn / dpn;
            z -= dz;
            if (fabs(dz) < 1e-17) break;
        }
        {  // derivative at the converged node
            double p0 = 1.0, p1 = z;
            for (int m = 2; m <= n; ++m) {
                double p2 = ((2 * m - 1) * z * p1 - (m - 1) * p0) / m;
                p0 = p1;
                p1 = p2;
            }
            double pm1 = (n == 1) ? 1.0 : p0;
            double pnn = (n == 1) ? z : p1;
            dpn = n * (pm1 - z * pnn) / (1.0 - z * z);
        }
        double wi = 2.0 / ((1.0 - z * z) * dpn * dpn);
        x[i] = -z;
        w[i] = wi;
        x[n - 1 - i] = z;
        w[n - 1 - i] = wi;
    }
    if (n & 1) x[n / 2] = 0.0;
}


__device__ __forceinline__ void build_ab(int k, double a, double* A, double* B)
{
    double xg[kMaxK], wg[kMaxK], Pj[kMaxK + 2], Pl[kMaxK + 2];
    dev_gauss(k, xg, wg);
    for (int j = 0; j < k * k; ++j) {
        A[j] = 0.0;
        B[j] = 0.0;
    }
    for (int g = 0; g < k; ++g) {
        // A: xi in [-1, 2a-1] -> xi = (a - 1) + a t ; integrand P_l(xi + 2 - 2a) P_j(xi)
        double xi = (a - 1.0) + a * xg[g];
        dev_legendre(k - 1, xi, Pj);
        dev_legendre(k - 1, xi + 2.0 - 2.0 * a, Pl);
        for (int j = 0; j < k; ++j)
            for (int l = 0; l < k; ++l) A[j * k + l] += wg[g] * (Pj[j] * Pl[l]);
        // B: xi in [2a-1, 1] -> xi = a + (1 - a) t ; integrand P_l(xi - 2a) P_j(xi)
        xi = a + (1.0 - a) * xg[g];
        dev_legendre(k - 1, xi, Pj);
        dev_legendre(k - 1, xi - 2.0 * a, Pl);
        for (int j = 0; j < k; ++j)
            for (int l = 0; l < k; ++l) B[j * k + l] += wg[g] * (Pj[j] * Pl[l]);
    }
    for (int j = 0; j < k; ++j) {
        double sa = 0.5 * (2 * j + 1) * a, sb = 0.5 * (2 * j + 1) * (1.0 - a);
        for (int l = 0; l < k; ++l) {
            A[j * k + l] *= sa;
            B[j * k + l] *= sb;
        }
    }
    // mass row, closed form (reading R3): int_x^1 P_l = -(P_{l+1}(x) - P_{l-1}(x))/(2l+1)
    {
        double P[kMaxK + 2];
        dev_legendre(k, 1.0 - 2.0 * a, P);
        for (int l = 1; l < k; ++l) {
            double v = -(P[l + 1] - P[l - 1]) / (2.0 * (2 * l + 1));
            A[l] = v;
            B[l] = -v;
        }
        if (a <= 0.5) {
            B[0] = 1.0 - a;
            A[0] = 1.0 - B[0];
        } else {
            A[0] = a;
            B[0] = 1.0 - a;
        }
    }
}


}  // namespace sldg
