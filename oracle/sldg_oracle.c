/*
 * sldg_oracle.c -- CPU ORACLE for the mixed-precision SLDG translate-and-project step
 * (Einkemmer, arXiv:1603.07008).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The product path
 * (paper_1603_07008_b200/) never imports, links or executes anything under oracle/.
 * It shares no code, headers, tables or constant generators with the CUDA path.
 *
 * Plain, slow, obviously-correct loops in fp64.  Build flags: -O2 -fno-fast-math
 * -ffp-contract=off (no FMA contraction, no reassociation).
 *
 * Citation keys: P:NNN = /root/reference/PAPER.md line NNN (section noted),
 *                S:NNN = /root/reference/SPEC.md line NNN,
 *                SURVEY 8(c) = /root/repo/SURVEY.md section 8(c) (the readings C1..C19).
 *
 * Host coefficient layout (shared with the C ABI's set/get, nothing else):
 *   c[cell * K + q],  K = k^D,
 *   cell = sum_d i_d * S_d,  S_0 = 1, S_d = prod_{e<d} n_e   (dim 0 fastest),
 *   q    = sum_d m_d * k^d                                     (m_0 fastest).
 *
 * Precision variants ("n_double"): coefficient slots q < n_double are kept in fp64; every
 * slot q >= n_double is stored as the nearest fp32 (round-to-nearest-even) and held here
 * as the double that fp32 value promotes to (exact).  n_double = 1 is the paper's
 * mixed scheme (c_0 in fp64, P:253-257 SS II-A; in multi-D only the all-zero multi-index,
 * SURVEY C8); n_double = K is the all-fp64 variant; n_double = 0 is pure fp32 (P:409-429
 * rows "0").
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py (see DESIGN.md
 * "Oracle pins").  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_ENOMEM 2

/* ------------------------------------------------------------------------------------ */
/* Legendre polynomials, three-term recurrence:                               */
/*   P_0 = 1, P_1 = x, (j+1) P_{j+1} = (2j+1) x P_j - j P_{j-1}.                        */
/* P_j is "the jth Legendre polynomial defined on [-1,1]" (SS II-A).          */
/* ------------------------------------------------------------------------------------ */
void or_legendre_all(int p, double x, double* out)
{
    out[0] = 1.0;
    if (p >= 1) out[1] = x;
    for (int j = 1; j < p; ++j)
        out[j + 1] = ((2.0 * j + 1.0) * x * out[j] - (double)j * out[j - 1]) / (j + 1.0);
}

/* ------------------------------------------------------------------------------------ */
/* Gauss-Legendre rule with n nodes on [-1,1] ("performing a Gauss-Legendre quadrature",  */
/* P:244, SS II-A).  Nodes = roots of P_n by Newton iteration from the standard guess    */
/* cos(pi (i - 1/4) / (n + 1/2)); weights w = 2 / ((1 - x^2) P_n'(x)^2).   */
/* Nodes returned in increasing order.                                                   */
/* ------------------------------------------------------------------------------------ */
int or_gauss_legendre(int n, double* nodes, double* weights)
{
    if (n < 1 || n > 64) return OR_EINVAL;
    const double pi = 3.14159265358979323846;
    for (int i = 1; i <= n; ++i) {
        double x = cos(pi * (i - 0.25) / (n + 0.5));
        double dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            /* P_n(x) and P_n'(x) by the recurrence */
            double p0 = 1.0, p1 = x;
            if (n == 1) { p1 = x; }
            for (int j = 1; j < n; ++j) {
                double p2 = ((2.0 * j + 1.0) * x * p1 - (double)j * p0) / (j + 1.0);
                p0 = p1;
                p1 = p2;
            }
            /* here p1 = P_n(x), p0 = P_{n-1}(x) (for n == 1: p0 = P_0 = 1) */
            dp = (double)n * (x * p1 - p0) / (x * x - 1.0);
            double dx = p1 / dp;
            x -= dx;
            if (fabs(dx) <= 1e-16) break;
        }
        /* recompute derivative at the converged root */
        {
            double p0 = 1.0, p1 = x;
            for (int j = 1; j < n; ++j) {
                double p2 = ((2.0 * j + 1.0) * x * p1 - (double)j * p0) / (j + 1.0);
                p0 = p1;
                p1 = p2;
            }
            dp = (double)n * (x * p1 - p0) / (x * x - 1.0);
        }
        /* guess i gives the i-th largest root; store ascending */
        nodes[n - i] = x;
        weights[n - i] = 2.0 / ((1.0 - x * x) * dp * dp);
    }
    if (n % 2 == 1) nodes[n / 2] = 0.0; /* the middle root of an odd-degree P_n is 0 */
    return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Shift decomposition ("i* is the integer part of the CFL number";            */
/* S:207-215): i* = floor(nu), alpha = nu - i* in [0,1).  If the rounded      */
/* alpha equals 1.0 (tiny negative nu), use (i*+1, 0).                                   */
/* ------------------------------------------------------------------------------------ */
int or_shift_decompose(double nu, int64_t* istar, double* alpha)
{
    if (!isfinite(nu) || fabs(nu) >= 4.0e18) return OR_EINVAL;
    double f = floor(nu);
    double a = nu - f;
    int64_t i = (int64_t)f;
    if (a >= 1.0) { i += 1; a = 0.0; }
    *istar = i;
    *alpha = a;
    return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Shift matrices A(alpha), B(alpha) in R^{k x k} (P:259-268 update rule, SS II-A;        */
/* S:216-224):                                              */
/*   A_jl = (2j+1)/2 * int_{-1}^{2a-1} P_l(xi + 2 - 2a) P_j(xi) dxi                      */
/*   B_jl = (2j+1)/2 * int_{2a-1}^{1}  P_l(xi - 2a)     P_j(xi) dxi                      */
/* each integral by a k-node Gauss rule mapped onto the sub-interval (exact: the         */
/* integrand has degree j+l <= 2k-2).  alpha = 0 gives exactly A = 0, B = I. */
/* Row-major: A[j*k + l].                                                                */
/* ------------------------------------------------------------------------------------ */
int or_shift_matrices(double alpha, int k, double* A, double* B)
{
    if (k < 1 || k > 16 || !(alpha >= 0.0) || !(alpha < 1.0)) return OR_EINVAL;
    for (int j = 0; j < k; ++j)
        for (int l = 0; l < k; ++l) {
            A[j * k + l] = 0.0;
            B[j * k + l] = (j == l) ? 1.0 : 0.0;
        }
    if (alpha == 0.0) return OR_OK;

    double xq[16], wq[16], Pj[16], Pl[16];
    or_gauss_legendre(k, xq, wq);

    /* A: sub-interval [lo, hi] = [-1, 2a-1] */
    {
        double lo = -1.0, hi = 2.0 * alpha - 1.0;
        double half = 0.5 * (hi - lo), mid = 0.5 * (hi + lo);
        for (int j = 0; j < k; ++j)
            for (int l = 0; l < k; ++l) A[j * k + l] = 0.0;
        for (int q = 0; q < k; ++q) {
            double xi = mid + half * xq[q];
            or_legendre_all(k - 1, xi, Pj);
            or_legendre_all(k - 1, xi + 2.0 - 2.0 * alpha, Pl);
            for (int j = 0; j < k; ++j)
                for (int l = 0; l < k; ++l) A[j * k + l] += wq[q] * Pl[l] * Pj[j];
        }
        for (int j = 0; j < k; ++j)
            for (int l = 0; l < k; ++l) A[j * k + l] *= half * (2.0 * j + 1.0) / 2.0;
    }
    /* B: sub-interval [lo, hi] = [2a-1, 1] */
    {
        double lo = 2.0 * alpha - 1.0, hi = 1.0;
        double half = 0.5 * (hi - lo), mid = 0.5 * (hi + lo);
        for (int j = 0; j < k; ++j)
            for (int l = 0; l < k; ++l) B[j * k + l] = 0.0;
        for (int q = 0; q < k; ++q) {
            double xi = mid + half * xq[q];
            or_legendre_all(k - 1, xi, Pj);
            or_legendre_all(k - 1, xi - 2.0 * alpha, Pl);
            for (int j = 0; j < k; ++j)
                for (int l = 0; l < k; ++l) B[j * k + l] += wq[q] * Pl[l] * Pj[j];
        }
        for (int j = 0; j < k; ++j)
            for (int l = 0; l < k; ++l) B[j * k + l] *= half * (2.0 * j + 1.0) / 2.0;
    }

    /* Mass row (j = 0) in closed form, reading R3.  The j = 0 integrand is a
     * single Legendre polynomial, and int_x^1 P_l = -(P_{l+1}(x) - P_{l-1}(x)) / (2l+1)
     * (l >= 1) gives, with x = 1 - 2 alpha,
     *   A_0l = -(P_{l+1}(x) - P_{l-1}(x)) / (2 (2l+1)),   B_0l = -A_0l,
     *   A_00 + B_00 = 1 with A_00 ~ alpha, both exact in floating point.
     * "storing c_0 in double precision ... automatically ensures conservation of mass up to
     * double precision accuracy" and Table II's 4e-15 mass error after 1e4
     * steps need the rounded mass row to sum to delta_0l exactly; a quadrature-
     * rounded row is off by an ulp with a fixed sign and drifts coherently (2.7e-12 after
     * 1e4 steps at k = 2, alpha = 1/4). */
    {
        double x = 1.0 - 2.0 * alpha;
        double P[18];
        or_legendre_all(k, x, P);
        for (int l = 1; l < k; ++l) {
            double a0l = -(P[l + 1] - P[l - 1]) / (2.0 * (2.0 * l + 1.0));
            A[l] = a0l;
            B[l] = -a0l;
        }
        if (alpha <= 0.5) {
            B[0] = 1.0 - alpha;  /* rounded, in [0.5, 1] */
            A[0] = 1.0 - B[0];   /* exact (Sterbenz) */
        } else {
            A[0] = alpha;
            B[0] = 1.0 - alpha;  /* exact (Sterbenz) */
        }
    }
    return OR_OK;
}

/* Store through the precision layout: q < n_double stays fp64, q >= n_double becomes the  */
/* nearest fp32 (RNE, the C cast under the default rounding mode). */
static double or_store(double v, int64_t q, int64_t n_double)
{
    if (q < n_double) return v;
    return (double)(float)v;
}

/* Round a whole host coefficient array through the precision layout (used to turn      */
/* generated fp64 inputs into the values a mixed grid holds after set_coeffs).          */
int or_round_layout(int64_t n_cells, int64_t K, int64_t n_double, double* c)
{
    for (int64_t cell = 0; cell < n_cells; ++cell)
        for (int64_t q = 0; q < K; ++q) c[cell * K + q] = or_store(c[cell * K + q], q, n_double);
    return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* One SLDG sweep along dimension `dim` (P:259-272 SS II-A).       */
/*                                                                                       */
/*   for every line along dim (fixed perpendicular indices) with CFL nu of that line:    */
/*     (i*, alpha) = decompose(nu); A, B = matrices(alpha)                               */
/*     for every target cell i and every coupled group (m_e fixed for e != dim):         */
/*       c'_{i,j} = sum_l A_jl c_{(i - i* - 1) mod n, l} + sum_l B_jl c_{(i - i*) mod n, l} */
/*     (alpha == 0: c'_i = c_{(i - i*) mod n}, an exact copy)                             */
/*     store through the precision layout.                                               */
/*                                                                                       */
/* Direction convention: u^{n+1}(x) = u^n(x - nu h); positive nu moves mass   */
/* toward +x.  Periodic in every dimension.                                  */
/*                                                                                       */
/* field == NULL: every line uses nu = shift.  Otherwise field holds one nu per           */
/* combination of the dims set in field_mask (bit dim must be clear), indexed            */
/* sum over masked dims e (ascending) of i_e * prod(n of the lower masked dims); the      */
/* unmasked perpendicular dims broadcast.                              */
/* src and dst are host arrays in the layout above; src != dst.                          */
/* ------------------------------------------------------------------------------------ */
int or_advect(int D, const int64_t* n, int k, int64_t n_double, const double* src, double* dst,
              int dim, double shift, const double* field, uint32_t field_mask)
{
    if (D < 1 || D > 6 || k < 1 || k > 16 || dim < 0 || dim >= D) return OR_EINVAL;
    if (src == dst) return OR_EINVAL;
    if (field && (field_mask & (1u << dim))) return OR_EINVAL;
    if (field_mask >> D) return OR_EINVAL;

    int64_t S[6], kp[6];
    int64_t cells = 1, K = 1;
    for (int d = 0; d < D; ++d) {
        if (n[d] < 1) return OR_EINVAL;
        S[d] = cells;
        kp[d] = K;
        cells *= n[d];
        K *= k;
    }
    int64_t n_field = 1;
    if (field)
        for (int d = 0; d < D; ++d)
            if (field_mask & (1u << d)) n_field *= n[d];

    /* steps 1-3: decompose each line's nu and build its matrices once per field entry
       ("precomputed at the beginning of each time step") */
    int64_t* istar = (int64_t*)malloc(sizeof(int64_t) * n_field);
    double* alpha = (double*)malloc(sizeof(double) * n_field);
    double* AB = (double*)malloc(sizeof(double) * n_field * 2 * k * k);
    if (!istar || !alpha || !AB) { free(istar); free(alpha); free(AB); return OR_ENOMEM; }
    for (int64_t f = 0; f < n_field; ++f) {
        double nu = field ? field[f] : shift;
        if (or_shift_decompose(nu, &istar[f], &alpha[f]) != OR_OK) {
            free(istar); free(alpha); free(AB);
            return OR_EINVAL;
        }
        or_shift_matrices(alpha[f], k, &AB[f * 2 * k * k], &AB[f * 2 * k * k + k * k]);
    }

    const int64_t nd = n[dim];
    for (int64_t cell = 0; cell < cells; ++cell) {
        int64_t idx[6];
        for (int d = 0; d < D; ++d) idx[d] = (cell / S[d]) % n[d];

        int64_t f = 0;
        if (field) {
            int64_t stride = 1;
            for (int d = 0; d < D; ++d)
                if (field_mask & (1u << d)) { f += idx[d] * stride; stride *= n[d]; }
        }
        const double* A = &AB[f * 2 * k * k];
        const double* B = &AB[f * 2 * k * k + k * k];

        /* source cells along dim: (i - i* - 1) mod n (weighted by A), (i - i*) mod n (by B) */
        int64_t i = idx[dim];
        int64_t iB = ((i - istar[f]) % nd + nd) % nd;
        int64_t iA = ((i - istar[f] - 1) % nd + nd) % nd;
        int64_t cellA = cell + (iA - i) * S[dim];
        int64_t cellB = cell + (iB - i) * S[dim];

        /* every coupled group: slots q0 with m_dim = 0; members q0 + l * k^dim */
        for (int64_t q0 = 0; q0 < K; ++q0) {
            if ((q0 / kp[dim]) % k != 0) continue;
            for (int j = 0; j < k; ++j) {
                int64_t qj = q0 + (int64_t)j * kp[dim];
                double v;
                if (alpha[f] == 0.0) {
                    v = src[cellB * K + qj]; /* integer shift: exact permutation */
                } else {
                    v = 0.0;
                    for (int l = 0; l < k; ++l) v += A[j * k + l] * src[cellA * K + q0 + (int64_t)l * kp[dim]];
                    for (int l = 0; l < k; ++l) v += B[j * k + l] * src[cellB * K + q0 + (int64_t)l * kp[dim]];
                }
                dst[cell * K + qj] = or_store(v, qj, n_double);
            }
        }
    }
    free(istar);
    free(alpha);
    free(AB);
    return OR_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Mass M = (prod_d h_d) * sum_cells c_{cell, 0}  ("c_0 corresponds to the     */
/* mass", SS II-A), summed with Neumaier compensation (SURVEY 8(c)   */
/* step 6, C14).                                                                          */
/* ------------------------------------------------------------------------------------ */
double or_mass(int64_t n_cells, int64_t K, double cell_volume, const double* c)
{
    double s = 0.0, comp = 0.0;
    for (int64_t cell = 0; cell < n_cells; ++cell) {
        double x = c[cell * K];
        double t = s + x;
        if (fabs(s) >= fabs(x)) comp += (s - t) + x;
        else comp += (x - t) + s;
        s = t;
    }
    return cell_volume * (s + comp);
}
