/*
 * oracle/mmse_oracle.c -- plain, slow, fp64 CPU oracle of the per-RE MMSE
 * detector + max-log soft demapper (arxiv 2510.07843 hot path).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2510_07843_b200/) never imports, links or executes anything here, and
 * this file shares no code, header, table or constant generator with the CUDA
 * path (DESIGN.md §"Oracle").
 *
 * What it computes (§IV; Fig. 4 caption PAPER.md:93): LMMSE
 * detection of every resource element (RE) of an H-unit, i.e. one channel H
 * (n_rx x n_layers) shared by the unit's REs (one H per subcarrier per slot,
 * SPEC.md:440), followed by max-log soft demapping (BASELINE.json north_star;
 * the paper is silent on demapping -- readings R3..R6 in DESIGN.md).
 *
 * Every function follows a definition or the paper's algorithm step by step:
 *   - oracle_gram            G = H^H H + s2 I         (north_star; "covariance")
 *   - oracle_covariance      R = H H^H + s2 I         ("received signal covariance matrix R")
 *   - oracle_cholesky        G = L L^H, Banachiewicz  (north_star; reading R2)
 *   - oracle_lu_factor / _forward / _backward / _invert
 *                            LU with partial pivoting, forward & backward
 *                            substitution, inversion
 *   - oracle_weights_chol    W = G^-1 H^H             (Gram form, reading R1)
 *   - oracle_weights_lu      W = H^H R^-1             (paper-literal covariance form)
 *   - oracle_detect          per-unit detector, Gram/Cholesky route
 *   - oracle_detect_irc      coloured-noise (interference-rejection) detector, W = H^H (H H^H + R_nn)^-1
 *   - oracle_bfp_decode      block-floating-point fronthaul decompression (reading R25)
 *   - oracle_detect_cov_lu   per-unit detector, covariance/LU route (paper-literal)
 *   - oracle_constellation   38.211 5.1 Gray QAM (reading R6)
 *   - oracle_maxlog          brute-force max-log over all 2^qm points (reading R5)
 *   - oracle_quantize        fp32 / fp16 (RNE, sat 65504) / int8 (rint, sat 127) (reading R10)
 *
 * Complex numbers are C99 `double complex`; complex arrays cross the ABI as
 * interleaved (re, im) pairs, row-major. Nothing is blocked, fused or
 * reordered beyond the definitions above.
 */
#include <complex.h>
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

#define ORACLE_VERSION 1
/* Reading R17: a unit is "not positive definite" when a Cholesky pivot
 * p_j = G_jj - sum_k |L_jk|^2 fails p_j > TAU * max_i G_ii with
 * TAU = 16 * 2^-24 (16 x the fp32 unit roundoff of the product's working
 * precision; scale-invariant like SPEC.md:266's eps_pivot). The oracle uses the
 * same TAU so flagged sets agree away from the boundary. */
#define ORACLE_PIVOT_TAU (16.0 * 5.9604644775390625e-08)

/* Reading R10: quantiser codes. */
#define ORACLE_LLR_F32 0
#define ORACLE_LLR_F16 1
#define ORACLE_LLR_I8 2

int oracle_version(void) { return ORACLE_VERSION; }
double oracle_pivot_tau(void) { return ORACLE_PIVOT_TAU; }

/* ---------------------------------------------------------------- QAM ---- */

/* 38.211 5.1 (reading R6): qm bits b_0..b_{qm-1}; b_0,b_2,.. drive I and
 * b_1,b_3,.. drive Q. With m = qm/2 and axis bits c_0..c_{m-1}:
 *   a = (1-2c_0)[2^{m-1} - (1-2c_1)[2^{m-2} - ... [2 - (1-2c_{m-1})]]]
 * normalised by 1/sqrt(2), 1/sqrt(10), 1/sqrt(42), 1/sqrt(170).
 * Point index L carries b_j = bit (qm-1-j) of L (b_0 is the MSB). */
int oracle_constellation(int qm, double* re, double* im)
{
    double norm;
    switch (qm) {
    case 2: norm = 2.0; break;
    case 4: norm = 10.0; break;
    case 6: norm = 42.0; break;
    case 8: norm = 170.0; break;
    default: return 0;
    }
    int m = qm / 2;
    for (int L = 0; L < (1 << qm); L++) {
        int b[8];
        for (int j = 0; j < qm; j++) b[j] = (L >> (qm - 1 - j)) & 1;
        double ax[2];
        for (int off = 0; off < 2; off++) {
            /* innermost bracket first: v = (1 - 2c_{m-1}) */
            double v = 1.0 - 2.0 * b[2 * (m - 1) + off];
            for (int i = m - 2; i >= 0; i--)
                v = (1.0 - 2.0 * b[2 * i + off]) * ((double)(1 << (m - 1 - i)) - v);
            ax[off] = v;
        }
        re[L] = ax[0] / sqrt(norm);
        im[L] = ax[1] / sqrt(norm);
    }
    return 1 << qm;
}

/* Brute-force max-log (reading R5): for bit j, D_v = min over all points s
 * whose label has b_j = v of |x - s|^2, and LLR_j = SINR (D_1 - D_0), i.e.
 * ln P(b=0)/P(b=1) under x~ = x + e, e ~ CN(0, 1/SINR). SINR = +inf
 * (sigma^2 = 0, reading R11): LLR = 0 if D_1 == D_0, else +-inf. */
static void maxlog_with(int qm, const double* cre, const double* cim,
                        double xr, double xi, double sinr, double* llr)
{
    int M = 1 << qm;
    for (int j = 0; j < qm; j++) {
        double d0 = INFINITY, d1 = INFINITY;
        for (int L = 0; L < M; L++) {
            double dr = xr - cre[L], di = xi - cim[L];
            double d = dr * dr + di * di;
            if ((L >> (qm - 1 - j)) & 1) {
                if (d < d1) d1 = d;
            } else {
                if (d < d0) d0 = d;
            }
        }
        double diff = d1 - d0;
        if (isinf(sinr))
            llr[j] = (diff == 0.0) ? 0.0 : copysign(INFINITY, diff);
        else
            llr[j] = sinr * diff;
    }
}

void oracle_maxlog(int qm, int n, const double* x /* complex [n] */, const double* sinr /* [n] */,
                   double* llr /* [n][qm] */)
{
    double cre[256], cim[256];
    oracle_constellation(qm, cre, cim);
    for (int i = 0; i < n; i++) maxlog_with(qm, cre, cim, x[2 * i], x[2 * i + 1], sinr[i], llr + (size_t)i * qm);
}

/* ------------------------------------------------------- linear algebra -- */

/* G = H^H H + s2 I  (n_layers x n_layers, full Hermitian). */
void oracle_gram(int nr, int nl, const double* Hd, double s2, double* Gd)
{
    const cplx* H = (const cplx*)Hd;
    cplx* G = (cplx*)Gd;
    for (int i = 0; i < nl; i++)
        for (int j = 0; j < nl; j++) {
            cplx s = 0;
            for (int r = 0; r < nr; r++) s += conj(H[r * nl + i]) * H[r * nl + j];
            if (i == j) s += s2;
            G[i * nl + j] = s;
        }
}

/* R = H H^H + s2 I  (n_rx x n_rx), the paper's covariance. */
void oracle_covariance(int nr, int nl, const double* Hd, double s2, double* Rd)
{
    const cplx* H = (const cplx*)Hd;
    cplx* R = (cplx*)Rd;
    for (int i = 0; i < nr; i++)
        for (int j = 0; j < nr; j++) {
            cplx s = 0;
            for (int l = 0; l < nl; l++) s += H[i * nl + l] * conj(H[j * nl + l]);
            if (i == j) s += s2;
            R[i * nr + j] = s;
        }
}

/* Cholesky-Banachiewicz, row by row: L_ij = (G_ij - sum_{k<j} L_ik conj(L_jk)) / L_jj,
 * L_ii = sqrt(G_ii - sum_{k<i} |L_ik|^2). Returns 1, or 0 if a pivot fails
 * the guard of reading R17 (the `!(p > t)` form also catches NaN). */
int oracle_cholesky(int n, const double* Gd, double* Ld)
{
    const cplx* G = (const cplx*)Gd;
    cplx* L = (cplx*)Ld;
    double gmax = 0.0;
    for (int i = 0; i < n; i++)
        if (creal(G[i * n + i]) > gmax) gmax = creal(G[i * n + i]);
    memset(L, 0, sizeof(cplx) * (size_t)n * n);
    for (int i = 0; i < n; i++) {
        for (int j = 0; j <= i; j++) {
            cplx s = 0;
            for (int k = 0; k < j; k++) s += L[i * n + k] * conj(L[j * n + k]);
            if (i == j) {
                double p = creal(G[i * n + i] - s);
                if (!(p > ORACLE_PIVOT_TAU * gmax)) return 0;
                L[i * n + i] = sqrt(p);
            } else {
                L[i * n + j] = (G[i * n + j] - s) / L[j * n + j];
            }
        }
    }
    return 1;
}

/* Forward substitution L w = z (L lower, non-unit diagonal). */
static void chol_forward(int n, const cplx* L, const cplx* z, cplx* w)
{
    for (int i = 0; i < n; i++) {
        cplx s = z[i];
        for (int k = 0; k < i; k++) s -= L[i * n + k] * w[k];
        w[i] = s / L[i * n + i];
    }
}

/* Backward substitution L^H x = w. */
static void chol_backward(int n, const cplx* L, const cplx* w, cplx* x)
{
    for (int i = n - 1; i >= 0; i--) {
        cplx s = w[i];
        for (int k = i + 1; k < n; k++) s -= conj(L[k * n + i]) * x[k];
        x[i] = s / conj(L[i * n + i]);
    }
}

/* LU with partial pivoting (largest |pivot| per column), PAPER.md:93, :115;
 * SPEC.md:211-216. LU holds L (unit diagonal, strictly lower) and U.
 * perm[i] = original row placed at row i. Returns 0 on a pivot below
 * 16 u_64 max|a_ij|. */
int oracle_lu_factor(int n, const double* Ad, double* LUd, int* perm)
{
    cplx* A = (cplx*)LUd;
    memcpy(A, Ad, sizeof(cplx) * (size_t)n * n);
    double amax = 0.0;
    for (int i = 0; i < n * n; i++)
        if (cabs(A[i]) > amax) amax = cabs(A[i]);
    for (int i = 0; i < n; i++) perm[i] = i;
    for (int k = 0; k < n; k++) {
        int p = k;
        for (int i = k + 1; i < n; i++)
            if (cabs(A[i * n + k]) > cabs(A[p * n + k])) p = i;
        if (!(cabs(A[p * n + k]) > 16.0 * DBL_EPSILON / 2.0 * amax)) return 0;
        if (p != k) {
            for (int j = 0; j < n; j++) {
                cplx t = A[k * n + j];
                A[k * n + j] = A[p * n + j];
                A[p * n + j] = t;
            }
            int t = perm[k];
            perm[k] = perm[p];
            perm[p] = t;
        }
        for (int i = k + 1; i < n; i++) {
            A[i * n + k] /= A[k * n + k];
            for (int j = k + 1; j < n; j++) A[i * n + j] -= A[i * n + k] * A[k * n + j];
        }
    }
    return 1;
}

/* Forward substitution L z = P b (unit lower L). */
void oracle_lu_forward(int n, const double* LUd, const int* perm, const double* bd, double* zd)
{
    const cplx* A = (const cplx*)LUd;
    const cplx* b = (const cplx*)bd;
    cplx* z = (cplx*)zd;
    for (int i = 0; i < n; i++) {
        cplx s = b[perm[i]];
        for (int k = 0; k < i; k++) s -= A[i * n + k] * z[k];
        z[i] = s;
    }
}

/* Backward substitution U x = z. */
void oracle_lu_backward(int n, const double* LUd, const double* zd, double* xd)
{
    const cplx* A = (const cplx*)LUd;
    const cplx* z = (const cplx*)zd;
    cplx* x = (cplx*)xd;
    for (int i = n - 1; i >= 0; i--) {
        cplx s = z[i];
        for (int k = i + 1; k < n; k++) s -= A[i * n + k] * x[k];
        x[i] = s / A[i * n + i];
    }
}

/* Inversion: one LU, then one forward + backward substitution per unit
 * vector ("LU decomposition, forward/backward substitution, and
 * matrix inversion"). X row-major, X[:, c] = A^-1 e_c. */
int oracle_lu_invert(int n, const double* Ad, double* Xd)
{
    cplx* LU = malloc(sizeof(cplx) * (size_t)n * n);
    int* perm = malloc(sizeof(int) * (size_t)n);
    cplx* e = malloc(sizeof(cplx) * (size_t)n * 3);
    cplx* X = (cplx*)Xd;
    int ok = oracle_lu_factor(n, Ad, (double*)LU, perm);
    if (ok) {
        for (int c = 0; c < n; c++) {
            cplx* z = e + n;
            cplx* x = e + 2 * n;
            for (int i = 0; i < n; i++) e[i] = (i == c) ? 1.0 : 0.0;
            oracle_lu_forward(n, (const double*)LU, perm, (const double*)e, (double*)z);
            oracle_lu_backward(n, (const double*)LU, (const double*)z, (double*)x);
            for (int i = 0; i < n; i++) X[i * n + c] = x[i];
        }
    }
    free(LU);
    free(perm);
    free(e);
    return ok;
}

/* W = G^-1 H^H (n_layers x n_rx) through Cholesky: column r of W solves
 * G w = conj(H[r, :])^T by forward + backward substitution. */
int oracle_weights_chol(int nr, int nl, const double* Hd, double s2, double* Wd)
{
    const cplx* H = (const cplx*)Hd;
    cplx* W = (cplx*)Wd;
    cplx* G = malloc(sizeof(cplx) * (size_t)nl * nl);
    cplx* L = malloc(sizeof(cplx) * (size_t)nl * nl);
    cplx* v = malloc(sizeof(cplx) * (size_t)nl * 3);
    oracle_gram(nr, nl, Hd, s2, (double*)G);
    int ok = oracle_cholesky(nl, (const double*)G, (double*)L);
    if (ok) {
        for (int r = 0; r < nr; r++) {
            for (int l = 0; l < nl; l++) v[l] = conj(H[r * nl + l]);
            chol_forward(nl, L, v, v + nl);
            chol_backward(nl, L, v + nl, v + 2 * nl);
            for (int l = 0; l < nl; l++) W[l * nr + r] = v[2 * nl + l];
        }
    }
    free(G);
    free(L);
    free(v);
    return ok;
}

/* W = H^H R^-1 (n_layers x n_rx), R = H H^H + s2 I inverted by LU +
 * substitution (the paper's literal pipeline). */
int oracle_weights_lu(int nr, int nl, const double* Hd, double s2, double* Wd)
{
    const cplx* H = (const cplx*)Hd;
    cplx* W = (cplx*)Wd;
    cplx* R = malloc(sizeof(cplx) * (size_t)nr * nr);
    cplx* Ri = malloc(sizeof(cplx) * (size_t)nr * nr);
    oracle_covariance(nr, nl, Hd, s2, (double*)R);
    int ok = oracle_lu_invert(nr, (const double*)R, (double*)Ri);
    if (ok) {
        for (int l = 0; l < nl; l++)
            for (int c = 0; c < nr; c++) {
                cplx s = 0;
                for (int r = 0; r < nr; r++) s += conj(H[r * nl + l]) * Ri[r * nr + c];
                W[l * nr + c] = s;
            }
    }
    free(R);
    free(Ri);
    return ok;
}

/* ------------------------------------------------------------ detector -- */

/* SINR and unbiasing (readings R3, R4, R11): mu_k = 1 - s2 A_kk with
 * A_kk = [G^-1]_kk, SINR_k = 1/(s2 A_kk) - 1; s2 == 0 gives mu = 1 and
 * SINR = +inf. A layer with !(mu_k > 0) carries no information: it is erased
 * (SINR 0, x~ 0, LLR 0). */
static void sinr_mu(double s2, double akk, double* sinr, double* mu)
{
    if (s2 == 0.0) {
        *mu = 1.0;
        *sinr = INFINITY;
        return;
    }
    *mu = 1.0 - s2 * akk;
    *sinr = 1.0 / (s2 * akk) - 1.0;
}

/* Detect one H-unit, Gram/Cholesky route:
 *  1 G = H^H H + s2 I;  2 G = L L^H (guard R17);  3 z = H^H y;
 *  4 L w = z, L^H xhat = w (PAPER.md:115 forward/backward substitution);
 *  5 A_kk from G a = e_k, mu_k, SINR_k;  6 x~_k = xhat_k / mu_k;
 *  7 brute-force max-log over all constellation points.
 * Hf, Yf: complex64 inputs widened to fp64 here. Returns 1, or 0 if flagged
 * (outputs zeroed). */
static int detect_unit_chol(int nr, int nl, int qm, int n_re, const float* Hf, const float* Yf,
                            double s2, const double* cre, const double* cim,
                            cplx* xt, double* sinr, double* llr)
{
    int ok = 1;
    cplx* H = malloc(sizeof(cplx) * (size_t)nr * nl);
    cplx* G = malloc(sizeof(cplx) * (size_t)nl * nl);
    cplx* L = malloc(sizeof(cplx) * (size_t)nl * nl);
    cplx* v = malloc(sizeof(cplx) * (size_t)(nl * 3 + nr));
    double* mu = malloc(sizeof(double) * (size_t)nl);
    for (int i = 0; i < nr * nl; i++) H[i] = (double)Hf[2 * i] + I * (double)Hf[2 * i + 1];

    oracle_gram(nr, nl, (const double*)H, s2, (double*)G);
    if (!oracle_cholesky(nl, (const double*)G, (double*)L)) {
        ok = 0;
        memset(xt, 0, sizeof(cplx) * (size_t)n_re * nl);
        memset(sinr, 0, sizeof(double) * (size_t)nl);
        memset(llr, 0, sizeof(double) * (size_t)n_re * nl * qm);
        goto done;
    }
    /* step 5: A_kk = e_k^T G^-1 e_k via the two substitutions */
    for (int k = 0; k < nl; k++) {
        for (int l = 0; l < nl; l++) v[l] = (l == k) ? 1.0 : 0.0;
        chol_forward(nl, L, v, v + nl);
        chol_backward(nl, L, v + nl, v + 2 * nl);
        sinr_mu(s2, creal(v[2 * nl + k]), &sinr[k], &mu[k]);
        if (!(mu[k] > 0.0)) sinr[k] = 0.0;
    }
    for (int e = 0; e < n_re; e++) {
        cplx* y = v + 3 * nl;
        for (int r = 0; r < nr; r++)
            y[r] = (double)Yf[((size_t)e * nr + r) * 2] + I * (double)Yf[((size_t)e * nr + r) * 2 + 1];
        /* step 3: z = H^H y */
        for (int l = 0; l < nl; l++) {
            cplx s = 0;
            for (int r = 0; r < nr; r++) s += conj(H[r * nl + l]) * y[r];
            v[l] = s;
        }
        /* step 4 */
        chol_forward(nl, L, v, v + nl);
        chol_backward(nl, L, v + nl, v + 2 * nl);
        for (int k = 0; k < nl; k++) {
            cplx* out = xt + (size_t)e * nl + k;
            double* lo = llr + ((size_t)e * nl + k) * qm;
            if (!(mu[k] > 0.0)) {
                *out = 0;
                for (int j = 0; j < qm; j++) lo[j] = 0.0;
                continue;
            }
            *out = v[2 * nl + k] / mu[k]; /* step 6 */
            maxlog_with(qm, cre, cim, creal(*out), cimag(*out), sinr[k], lo); /* step 7 */
        }
    }
done:
    free(H);
    free(G);
    free(L);
    free(v);
    free(mu);
    return ok;
}

/* Detect one H-unit, paper-literal route: R = H H^H + s2 I, LU + substitution
 * inversion, W = H^H R^-1, xhat = W y;
 * mu_k = [W H]_kk (unbiasing identity, pin P7), SINR_k = mu_k / (1 - mu_k). */
static int detect_unit_cov_lu(int nr, int nl, int qm, int n_re, const float* Hf, const float* Yf,
                              double s2, const double* cre, const double* cim,
                              cplx* xt, double* sinr, double* llr)
{
    cplx* H = malloc(sizeof(cplx) * (size_t)nr * nl);
    cplx* W = malloc(sizeof(cplx) * (size_t)nl * nr);
    double* mu = malloc(sizeof(double) * (size_t)nl);
    for (int i = 0; i < nr * nl; i++) H[i] = (double)Hf[2 * i] + I * (double)Hf[2 * i + 1];
    int ok = oracle_weights_lu(nr, nl, (const double*)H, s2, (double*)W);
    if (!ok) {
        memset(xt, 0, sizeof(cplx) * (size_t)n_re * nl);
        memset(sinr, 0, sizeof(double) * (size_t)nl);
        memset(llr, 0, sizeof(double) * (size_t)n_re * nl * qm);
        goto done;
    }
    for (int k = 0; k < nl; k++) {
        cplx s = 0;
        for (int r = 0; r < nr; r++) s += W[k * nr + r] * H[r * nl + k];
        mu[k] = creal(s);
        if (s2 == 0.0) {
            mu[k] = 1.0;
            sinr[k] = INFINITY;
        } else {
            sinr[k] = mu[k] / (1.0 - mu[k]);
        }
        if (!(mu[k] > 0.0)) sinr[k] = 0.0;
    }
    for (int e = 0; e < n_re; e++) {
        for (int k = 0; k < nl; k++) {
            cplx* out = xt + (size_t)e * nl + k;
            double* lo = llr + ((size_t)e * nl + k) * qm;
            if (!(mu[k] > 0.0)) {
                *out = 0;
                for (int j = 0; j < qm; j++) lo[j] = 0.0;
                continue;
            }
            cplx s = 0;
            for (int r = 0; r < nr; r++)
                s += W[k * nr + r] * ((double)Yf[((size_t)e * nr + r) * 2] + I * (double)Yf[((size_t)e * nr + r) * 2 + 1]);
            *out = s / mu[k];
            maxlog_with(qm, cre, cim, creal(*out), cimag(*out), sinr[k], lo);
        }
    }
done:
    free(H);
    free(W);
    free(mu);
    return ok;
}

/* Detect one H-unit with a coloured-noise covariance R_nn (SURVEY.md §8(f)
 * NEXT-3, interference-rejection combining; reading R24). The LMMSE filter for
 * y = H x + n, n ~ CN(0, R_nn), E[x x^H] = I, written out as its definition:
 *   W = H^H (H H^H + R_nn)^-1           (R_nn = s2 I gives the paper's R)
 * with the inverse formed by the LU + substitution inversion above; then, as in
 * the white case, mu_k = [W H]_kk, SINR_k = mu_k / (1 - mu_k), x~ = (W y)_k / mu_k,
 * brute-force max-log. Rf: complex64 [nr][nr] (full Hermitian matrix). */
static int detect_unit_irc(int nr, int nl, int qm, int n_re, const float* Hf, const float* Yf, const float* Rf,
                           const double* cre, const double* cim, cplx* xt, double* sinr, double* llr)
{
    cplx* H = malloc(sizeof(cplx) * (size_t)nr * nl);
    cplx* Rt = malloc(sizeof(cplx) * (size_t)nr * nr);
    cplx* Ri = malloc(sizeof(cplx) * (size_t)nr * nr);
    cplx* W = malloc(sizeof(cplx) * (size_t)nl * nr);
    double* mu = malloc(sizeof(double) * (size_t)nl);
    for (int i = 0; i < nr * nl; i++) H[i] = (double)Hf[2 * i] + I * (double)Hf[2 * i + 1];
    /* R_total = H H^H + R_nn */
    for (int i = 0; i < nr; i++)
        for (int j = 0; j < nr; j++) {
            cplx s = (double)Rf[2 * (i * nr + j)] + I * (double)Rf[2 * (i * nr + j) + 1];
            for (int l = 0; l < nl; l++) s += H[i * nl + l] * conj(H[j * nl + l]);
            Rt[i * nr + j] = s;
        }
    int ok = oracle_lu_invert(nr, (const double*)Rt, (double*)Ri);
    if (!ok) {
        memset(xt, 0, sizeof(cplx) * (size_t)n_re * nl);
        memset(sinr, 0, sizeof(double) * (size_t)nl);
        memset(llr, 0, sizeof(double) * (size_t)n_re * nl * qm);
        goto done;
    }
    for (int l = 0; l < nl; l++)
        for (int c = 0; c < nr; c++) {
            cplx s = 0;
            for (int r = 0; r < nr; r++) s += conj(H[r * nl + l]) * Ri[r * nr + c];
            W[l * nr + c] = s;
        }
    for (int k = 0; k < nl; k++) {
        cplx s = 0;
        for (int r = 0; r < nr; r++) s += W[k * nr + r] * H[r * nl + k];
        mu[k] = creal(s);
        sinr[k] = mu[k] / (1.0 - mu[k]);
        if (!(mu[k] > 0.0)) sinr[k] = 0.0;
    }
    for (int e = 0; e < n_re; e++) {
        for (int k = 0; k < nl; k++) {
            cplx* out = xt + (size_t)e * nl + k;
            double* lo = llr + ((size_t)e * nl + k) * qm;
            if (!(mu[k] > 0.0)) {
                *out = 0;
                for (int j = 0; j < qm; j++) lo[j] = 0.0;
                continue;
            }
            cplx s = 0;
            for (int r = 0; r < nr; r++)
                s += W[k * nr + r] * ((double)Yf[((size_t)e * nr + r) * 2] + I * (double)Yf[((size_t)e * nr + r) * 2 + 1]);
            *out = s / mu[k];
            maxlog_with(qm, cre, cim, creal(*out), cimag(*out), sinr[k], lo);
        }
    }
done:
    free(H);
    free(Rt);
    free(Ri);
    free(W);
    free(mu);
    return ok;
}

/* Batch driver of the coloured-noise route: R complex64 [n_units][nr][nr]. */
long oracle_detect_irc(int nr, int nl, int qm, long n_units, int n_re, const float* H, const float* Y,
                       const float* R, double* xt, double* sinr, double* llr, signed char* ok, int n_threads)
{
    double cre[256], cim[256];
    if (oracle_constellation(qm, cre, cim) == 0) return -1;
    long n_bad = 0;
    if (n_threads < 1) n_threads = 1;
#pragma omp parallel for schedule(dynamic, 4) num_threads(n_threads) reduction(+ : n_bad)
    for (long u = 0; u < n_units; u++) {
        int r = detect_unit_irc(nr, nl, qm, n_re, H + (size_t)u * nr * nl * 2, Y + (size_t)u * n_re * nr * 2,
                                R + (size_t)u * nr * nr * 2, cre, cim, (cplx*)xt + (size_t)u * n_re * nl,
                                sinr + (size_t)u * nl, llr + (size_t)u * n_re * nl * qm);
        ok[u] = (signed char)r;
        if (!r) n_bad++;
    }
    return n_bad;
}

/* Batch driver over H-units (units are independent: SPEC.md:470-471).
 *   H    complex64 [n_units][nr][nl]
 *   Y    complex64 [n_units][n_re][nr]       (REs of each unit, unit order)
 *   xt   complex128 [n_units][n_re][nl]      unbiased x~
 *   sinr double [n_units][nl]
 *   llr  double [n_units][n_re][nl][qm]      natural-log units, before scaling
 *   ok   int8 [n_units]                      1 = detected, 0 = flagged (R17)
 * route 0 = Gram/Cholesky, 1 = covariance/LU. Returns the number of flagged
 * units. n_threads <= 0 means 1 thread. */
long oracle_detect(int route, int nr, int nl, int qm, long n_units, int n_re,
                   const float* H, const float* Y, float sigma2,
                   double* xt, double* sinr, double* llr, signed char* ok, int n_threads)
{
    double cre[256], cim[256];
    if (oracle_constellation(qm, cre, cim) == 0) return -1;
    long n_bad = 0;
    if (n_threads < 1) n_threads = 1;
#pragma omp parallel for schedule(dynamic, 4) num_threads(n_threads) reduction(+ : n_bad)
    for (long u = 0; u < n_units; u++) {
        const float* Hu = H + (size_t)u * nr * nl * 2;
        const float* Yu = Y + (size_t)u * n_re * nr * 2;
        cplx* xu = (cplx*)xt + (size_t)u * n_re * nl;
        double* su = sinr + (size_t)u * nl;
        double* lu = llr + (size_t)u * n_re * nl * qm;
        int r = route == 1 ? detect_unit_cov_lu(nr, nl, qm, n_re, Hu, Yu, (double)sigma2, cre, cim, xu, su, lu)
                           : detect_unit_chol(nr, nl, qm, n_re, Hu, Yu, (double)sigma2, cre, cim, xu, su, lu);
        ok[u] = (signed char)r;
        if (!r) n_bad++;
    }
    return n_bad;
}

/* ------------------------------------------------------- BFP fronthaul -- */

/* Block-floating-point decompression (the O-RAN format
 * is not in the container, reading R25 fixes it): one block = one PRB (12
 * subcarriers) of one antenna in one OFDM symbol, block_bytes = roundup4(1 + 3 W):
 *   byte 0        exponent e in bits 0..3
 *   bytes 1..     24 two's-complement W-bit mantissas m_j, j = 2 f + {0: I, 1: Q},
 *                 packed MSB-first (stream bit 0 = bit 7 of byte 1)
 *   value_j = m_j * 2^e * scale.
 * Decoded bit by bit, in fp64, rounded once to fp32: out complex64 [n_blocks][12]. */
void oracle_bfp_decode(long n_blocks, int W, double scale, const unsigned char* blocks, float* out)
{
    const int bb = ((1 + 3 * W) + 3) & ~3;
    for (long b = 0; b < n_blocks; b++) {
        const unsigned char* blk = blocks + (size_t)b * bb;
        const int e = blk[0] & 0xF;
        for (int j = 0; j < 24; j++) {
            long m = 0;
            for (int t = 0; t < W; t++) {
                const int bit = j * W + t; /* stream bit index, MSB-first */
                const int v = (blk[1 + bit / 8] >> (7 - bit % 8)) & 1;
                m = (m << 1) | v;
            }
            if (m >= (1L << (W - 1))) m -= (1L << W); /* two's complement */
            out[(size_t)b * 24 + j] = (float)((double)m * ldexp(1.0, e) * scale);
        }
    }
}

/* ----------------------------------------------------------- quantisers -- */

/* Scale and quantise (reading R10):
 *   F32: round to nearest fp32, saturate at +-FLT_MAX;
 *   F16: saturate at +-65504, round-to-nearest-even to IEEE binary16;
 *   I8 : saturate at +-127, rint (round half to even).
 * out: float32 / uint16 (binary16 bits) / int8 arrays. */
void oracle_quantize(int type, long n, const double* llr, double scale, void* out)
{
    for (long i = 0; i < n; i++) {
        double v = llr[i] * scale;
        if (isnan(v)) v = 0.0;
        if (type == ORACLE_LLR_F32) {
            if (v > FLT_MAX) v = FLT_MAX;
            if (v < -FLT_MAX) v = -FLT_MAX;
            ((float*)out)[i] = (float)v;
        } else if (type == ORACLE_LLR_F16) {
            if (v > 65504.0) v = 65504.0;
            if (v < -65504.0) v = -65504.0;
            _Float16 h = (_Float16)v;
            memcpy((uint16_t*)out + i, &h, 2);
        } else {
            if (v > 127.0) v = 127.0;
            if (v < -127.0) v = -127.0;
            ((int8_t*)out)[i] = (int8_t)rint(v);
        }
    }
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
