/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the LogosQ dense
 * state-vector hot path (arXiv 2512.23183, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg / `--impl reference` arm may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2512_23183_b200/); the only shared module is workloads/ (seeded
 * input generators, no arithmetic of the method).
 *
 * Precision: complex128 (C99 `double complex`), as the paper's Complex64
 * (= two f64).  Single-threaded, no SIMD intrinsics, no
 * blocking or fusion: every gate is one full sweep over the 2^n amplitudes,
 * in the order the circuit lists it (Circuit::execute).
 *
 * Conventions
 *   qubit q <-> index bit n-1-q (MSB first; Alg. 1 line "c_bit <- n-1-c",
 *   PAPER.md:579; App. B).
 *   2q matrices act on the sub-index 2*bit(q0) + bit(q1): q0 is the high bit
 *   (reading A2); CNOT/CP/CRY list the control first.
 *   Rotations R_G(theta) = exp(-i theta G / 2) (reading A3).
 *
 * Parity status of each function is recorded in DESIGN.md ("Oracle pins").
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

/* Oracle-private gate codes (the Python wrapper maps gate names to these). */
enum {
    OR_H = 0, OR_X, OR_Y, OR_Z, OR_S, OR_SDG, OR_T, OR_TDG,
    OR_RX, OR_RY, OR_RZ,
    OR_CNOT, OR_CZ, OR_CP, OR_SWAP, OR_U1, OR_U2, OR_CRY,
    OR_CCX, OR_RXX, OR_RYY, OR_RZZ,
    OR_NKINDS
};

#define OR_OK 0
#define OR_EARG (-1)
#define OR_EIMAG (-2)
#define OR_ENOMEM (-3)

static const double OR_PI = 3.14159265358979323846264338327950288;

/* ------------------------------------------------------------------ */
/* Compensated (Neumaier) summation -- SURVEY.md §8(c) c.3.           */
/* ------------------------------------------------------------------ */
typedef struct { double s, c; } neumaier;

static void neu_add(neumaier *acc, double x)
{
    double t = acc->s + x;
    if (fabs(acc->s) >= fabs(x))
        acc->c += (acc->s - t) + x;
    else
        acc->c += (x - t) + acc->s;
    acc->s = t;
}

static double neu_value(const neumaier *acc) { return acc->s + acc->c; }

/* ------------------------------------------------------------------ */
/* Basis / random states  */
/* ------------------------------------------------------------------ */
void or_init_basis(cplx *psi, int n, uint64_t k)
{
    uint64_t N = (uint64_t)1 << n;
    for (uint64_t i = 0; i < N; i++)
        psi[i] = 0.0;
    psi[k] = 1.0;
}

uint64_t or_splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* The unnormalised amplitude of index i:
 * a_i = r (cos 2 pi u1 + i sin 2 pi u1), r = sqrt(-2 ln u0) (Box-Muller),
 * u_j = ((x_j >> 11) + 0.5) 2^-53, x0 = splitmix64(seed ^ 2i),
 * x1 = splitmix64(seed ^ (2i+1)). */
/* u = ((x >> 11) + 0.5) 2^-53: the midpoint of one of 2^53 equal cells of
 * (0, 1), never 0 (log u0 stays finite) and never 1. */
double or_u53(uint64_t x)
{
    return ((double)(x >> 11) + 0.5) * 0x1.0p-53;
}

static void gauss_at(uint64_t seed, uint64_t i, double *re, double *im)
{
    uint64_t x0 = or_splitmix64(seed ^ (2 * i));
    uint64_t x1 = or_splitmix64(seed ^ (2 * i + 1));
    double u0 = or_u53(x0);
    double u1 = or_u53(x1);
    double r = sqrt(-2.0 * log(u0));
    *re = r * cos(2.0 * OR_PI * u1);
    *im = r * sin(2.0 * OR_PI * u1);
}

/* init_random: a_i as above for every i, then a /= sqrt(sum |a|^2)
 * (Neumaier sum). */
void or_init_random(cplx *psi, int n, uint64_t seed)
{
    uint64_t N = (uint64_t)1 << n;
    neumaier norm = {0.0, 0.0};
    for (uint64_t i = 0; i < N; i++) {
        double re, im;
        gauss_at(seed, i, &re, &im);
        psi[i] = re + I * im;
        neu_add(&norm, re * re);
        neu_add(&norm, im * im);
    }
    double s = 1.0 / sqrt(neu_value(&norm));
    for (uint64_t i = 0; i < N; i++)
        psi[i] *= s;
}

/* The unnormalised a_i at `count` indices (for states too large for the
 * host: the normalised state is a_i / sqrt(S) with one constant S). */
void or_random_gaussian_at(uint64_t seed, const uint64_t *idx, uint64_t count, cplx *out)
{
    for (uint64_t k = 0; k < count; k++) {
        double re, im;
        gauss_at(seed, idx[k], &re, &im);
        out[k] = re + I * im;
    }
}

/* ------------------------------------------------------------------ */
/* Gate matrices: textbook definitions (reading A4) and the rotation   */
/* generators of PAPER.md:373,380.                                      */
/* ------------------------------------------------------------------ */
static void mat1(int kind, double theta, cplx U[2][2])
{
    double c = cos(theta / 2.0), s = sin(theta / 2.0);
    const double r2 = 1.0 / sqrt(2.0);
    switch (kind) {
    case OR_H:   U[0][0] = r2; U[0][1] = r2; U[1][0] = r2; U[1][1] = -r2; break;
    case OR_X:   U[0][0] = 0; U[0][1] = 1; U[1][0] = 1; U[1][1] = 0; break;
    case OR_Y:   U[0][0] = 0; U[0][1] = -I; U[1][0] = I; U[1][1] = 0; break;
    case OR_Z:   U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = -1; break;
    case OR_S:   U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = I; break;
    case OR_SDG: U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = -I; break;
    case OR_T:   U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = cexp(I * OR_PI / 4.0); break;
    case OR_TDG: U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = cexp(-I * OR_PI / 4.0); break;
    /* R_G(theta) = cos(theta/2) I - i sin(theta/2) G */
    case OR_RX:  U[0][0] = c; U[0][1] = -I * s; U[1][0] = -I * s; U[1][1] = c; break;
    case OR_RY:  U[0][0] = c; U[0][1] = -s; U[1][0] = s; U[1][1] = c; break;
    case OR_RZ:  U[0][0] = c - I * s; U[0][1] = 0; U[1][0] = 0; U[1][1] = c + I * s; break;
    default:     U[0][0] = 1; U[0][1] = 0; U[1][0] = 0; U[1][1] = 1; break;
    }
}

/* 1q apply: for i with bit b clear, j = i | 2^b:
 * (a_i, a_j) <- (U00 a_i + U01 a_j, U10 a_i + U11 a_j). */
static void apply_1q(cplx *psi, int n, int q, cplx U[2][2])
{
    uint64_t N = (uint64_t)1 << n;
    uint64_t m = (uint64_t)1 << (n - 1 - q);
    for (uint64_t i = 0; i < N; i++) {
        if (i & m)
            continue;
        uint64_t j = i | m;
        cplx a = psi[i], b = psi[j];
        psi[i] = U[0][0] * a + U[0][1] * b;
        psi[j] = U[1][0] * a + U[1][1] * b;
    }
}

/* 2q apply: quads with sub-index k = 2*bit(qa) + bit(qb). */
static void apply_2q(cplx *psi, int n, int qa, int qb, cplx U[4][4])
{
    uint64_t N = (uint64_t)1 << n;
    uint64_t ma = (uint64_t)1 << (n - 1 - qa);
    uint64_t mb = (uint64_t)1 << (n - 1 - qb);
    for (uint64_t i = 0; i < N; i++) {
        if ((i & ma) || (i & mb))
            continue;
        uint64_t idx[4] = { i, i | mb, i | ma, i | ma | mb };
        cplx v[4], w[4];
        for (int k = 0; k < 4; k++)
            v[k] = psi[idx[k]];
        for (int r = 0; r < 4; r++) {
            w[r] = 0;
            for (int k = 0; k < 4; k++)
                w[r] += U[r][k] * v[k];
        }
        for (int k = 0; k < 4; k++)
            psi[idx[k]] = w[k];
    }
}

/* Alg. 1 "Direct State Vector CNOT", literally. */
static void apply_cnot(cplx *psi, int n, int c, int t)
{
    uint64_t N = (uint64_t)1 << n;
    int c_bit = n - 1 - c;
    int t_bit = n - 1 - t;
    uint64_t c_mask = (uint64_t)1 << c_bit;
    uint64_t t_mask = (uint64_t)1 << t_bit;
    for (uint64_t i = 0; i < N; i++) {
        if ((i & c_mask) != 0 && (i & t_mask) == 0) {
            uint64_t j = i ^ t_mask;
            cplx tmp = psi[i];
            psi[i] = psi[j];
            psi[j] = tmp;
        }
    }
}

/* App. B "Direct State Vector Toffoli", literally. */
static void apply_ccx(cplx *psi, int n, int c1, int c2, int t)
{
    uint64_t N = (uint64_t)1 << n;
    uint64_t c1_mask = (uint64_t)1 << (n - 1 - c1);
    uint64_t c2_mask = (uint64_t)1 << (n - 1 - c2);
    uint64_t t_mask = (uint64_t)1 << (n - 1 - t);
    uint64_t both = c1_mask | c2_mask;
    for (uint64_t i = 0; i < N; i++) {
        if ((i & both) == both && (i & t_mask) == 0) {
            uint64_t j = i ^ t_mask;
            cplx tmp = psi[i];
            psi[i] = psi[j];
            psi[j] = tmp;
        }
    }
}

/* Controlled phase: multiply by e^{i phi} where both bits are set
 * ("phase rotations based on bitwise masks"). */
static void apply_cphase(cplx *psi, int n, int a, int b, cplx phase)
{
    uint64_t N = (uint64_t)1 << n;
    uint64_t ma = (uint64_t)1 << (n - 1 - a);
    uint64_t mb = (uint64_t)1 << (n - 1 - b);
    for (uint64_t i = 0; i < N; i++)
        if ((i & ma) && (i & mb))
            psi[i] *= phase;
}

static void apply_swap(cplx *psi, int n, int a, int b)
{
    uint64_t N = (uint64_t)1 << n;
    uint64_t ma = (uint64_t)1 << (n - 1 - a);
    uint64_t mb = (uint64_t)1 << (n - 1 - b);
    for (uint64_t i = 0; i < N; i++) {
        if ((i & ma) && !(i & mb)) {
            uint64_t j = (i ^ ma) | mb;
            cplx tmp = psi[i];
            psi[i] = psi[j];
            psi[j] = tmp;
        }
    }
}

/* CRY(theta): RY(theta) on target q1 when control q0 is |1>. */
static void apply_cry(cplx *psi, int n, int c, int t, double theta)
{
    cplx U[2][2];
    mat1(OR_RY, theta, U);
    uint64_t N = (uint64_t)1 << n;
    uint64_t cm = (uint64_t)1 << (n - 1 - c);
    uint64_t tm = (uint64_t)1 << (n - 1 - t);
    for (uint64_t i = 0; i < N; i++) {
        if (!(i & cm) || (i & tm))
            continue;
        uint64_t j = i | tm;
        cplx a = psi[i], b = psi[j];
        psi[i] = U[0][0] * a + U[0][1] * b;
        psi[j] = U[1][0] * a + U[1][1] * b;
    }
}

/* R_PP(theta) = exp(-i theta P(x)P / 2) = cos(theta/2) I - i sin(theta/2) P(x)P
 * (SPEC.md:114), built as a plain Kronecker product. */
static void apply_rpp(cplx *psi, int n, int a, int b, int kind, double theta)
{
    cplx P[2][2], K[4][4], U[4][4];
    mat1(kind == OR_RXX ? OR_X : kind == OR_RYY ? OR_Y : OR_Z, 0.0, P);
    for (int r = 0; r < 4; r++)
        for (int k = 0; k < 4; k++)
            K[r][k] = P[r >> 1][k >> 1] * P[r & 1][k & 1];
    double c = cos(theta / 2.0), s = sin(theta / 2.0);
    for (int r = 0; r < 4; r++)
        for (int k = 0; k < 4; k++)
            U[r][k] = (r == k ? c : 0.0) - I * s * K[r][k];
    apply_2q(psi, n, a, b, U);
}

static int valid_qubit(int n, int q) { return q >= 0 && q < n; }

/* One gate.  mat: LQ-style row-major (re, im) pairs, 8 doubles for U1,
 * 32 for U2.  Returns OR_OK or OR_EARG. */
int or_apply_gate(cplx *psi, int n, int kind, int q0, int q1, int q2,
                  double angle, const double *mat)
{
    cplx U[2][2], U4[4][4];
    if (kind < 0 || kind >= OR_NKINDS || !valid_qubit(n, q0))
        return OR_EARG;
    int two = (kind >= OR_CNOT && kind != OR_U1);
    if (two && (!valid_qubit(n, q1) || q1 == q0))
        return OR_EARG;
    if (kind == OR_CCX && (!valid_qubit(n, q2) || q2 == q0 || q2 == q1))
        return OR_EARG;
    switch (kind) {
    case OR_H: case OR_X: case OR_Y: case OR_Z: case OR_S: case OR_SDG:
    case OR_T: case OR_TDG: case OR_RX: case OR_RY: case OR_RZ:
        mat1(kind, angle, U);
        apply_1q(psi, n, q0, U);
        break;
    case OR_U1:
        for (int r = 0; r < 2; r++)
            for (int k = 0; k < 2; k++)
                U[r][k] = mat[2 * (2 * r + k)] + I * mat[2 * (2 * r + k) + 1];
        apply_1q(psi, n, q0, U);
        break;
    case OR_U2:
        for (int r = 0; r < 4; r++)
            for (int k = 0; k < 4; k++)
                U4[r][k] = mat[2 * (4 * r + k)] + I * mat[2 * (4 * r + k) + 1];
        apply_2q(psi, n, q0, q1, U4);
        break;
    case OR_CNOT: apply_cnot(psi, n, q0, q1); break;
    case OR_CZ:   apply_cphase(psi, n, q0, q1, -1.0); break;
    case OR_CP:   apply_cphase(psi, n, q0, q1, cexp(I * angle)); break;
    case OR_SWAP: apply_swap(psi, n, q0, q1); break;
    case OR_CRY:  apply_cry(psi, n, q0, q1, angle); break;
    case OR_CCX:  apply_ccx(psi, n, q0, q1, q2); break;
    case OR_RXX: case OR_RYY: case OR_RZZ:
        apply_rpp(psi, n, q0, q1, kind, angle);
        break;
    default:
        return OR_EARG;
    }
    return OR_OK;
}

/* Circuit::execute: gates applied in list order.
 * Angle of gate g = theta[pidx[g]] if pidx[g] >= 0, else angles[g].
 * mats: 32 doubles per gate (only read for U1/U2). */
int or_apply_circuit(cplx *psi, int n, int n_gates, const int *kinds,
                     const int *q0, const int *q1, const int *q2,
                     const int *pidx, const double *angles, const double *mats,
                     const double *theta)
{
    for (int g = 0; g < n_gates; g++) {
        double a = pidx[g] >= 0 ? theta[pidx[g]] : angles[g];
        int rc = or_apply_gate(psi, n, kinds[g], q0[g], q1[g], q2[g], a,
                               mats ? mats + 32 * (size_t)g : NULL);
        if (rc != OR_OK)
            return rc;
    }
    return OR_OK;
}

/* Alg. 3 "Gate-Based QFT": for i: H(i); for j>i:
 * CP(pi/2^{j-i}) control i target j; then SWAP(i, n-1-i) for i < floor(n/2).
 * The inverse runs the gates in reverse order with negated phases
 * (SPEC.md:368).  Under MSB-first this equals QFT|x> =
 * N^-1/2 sum_k e^{2 pi i x k / N}|k> with no extra
 * permutation (reading A5). */
void or_qft(cplx *psi, int n, int inverse)
{
    if (!inverse) {
        for (int i = 0; i < n; i++) {
            or_apply_gate(psi, n, OR_H, i, -1, -1, 0.0, NULL);
            for (int j = i + 1; j < n; j++)
                or_apply_gate(psi, n, OR_CP, i, j, -1, OR_PI / ldexp(1.0, j - i), NULL);
        }
        for (int i = 0; i < n / 2; i++)
            or_apply_gate(psi, n, OR_SWAP, i, n - 1 - i, -1, 0.0, NULL);
    } else {
        for (int i = n / 2 - 1; i >= 0; i--)
            or_apply_gate(psi, n, OR_SWAP, i, n - 1 - i, -1, 0.0, NULL);
        for (int i = n - 1; i >= 0; i--) {
            for (int j = n - 1; j > i; j--)
                or_apply_gate(psi, n, OR_CP, i, j, -1, -OR_PI / ldexp(1.0, j - i), NULL);
            or_apply_gate(psi, n, OR_H, i, -1, -1, 0.0, NULL);
        }
    }
}

/* <psi|phi> with Neumaier-summed real and imaginary parts. */
static cplx inner(const cplx *psi, const cplx *phi, int n)
{
    uint64_t N = (uint64_t)1 << n;
    neumaier re = {0, 0}, im = {0, 0};
    for (uint64_t i = 0; i < N; i++) {
        cplx v = conj(psi[i]) * phi[i];
        neu_add(&re, creal(v));
        neu_add(&im, cimag(v));
    }
    return neu_value(&re) + I * neu_value(&im);
}

/* E = sum_t c_t <psi|P_t|psi>: for each term copy psi,
 * apply the Pauli factors as 1q gates (Y where x&z, X where x, Z where z;
 * bit q of a mask = qubit q), take Re<psi|P psi>.
 * Fails with OR_EIMAG unless |Im<psi|P psi>| <= 1e-10 and the value is finite
 * ("explicit, never silent"). */
int or_expval(const cplx *psi, int n, int n_terms, const double *coeffs,
              const uint64_t *xm, const uint64_t *zm, double *out)
{
    uint64_t N = (uint64_t)1 << n;
    cplx *phi = (cplx *)malloc(N * sizeof(cplx));
    if (!phi)
        return OR_ENOMEM;
    neumaier e = {0, 0};
    for (int t = 0; t < n_terms; t++) {
        memcpy(phi, psi, N * sizeof(cplx));
        for (int q = 0; q < n; q++) {
            int xb = (int)((xm[t] >> q) & 1), zb = (int)((zm[t] >> q) & 1);
            if (xb && zb)
                or_apply_gate(phi, n, OR_Y, q, -1, -1, 0.0, NULL);
            else if (xb)
                or_apply_gate(phi, n, OR_X, q, -1, -1, 0.0, NULL);
            else if (zb)
                or_apply_gate(phi, n, OR_Z, q, -1, -1, 0.0, NULL);
        }
        cplx v = inner(psi, phi, n);
        if (!(fabs(cimag(v)) <= 1e-10) || !isfinite(creal(v))) {   /* NaN/Inf too: never silent */
            free(phi);
            return OR_EIMAG;
        }
        neu_add(&e, coeffs[t] * creal(v));
    }
    free(phi);
    *out = neu_value(&e);
    return OR_OK;
}

/* E(theta): fresh |0...0> (State::zero_state), apply the
 * ansatz built with theta, take the expectation. */
int or_energy(int n, int n_gates, const int *kinds, const int *q0, const int *q1,
              const int *q2, const int *pidx, const double *angles,
              const double *mats, const double *theta, int n_terms,
              const double *coeffs, const uint64_t *xm, const uint64_t *zm,
              double *out)
{
    uint64_t N = (uint64_t)1 << n;
    cplx *psi = (cplx *)malloc(N * sizeof(cplx));
    if (!psi)
        return OR_ENOMEM;
    or_init_basis(psi, n, 0);
    int rc = or_apply_circuit(psi, n, n_gates, kinds, q0, q1, q2, pidx, angles, mats, theta);
    if (rc == OR_OK)
        rc = or_expval(psi, n, n_terms, coeffs, xm, zm, out);
    free(psi);
    return rc;
}

/* Parameter-shift rule (Eq. parameter_shift; loop of
 * ParameterShift::compute_gradient) with s = pi/2 and the
 * fixed prefactor 1/2 (reading A6):
 *   g_p = ( E(theta + s e_p) - E(theta - s e_p) ) / 2
 * for each p in which[0..n_which).  Each evaluation rebuilds the circuit from
 * a fresh |0...0>.
 * A parameter of a CRY gate (generator |1><1| (x) Y/2, eigenvalues 0, +-1/2:
 * E(theta) = a0 + a1 cos(theta/2) + b1 sin(theta/2) + a2 cos(theta) +
 * b2 sin(theta), for which the two-term rule is not exact -- reading A8;
 * the paper is silent) takes the four-term rule that is exact for those two
 * frequencies (reading A8):
 *   g_p = c1 [E(+pi/2) - E(-pi/2)] - c2 [E(+3pi/2) - E(-3pi/2)],
 *   c1 = (sqrt2 + 1)/(4 sqrt2), c2 = (sqrt2 - 1)/(4 sqrt2). */
int or_param_shift(int n, int n_gates, const int *kinds, const int *q0, const int *q1,
                   const int *q2, const int *pidx, const double *angles,
                   const double *mats, const double *theta, int n_params,
                   int n_terms, const double *coeffs, const uint64_t *xm,
                   const uint64_t *zm, const int *which, int n_which, double *grad)
{
    const double shift = OR_PI / 2.0;
    double *tp = (double *)malloc((size_t)(n_params > 0 ? n_params : 1) * sizeof(double));
    if (!tp)
        return OR_ENOMEM;
    for (int w = 0; w < n_which; w++) {
        int i = which[w];
        double e_plus, e_minus;
        int controlled = 0;
        for (int k = 0; k < n_gates; k++)
            if (pidx[k] == i && kinds[k] == OR_CRY)
                controlled = 1;
        if (controlled) {
            const double s[4] = {OR_PI / 2.0, -OR_PI / 2.0, 3.0 * OR_PI / 2.0, -3.0 * OR_PI / 2.0};
            double e[4];
            for (int k = 0; k < 4; k++) {
                memcpy(tp, theta, (size_t)n_params * sizeof(double));
                tp[i] += s[k];
                int rc = or_energy(n, n_gates, kinds, q0, q1, q2, pidx, angles, mats, tp,
                                   n_terms, coeffs, xm, zm, &e[k]);
                if (rc != OR_OK) { free(tp); return rc; }
            }
            const double r2 = sqrt(2.0);
            const double c1 = (r2 + 1.0) / (4.0 * r2), c2 = (r2 - 1.0) / (4.0 * r2);
            grad[w] = c1 * (e[0] - e[1]) - c2 * (e[2] - e[3]);
            continue;
        }
        memcpy(tp, theta, (size_t)n_params * sizeof(double));
        tp[i] += shift;
        int rc = or_energy(n, n_gates, kinds, q0, q1, q2, pidx, angles, mats, tp,
                           n_terms, coeffs, xm, zm, &e_plus);
        if (rc != OR_OK) { free(tp); return rc; }
        memcpy(tp, theta, (size_t)n_params * sizeof(double));
        tp[i] -= shift;
        rc = or_energy(n, n_gates, kinds, q0, q1, q2, pidx, angles, mats, tp,
                       n_terms, coeffs, xm, zm, &e_minus);
        if (rc != OR_OK) { free(tp); return rc; }
        grad[w] = (e_plus - e_minus) / 2.0;
    }
    free(tp);
    return OR_OK;
}

/* sum_i |a_i|^2 (Neumaier). */
double or_norm2(const cplx *psi, int n)
{
    uint64_t N = (uint64_t)1 << n;
    neumaier s = {0, 0};
    for (uint64_t i = 0; i < N; i++) {
        neu_add(&s, creal(psi[i]) * creal(psi[i]));
        neu_add(&s, cimag(psi[i]) * cimag(psi[i]));
    }
    return neu_value(&s);
}
