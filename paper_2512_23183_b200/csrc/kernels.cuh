// kernels.cuh -- sm_100a kernels of liblq (included once, by lq_api.cu):
// the tile kernel (tile.cuh) plus the pair, diagonal, matrix-builder, init,
// readback, Pauli and PSR kernels.  All are HBM-streaming FP64 kernels; see
// DESIGN.md §5 for the roofline of each.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tile.cuh"
#include "../../include/lq.h"

namespace lq {

// ---------------------------------------------------------------- pair kernel (a4)
// One 1q/2q gate on arbitrary physical bits: strided pairs (i, i | 2^b) or
// quads, 16-byte loads, controls as a bit mask (Alg. 1 generalised).
__global__ void __launch_bounds__(256) k_pair(int n, uint64_t gofs, const KOp op, const double2 *__restrict__ mats,
                                              uint64_t mat_stride, double2 *__restrict__ state,
                                              uint64_t state_stride) {
    // n: local index bits; gofs: this shard's physical global bits (controls only)
    double2 *__restrict__ psi = state + (uint64_t)blockIdx.y * state_stride;
    const double2 *__restrict__ M = mats + (uint64_t)blockIdx.y * mat_stride;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (op.type == K_U1 || op.type == K_X || op.type == K_G) {
        const uint64_t np = 1ull << (n - 1);
        const uint64_t mb = 1ull << op.b0;
        double2 u00 = make_double2(0, 0), u01 = u00, u10 = u00, u11 = u00;
        if (op.type == K_U1) { u00 = M[op.mat]; u01 = M[op.mat + 1]; u10 = M[op.mat + 2]; u11 = M[op.mat + 3]; }
        if (op.type == K_G) {   // expand lambda * M (lq_internal.h GKind)
            const double p = M[op.mat].x, l = M[op.mat].y;
            const bool alt = M[op.mat + 1].x != 0.0;
            const double one = alt ? p : 1.0, off = alt ? 1.0 : p;
            if (op.qj == GK_REAL) {
                u00 = make_double2(l * one, 0); u01 = make_double2(-l * off, 0);
                u10 = make_double2(l * off, 0); u11 = u00;
            } else if (op.qj == GK_IMAG) {
                u00 = make_double2(l * one, 0); u01 = make_double2(0, -l * off); u10 = u01; u11 = u00;
            } else {
                u00 = make_double2(l, 0); u01 = u00; u10 = u00; u11 = make_double2(-l, 0);
            }
        }
        // four pairs per thread and iteration, all loads issued before any
        // store: 128 bytes in flight per thread (HBM latency hiding)
        constexpr int U = 4;
        for (; i < np; i += U * stride) {
            uint64_t i0[U];
            bool on[U];
            double2 x[U], y[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint64_t j = i + (uint64_t)u * stride;
                i0[u] = insert_zero64(j, op.b0);
                on[u] = j < np && ((i0[u] | gofs) & op.cmask) == op.cmask;
                if (on[u]) { x[u] = psi[i0[u]]; y[u] = psi[i0[u] | mb]; }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (!on[u]) continue;
                if (op.type == K_X) { psi[i0[u]] = y[u]; psi[i0[u] | mb] = x[u]; }
                else {
                    psi[i0[u]] = cfma(u00, x[u], cmul(u01, y[u]));
                    psi[i0[u] | mb] = cfma(u10, x[u], cmul(u11, y[u]));
                }
            }
        }
    } else {
        const uint64_t nq = 1ull << (n - 2);
        const int hb = op.b0 > op.b1 ? op.b0 : op.b1, lb = op.b0 > op.b1 ? op.b1 : op.b0;
        const uint64_t m0 = 1ull << op.b0, m1 = 1ull << op.b1;   // b0: high sub-index bit
        double2 U[16];
        if (op.type == K_U2)
            for (int k = 0; k < 16; k++) U[k] = M[op.mat + k];
        for (; i < nq; i += stride) {
            const uint64_t base = insert_zero64(insert_zero64(i, lb), hb);
            if (((base | gofs) & op.cmask) != op.cmask) continue;
            const uint64_t j0 = base, j1 = base | m1, j2 = base | m0, j3 = base | m0 | m1;
            if (op.type == K_SWAP) {
                double2 x = psi[j1];
                psi[j1] = psi[j2];
                psi[j2] = x;
            } else {
                double2 x0 = psi[j0], x1 = psi[j1], x2 = psi[j2], x3 = psi[j3];
                psi[j0] = cfma(U[0], x0, cfma(U[1], x1, cfma(U[2], x2, cmul(U[3], x3))));
                psi[j1] = cfma(U[4], x0, cfma(U[5], x1, cfma(U[6], x2, cmul(U[7], x3))));
                psi[j2] = cfma(U[8], x0, cfma(U[9], x1, cfma(U[10], x2, cmul(U[11], x3))));
                psi[j3] = cfma(U[12], x0, cfma(U[13], x1, cfma(U[14], x2, cmul(U[15], x3))));
            }
        }
    }
}

// ---------------------------------------------------------------- diagonal kernel (a3)
// a_i <- a_i * prod_ops d_op(bits of i): any number of fused Z/S/T/RZ/CZ/CP/RZZ
// factors in one read-modify-write pass ("phase rotations based on bitwise
// masks").
constexpr int DIAG_MAX_OPS = 128;
__global__ void __launch_bounds__(256) k_diag(int n, uint64_t gofs, const KOp *__restrict__ ops, int n_ops,
                                              const double2 *__restrict__ mats, uint64_t mat_stride,
                                              double2 *__restrict__ state, uint64_t state_stride) {
    __shared__ KOp sop[DIAG_MAX_OPS];
    __shared__ double2 sd[DIAG_MAX_OPS][4];
    const double2 *__restrict__ M = mats + (uint64_t)blockIdx.y * mat_stride;
    double2 *__restrict__ psi = state + (uint64_t)blockIdx.y * state_stride;
    for (int k = threadIdx.x; k < n_ops; k += blockDim.x) {
        sop[k] = ops[k];
        const int cnt = ops[k].type == K_D2 ? 4 : 2;
        for (int e = 0; e < 4; e++) sd[k][e] = e < cnt ? M[ops[k].mat + e] : make_double2(1, 0);
    }
    __syncthreads();
    const uint64_t N = 1ull << n;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
        double2 ph = make_double2(1.0, 0.0);
        const uint64_t x = i | gofs;   // logic index (global bits of a shard are constants)
        for (int k = 0; k < n_ops; k++) {
            const KOp &o = sop[k];
            if ((x & o.cmask) != o.cmask) continue;
            uint32_t idx = (uint32_t)((x >> o.b0) & 1);
            if (o.type == K_D2) idx = 2 * idx + (uint32_t)((x >> o.b1) & 1);
            ph = cmul(ph, sd[k][idx]);
        }
        psi[i] = cmul(psi[i], ph);
    }
}

// ---------------------------------------------------------------- matrices
// Gate matrices (textbook, reading A4; rotations exp(-i theta G/2),
// PAPER.md:373, 380), computed per circuit from theta on the device.
__device__ void gate2x2(int kind, double th, const double2 *c, double2 (&U)[4]) {
    const double r2 = 0.70710678118654752440;
    double s, co;
    sincos(0.5 * th, &s, &co);
    const double2 z = make_double2(0, 0), one = make_double2(1, 0);
    switch (kind) {
    case LQ_H:   U[0] = make_double2(r2, 0); U[1] = U[0]; U[2] = U[0]; U[3] = make_double2(-r2, 0); break;
    case LQ_X:   U[0] = z; U[1] = one; U[2] = one; U[3] = z; break;
    case LQ_Y:   U[0] = z; U[1] = make_double2(0, -1); U[2] = make_double2(0, 1); U[3] = z; break;
    case LQ_Z:   U[0] = one; U[1] = z; U[2] = z; U[3] = make_double2(-1, 0); break;
    case LQ_S:   U[0] = one; U[1] = z; U[2] = z; U[3] = make_double2(0, 1); break;
    case LQ_SDG: U[0] = one; U[1] = z; U[2] = z; U[3] = make_double2(0, -1); break;
    case LQ_T:   U[0] = one; U[1] = z; U[2] = z; U[3] = make_double2(r2, r2); break;
    case LQ_TDG: U[0] = one; U[1] = z; U[2] = z; U[3] = make_double2(r2, -r2); break;
    case LQ_RX:  U[0] = make_double2(co, 0); U[1] = make_double2(0, -s); U[2] = U[1]; U[3] = U[0]; break;
    case LQ_RY:  U[0] = make_double2(co, 0); U[1] = make_double2(-s, 0); U[2] = make_double2(s, 0); U[3] = U[0]; break;
    case LQ_RZ:  U[0] = make_double2(co, -s); U[1] = z; U[2] = z; U[3] = make_double2(co, s); break;
    case LQ_CP: {
        double s1, c1;
        sincos(th, &s1, &c1);
        U[0] = one; U[1] = z; U[2] = z; U[3] = make_double2(c1, s1);
        break;
    }
    case LQ_U1:  U[0] = c[0]; U[1] = c[1]; U[2] = c[2]; U[3] = c[3]; break;
    case FK_YDIAG: U[0] = make_double2(0, 1); U[1] = z; U[2] = z; U[3] = make_double2(0, -1); break;
    default:     U[0] = one; U[1] = z; U[2] = z; U[3] = one; break;
    }
}

__global__ void k_build_mats(const MSpec *__restrict__ specs, int n_specs, const MFactor *__restrict__ factors,
                             const double *__restrict__ theta, const Shift *__restrict__ shifts,
                             const double2 *__restrict__ cst, double2 *__restrict__ mats, uint64_t mat_stride,
                             int n_circ) {
    const uint64_t total = (uint64_t)n_specs * n_circ;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const int c = (int)(idx / n_specs), si = (int)(idx % n_specs);
        const MSpec sp = specs[si];
        Shift sh;
        sh.pidx = -1;
        sh.delta = 0.0;
        if (shifts) sh = shifts[c];
        double2 *out = mats + (uint64_t)c * mat_stride + sp.out;
        auto angle = [&](const MFactor &f) {
            if (f.pidx < 0) return f.angle;
            double a = theta[f.pidx];
            if (f.pidx == sh.pidx) a += sh.delta;
            return a;
        };
        if (sp.form == MF_U2x2 || sp.form == MF_DIAG2) {
            double2 A[4] = {make_double2(1, 0), make_double2(0, 0), make_double2(0, 0), make_double2(1, 0)};
            for (uint32_t fi = sp.f_begin; fi < sp.f_end; fi++) {
                const MFactor f = factors[fi];
                double2 F[4];
                gate2x2(f.kind, angle(f), f.cst >= 0 ? cst + f.cst : nullptr, F);
                double2 B[4];
                B[0] = cfma(F[0], A[0], cmul(F[1], A[2]));
                B[1] = cfma(F[0], A[1], cmul(F[1], A[3]));
                B[2] = cfma(F[2], A[0], cmul(F[3], A[2]));
                B[3] = cfma(F[2], A[1], cmul(F[3], A[3]));
                A[0] = B[0]; A[1] = B[1]; A[2] = B[2]; A[3] = B[3];
            }
            if (sp.form == MF_U2x2) { out[0] = A[0]; out[1] = A[1]; out[2] = A[2]; out[3] = A[3]; }
            else {   // diagonal: d0, d1 and the ratio d1/d0 (register-bit ops defer d0)
                out[0] = A[0];
                out[1] = A[3];
                const double nn = A[0].x * A[0].x + A[0].y * A[0].y;
                const double2 r = cmul(A[3], make_double2(A[0].x, -A[0].y));
                out[2] = make_double2(r.x / nn, r.y / nn);
            }
        } else if (sp.form == MF_G) {
            // lambda * M (GKind table layout, lq_internal.h): the larger of
            // |cos|, |sin| becomes lambda so |p| <= 1
            const MFactor f = factors[sp.f_begin];
            if (f.kind == LQ_H) {
                out[0] = make_double2(0.0, 0.70710678118654752440);
                out[1] = make_double2(0.0, 0.0);
            } else {
                double s, co;
                sincos(0.5 * angle(f), &s, &co);
                if (fabs(co) >= fabs(s)) { out[0] = make_double2(s / co, co); out[1] = make_double2(0.0, 0.0); }
                else { out[0] = make_double2(co / s, s); out[1] = make_double2(1.0, 0.0); }
            }
        } else {
            const MFactor f = factors[sp.f_begin];
            const double th = angle(f);
            double s, co;
            sincos(0.5 * th, &s, &co);
            if (sp.form == MF_DIAG4) {   // RZZ: diag(e^{-i t/2}, e^{i t/2}, e^{i t/2}, e^{-i t/2})
                out[0] = make_double2(co, -s); out[1] = make_double2(co, s);
                out[2] = make_double2(co, s);  out[3] = make_double2(co, -s);
            } else if (f.kind == LQ_U2) {
                for (int e = 0; e < 16; e++) out[e] = cst[f.cst + e];
            } else {
                // RXX / RYY = cos(t/2) I - i sin(t/2) P(x)P
                for (int e = 0; e < 16; e++) out[e] = make_double2(0, 0);
                for (int d = 0; d < 4; d++) out[5 * d] = make_double2(co, 0);
                const double yy = (f.kind == LQ_RYY) ? -1.0 : 1.0;   // Y(x)Y anti-diagonal: -1, 1, 1, -1
                out[0 * 4 + 3] = make_double2(0, -s * yy);
                out[1 * 4 + 2] = make_double2(0, -s);
                out[2 * 4 + 1] = make_double2(0, -s);
                out[3 * 4 + 0] = make_double2(0, -s * yy);
            }
        }
    }
}

// ---------------------------------------------------------------- init
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// counter-based complex Gaussian of SURVEY.md §8(c) c.1 (lq.h lq_sv_init_random)
__device__ __forceinline__ double2 gauss_amp(uint64_t seed, uint64_t i) {
    const uint64_t x0 = splitmix64(seed ^ (2 * i)), x1 = splitmix64(seed ^ (2 * i + 1));
    const double u0 = ((double)(x0 >> 11) + 0.5) * 0x1.0p-53;
    const double u1 = ((double)(x1 >> 11) + 0.5) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u0));
    double s, c;
    sincospi(2.0 * u1, &s, &c);
    return make_double2(r * c, r * s);
}

constexpr int RED_BLOCKS = 1184;   // 8 x 148 SMs; fixed => deterministic reduction order

// off: logical index of the shard's first amplitude (sharded states).
// |a_i|^2 = r_i^2 = -2 ln u0_i: the phase draw never enters the norm, and
// the sum of logs is the log of a running product (renormalised with frexp
// every 16 factors: u0 >= 2^-54, so 16 factors stay above 2^-1022), so this
// sweep costs one splitmix64 and one DMUL per amplitude instead of a log, a
// sqrt and a sincospi.
__global__ void __launch_bounds__(256) k_random_norm(uint64_t N, uint64_t off, uint64_t seed, double *partial) {
    double p = 1.0;
    int e = 0, cnt = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < N; i += (uint64_t)gridDim.x * 256) {
        const uint64_t x0 = splitmix64(seed ^ (2 * (off + i)));
        p *= ((double)(x0 >> 11) + 0.5) * 0x1.0p-53;
        if (++cnt == 16) {
            int ex;
            p = frexp(p, &ex);
            e += ex;
            cnt = 0;
        }
    }
    const double acc = -2.0 * (log(p) + (double)e * 0.69314718055994530942);
    __shared__ double red[256];
    double r = block_sum(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = r;
}

// The write sweep evaluates the same formula as gauss_amp with table-driven
// log and sincospi (the libdevice FP64 routines cost ~100 FP64 instructions
// per amplitude and made this sweep FP64-bound at a quarter of the write
// roofline):
//   log u0 = e ln2 + log c + log1p(r), u0 = 2^e m, m in [0.75, 1.5)
//            (m in [1.5, 2) is halved and e incremented), c = the nearest
//            node of spacing 1/128 above 1 and 1/256 below it (130 nodes),
//            r = (m - c) / c, |r| <= 1/256, log1p by its Taylor series to
//            r^8 (remainder < 2^-75 relative).  Reducing to m around 1 keeps the
//            relative error at a few ulp where log u0 -> 0 (u0 -> 1): there
//            c = 1, log c = 0 and log u0 = log1p(r) with r exact; a fixed
//            m in [1, 2) would cancel -ln2 against log c ~ ln2 (4e-9 relative
//            at u0 = 1 - 1e-6);
//   (cos, sin)(pi x), x = 2 u1 in (0, 2): x = j/128 + t, t in [0, 1/128),
//            rotate the tabulated (cos, sin)(pi j/128) by (cos, sin)(pi t)
//            from their Taylor series (degree 8 / 9, remainder < 2^-70).
// m - c and x - j/128 are exact; the tables are computed per block with
// the libdevice routines.  Relative error of the amplitude a few 1e-16
// everywhere (lq.h lq_sv_init_random; test_gpu_fullsize checks the ratio to
// the oracle's unnormalised amplitudes to 1e-12 relative at n = 33).
__device__ __forceinline__ double2 gauss_amp_tab(uint64_t seed, uint64_t i, const double2 *__restrict__ lt,
                                                 const double2 *__restrict__ sc) {
    const uint64_t x0 = splitmix64(seed ^ (2 * i)), x1 = splitmix64(seed ^ (2 * i + 1));
    const double u0 = ((double)(x0 >> 11) + 0.5) * 0x1.0p-53;
    const double u1 = ((double)(x1 >> 11) + 0.5) * 0x1.0p-53;
    // log u0
    const uint64_t b = (uint64_t)__double_as_longlong(u0);
    int e = (int)((b >> 52) & 0x7FF) - 1023;         // u0 >= 2^-54: normal
    const uint32_t mt = (uint32_t)((b >> 44) & 255u); // top 8 mantissa bits
    const uint32_t kk = (mt + 1) >> 1;                // nearest 1/128 step: 0..128
    double m = __longlong_as_double((long long)((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
    double cn;
    uint32_t j;
    if (mt >= 128) {                                   // m in [1.5, 2): m/2 in [0.75, 1)
        m *= 0.5;
        e += 1;
        cn = 0.5 + (double)kk * 0.00390625;           // kk in 64..128: c in [0.75, 1]
        j = kk + 1;
    } else {
        cn = 1.0 + (double)kk * 0.0078125;            // kk in 0..64: c in [1, 1.5]
        j = kk;
    }
    const double2 L = lt[j];                          // (1 / c, log c)
    const double r = (m - cn) * L.x;                  // m - c exact (Sterbenz)
    double p = -1.0 / 8.0;
    p = fma(p, r, 1.0 / 7.0);
    p = fma(p, r, -1.0 / 6.0);
    p = fma(p, r, 1.0 / 5.0);
    p = fma(p, r, -1.0 / 4.0);
    p = fma(p, r, 1.0 / 3.0);
    p = fma(p, r, -0.5);
    p = p * r * r + r;                                 // log1p(r)
    const double lg = fma((double)e, 0.69314718055994530942, L.y + p);
    const double rad = sqrt(-2.0 * lg);
    // (cos, sin)(2 pi u1)
    const double x = 2.0 * u1;
    const uint32_t k = (uint32_t)(x * 128.0);         // 0..255
    const double t = (x - (double)k * 0.0078125) * 3.14159265358979323846;
    const double t2 = t * t;
    double cs = 1.0 / 40320.0;
    cs = fma(cs, t2, -1.0 / 720.0);
    cs = fma(cs, t2, 1.0 / 24.0);
    cs = fma(cs, t2, -0.5);
    cs = fma(cs, t2, 1.0);
    double sn = 1.0 / 362880.0;
    sn = fma(sn, t2, -1.0 / 5040.0);
    sn = fma(sn, t2, 1.0 / 120.0);
    sn = fma(sn, t2, -1.0 / 6.0);
    sn = fma(sn * t2, t, t);
    const double2 T = sc[k];                          // (cos, sin)(pi k / 128)
    const double c = fma(T.x, cs, -T.y * sn), s = fma(T.y, cs, T.x * sn);
    return make_double2(rad * c, rad * s);
}

__global__ void __launch_bounds__(256) k_random_write(uint64_t N, uint64_t off, uint64_t seed, const double *norm2,
                                                      double2 *__restrict__ psi) {
    __shared__ double2 lt[130], sc[256];
    {
        const uint32_t q = threadIdx.x;   // blockDim = 256
        double s, c;
        sincospi((double)q / 128.0, &s, &c);
        sc[q] = make_double2(c, s);
        if (q < 130) {   // nodes of gauss_amp_tab: 1 + q/128 (q <= 64), 0.5 + (q - 1)/256 (q >= 65)
            const double cj = q <= 64 ? 1.0 + (double)q * 0.0078125 : 0.5 + (double)(q - 1) * 0.00390625;
            lt[q] = make_double2(1.0 / cj, log(cj));
        }
    }
    __syncthreads();
    const double inv = 1.0 / sqrt(*norm2);
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < N; i += (uint64_t)gridDim.x * 256)
        psi[i] = cscale(gauss_amp_tab(seed, off + i, lt, sc), inv);
}

// ---------------------------------------------------------------- global-qubit exchange (a9)
// Sharded states (dist.h): exchanging k global bits g_j with k local bits
// l_j (ascending), a shard splits into 2^k parts by the value b of its
// l-bits (bit j of b <-> l_j); part b travels to the rank whose g-bits are b
// and the part coming back lands in the same positions.  Part index i (the
// other nl - k bits, ascending) <-> shard position with b deposited at the
// l positions.  k = 1 is the pairwise half-shard swap.
struct PartSpec {
    int k;
    int l[4];   // ascending local bit positions (dist.h MAX_SWAP_K)
};
__device__ __forceinline__ uint64_t insert_bit64(uint64_t x, int b, uint64_t v) {
    const uint64_t lo = x & ((1ull << b) - 1);
    return ((x ^ lo) << 1) | (v << b) | lo;
}
__device__ __forceinline__ uint64_t part_pos(const PartSpec &ps, uint64_t i, uint32_t b) {
    for (int j = 0; j < ps.k; j++) i = insert_bit64(i, ps.l[j], (b >> j) & 1u);
    return i;
}

// both shards in this process (group mode): part va of shard a <-> part vb
// of shard b, element-wise in place.  All three kernels move U elements per
// thread per iteration, loads first (HBM latency hiding, as k_pair).
constexpr int MOVE_U = 4;
__global__ void __launch_bounds__(256) k_swap_parts(double2 *__restrict__ a, double2 *__restrict__ b, PartSpec ps,
                                                    uint32_t va, uint32_t vb, uint64_t cnt) {
    const uint64_t stride = (uint64_t)gridDim.x * 256;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < cnt; i += MOVE_U * stride) {
        uint64_t pa[MOVE_U], pb[MOVE_U];
        double2 x[MOVE_U], y[MOVE_U];
#pragma unroll
        for (int u = 0; u < MOVE_U; u++) {
            const uint64_t j = i + u * stride;
            pa[u] = part_pos(ps, j, va);
            pb[u] = part_pos(ps, j, vb);
            if (j < cnt) { x[u] = a[pa[u]]; y[u] = b[pb[u]]; }
        }
#pragma unroll
        for (int u = 0; u < MOVE_U; u++)
            if (i + u * stride < cnt) { a[pa[u]] = y[u]; b[pb[u]] = x[u]; }
    }
}

// NCCL mode: chunk [off, off + cnt) of every outgoing part -> contiguous
// staging (blockIdx.y = peer slot p: part b = p < own ? p : p + 1), and back
__global__ void __launch_bounds__(256) k_pack_parts(const double2 *__restrict__ src, double2 *__restrict__ dst,
                                                    PartSpec ps, uint32_t own, uint64_t off, uint64_t cnt) {
    const uint32_t p = blockIdx.y, bv = p < own ? p : p + 1;
    double2 *d = dst + (uint64_t)p * cnt;
    const uint64_t stride = (uint64_t)gridDim.x * 256;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < cnt; i += MOVE_U * stride) {
        double2 x[MOVE_U];
#pragma unroll
        for (int u = 0; u < MOVE_U; u++)
            if (i + u * stride < cnt) x[u] = src[part_pos(ps, off + i + u * stride, bv)];
#pragma unroll
        for (int u = 0; u < MOVE_U; u++)
            if (i + u * stride < cnt) d[i + u * stride] = x[u];
    }
}
__global__ void __launch_bounds__(256) k_unpack_parts(double2 *__restrict__ dst, const double2 *__restrict__ src,
                                                      PartSpec ps, uint32_t own, uint64_t off, uint64_t cnt) {
    const uint32_t p = blockIdx.y, bv = p < own ? p : p + 1;
    const double2 *s = src + (uint64_t)p * cnt;
    const uint64_t stride = (uint64_t)gridDim.x * 256;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < cnt; i += MOVE_U * stride) {
        double2 x[MOVE_U];
#pragma unroll
        for (int u = 0; u < MOVE_U; u++)
            if (i + u * stride < cnt) x[u] = s[i + u * stride];
#pragma unroll
        for (int u = 0; u < MOVE_U; u++)
            if (i + u * stride < cnt) dst[part_pos(ps, off + i + u * stride, bv)] = x[u];
    }
}

__global__ void __launch_bounds__(256) k_fill_basis(uint64_t N, uint64_t k, double2 *__restrict__ state,
                                                    uint64_t state_stride) {
    double2 *psi = state + (uint64_t)blockIdx.y * state_stride;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < N; i += (uint64_t)gridDim.x * 256)
        psi[i] = make_double2(i == k ? 1.0 : 0.0, 0.0);
}

// ---------------------------------------------------------------- access-pattern ceiling (measurement)
// The memory traffic of a tile pass without its arithmetic: every tile (the
// 2^K amplitudes whose bits outside the tile set are fixed) is read and
// written back in place (re and im swapped), 16 amplitudes per thread, loads
// first, tiles in the order of their free bits over a persistent grid, as in
// the tile kernel.  Its time is the ceiling an HBM-bound pass with that tile
// set can reach (bench.py roofline.access_pattern_ceiling).
struct SweepSpec {
    int K, nfree;
    uint8_t tpos[16];   // tile bit positions, ascending
    uint8_t fpos[48];   // free bit positions, ascending
};
__device__ __forceinline__ uint64_t deposit_bits(uint64_t v, const uint8_t *pos, int cnt) {
    uint64_t a = 0;
    for (int i = 0; i < cnt; i++) a |= ((v >> i) & 1ull) << pos[i];
    return a;
}
__global__ void __launch_bounds__(256) k_tile_sweep(double2 *__restrict__ s, uint64_t n_tiles, SweepSpec P) {
    constexpr int U = 16;
    const uint32_t per = (1u << P.K) / U;   // threads per tile
    const uint32_t lane = threadIdx.x % per, slot = threadIdx.x / per, tpc = blockDim.x / per;
    uint64_t off[U];
#pragma unroll
    for (int u = 0; u < U; u++) off[u] = deposit_bits(lane + u * per, P.tpos, P.K);
    for (uint64_t t = (uint64_t)blockIdx.x * tpc + slot; t < n_tiles; t += (uint64_t)gridDim.x * tpc) {
        const uint64_t base = deposit_bits(t, P.fpos, P.nfree);
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; u++) a[u] = s[base | off[u]];
#pragma unroll
        for (int u = 0; u < U; u++) s[base | off[u]] = make_double2(a[u].y, a[u].x);
    }
}

__global__ void __launch_bounds__(256) k_norm2(uint64_t N, const double2 *__restrict__ psi, double *partial) {
    double acc = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < N; i += (uint64_t)gridDim.x * 256) {
        double2 a = psi[i];
        acc = fma(a.x, a.x, fma(a.y, a.y, acc));
    }
    __shared__ double red[256];
    double r = block_sum(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = r;
}

// out[c] = sum_{s < n} partial[c * stride + s], fixed order (one block per c)
__global__ void __launch_bounds__(256) k_sum_partials(const double *__restrict__ partial, uint64_t stride,
                                                      uint32_t n, double *out) {
    const double *p = partial + (uint64_t)blockIdx.x * stride;
    double acc = 0.0;
    for (uint32_t i = threadIdx.x; i < n; i += 256) acc += p[i];
    __shared__ double red[256];
    double r = block_sum(acc, red);
    if (threadIdx.x == 0) out[blockIdx.x] = r;
}

// chunk sums: out[c * stride + b] = sum of partial[c * stride + b * chunk ..
// + chunk) (clipped to n), fixed order; grid (n_chunks, n_circ)
__global__ void __launch_bounds__(256) k_sum_chunks(const double *__restrict__ partial, uint64_t stride, uint32_t n,
                                                    uint32_t chunk, double *out) {
    const double *p = partial + (uint64_t)blockIdx.y * stride;
    const uint32_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    double acc = 0.0;
    for (uint32_t i = lo + threadIdx.x; i < hi; i += 256) acc += p[i];
    __shared__ double red[256];
    double r = block_sum(acc, red);
    if (threadIdx.x == 0) out[(uint64_t)blockIdx.y * stride + blockIdx.x] = r;
}

// ---------------------------------------------------------------- logical <-> physical
struct QMap { int8_t q[64]; };

__device__ __forceinline__ uint64_t logical_to_phys(uint64_t x, int n, const QMap &m) {
    uint64_t g = 0;
    for (int q = 0; q < n; q++)
        if ((x >> (n - 1 - q)) & 1) g |= 1ull << m.q[q];
    return g;
}

__global__ void k_gather(int n, QMap m, const double2 *__restrict__ psi, const uint64_t *__restrict__ idx,
                         uint64_t offset, uint64_t count, double2 *__restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x = idx ? idx[i] : offset + i;
        out[i] = psi[logical_to_phys(x, n, m)];
    }
}

// idx (nullable): explicit indices instead of offset + i (sharded writes)
__global__ void k_scatter(int n, QMap m, double2 *__restrict__ psi, const uint64_t *__restrict__ idx, uint64_t offset,
                          uint64_t count, const double2 *__restrict__ in) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        psi[logical_to_phys(idx ? idx[i] : offset + i, n, m)] = in[i];
}

// ---------------------------------------------------------------- Pauli expectation (a7)
// E = sum_t c_t Re <psi|P_t|psi>,  P|j> = i^{y} (-1)^{popcount(j & z)} |j ^ x>
// (PAPER.md:733-734).  One CTA per tile: the tile holds every pair (j, j^x)
// of the pass's x masks; per-CTA partial sums are reduced in fixed order.

__device__ __forceinline__ double re_iy(double2 w, uint32_t y) {
    switch (y & 3) {
    case 0: return w.x;
    case 1: return -w.y;
    case 2: return -w.x;
    default: return w.y;
    }
}

// Direct (non-tiled) pass for x masks wider than a tile.
__global__ void __launch_bounds__(256) k_pauli_direct(int n, uint64_t gofs, uint64_t x, const PTerm *__restrict__ terms,
                                                      uint32_t nterm, const double2 *__restrict__ state,
                                                      uint64_t state_stride, double *__restrict__ partial,
                                                      uint64_t slot_stride, uint32_t slot) {
    const double2 *__restrict__ psi = state + (uint64_t)blockIdx.y * state_stride;
    const uint64_t N = 1ull << n;
    double acc = 0.0;
    for (uint64_t j = (uint64_t)blockIdx.x * 256 + threadIdx.x; j < N; j += (uint64_t)gridDim.x * 256) {
        const double2 a = psi[j], p = psi[j ^ x];
        const double2 w = make_double2(fma(p.x, a.x, p.y * a.y), fma(p.x, a.y, -p.y * a.x));
        for (uint32_t k = 0; k < nterm; k++) {
            const PTerm pt = terms[k];
            const double c = (__popcll((j | gofs) & pt.zfull) & 1) ? -pt.coeff : pt.coeff;
            acc = fma(c, re_iy(w, pt.yph), acc);
        }
    }
    __shared__ double red[256];
    double r = block_sum(acc, red);
    if (threadIdx.x == 0) partial[(uint64_t)blockIdx.y * slot_stride + slot + blockIdx.x] = r;
}

// ---------------------------------------------------------------- constant op tables
// Stage every JIT pass's op tables for circuits 0..n_circ-1 of a launch into
// `out` (layout: CtabDesc); the host then copies each pass's slice into the
// pass module's __constant__ bank.  grid (n_pass, n_circ).
__global__ void k_stage_ctab(const KOp *__restrict__ kops, const CtabDesc *__restrict__ desc,
                             const double2 *__restrict__ mats, uint64_t mat_stride, const double2 *__restrict__ cst,
                             double2 *__restrict__ out) {
    const CtabDesc D = desc[blockIdx.x];
    const uint32_t c = blockIdx.y;
    double2 *o = out + D.out + (uint64_t)c * D.smat;
    const double2 *M = mats ? mats + (uint64_t)c * mat_stride : nullptr;
    for (uint32_t k = D.op_begin + threadIdx.x; k < D.op_end; k += blockDim.x) stage_table(kops[k], o, M, cst);
}

// ---------------------------------------------------------------- PSR combine (a8)
// g_p = sum_k w_k E(theta + s_k e_p).  Rotations exp(-i theta G / 2) with
// G^2 = 1 take the paper's two-term rule, s = +-pi/2, w = +-1/2
// (PAPER.md:374-377, 533-534).  A controlled rotation (CRY) has generator
// eigenvalues {0, +-1/2}, so E(theta) carries frequencies 1/2 and 1 and the
// two-term rule is not exact (reading A8): it takes the four-term rule
// s = +-pi/2, +-3pi/2 with w = +-(sqrt2+1)/(4 sqrt2), -+(sqrt2-1)/(4 sqrt2)
// (reading A8; derived there).  One component per thread, terms
// summed in fixed order.
struct PsrRule { int32_t p, nc; int32_t c[4]; double w[4]; };
__global__ void k_psr_combine(const double *__restrict__ E, const PsrRule *__restrict__ rules, int n_rules,
                              int base_idx, double *__restrict__ grad, int n_params, double *energy) {
    // launched as ONE block: zero, barrier, then the owned components
    for (int i = threadIdx.x; i < n_params; i += blockDim.x) grad[i] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < n_rules; i += blockDim.x) {
        const PsrRule r = rules[i];
        double g = 0.0;
        for (int k = 0; k < r.nc; k++) g = fma(r.w[k], E[r.c[k]], g);
        grad[r.p] = g;
    }
    if (energy && threadIdx.x == 0) *energy = base_idx >= 0 ? E[base_idx] : 0.0;
}

// ---------------------------------------------------------------- Adam (VQE outer loop)
// theta^{t+1} = theta^t - lr * Adam(g^t) (Adam of the cited
// Kingma & Ba: bias-corrected first and second moments).  bc1 = 1 - b1^t,
// bc2 = 1 - b2^t.  Explicit _rn intrinsics keep the update free of FMA
// contraction (the update is O(P) work; exact rounding is worth more).
__global__ void k_adam_step(double *__restrict__ theta, double *__restrict__ m, double *__restrict__ v,
                            const double *__restrict__ g, int n, double lr, double b1, double b2, double eps,
                            double bc1, double bc2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double gi = g[i];
        const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dadd_rn(1.0, -b1), gi));
        const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dadd_rn(1.0, -b2), __dmul_rn(gi, gi)));
        m[i] = mi;
        v[i] = vi;
        const double mh = __ddiv_rn(mi, bc1), vh = __ddiv_rn(vi, bc2);
        theta[i] = __dadd_rn(theta[i], -__ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps)));
    }
}

// One VQE iteration's bookkeeping on the device (lq_vqe_adam's graph path,
// PAPER.md:739-762; stopping rule reading A21): record E_t, decide the stop
// exactly as the host loop does -- non-finite E (state 2), or
// |E_t - E_{t-1}| < tol for t >= 1, or t == max_iter (state 1) -- and
// otherwise take the Adam step with the host-computed bias corrections
// bc[2t], bc[2t+1] (the same _rn arithmetic as k_adam_step).  Once stopped,
// later iterations of the replayed graph leave theta, the trace and the
// counter alone.  One block.
struct VqeCtl {
    int32_t t;        // iteration index
    int32_t state;    // 0 running, 1 stopped, 2 non-finite energy
    double prev;      // E_{t-1}
};
__global__ void k_vqe_step(double *__restrict__ theta, double *__restrict__ m, double *__restrict__ v,
                           const double *__restrict__ g, int n, double lr, double b1, double b2, double eps,
                           double tol, int max_iter, const double *__restrict__ bc, const double *__restrict__ E,
                           double *__restrict__ trace, VqeCtl *__restrict__ ctl) {
    __shared__ int go, t;
    if (threadIdx.x == 0) {
        go = 0;
        t = ctl->t;
        if (ctl->state == 0) {
            const double e = *E;
            trace[t] = e;
            if (!isfinite(e)) ctl->state = 2;
            else if ((t >= 1 && fabs(e - ctl->prev) < tol) || t == max_iter) ctl->state = 1;
            else {
                ctl->prev = e;
                go = 1;
            }
        }
    }
    __syncthreads();
    if (!go) return;
    const double bc1 = bc[2 * t], bc2 = bc[2 * t + 1];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double gi = g[i];
        const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dadd_rn(1.0, -b1), gi));
        const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dadd_rn(1.0, -b2), __dmul_rn(gi, gi)));
        m[i] = mi;
        v[i] = vi;
        const double mh = __ddiv_rn(mi, bc1), vh = __ddiv_rn(vi, bc2);
        theta[i] = __dadd_rn(theta[i], -__ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps)));
    }
    if (threadIdx.x == 0) ctl->t = t + 1;
}

}  // namespace lq
