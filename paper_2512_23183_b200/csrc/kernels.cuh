// kernels.cuh -- sm_100a kernels of liblq (included once, by lq_api.cu).
//
// All kernels are HBM-streaming FP64 kernels: a dense complex128 gate update
// is 6-14 flop per 32 B of traffic, far below the
// FP64 ridge, and tcgen05 has no FP64 kind, so the design target is
// coalesced 16-byte accesses, enough bytes in flight, and as many gates per
// HBM round trip as possible (tile passes).  See DESIGN.md §4 for the
// roofline of each kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "lq_internal.h"
#include "../../include/lq.h"

namespace lq {

// ---------------------------------------------------------------- complex
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a*b + c
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// Deterministic block reduction (fixed shuffle tree + fixed smem tree).
// red: >= max(32, blockDim.x) doubles of shared memory.  blockDim.x must be
// a power of two.  Result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double *red) {
    const int nt = blockDim.x, t = threadIdx.x;
    if (nt >= 32) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        const int w = t >> 5, l = t & 31;
        if (l == 0) red[w] = v;
        __syncthreads();
        double r = 0.0;
        if (w == 0) {
            r = (l < (nt >> 5)) ? red[l] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
        }
        __syncthreads();
        return r;
    }
    red[t] = v;
    __syncthreads();
    for (int s = nt >> 1; s > 0; s >>= 1) {
        if (t < s) red[t] += red[t + s];
        __syncthreads();
    }
    double r = red[0];
    __syncthreads();
    return r;
}

// In-place register swap the compiler cannot turn into a renaming (a
// renaming would force loop-carried copies of the whole register tile).
__device__ __forceinline__ void swap_inplace(double2 &x, double2 &y) {
    asm volatile("{\n\t.reg .f64 t;\n\tmov.f64 t, %0;\n\tmov.f64 %0, %2;\n\tmov.f64 %2, t;\n\t"
                 "mov.f64 t, %1;\n\tmov.f64 %1, %3;\n\tmov.f64 %3, t;\n\t}"
                 : "+d"(x.x), "+d"(x.y), "+d"(y.x), "+d"(y.y));
}

__device__ __forceinline__ uint64_t insert_zero64(uint64_t x, int b) {
    uint64_t lo = x & ((1ull << b) - 1);
    return ((x ^ lo) << 1) | lo;
}
__device__ __forceinline__ uint32_t insert_zero32(uint32_t x, int b) {
    uint32_t lo = x & ((1u << b) - 1);
    return ((x ^ lo) << 1) | lo;
}

// ---------------------------------------------------------------- tile kernel
// Shared-memory index swizzle for the 16-byte exchange buffer: XOR-folds the
// higher 3-bit groups into the bank-group bits (idx mod 8), so the 8 lanes
// of a quarter warp hit distinct bank groups whenever the lowest three
// non-register local bits have distinct residues mod 3.  GF(2)-linear, so
// swz(a ^ b) = swz(a) ^ swz(b).
__device__ __forceinline__ uint32_t swz(uint32_t x) {
    return x ^ (((x >> 3) ^ (x >> 6) ^ (x >> 9) ^ (x >> 12)) & 7u);
}

// Register mapping of a sub-block: thread t holds the 2^RR amplitudes with
// local index lt + loff(v), loff(v) = sum_{i: v_i} 2^{S[i]}; global index
// gt + goff(v), goff(v) = sum_{i: v_i} 2^{T[S[i]]}.  Shared-memory slots
// are swizzled: slot = swz(lt) ^ swz(loff(v)).
template <int RR>
struct Mapping {
    uint32_t lt;         // local index of v = 0
    uint32_t slt;        // shared-memory slot of v = 0 (plain, used for writes)
    uint32_t slm[RR];    // slot offsets (XOR) of the register bits
    uint64_t gt;         // global index of v = 0
    uint64_t gm[RR];     // global offsets of the register bits
    // dep: deposit tables of the local->global bit map (dep[0][l & 255] |
    // dep[1][l >> 8] = the global bits of local index l)
    __device__ __forceinline__ void make(uint32_t t, const uint8_t *S, const uint64_t *dlo, const uint64_t *dhi,
                                         uint64_t tb) {
        uint32_t l = t;
#pragma unroll
        for (int i = 0; i < RR; i++) l = insert_zero32(l, S[i]);
        lt = l;
        gt = tb | dlo[l & 255] | dhi[l >> 8];
        slt = swz(l);
#pragma unroll
        for (int i = 0; i < RR; i++) {
            slm[i] = swz(1u << S[i]);
            gm[i] = S[i] < 8 ? dlo[1u << S[i]] : dhi[1u << (S[i] - 8)];
        }
    }
    template <int V>
    __device__ __forceinline__ uint32_t sidx() const {
        uint32_t o = slt;
#pragma unroll
        for (int i = 0; i < RR; i++)
            if (V & (1 << i)) o ^= slm[i];
        return o;
    }
    // slot offset of a runtime register index u (folds the flip mask)
    __device__ __forceinline__ uint32_t soff_dyn(uint32_t u) const {
        uint32_t o = 0;
#pragma unroll
        for (int i = 0; i < RR; i++)
            if ((u >> i) & 1) o ^= slm[i];
        return o;
    }
    template <int V>
    __device__ __forceinline__ uint64_t goff() const {
        uint64_t o = 0;
#pragma unroll
        for (int i = 0; i < RR; i++)
            if (V & (1 << i)) o |= gm[i];
        return o;
    }
};

// Read slots of a mapping through an entry permutation: register slot l
// reads position P^-1(l) = Ainv l + binv.
template <int RR>
struct PermSlots {
    uint32_t slt, slm[RR];
    __device__ __forceinline__ void make(const Mapping<RR> &m, const uint8_t *S, int K, const KPerm &pm,
                                         uint32_t binv) {
        uint32_t lp = binv;
        for (int i = 0; i < K; i++)
            if ((m.lt >> i) & 1) lp ^= pm.col[i];
        slt = swz(lp);
#pragma unroll
        for (int i = 0; i < RR; i++) slm[i] = swz(pm.col[S[i]]);
    }
    template <int V>
    __device__ __forceinline__ uint32_t sidx() const {
        uint32_t o = slt;
#pragma unroll
        for (int i = 0; i < RR; i++)
            if (V & (1 << i)) o ^= slm[i];
        return o;
    }
};

template <int RR, int V = 0>
struct Unroll {
    template <class F>
    __device__ __forceinline__ static void run(F &&f) {
        f(std::integral_constant<int, V>());
        Unroll<RR, V + 1>::run(f);
    }
};
template <int RR>
struct Unroll<RR, (1 << RR)> {
    template <class F>
    __device__ __forceinline__ static void run(F &&) {}
};

template <int RR, int P>
__device__ __forceinline__ void ap_u1(double2 (&a)[1 << RR], double2 u00, double2 u01, double2 u10,
                                      double2 u11, uint32_t rcm) {
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if (v & (1 << P)) continue;
        if ((v & rcm) != rcm) continue;
        const int w = v | (1 << P);
        double2 x = a[v], y = a[w];
        a[v] = cfma(u00, x, cmul(u01, y));
        a[w] = cfma(u10, x, cmul(u11, y));
    }
}

template <int RR, int P>
__device__ __forceinline__ void ap_x(double2 (&a)[1 << RR], uint32_t rcm) {
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if (v & (1 << P)) continue;
        if ((v & rcm) != rcm) continue;
        const int w = v | (1 << P);
        swap_inplace(a[v], a[w]);
    }
}

template <int RR, int P0, int P1>
__device__ __forceinline__ void ap_u2(double2 (&a)[1 << RR], const double2 *U, uint32_t rcm) {
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if (v & ((1 << P0) | (1 << P1))) continue;
        if ((v & rcm) != rcm) continue;
        const int i0 = v, i1 = v | (1 << P1), i2 = v | (1 << P0), i3 = v | (1 << P0) | (1 << P1);
        double2 x0 = a[i0], x1 = a[i1], x2 = a[i2], x3 = a[i3];
        a[i0] = cfma(U[0], x0, cfma(U[1], x1, cfma(U[2], x2, cmul(U[3], x3))));
        a[i1] = cfma(U[4], x0, cfma(U[5], x1, cfma(U[6], x2, cmul(U[7], x3))));
        a[i2] = cfma(U[8], x0, cfma(U[9], x1, cfma(U[10], x2, cmul(U[11], x3))));
        a[i3] = cfma(U[12], x0, cfma(U[13], x1, cfma(U[14], x2, cmul(U[15], x3))));
    }
}

template <int RR, int P0, int P1>
__device__ __forceinline__ void ap_swap(double2 (&a)[1 << RR], uint32_t rcm) {
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if (v & ((1 << P0) | (1 << P1))) continue;
        if ((v & rcm) != rcm) continue;
        const int i1 = v | (1 << P1), i2 = v | (1 << P0);
        swap_inplace(a[i1], a[i2]);
    }
}

// QFT stage on register position P (see planner.cpp plan_qft).
template <int RR, int P>
__device__ __forceinline__ void ap_qft(double2 (&a)[1 << RR], double2 tt, const double2 *__restrict__ W,
                                       bool inverse) {
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if (v & (1 << P)) continue;
        const int w = v | (1 << P);
        double2 tw = cmul(tt, W[w]);
        if (!inverse) {
            double2 u = a[v], x = a[w];
            a[v] = cadd(u, x);
            a[w] = cmul(csub(u, x), tw);
        } else {
            double2 u = a[v], y = cmul(a[w], tw);
            a[v] = cadd(u, y);
            a[w] = csub(u, y);
        }
    }
}

#define LQ_SW4(r, CALL)                         \
    switch (r) {                                \
    case 0: CALL(0); break;                     \
    case 1: if (RR > 1) CALL((RR > 1 ? 1 : 0)); break; \
    case 2: if (RR > 2) CALL((RR > 2 ? 2 : 0)); break; \
    case 3: if (RR > 3) CALL((RR > 3 ? 3 : 0)); break; \
    default: break;                             \
    }

// QFT thread twiddle exp(+-i pi Lt / 2^j), Lt = logical(gbase) mod 2^j: one
// sincospi per sub-block (at its largest j), then the exact recurrence
// tt_{k-1} = tt_k^2 (-1)^{bit k-1 of Lt}.
__device__ __forceinline__ double2 qft_thread_twiddle(const KOp &op, uint64_t gbase, int n, double2 &ttmax,
                                                      uint64_t &lg) {
    const bool inv = op.flags & QF_INVERSE;
    if (op.flags & QF_HEAD) {
        const int jm = op.b1;
        lg = (op.flags & QF_REVERSED) ? (__brevll(gbase) >> (64 - n)) : gbase;
        const uint64_t Lt = (jm == 0) ? 0ull : (lg & ((1ull << jm) - 1));
        double s, c;
        sincospi(ldexp((double)Lt, -jm), &s, &c);
        ttmax = make_double2(c, inv ? -s : s);
    }
    double2 tt = ttmax;
    for (int k = op.b1; k > op.qj; k--) {
        tt = cmul(tt, tt);
        if ((lg >> (k - 1)) & 1) tt = make_double2(-tt.x, -tt.y);
    }
    return tt;
}

template <int RR, int C, int T>
__device__ __forceinline__ void ap_cx(double2 (&a)[1 << RR]) {
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if ((v & (1 << T)) || !(v & (1 << C))) continue;
        const int w = v | (1 << T);
        swap_inplace(a[v], a[w]);
    }
}

template <int RR, int C, int T>
__device__ __forceinline__ void ap_cx_n(double2 (&a)[1 << RR]) {   // control bit sense inverted
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if ((v & (1 << T)) || (v & (1 << C))) continue;
        const int w = v | (1 << T);
        swap_inplace(a[v], a[w]);
    }
}

// Materialise a pending register flip mask (see apply_ops).
template <int RR>
__device__ __forceinline__ void flush_flips(double2 (&a)[1 << RR], uint32_t &fb) {
    if (fb == 0) return;
#pragma unroll
    for (int p = 0; p < RR; p++)
        if ((fb >> p) & 1) {
#pragma unroll
            for (int v = 0; v < (1 << RR); v++)
                if (!(v & (1 << p))) swap_inplace(a[v], a[v | (1 << p)]);
        }
    fb = 0;
}

// Rare op shapes (register-controlled U1/D1, multi-register controls, U2,
// D2, SWAP): a switch on the op type.
template <int RR>
__device__ __forceinline__ void apply_generic(double2 (&a)[1 << RR], const KOp &op, const double2 *M, uint64_t gbase) {
    const uint32_t rcm = op.rcm;
    switch (op.type) {
    case K_U1: {
        const double2 u00 = M[0], u01 = M[1], u10 = M[2], u11 = M[3];
#define CALL_U1(P) ap_u1<RR, P>(a, u00, u01, u10, u11, rcm)
        LQ_SW4(op.r0, CALL_U1)
#undef CALL_U1
        break;
    }
    case K_X: {
#define CALL_X(P) ap_x<RR, P>(a, rcm)
        LQ_SW4(op.r0, CALL_X)
#undef CALL_X
        break;
    }
    case K_D1: {
        const double2 d0 = M[0], d1 = M[1];
        if (op.r0 != NOREG) {
#pragma unroll
            for (int v = 0; v < (1 << RR); v++) {
                if ((v & rcm) != rcm) continue;
                a[v] = cmul(a[v], ((v >> op.r0) & 1) ? d1 : d0);
            }
        } else {
            const double2 d = ((gbase >> op.b0) & 1) ? d1 : d0;
#pragma unroll
            for (int v = 0; v < (1 << RR); v++) {
                if ((v & rcm) != rcm) continue;
                a[v] = cmul(a[v], d);
            }
        }
        break;
    }
    case K_D2: {
        const uint32_t ha = (op.r0 == NOREG) ? (uint32_t)((gbase >> op.b0) & 1) : 0u;
        const uint32_t hb = (op.r1 == NOREG) ? (uint32_t)((gbase >> op.b1) & 1) : 0u;
#pragma unroll
        for (int v = 0; v < (1 << RR); v++) {
            if ((v & rcm) != rcm) continue;
            uint32_t ia = (op.r0 == NOREG) ? ha : ((v >> op.r0) & 1);
            uint32_t ib = (op.r1 == NOREG) ? hb : ((v >> op.r1) & 1);
            a[v] = cmul(a[v], M[2 * ia + ib]);
        }
        break;
    }
    case K_U2: {
        if constexpr (RR >= 2) {
            const double2 *U = M;   // shared memory: entries are re-read per quad
            const int code = op.r0 * 4 + op.r1;
            switch (code) {
#define CU2(p0, p1) case p0 * 4 + p1: if (RR > p0 && RR > p1) ap_u2<RR, (RR > p0 ? p0 : 0), (RR > p1 ? p1 : 1)>(a, U, rcm); break;
            CU2(0, 1) CU2(1, 0) CU2(0, 2) CU2(2, 0) CU2(0, 3) CU2(3, 0)
            CU2(1, 2) CU2(2, 1) CU2(1, 3) CU2(3, 1) CU2(2, 3) CU2(3, 2)
#undef CU2
            default: break;
            }
        }
        break;
    }
    case K_SWAP: {
        if constexpr (RR >= 2) {
            const int lo = op.r0 < op.r1 ? op.r0 : op.r1, hi = op.r0 < op.r1 ? op.r1 : op.r0;
            const int code = hi * 4 + lo;
            switch (code) {
#define CSW(p0, p1) case p0 * 4 + p1: if (RR > p0) ap_swap<RR, (RR > p0 ? p0 : 1), (RR > p0 ? p1 : 0)>(a, rcm); break;
            CSW(1, 0) CSW(2, 0) CSW(2, 1) CSW(3, 0) CSW(3, 1) CSW(3, 2)
#undef CSW
            default: break;
            }
        }
        break;
    }
    default:
        break;
    }
}

// Pauli-group expectation on the register tile (SURVEY
// §8(a) a7).  For the group's x mask X (register positions) and register
// index v: w_v = conj(a[v ^ X]) a[v]; a term (c, z, y) contributes
//   c (-1)^{popcount(gbase & znr)} Re[ i^y sum_v chi_zreg(v) w_v ].
// sum_v chi_p(v) w_v for all 16 patterns p is one Walsh-Hadamard transform
// of w.  Pairs (v, v ^ X) give conjugate w, so only half are formed.
template <int RR, int X, bool IM>
__device__ __forceinline__ void expv_w(const double2 (&a)[1 << RR], double (&w)[1 << RR]) {
    if constexpr (X == 0) {
#pragma unroll
        for (int v = 0; v < (1 << RR); v++) w[v] = IM ? 0.0 : fma(a[v].x, a[v].x, a[v].y * a[v].y);
    } else {
        constexpr int lowb = X & -X;
#pragma unroll
        for (int v = 0; v < (1 << RR); v++) {
            if (v & lowb) continue;
            const double2 p = a[v ^ X], q = a[v];
            if constexpr (IM) {
                const double im = fma(p.x, q.y, -p.y * q.x);
                w[v] = im;
                w[v ^ X] = -im;
            } else {
                const double r = fma(p.x, q.x, p.y * q.y);
                w[v] = r;
                w[v ^ X] = r;
            }
        }
    }
}

template <int RR>
__device__ __forceinline__ void wht(double (&w)[1 << RR]) {
#pragma unroll
    for (int b = 0; b < RR; b++)
#pragma unroll
        for (int v = 0; v < (1 << RR); v++) {
            if (v & (1 << b)) continue;
            const double x = w[v], y = w[v | (1 << b)];
            w[v] = x + y;
            w[v | (1 << b)] = x - y;
        }
}

template <int RR>
__device__ __forceinline__ double pick(const double (&w)[1 << RR], uint32_t p) {
    double r = 0.0;
#pragma unroll
    for (int v = 0; v < (1 << RR); v++)
        if (p == (uint32_t)v) r = w[v];
    return r;
}

template <int RR, bool IM>
__device__ __forceinline__ double expv_part(const double2 (&a)[1 << RR], uint32_t xreg, const ETerm *et, uint32_t nt,
                                            uint64_t gbase) {
    double w[1 << RR];
    switch (xreg) {
#define EW(X) case X: if constexpr (X < (1 << RR)) expv_w<RR, (X < (1 << RR) ? X : 0), IM>(a, w); break;
    EW(0) EW(1) EW(2) EW(3) EW(4) EW(5) EW(6) EW(7) EW(8) EW(9) EW(10) EW(11) EW(12) EW(13) EW(14) EW(15)
#undef EW
    default: break;
    }
    wht<RR>(w);
    double e = 0.0;
    uint32_t k = 0;
    while (k < nt) {
        const uint32_t z = et[k].zreg;
        double cz = 0.0;
        for (; k < nt && et[k].zreg == z; k++) {
            const ETerm t = et[k];
            if ((bool)(t.y & 1) != IM) continue;
            double c = (__popcll(gbase & t.znr) & 1) ? -t.c : t.c;
            if (t.y & 2) c = -c;
            cz += IM ? -c : c;   // Re[i w] = -Im w, Re[-i w] = Im w
        }
        if (cz != 0.0) e = fma(cz, pick<RR>(w, z), e);
    }
    return e;
}

template <int RR>
__device__ __forceinline__ double expv_group(const double2 (&a)[1 << RR], uint32_t xreg, const ETerm *et, uint32_t nt,
                                             uint64_t gbase) {
    double e = expv_part<RR, false>(a, xreg, et, nt, gbase);
    bool need_im = false;
    for (uint32_t k = 0; k < nt; k++) need_im |= (et[k].y & 1);
    if (need_im) e += expv_part<RR, true>(a, xreg, et, nt, gbase);
    return e;
}

// Apply the ops [ob, oe) of a sub-block to the register tile.
// fb is a pending flip mask over register positions: register v holds the
// amplitude of logical register index v ^ fb.  X, and CNOT/CCX whose
// controls are thread constants, only toggle fb (no data movement); the
// mask is absorbed into the next shared-memory write or global store
// address.  Other ops read logical bit values through fb.
template <int RR>
__device__ __forceinline__ void apply_ops(double2 (&a)[1 << RR], const KOp *ops, uint32_t ob, uint32_t oe,
                                          uint64_t gbase, int n, const double2 *tab, uint32_t &fb,
                                          const ETerm *et, double &eacc) {
    double2 ttmax = make_double2(1.0, 0.0);
    uint64_t lg = 0;
    for (uint32_t oi = ob; oi < oe; oi++) {
        const KOp op = ops[oi];
        if (op.cmask && (gbase & op.cmask) != op.cmask) continue;
        const double2 *M = tab + op.aux;
        const int code = op.code;
        switch (code) {
#define U1C(P)                                                                         \
        case C_U1 + P:                                                                 \
            if (RR > P) {                                                              \
                const bool f = (fb >> P) & 1;                                          \
                const double2 m00 = M[0], m01 = M[1], m10 = M[2], m11 = M[3];          \
                ap_u1<RR, (RR > P ? P : 0)>(a, f ? m11 : m00, f ? m10 : m01,            \
                                            f ? m01 : m10, f ? m00 : m11, 0u);          \
            }                                                                          \
            break;
        U1C(0) U1C(1) U1C(2) U1C(3)
#undef U1C
#define XC(P) case C_X + P: fb ^= 1u << P; break;
        XC(0) XC(1) XC(2) XC(3)
#undef XC
#define CXC(C, T)                                                                      \
        case C_CX + 4 * C + T:                                                         \
            if (RR > C && RR > T) {                                                    \
                if ((fb >> C) & 1) ap_cx_n<RR, (RR > C ? C : 0), (RR > T ? T : 1)>(a);  \
                else ap_cx<RR, (RR > C ? C : 0), (RR > T ? T : 1)>(a);                  \
            }                                                                          \
            break;
        CXC(0, 1) CXC(0, 2) CXC(0, 3) CXC(1, 0) CXC(1, 2) CXC(1, 3)
        CXC(2, 0) CXC(2, 1) CXC(2, 3) CXC(3, 0) CXC(3, 1) CXC(3, 2)
#undef CXC
#define D1C(P)                                                                      \
        case C_D1R + P:                                                             \
            if (RR > P) {                                                           \
                const bool f = (fb >> P) & 1;                                       \
                const double2 d0 = f ? M[1] : M[0], d1 = f ? M[0] : M[1];           \
                _Pragma("unroll") for (int v = 0; v < (1 << RR); v++)              \
                    a[v] = cmul(a[v], ((v >> (RR > P ? P : 0)) & 1) ? d1 : d0);     \
            }                                                                       \
            break;
        D1C(0) D1C(1) D1C(2) D1C(3)
#undef D1C
        case C_D1T: {
            const double2 d = ((gbase >> op.b0) & 1) ? M[1] : M[0];
            if (d.x != 1.0 || d.y != 0.0) {
#pragma unroll
                for (int v = 0; v < (1 << RR); v++) a[v] = cmul(a[v], d);
            }
            break;
        }
#define QC(P)                                                                          \
        case C_QFT + P:                                                                \
            if (RR > P) {                                                              \
                flush_flips<RR>(a, fb);                                                \
                const double2 tt = qft_thread_twiddle(op, gbase, n, ttmax, lg);         \
                ap_qft<RR, (RR > P ? P : 0)>(a, tt, M, op.flags & QF_INVERSE);          \
            }                                                                          \
            break;
        QC(0) QC(1) QC(2) QC(3)
#undef QC
        case C_SCALE: {
            const double sc = M[0].x;
#pragma unroll
            for (int v = 0; v < (1 << RR); v++) a[v] = cscale(a[v], sc);
            break;
        }
        case C_EXPV:
            flush_flips<RR>(a, fb);
            eacc += expv_group<RR>(a, op.rcm, et + op.mat, op.aux, gbase);
            break;
        default:
            flush_flips<RR>(a, fb);
            apply_generic<RR>(a, op, M, gbase);
            break;
        }
    }
}

template <int RR>
__device__ __forceinline__ uint32_t smask(const uint8_t *S) {
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < RR; i++) m |= 1u << S[i];
    return m;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Persistent tile kernel.  One CTA per SM walks the
// tiles of all circuits of the launch (tile g = circuit * tiles_per_circ +
// tile).  While it computes tile i out of shared buffer i&1 it streams tile
// i+1 into the other buffer with cp.async (LDGSTS), so HBM reads overlap the
// FP64 work; results go back to HBM with plain 16-byte stores.
// Shared memory: [buf0 2^K][buf1 2^K][staged op tables][ops].
template <int RR>
__global__ void __launch_bounds__(RR >= 4 ? 256 : 512, 1) k_tile(const __grid_constant__ KPass P, const KSub *__restrict__ subs,
                                                 const KOp *__restrict__ ops, const KPerm *__restrict__ perms,
                                                 const KPermTerm *__restrict__ pterms, const ETerm *__restrict__ eterms,
                                                 const double2 *__restrict__ mats,
                                                 uint64_t mat_stride, const double2 *__restrict__ cst,
                                                 double2 *__restrict__ state, uint64_t state_stride,
                                                 uint32_t tiles_log2, uint32_t total_tiles,
                                                 double *__restrict__ partials, uint64_t slot_stride) {
    extern __shared__ double2 sm[];
    constexpr int NV = 1 << RR;
    const int K = P.K;
    const uint32_t TS = 1u << K;
    const uint32_t NT = 1u << (K - RR);
    const uint32_t t = threadIdx.x;
    double2 *s_tab = sm + 2 * TS;
    KOp *s_ops = reinterpret_cast<KOp *>(s_tab + P.smat);
    const uint32_t nops = P.op_end - P.op_begin;
    const uint32_t nperm = P.perm_end - P.perm_begin;
    KPerm *s_perm = reinterpret_cast<KPerm *>(s_ops + nops);
    const uint32_t pt0 = nperm ? perms[P.perm_begin].term_begin : 0;
    const uint32_t npt = nperm ? perms[P.perm_end - 1].term_end - pt0 : 0;
    KPermTerm *s_pt = reinterpret_cast<KPermTerm *>(s_perm + nperm);
    uint64_t *s_dlo = reinterpret_cast<uint64_t *>(s_pt + npt);
    uint64_t *s_dhi = s_dlo + 256;
    KSub *s_sub = reinterpret_cast<KSub *>(s_dhi + 32);
    const uint32_t nsub = P.sub_end - P.sub_begin;
    const uint32_t net = P.eterm_end - P.eterm_begin;
    ETerm *s_et = reinterpret_cast<ETerm *>(s_sub + nsub + (nsub & 1));   // 8-byte aligned
    for (uint32_t k = threadIdx.x; k < net; k += blockDim.x) s_et[k] = eterms[P.eterm_begin + k];
    const bool zero = P.flags & PF_LOAD_ZERO;
    for (uint32_t k = threadIdx.x; k < 256 + 32; k += blockDim.x) {
        uint64_t g = 0;
        const uint32_t l = k < 256 ? k : (k - 256) << 8;
        for (int i = 0; i < K; i++)
            if ((l >> i) & 1) g |= 1ull << P.T[i];
        s_dlo[k] = g;   // s_dhi = s_dlo + 256
    }
    for (uint32_t k = threadIdx.x; k < P.sub_end - P.sub_begin; k += blockDim.x) s_sub[k] = subs[P.sub_begin + k];
    for (uint32_t k = threadIdx.x; k < nperm; k += blockDim.x) s_perm[k] = perms[P.perm_begin + k];
    for (uint32_t k = threadIdx.x; k < npt; k += blockDim.x) s_pt[k] = pterms[pt0 + k];
    // translation of an entry permutation for this tile
    auto binv_of = [&](int pi, uint64_t tb) {
        uint32_t b = 0;
        const KPerm &pm = s_perm[pi];
        for (uint32_t k = pm.term_begin - pt0; k < pm.term_end - pt0; k++)
            if ((tb & s_pt[k].cmask) == s_pt[k].cmask) b ^= s_pt[k].vec;
        return b;
    };

    // this thread's copy slots: local index l = t + v * NT (top RR bits = v)
    uint64_t dep_t = 0;
    for (int i = 0; i < K - RR; i++)
        if ((t >> i) & 1) dep_t |= 1ull << P.T[i];
    const uint32_t sw_t = swz(t);

    auto tile_base = [&](uint32_t g) {
        uint64_t tb = g & ((1u << tiles_log2) - 1);
        for (int i = 0; i < K; i++) tb = insert_zero64(tb, P.T[i]);
        return tb;
    };
    auto issue = [&](uint32_t g, double2 *buf) {
        const double2 *psi = state + (uint64_t)(g >> tiles_log2) * state_stride + tile_base(g) + dep_t;
        Unroll<RR>::run([&](auto V) {
            constexpr int v = decltype(V)::value;
            uint64_t o = 0;
#pragma unroll
            for (int i = 0; i < RR; i++)
                if (v & (1 << i)) o |= 1ull << P.T[K - RR + i];
            cp_async16(buf + (sw_t ^ swz((uint32_t)v * NT)), psi + o);
        });
    };

    uint32_t g = blockIdx.x;
    if (g >= total_tiles) return;
    if (!zero) issue(g, sm);
    cp_async_commit();
    int cur_circ = -1;
    for (uint32_t i = 0; g < total_tiles; i++, g += gridDim.x) {
        const uint32_t gn = g + gridDim.x;
        double2 *b = sm + (i & 1) * TS;
        if (gn < total_tiles && !zero) issue(gn, sm + ((i + 1) & 1) * TS);
        cp_async_commit();
        const int circ = (int)(g >> tiles_log2);
        if (circ != cur_circ) {   // (re)stage the ops and this circuit's matrices
            const double2 *M = mats + (uint64_t)circ * mat_stride;
            for (uint32_t k = t; k < nops; k += blockDim.x) {
                const KOp o = ops[P.op_begin + k];
                s_ops[k] = o;
                const int sz = op_table_size(o.type);
                const double2 *src = ((o.type == K_QFT || o.type == K_SCALE) ? cst : M) + o.mat;
                for (int e = 0; e < sz; e++) s_tab[o.aux + e] = src[e];
            }
            cur_circ = circ;
        }
        cp_async_wait1();
        __syncthreads();

        const uint64_t tb = tile_base(g);
        double2 a[NV];
        Mapping<RR> cur;
        KSub sb = s_sub[0];
        cur.make(t, sb.S, s_dlo, s_dhi, tb);
        uint32_t cur_m = smask<RR>(sb.S);
        // registers <- buffer (through the entry permutation, if any)
        auto load_regs = [&](int perm, const uint8_t *S) {
            if (perm >= 0) {
                PermSlots<RR> ps;
                ps.make(cur, S, K, s_perm[perm], binv_of(perm, tb));
                Unroll<RR>::run([&](auto V) { a[decltype(V)::value] = b[ps.template sidx<decltype(V)::value>()]; });
            } else {
                Unroll<RR>::run([&](auto V) { a[decltype(V)::value] = b[cur.template sidx<decltype(V)::value>()]; });
            }
        };
        if (zero) {   // |0...0>: amplitude 1 where the source position is local 0 of tile 0
            if (sb.perm >= 0) {
                PermSlots<RR> ps;
                ps.make(cur, sb.S, K, s_perm[sb.perm], binv_of(sb.perm, tb));
                Unroll<RR>::run([&](auto V) {
                    a[decltype(V)::value] = make_double2((tb == 0 && ps.template sidx<decltype(V)::value>() == 0) ? 1.0 : 0.0, 0.0);
                });
            } else {
                Unroll<RR>::run([&](auto V) {
                    a[decltype(V)::value] = make_double2((tb == 0 && cur.template sidx<decltype(V)::value>() == 0) ? 1.0 : 0.0, 0.0);
                });
            }
        } else {
            load_regs(sb.perm, sb.S);
        }
        uint32_t fb = 0;   // pending register flip mask (apply_ops)
        double eacc = 0.0; // Pauli-group contributions of this thread
        for (uint32_t s = P.sub_begin; s < P.sub_end; s++) {
            if (s != P.sub_begin) {
                sb = s_sub[s - P.sub_begin];
                const uint32_t m = smask<RR>(sb.S);
                if (m != cur_m || sb.perm >= 0) {
                    __syncthreads();   // everyone has read the previous mapping's slots
                    const uint32_t adj = cur.soff_dyn(fb);
                    Unroll<RR>::run([&](auto V) { b[cur.template sidx<decltype(V)::value>() ^ adj] = a[decltype(V)::value]; });
                    fb = 0;
                    __syncthreads();
                    cur.make(t, sb.S, s_dlo, s_dhi, tb);
                    cur_m = m;
                    load_regs(sb.perm, sb.S);
                }
            }
            apply_ops<RR>(a, s_ops, sb.op_begin - P.op_begin, sb.op_end - P.op_begin, cur.gt, P.n, s_tab, fb, s_et,
                          eacc);
        }
        double2 *psi = state + (uint64_t)circ * state_stride;
        if (P.flags & PF_EXPV) {   // one deterministic partial per tile
            __syncthreads();       // all reads of b done: reuse it as reduction scratch
            const double r = block_sum(eacc, reinterpret_cast<double *>(b));
            if (t == 0) partials[(uint64_t)circ * slot_stride + P.eslot + (g & ((1u << tiles_log2) - 1))] = r;
        }
        if (P.flags & PF_NO_STORE) {
            __syncthreads();
            continue;
        }
        const uint32_t ms = smask<RR>(P.Sstore);
        // a non-zero flip mask would scatter the lanes of each store: go
        // through shared memory (collective decision: the exchange syncs)
        if (__syncthreads_or(ms != cur_m || fb != 0 || P.store_perm >= 0)) {
            const uint32_t adj = cur.soff_dyn(fb);
            Unroll<RR>::run([&](auto V) { b[cur.template sidx<decltype(V)::value>() ^ adj] = a[decltype(V)::value]; });
            fb = 0;
            __syncthreads();
            cur.make(t, P.Sstore, s_dlo, s_dhi, tb);
            load_regs(P.store_perm, P.Sstore);
        }
        Unroll<RR>::run([&](auto V) {
            psi[cur.gt + cur.template goff<decltype(V)::value>()] = a[decltype(V)::value];
        });
        __syncthreads();   // buffer b is refilled by the next iteration's prefetch
    }
}

// ---------------------------------------------------------------- pair kernel (a4)
// One 1q/2q gate on arbitrary physical bits: strided pairs (i, i | 2^b) or
// quads, 16-byte loads, controls as a bit mask (Alg. 1 generalised).
__global__ void __launch_bounds__(256) k_pair(int n, const KOp op, const double2 *__restrict__ mats,
                                              uint64_t mat_stride, double2 *__restrict__ state,
                                              uint64_t state_stride) {
    double2 *__restrict__ psi = state + (uint64_t)blockIdx.y * state_stride;
    const double2 *__restrict__ M = mats + (uint64_t)blockIdx.y * mat_stride;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (op.type == K_U1 || op.type == K_X) {
        const uint64_t np = 1ull << (n - 1);
        const uint64_t mb = 1ull << op.b0;
        double2 u00 = make_double2(0, 0), u01 = u00, u10 = u00, u11 = u00;
        if (op.type == K_U1) { u00 = M[op.mat]; u01 = M[op.mat + 1]; u10 = M[op.mat + 2]; u11 = M[op.mat + 3]; }
        for (; i < np; i += stride) {
            const uint64_t i0 = insert_zero64(i, op.b0);
            if ((i0 & op.cmask) != op.cmask) continue;
            const uint64_t i1 = i0 | mb;
            double2 x = psi[i0], y = psi[i1];
            if (op.type == K_X) { psi[i0] = y; psi[i1] = x; }
            else { psi[i0] = cfma(u00, x, cmul(u01, y)); psi[i1] = cfma(u10, x, cmul(u11, y)); }
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
            if ((base & op.cmask) != op.cmask) continue;
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
__global__ void __launch_bounds__(256) k_diag(int n, const KOp *__restrict__ ops, int n_ops,
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
        for (int k = 0; k < n_ops; k++) {
            const KOp &o = sop[k];
            if ((i & o.cmask) != o.cmask) continue;
            uint32_t idx = (uint32_t)((i >> o.b0) & 1);
            if (o.type == K_D2) idx = 2 * idx + (uint32_t)((i >> o.b1) & 1);
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
            else { out[0] = A[0]; out[1] = A[3]; }
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

__global__ void __launch_bounds__(256) k_random_norm(uint64_t N, uint64_t seed, double *partial) {
    double acc = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < N; i += (uint64_t)gridDim.x * 256) {
        double2 a = gauss_amp(seed, i);
        acc = fma(a.x, a.x, fma(a.y, a.y, acc));
    }
    __shared__ double red[256];
    double r = block_sum(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = r;
}

__global__ void __launch_bounds__(256) k_random_write(uint64_t N, uint64_t seed, const double *norm2,
                                                      double2 *__restrict__ psi) {
    const double inv = 1.0 / sqrt(*norm2);
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < N; i += (uint64_t)gridDim.x * 256)
        psi[i] = cscale(gauss_amp(seed, i), inv);
}

__global__ void __launch_bounds__(256) k_fill_basis(uint64_t N, uint64_t k, double2 *__restrict__ state,
                                                    uint64_t state_stride) {
    double2 *psi = state + (uint64_t)blockIdx.y * state_stride;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < N; i += (uint64_t)gridDim.x * 256)
        psi[i] = make_double2(i == k ? 1.0 : 0.0, 0.0);
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

__global__ void k_scatter(int n, QMap m, double2 *__restrict__ psi, uint64_t offset, uint64_t count,
                          const double2 *__restrict__ in) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        psi[logical_to_phys(offset + i, n, m)] = in[i];
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
__global__ void __launch_bounds__(256) k_pauli_direct(int n, uint64_t x, const PTerm *__restrict__ terms,
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
            const double c = (__popcll(j & pt.zfull) & 1) ? -pt.coeff : pt.coeff;
            acc = fma(c, re_iy(w, pt.yph), acc);
        }
    }
    __shared__ double red[256];
    double r = block_sum(acc, red);
    if (threadIdx.x == 0) partial[(uint64_t)blockIdx.y * slot_stride + slot + blockIdx.x] = r;
}

// ---------------------------------------------------------------- PSR combine (a8)
// g_p = (E(theta + pi/2 e_p) - E(theta - pi/2 e_p)) / 2
struct PsrPair { int32_t p, plus, minus, pad; };
__global__ void k_psr_combine(const double *__restrict__ E, const PsrPair *__restrict__ pairs, int n_pairs,
                              int base_idx, double *__restrict__ grad, int n_params, double *energy) {
    // launched as ONE block: zero, barrier, then the owned components
    for (int i = threadIdx.x; i < n_params; i += blockDim.x) grad[i] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < n_pairs; i += blockDim.x) {
        const PsrPair pr = pairs[i];
        grad[pr.p] = 0.5 * (E[pr.plus] - E[pr.minus]);
    }
    if (energy && threadIdx.x == 0) *energy = base_idx >= 0 ? E[base_idx] : 0.0;
}

}  // namespace lq
