// tile.cuh -- the fused tile-pass kernel of liblq.
//
// Included by kernels.cuh (nvcc) and embedded verbatim in liblq.so as the
// prelude of JIT-compiled pass programs (NVRTC, jit.cpp): it must compile
// without host headers.  Every dense complex128 gate update is 2-14 FP64
// ops per 32 B of HBM traffic, far below the FP64 ridge, and tcgen05 has no
// FP64 kind: the design target is coalesced 16-byte accesses, enough bytes
// in flight, as many gates per HBM round trip as possible and as few
// instructions per gate as possible.  See DESIGN.md §5, §7.
#pragma once
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#endif
#include "lq_internal.h"

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

// Expectation partial of one tile (a7): with >= 32 threads every warp
// writes its own fixed-order shuffle sum to slot base + tile * W + warp (W =
// warps per tile) -- no barrier; smaller tiles reduce through `red` (block
// tree, W = 1).  Deterministic either way; k_sum_partials adds the slots in
// index order.
__device__ __forceinline__ void expv_partial(double v, double *red, double *slots, uint64_t tile) {
    const int nt = blockDim.x, t = threadIdx.x;
    if (nt >= 32) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if ((t & 31) == 0) slots[tile * (uint64_t)(nt >> 5) + (t >> 5)] = v;
        return;
    }
    __syncthreads();   // all reads of `red` (the tile buffer) are done
    const double r = block_sum(v, red);
    if (t == 0) slots[tile] = r;
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
__host__ __device__ constexpr uint32_t swz(uint32_t x) {
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

template <int V> struct IC { static constexpr int value = V; };

template <int RR, int V = 0>
struct Unroll {
    template <class F>
    __device__ __forceinline__ static void run(F &&f) {
        f(IC<V>());
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

// Scaled rotation lambda * M on one amplitude pair (x: logical bit 0, y:
// logical bit 1); the GKind table of lq_internal.h.  4 DFMA (or 4 DADD) per
// pair; lambda is deferred by the caller.
template <int GK, bool ALT>
__device__ __forceinline__ void g_pair(double2 &x, double2 &y, double p) {
    const double2 X = x, Y = y;
    if constexpr (GK == GK_REAL) {
        if constexpr (!ALT) {   // [[1, -p], [p, 1]]
            x = make_double2(fma(-p, Y.x, X.x), fma(-p, Y.y, X.y));
            y = make_double2(fma(p, X.x, Y.x), fma(p, X.y, Y.y));
        } else {                // [[p, -1], [1, p]]
            x = make_double2(fma(p, X.x, -Y.x), fma(p, X.y, -Y.y));
            y = make_double2(fma(p, Y.x, X.x), fma(p, Y.y, X.y));
        }
    } else if constexpr (GK == GK_IMAG) {
        if constexpr (!ALT) {   // [[1, -ip], [-ip, 1]]
            x = make_double2(fma(p, Y.y, X.x), fma(-p, Y.x, X.y));
            y = make_double2(fma(p, X.y, Y.x), fma(-p, X.x, Y.y));
        } else {                // [[p, -i], [-i, p]]
            x = make_double2(fma(p, X.x, Y.y), fma(p, X.y, -Y.x));
            y = make_double2(fma(p, Y.x, X.y), fma(p, Y.y, -X.x));
        }
    } else {                    // [[1, 1], [1, -1]]
        x = cadd(X, Y);
        y = csub(X, Y);
    }
}

template <int RR, int P, int GK, bool ALT, bool F>
__device__ __forceinline__ void ap_g_(double2 (&a)[1 << RR], double p) {
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if (v & (1 << P)) continue;
        const int w = v | (1 << P);
        if constexpr (!F) g_pair<GK, ALT>(a[v], a[w], p);
        else g_pair<GK, ALT>(a[w], a[v], p);   // flipped: register w holds logical bit 0
    }
}

template <int RR, int P, int GK>
__device__ __forceinline__ void ap_g(double2 (&a)[1 << RR], const double2 *M, bool f) {
    const double p = M[0].x;
    if constexpr (GK == GK_HAD) {
        if (f) ap_g_<RR, P, GK, false, true>(a, p);
        else ap_g_<RR, P, GK, false, false>(a, p);
    } else {
        if (M[1].x != 0.0) {
            if (f) ap_g_<RR, P, GK, true, true>(a, p);
            else ap_g_<RR, P, GK, true, false>(a, p);
        } else {
            if (f) ap_g_<RR, P, GK, false, true>(a, p);
            else ap_g_<RR, P, GK, false, false>(a, p);
        }
    }
}

// RXX / RYY on register positions (P0, P1):
// RXX(t) = cos(t/2) I - i sin(t/2) X(x)X rotates every pair (v, v ^ m),
// m = 2^P0 | 2^P1, by [[c, -is], [-is, c]] = lambda * (GK_IMAG table); RYY
// does the same on the 01<->10 pairs and the opposite rotation on the
// 00<->11 pairs (Y(x)Y|00> = -|11>).  NEG flips the sign of the imaginary
// off-diagonal: [[1, +ip], [+ip, 1]] (variant 0) or [[p, +i], [+i, p]]
// (variant 1).  Register flips (fb) keep the pairing; they swap the RYY
// classes when exactly one of the two bits is flipped.
template <bool ALT, bool NEG>
__device__ __forceinline__ void gg_pair(double2 &x, double2 &y, double p) {
    const double2 X = x, Y = y;
    if constexpr (!ALT) {
        const double q = NEG ? -p : p;
        x = make_double2(fma(q, Y.y, X.x), fma(-q, Y.x, X.y));
        y = make_double2(fma(q, X.y, Y.x), fma(-q, X.x, Y.y));
    } else if constexpr (!NEG) {
        x = make_double2(fma(p, X.x, Y.y), fma(p, X.y, -Y.x));
        y = make_double2(fma(p, Y.x, X.y), fma(p, Y.y, -X.x));
    } else {
        x = make_double2(fma(p, X.x, -Y.y), fma(p, X.y, Y.x));
        y = make_double2(fma(p, Y.x, -X.y), fma(p, Y.y, X.x));
    }
}

template <int RR, int P0, int P1, bool ALT>
__device__ __forceinline__ void ap_gg_(double2 (&a)[1 << RR], double p, bool yy, bool swapc) {
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if (v & (1 << P0)) continue;
        const int w = v ^ ((1 << P0) | (1 << P1));
        const bool same = !((v >> P1) & 1);   // v, w hold 00 / 11 (before flips)
        if (yy && (same != swapc)) gg_pair<ALT, true>(a[v], a[w], p);
        else gg_pair<ALT, false>(a[v], a[w], p);
    }
}

template <int RR, int P0, int P1>
__device__ __forceinline__ void ap_gg(double2 (&a)[1 << RR], const double2 *M, bool yy, uint32_t fb) {
    const double p = M[0].x;
    const bool swapc = (((fb >> P0) ^ (fb >> P1)) & 1) != 0;
    if (M[1].x != 0.0) ap_gg_<RR, P0, P1, true>(a, p, yy, swapc);
    else ap_gg_<RR, P0, P1, false>(a, p, yy, swapc);
}

// Deferred scalars.  The register tile holds
// psi / (tsc * ph):
//   tsc (complex) collects factors identical on every thread of the tile --
//       scaled-rotation lambdas, QFT scales, d0 of register-bit diagonals and
//       diagonal factors on bits outside the tile -- and may stay pending
//       across exchanges; it is applied once, before the store;
//   ph  (complex, unit modulus) collects thread-dependent diagonal factors and
//       is applied before amplitudes move between threads.
struct TState {
    uint32_t fb;       // pending register flip mask
    bool hph;          // ph != 1
    double eacc;       // Pauli-group contributions of this thread
    double2 tsc, ph;
    double2 ttmax;     // QFT twiddle state of the current sub-block (at its largest j)
    double2 ttcur;     // ... and at the last stage applied, j = tj
    int tj;
    uint64_t lg;
    const uint8_t *lpos;   // physical -> logical bit map of the pass (QF_GENERAL stages)
    uint32_t cbase;        // this circuit's offset in the pass's constant op-table bank (JIT, D::CTAB)
    __device__ __forceinline__ void reset() {
        fb = 0;
        hph = false;
        eacc = 0.0;
        tsc = make_double2(1.0, 0.0);
        ph = make_double2(1.0, 0.0);
        ttmax = ttcur = make_double2(1.0, 0.0);
        tj = -1;
        lg = 0;
    }
};

// apply ph (exchange) or tsc * ph (store) to the register tile
template <int RR>
__device__ __forceinline__ void materialize(double2 (&a)[1 << RR], TState &ts, bool with_tsc) {
    if (with_tsc) {
        const double2 s = ts.hph ? cmul(ts.tsc, ts.ph) : ts.tsc;
        if (s.x != 1.0 || s.y != 0.0) {
            if (s.y == 0.0) {
#pragma unroll
                for (int v = 0; v < (1 << RR); v++) a[v] = cscale(a[v], s.x);
            } else {
#pragma unroll
                for (int v = 0; v < (1 << RR); v++) a[v] = cmul(a[v], s);
            }
        }
        ts.tsc = make_double2(1.0, 0.0);
    } else if (ts.hph) {
#pragma unroll
        for (int v = 0; v < (1 << RR); v++) a[v] = cmul(a[v], ts.ph);
    }
    ts.ph = make_double2(1.0, 0.0);
    ts.hph = false;
}

// QFT stage on register position P (see planner.cpp plan_qft).  The
// twiddle of pair (v, w) is tt * W[w]; W[w] depends only on the register
// positions in tdep (logical bits below j), so with tdep known at compile
// time (JIT) the 8 butterflies share 2^|tdep| distinct twiddles and pairs
// with no such bit set use tt itself (W = 1 exactly there).
//
// qi = the register position of logical bit j - 1 when it is in tdep: its
// share of the twiddle is e^{+-i pi 2^(j-1) / 2^j} = +-i exactly, so a pair
// with that bit takes +-i times its partner pattern's twiddle (a swap and a
// sign) instead of another complex multiply: half of the stage's twiddle
// products are free (radix-4 structure of adjacent stages).
template <int RR, int P>
__device__ __forceinline__ void ap_qft(double2 (&a)[1 << RR], double2 tt, const double2 *__restrict__ W,
                                       bool inverse, uint32_t tdep, uint32_t qi) {
#pragma unroll
    for (int v = 0; v < (1 << RR); v++) {
        if (v & (1 << P)) continue;
        const int w = v | (1 << P);
        const bool known = tdep & 0x80u;
        const int lo = (int)(w & tdep & 0x7Fu);
        const int qb = (known && qi < 8u) ? (lo & (1 << qi)) : 0;
        const int lo2 = lo & ~qb;
        double2 tw;
        if (known && lo2 == 0) tw = tt;
        else tw = cmul(tt, W[known ? (lo2 | (1 << P)) : w]);
        if (qb) tw = inverse ? make_double2(tw.y, -tw.x) : make_double2(-tw.y, tw.x);
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
// tt_{k-1} = tt_k^2 (-1)^{bit k-1 of Lt}.  Stages of a forward QFT come in
// descending j, so each continues the recurrence from the previous stage's
// value (one squaring per stage, the same operations in the same order as
// restarting from the head); the inverse's ascending stages restart.
__device__ __forceinline__ double2 qft_thread_twiddle(const KOp &op, uint64_t gbase, int n, TState &ts,
                                                      const uint8_t *lpos) {
    double2 &ttmax = ts.ttmax;
    uint64_t &lg = ts.lg;
    const bool inv = op.flags & QF_INVERSE;
    if (op.flags & QF_HEAD) {
        const int jm = op.b1;
        if (op.flags & QF_LGSET) {
            // lg set by the JIT program (straight-line bit map, no table reads)
        } else if (op.flags & QF_GENERAL) {   // logical bits of this thread's base index
            lg = 0;
            for (uint64_t g = gbase; g; g &= g - 1) {
                const uint32_t l = lpos[__ffsll((long long)g) - 1];
                if (l < 64) lg |= 1ull << l;
            }
        } else {
            lg = (op.flags & QF_REVERSED) ? (__brevll(gbase) >> (64 - n)) : gbase;
        }
        const uint64_t Lt = (jm == 0) ? 0ull : (lg & ((1ull << jm) - 1));
        double s, c;
#ifdef LQ_EXP_NOSINCOS   // timing experiment only: wrong twiddles
        s = ldexp((double)Lt, -jm); c = 1.0 - s;
#else
        sincospi(ldexp((double)Lt, -jm), &s, &c);
#endif
        ttmax = make_double2(c, inv ? -s : s);
        ts.ttcur = ttmax;
        ts.tj = jm;
    }
    const bool cont = ts.tj >= (int)op.qj && ts.tj <= (int)op.b1;
    double2 tt = cont ? ts.ttcur : ttmax;
    for (int k = cont ? ts.tj : op.b1; k > op.qj; k--) {
        tt = cmul(tt, tt);
        if ((lg >> (k - 1)) & 1) tt = make_double2(-tt.x, -tt.y);
    }
    ts.ttcur = tt;
    ts.tj = op.qj;
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
    case K_G: {   // register-controlled scaled rotation (CRY): lambda * M applied in full on the controlled half
        const double p = M[0].x, l = M[0].y;
        const bool alt = M[1].x != 0.0;
        const double one = alt ? p : 1.0, off = alt ? 1.0 : p;
        double2 u00, u01, u10, u11;
        if (op.qj == GK_REAL) {
            u00 = make_double2(l * one, 0); u01 = make_double2(-l * off, 0); u10 = make_double2(l * off, 0); u11 = u00;
        } else if (op.qj == GK_IMAG) {
            u00 = make_double2(l * one, 0); u01 = make_double2(0, -l * off); u10 = u01; u11 = u00;
        } else {
            u00 = make_double2(l, 0); u01 = u00; u10 = u00; u11 = make_double2(-l, 0);
        }
#define CALL_U1(P) ap_u1<RR, P>(a, u00, u01, u10, u11, rcm)
        LQ_SW4(op.r0, CALL_U1)
#undef CALL_U1
        break;
    }
    case K_GG: {   // (normally specialised as C_GG; kept complete for the generic path)
        if constexpr (RR >= 2) {
            const int lo = op.r0 < op.r1 ? op.r0 : op.r1, hi = op.r0 < op.r1 ? op.r1 : op.r0;
            const bool yy = op.flags & GG_YY;
            switch (lo * 4 + hi) {
#define CGG(p0, p1) case p0 * 4 + p1: if (RR > p1) ap_gg<RR, p0, (RR > p1 ? p1 : 1)>(a, M, yy, 0u); break;
            CGG(0, 1) CGG(0, 2) CGG(0, 3) CGG(1, 2) CGG(1, 3) CGG(2, 3)
#undef CGG
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

// One lowered op with its code known at compile time (the interpreter's
// switch and the JIT-generated programs both land here).  op.cmask has
// already been checked by the caller.  Register v holds logical register
// index v ^ fb: X, and CNOT/CCX whose controls are thread constants, only
// toggle fb; other ops read logical bit values through it.
template <int RR, int CODE>
__device__ __forceinline__ void exec_op(double2 (&a)[1 << RR], const KOp &op, const double2 *M, uint64_t gbase,
                                        int n, TState &ts, const ETerm *et) {
    if constexpr (CODE >= C_U1 && CODE < C_U1 + 4) {
        constexpr int P = CODE - C_U1;
        if constexpr (RR > P) {
            const bool f = (ts.fb >> P) & 1;
            const double2 m00 = M[0], m01 = M[1], m10 = M[2], m11 = M[3];
            ap_u1<RR, P>(a, f ? m11 : m00, f ? m10 : m01, f ? m01 : m10, f ? m00 : m11, 0u);
        }
    } else if constexpr (CODE >= C_X && CODE < C_X + 4) {
        ts.fb ^= 1u << (CODE - C_X);
    } else if constexpr (CODE >= C_CX && CODE < C_CX + 16) {
        constexpr int Cc = (CODE - C_CX) / 4, Tt = (CODE - C_CX) % 4;
        if constexpr (RR > Cc && RR > Tt && Cc != Tt) {
            if ((ts.fb >> Cc) & 1) ap_cx_n<RR, Cc, Tt>(a);
            else ap_cx<RR, Cc, Tt>(a);
        }
    } else if constexpr (CODE >= C_D1R && CODE < C_D1R + 4) {
        // register-bit diagonal: d0 joins a deferred scalar, only the
        // logical-bit-1 half is multiplied by d1/d0
        constexpr int P = CODE - C_D1R;
        if constexpr (RR > P) {
            const double2 r = M[2];
            if (op.flags & OF_UNIFORM) ts.tsc = cmul(ts.tsc, M[0]);
            else { ts.ph = cmul(ts.ph, M[0]); ts.hph = true; }
            if ((ts.fb >> P) & 1) {
#pragma unroll
                for (int v = 0; v < (1 << RR); v++)
                    if (!(v & (1 << P))) a[v] = cmul(a[v], r);
            } else {
#pragma unroll
                for (int v = 0; v < (1 << RR); v++)
                    if (v & (1 << P)) a[v] = cmul(a[v], r);
            }
        }
    } else if constexpr (CODE == C_D1T) {   // thread-dependent constant bit: one multiply per thread
        ts.ph = cmul(ts.ph, ((gbase >> op.b0) & 1) ? M[1] : M[0]);
        ts.hph = true;
    } else if constexpr (CODE == C_D1U) {   // bit (and controls) outside the tile: tile-uniform
        ts.tsc = cmul(ts.tsc, ((gbase >> op.b0) & 1) ? M[1] : M[0]);
    } else if constexpr (CODE >= C_G && CODE < C_G + 12) {
        constexpr int GK = (CODE - C_G) / 4, P = (CODE - C_G) % 4;
        if constexpr (RR > P) {
            ap_g<RR, P, GK>(a, M, (ts.fb >> P) & 1);
            if (op.cmask) {   // thread-constant control (CRY): only this thread's amplitudes carry lambda
                ts.ph = cscale(ts.ph, M[0].y);
                ts.hph = true;
            } else {
                ts.tsc = cscale(ts.tsc, M[0].y);
            }
        }
    } else if constexpr (CODE >= C_QFT && CODE < C_QFT + 4) {
        constexpr int P = CODE - C_QFT;
        if constexpr (RR > P) {
            flush_flips<RR>(a, ts.fb);
            const double2 tt = qft_thread_twiddle(op, gbase, n, ts, ts.lpos);
            ap_qft<RR, P>(a, tt, M, op.flags & QF_INVERSE, op.tdep, op.qi);
            if (op.flags & QF_SCALE) ts.tsc = cscale(ts.tsc, 0.70710678118654752440);
        }
    } else if constexpr (CODE == C_DT) {
        // several register-bit diagonals at once: one complex multiply per
        // amplitude (v = 0 is 1), their d0 product joins the tile scalar
        ts.tsc = cmul(ts.tsc, M[0]);
        if (ts.fb == 0) {
#pragma unroll
            for (int v = 1; v < (1 << RR); v++) a[v] = cmul(a[v], M[1 + v]);
        } else {
#pragma unroll
            for (int v = 0; v < (1 << RR); v++) a[v] = cmul(a[v], M[1 + (v ^ ts.fb)]);
        }
    } else if constexpr (CODE >= C_GG && CODE < C_GG + 6) {
        constexpr int PI = CODE - C_GG;
        constexpr int P0 = PI < 3 ? 0 : (PI < 5 ? 1 : 2);
        constexpr int P1 = PI < 3 ? PI + 1 : (PI < 5 ? PI - 1 : 3);
        if constexpr (RR > P1) {
            ap_gg<RR, P0, P1>(a, M, (op.flags & GG_YY) != 0, ts.fb);
            ts.tsc = cscale(ts.tsc, M[0].y);
        }
    } else if constexpr (CODE == C_SCALE) {
        ts.tsc = cscale(ts.tsc, M[0].x);
    } else if constexpr (CODE == C_EXPV) {
        flush_flips<RR>(a, ts.fb);
        // the registers hold psi / (tsc * ph)
        double sc = fma(ts.tsc.x, ts.tsc.x, ts.tsc.y * ts.tsc.y);
        if (ts.hph) sc *= fma(ts.ph.x, ts.ph.x, ts.ph.y * ts.ph.y);
        ts.eacc = fma(sc, expv_group<RR>(a, op.rcm, et + op.mat, op.aux, gbase), ts.eacc);
    } else {
        flush_flips<RR>(a, ts.fb);
        apply_generic<RR>(a, op, M, gbase);
        if (op.type == K_GG) ts.tsc = cscale(ts.tsc, M[0].y);   // the deferred lambda
    }
}

#define LQ_OP_CODES(X)                                                                                    \
    X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17)   \
    X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31) X(32) X(33)     \
    X(34) X(35) X(36) X(37) X(38) X(39) X(40) X(41) X(42) X(43) X(44) X(45) X(46) X(47) X(48) X(49)     \
    X(50) X(51) X(52) X(53) X(54) X(55)

// The interpreter: walks the sub-block's op list in shared memory.
struct InterpProg {
    template <int RR>
    __device__ __forceinline__ static void run(uint32_t /*sub*/, const KSub &sb, uint32_t op0, double2 (&a)[1 << RR],
                                               const KOp *ops, uint64_t gbase, int n, const double2 *tab,
                                               TState &ts, const ETerm *et) {
        ts.ttmax = ts.ttcur = make_double2(1.0, 0.0);
        ts.tj = -1;
        ts.lg = 0;
        for (uint32_t oi = sb.op_begin - op0; oi < sb.op_end - op0; oi++) {
            const KOp op = ops[oi];
            if (op.cmask && (gbase & op.cmask) != op.cmask) continue;
            const double2 *M = tab + op.aux;
            switch (op.code) {
#define LQ_CASE(c) case c: exec_op<RR, c>(a, op, M, gbase, n, ts, et); break;
                LQ_OP_CODES(LQ_CASE)
#undef LQ_CASE
            default: break;
            }
        }
    }
};

// Stage one op's table into shared memory (once per circuit per CTA): a copy
// of the circuit's matrices (M) or of the plan constants (cst); a K_DT table
// is built here from its members' diagonal tables (d0, d1, d1/d0).
__device__ __forceinline__ void stage_table(const KOp &o, double2 *s_tab, const double2 *M, const double2 *cst) {
    if (o.type == K_DT) {
        double2 T[16], D0 = make_double2(1.0, 0.0);
        for (int v = 0; v < 16; v++) T[v] = make_double2(1.0, 0.0);
        for (int i = 0; i < (int)o.flags; i++) {
            const double2 mem = cst[o.mat + i];   // (register position, table offset)
            const int pos = (int)mem.x;
            const double2 *d = M + (uint32_t)mem.y;
            D0 = cmul(D0, d[0]);
            for (int v = 0; v < 16; v++)
                if ((v >> pos) & 1) T[v] = cmul(T[v], d[2]);
        }
        s_tab[o.aux] = D0;
        for (int v = 0; v < 16; v++) s_tab[o.aux + 1 + v] = T[v];
        return;
    }
    const int sz = op_table_size(o.type);
    const double2 *src = ((o.type == K_QFT || o.type == K_SCALE) ? cst : M) + o.mat;
    for (int e = 0; e < sz; e++) s_tab[o.aux + e] = src[e];
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
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Bulk (TMA) copies of whole contiguous tiles (JIT Desc::BULK): one thread
// arms the buffer's mbarrier with the tile's byte count and issues one
// cp.async.bulk; the others wait on the barrier's phase.  Frees the LSU of
// 2^K per-thread LDGSTS per tile (the 12-bit contiguous QFT pass).
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    // order this CTA's earlier generic-proxy accesses of dst before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done)
                     : "r"(smem_addr(bar)), "r"(parity)
                     : "memory");
}

// Persistent tile kernel.  One CTA per SM walks the
// tiles of all circuits of the launch (tile g = circuit * tiles_per_circ +
// tile).  While it computes tile i out of shared buffer i&1 it streams tile
// i+1 into the other buffer with cp.async (LDGSTS), so HBM reads overlap the
// FP64 work; results go back to HBM with plain 16-byte stores.
// Shared memory: [buf0 2^K][buf1 2^K][staged op tables][ops]...
// Prog executes the ops of one sub-block: InterpProg (op list in shared
// memory) or a JIT-generated straight-line program (jit.cpp).
#define LQ_TILE_PARAMS                                                                                   \
    const __grid_constant__ lq::KPass P, const lq::KSub *__restrict__ subs, const lq::KOp *__restrict__ ops, \
        const lq::KPerm *__restrict__ perms, const lq::KPermTerm *__restrict__ pterms,                      \
        const lq::ETerm *__restrict__ eterms, const double2 *__restrict__ mats, uint64_t mat_stride,        \
        const double2 *__restrict__ cst, double2 *__restrict__ state, uint64_t state_stride,                 \
        uint32_t tiles_log2, uint32_t total_tiles, double *__restrict__ partials, uint64_t slot_stride,       \
        double2 *__restrict__ state_out
// state_out: where a relabelling out-of-place pass (JIT Desc::OOP, PlanPass::oop) stores the state in the
// next frame; every other pass updates `state` in place and ignores it
#define LQ_TILE_ARGS \
    P, subs, ops, perms, pterms, eterms, mats, mat_stride, cst, state, state_stride, tiles_log2, total_tiles, partials, slot_stride

template <int RR, class Prog>
__device__ __forceinline__ void tile_body(const KPass &P, const KSub *__restrict__ subs,
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
                stage_table(o, s_tab, M, cst);
            }
            cur_circ = circ;
        }
        cp_async_wait1();
        __syncthreads();

        const uint64_t tb = tile_base(g);
        if (zero && (tb | P.gofs) != 0 && !(P.flags & PF_EXPV)) {   // an all-zero tile (tile_body_static)
            if (!(P.flags & PF_NO_STORE)) {
                Mapping<RR> st;
                st.make(t, P.Sstore, s_dlo, s_dhi, tb);
                double2 *psi = state + (uint64_t)circ * state_stride;
                Unroll<RR>::run([&](auto V) { psi[st.gt + st.template goff<decltype(V)::value>()] = make_double2(0.0, 0.0); });
            }
            __syncthreads();
            continue;
        }
        double2 a[NV];
        Mapping<RR> cur;
        KSub sb = s_sub[0];
        cur.make(t, sb.S, s_dlo, s_dhi, tb);
        uint32_t cur_m = smask<RR>(sb.S);
        // registers <- buffer (through the entry permutation, if any)
        auto load_regs = [&](int perm, const uint8_t *S) {
            if (perm >= 0) {
                PermSlots<RR> ps;
                ps.make(cur, S, K, s_perm[perm], binv_of(perm, tb | P.gofs));
                Unroll<RR>::run([&](auto V) { a[decltype(V)::value] = b[ps.template sidx<decltype(V)::value>()]; });
            } else {
                Unroll<RR>::run([&](auto V) { a[decltype(V)::value] = b[cur.template sidx<decltype(V)::value>()]; });
            }
        };
        if (zero) {   // |0...0>: amplitude 1 where the source position is local 0 of tile 0
            if (sb.perm >= 0) {
                PermSlots<RR> ps;
                ps.make(cur, sb.S, K, s_perm[sb.perm], binv_of(sb.perm, tb | P.gofs));
                Unroll<RR>::run([&](auto V) {
                    a[decltype(V)::value] = make_double2(((tb | P.gofs) == 0 && ps.template sidx<decltype(V)::value>() == 0) ? 1.0 : 0.0, 0.0);
                });
            } else {
                Unroll<RR>::run([&](auto V) {
                    a[decltype(V)::value] = make_double2(((tb | P.gofs) == 0 && cur.template sidx<decltype(V)::value>() == 0) ? 1.0 : 0.0, 0.0);
                });
            }
        } else {
            load_regs(sb.perm, sb.S);
        }
        TState ts;
        ts.reset();
        ts.lpos = P.lpos;
        for (uint32_t s = P.sub_begin; s < P.sub_end; s++) {
            if (s != P.sub_begin) {
                sb = s_sub[s - P.sub_begin];
                const uint32_t m = smask<RR>(sb.S);
                if (m != cur_m || sb.perm >= 0) {
                    materialize<RR>(a, ts, false);
                    __syncthreads();   // everyone has read the previous mapping's slots
                    const uint32_t adj = cur.soff_dyn(ts.fb);
                    Unroll<RR>::run([&](auto V) { b[cur.template sidx<decltype(V)::value>() ^ adj] = a[decltype(V)::value]; });
                    ts.fb = 0;
                    __syncthreads();
                    cur.make(t, sb.S, s_dlo, s_dhi, tb);
                    cur_m = m;
                    load_regs(sb.perm, sb.S);
                }
            }
            Prog::template run<RR>(s - P.sub_begin, sb, P.op_begin, a, s_ops, cur.gt | P.gofs, P.n, s_tab, ts, s_et);
        }
        double2 *psi = state + (uint64_t)circ * state_stride;
        if (P.flags & PF_EXPV)     // deterministic partials: one per warp of the tile
            expv_partial(ts.eacc, reinterpret_cast<double *>(b), partials + (uint64_t)circ * slot_stride + P.eslot,
                         g & ((1u << tiles_log2) - 1));
        if (P.flags & PF_NO_STORE) {
            __syncthreads();
            continue;
        }
        materialize<RR>(a, ts, true);
        const uint32_t ms = smask<RR>(P.Sstore);
        if (P.flags & PF_RELABEL) {   // no exchange: registers to the Sstore mapping's positions
            flush_flips<RR>(a, ts.fb);
            cur.make(t, P.Sstore, s_dlo, s_dhi, tb);
        } else if (__syncthreads_or(ms != cur_m || ts.fb != 0 || P.store_perm >= 0)) {
            // a non-zero flip mask would scatter the lanes of each store: go
            // through shared memory (collective decision: the exchange syncs)
            const uint32_t adj = cur.soff_dyn(ts.fb);
            Unroll<RR>::run([&](auto V) { b[cur.template sidx<decltype(V)::value>() ^ adj] = a[decltype(V)::value]; });
            ts.fb = 0;
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



// ---------------------------------------------------------------- static skeleton (JIT)
// tile_body_static<RR, D, Prog> is tile_body with the pass's layout known at
// compile time.  D (generated by jit.cpp) holds K, NSUB; SM[s] = local
// register-bit mask of sub-block s; PERM[s] = entry permutation (-1: none);
// SSTORE, STORE_PERM; and generated functions dep(l) (local index ->
// physical bits), tbase(g) (tile index -> the physical bits outside the
// tile), ainv<p>(l) and binv<p>(tile base) (permutation p's inverse map and
// its tile-dependent translation), and swz(x), the pass's shared-memory
// swizzle: x ^ (a GF(2)-linear function of x >> 3 into the low 3 bits), chosen
// by jit.cpp so that the 8 lanes of every quarter-warp hit distinct 16-byte
// bank groups in every exchange of the pass.  Every shared-memory slot offset and global offset
// of a register then folds to a constant; per tile only the tile base, one
// XOR per register access and one add per global address remain.
__host__ __device__ constexpr int nth_set_bit(uint32_t m, int i) {
    for (int b = 0; b < 32; b++)
        if ((m >> b) & 1) {
            if (i == 0) return b;
            i--;
        }
    return 0;
}
template <uint32_t SMm>
__host__ __device__ constexpr uint32_t loff_c(uint32_t v) {   // register index -> local offset
    uint32_t o = 0;
    for (int i = 0; i < 4; i++)
        if ((v >> i) & 1) o |= 1u << nth_set_bit(SMm, i);
    return o;
}
template <uint32_t SMm, int K>
__device__ __forceinline__ uint32_t ins_zeros(uint32_t t) {   // thread -> local index of register 0
#pragma unroll
    for (int b = 0; b < K; b++)
        if ((SMm >> b) & 1) t = ((t >> b) << (b + 1)) | (t & ((1u << b) - 1u));
    return t;
}
// The dynamic shared memory base (both tile buffers, then the tables).  The
// swizzled accesses below index it with (base | boff) ^ offset, boff = the
// buffer's element offset (0 or 2^K, above every slot bit), so a slot costs
// one XOR and one LEA with the buffer choice folded into the per-exchange base.
__device__ __forceinline__ double2 *dyn_smem() {
    extern __shared__ double2 lq_dyn_smem[];
    return lq_dyn_smem;
}

// registers -> shared slots of mapping SMm (pending flips folded into the address).
// ADD: identity layout (an additive epoch, jit.cpp): slot = the thread's base
// plus a compile-time register offset, so each store is [base + immediate].
template <int RR, class D, uint32_t SMm, bool ADD = false>
__device__ __forceinline__ void xwrite_c(double2 *b, const double2 (&a)[1 << RR], uint32_t t, uint32_t fb) {
    if constexpr (ADD) {
        double2 *p = b + ins_zeros<SMm, D::K>(t);
        if (fb == 0) {
            Unroll<RR>::run([&](auto V) { p[loff_c<SMm>(decltype(V)::value)] = a[decltype(V)::value]; });
        } else {
            const uint32_t adj = loff_c<SMm>(fb);   // register v holds logical v ^ fb
            Unroll<RR>::run([&](auto V) { p[loff_c<SMm>(decltype(V)::value) ^ adj] = a[decltype(V)::value]; });
        }
        return;
    }
    const uint32_t slt = D::swz(ins_zeros<SMm, D::K>(t));
    uint32_t adj = 0;
#pragma unroll
    for (int i = 0; i < RR; i++)
        if ((fb >> i) & 1) adj ^= D::swz(1u << nth_set_bit(SMm, i));
    double2 *const s0 = dyn_smem();
    const uint32_t base = (slt ^ adj) | (uint32_t)(b - s0);
    Unroll<RR>::run([&](auto V) {
        constexpr uint32_t so = D::swz(loff_c<SMm>(decltype(V)::value));
        s0[base ^ so] = a[decltype(V)::value];
    });
}
// shared slots -> registers of mapping SMm, through entry permutation PI
// (ZERO: synthesise |0...0> -- amplitude 1 at position 0 of tile 0)
template <int RR, class D, uint32_t SMm, int PI, bool ZERO, bool ADD = false>
__device__ __forceinline__ void xread_c(const double2 *b, double2 (&a)[1 << RR], uint32_t t, uint64_t tb,
                                        uint64_t gofs) {
    const uint32_t lt = ins_zeros<SMm, D::K>(t);
    if constexpr (ADD && !ZERO) {   // identity layout, no permutation (an additive epoch)
        static_assert(PI < 0, "additive epochs read through no permutation");
        const double2 *p = b + lt;
        Unroll<RR>::run([&](auto V) { a[decltype(V)::value] = p[loff_c<SMm>(decltype(V)::value)]; });
        return;
    }
    const double2 *const s0 = dyn_smem();
    const uint32_t boff = (uint32_t)(b - s0);
    if constexpr (PI < 0) {
        const uint32_t base = D::swz(lt);
        Unroll<RR>::run([&](auto V) {
            constexpr uint32_t so = D::swz(loff_c<SMm>(decltype(V)::value));
            if constexpr (ZERO) a[decltype(V)::value] = make_double2(((tb | gofs) == 0 && (base ^ so) == 0) ? 1.0 : 0.0, 0.0);
            else a[decltype(V)::value] = s0[(base | boff) ^ so];
        });
    } else {
        const uint32_t base = D::swz(D::template ainv<PI>(lt) ^ D::template binv<PI>(tb | gofs));
        Unroll<RR>::run([&](auto V) {
            constexpr uint32_t so = D::swz(D::template ainv<PI>(loff_c<SMm>(decltype(V)::value)));
            if constexpr (ZERO) a[decltype(V)::value] = make_double2(((tb | gofs) == 0 && (base ^ so) == 0) ? 1.0 : 0.0, 0.0);
            else a[decltype(V)::value] = s0[(base | boff) ^ so];
        });
    }
}

template <int RR, class D, class Prog, int S>
__device__ __forceinline__ void run_subs_c(double2 (&a)[1 << RR], double2 *b, TState &ts, uint64_t tb, uint64_t gofs,
                                           uint32_t t, const double2 *tab, const ETerm *et, int n, bool zero) {
    if constexpr (S < D::NSUB) {
        if constexpr (S > 0 && (D::SM[S] != D::SM[S - 1] || D::PERM[S] >= 0)) {
            // The buffer still holds the register contents (jit.cpp RO: only
            // Pauli groups since it was filled), so the new mapping reads it
            // directly -- no write-back, no barrier -- unless the pass never
            // loaded it (PF_LOAD_ZERO).
            if constexpr (D::RO[S - 1]) {
                xread_c<RR, D, D::SM[S], D::PERM[S], false, D::RADD[S]>(b, a, t, tb, gofs);
            } else {
                materialize<RR>(a, ts, false);
                // everyone has read the previous mapping's slots -- needed only
                // if this thread's writes can reach slots another thread reads
                if constexpr (!D::WSAFE[S - 1]) __syncthreads();
                xwrite_c<RR, D, D::SM[S - 1], D::WADD[S - 1]>(b, a, t, ts.fb);
                ts.fb = 0;
                __syncthreads();
                xread_c<RR, D, D::SM[S], D::PERM[S], false, D::RADD[S]>(b, a, t, tb, gofs);
            }
        }
        const uint64_t gbase = tb | gofs | D::dep(ins_zeros<D::SM[S], D::K>(t));
        Prog::template run<S, RR>(a, gbase, n, tab, ts, et);
        run_subs_c<RR, D, Prog, S + 1>(a, b, ts, tb, gofs, t, tab, et, n, zero);
    }
}

template <int RR, class D, class Prog>
__device__ __forceinline__ void tile_body_static(const KPass &P, const KOp *__restrict__ ops,
                                                 const ETerm *__restrict__ eterms, const double2 *__restrict__ mats,
                                                 uint64_t mat_stride, const double2 *__restrict__ cst,
                                                 double2 *__restrict__ state, uint64_t state_stride,
                                                 uint32_t tiles_log2, uint32_t total_tiles,
                                                 double *__restrict__ partials, uint64_t slot_stride,
                                                 double2 *__restrict__ state_out) {
    extern __shared__ double2 sm[];
    constexpr int K = D::K;
    // the store frame (D::OOP: the next pass's frame in the other buffer,
    // D::sdep / D::stbase = the pass's bit permutation applied to dep / tbase;
    // otherwise the same addresses in place)
    double2 *const store_base = D::OOP ? state_out : state;
    constexpr int NV = 1 << RR;
    constexpr uint32_t TS = 1u << K;
    constexpr uint32_t NT = 1u << (K - RR);
    constexpr int LAST = D::NSUB - 1;
    const uint32_t t = threadIdx.x;
    double2 *s_tab = sm + 2 * TS;
    ETerm *s_et = reinterpret_cast<ETerm *>(s_tab + P.smat);
    const uint32_t nops = P.op_end - P.op_begin;
    const uint32_t net = P.eterm_end - P.eterm_begin;
    for (uint32_t k = t; k < net; k += blockDim.x) s_et[k] = eterms[P.eterm_begin + k];
    const bool zero = P.flags & PF_LOAD_ZERO;
    const uint64_t dep_t = D::dep(t);
    const uint32_t sw_t = D::swz(t);
    const uint32_t tmask = (1u << tiles_log2) - 1u;
    // BULK: a contiguous tile (bits 0..K-1) filled in the identity layout is
    // one 2^K * 16-byte block of HBM -- one TMA bulk copy per tile
    __shared__ __align__(8) uint64_t s_bar[2];
    if constexpr (D::BULK) {
        if (t == 0) {
            mbar_init(&s_bar[0], 1);
            mbar_init(&s_bar[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
    }
    auto issue = [&](uint32_t g, double2 *buf) {
        if constexpr (D::BULK) {
            if (t == 0)
                bulk_load(buf, state + (uint64_t)(g >> tiles_log2) * state_stride + D::tbase(g & tmask), TS * 16u,
                          &s_bar[buf == sm ? 0 : 1]);
            return;
        }
        const uint64_t tbg = D::tbase(g & tmask);
        const double2 *psi = state + (uint64_t)(g >> tiles_log2) * state_stride + tbg + dep_t;
        // UMASK (zero-first plans, lq_api.cu prepare()): the state is zero at
        // every index with a bit outside UMASK and HBM holds garbage there --
        // write zeros into those slots instead of loading them
        const bool tok = D::UMASK == ~0ull || ((tbg | dep_t) & ~D::UMASK) == 0;
        Unroll<RR>::run([&](auto V) {
            constexpr uint32_t l = (uint32_t)decltype(V)::value * NT;
            constexpr uint64_t o = D::dep(l);
            double2 *dst = D::ADD_F ? buf + t + l : buf + (sw_t ^ D::swz(l));
            if constexpr ((o & ~D::UMASK) != 0) {
                *dst = make_double2(0.0, 0.0);
            } else {
                if (tok) cp_async16(dst, psi + o);
                else *dst = make_double2(0.0, 0.0);
            }
        });
    };
    uint32_t g = blockIdx.x;
    if (g >= total_tiles) return;
    if (!zero) issue(g, sm);
    cp_async_commit();
    int cur_circ = -1;
    // LATE (constant op tables): the next tile's prefetch is
    // issued right after the barrier that starts this tile -- every thread has
    // then finished the previous tile, whose buffer the prefetch refills -- so
    // no barrier is needed at the end of a tile.
    constexpr bool LATE = D::CTAB;
    for (uint32_t i = 0; g < total_tiles; i++, g += gridDim.x) {
        const uint32_t gn = g + gridDim.x;
        double2 *b = sm + (i & 1) * TS;
        if constexpr (!LATE) {
            if (gn < total_tiles && !zero) issue(gn, sm + ((i + 1) & 1) * TS);
            cp_async_commit();
        }
        const int circ = (int)(g >> tiles_log2);
        if constexpr (!D::CTAB) {
            if (circ != cur_circ) {   // (re)stage this circuit's op tables
                const double2 *M = mats + (uint64_t)circ * mat_stride;
                if constexpr (D::FLAT) {   // staged by k_stage_ctab: one flat block of P.smat entries
                    for (uint32_t k = t; k < P.smat; k += blockDim.x) s_tab[k] = M[k];
                } else {
                    for (uint32_t k = t; k < nops; k += blockDim.x) stage_table(ops[P.op_begin + k], s_tab, M, cst);
                }
                cur_circ = circ;
            }
        }
        if constexpr (D::BULK) {
            if (!zero) mbar_wait(&s_bar[i & 1], (i >> 1) & 1u);   // fill i>>1 of buffer i&1
        } else if constexpr (LATE) {
            cp_async_wait0();
        } else {
            cp_async_wait1();
        }
        __syncthreads();
        if constexpr (LATE) {
            if (gn < total_tiles && !zero) issue(gn, sm + ((i + 1) & 1) * TS);
            cp_async_commit();
        }

        const uint64_t tb = D::tbase(g & tmask);
        if (D::ZSKIP && zero && (tb | P.gofs) != 0 && !(P.flags & PF_EXPV)) {
            // |0...0> lives in tile 0 and the pass's ops act inside a tile:
            // every other tile is zero before and after the pass -- store
            // zeros, skip the arithmetic (CTA-uniform branch)
            if (!(P.flags & PF_NO_STORE)) {
                double2 *psi = store_base + (uint64_t)circ * state_stride;
                const uint64_t gst = D::stbase(g & tmask) | D::sdep(ins_zeros<D::SSTORE, K>(t));
                Unroll<RR>::run([&](auto V) {
                    constexpr uint64_t go = D::sdep(loff_c<D::SSTORE>(decltype(V)::value));
                    psi[gst + go] = make_double2(0.0, 0.0);
                });
            }
            if constexpr (!LATE) __syncthreads();
            continue;
        }
        // CIRC: the launch's circuit index as a compile-time value (D::NCIRC
        // copies of the body, chosen by a CTA-uniform branch), so the op-table
        // offsets fold into immediate constant-bank operands; -1: runtime
        auto body = [&](auto CV) {
            constexpr int CIRC = decltype(CV)::value;
            double2 a[NV];
            if (zero) xread_c<RR, D, D::SM[0], D::PERM[0], true>(b, a, t, tb, P.gofs);
            else xread_c<RR, D, D::SM[0], D::PERM[0], false, D::RADD[0]>(b, a, t, tb, P.gofs);
            TState ts;
            ts.reset();
            ts.lpos = P.lpos;
            ts.cbase = CIRC >= 0 ? (uint32_t)CIRC * D::SMAT : (uint32_t)circ * D::SMAT;
            run_subs_c<RR, D, Prog, 0>(a, b, ts, tb, P.gofs, t, s_tab, s_et, P.n, zero);
            double2 *psi = store_base + (uint64_t)circ * state_stride;
            if (P.flags & PF_EXPV)     // deterministic partials: one per warp of the tile
                expv_partial(ts.eacc, reinterpret_cast<double *>(b), partials + (uint64_t)circ * slot_stride + P.eslot,
                             g & tmask);
            if (P.flags & PF_NO_STORE) {
                if constexpr (!LATE) __syncthreads();
                return;
            }
            materialize<RR>(a, ts, true);
            // RELABEL (PF_RELABEL): no store exchange -- the registers go to
            // the SSTORE mapping's positions, a local-bit permutation the
            // plan absorbed into the qubit map
            constexpr bool need_x = !D::RELABEL && (D::SSTORE != D::SM[LAST] || D::STORE_PERM >= 0);
            bool ex = need_x;
            if constexpr (D::RELABEL) flush_flips<RR>(a, ts.fb);
            else if constexpr (!need_x) ex = __syncthreads_or(ts.fb != 0);
            if (ex) {
                if constexpr (need_x && !D::WSAFE[LAST]) __syncthreads();
                xwrite_c<RR, D, D::SM[LAST], D::ADD_S>(b, a, t, ts.fb);
                __syncthreads();
                xread_c<RR, D, D::SSTORE, D::STORE_PERM, false, D::ADD_S>(b, a, t, tb, P.gofs);
            }
            const uint64_t gst = (D::OOP ? D::stbase(g & tmask) : tb) | D::sdep(ins_zeros<D::SSTORE, K>(t));
            Unroll<RR>::run([&](auto V) {
                constexpr uint64_t go = D::sdep(loff_c<D::SSTORE>(decltype(V)::value));
                psi[gst + go] = a[decltype(V)::value];
            });
            if constexpr (!LATE) __syncthreads();   // buffer b is refilled by the next iteration's prefetch
        };
        if constexpr (D::CTAB && D::NCIRC >= 1 && D::NCIRC <= 4) {
            if (D::NCIRC == 1 || circ == 0) body(IC<0>());
            else if (D::NCIRC == 2 || circ == 1) body(IC<(D::NCIRC > 1 ? 1 : 0)>());
            else if (D::NCIRC == 3 || circ == 2) body(IC<(D::NCIRC > 2 ? 2 : 0)>());
            else body(IC<(D::NCIRC > 3 ? 3 : 0)>());
        } else {
            body(IC<-1>());
        }
    }
}

template <int RR>
__global__ void __launch_bounds__(RR >= 4 ? 256 : 512, 1) k_tile(LQ_TILE_PARAMS) {
    tile_body<RR, InterpProg>(LQ_TILE_ARGS);   // in place only (the planner's oop passes are JIT-only)
}

}  // namespace lq
