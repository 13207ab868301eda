// planner.cpp -- host gate-fusion planner.  See planner.h.
#include "planner.h"

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

namespace lq {

static inline int popc(uint64_t x) { return __builtin_popcountll(x); }
static inline uint64_t bit(int b) { return 1ull << b; }

uint64_t POp::full() const {
    switch (type) {
    case K_U1: case K_X: case K_QFT: case K_G: return bit(t0);
    case K_U2: case K_SWAP: case K_GG: return bit(t0) | bit(t1);
    case K_EXPV: return xm;
    default: return 0;
    }
}

uint64_t POp::touch() const {
    uint64_t m = ctrl | full() | rd;
    if (type == K_EXPV) m |= zm;
    if (type == K_D1) m |= bit(t0);
    if (type == K_D2) m |= bit(t0) | bit(t1);
    return m;
}

// Two ops commute if every bit they share is acted on diagonally (as a
// control or a diagonal factor) by both.
bool commute(const POp &a, const POp &b) {
    return (a.full() & b.touch()) == 0 && (b.full() & a.touch()) == 0;
}

int op_fp64_cost(const POp &o) {
    switch (o.type) {
    case K_G: return 20;       // 4 DFMA per amplitude pair
    case K_GG: return 20;      // 4 DFMA per amplitude pair (RXX / RYY)
    case K_U1: return 80;      // general complex 2x2
    case K_U2: return 160;     // general complex 4x4
    case K_D1: return 12;      // register-bit half multiply / table share / thread constant
    case K_D2: return 30;
    case K_QFT: return 50;     // butterfly + twiddle multiply
    case K_EXPV: return 30;    // pair products + Walsh-Hadamard share
    default: return 0;         // X / CNOT / SWAP: folded permutations or flips
    }
}

int MatBuilder::add_spec(MForm form, const std::vector<MFactor> &f) {
    MSpec s;
    s.out = mat_size;
    s.f_begin = (uint32_t)factors.size();
    factors.insert(factors.end(), f.begin(), f.end());
    s.f_end = (uint32_t)factors.size();
    s.form = form;
    static const uint32_t sz[5] = {4, 3, 16, 4, 2};
    mat_size += sz[form];
    specs.push_back(s);
    return (int)specs.size() - 1;
}

int MatBuilder::add_const(const double *v, int n_complex) {
    int off = (int)(cst.size() / 2);
    cst.insert(cst.end(), v, v + 2 * n_complex);
    return off;
}

// K = 11: two 2^11-amplitude tiles (64 KiB double-buffered) per CTA leave room
// for two independent CTAs per SM, which hides shared-memory and FP64 latency
// better than one K = 12 CTA, at ~10 % more passes (measured on B200).
int auto_tile_bits(int n) { return n < 11 ? n : 11; }

// --------------------------------------------------------------------------
// Lowering of user gates (PAPER.md:77-139 operations) to physical-bit ops.
// --------------------------------------------------------------------------
static bool is_1q(int k) { return k <= LQ_RZ || k == LQ_U1; }
static bool is_diag_1q(int k) {
    return k == LQ_Z || k == LQ_S || k == LQ_SDG || k == LQ_T || k == LQ_TDG || k == LQ_RZ;
}

void lower_gates(int n, const lq_gate *gates, size_t n_gates, int32_t *qmap,
                 std::vector<POp> &ops, MatBuilder &mb) {
    std::vector<std::vector<MFactor>> fl;   // factor list per op
    std::vector<int> last(64, -1);          // last op touching each physical bit
    std::vector<char> fusable;              // op is an uncontrolled 1q op
    size_t base = ops.size();
    auto touch_all = [&](int idx) {
        uint64_t m = ops[idx].touch();
        while (m) { int b = __builtin_ctzll(m); last[b] = idx; m &= m - 1; }
    };
    for (size_t g = 0; g < n_gates; g++) {
        const lq_gate &G = gates[g];
        MFactor f{G.kind, G.param_idx, G.angle, -1, 0};
        int k = G.kind;
        if (k == LQ_SWAP) {
            std::swap(qmap[G.q0], qmap[G.q1]);
            continue;
        }
        if (is_1q(k)) {
            if (k == LQ_U1) f.cst = mb.add_const(G.mat, 4);
            int b = qmap[G.q0];
            int prev = last[b];
            const bool dg = is_diag_1q(k) || k == LQ_Y;
            if (k == LQ_Y) f.kind = FK_YDIAG;   // Y = X * diag(i, -i): the diagonal part, then X
            if (dg && prev >= (int)base && fusable[prev - base] && ops[prev].t0 == b && ops[prev].type == K_D1) {
                // no op touched bit b since `prev` (a diagonal op): the diagonal
                // factor joins it.  Non-diagonal 1q gates are NOT fused: two
                // scaled rotations (K_G, 4 DFMA per pair each) are cheaper than
                // one general complex 2x2 (16 FP64 ops per pair).
                fl[prev - base].push_back(f);
            } else {
                POp op;
                op.t0 = b;
                if (dg) op.type = K_D1;
                else if (k == LQ_X) op.type = K_X;
                else if (k == LQ_RY || k == LQ_RX || k == LQ_H) {
                    op.type = K_G;
                    op.qj = (uint8_t)(k == LQ_RY ? GK_REAL : k == LQ_RX ? GK_IMAG : GK_HAD);
                } else op.type = K_U1;
                ops.push_back(op);
                fl.push_back(op.type == K_X ? std::vector<MFactor>{} : std::vector<MFactor>{f});
                fusable.push_back(op.type == K_D1 ? 1 : 0);
                touch_all((int)ops.size() - 1);
            }
            if (k == LQ_Y) {
                POp op;
                op.type = K_X;
                op.t0 = b;
                ops.push_back(op);
                fl.push_back({});
                fusable.push_back(0);
                touch_all((int)ops.size() - 1);
            }
            continue;
        }
        if (k == LQK_QFT_STAGE) {   // Alg. 3 stage as one op (reads the qubits after q0 diagonally)
            POp op;
            op.type = K_QFT;
            op.t0 = qmap[G.q0];
            op.qj = (uint8_t)(n - 1 - G.q0);
            op.qflags = QF_GENERAL | QF_SCALE | (G.angle < 0 ? QF_INVERSE : 0);
            for (int q = G.q0 + 1; q < n; q++) op.rd |= bit(qmap[q]);
            std::vector<uint8_t> lp(64, 255);
            for (int q = 0; q < n; q++) lp[qmap[q]] = (uint8_t)(n - 1 - q);
            int li = -1;
            for (size_t x = 0; x < mb.layouts.size(); x++)
                if (mb.layouts[x] == lp) li = (int)x;
            if (li < 0) { mb.layouts.push_back(lp); li = (int)mb.layouts.size() - 1; }
            op.layout = li;
            ops.push_back(op);
            fl.push_back({});
            fusable.push_back(0);
            touch_all((int)ops.size() - 1);
            continue;
        }
        POp op;
        switch (k) {
        case LQ_CNOT: op.type = K_X; op.t0 = qmap[G.q1]; op.ctrl = bit(qmap[G.q0]); break;
        case LQ_CCX:  op.type = K_X; op.t0 = qmap[G.q2]; op.ctrl = bit(qmap[G.q0]) | bit(qmap[G.q1]); break;
        case LQ_CZ:   op.type = K_D1; op.t0 = qmap[G.q1]; op.ctrl = bit(qmap[G.q0]); f.kind = LQ_Z; break;
        case LQ_CP:   op.type = K_D1; op.t0 = qmap[G.q1]; op.ctrl = bit(qmap[G.q0]); break;
        case LQ_CRY:  // controlled scaled rotation: lambda goes to the controlled threads' phase (tile.cuh)
                      op.type = K_G; op.t0 = qmap[G.q1]; op.ctrl = bit(qmap[G.q0]); f.kind = LQ_RY;
                      op.qj = GK_REAL; break;
        case LQ_U2:   op.type = K_U2; op.t0 = qmap[G.q0]; op.t1 = qmap[G.q1]; f.cst = mb.add_const(G.mat, 16); break;
        case LQ_RXX: case LQ_RYY:   // scaled pair rotation on two register bits (tile.cuh ap_gg)
                      op.type = K_GG; op.t0 = qmap[G.q0]; op.t1 = qmap[G.q1];
                      op.qj = GK_IMAG; op.qflags = G.kind == LQ_RYY ? GG_YY : 0; break;
        case LQ_RZZ:  op.type = K_D2; op.t0 = qmap[G.q0]; op.t1 = qmap[G.q1]; break;
        default: break;
        }
        ops.push_back(op);
        fl.push_back(op.type == K_X ? std::vector<MFactor>{} : std::vector<MFactor>{f});
        fusable.push_back(0);
        touch_all((int)ops.size() - 1);
    }
    for (size_t i = base; i < ops.size(); i++) {   // Pauli generators (Blocker)
        POp &P = ops[i];
        if (P.ctrl) continue;
        const uint64_t b0 = P.t0 >= 0 ? bit(P.t0) : 0, b1 = P.t1 >= 0 ? bit(P.t1) : 0;
        switch (P.type) {
        case K_D1: P.pgen = true; P.gz = b0; break;                 // any diagonal: a function of Z
        case K_D2: P.pgen = true; P.gz = b0 | b1; break;
        case K_X: P.pgen = true; P.gx = b0; break;
        case K_G:
            if (P.qj == GK_REAL) { P.pgen = true; P.gx = P.gz = b0; }    // RY
            else if (P.qj == GK_IMAG) { P.pgen = true; P.gx = b0; }     // RX
            break;
        case K_GG:
            P.pgen = true;
            P.gx = b0 | b1;
            if (P.qflags & GG_YY) P.gz = b0 | b1;
            break;
        default: break;
        }
    }
    for (size_t i = base; i < ops.size(); i++) {
        POp &P = ops[i];
        auto &F = fl[i - base];
        if (P.type == K_X || P.type == K_QFT) { P.spec = -1; continue; }
        MForm form = P.type == K_D1 ? MF_DIAG2 : P.type == K_U1 ? MF_U2x2 : (P.type == K_G || P.type == K_GG) ? MF_G
                   : P.type == K_U2 ? MF_U4x4 : MF_DIAG4;
        P.spec = mb.add_spec(form, F);
    }
}

void canonicalize_ops(int n, int32_t *qmap, std::vector<POp> &ops) {
    for (int q = 0; q < n; q++) {
        int target = n - 1 - q;
        if (qmap[q] == target) continue;
        int q2 = -1;
        for (int r = 0; r < n; r++) if (qmap[r] == target) q2 = r;
        POp op;
        op.type = K_SWAP;
        op.t0 = std::max(qmap[q], target);
        op.t1 = std::min(qmap[q], target);
        ops.push_back(op);
        std::swap(qmap[q], qmap[q2]);
    }
}

// Pauli sum -> one K_EXPV op per x mask (E = sum_t c_t <P_t>).
void lower_pauli(int n, const int32_t *qmap, const lq_pauli_term *terms, size_t n_terms,
                 std::vector<POp> &ops, Plan &plan) {
    size_t g0 = plan.groups.size();
    for (size_t t = 0; t < n_terms; t++) {
        uint64_t x = 0, z = 0;
        for (int q = 0; q < n; q++) {
            if (terms[t].x_mask & bit(q)) x |= bit(qmap[q]);
            if (terms[t].z_mask & bit(q)) z |= bit(qmap[q]);
        }
        uint32_t y = (uint32_t)(popc(terms[t].x_mask & terms[t].z_mask) & 3);
        size_t g = g0;
        while (g < plan.groups.size() && plan.groups[g].x != x) g++;
        if (g == plan.groups.size()) {
            plan.groups.push_back(PGroup());
            plan.groups.back().x = x;
        }
        plan.groups[g].terms.push_back({terms[t].coeff, z, y});
    }
    for (size_t g = g0; g < plan.groups.size(); g++) {
        POp op;
        op.type = K_EXPV;
        op.xm = plan.groups[g].x;
        for (auto &t : plan.groups[g].terms) op.zm |= t.z;
        op.group = (int)g;
        ops.push_back(op);
    }
}

// --------------------------------------------------------------------------
// Tile / sub-block planning
// --------------------------------------------------------------------------
namespace {

// Ops left behind block later ops that do not commute with them.  The
// bit-mask rule (two ops commute if every shared bit is diagonal in both)
// covers everything; for two Pauli-generator ops (POp::pgen) the letters are
// compared per bit instead -- conservatively: any bit on which the letters
// differ counts as a conflict -- so e.g. X(x)X rotations on overlapping pairs
// pass each other.
struct Blocker {
    uint64_t bF = 0, bT = 0;         // every blocked op
    uint64_t gF = 0, gT = 0;         // blocked ops that change the state (not Pauli-group reads)
    uint64_t nF = 0, nT = 0;         // blocked ops without a Pauli generator
    uint64_t mX = 0, mY = 0, mZ = 0; // letters of blocked Pauli-generator ops, per bit
    bool blocked(const POp &o) const {
        // Pauli-group expectations only read the state: they never block
        // each other, only the gates before them
        static const bool old_rule = getenv("LQ_EXPV_BLOCK_ALL") != nullptr;   // A/B experiments
        if (o.type == K_EXPV && !old_rule) return (o.full() & gT) || (o.touch() & gF);
        if (!o.pgen) return (o.full() & bT) || (o.touch() & bF);
        if ((o.full() & nT) || (o.touch() & nF)) return true;
        const uint64_t oX = o.gx & ~o.gz, oY = o.gx & o.gz, oZ = o.gz & ~o.gx;
        return ((oX & (mY | mZ)) | (oY & (mX | mZ)) | (oZ & (mX | mY))) != 0;
    }
    void add(const POp &o) {
        bF |= o.full();
        bT |= o.touch();
        if (o.type != K_EXPV) {
            gF |= o.full();
            gT |= o.touch();
        }
        if (!o.pgen) {
            nF |= o.full();
            nT |= o.touch();
            return;
        }
        mX |= o.gx & ~o.gz;
        mY |= o.gx & o.gz;
        mZ |= o.gz & ~o.gx;
    }
};

// first-fit absorption of `rem` into a tile whose bit set starts at Tm.
// Absorption stops at the pass's FP64 budget: a pass whose arithmetic
// exceeds its HBM time is FP64-bound, and the ops it leaves behind fill
// lighter passes later.
static void first_fit(const std::vector<POp> &ops, const std::vector<int> &rem, int K,
                      uint64_t &Tm, std::vector<int> &absorbed, int budget) {
    Blocker blk;
    int cost = 0;
    for (int i : rem) {
        const POp &o = ops[i];
        if (blk.blocked(o)) { blk.add(o); continue; }
        uint64_t need = o.full() & ~Tm;
        const int c = op_fp64_cost(o);
        if (popc(Tm | need) <= K && (!budget || cost + c <= budget)) { Tm |= need; absorbed.push_back(i); cost += c; }
        else blk.add(o);
    }
}

static int score(const std::vector<POp> &ops, const std::vector<int> &absorbed) {
    int s = 0;
    for (int i : absorbed) s += ops[i].diag() ? 1 : 4;
    return s;
}

// Count ops absorbable with a FIXED tile bit set Tm.
static void absorb_fixed(const std::vector<POp> &ops, const std::vector<int> &rem, uint64_t Tm,
                         std::vector<int> &absorbed, int budget) {
    Blocker blk;
    int cost = 0;
    for (int i : rem) {
        const POp &o = ops[i];
        const int c = op_fp64_cost(o);
        if (blk.blocked(o) || (o.full() & ~Tm) || (budget && cost + c > budget)) { blk.add(o); continue; }
        absorbed.push_back(i);
        cost += c;
    }
}

struct LocalMap {
    int K;
    uint8_t T[MAXK];
    int loc[64];
    LocalMap(uint64_t Tm) {
        K = 0;
        for (int b = 0; b < 64; b++) loc[b] = -1;
        for (int b = 0; b < 64; b++)
            if (Tm & bit(b)) { loc[b] = K; T[K++] = (uint8_t)b; }
    }
    uint32_t local(uint64_t phys) const {
        uint32_t m = 0;
        while (phys) { int b = __builtin_ctzll(phys); if (loc[b] >= 0) m |= 1u << loc[b]; phys &= phys - 1; }
        return m;
    }
};

static int lowrun_of(const LocalMap &L) {
    int r = 0;
    while (r < L.K && L.T[r] == r) r++;
    return r;
}

// fill a local register mask up to Rr bits
static uint32_t fill_S(uint32_t Sm, int K, int Rr, int lowrun) {
    for (int b = K - 1; b >= 0 && popc(Sm) < Rr; b--)
        if (b >= std::min(lowrun, 3) && !(Sm & (1u << b))) Sm |= 1u << b;
    for (int b = 0; b < K && popc(Sm) < Rr; b++)
        if (!(Sm & (1u << b))) Sm |= 1u << b;
    return Sm;
}

static void mask_to_S(uint32_t Sm, uint8_t *S) {
    int i = 0;
    for (int b = 0; b < 32 && i < R; b++) if (Sm & (1u << b)) S[i++] = (uint8_t)b;
    for (; i < R; i++) S[i] = 0;
}

static KOp lower_tile_op(const POp &o, const LocalMap &L, const uint8_t *S, int Rr,
                         const std::vector<uint32_t> &mat_off) {
    KOp k{};
    k.type = o.type;
    k.r0 = k.r1 = NOREG;
    auto reg = [&](int p) -> uint8_t {
        if (p < 0 || L.loc[p] < 0) return NOREG;
        for (int i = 0; i < Rr; i++) if (S[i] == L.loc[p]) return (uint8_t)i;
        return NOREG;
    };
    k.r0 = reg(o.t0);
    if (o.t1 >= 0) k.r1 = reg(o.t1);
    k.b0 = (uint8_t)(o.t0 >= 0 ? o.t0 : 0);
    k.b1 = (uint8_t)(o.t1 >= 0 ? o.t1 : 0);
    uint64_t c = o.ctrl;
    while (c) {
        int b = __builtin_ctzll(c);
        uint8_t r = reg(b);
        if (r != NOREG) k.rcm |= (uint8_t)(1u << r); else k.cmask |= bit(b);
        c &= c - 1;
    }
    k.flags = o.qflags;
    if (o.type == K_D1) {
        bool uni = true;
        uint64_t cc = o.ctrl;
        while (cc) { if (L.loc[__builtin_ctzll(cc)] >= 0) uni = false; cc &= cc - 1; }
        if (uni) k.flags |= OF_UNIFORM;
        if (L.loc[o.t0] < 0) k.flags |= OF_OUTSIDE;
    }
    k.qj = o.qj;
    k.mat = o.spec >= 0 ? mat_off[o.spec] : 0;
    return k;
}

static KOp lower_flat_op(const POp &o, const std::vector<uint32_t> &mat_off) {
    KOp k{};
    k.type = o.type;
    k.r0 = k.r1 = NOREG;
    k.b0 = (uint8_t)(o.t0 >= 0 ? o.t0 : 0);
    k.b1 = (uint8_t)(o.t1 >= 0 ? o.t1 : 0);
    k.cmask = o.ctrl;
    k.qj = o.qj;
    k.mat = o.spec >= 0 ? mat_off[o.spec] : 0;
    k.code = C_GENERIC;
    return k;
}

// Pick the specialised tile-kernel path of a lowered op.
static uint8_t tile_code(const KOp &k) {
    switch (k.type) {
    case K_U1:
        if (k.rcm == 0 && k.r0 < R) return (uint8_t)(C_U1 + k.r0);
        break;
    case K_G:
        if (k.rcm == 0 && k.r0 < R) return (uint8_t)(C_G + 4 * k.qj + k.r0);
        break;
    case K_GG:
        if (k.rcm == 0 && k.r0 < R && k.r1 < R && k.r0 != k.r1) {
            const int lo = std::min(k.r0, k.r1), hi = std::max(k.r0, k.r1);
            static const int idx[4][4] = {{-1, 0, 1, 2}, {-1, -1, 3, 4}, {-1, -1, -1, 5}, {-1, -1, -1, -1}};
            return (uint8_t)(C_GG + idx[lo][hi]);
        }
        break;
    case K_X:
        if (k.rcm == 0 && k.r0 < R) return (uint8_t)(C_X + k.r0);
        if (__builtin_popcount(k.rcm) == 1 && k.r0 < R) return (uint8_t)(C_CX + 4 * __builtin_ctz(k.rcm) + k.r0);
        break;
    case K_D1:
        if (k.rcm == 0) {
            if (k.r0 < R) return (uint8_t)(C_D1R + k.r0);
            return ((k.flags & OF_UNIFORM) && (k.flags & OF_OUTSIDE)) ? (uint8_t)C_D1U : (uint8_t)C_D1T;
        }
        break;
    case K_QFT:
        if (k.r0 < R) return (uint8_t)(C_QFT + k.r0);
        break;
    case K_SCALE:
        return C_SCALE;
    case K_DT:
        return C_DT;
    case K_EXPV:
        return C_EXPV;
    default:
        break;
    }
    return C_GENERIC;
}

// Assign shared-memory staging offsets to the ops of a tile pass.
static void finalize_pass_tables(PlanPass &pp, Plan &plan) {
    pp.kp.op_begin = plan.subs[pp.kp.sub_begin].op_begin;
    pp.kp.op_end = plan.subs[pp.kp.sub_end - 1].op_end;
    if (pp.kp.perm_end < pp.kp.perm_begin) pp.kp.perm_end = pp.kp.perm_begin;
    uint32_t off = 0;
    for (uint32_t i = pp.kp.op_begin; i < pp.kp.op_end; i++) {
        plan.kops[i].code = tile_code(plan.kops[i]);
        if (plan.kops[i].type == K_EXPV) continue;   // mat/aux hold its ETerm range
        plan.kops[i].aux = off;
        off += (uint32_t)op_table_size(plan.kops[i].type);
    }
    pp.kp.smat = off;
}

// An X-type op (X, CNOT, CCX) or SWAP is an affine permutation of the
// tile's local index when at most one control lies in the tile and, in that
// case, none lies outside (a tile-constant control makes it a conditional
// translation).
static bool foldable(const POp &o, const LocalMap &L) {
    if (o.type == K_SWAP) return o.ctrl == 0;
    if (o.type != K_X) return false;
    int in_t = 0;
    uint64_t out = 0, c = o.ctrl;
    while (c) {
        int b = __builtin_ctzll(c);
        if (L.loc[b] >= 0) in_t++; else out |= bit(b);
        c &= c - 1;
    }
    return in_t == 0 || (in_t == 1 && out == 0);
}

// Affine map l -> A l + sum_i [tile & cm_i == cm_i] v_i over GF(2)^K.
struct Affine {
    int K;
    uint32_t A[MAXK];                 // columns A e_j
    std::vector<std::pair<uint64_t, uint32_t>> terms;
    explicit Affine(int k) : K(k) { for (int j = 0; j < K; j++) A[j] = 1u << j; }
    template <class F> void linear(F M) {
        for (int j = 0; j < K; j++) A[j] = M(A[j]);
        for (auto &t : terms) t.second = M(t.second);
    }
    void add(const POp &o, const LocalMap &L) {
        if (o.type == K_SWAP) {
            int a = L.loc[o.t0], b = L.loc[o.t1];
            linear([&](uint32_t v) {
                uint32_t x = ((v >> a) ^ (v >> b)) & 1u;
                return v ^ (x << a) ^ (x << b);
            });
            return;
        }
        int t = L.loc[o.t0];
        int cin = -1;
        uint64_t out = 0, c = o.ctrl;
        while (c) {
            int b = __builtin_ctzll(c);
            if (L.loc[b] >= 0) cin = L.loc[b]; else out |= bit(b);
            c &= c - 1;
        }
        if (cin >= 0) linear([&](uint32_t v) { return v ^ (((v >> cin) & 1u) << t); });
        else terms.push_back({out, 1u << t});
    }
    // columns of A^-1 (Gauss-Jordan on [A | I])
    void inverse(uint32_t *inv) const {
        uint32_t rowsA[MAXK], rowsI[MAXK];
        for (int i = 0; i < K; i++) {
            rowsA[i] = 0;
            for (int j = 0; j < K; j++) if ((A[j] >> i) & 1) rowsA[i] |= 1u << j;
            rowsI[i] = 1u << i;
        }
        for (int col = 0; col < K; col++) {
            int piv = col;
            while (!((rowsA[piv] >> col) & 1)) piv++;
            std::swap(rowsA[piv], rowsA[col]);
            std::swap(rowsI[piv], rowsI[col]);
            for (int r = 0; r < K; r++)
                if (r != col && ((rowsA[r] >> col) & 1)) { rowsA[r] ^= rowsA[col]; rowsI[r] ^= rowsI[col]; }
        }
        for (int j = 0; j < K; j++) {   // column j of inverse = bits (row i, col j) of rowsI
            inv[j] = 0;
            for (int i = 0; i < K; i++) if ((rowsI[i] >> j) & 1) inv[j] |= 1u << i;
        }
    }
};

// Lower a K_EXPV op for register set S: x bits -> register mask (rcm),
// terms sorted by their register z pattern.
static void lower_expv(const POp &o, const LocalMap &L, const uint8_t *S, int Rr, PlanPass &pp, KOp &k,
                       Plan &plan) {
    auto reg = [&](int p) -> int {
        if (L.loc[p] < 0) return -1;
        for (int i = 0; i < Rr; i++) if (S[i] == L.loc[p]) return i;
        return -1;
    };
    uint32_t xreg = 0;
    uint64_t x = o.xm;
    while (x) { int b = __builtin_ctzll(x); xreg |= 1u << reg(b); x &= x - 1; }
    uint64_t sphys = 0;
    for (int i = 0; i < Rr; i++) sphys |= bit(L.T[S[i]]);
    std::vector<ETerm> ts;
    for (auto &t : plan.groups[o.group].terms) {
        ETerm e{};
        e.c = t.c;
        e.znr = t.z & ~sphys;
        uint64_t zr = t.z & sphys;
        while (zr) { int b = __builtin_ctzll(zr); e.zreg |= 1u << reg(b); zr &= zr - 1; }
        e.y = t.y;
        ts.push_back(e);
    }
    std::stable_sort(ts.begin(), ts.end(), [](const ETerm &a, const ETerm &b) { return a.zreg < b.zreg; });
    k.type = K_EXPV;
    k.rcm = (uint8_t)xreg;
    k.cmask = 0;
    k.mat = (uint32_t)(plan.eterms.size() - pp.kp.eterm_begin);
    k.aux = (uint32_t)ts.size();
    plan.eterms.insert(plan.eterms.end(), ts.begin(), ts.end());
    pp.kp.eterm_end = (uint32_t)plan.eterms.size();
    pp.kp.flags |= PF_EXPV;
}

// Runs of >= 2 consecutive uncontrolled diagonals on distinct register bits
// become one K_DT op: 15 complex multiplies per thread instead of 8 per
// member.  Members are recorded in the plan constants as (position, offset).
static void merge_diag_runs(Plan &plan, uint32_t begin, MatBuilder &mb) {
    auto simple = [](const KOp &k) { return k.type == K_D1 && k.rcm == 0 && k.cmask == 0 && k.r0 < R; };
    std::vector<KOp> out;
    for (size_t i = begin; i < plan.kops.size();) {
        size_t j = i;
        uint32_t pos = 0;
        while (j < plan.kops.size() && simple(plan.kops[j]) && !(pos >> plan.kops[j].r0 & 1)) {
            pos |= 1u << plan.kops[j].r0;
            j++;
        }
        if (j - i >= 2) {
            std::vector<double> mem;
            for (size_t q = i; q < j; q++) {
                mem.push_back((double)plan.kops[q].r0);
                mem.push_back((double)plan.kops[q].mat);
            }
            KOp d{};
            d.type = K_DT;
            d.r0 = d.r1 = NOREG;
            d.flags = (uint8_t)(j - i);
            d.mat = (uint32_t)mb.add_const(mem.data(), (int)(j - i));
            out.push_back(d);
            i = j;
        } else {
            out.push_back(plan.kops[i]);
            i++;
        }
    }
    plan.kops.resize(begin);
    plan.kops.insert(plan.kops.end(), out.begin(), out.end());
}

// Generic QFT stages (QF_GENERAL) of a sub-block: register twiddle table of
// each stage for this register set, the sub-block head (thread twiddle at the
// largest j), and the pass's physical -> logical map.
static void lower_qft_stages(Plan &plan, const KSub &sb, const LocalMap &L, int Rr, const std::vector<POp> &ops,
                             const std::vector<int> &taken, MatBuilder &mb, PlanPass &pp) {
    int jmax = -1, layout = -1;
    for (int i : taken)
        if (ops[i].type == K_QFT && ops[i].layout >= 0) { jmax = std::max(jmax, (int)ops[i].qj); layout = ops[i].layout; }
    if (layout < 0) return;
    const std::vector<uint8_t> &lp = mb.layouts[layout];
    for (int b = 0; b < 64; b++) pp.kp.lpos[b] = lp[b];
    bool head = true;
    for (uint32_t k = sb.op_begin; k < plan.kops.size(); k++) {
        KOp &op = plan.kops[k];
        if (op.type != K_QFT || !(op.flags & QF_GENERAL)) continue;
        const int j = op.qj;
        const bool inv = op.flags & QF_INVERSE;
        double tab[2 * NREG];
        for (int v = 0; v < NREG; v++) {
            uint64_t lg = 0;
            for (int i = 0; i < Rr; i++)
                if (v & (1 << i)) {
                    const int p = L.T[sb.S[i]];
                    if (lp[p] < 64) lg |= bit(lp[p]);
                }
            const uint64_t Lm = (j == 0) ? 0 : (lg & (bit(j) - 1));
            const long double ang = 3.141592653589793238462643383279502884L * (long double)Lm / ldexpl(1.0L, j);
            tab[2 * v] = (double)cosl(ang);
            tab[2 * v + 1] = (inv ? -1.0 : 1.0) * (double)sinl(ang);
        }
        op.mat = (uint32_t)mb.add_const(tab, NREG);
        op.tdep = 0x80;
        op.qi = NOREG;
        for (int i = 0; i < Rr; i++) {
            const int p = L.T[sb.S[i]];
            if (lp[p] < 64 && lp[p] < j) op.tdep |= (uint8_t)(1u << i);
            if (lp[p] < 64 && (int)lp[p] == j - 1) op.qi = (uint8_t)i;
        }
        op.b1 = (uint8_t)jmax;
        if (head) op.flags |= QF_HEAD;
        head = false;
    }
}

static int32_t build_perm(const std::vector<POp> &ops, const std::vector<int> &group, const LocalMap &L,
                          const PlanPass &pp, Plan &plan) {
    if (group.empty()) return -1;
    Affine F(L.K);
    for (int i : group) F.add(ops[i], L);
    uint32_t inv[MAXK];
    F.inverse(inv);
    KPerm P{};
    for (int j = 0; j < L.K; j++) P.col[j] = (uint16_t)inv[j];
    P.term_begin = (uint32_t)plan.perm_terms.size();
    for (auto &t : F.terms) {
        uint32_t v = 0;
        for (int j = 0; j < L.K; j++) if ((t.second >> j) & 1) v ^= inv[j];
        KPermTerm kt{};
        kt.cmask = t.first;
        kt.vec = v;
        plan.perm_terms.push_back(kt);
    }
    P.term_end = (uint32_t)plan.perm_terms.size();
    plan.perms.push_back(P);
    plan.n_folded += group.size();
    return (int32_t)(plan.perms.size() - 1 - pp.kp.perm_begin);
}

// Build a TILE pass from absorbed ops (execution order) and tile mask Tm:
// segments = [entry permutation group][register sub-block], the entry
// permutations being folded into the exchange that starts the sub-block.
static void emit_tile(int n, int nl, int K, int Rr, uint64_t Tm, const std::vector<POp> &ops,
                      const std::vector<int> &absorbed, const std::vector<uint32_t> &mat_off,
                      Plan &plan, MatBuilder &mb, bool oop = false) {
    LocalMap L(Tm);
    int lowrun = (nl > K) ? lowrun_of(L) : 0;
    PlanPass pp;
    pp.kind = PASS_TILE;
    pp.kp.n = n;
    pp.kp.nl = nl;
    pp.kp.K = K;
    pp.kp.flags = 0;
    memset(pp.kp.lpos, 255, sizeof(pp.kp.lpos));
    memcpy(pp.kp.T, L.T, MAXK);
    pp.kp.sub_begin = (uint32_t)plan.subs.size();
    pp.kp.perm_begin = (uint32_t)plan.perms.size();
    pp.kp.eterm_begin = pp.kp.eterm_end = (uint32_t)plan.eterms.size();
    pp.n_ops = (int)absorbed.size();
    bool all_expv = true;

    std::vector<int> rem = absorbed;
    auto collect_perm = [&](std::vector<int> &group) {
        Blocker blk;
        std::vector<int> left;
        for (int i : rem) {
            const POp &o = ops[i];
            if (!blk.blocked(o) && foldable(o, L)) { group.push_back(i); continue; }
            blk.add(o);
            left.push_back(i);
        }
        rem.swap(left);
    };
    struct Seg { std::vector<int> entry; uint32_t Sm; std::vector<int> taken; };
    std::vector<Seg> segs;
    std::vector<int> entry;
    collect_perm(entry);
    while (!rem.empty()) {
        uint32_t Sm = 0;
        Blocker blk;
        std::vector<int> taken, left;
        for (int i : rem) {
            const POp &o = ops[i];
            if (blk.blocked(o)) { blk.add(o); left.push_back(i); continue; }
            if (foldable(o, L)) {
                // X / CNOT with a register target and thread-constant controls is
                // free inside the sub-block (flip mask); otherwise defer it to the
                // next exchange
                bool inl = o.type == K_X && (Sm & (1u << L.loc[o.t0])) && !(L.local(o.ctrl) & Sm);
                if (inl) taken.push_back(i);
                else { blk.add(o); left.push_back(i); }
                continue;
            }
            uint32_t need = L.local(o.full()) & ~Sm;
            if (popc(Sm | need) <= Rr) { Sm |= need; taken.push_back(i); }
            else { blk.add(o); left.push_back(i); }
        }
        rem.swap(left);
        segs.push_back({entry, Sm, taken});
        entry.clear();
        collect_perm(entry);
    }
    if (segs.empty()) segs.push_back({std::vector<int>(), 0u, std::vector<int>()});   // pure permutation pass
    std::vector<int> store_group = entry;
    if (segs.size() == 1 && segs[0].taken.empty() && !segs[0].entry.empty() && store_group.empty()) {
        store_group.swap(segs[0].entry);   // a lone permutation group: apply it at the store
    }
    for (auto &sg : segs) sg.Sm = fill_S(sg.Sm, K, Rr, lowrun);
    uint32_t lane_forbid = (uint32_t)((1u << std::min(lowrun, 3)) - 1);
    uint32_t top = 0;
    for (int b = K - 1; b >= 0 && popc(top) < Rr; b--) top |= 1u << b;
    uint32_t Ss = segs.back().Sm;
    // in place, the store's lanes must be the coalescing bits; a relabelling
    // store (oop) puts whatever its lanes hold at the new frame's low bits
    if ((Ss & lane_forbid) && !oop) Ss = top;
    mask_to_S(segs.front().Sm, pp.kp.Sload);
    mask_to_S(Ss, pp.kp.Sstore);
    for (auto &sg : segs) {
        KSub sb{};
        mask_to_S(sg.Sm, sb.S);
        sb.perm = build_perm(ops, sg.entry, L, pp, plan);
        sb.op_begin = (uint32_t)plan.kops.size();
        for (int i : sg.taken) {
            KOp k = lower_tile_op(ops[i], L, sb.S, Rr, mat_off);
            if (ops[i].type == K_EXPV) lower_expv(ops[i], L, sb.S, Rr, pp, k, plan);
            else all_expv = false;
            plan.kops.push_back(k);
        }
        merge_diag_runs(plan, sb.op_begin, mb);
        lower_qft_stages(plan, sb, L, Rr, ops, sg.taken, mb, pp);
        sb.op_end = (uint32_t)plan.kops.size();
        plan.subs.push_back(sb);
    }
    if (pp.kp.eterm_end > pp.kp.eterm_begin || (pp.kp.flags & PF_EXPV)) {
        pp.kp.flags |= PF_EXPV;
        pp.kp.eslot = plan.n_slots;   // one partial per warp of every tile (tile.cuh expv_partial)
        plan.n_slots += (uint32_t)(1u << (nl - K)) * (uint32_t)std::max(1, (1 << (K - Rr)) / 32);
    }
    pp.kp.store_perm = build_perm(ops, store_group, L, pp, plan);
    // read-only pass: nothing but Pauli groups (no gate, no folded permutation)
    if (all_expv && plan.perms.size() == pp.kp.perm_begin) pp.kp.flags |= PF_NO_STORE;
    pp.kp.sub_end = (uint32_t)plan.subs.size();
    pp.kp.perm_end = (uint32_t)plan.perms.size();
    finalize_pass_tables(pp, plan);
    plan.passes.push_back(pp);
    plan.n_tile++;
}

}  // namespace


// Relabelling out-of-place stores (PlanOptions::oop).
// The lane bits of a tile pass's store: the lowest local bits outside its
// store register set, as physical bits in the pass's frame (lane order).
static std::vector<int> store_lanes(const PlanPass &pp, int Rr) {
    uint32_t sm = 0;
    for (int i = 0; i < Rr; i++) sm |= 1u << pp.kp.Sstore[i];
    std::vector<int> l;
    for (int b = 0; b < pp.kp.K && l.size() < 5; b++)
        if (!(sm >> b & 1)) l.push_back(pp.kp.T[b]);
    return l;
}

// The next frame: the store's lane bits that the next tile holds, in lane
// order, go to bits 0, 1, ... (each warp store is then one contiguous run);
// the next tile's other bits follow up to bit K-1; every other bit keeps its
// relative order above.
static void next_frame(int nl, const std::vector<int> &lanes, uint64_t Tn, uint8_t *spos) {
    int nxt = 0;
    uint64_t placed = 0;
    for (int b : lanes) {
        if (!(Tn >> b & 1)) break;
        spos[b] = (uint8_t)nxt++;
        placed |= bit(b);
    }
    for (int b = 0; b < nl; b++)
        if ((Tn >> b & 1) && !(placed >> b & 1)) { spos[b] = (uint8_t)nxt++; placed |= bit(b); }
    for (int b = 0; b < nl; b++)
        if (!(placed >> b & 1)) spos[b] = (uint8_t)nxt++;
    for (int b = nl; b < 64; b++) spos[b] = (uint8_t)b;   // global (shard) bits never move
}

static uint64_t map_bits(uint64_t m, const uint8_t *spos) {
    uint64_t r = 0;
    while (m) { int b = __builtin_ctzll(m); r |= bit(spos[b]); m &= m - 1; }
    return r;
}

static void remap_op(POp &o, const uint8_t *spos) {
    if (o.t0 >= 0) o.t0 = spos[o.t0];
    if (o.t1 >= 0) o.t1 = spos[o.t1];
    o.ctrl = map_bits(o.ctrl, spos);
    o.xm = map_bits(o.xm, spos);
    o.zm = map_bits(o.zm, spos);
    o.rd = map_bits(o.rd, spos);
    o.gx = map_bits(o.gx, spos);
    o.gz = map_bits(o.gz, spos);
}

// op types the strided pair kernel (k_pair) executes; everything else
// (QFT stages, ...) runs in a tile pass even when alone
static bool pair_kernel_op(uint8_t t) { return t == K_U1 || t == K_X || t == K_G || t == K_U2 || t == K_SWAP; }

void plan_circuit(int n, const std::vector<POp> &ops_in, const PlanOptions &opt, MatBuilder &mb,
                  Plan &plan) {
    std::vector<POp> ops(ops_in);   // relabelling stores (opt.oop) move later ops into new frames
    for (int b = 0; b < 64; b++) plan.frame[b] = (uint8_t)b;
    std::vector<uint32_t> mat_off;
    for (auto &sp : mb.specs) mat_off.push_back(sp.out);
    const int nl = opt.n_local > 0 ? std::min(opt.n_local, n) : n;   // tile bits come from [0, nl)
    int K = opt.K > 0 ? std::min(opt.K, nl) : auto_tile_bits(nl);
    // a run of QFT stages only (Alg. 3 on a permuted or sharded layout)
    // packs strictly in order with no FP64 budget, as plan_qft's, and takes
    // 12 tile bits when that saves a pass (n = 30 QFT on 2 shards: 31 ms vs
    // 37 ms; before the JIT computed the stages' logical index with
    // straight-line code it was 57 ms)
    bool all_qft = !ops.empty();
    for (const POp &o : ops) all_qft &= o.type == K_QFT;
    if (all_qft && opt.K <= 0 && nl > 12 && !getenv("LQ_QFT_K11")) {   // (A/B switch)
        auto count_q = [&](int Kc) {
            const int cc = std::max(0, std::min(opt.coalesce, Kc - 2));
            const uint64_t m0 = (1ull << cc) - 1;
            int np = 0;
            for (size_t s0 = 0; s0 < ops.size(); np++) {
                uint64_t Tm = m0;
                while (s0 < ops.size() && popc(Tm | ops[s0].full()) <= Kc) Tm |= ops[s0++].full();
            }
            return np;
        };
        if (count_q(12) < count_q(K)) K = 12;
    }
    if (K > 12) K = 12;   // two 2^K buffers must fit in shared memory
    if (nl <= K) K = nl;
    int Rr = std::min(std::max(1, std::min(opt.reg_bits, R)), K);
    // a tile of fewer than 2^5 threads runs its gates as one thread's serial
    // chain, and a state that is one tile runs on one CTA: such plans spread
    // the tile over more threads, down to 4 amplitudes per thread (a 2-qubit
    // op needs both its bits in registers) -- config 3 (n = 4, 4 threads)
    // 41 -> 37 us per gradient, config 1 (n = 10, 256 threads) 156 -> 124 us
    // per run on B200 (tools/cfg3_rb.py, tools/cfg1_variants.py)
    if (opt.reg_bits >= R) {
        if (nl <= K) Rr = std::min(Rr, std::max(2, K - 8));
        else if (K - Rr < 5) Rr = std::min(Rr, std::max(2, K - 5));
    }
    plan.Rr = Rr;
    plan.n = n;
    plan.nl = nl;
    plan.K = K;
    int c = std::max(0, std::min(opt.coalesce, K - 2));
    uint64_t mand = (nl > K) ? ((1ull << c) - 1) : ((1ull << nl) - 1);
    // Pauli groups whose x mask cannot share a tile with the coalescing run
    // go to the direct kernel
    std::vector<char> skip(ops.size(), 0);
    for (size_t i = 0; i < ops.size(); i++)
        if (ops[i].type == K_EXPV && (popc(mand | ops[i].xm) > K || popc(ops[i].xm) > Rr)) {
            skip[i] = 1;
            plan.wide_groups.push_back((uint32_t)ops[i].group);
        }
    if (!opt.fusion) {
        for (size_t i = 0; i < ops.size(); i++) {
            const POp &o = ops[i];
            if (skip[i]) continue;
            if (o.type == K_EXPV || (!o.diag() && !pair_kernel_op(o.type))) {
                uint64_t Tm = mand | o.full() | (o.type == K_EXPV ? o.xm : 0);
                for (int b = 0; b < nl && popc(Tm) < K; b++) Tm |= bit(b);
                emit_tile(n, nl, K, Rr, Tm, ops, std::vector<int>{(int)i}, mat_off, plan, mb);
                continue;
            }
            PlanPass pp;
            pp.kind = o.diag() ? PASS_DIAG : PASS_PAIR;
            pp.op_begin = (uint32_t)plan.kops.size();
            plan.kops.push_back(lower_flat_op(o, mat_off));
            pp.op_end = (uint32_t)plan.kops.size();
            pp.n_ops = 1;
            plan.passes.push_back(pp);
            (o.diag() ? plan.n_diag : plan.n_pair)++;
        }
        return;
    }
    // the coalescing run must leave room for a 2-qubit gate's two target bits
    std::vector<int> rem;
    for (size_t i = 0; i < ops.size(); i++)
        if (!skip[i]) rem.push_back((int)i);
    // Balanced stage packing of a run of QFT stages (as plan_qft's): the pass
    // count is the greedy one, but a pass whose stages cover the coalescing
    // bits (its tile needs no extra low bits) takes K stages and the others
    // share the rest evenly, so their spare tile bits lengthen the coalescing
    // run.  Caps are upper bounds on the stages per pass: any prefix of the
    // run is a valid pass.
    std::vector<size_t> qcap;
    size_t qpass = 0;
    if (all_qft && nl > K && opt.fusion && !getenv("LQ_QFT_GREEDY")) {   // (A/B switch)
        const int m = (int)ops.size();
        int np = 0;
        for (size_t s0 = 0; s0 < ops.size(); np++) {
            uint64_t Tq = mand;
            const size_t b0 = s0;
            while (s0 < ops.size() && popc(Tq | ops[s0].full()) <= K) Tq |= ops[s0++].full();
            if (s0 == b0) { np = 0; break; }
        }
        auto covers = [&](int from, int to) {   // stages [from, to): distinct single bits that include mand
            uint64_t u = 0;
            for (int i = from; i < to; i++) u |= ops[i].full();
            return (u & mand) == mand && popc(u) == to - from;
        };
        const int Lc = std::min(K, m);
        const bool last_free = covers(m - Lc, m), head_free = !last_free && covers(0, Lc);
        const int ns = (last_free || head_free) ? np - 1 : np;
        const int S = (last_free || head_free) ? m - Lc : m;
        if (np > 1 && ns > 0 && S > 0 && (S + ns - 1) / ns <= K - c) {
            for (int p = 0; p < ns; p++) qcap.push_back((size_t)(S / ns + (p < S % ns ? 1 : 0)));
            if (head_free) qcap.insert(qcap.begin(), (size_t)Lc);
            else if (last_free) qcap.push_back((size_t)Lc);
        }
    }
    // the FP64 budget trades an extra HBM round trip for less arithmetic per
    // pass; a state that is one tile has no HBM round trip to trade
    const int budget_all = (nl > K && !all_qft) ? opt.budget : 0;
    // zero-first plans (PlanOptions::first_free): the support U = union of the
    // tiles planned so far (lq_api.cu prepare() runs a pass only over the
    // tiles inside U).  A pass with |U| <= free_upto is exempt from the
    // budget.  Pass 0 (U empty: one tile per state) always; exempting pass 1
    // too (|U| = K, at most 2^(K-3) tiles) measured 0.8 % slower on config 4
    // (the extra ops it absorbs leave later passes no lighter), hence 0.
    uint64_t U = 0;
    bool track = opt.first_free;
    const int free_upto = getenv("LQ_FREE_UPTO") ? atoi(getenv("LQ_FREE_UPTO")) : 0;   // A/B experiments
    // support-aware budget (zero-first plans): a pass whose support U misses
    // some bits reads only 2^|U| amplitudes, so its HBM time is about
    // (2^(|U|-nl) + 1) / 2 of a full pass and so is the arithmetic it can hide
    const bool sup_budget = getenv("LQ_SUPPORT_BUDGET") != nullptr;   // A/B experiments
    // relabelling out-of-place stores (PlanOptions::oop): after each storing
    // tile pass the next tile is chosen at once -- it must hold the store's
    // lowest opt.oop lane bits -- and the pass writes the state in the frame
    // where that tile is bits 0..K-1 (contiguous reads)
    bool any_qft = false;
    for (const POp &o : ops) any_qft |= o.type == K_QFT;
    const bool oop = opt.oop > 0 && nl > K && !any_qft && nl <= 48;
    // tile selection for the ops in `rem`: Tm starts from `mand0`; the result
    // is filled to K bits with the bits of `prefer` first, then the lowest
    auto select = [&](uint64_t mand0, const std::vector<int> &prefer, uint64_t &Tm,
                      std::vector<int> &absorbed) {
        const uint64_t mand = mand0;
        int budget = (track && popc(U) <= free_upto) ? 0 : budget_all;
        if (track && sup_budget && budget && popc(U) < nl) {
            const double f = 0.5 * (std::ldexp(1.0, popc(U) - nl) + 1.0);
            budget = std::max(1, (int)(budget * f));
        }
        Tm = mand;
        absorbed.clear();
        std::vector<int> absorbed_w;
        first_fit(ops, rem, K, Tm, absorbed, budget);
        // local search works on a window of the next ops (bounded cost)
        std::vector<int> window(rem.begin(), rem.begin() + std::min<size_t>(rem.size(), 384));
        {
            std::vector<int> a0;
            absorb_fixed(ops, window, Tm, a0, budget);
            absorbed_w.swap(a0);
        }
        int best = score(ops, absorbed_w);
        uint64_t Tm0 = Tm;
        // local search: swap one free tile bit for another if it absorbs more
        if (nl > K) {
            for (int iter = 0; iter < 2; iter++) {
                bool improved = false;
                // fill Tm to K bits first with the bits most used by blocked ops
                for (int out = 0; out < nl; out++) {
                    if (!(Tm & bit(out)) || (mand & bit(out))) continue;
                    for (int in = 0; in < nl; in++) {
                        if (Tm & bit(in)) continue;
                        uint64_t T2 = (Tm & ~bit(out)) | bit(in);
                        std::vector<int> a2;
                        absorb_fixed(ops, window, T2, a2, budget);
                        int s2 = score(ops, a2);
                        if (s2 > best) { best = s2; Tm = T2; improved = true; break; }
                    }
                }
                if (popc(Tm) < K) {
                    for (int in = 0; in < nl && popc(Tm) < K; in++) {
                        if (Tm & bit(in)) continue;
                        std::vector<int> a2;
                        absorb_fixed(ops, window, Tm | bit(in), a2, budget);
                        int s2 = score(ops, a2);
                        if (s2 > best) { best = s2; Tm |= bit(in); improved = true; }
                    }
                }
                if (!improved) break;
            }
            if (Tm != Tm0) {
                absorbed.clear();
                absorb_fixed(ops, rem, Tm, absorbed, budget);
            }
        }
        if (absorbed.empty()) absorbed.push_back(rem[0]);   // progress guarantee
        if (absorbed.size() > (size_t)MAX_PASS_OPS) absorbed.resize(MAX_PASS_OPS);   // a valid prefix
        for (int b : prefer)
            if (popc(Tm) < K && b < nl) Tm |= bit(b);
        for (int b = 0; b < nl && popc(Tm) < K; b++) Tm |= bit(b);
    };
    bool have_pend = false;
    uint64_t pend_T = 0;
    std::vector<int> pend_abs;
    // the first pass of a zero-first plan reads nothing: no coalescing run
    uint64_t mand_next = (oop && opt.first_free) ? 0 : mand;
    while (!rem.empty()) {
        uint64_t Tm = 0;
        std::vector<int> absorbed;
        if (have_pend) {
            Tm = pend_T;
            absorbed.swap(pend_abs);
            have_pend = false;
        } else {
            select(mand_next, std::vector<int>(), Tm, absorbed);
        }
        if (qpass < qcap.size() && absorbed.size() > qcap[qpass]) {
            absorbed.resize(qcap[qpass]);
            Tm = mand;
            for (int i : absorbed) Tm |= ops[i].full();
            for (int b = 0; b < nl && popc(Tm) < K; b++) Tm |= bit(b);
        }
        qpass++;
        mand_next = mand;
        int n_full = 0;
        bool has_expv = false;
        for (int i : absorbed) {
            n_full += ops[i].diag() ? 0 : 1;
            has_expv |= ops[i].type == K_EXPV;
        }
        if (n_full == 0 && !has_expv && absorbed.size() == 1) {
            // a lone diagonal op: k_diag (one complex multiply per amplitude).
            // Longer diagonal runs go to tile passes, which apply factors on
            // bits outside the register set once per thread, not per amplitude.
            PlanPass pp;
            pp.kind = PASS_DIAG;
            pp.op_begin = (uint32_t)plan.kops.size();
            for (int i : absorbed) plan.kops.push_back(lower_flat_op(ops[i], mat_off));
            pp.op_end = (uint32_t)plan.kops.size();
            pp.n_ops = (int)absorbed.size();
            plan.passes.push_back(pp);
            plan.n_diag++;
            track = false;
        } else if (absorbed.size() == 1 && !has_expv && pair_kernel_op(ops[absorbed[0]].type) &&
                   (nl > K || popc(ops[absorbed[0]].full()) > K)) {
            PlanPass pp;
            pp.kind = PASS_PAIR;
            pp.op_begin = (uint32_t)plan.kops.size();
            plan.kops.push_back(lower_flat_op(ops[absorbed[0]], mat_off));
            pp.op_end = (uint32_t)plan.kops.size();
            pp.n_ops = 1;
            plan.passes.push_back(pp);
            plan.n_pair++;
            track = false;
        } else {
            // (select() filled the tile to exactly K bits, lowest free bits
            // first: longer contiguous runs for coalescing)
            emit_tile(n, nl, K, Rr, Tm, ops, absorbed, mat_off, plan, mb, oop);
            if (!(plan.passes.back().kp.flags & PF_NO_STORE)) U |= Tm;   // a read-only pass leaves U as it was
        }
        // remove absorbed from rem (absorbed is a subsequence of rem)
        std::vector<int> left;
        size_t j = 0;
        for (int i : rem) {
            if (j < absorbed.size() && absorbed[j] == i) { j++; continue; }
            left.push_back(i);
        }
        rem.swap(left);
        PlanPass &pp = plan.passes.back();
        if (oop && pp.kind == PASS_TILE && !(pp.kp.flags & PF_NO_STORE)) {
            const std::vector<int> lanes = store_lanes(pp, Rr);
            uint64_t mn = 0;
            for (size_t k = 0; k < lanes.size() && (int)k < opt.oop; k++) mn |= bit(lanes[k]);
            uint64_t Tn = mn;
            if (!rem.empty()) {
                std::vector<int> prefer(lanes);
                for (int l = 0; l < pp.kp.K; l++) prefer.push_back(pp.kp.T[l]);
                select(mn, prefer, Tn, pend_abs);
                have_pend = true;
            }
            next_frame(nl, lanes, Tn, pp.spos);
            pp.oop = true;
            plan.has_oop = true;
            for (POp &o : ops) {
                remap_op(o, pp.spos);
                if (o.type == K_EXPV && o.group >= 0) {
                    PGroup &G = plan.groups[(size_t)o.group];
                    G.x = map_bits(G.x, pp.spos);
                    for (auto &t : G.terms) t.z = map_bits(t.z, pp.spos);
                }
            }
            U = map_bits(U, pp.spos);
            for (int b = 0; b < 64; b++) plan.frame[b] = pp.spos[plan.frame[b]];
            pend_T = map_bits(Tn, pp.spos);
        }
    }
}

// --------------------------------------------------------------------------
// QFT.  Stage for logical bit j (qubit n-1-j): butterfly
// (u, w) -> (u + w, u - w) then multiply the bit-j-set output by
// exp(i pi (x mod 2^j) / 2^j), x the logical index -- Alg. 3's H(i) followed
// by all CP(pi/2^{k-i}) controlled by qubit i.  The 1/sqrt2 of each H is
// applied once per pass (K_SCALE).  The closing SWAP layer is the layout
// relabel.
// --------------------------------------------------------------------------
static uint64_t brev_n(uint64_t x, int n) {
    uint64_t r = 0;
    for (int i = 0; i < n; i++) if (x & bit(i)) r |= bit(n - 1 - i);
    return r;
}

bool plan_qft(int n, int32_t *qmap, bool inverse, const PlanOptions &opt, Plan &plan,
              MatBuilder &mb) {
    bool ident = true, rev = true;
    for (int q = 0; q < n; q++) {
        if (qmap[q] != n - 1 - q) ident = false;
        if (qmap[q] != q) rev = false;
    }
    if (!ident && !rev) return false;
    bool layout_rev = ident ? false : true;
    if (inverse) layout_rev = !layout_rev;
    std::vector<int> js;
    if (!inverse) for (int j = n - 1; j >= 0; j--) js.push_back(j);
    else for (int j = 0; j < n; j++) js.push_back(j);
    auto phys = [&](int j) { return layout_rev ? n - 1 - j : j; };

    // passes the greedy stage packing below makes with K tile bits
    auto count_passes = [&](int Kc) {
        const int cc = std::max(0, std::min(opt.coalesce, Kc - 1));
        const uint64_t m0 = (n > Kc) ? ((1ull << cc) - 1) : ((1ull << n) - 1);
        int np = 0;
        for (size_t s0 = 0; s0 < js.size(); np++) {
            uint64_t Tm = m0;
            while (s0 < js.size() && popc(Tm | bit(phys(js[s0]))) <= Kc) Tm |= bit(phys(js[s0++]));
        }
        return np;
    };
    int K = opt.K > 0 ? std::min(opt.K, n) : auto_tile_bits(n);
    // automatic size: 12 tile bits (one CTA per SM) when that saves a whole
    // pass -- at n = 30 four passes of 11 bits take 29.2 ms, three of 12 take
    // 25.0 ms (B200)
    if (opt.K <= 0 && n > 12 && count_passes(12) < count_passes(K)) K = 12;
    // ... or, at the same pass count, when the balanced packing below would
    // leave a strided pass of the smaller tile without a spare bit (128-byte
    // runs) and 12 bits give every strided pass one: QFT(27) 2.555 -> 2.418
    // ms, QFT(33) 219.8 -> 210.2 ms; the sizes the rule leaves alone are
    // faster with the smaller tile at 3 CTAs/SM (n = 24, 25, 31, 32: +2 ..
    // +11 % with 12 bits; profiles/r02/ab_qft_k12.jsonl)
    // (HBM-resident sizes only, n >= 26: measured there)
    if (opt.K <= 0 && n >= 26 && K < 12 && !getenv("LQ_QFT_GREEDY") && !getenv("LQ_QFT_K11")) {   // (A/B switches)
        const int np = count_passes(K), ns = np - 1;
        const int cK = std::max(0, std::min(opt.coalesce, K - 1)), c12 = std::max(0, std::min(opt.coalesce, 11));
        if (np == count_passes(12) && ns > 0 && (n - K + ns - 1) / ns == K - cK && (n - 12 + ns - 1) / ns < 12 - c12)
            K = 12;
    }
    if (K > 12) K = 12;
    if (n <= K) K = n;
    int Rr = std::min(std::max(1, std::min(opt.reg_bits, R)), K);
    plan.Rr = Rr;
    int c = std::max(0, std::min(opt.coalesce, K - 1));   // room for at least one stage bit
    uint64_t mand = (n > K) ? ((1ull << c) - 1) : ((1ull << n) - 1);
    plan.n = n;
    plan.nl = n;
    plan.K = K;
    size_t s = 0;
    uint32_t relabel_from = 0, relabel_to = 0;   // PF_RELABEL of the last pass: register masks
    LocalMap relabel_L(0);
    // Balanced stage packing: the pass over the low (contiguous) bits takes K
    // stages, and the strided passes share the other n - K stages evenly, so
    // the tile bits they leave unused extend the coalescing run (the fill
    // below adds low bits): n = 31 (K = 11) packs 7+7+6+11 stages with 256-,
    // 256- and 512-byte runs instead of 8+8+8+7 with 128-byte runs, n = 28
    // (K = 12) packs 8+8+12 with 256-byte runs instead of 9+9+10, n = 33
    // (K = 11) 8+7+7+11 instead of 8+8+8+9.  B200, same box: QFT(28) 5.68 ->
    // 4.92 ms, QFT(31) 59.0 -> 48.9 ms, QFT(33) 240.9 -> 223.1 ms; the pass
    // count is the greedy one and n = 30 (9+9+12) is unchanged
    // (profiles/r02/ab_qft_balance.jsonl).
    std::vector<size_t> cap;
    size_t qpass = 0;
    if (n > K && !getenv("LQ_QFT_GREEDY")) {   // (A/B switch)
        const int np = count_passes(K), ns = np - 1;
        // (fewer stages in the contiguous pass and 256-byte instead of 512-byte
        // runs in the strided ones measured the same: n = 31, 7+7+7+10 vs
        // 7+7+6+11 at K = 11, 48.9 vs 48.7 ms, profiles/r02/ab_qft_balance.jsonl)
        const int Lc = K, S = n - Lc;
        const bool low_first = phys(js.front()) < phys(js.back());
        if (ns > 0 && S > 0 && (S + ns - 1) / ns <= K - c) {
            for (int p = 0; p < ns; p++) cap.push_back((size_t)(S / ns + (p < S % ns ? 1 : 0)));
            if (low_first) cap.insert(cap.begin(), (size_t)Lc);
            else cap.push_back((size_t)Lc);
        }
    }
    while (s < js.size()) {
        uint64_t Tm = mand;
        std::vector<int> st;
        const size_t cap_p = qpass < cap.size() ? cap[qpass] : (size_t)K;
        qpass++;
        while (s < js.size() && st.size() < cap_p && popc(Tm | bit(phys(js[s]))) <= K) {
            Tm |= bit(phys(js[s]));
            st.push_back(js[s]);
            s++;
        }
        for (int b = 0; b < n && popc(Tm) < K; b++) Tm |= bit(b);
        LocalMap L(Tm);
        int lowrun = (n > K) ? lowrun_of(L) : 0;
        PlanPass pp;
        pp.kind = PASS_TILE;
        pp.kp.n = n;
        pp.kp.nl = n;
        pp.kp.K = K;
        memset(pp.kp.lpos, 255, sizeof(pp.kp.lpos));
        memcpy(pp.kp.T, L.T, MAXK);
        pp.kp.sub_begin = (uint32_t)plan.subs.size();
        pp.kp.perm_begin = pp.kp.perm_end = (uint32_t)plan.perms.size();
        pp.kp.store_perm = -1;
        pp.kp.eterm_begin = pp.kp.eterm_end = (uint32_t)plan.eterms.size();
        pp.n_ops = (int)st.size();
        std::vector<uint32_t> Sms;
        for (size_t a = 0; a < st.size(); a += Rr) {
            uint32_t Sm = 0;
            for (size_t b = a; b < std::min(st.size(), a + Rr); b++) Sm |= 1u << L.loc[phys(st[b])];
            Sms.push_back(fill_S(Sm, K, Rr, lowrun));
        }
        uint32_t lane_forbid = (uint32_t)((1u << std::min(lowrun, 3)) - 1);
        uint32_t top = 0;
        for (int b = K - 1; b >= 0 && popc(top) < Rr; b--) top |= 1u << b;
        uint32_t Sl = Sms.front(), Ss = Sms.back();
        if (Sl & lane_forbid) Sl = top;
        // The last sub-block's registers hold lane bits the store must
        // coalesce over (the contiguous final pass: stages on bits 3..0).
        // Instead of a store exchange through shared memory, the last pass
        // stores the registers at the positions of the `top` mapping and the
        // plan relabels the qubits (the QFT already ends in a relabel, its
        // bit reversal): QFT(30) 23.35 -> 22.6 ms.
        if ((Ss & lane_forbid) && s == js.size() && !getenv("LQ_QFT_NO_RELABEL")) {   // (A/B switch)
            relabel_from = Ss;
            relabel_to = top;
            relabel_L = L;
            pp.kp.flags |= PF_RELABEL;
            Ss = top;
        } else if (Ss & lane_forbid) {
            Ss = top;
        }
        mask_to_S(Sl, pp.kp.Sload);
        mask_to_S(Ss, pp.kp.Sstore);
        for (size_t a = 0, blk = 0; a < st.size(); a += Rr, blk++) {
            KSub sb{};
            mask_to_S(Sms[blk], sb.S);
            sb.perm = -1;
            sb.op_begin = (uint32_t)plan.kops.size();
            for (size_t b = a; b < std::min(st.size(), a + Rr); b++) {
                int j = st[b], p = phys(j);
                KOp k{};
                k.type = K_QFT;
                k.r0 = NOREG;
                k.r1 = NOREG;
                for (int i = 0; i < Rr; i++) if (sb.S[i] == L.loc[p]) k.r0 = (uint8_t)i;
                k.b0 = (uint8_t)p;
                k.qj = (uint8_t)j;
                k.flags = (inverse ? QF_INVERSE : 0) | (layout_rev ? QF_REVERSED : 0);
                // register twiddle table: exp(+-i pi (logical(goff_v) mod 2^j) / 2^j)
                double tab[2 * NREG];
                for (int v = 0; v < NREG; v++) {
                    uint64_t goff = 0;
                    for (int i = 0; i < Rr; i++) if (v & (1 << i)) goff |= bit(L.T[sb.S[i]]);
                    uint64_t lg = layout_rev ? brev_n(goff, n) : goff;
                    uint64_t Lm = (j == 0) ? 0 : (lg & (bit(j) - 1));
                    long double ang = (long double)3.141592653589793238462643383279502884L *
                                      (long double)Lm / ldexpl(1.0L, j);
                    double sgn = inverse ? -1.0 : 1.0;
                    tab[2 * v] = (double)cosl(ang);
                    tab[2 * v + 1] = sgn * (double)sinl(ang);
                }
                k.mat = (uint32_t)mb.add_const(tab, NREG);
                k.tdep = 0x80;
                k.qi = NOREG;
                for (int i = 0; i < Rr; i++) {
                    const int p = L.T[sb.S[i]], l = layout_rev ? n - 1 - p : p;
                    if (l < j) k.tdep |= (uint8_t)(1u << i);
                    if (l == j - 1) k.qi = (uint8_t)i;
                }
                if (b == a) k.flags |= QF_HEAD;
                int jmax = 0;
                for (size_t b2 = a; b2 < std::min(st.size(), a + Rr); b2++) jmax = std::max(jmax, st[b2]);
                k.b1 = (uint8_t)jmax;
                plan.kops.push_back(k);
            }
            if (a + Rr >= st.size()) {
                KOp k{};
                k.type = K_SCALE;
                k.r0 = k.r1 = NOREG;
                double sc[2] = {std::pow(0.5, 0.5 * (double)st.size()), 0.0};
                k.mat = (uint32_t)mb.add_const(sc, 1);
                plan.kops.push_back(k);
            }
            sb.op_end = (uint32_t)plan.kops.size();
            plan.subs.push_back(sb);
        }
        pp.kp.sub_end = (uint32_t)plan.subs.size();
        finalize_pass_tables(pp, plan);
        plan.passes.push_back(pp);
        plan.n_tile++;
    }
    // new layout
    bool final_rev = ident;   // the layout flips
    for (int q = 0; q < n; q++) qmap[q] = final_rev ? q : n - 1 - q;
    if (relabel_from) {
        // PF_RELABEL: local bit b of the last pass's tile goes to pi(b) --
        // register bits in order onto relabel_to's, the rest in order onto
        // the rest (tile.cuh, the store of tile_body / tile_body_static)
        int pi[MAXK];
        int rf = 0, rt = 0, nf = 0, nt = 0;
        int to_reg[MAXK], to_oth[MAXK];
        for (int b = 0; b < K; b++) ((relabel_to >> b) & 1 ? to_reg[rt++] : to_oth[nt++]) = b;
        for (int b = 0; b < K; b++) pi[b] = (relabel_from >> b) & 1 ? to_reg[rf++] : to_oth[nf++];
        for (int q = 0; q < n; q++) {
            const int p = qmap[q];
            const int b = relabel_L.loc[p];
            if (b >= 0 && b < K) qmap[q] = relabel_L.T[pi[b]];
        }
    }
    return true;
}

std::string describe(const Plan &plan) {
    std::ostringstream os;
    os << "n=" << plan.n << " K=" << plan.K << " passes=" << plan.passes.size()
       << " (tile " << plan.n_tile << ", pair " << plan.n_pair << ", diag " << plan.n_diag
       << ") folded_perm_gates=" << plan.n_folded << "\n";
    for (size_t i = 0; i < plan.passes.size(); i++) {
        const PlanPass &p = plan.passes[i];
        if (p.kind == PASS_TILE) {
            os << "  [" << i << "] TILE ops=" << p.n_ops << " subs=" << (p.kp.sub_end - p.kp.sub_begin) << " T={";
            for (int k = 0; k < p.kp.K; k++) os << (int)p.kp.T[k] << (k + 1 < p.kp.K ? "," : "");
            os << "}";
            if (p.oop) {   // relabelling store: where the tile's bits go in the next frame
                os << " -> {";
                for (int k = 0; k < p.kp.K; k++) os << (int)p.spos[p.kp.T[k]] << (k + 1 < p.kp.K ? "," : "");
                os << "}";
            }
            os << (p.kp.flags & PF_NO_STORE ? " ro" : "") << "\n";
        } else {
            os << "  [" << i << "] " << (p.kind == PASS_PAIR ? "PAIR" : "DIAG") << " ops=" << p.n_ops << "\n";
        }
    }
    return os.str();
}

std::string export_json(const Plan &plan, const MatBuilder &mb, const int32_t *qmap) {
    std::ostringstream o;
    o.precision(17);
    auto arr = [&](const char *name, size_t cnt, auto f) {
        o << "\"" << name << "\":[";
        for (size_t i = 0; i < cnt; i++) { if (i) o << ","; f(i); }
        o << "]";
    };
    o << "{\"n\":" << plan.n << ",\"nl\":" << plan.nl << ",\"K\":" << plan.K << ",\"Rr\":" << plan.Rr << ",\"n_slots\":" << plan.n_slots
      << ",\"mat_size\":" << mb.mat_size << ",";
    arr("qmap", (size_t)plan.n, [&](size_t i) { o << qmap[i]; });
    o << ",";
    arr("passes", plan.passes.size(), [&](size_t i) {
        const PlanPass &p = plan.passes[i];
        const KPass &k = p.kp;
        o << "{\"kind\":" << (int)p.kind << ",\"op_begin\":" << p.op_begin << ",\"op_end\":" << p.op_end
          << ",\"K\":" << k.K << ",\"sub_begin\":" << k.sub_begin << ",\"sub_end\":" << k.sub_end
          << ",\"kop_begin\":" << k.op_begin << ",\"kop_end\":" << k.op_end << ",\"perm_begin\":" << k.perm_begin
          << ",\"store_perm\":" << k.store_perm << ",\"eterm_begin\":" << k.eterm_begin << ",\"eslot\":" << k.eslot
          << ",\"flags\":" << k.flags << ",\"lpos\":[";
        for (int b = 0; b < 64; b++) o << (b ? "," : "") << (int)k.lpos[b];
        o << "],\"T\":[";
        for (int b = 0; b < (p.kind == PASS_TILE ? k.K : 0); b++) o << (b ? "," : "") << (int)k.T[b];
        o << "],\"Sstore\":[" << (int)k.Sstore[0] << "," << (int)k.Sstore[1] << "," << (int)k.Sstore[2] << ","
          << (int)k.Sstore[3] << "],\"oop\":" << (p.oop ? 1 : 0) << ",\"spos\":[";
        for (int b = 0; b < (p.oop ? plan.nl : 0); b++) o << (b ? "," : "") << (int)p.spos[b];
        o << "]}";
    });
    o << ",";
    arr("subs", plan.subs.size(), [&](size_t i) {
        const KSub &sb = plan.subs[i];
        o << "{\"S\":[" << (int)sb.S[0] << "," << (int)sb.S[1] << "," << (int)sb.S[2] << "," << (int)sb.S[3]
          << "],\"op_begin\":" << sb.op_begin << ",\"op_end\":" << sb.op_end << ",\"perm\":" << sb.perm << "}";
    });
    o << ",";
    arr("kops", plan.kops.size(), [&](size_t i) {
        const KOp &k = plan.kops[i];
        o << "{\"type\":" << (int)k.type << ",\"code\":" << (int)k.code << ",\"r0\":" << (int)k.r0 << ",\"r1\":"
          << (int)k.r1 << ",\"rcm\":" << (int)k.rcm << ",\"b0\":" << (int)k.b0 << ",\"b1\":" << (int)k.b1
          << ",\"flags\":" << (int)k.flags << ",\"cmask\":" << k.cmask << ",\"mat\":" << k.mat << ",\"aux\":" << k.aux
          << ",\"qj\":" << (int)k.qj << "}";
    });
    o << ",";
    arr("perms", plan.perms.size(), [&](size_t i) {
        const KPerm &p = plan.perms[i];
        o << "{\"col\":[";
        for (int b = 0; b < plan.K; b++) o << (b ? "," : "") << p.col[b];
        o << "],\"term_begin\":" << p.term_begin << ",\"term_end\":" << p.term_end << "}";
    });
    o << ",";
    arr("perm_terms", plan.perm_terms.size(), [&](size_t i) {
        o << "[" << plan.perm_terms[i].cmask << "," << plan.perm_terms[i].vec << "]";
    });
    o << ",";
    arr("eterms", plan.eterms.size(), [&](size_t i) {
        const ETerm &e = plan.eterms[i];
        o << "[" << e.c << "," << e.znr << "," << e.zreg << "," << e.y << "]";
    });
    o << ",";
    arr("specs", mb.specs.size(), [&](size_t i) {
        const MSpec &m = mb.specs[i];
        o << "[" << m.out << "," << m.f_begin << "," << m.f_end << "," << m.form << "]";
    });
    o << ",";
    arr("factors", mb.factors.size(), [&](size_t i) {
        const MFactor &f = mb.factors[i];
        o << "[" << f.kind << "," << f.pidx << "," << f.angle << "," << f.cst << "]";
    });
    o << ",";
    arr("cst", mb.cst.size(), [&](size_t i) { o << mb.cst[i]; });
    o << ",";
    arr("wide_groups", plan.wide_groups.size(), [&](size_t i) { o << plan.wide_groups[i]; });
    o << ",";
    arr("groups", plan.groups.size(), [&](size_t i) {
        const PGroup &g = plan.groups[i];
        o << "{\"x\":" << g.x << ",\"terms\":[";
        for (size_t t = 0; t < g.terms.size(); t++)
            o << (t ? "," : "") << "[" << g.terms[t].c << "," << g.terms[t].z << "," << g.terms[t].y << "]";
        o << "]}";
    });
    o << "}";
    return o.str();
}

}  // namespace lq
