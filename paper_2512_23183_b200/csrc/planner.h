// planner.h -- host-side gate-fusion planner.
//
// Turns a circuit (an ordered gate list) into passes over
// the state: commutation-aware first-fit tile selection, register sub-blocks
// inside each tile, 1q gate fusion, and lowering of every op into the
// register-position form the kernels execute.  Also plans the QFT stage
// passes and the Pauli-expectation tile passes
// (PAPER.md:733-734).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "lq_internal.h"
#include "../../include/lq.h"

namespace lq {

// Abstract op on physical bits, before tiling.
struct POp {
    uint8_t type = K_U1;      // KOpType
    int t0 = -1, t1 = -1;     // target bits (U1/X/QFT: t0; U2/SWAP: t0 high, t1 low; D1: t0; D2: t0 high, t1 low)
    uint64_t ctrl = 0;        // control bits (DIAG role)
    int spec = -1;            // MSpec index (matrix), -1 if none
    uint8_t qflags = 0, qj = 0;
    double scale = 1.0;
    uint64_t xm = 0, zm = 0;  // K_EXPV: group x mask, union of the terms' z masks (physical)
    int group = -1;           // K_EXPV: index into Plan::groups
    uint64_t rd = 0;          // bits read diagonally without being controls (QFT stage twiddle inputs)
    int layout = -1;          // K_QFT (QF_GENERAL): index into MatBuilder::layouts
    // Pauli generator: an uncontrolled op exp(-i t P / 2) (or P itself) with
    // P = X^gx Z^gz up to a phase.  Two such ops commute when P and P' do,
    // which the planner's blocker uses beyond the bit-mask rule (Trotter
    // chains: X(x)X rotations on overlapping pairs commute).
    bool pgen = false;
    uint64_t gx = 0, gz = 0;
    uint64_t full() const;    // bits on which the op is not diagonal
    uint64_t touch() const;   // every bit the op reads
    bool diag() const { return type == K_D1 || type == K_D2 || type == K_SCALE; }
};

// A Pauli group: the terms of a Pauli sum that share one x mask.
struct PGroup {
    uint64_t x = 0;
    struct Term { double c; uint64_t z; uint32_t y; };
    std::vector<Term> terms;
};

bool commute(const POp &a, const POp &b);

enum PassKind { PASS_TILE = 0, PASS_PAIR = 1, PASS_DIAG = 2 };

struct PlanPass {
    PassKind kind = PASS_TILE;
    KPass kp{};               // TILE: descriptor (sub range into Plan::subs)
    uint32_t op_begin = 0, op_end = 0;   // PAIR/DIAG: range into Plan::kops (physical-bit form)
    int n_ops = 0;            // user-level ops fused into this pass (for stats)
    // zero_first plans (JIT, lq_api.cu prepare()): the state entering the
    // pass is zero at every index with a local bit outside `support`, and HBM
    // holds it only at the other indices.  The pass loads those and
    // synthesises zeros for the rest; tiles whose free bits leave sup_free =
    // support minus the tile hold zeros before and after and are not launched.
    uint64_t support = ~0ull;
    uint64_t sup_free = ~0ull;
    int tiles_log2 = -1;      // popcount(sup_free) when restricted, else -1 (nl - K)
    // Relabelling out-of-place store (PlanOptions::oop, TILE passes): the pass
    // reads the state in its own frame and writes it to the other buffer of a
    // ping-pong pair with physical bit b moved to bit spos[b] -- the frame of
    // the next pass, whose tile bits are there the contiguous bits 0..K-1
    // (DESIGN.md §7).  The plan's ops after this pass are in the new frame.
    bool oop = false;
    uint8_t spos[64];
    uint64_t map_store(uint64_t m) const {   // a physical bit mask in the store frame
        if (!oop) return m;
        uint64_t r = 0;
        while (m) { int b = __builtin_ctzll(m); r |= 1ull << spos[b]; m &= m - 1; }
        return r;
    }
};

struct Plan {
    int n = 0;
    int nl = 0;               // local index bits (tile bits are chosen among [0, nl)); n for an unsharded state
    int K = 0;
    int Rr = 0;               // register bits of the tile passes
    std::vector<PlanPass> passes;
    std::vector<KSub> subs;
    std::vector<KOp> kops;
    std::vector<KPerm> perms;
    std::vector<KPermTerm> perm_terms;
    std::vector<PGroup> groups;       // Pauli groups referenced by K_EXPV ops
    std::vector<ETerm> eterms;        // their terms lowered per tile pass
    uint32_t n_slots = 0;             // partial sums per circuit (tile passes with PF_EXPV)
    std::vector<uint32_t> wide_groups;   // groups whose x mask exceeds a tile (direct kernel)
    size_t n_tile = 0, n_pair = 0, n_diag = 0;
    size_t n_folded = 0;      // permutation gates folded into exchanges
    std::vector<const void *> jit;    // per pass: JIT-compiled tile kernel (cudaKernel_t) or nullptr (jit.h)
    bool prepared = false;            // jit resolved (prepare() in lq_api.cu)
    bool zero_first = false;          // the first pass synthesises |0...0> (PSR plans: PF_LOAD_ZERO)
    bool ctab = false;                // JIT passes read op tables from a __constant__ bank (jit.cpp)
    int ctab_circ = 1;                // circuits per launch the constant tables are sized for
    std::vector<void *> jit_ctab;     // per pass: device address of its lqj_ctab, or nullptr (smem tables)
    std::vector<CtabDesc> ctab_desc;  // the passes with jit_ctab, in pass order (staging layout)
    uint32_t ctab_total = 0;          // staging buffer size (double2) for ctab_circ circuits
    uint64_t uid = 0;                 // nonzero: identity of a cached plan's device tables (lq_api.cu
                                      // re-uploads them to a state only when it changes)
    bool has_oop = false;             // some pass stores out of place (the state needs a ping-pong buffer)
    uint8_t frame[64];                // frame[b]: physical bit, after the plan, of the plan's input bit b
    uint64_t stream_tag = 0;          // the stream the plan runs on: constant banks are per module, so
                                      // JIT modules with constant tables are private to one stream
};

struct MatBuilder {
    std::vector<MSpec> specs;
    std::vector<MFactor> factors;
    std::vector<double> cst;      // constant complex entries (re, im) -- U1/U2 user matrices, QFT twiddles
    std::vector<std::vector<uint8_t>> layouts;   // physical -> logical bit maps (64 entries, 255 = none)
    uint32_t mat_size = 0;        // per-circuit matrix block size (double2 units)
    int add_spec(MForm form, const std::vector<MFactor> &f);
    int add_const(const double *re_im_pairs, int n_complex);
};

struct PlanOptions {
    int K = 0;               // tile bits (0 = automatic)
    int coalesce = 3;        // low physical bits a strided tile always holds
    bool fusion = true;      // false: one PAIR/DIAG pass per op
    int reg_bits = 4;        // register bits per thread (R); tile kernels run 2^(K-R) threads
    int n_local = 0;         // sharded state: only bits [0, n_local) are local (0 = all n bits)
    int budget = 0;          // FP64 budget of a tile pass in tenths of an instruction per amplitude (0: none)
    bool first_free = false; // the first pass starts from |0...0> (PSR plans): exempt from the budget
    int oop = 0;             // > 0: relabelling out-of-place stores (PlanPass::oop); the next tile must hold
                             // the `oop` lowest lane bits of each store (128 B runs at 3)
};

// Estimated FP64 instructions per amplitude (x10) an op costs in a tile pass.
int op_fp64_cost(const POp &o);

// Lower user gates (already validated) to POps on physical bits.  SWAP
// gates update qmap (relabel) and emit nothing.  Adjacent 1q gates on the
// same qubit are fused into one op (product of factors).
void lower_gates(int n, const lq_gate *gates, size_t n_gates, int32_t *qmap,
                 std::vector<POp> &ops, MatBuilder &mb);

// Physical SWAP ops that permute the layout `qmap` into the identity.
void canonicalize_ops(int n, int32_t *qmap, std::vector<POp> &ops);

// Plan generic passes for `ops`.
void plan_circuit(int n, const std::vector<POp> &ops, const PlanOptions &opt, MatBuilder &mb,
                  Plan &plan);

// Pauli groups of a Pauli sum (bit q of a mask = qubit q -> physical
// qmap[q]) as K_EXPV ops appended to `ops`; groups are stored in plan.groups.
void lower_pauli(int n, const int32_t *qmap, const lq_pauli_term *terms, size_t n_terms,
                 std::vector<POp> &ops, Plan &plan);

// Plan the QFT (forward or inverse) as tile passes; updates qmap (layout
// flips between identity and reversed).  Requires qmap identity or reversed.
bool plan_qft(int n, int32_t *qmap, bool inverse, const PlanOptions &opt, Plan &plan,
              MatBuilder &mb);

int auto_tile_bits(int n);

std::string describe(const Plan &plan);
std::string export_json(const Plan &plan, const MatBuilder &mb, const int32_t *qmap);

}  // namespace lq
