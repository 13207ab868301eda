// dist.h -- schedules for states sharded on their top log2 G physical bits
// (SURVEY.md §8(a) a9, §8(e) item 2).
//
// A sharded state of n qubits on G = 2^m ranks keeps 2^(n-m) amplitudes per
// rank: physical index = (global bits << nl) | local index, nl = n - m, and
// rank r holds the global bits r ^ xmask (xmask = pending rank relabel).
// A circuit becomes a list of steps:
//   LOCAL : ops whose non-diagonal bits are all local; controls and diagonal
//           factors on global bits are rank constants (the kernels OR the
//           shard's global bits, gofs, into their logic index).  Planned into
//           tile passes over the local bits like any single-GPU circuit.
//   SWAP  : exchange global physical bit g with local physical bit l: rank r
//           and its partner r ^ (1 << (g - nl)) trade the half of their
//           shard whose l-bit differs from their own g-bit; the qubit map
//           swaps the two qubits' physical positions.
// Uncontrolled X on a global qubit is a rank relabel (xmask), Y = X * diag(i,
// -i) a rank-constant phase plus the relabel: no data moves.  Gates that act
// non-diagonally on a global qubit first swap it in; the local victim is the
// qubit whose next non-diagonal use lies furthest ahead (Belady).  The
// schedule is a pure function of its inputs: every rank computes the same.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "planner.h"

namespace lq {

struct DStep {
    int kind = 0;                 // 0 LOCAL, 1 SWAP
    std::vector<POp> ops;         // LOCAL
    uint32_t xmask = 0;           // rank relabel in effect (physical global bits of rank r = r ^ xmask)
    int g = -1, l = -1;           // SWAP: global / local physical bits
    bool expv = false;            // LOCAL: evaluates a Pauli sum
    Plan plan;                    // LOCAL: planned passes (plan_steps)
};

struct Schedule {
    int n = 0, m = 0, nl = 0;
    std::vector<DStep> steps;
    MatBuilder mb;
    size_t n_swaps = 0, n_relabels = 0;
};

// Append the steps of `gates` to `sc`; qmap (logical -> physical, n entries)
// and xmask are updated to the layout after the circuit.
// Returns false (schedule unusable) if a gate cannot be made local -- only
// possible when a shard holds fewer than 3 qubits (sh_check forbids that).
bool schedule_gates(Schedule &sc, const lq_gate *gates, size_t n_gates, int32_t *qmap, uint32_t &xmask);

// Alg. 3 as n stage ops (LQK_QFT_STAGE: H(i) and the CPs
// controlled by the later qubits, one butterfly-with-twiddle each) followed
// by the SWAP layer (relabels); inverse: the reversed sequence of inverse
// stages.
std::vector<lq_gate> qft_gates(int n, bool inverse);

// LOCAL steps (expv = true) whose K_EXPV ops evaluate the Pauli sum
// (groups live in each step's plan): first every term whose
// X/Y qubits are all local, then each remaining x mask after swapping its
// global X/Y qubits in.  E = the sum over the expv steps.  Returns false if
// one term has more X/Y qubits than local bits.
bool schedule_expval(Schedule &sc, const lq_pauli_term *terms, size_t n_terms, int32_t *qmap, uint32_t &xmask);

// Plan the LOCAL steps' tile passes (restricted to the local bits).
void plan_steps(Schedule &sc, const PlanOptions &opt);

std::string schedule_json(const Schedule &sc, const int32_t *qmap, uint32_t xmask);

}  // namespace lq
