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
//   SWAP  : exchange k global physical bits g_0..g_{k-1} with k local
//           physical bits l_0..l_{k-1} at once (k = 1: a pairwise half-shard
//           exchange; k > 1: an all-to-all among the 2^k ranks that differ
//           in those global bits).  Rank r (physical global bits R = r ^
//           xmask) splits its shard into 2^k parts by the values b of its
//           l-bits; part b goes to the rank whose g-bits equal b and lands
//           in that rank's part a, a = r's own g-bits (part a stays).  Each
//           rank sends (2^k - 1) / 2^k of its shard.  The qubit map swaps
//           the qubits' physical positions pairwise (g_j <-> l_j).
// Uncontrolled X on a global qubit is a rank relabel (xmask), Y = X * diag(i,
// -i) a rank-constant phase plus the relabel: no data moves.  Gates that act
// non-diagonally on a global qubit first swap it in; the local victim is the
// qubit whose next non-diagonal use lies furthest ahead (Belady).  A swap
// also brings in every other global qubit whose next non-diagonal use comes
// before the next use of the local qubit it would displace (the Belady rule
// applied to the whole exchange), up to max_k qubits per exchange: one
// all-to-all instead of several pairwise swaps (the distributed QFT needs
// two).  For a QFT stage (qft_pass_stages = P > 0) the victims are instead
// the qubits needed first AFTER the next P stages: the local run then ends
// exactly at a tile-pass boundary and the second exchange brings them back,
// so the sharded QFT makes as many local passes as the unsharded one
// (ceil(n / P)) plus two exchanges.  The schedule is a pure function of its
// inputs: every rank computes the same.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "planner.h"

namespace lq {

constexpr int MAX_SWAP_K = 4;     // qubits per exchange (2^k - 1 peers)

struct DStep {
    int kind = 0;                 // 0 LOCAL, 1 SWAP
    std::vector<POp> ops;         // LOCAL
    uint32_t xmask = 0;           // rank relabel in effect (physical global bits of rank r = r ^ xmask)
    int k = 0;                    // SWAP: number of exchanged qubit pairs
    int g[MAX_SWAP_K], l[MAX_SWAP_K];   // SWAP: global / local physical bits, l ascending
    bool expv = false;            // LOCAL: evaluates a Pauli sum
    Plan plan;                    // LOCAL: planned passes (plan_steps)
};

struct Schedule {
    int n = 0, m = 0, nl = 0;
    int max_k = MAX_SWAP_K;       // qubits per exchange (1: pairwise swaps only)
    int qft_pass_stages = 0;      // QFT stages one local tile pass holds (0: plain Belady victims)
    std::vector<DStep> steps;
    MatBuilder mb;
    size_t n_swaps = 0, n_relabels = 0;
    size_t n_swapped_qubits = 0;  // sum of k over the swap steps
    double shard_fraction_sent = 0.0;   // sum over swaps of (2^k - 1) / 2^k
};

// Append a k-qubit exchange step (pairs sorted by local bit) and update the
// layout: qm[logical] = physical, at[physical] = logical (-1: none).
void push_swap(Schedule &sc, int k, const int *g, const int *l, uint32_t xmask, int32_t *qm, int *at);

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
