// lq_internal.h -- data structures shared by the host planner (planner.cpp)
// and the sm_100a kernels (kernels.cuh).  Product code; shares nothing with
// oracle/.
//
// Execution model.  A state of n qubits is 2^n complex128
// amplitudes in HBM.  Work is a list of PASSES; each pass streams the whole
// state through the SMs exactly once (32 B/amp of HBM traffic) and applies
// many gates on the way:
//
//   TILE pass  : a CTA owns one tile = the 2^K amplitudes whose index bits
//                outside the tile-bit set T are fixed.  Each thread keeps
//                2^R amplitudes in registers (the "register bits" S of the
//                current sub-block); gates whose target bits lie in S are
//                applied in registers; sub-blocks with different S exchange
//                amplitudes through shared memory.  Controls and diagonal
//                factors on bits outside S are thread constants, so they
//                never constrain T.
//   PAIR pass  : one 1q/2q gate on arbitrary bits, strided pairs/quads with
//                16-byte loads (a4).
//   DIAG pass  : any number of diagonal/phase gates on any bits (a3).
//
// Physical bit p of an amplitude index holds logical qubit q with
// qmap[q] = p (identity: p = n-1-q).
#pragma once
#ifdef __CUDACC_RTC__   // JIT (NVRTC): no host headers
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
#else
#include <cstddef>
#include <cstdint>
#endif

#ifdef __CUDACC__
#define LQ_HD __host__ __device__
#else
#define LQ_HD
#endif

namespace lq {

constexpr int R = 4;          // register bits per thread: 16 amplitudes in registers
constexpr int NREG = 1 << R;
constexpr int MAXK = 14;      // max tile bits (2^14 * 16 B = 256 KiB > smem; 13 is the practical max)
constexpr uint8_t NOREG = 0xFF;

enum KOpType : uint8_t {
    K_U1 = 0,   // general 2x2 on register bit r0 (mat: U00 U01 U10 U11)
    K_D1 = 1,   // diagonal (d0, d1) on one bit: register r0, or thread-constant physical bit b0
    K_X = 2,    // X-type permutation on register bit r0 (CNOT/CCX/X)
    K_U2 = 3,   // general 4x4 on register bits (r0 high, r1 low)
    K_D2 = 4,   // diagonal on two bits (r0|b0 high, r1|b1 low): mat d[4]
    K_SWAP = 5, // exchange register bits r0, r1
    K_QFT = 6,  // QFT stage on register bit r0 (logical bit qj); aux = twiddle table
    K_SCALE = 7, // multiply every amplitude by `scale`
    K_EXPV = 8,  // Pauli-group expectation contribution (read-only; see ETerm)
    K_G = 9,     // scaled 2x2 rotation on register bit r0 (RY / RX / H, see GKind)
    K_DT = 10,   // run of uncontrolled register-bit diagonals as one 16-entry phase table (flags = count;
                 // mat = offset in cst of the members' (register position, table offset) pairs)
    K_GG = 11    // RXX / RYY: scaled rotation on the register pairs (v, v ^ (r0 | r1)) (GK_IMAG table;
                 // flags & GG_YY: RYY, whose 00<->11 pairs rotate the other way)
};
constexpr uint8_t GG_YY = 1;

// Scaled rotation families (K_G; qj holds the family).  Every matrix is
// lambda * M with M having unit entries, so an amplitude pair costs 4 DFMA
// (or 4 DADD) instead of 16 FP64 ops; lambda is a real scalar the kernel
// defers.  Table: [0] = (p, lambda), [1] = (variant, 0).
//   GK_REAL (RY):  variant 0: M = [[1, -p], [p, 1]]   (p = tan(theta/2), lambda = cos)
//                  variant 1: M = [[p, -1], [1, p]]   (p = cot(theta/2), lambda = sin)
//   GK_IMAG (RX):  variant 0: M = [[1, -ip], [-ip, 1]]; variant 1: M = [[p, -i], [-i, p]]
//   GK_HAD  (H):   M = [[1, 1], [1, -1]], lambda = 1/sqrt(2)
enum GKind : uint8_t { GK_REAL = 0, GK_IMAG = 1, GK_HAD = 2 };

// Internal factor kinds (beyond lq_kind) used by the matrix builder.
constexpr int FK_YDIAG = 100;   // diag(i, -i): Y = X * diag(i, -i)
// Internal gate kind (never accepted at the ABI): one QFT stage of Alg. 3 --
// H on qubit q0 then every CP(pi / 2^(k - q0)) controlled by qubit k > q0 --
// as a single butterfly-with-twiddle op; angle < 0: the inverse stage.
constexpr int LQK_QFT_STAGE = 200;

enum KOpFlags : uint8_t {
    QF_INVERSE = 1,   // inverse stage (conj twiddle before the butterfly)
    QF_REVERSED = 2,  // layout is bit-reversed (logical index = brev(physical))
    QF_HEAD = 4,      // first QFT op of its sub-block: compute the thread twiddle for j = b1
    QF_GENERAL = 8,   // any layout: logical index from the pass's physical->logical map (KPass::lpos)
    QF_SCALE = 16,    // the stage carries its own 1/sqrt(2) (deferred into the tile scalar)
    QF_LGSET = 32     // QF_GENERAL head: the caller (JIT program) already put the thread's logical
                      // index into TState::lg with the pass's compile-time bit map
};

// One op inside a sub-block.  Controls on register bits are the register
// mask rcm (all must be 1); controls on other bits are the physical mask
// cmask, a thread constant.  `code` selects a specialised code path in the
// tile kernel (CodeTile); C_GENERIC falls back to a switch on `type`.
struct KOp {
    uint8_t type;
    uint8_t code;
    uint8_t r0, r1;      // register positions (NOREG if not a register bit)
    uint8_t rcm;         // register-position control mask
    uint8_t b0, b1;      // physical bits for thread-constant diagonal bits (QFT: b1 = largest j of the sub-block)
    uint8_t flags;       // QF_*
    uint64_t cmask;      // physical non-register control mask
    uint32_t mat;        // source of the op's table (double2 units): per-circuit matrix block, or cst
    uint32_t aux;        // where the kernel stages that table in shared memory (pass-local, double2 units)
    uint8_t qj;          // QFT: logical bit j of the stage
    uint8_t tdep;        // QFT: 0x80 | register positions whose logical bit is below j (the
                         // only ones the register twiddle depends on); 0: unknown
    uint8_t qi;          // QFT: register position of logical bit j - 1 when it is in tdep (its
                         // twiddle factor is exactly +-i), else NOREG
    uint8_t pad[5];
};
static_assert(sizeof(KOp) == 32, "KOp layout");

// Specialised tile-kernel code paths.
enum CodeTile : uint8_t {
    C_U1 = 0,        // + r0 (0..3): general 2x2, no register control
    C_X = 4,         // + r0: X, no register control
    C_CX = 8,        // + 4*c + t: X on register t controlled by register c
    C_D1R = 24,      // + r0: diagonal on a register bit, no register control
    C_D1T = 28,      // diagonal on a thread-constant bit, no register control
    C_QFT = 29,      // + r0
    C_SCALE = 33,
    C_GENERIC = 34,
    C_EXPV = 35,     // Pauli group: rcm = x mask in register positions, mat/aux = ETerm range
    C_G = 36,        // + 4*GKind + r0: scaled rotation on a register bit, no register control
    C_D1U = 48,      // diagonal on a bit outside the tile, controls outside the tile (tile-uniform factor)
    C_DT = 49,       // K_DT phase table
    C_GG = 50,       // + pair index of (r0, r1): (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)
    C_NUM = 56
};

// KOp.flags bits for diagonal ops (QF_* are QFT-only)
enum KOpDiagFlags : uint8_t {
    OF_UNIFORM = 8,   // every control bit lies outside the tile: the op acts alike on all threads of a tile
    OF_OUTSIDE = 16   // the target bit lies outside the tile
};

// One Pauli term of a group lowered to a sub-block:
// contribution c * Re[ i^y sum_v chi_zreg(v) conj(a[v ^ x]) a[v] ]
// times the thread-constant sign (-1)^{popcount(gbase & znr)}.
struct ETerm {
    double c;
    uint64_t znr;        // z bits that are not register bits (physical)
    uint32_t zreg;       // z bits in register positions
    uint32_t y;          // number of Y factors mod 4
};

struct KSub {
    uint8_t S[R];        // local bit positions held in registers (ascending)
    uint32_t op_begin, op_end;
    int32_t perm;        // entry permutation (pass-local index into the KPerm list), -1: none
};

// An affine permutation of the tile's local index, folded into a shared
// memory exchange: gates X, CNOT, SWAP, and multi-controlled X whose
// controls are tile constants map basis state |l> to |A l + b> over GF(2).
// The kernel reads register slot l' of the next mapping from position
// P^-1(l') = Ainv l' + binv, binv = sum over terms with (tile & cmask) ==
// cmask of vec.  Permutation gates folded this way cost no instructions
// beyond the exchange itself.
struct KPerm {
    uint16_t col[MAXK];  // columns of Ainv (local bit masks)
    uint32_t term_begin, term_end;
    uint32_t pad;        // keeps sizeof a multiple of 8 (KPermTerm follows in shared memory)
};
static_assert(sizeof(KPerm) % 8 == 0, "KPerm alignment");
struct KPermTerm {
    uint64_t cmask;      // physical tile-constant condition bits (0 = always)
    uint32_t vec;        // local translation (already multiplied by Ainv)
    uint32_t pad;
};

enum PassFlags : uint32_t {
    PF_LOAD_ZERO = 1,    // synthesise |0...0> instead of loading (fused init_basis(0))
    PF_EXPV = 2,         // the pass evaluates Pauli groups: write one partial sum per tile
    PF_NO_STORE = 4,     // the state after the pass is not needed (read-only pass / final PSR pass)
    PF_RELABEL = 8       // store without the store exchange: register i of the last mapping goes to the
                         // i-th register bit of Sstore and its other bits, in order, to Sstore's other
                         // bits -- a permutation of the tile's local bits the plan absorbs into the
                         // qubit map (plan_qft's last pass)
};

// Tile pass descriptor, passed by value to the kernel.
constexpr int MAX_PASS_OPS = 192;  // ops staged in shared memory per tile pass

// table size (double2) an op stages in shared memory
LQ_HD inline int op_table_size(uint8_t type) {
    switch (type) {
    case K_U1: return 4;
    case K_D1: return 3;      // d0, d1, d1/d0
    case K_U2: return 16;
    case K_D2: return 4;
    case K_QFT: return 16;
    case K_SCALE: return 1;
    case K_G: return 2;
    case K_GG: return 2;
    case K_DT: return 17;     // prod d0, then T[v] = prod over members with bit set of d1/d0
    default: return 0;
    }
}

struct KPass {
    int32_t n;           // index bits of the (logical) state
    int32_t nl;          // index bits held locally (n - log2 G for a sharded state, else n)
    uint64_t gofs;       // physical global bits of this shard (OR-ed into the logic index, never into addresses)
    int32_t K;           // tile bits
    uint32_t sub_begin, sub_end;
    uint32_t op_begin, op_end;   // contiguous op range of the pass
    uint32_t smat;       // staged table size (double2)
    uint32_t perm_begin, perm_end;   // KPerm range of the pass (global indices)
    int32_t store_perm;  // permutation applied before the store (pass-local), -1: none
    uint32_t eterm_begin, eterm_end;   // ETerm range of the pass (global indices)
    uint32_t eslot;      // first partial-sum slot of the pass (one per tile)
    uint32_t flags;
    uint8_t T[MAXK];     // physical bit of each local bit, ascending
    uint8_t Sload[R];    // (unused by the persistent kernel; kept for layout)
    uint8_t Sstore[R];   // local bits of the register mapping used for the HBM store
    uint8_t pad[6];
    uint8_t lpos[64];    // QFT stages (QF_GENERAL): logical bit held by physical bit p (255: none)
};

// Constant-bank op tables (JIT passes): pass p's staged
// tables for circuit c live at out + c * smat in the staging buffer and are
// copied to the pass module's __constant__ lqj_ctab before its launch.
struct CtabDesc {
    uint32_t op_begin, op_end;   // the pass's ops (global kop indices)
    uint32_t smat;               // staged table size of one circuit (double2)
    uint32_t out;                // offset of circuit 0's tables in the staging buffer (double2)
};

// Matrix construction (device-side, per circuit): every fused op has a
// MSpec that multiplies its factor gates (later factors on the left).
enum MForm : uint8_t { MF_U2x2 = 0, MF_DIAG2 = 1, MF_U4x4 = 2, MF_DIAG4 = 3, MF_G = 4 };

// Factor kinds use lq_kind numbering for gates; the angle is theta[pidx]
// (+ the circuit's shift if pidx is the shifted parameter) or `angle`.
struct MFactor {
    int32_t kind;
    int32_t pidx;
    double angle;
    int32_t cst;         // offset of a constant matrix (U1: 4, U2: 16 double2) in cst, else -1
    int32_t pad;
};

struct MSpec {
    uint32_t out;        // output offset (double2 units) in the circuit's matrix block
    uint32_t f_begin, f_end;
    uint32_t form;       // MForm
};

// Per-circuit parameter shift (PSR): theta[pidx] += delta.
struct Shift {
    int32_t pidx;        // -1: unshifted
    int32_t pad;
    double delta;
};

// Pauli term of a wide group (direct kernel): coeff * i^yph (-1)^{popcount(j & zfull)}.
struct PTerm {
    double coeff;
    uint64_t zfull;      // physical z mask
    uint32_t zloc, xloc; // (unused)
    uint32_t yph;        // number of Y factors mod 4
    uint32_t pad;
};

}  // namespace lq
