/*
 * lq.h -- C ABI of liblq.so: B200-native dense complex128 state-vector
 * simulation of parameterised circuits (the data-parallel hot path of
 * LogosQ, arXiv 2512.23183; /root/reference/PAPER.md).
 *
 * Conventions (all entry points)
 *   - A state on n qubits holds N = 2^n complex128 amplitudes (interleaved
 *     re, im doubles), the paper's DenseState of Complex64.
 *   - Qubit q <-> logical index bit n-1-q (MSB first; Alg. 1).
 *     The library may keep amplitudes in a permuted physical layout (a qubit
 *     map); every call that takes or returns indices uses LOGICAL indices.
 *   - Rotations R_G(theta) = exp(-i theta G / 2).
 *   - 2-qubit matrices act on the sub-index 2*bit(q0) + bit(q1) (q0 is the
 *     high bit).  Controlled gates list the control first.
 *   - Every call validates all arguments before any device work: a rejected
 *     call returns a negative lq_status, sets lq_last_error() and leaves the
 *     state untouched.  No exception or abort crosses this ABI.
 *   - Device work is enqueued on the handle's CUDA stream (cudaStream_t passed
 *     as void*; NULL = legacy default stream).  Calls documented "syncs"
 *     block until their results are on the host.
 *   - Handles are single-writer: do not call into one handle
 *     from two threads at once.
 *   - No CPU fallback: if no CUDA device is present every call that needs one
 *     fails with LQ_ERR_CUDA.
 */
#ifndef LQ_C_ABI_H_
#define LQ_C_ABI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LQ_VERSION 1

typedef enum {
    LQ_OK = 0,
    LQ_ERR_ARG = -1,        /* bad argument (qubit range, duplicate qubits, angle on a fixed gate, ...) */
    LQ_ERR_OOM = -2,        /* device allocation failed / state too large */
    LQ_ERR_CUDA = -3,       /* CUDA runtime error (incl. no device) */
    LQ_ERR_NCCL = -4,       /* collective failure (NCCL error, asynchronous error or timeout) */
    LQ_ERR_DIM = -5,        /* size mismatch (wrapped buffer too small, count out of range) */
    LQ_ERR_NONFINITE = -6,  /* NaN/Inf angle, parameter or coefficient */
    LQ_ERR_STATE = -7       /* handle unusable after an earlier asynchronous failure: once a call on a
                               state / gradient plan / comm returned LQ_ERR_CUDA or LQ_ERR_NCCL from
                               work it had enqueued, every later call on it returns LQ_ERR_STATE */
} lq_status;

/* Gate kinds.  Fixed gates take no angle; rotation
 * kinds take exactly one angle (literal or theta[param_idx]). */
typedef enum {
    LQ_H = 0, LQ_X, LQ_Y, LQ_Z, LQ_S, LQ_SDG, LQ_T, LQ_TDG,
    LQ_RX, LQ_RY, LQ_RZ,          /* exp(-i theta {X,Y,Z} / 2) */
    LQ_CNOT,                      /* q0 control, q1 target (Alg. 1) */
    LQ_CZ,                        /* diag(1,1,1,-1) */
    LQ_CP,                        /* diag(1,1,1,e^{i theta}) (Alg. 3 CP) */
    LQ_SWAP,
    LQ_U1,                        /* arbitrary 2x2, row-major complex128 in .mat (8 doubles) */
    LQ_U2,                        /* arbitrary 4x4 on (q0 high, q1 low), .mat (32 doubles) */
    LQ_CRY,                       /* RY(theta) on q1 when q0 = |1> (App. E circuit) */
    LQ_CCX,                       /* Toffoli: q0, q1 controls, q2 target (App. B) */
    LQ_RXX, LQ_RYY, LQ_RZZ,       /* exp(-i theta P(x)P / 2) (Trotter gates) */
    LQ_NUM_KINDS
} lq_kind;

/* One circuit operation ("Operation").  Unused qubit slots
 * are -1.  angle source: param_idx >= 0 -> theta[param_idx] (an ansatz
 * parameter); param_idx == -1 -> .angle.  Fixed gates
 * must have param_idx == -1 and angle == 0.  mat is read only for
 * LQ_U1/LQ_U2 and is borrowed for the call. */
typedef struct lq_gate {
    int32_t kind;
    int32_t q0, q1, q2;
    int32_t param_idx;
    int32_t reserved;             /* must be 0 */
    double angle;
    const double *mat;
} lq_gate;

/* Real-weighted Pauli string coeff * P, P = prod_q sigma_q:
 * bit q of x_mask / z_mask = qubit q; X: x only, Z: z only, Y: both. */
typedef struct lq_pauli_term {
    double coeff;
    uint64_t x_mask;
    uint64_t z_mask;
} lq_pauli_term;

typedef struct lq_sv lq_sv;       /* opaque state-vector handle */
typedef struct lq_psr lq_psr;     /* opaque parameter-shift gradient plan */

/* Thread-local message for the last failing call on this thread. */
const char *lq_last_error(void);
int lq_version(void);

/* Number of CUDA devices visible (0 on a host without a GPU; never fails). */
int lq_device_count(void);

/* ---- state vectors (DenseState) ---------------------- */

/* Allocate 2^n_qubits amplitudes on the current CUDA device; the library
 * owns the memory.  Contents are undefined until an init call.
 * n_qubits in [1, 40]; LQ_ERR_OOM if the device cannot hold the state. */
lq_status lq_sv_alloc(int n_qubits, void *cuda_stream, lq_sv **out);

/* Wrap caller-owned device memory (e.g. a torch complex128 tensor the
 * caller keeps alive).  bytes >= 16 * 2^n_qubits; dev_ptr 16-byte aligned.
 * The library never frees wrapped memory. */
lq_status lq_sv_wrap(int n_qubits, void *cuda_stream, void *dev_ptr, size_t bytes, lq_sv **out);

/* Free the handle (and its memory unless wrapped).  NULL is a no-op. */
lq_status lq_sv_free(lq_sv *sv);

/* Change the stream later calls enqueue on. */
lq_status lq_sv_set_stream(lq_sv *sv, void *cuda_stream);

int lq_sv_num_qubits(const lq_sv *sv);

/* Raw device pointer of the amplitudes in the current PHYSICAL layout. */
void *lq_sv_device_ptr(const lq_sv *sv);

/* Physical bit of each qubit: map_out[q] for q < n (identity = n-1-q). */
lq_status lq_sv_qubit_map(const lq_sv *sv, int32_t *map_out);

/* |k>.  k < 2^n (logical index). Resets the qubit map. */
lq_status lq_sv_init_basis(lq_sv *sv, uint64_t k);

/* Seeded random normalised state: for logical index i,
 *   x0 = splitmix64(seed ^ 2i), x1 = splitmix64(seed ^ (2i+1)),
 *   u_j = ((x_j >> 11) + 0.5) 2^-53,
 *   a_i = sqrt(-2 ln u0) (cos 2 pi u1 + i sin 2 pi u1),
 * then a /= sqrt(sum |a|^2).  splitmix64(x): z = x + 0x9E3779B97F4A7C15;
 * z = (z ^ z>>30) * 0xBF58476D1CE4E5B9; z = (z ^ z>>27) * 0x94D049BB133111EB;
 * return z ^ z>>31.  The hashes and u_j are exact; ln, sqrt, cos and sin are
 * evaluated to ~1e-16 relative error (table-driven on the device), so the
 * amplitudes match the formula to ~1e-15 relative.  Resets the qubit map. */
lq_status lq_sv_init_random(lq_sv *sv, uint64_t seed);

/* Copy amplitudes from/to host memory in LOGICAL order (syncs).
 * host buffers hold 2*count doubles (re, im).  offset + count <= 2^n. */
lq_status lq_sv_read(lq_sv *sv, uint64_t offset, uint64_t count, double *host_out);
lq_status lq_sv_write(lq_sv *sv, uint64_t offset, uint64_t count, const double *host_in);

/* Amplitudes at arbitrary logical indices (syncs); host_out: 2*count doubles. */
lq_status lq_sv_gather(lq_sv *sv, const uint64_t *idx, size_t count, double *host_out);

/* sum_i |a_i|^2 with a deterministic fixed-order reduction (syncs). */
lq_status lq_sv_norm2(lq_sv *sv, double *out);

/* Physically permute amplitudes so the qubit map is the identity
 * (natural MSB-first order in device memory). */
lq_status lq_sv_canonicalize(lq_sv *sv);

/* ---- sharded states --------------------------
 * A state too large for one GPU is split over G = 2^m ranks on its top m
 * physical bits: rank r holds the 2^(n-m) amplitudes whose global bits are
 * r ^ xmask (xmask: pending rank relabel; 0 after an init).  Gates acting
 * non-diagonally on a global qubit are preceded by a global<->local qubit
 * exchange (k global with k local qubits at once: an all-to-all among 2^k
 * ranks, chunked and in place, transfers overlapped with packing on a second
 * stream; LQ_OPT_SWAP_QUBITS); controls, diagonal gates and Pauli Z
 * factors on global qubits are rank constants; an uncontrolled X (or Y) on a
 * global qubit is a rank relabel.  Every call on a sharded handle is
 * COLLECTIVE: all ranks make the same calls with the same arguments, in the
 * same order; host results (norm, expectation, read/gather) are returned on
 * every rank.  lq_sv_write on a sharded handle writes the logical range on
 * the ranks that own it (every rank passes the same host data: checkpoint
 * restore); lq_sv_canonicalize rejects sharded handles. */
typedef struct lq_comm lq_comm;   /* NCCL communicator (one process per GPU) */

/* ncclUniqueId for lq_comm_init (len >= 128): call on rank 0 and broadcast
 * the bytes (e.g. torch.distributed.broadcast_object_list). */
lq_status lq_comm_unique_id(void *out, size_t len);
/* Join the communicator (collective over `world` processes).  NCCL is loaded
 * at run time (the copy torch already loaded, else libnccl.so.2);
 * LQ_ERR_NCCL if it is unavailable. */
lq_status lq_comm_init(const void *unique_id, size_t len, int rank, int world, lq_comm **out);
/* A communicator WITHOUT transport: (rank, world) only.  Work partitioned over
 * ranks (lq_psr_create / lq_param_shift_grad) computes this rank's share and
 * the collectives are the identity, so every host or device result is the
 * rank's PARTIAL one (gradient components it does not own are 0; E only on
 * rank 0).  For callers that reduce themselves and for testing the partition
 * on one device.  Sharded states reject it (they need a transport). */
lq_status lq_comm_init_local(int rank, int world, lq_comm **out);
/* rank, world, and whether NCCL carries data (0 for lq_comm_init_local).
 * LQ_ERR_STATE once the communicator was aborted (LQ_OPT_COMM_TIMEOUT_MS). */
lq_status lq_comm_info(const lq_comm *comm, int *rank, int *world, int *has_transport);
lq_status lq_comm_free(lq_comm *comm);

/* This process's shard of an n-qubit state on comm's ranks (world a power of
 * two, n - log2(world) >= 1); world == 1 is lq_sv_alloc.  The handle keeps
 * the comm pointer: free the state before the comm. */
lq_status lq_sv_alloc_sharded(int n_qubits, lq_comm *comm, void *cuda_stream, lq_sv **out);

/* All `world` shards of an n-qubit state in THIS process, exchanging halves
 * with device copies instead of NCCL: the same schedules and kernels on one
 * GPU (tests and single-GPU runs of the sharded data path). */
lq_status lq_sv_alloc_group(int n_qubits, int world, void *cuda_stream, lq_sv **out);

/* log2 of the number of shards (0: unsharded), rank of this process's first
 * shard, number of shards held here, current rank relabel.  NULLs allowed. */
lq_status lq_sv_shard_info(const lq_sv *sv, int *log2_world, int *first_rank, int *n_local_shards,
                           uint32_t *xmask);
/* Device pointer of local shard k (2^(n-m) amplitudes, physical local order). */
void *lq_sv_shard_ptr(const lq_sv *sv, int k);
/* Global-qubit exchanges run on this handle so far, and the bytes each rank
 * sent in them (a k-qubit exchange sends (2^k - 1) / 2^k of a shard). */
lq_status lq_sv_exchange_stats(const lq_sv *sv, uint64_t *n_exchanges, uint64_t *bytes_sent_per_rank);

/* Host-only: the distributed schedule (steps: local tile plans with the rank
 * relabel in effect, global<->local swaps) of `gates`, then an optional QFT
 * (qft = 1 forward, -1 inverse, 0 none), then an optional Pauli sum, for an
 * n-qubit state on 2^log2_world ranks starting in the identity layout, as
 * JSON (final qmap and xmask included).  *needed = buffer size required. */
lq_status lq_dist_schedule_json(int n_qubits, int log2_world, const lq_gate *gates, size_t n_gates, int qft,
                                const lq_pauli_term *terms, size_t n_terms, char *buf, size_t buf_len,
                                size_t *needed);

/* ---- circuits (Circuit::execute) ----------------------- */

/* Apply gates[0..n_gates) in order (Circuit::execute semantics).  theta
 * (host, n_theta doubles) supplies angles for gates with param_idx >= 0;
 * it may be NULL when no gate uses a parameter.  The library fuses gates
 * into shared-memory tile passes; the result equals sequential application
 * up to floating-point rounding.  SWAP gates are applied as qubit-map
 * relabels (no data movement). */
lq_status lq_apply_circuit(lq_sv *sv, const lq_gate *gates, size_t n_gates,
                           const double *theta, size_t n_theta);

/* QFT|x> = N^-1/2 sum_k e^{2 pi i x k / N}|k>, i.e.
 * Alg. 2's InverseFFT / sqrt(N) and Alg. 3's gate
 * sequence.  inverse != 0 applies QFT^-1.  Computed as
 * fused radix-2 butterfly tiles; the final bit reversal is a qubit-map
 * relabel (call lq_sv_canonicalize to materialise natural order). */
lq_status lq_qft(lq_sv *sv, int inverse);

/* ---- observables ---------------------------- */

/* E = sum_t coeff_t <psi|P_t|psi> (syncs).  Deterministic reduction. */
lq_status lq_expval_pauli_sum(lq_sv *sv, const lq_pauli_term *terms, size_t n_terms,
                              double *out_energy);

/* ---- parameter-shift gradients -------------- */

/* g_p = ( E(theta + (pi/2) e_p) - E(theta - (pi/2) e_p) ) / 2 for the ansatz
 * ansatz[0..n_gates) run from |0...0> and the Pauli sum
 * terms.  A parameter of a controlled rotation (LQ_CRY: generator
 * eigenvalues {0, +-1/2}, where the two-term rule is not exact, reading A8)
 * takes the exact four-term rule
 *   g_p = c1 (E(+pi/2) - E(-pi/2)) - c2 (E(+3pi/2) - E(-3pi/2)),
 *   c1 = (sqrt2 + 1) / (4 sqrt2), c2 = (sqrt2 - 1) / (4 sqrt2)
 * (shifts of theta_p; reading A8).  Each parameter must be used by
 * exactly one rotation gate (reading A7); all shifted circuits are
 * independent and are batched.
 * comm (nullable): with a communicator of `world`
 * ranks the call is COLLECTIVE (same arguments on every rank): rank r
 * evaluates the circuits of the parameters p with p % world == r (and rank 0
 * the unshifted circuit), then one NCCL all-reduce over the n_params + 1
 * values returns the full gradient and E(theta) on EVERY rank.  Each value
 * comes from exactly one rank (zeros elsewhere), so the result is
 * bit-identical to the 1-GPU one.  A transport-less comm
 * (lq_comm_init_local) returns the rank's partial gradient instead.
 * energy_out (nullable) receives E(theta).  Host in/out (syncs; with NCCL the
 * wait polls for asynchronous errors, LQ_OPT_COMM_TIMEOUT_MS). */
lq_status lq_param_shift_grad(int n_qubits, const lq_gate *ansatz, size_t n_gates,
                              const double *theta, size_t n_params,
                              const lq_pauli_term *terms, size_t n_terms,
                              lq_comm *comm, void *cuda_stream,
                              double *grad_out, double *energy_out);

/* lq_param_shift_grad keeps the plans (and device buffers) of its two most
 * recent distinct (circuit, Hamiltonian, shard, stream, options) arguments
 * and reuses them, and lq_apply_circuit / lq_qft / lq_expval_pauli_sum keep
 * the plans of their 32 most recent distinct (gates or terms, n, qubit
 * map, options) arguments (theta is not part of a plan); this frees both. */
lq_status lq_psr_cache_clear(void);

/* Same computation split into a reusable plan and an asynchronous run on
 * DEVICE pointers (theta_dev: n_params doubles; grad_dev: n_params doubles;
 * energy_dev: 1 double or NULL).  lq_psr_run does not sync.  Every circuit
 * starts from |0...0>: the first tile pass synthesises it,
 * and while the tiles run so far leave some qubits untouched the state is zero
 * outside their union, so passes read and run only inside it (support
 * tracking; results are bit-identical to full passes, lq_psr_pass_bytes).
 * comm: as lq_param_shift_grad -- the plan holds this rank's circuits and
 * lq_psr_run ends with the all-reduce (enqueued on the stream; the comm must
 * outlive the plan).  A plan that met an asynchronous CUDA / NCCL failure
 * returns LQ_ERR_STATE from every later run. */
lq_status lq_psr_create(int n_qubits, const lq_gate *ansatz, size_t n_gates, size_t n_params,
                        const lq_pauli_term *terms, size_t n_terms, lq_comm *comm,
                        void *cuda_stream, lq_psr **out);
lq_status lq_psr_run(lq_psr *plan, const double *theta_dev, double *grad_dev, double *energy_dev);
lq_status lq_psr_free(lq_psr *plan);
/* ---- Trotterised XYZ time evolution --- */

typedef struct lq_xyz_model {
    double jx, jy, jz;            /* couplings J_x, J_y, J_z */
    double amp, omega;            /* field h(t) = amp * sin(omega * t) */
} lq_xyz_model;

/* Evolve sv in place under H(t) = -sum_{i<n-1} (J_x X_i X_{i+1} + J_y Y_i Y_{i+1}
 * + J_z Z_i Z_{i+1}) - h(t) sum_i Z_i (Eq. 9, open chain) by n_steps
 * first-order Trotter steps of size dt starting at time t0 (Eq. 12):
 * step j applies RXX(-2 J_x dt) on every pair (i, i+1), i ascending, then
 * RYY(-2 J_y dt), then RZZ(-2 J_z dt), then RZ(-2 h(t0 + j dt) dt) on every
 * qubit (the gates of P:825-831 with the signs of Eq. 9, reading A20).  The
 * caller prepares the initial state (the paper starts from |1...1>:
 * lq_sv_init_basis(sv, 2^n - 1)).  energy_out (nullable, host):
 * E(t) = <psi(t)|H(t)|psi(t)> (Eq. 13) at t0 and after every record_every
 * steps -- 1 + n_steps / record_every values.  Sharded states are supported
 * (the gates go through the usual scheduler).  LQ_ERR_ARG for n < 2, dt <= 0,
 * n_steps < 0 or record_every < 1; LQ_ERR_NONFINITE for a non-finite model. */
lq_status lq_trotter_xyz(lq_sv *sv, const lq_xyz_model *model, double t0, double dt, int n_steps,
                         int record_every, double *energy_out);

/* ---- VQE outer loop ---------------- */

/* Adam settings.  The paper fixes lr = 1e-2, at most 350 iterations and a
 * convergence tolerance of 1e-7; beta1 = 0.9, beta2 = 0.999,
 * eps = 1e-8 are Adam's standard constants. */
typedef struct lq_adam_cfg {
    double lr, beta1, beta2, eps, tol;
    int32_t max_iter;
    int32_t reserved;             /* must be 0 */
} lq_adam_cfg;

/* Minimise E(theta) = <0|U(theta)^+ H U(theta)|0> for the ansatz and Pauli
 * sum (same rules as lq_param_shift_grad) with Adam on parameter-shift
 * gradients: for t = 0, 1, ...: evaluate E_t and g_t at theta^t (one batched
 * gradient, "2 N_theta circuit evaluations per gradient");
 * stop if t >= 1 and |E_t - E_{t-1}| < tol, or t == max_iter; otherwise
 * theta^{t+1} = theta^t - lr m_hat / (sqrt(v_hat) + eps) with
 * m = beta1 m + (1 - beta1) g, v = beta2 v + (1 - beta2) g^2,
 * m_hat = m / (1 - beta1^{t+1}), v_hat = v / (1 - beta2^{t+1}).
 * theta: host, in/out (n_params; the final iterate).  energy_trace
 * (nullable, host, >= max_iter + 1 entries): E_0 .. E_T.  iters_out
 * (nullable): T = number of Adam updates taken.  One GPU; syncs every
 * iteration (8 bytes).  LQ_ERR_NONFINITE for non-finite settings, theta or
 * an energy (with its iteration index in lq_last_error). */
lq_status lq_vqe_adam(int n_qubits, const lq_gate *ansatz, size_t n_gates, double *theta, size_t n_params,
                      const lq_pauli_term *terms, size_t n_terms, const lq_adam_cfg *cfg, void *cuda_stream,
                      double *energy_trace, int32_t *iters_out);

/* Accounting for one lq_psr_run on this shard: circuits evaluated, kernel
 * launches issued (by the last run), bytes of the uploaded plan, tile passes
 * per circuit.  Any output pointer may be NULL. */
lq_status lq_psr_stats(const lq_psr *plan, uint64_t *n_circuits, uint64_t *n_launches, uint64_t *plan_bytes,
                       uint64_t *tile_passes);
/* Algorithmic HBM bytes ONE circuit of the plan moves: through tile passes
 * (16 B/amp per load, 16 B/amp per store; the first pass synthesises
 * |0...0> without a load, read-only and final passes skip the store) and
 * through other kernels (pair/diag passes, wide Pauli groups).  Either
 * pointer may be NULL.  This is the numerator of the roofline bench.py
 * reports. */
lq_status lq_psr_traffic(const lq_psr *plan, uint64_t *tile_bytes_per_circuit, uint64_t *other_bytes_per_circuit);

/* The same per launched pass, in launch order: bytes_out[i] = algorithmic
 * HBM bytes of pass i for one circuit, kind_out[i] = 0 tile / 1 pair / 2
 * diagonal.  Passes of a zero-first plan under support tracking (lq_psr_run:
 * while the union U of the tiles run so far misses some local bits, the state
 * is zero at every index outside U, a pass reads only the indices inside U and
 * runs only the tiles whose free bits lie in U) count only those reads and
 * tiles.  support_amps_out (may be NULL) receives the amplitudes per circuit
 * the pass's gates act on: 2^n, or fewer for a pass that runs only the tiles
 * inside its support (the others are provably zero); ops_out (may be NULL)
 * the planner ops fused into the pass (fused gates, Pauli groups).
 * Fills min(cap, *n_passes) entries; cap may be 0 to query the count. */
lq_status lq_psr_pass_bytes(const lq_psr *plan, uint64_t *bytes_out, int32_t *kind_out, uint64_t *support_amps_out,
                            uint32_t *ops_out, size_t cap, size_t *n_passes);

/* The tile bit set of each launched pass of the plan (bit b set = physical
 * bit b is in the pass's tile; 0 for pair / diagonal passes), in launch
 * order; fills min(cap, *n_passes) entries. */
lq_status lq_psr_pass_tiles(const lq_psr *plan, uint64_t *tile_masks_out, size_t cap, size_t *n_passes);

/* Measurement: the access-pattern ceiling of a tile pass.  Sweeps the
 * 2^n_bits complex128 amplitudes of dev_buf (bytes >= 16 * 2^n_bits; the
 * contents are scrambled) in place, tile by tile -- a tile = the amplitudes
 * whose bits outside tile_mask (4..12 bits) are fixed -- with the tile
 * kernel's access pattern and no arithmetic (read 16 B + write 16 B per
 * amplitude); *ms_per_sweep = mean time of `reps` sweeps after a warm-up
 * (CUDA events on cuda_stream; syncs).  HBM3e serves short runs at large
 * strides below its copy rate: this is the bandwidth a pass with that tile
 * set can reach. */
lq_status lq_tile_sweep(void *dev_buf, size_t bytes, int n_bits, uint64_t tile_mask, int reps, void *cuda_stream,
                        double *ms_per_sweep);

/* ---- execution options (testing / measurement) -------------------------- */
typedef enum {
    LQ_OPT_FUSION = 0,     /* 1 (default): tile-fused passes; 0: one pass per gate (pair/diag kernels) */
    LQ_OPT_TILE_BITS = 1,  /* tile size K in bits (default 0 = automatic) */
    LQ_OPT_COALESCE_BITS = 2, /* low physical bits every strided tile includes (default 3) */
    LQ_OPT_REG_BITS = 3,      /* amplitudes per thread in tile passes = 2^value, 2..4 (default 4;
                                 states under 9 qubits use down to 2 so a tile spans more threads) */
    LQ_OPT_KERNEL_TIMING = 4, /* 1: bracket every launch with CUDA events on its stream (lq_kernel_timing) */
    LQ_OPT_JIT = 5,           /* tile passes as per-plan specialised kernels compiled with NVRTC for
                                 sm_100a (cached per process) instead of the op-list interpreter kernel;
                                 both execute the same device op templates (tile.cuh).  0: off;
                                 1 (default): auto -- PSR plans and states with n >= 26; 2: always. */
    LQ_OPT_PASS_BUDGET = 6,   /* planner, parameter-shift plans: estimated FP64 instructions per amplitude
                                 (x10) a tile pass may absorb before it stops (default 400; 0 = no limit) */
    LQ_OPT_FIRST_PASS_FREE = 7, /* PSR plans: 1 (default) exempts the first pass -- it synthesises |0...0>,
                                 so every tile but one is stored as zeros without arithmetic -- from
                                 the pass budget; 0: budget it like the others */
    LQ_OPT_POISON_ALLOC = 8,  /* testing: 1 fills every fresh library work allocation (PSR state batches,
                                 scratch, staging) with 0xFF bytes (NaN doubles), so a kernel that reads
                                 memory nothing wrote fails loudly instead of seeing leftover zeros */
    LQ_OPT_COMM_TIMEOUT_MS = 9, /* host waits on work that includes NCCL operations poll the stream and
                                 ncclCommGetAsyncError; after this many ms (default 600000; 0 = forever)
                                 or on an asynchronous NCCL error the communicator is aborted and the
                                 call returns LQ_ERR_NCCL (later calls on its handles: LQ_ERR_STATE) */
    LQ_OPT_SWAP_QUBITS = 10,  /* sharded states: most global qubits one exchange may move (1..4, default
                                 4; 1 = pairwise half-shard swaps only, k > 1 = all-to-all among 2^k ranks) */
    LQ_OPT_STATE_PASS_BUDGET = 11, /* the same budget for every other plan (circuits, QFT, expectations,
                                 Trotter, sharded steps; default 800) */
    LQ_OPT_GROUP_STAGED = 12, /* testing: 1 runs group-mode exchanges (lq_sv_alloc_group) through the
                                 NCCL path's pack / unpack kernels and peer map, device copies standing
                                 in for the send / receive (default 0: in-place k_swap_parts); staging
                                 2 * G * (2^k - 1) * 16 MiB of device memory */
    LQ_OPT_RELABEL_STORES = 13, /* parameter-shift plans (JIT): 0 (default) = every tile pass updates the
                                 state in place; 3..5 = relabelling out-of-place stores -- each tile
                                 pass writes the state to a second buffer in the frame where the next
                                 pass's tile bits are the contiguous low bits (contiguous reads), its
                                 lowest `value` lane bits held by that tile (128..512-byte write runs);
                                 doubles the batch's state memory.  Same results; on config 4 it
                                 measured 2 % slower than in place */
    LQ_OPT_EXPORT_PSR = 14,   /* testing: 1 makes lq_plan_export_json plan like lq_psr_create (pass
                                 budget, first-pass exemption, relabelling stores) */
    LQ_OPT_GRAPHS = 15        /* 1 (default): parameter-shift runs (no communicator, no kernel timing)
                                 are captured as a CUDA graph on their second run with the same device
                                 pointers and replayed after; lq_vqe_adam runs its loop on the device
                                 (stopping rule and Adam step in one kernel of the graph; runs of at most
                                 2^24 amplitudes read the status once per chunk of up to 32 iterations,
                                 larger ones after every iteration).  0: plain stream launches */
} lq_option;
lq_status lq_set_option(int option, int64_t value);
int64_t lq_get_option(int option);

/* Host-only planning diagnostics (no device needed): plan `gates` on
 * n_qubits with the current options; report the number of passes, of tile
 * passes, and a text description (truncated to buf_len). */
lq_status lq_plan_describe(int n_qubits, const lq_gate *gates, size_t n_gates, uint64_t *n_passes,
                           uint64_t *n_tile, char *buf, size_t buf_len);

/* Host-only: the full plan (passes, sub-blocks, lowered ops, folded
 * permutations, Pauli-group terms, matrix specs) of `gates` followed by the
 * Pauli sum `terms` (may be empty), as JSON text.  *needed receives the
 * buffer size required (including the terminating NUL). */
lq_status lq_plan_export_json(int n_qubits, const lq_gate *gates, size_t n_gates, const lq_pauli_term *terms,
                              size_t n_terms, char *buf, size_t buf_len, size_t *needed);

/* Host-only: generate and NVRTC-compile (for sm_100a, without loading) the
 * JIT pass programs of `gates` followed by the Pauli sum `terms` (may be
 * empty).  No device needed; LQ_ERR_CUDA with the compiler log on failure. */
lq_status lq_jit_compile_check(int n_qubits, const lq_gate *gates, size_t n_gates, const lq_pauli_term *terms,
                               size_t n_terms, uint64_t *n_kernels);

/* Host-only: the same for the JIT pass programs of the QFT (inverse != 0:
 * QFT^-1) on n qubits in the identity layout. */
lq_status lq_qft_jit_compile_check(int n_qubits, int inverse, uint64_t *n_kernels);

/* Host-only: the tile-pass plan of the QFT (inverse != 0: QFT^-1) on n
 * qubits, PAPER.md:597-641 (Alg. 2/3), as JSON in the format of
 * lq_plan_export_json, with the qubit map the plan leaves behind (the bit
 * reversal and the last pass's store relabel are relabels, not data moves).
 * reversed_layout != 0 plans for the layout a forward QFT leaves (qubit q on
 * physical bit q) instead of the identity layout (qubit q on bit n-1-q); the
 * JSON's "qmap_in" is that input layout.  Same buffer protocol as
 * lq_plan_export_json (LQ_ERR_ARG for n outside [1, 40]).  No device needed:
 * the CPU tests execute these plans with tests/plan_emulator.py against the
 * oracle. */
lq_status lq_qft_plan_export_json(int n_qubits, int inverse, int reversed_layout, char *buf, size_t buf_len,
                                  size_t *needed);

/* Accumulated device time of launches made while LQ_OPT_KERNEL_TIMING was
 * on, per kernel class: 0 tile pass, 1 pair pass, 2 diagonal pass,
 * 3 Pauli expectation, 4 other, 5 global-qubit exchange of a sharded state
 * (one record per exchange step: pack, transfer and unpack on the handle's
 * stream).  Synchronises on the recorded events. */
lq_status lq_kernel_timing(int kernel_class, double *total_ms, uint64_t *count);
lq_status lq_kernel_timing_reset(void);

/* JIT compiler accounting (LQ_OPT_JIT): pass kernels compiled, cache hits,
 * total compile wall time.  Any output pointer may be NULL. */
lq_status lq_jit_stats(uint64_t *compiled, uint64_t *cache_hits, double *compile_seconds);

/* Kernel launches issued by this process so far (all entry points). */
uint64_t lq_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LQ_C_ABI_H_ */
