// lq_api.cu -- C ABI of liblq.so (include/lq.h): handles, validation,
// launch orchestration, the batched parameter-shift driver.
//
// Every numerical step runs in the kernels of kernels.cuh; this file only
// validates arguments, plans (planner.cpp), uploads plans and launches.
// There is no CPU fallback: without a CUDA device every call that needs one
// returns LQ_ERR_CUDA.
#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstddef>
#include <list>
#include <memory>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "planner.h"
#include "jit.h"
#include "dist.h"

#include <dlfcn.h>
#include <nccl.h>   // types only: the functions are resolved with dlsym (liblq loads without NCCL)

using namespace lq;

struct lq_sv;
struct lq_psr;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
std::atomic<int64_t> g_opt_fusion{1};
std::atomic<int64_t> g_opt_K{0};
std::atomic<int64_t> g_opt_coalesce{3};
std::atomic<int64_t> g_opt_regbits{4};
std::atomic<int64_t> g_opt_jit{1};
std::atomic<int64_t> g_opt_first_free{1};   // PSR plans: the |0...0> pass is exempt from the budget
std::atomic<int64_t> g_opt_poison{0};   // LQ_OPT_POISON_ALLOC
std::atomic<int64_t> g_opt_comm_timeout{600000};   // LQ_OPT_COMM_TIMEOUT_MS
std::atomic<int64_t> g_opt_swap_k{4};   // LQ_OPT_SWAP_QUBITS: qubits per global exchange (dist.h)
std::atomic<int64_t> g_opt_group_staged{0};   // LQ_OPT_GROUP_STAGED: group mode through NCCL mode's pack/unpack
// FP64 pass budgets, swept on B200: PSR plans (config 4:
// 2.540 s at 400 vs 2.555 / 2.559 s at 600 / 800) and single-state or
// sharded plans (n = 30: 8 Trotter steps 371 -> 279 ms, the config-5
// circuit 186 -> 151 ms, 200 random gates 40.5 -> 35.9 ms at 800 vs 400)
std::atomic<int64_t> g_opt_budget{400};         // LQ_OPT_PASS_BUDGET (PSR plans)
std::atomic<int64_t> g_opt_state_budget{800};   // LQ_OPT_STATE_PASS_BUDGET (every other plan)
std::atomic<int64_t> g_opt_relabel{0};          // LQ_OPT_RELABEL_STORES (PSR plans; measured, off)
std::atomic<int64_t> g_opt_export_psr{0};       // LQ_OPT_EXPORT_PSR (testing)
std::atomic<int64_t> g_opt_graphs{1};           // LQ_OPT_GRAPHS
std::atomic<uint64_t> g_plan_uid{1};            // Plan::uid of cached plans
uint64_t next_plan_uid() { return g_plan_uid.fetch_add(1); }
const double PI = 3.14159265358979323846264338327950288;

lq_status fail(lq_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

#define CUDA_TRY(x)                                                                         \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess)                                                              \
            return fail(LQ_ERR_CUDA, std::string(#x) + " failed: " + cudaGetErrorString(e_)); \
    } while (0)

#define LQ_TRY(x)                          \
    do {                                   \
        lq_status s_ = (x);                \
        if (s_ != LQ_OK) return s_;        \
    } while (0)

// ---- optional per-launch CUDA-event timing (LQ_OPT_KERNEL_TIMING) ----
enum KClass { KC_TILE = 0, KC_PAIR = 1, KC_DIAG = 2, KC_PAULI = 3, KC_OTHER = 4, KC_SWAP = 5, KC_N = 6 };
std::atomic<int64_t> g_opt_timing{0};
struct TimedLaunch { int cls; cudaEvent_t a, b; };
std::vector<TimedLaunch> g_timed;
std::vector<cudaEvent_t> g_event_pool;
double g_time_ms[KC_N] = {0, 0, 0, 0, 0, 0};
uint64_t g_time_cnt[KC_N] = {0, 0, 0, 0, 0, 0};

cudaEvent_t pool_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
struct LaunchTimer {
    int cls;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    LaunchTimer(int c, cudaStream_t s) : cls(c), st(s) {
        if (g_opt_timing.load()) { a = pool_event(); cudaEventRecord(a, st); }
    }
    ~LaunchTimer() {
        if (a) {
            cudaEvent_t b = pool_event();
            cudaEventRecord(b, st);
            g_timed.push_back({cls, a, b});
        }
    }
};
// NVTX ranges (nsys / ncu --nvtx): one per tile pass launch, exchange and
// collective; a no-op unless a tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

void harvest_timing() {
    for (auto &t : g_timed) {
        float ms = 0.f;
        if (cudaEventSynchronize(t.b) == cudaSuccess && cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
            g_time_ms[t.cls] += ms;
            g_time_cnt[t.cls] += 1;
        }
        g_event_pool.push_back(t.a);
        g_event_pool.push_back(t.b);
    }
    g_timed.clear();
    cudaGetLastError();
}

lq_status check_launch(const char *what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(LQ_ERR_CUDA, std::string(what) + " launch failed: " + cudaGetErrorString(e));
    return LQ_OK;
}

template <class F>
static lq_status capture_graph(F body, cudaGraphExec_t *out, uint64_t *kernels) {
    *out = nullptr;
    cudaStream_t cs = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    const uint64_t l0 = g_launches.load();
    lq_status s = LQ_OK;
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    else s = body(cs);
    cudaGraph_t g = nullptr;
    if (e == cudaSuccess) {
        const cudaError_t e2 = cudaStreamEndCapture(cs, &g);   // always end a begun capture
        if (s == LQ_OK && e2 != cudaSuccess) s = fail(LQ_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e2));
    }
    if (s == LQ_OK) {
        e = cudaGraphInstantiate(out, g, 0);
        if (e != cudaSuccess) {
            *out = nullptr;
            s = fail(LQ_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
        }
    }
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cs);
    // the captured launches have not run: count them when the graph replays
    *kernels = g_launches.load() - l0;
    g_launches.fetch_sub(*kernels);
    cudaGetLastError();
    return s;
}

lq_status have_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(LQ_ERR_CUDA, "no CUDA device available (liblq has no CPU fallback)");
    }
    return LQ_OK;
}

// QFT stages one local tile pass of a sharded state holds (dist.h): the
// tile bits the planner takes for a run of stages minus the coalescing
// bits; 0 (plain Belady) for small shards.
int qft_pass_stages(int nl) {
    // plan_circuit gives a run of QFT stages 12 tile bits when that saves a pass
    const int K = g_opt_K.load() > 0 ? (int)g_opt_K.load() : (getenv("LQ_QFT_K11") ? auto_tile_bits(nl) : 12);
    if (getenv("LQ_QFT_BELADY") || nl <= K) return 0;   // A/B experiments
    return std::max(1, K - (int)g_opt_coalesce.load());
}

PlanOptions options() {
    PlanOptions o;
    o.K = (int)g_opt_K.load();
    o.coalesce = (int)g_opt_coalesce.load();
    o.fusion = g_opt_fusion.load() != 0;
    o.reg_bits = (int)g_opt_regbits.load();
    o.budget = (int)g_opt_state_budget.load();   // lq_psr_create overrides with g_opt_budget
    return o;
}

// Planner options of lq_plan_describe / lq_plan_export_json: the generic
// ones, or (LQ_OPT_EXPORT_PSR) those of the parameter-shift planner.
PlanOptions export_options() {
    PlanOptions po = options();
    if (g_opt_export_psr.load()) {
        po.budget = (int)g_opt_budget.load();
        po.first_free = g_opt_first_free.load() != 0;
        po.oop = (int)g_opt_relabel.load();
    }
    return po;
}

// JIT-specialise the plan's tile passes (LQ_OPT_JIT).  Auto mode (1)
// compiles plans that will stream enough amplitudes to amortise NVRTC
// (~1-5 s per pass): every PSR plan (it runs 2P+1 circuits) and single
// states with n >= 26; 2 forces it, 0 disables it.
lq_status prepare(Plan &plan, bool reused = false) {
    if (plan.prepared) return LQ_OK;   // a cached plan (PlanCache) keeps its kernels
    plan.jit.clear();
    const int64_t mode = g_opt_jit.load();
    if (mode == 0 || plan.n_tile == 0) return LQ_OK;
    if (mode == 1 && !reused && plan.n < 26) return LQ_OK;
    for (PlanPass &p : plan.passes) {
        p.support = p.sup_free = ~0ull;
        p.tiles_log2 = -1;
    }
    if (plan.zero_first && getenv("LQ_NO_SUPPORT") == nullptr) {
        // Support tracking.  The state starts as |0...0> and a tile pass
        // changes only its own tile bits, so the state entering pass i is zero
        // wherever a local bit outside U_i = T_0 | ... | T_{i-1} is set.
        // Invariant: HBM holds the state at the indices inside U_i (garbage
        // elsewhere).  Pass i loads only those indices (zeros synthesised for
        // the rest of its tiles), runs only the tiles whose free bits lie in
        // U_i (every other tile is zero and stays zero) and stores them whole:
        // indices inside U_{i+1} = U_i | T_i, so the invariant carries over.
        // Pass 0 (U = 0) is tile 0 only, |0...0> synthesised: no HBM read and
        // 2^K amplitudes written.  Passes with Pauli groups run every tile
        // (one partial per tile).  Valid when no non-tile pass comes before U
        // covers every local bit, and the state after the plan is either whole
        // (U = all) or read by nothing but the tile passes' own Pauli groups.
        const uint64_t all = plan.nl >= 64 ? ~0ull : ((1ull << plan.nl) - 1);
        uint64_t U = 0;
        bool ok = true;
        // A read-only pass (PF_NO_STORE) writes nothing to HBM: it leaves the
        // support where it was.
        for (const PlanPass &p : plan.passes) {
            if (U == all) break;
            if (p.kind != PASS_TILE) { ok = false; break; }
            if (p.kp.flags & PF_NO_STORE) continue;
            for (int b = 0; b < p.kp.K; b++) U |= 1ull << p.kp.T[b];
            U = p.map_store(U);   // a relabelling store moves the support into the next frame
        }
        if (U != all && !plan.wide_groups.empty()) ok = false;
        U = 0;
        for (size_t i = 0; ok && i < plan.passes.size() && U != all; i++) {
            PlanPass &p = plan.passes[i];
            uint64_t tm = 0;
            for (int b = 0; b < p.kp.K; b++) tm |= 1ull << p.kp.T[b];
            p.support = U;
            if (!(p.kp.flags & PF_EXPV)) {
                p.sup_free = U & ~tm & all;
                p.tiles_log2 = __builtin_popcountll(p.sup_free);
            }
            if (!(p.kp.flags & PF_NO_STORE)) U = p.map_store(U | tm);
        }
    }
    plan.ctab = getenv("LQ_JIT_NO_CTAB") == nullptr;   // constant-bank op tables (A/B switch for experiments)
    std::string err;
    if (!jit_plan(plan, plan.jit, plan.jit_ctab, err)) {
        plan.jit.clear();
        plan.jit_ctab.clear();
        return fail(LQ_ERR_CUDA, err);
    }
    plan.ctab_desc.clear();
    plan.ctab_total = 0;
    for (size_t i = 0; i < plan.passes.size(); i++) {
        // bank passes and flat-staged passes (jit.h plan_flat_tables) both stage through k_stage_ctab
        const bool flat = plan.jit[i] && plan.passes[i].kind == PASS_TILE && plan_flat_tables(plan, plan.passes[i].kp);
        if (!plan.jit_ctab[i] && !flat) continue;
        const KPass &kp = plan.passes[i].kp;
        plan.ctab_desc.push_back({kp.op_begin, kp.op_end, kp.smat, plan.ctab_total});
        plan.ctab_total += kp.smat * (uint32_t)plan.ctab_circ;
    }
    return LQ_OK;
}

// Plans of single-state calls (apply, QFT, expectation) for repeated use:
// an LRU keyed by everything the plan depends on -- the call kind, n, the
// qubit map, the planner options and the gate / term arrays (U1/U2 matrices
// by value, angles included; theta is not part of a plan: parameterised
// angles are resolved on the device by k_build_mats).  A hit skips
// planning and JIT source generation, which otherwise cost 0.1-30 ms per
// call on the host.
struct CachedPlan {
    Plan plan;
    MatBuilder mb;
    int32_t qmap_after[64];
    int uses = 0;
    bool promoted = false;
    // CUDA graph of this plan's launches on one state (LQ_OPT_GRAPHS; run_single):
    // captured on the second run with the same buffers, replayed after
    std::mutex gmu;
    cudaGraphExec_t gexec = nullptr;
    uint64_t gkernels = 0;
    std::array<const void *, 6> gkey{}, gseen{};
    bool gdisabled = false;   // a capture failed: stream launches only
    ~CachedPlan() {
        if (gexec) cudaGraphExecDestroy(gexec);
    }
};

// Compile on second use: in auto JIT mode small single-state plans start on
// the interpreter (NVRTC costs ~1 s per pass); a cached plan that runs a
// second time is specialised like a PSR plan (config 1 / config 2 shapes).
lq_status promote(CachedPlan &cp) {
    if (++cp.uses < 2 || cp.promoted || g_opt_jit.load() != 1) return LQ_OK;
    cp.promoted = true;
    if (cp.plan.passes.empty() || cp.plan.n_tile == 0 || !cp.plan.jit.empty()) return LQ_OK;
    cp.plan.prepared = false;
    lq_status s = prepare(cp.plan, true);
    cp.plan.prepared = true;
    cp.plan.uid = next_plan_uid();   // its tables changed (constant-bank descriptors)
    return s;
}
struct PlanCache {
    std::mutex mu;
    std::list<std::pair<std::string, std::shared_ptr<CachedPlan>>> lru;
    static constexpr size_t CAP = 32;
    std::shared_ptr<CachedPlan> get(const std::string &k) {
        std::lock_guard<std::mutex> lk(mu);
        for (auto it = lru.begin(); it != lru.end(); ++it)
            if (it->first == k) {
                lru.splice(lru.begin(), lru, it);
                return it->second;
            }
        return nullptr;
    }
    void put(const std::string &k, std::shared_ptr<CachedPlan> p) {
        std::lock_guard<std::mutex> lk(mu);
        lru.emplace_front(k, std::move(p));
        if (lru.size() > CAP) lru.pop_back();
    }
    void clear() {
        std::lock_guard<std::mutex> lk(mu);
        lru.clear();
    }
};
PlanCache g_plan_cache;

std::string plan_key(char kind, int n, const int32_t *qmap, const void *payload, size_t bytes, const void *stream) {
    std::string k(1, kind);
    int64_t o[8] = {n, g_opt_K.load(), g_opt_coalesce.load(), g_opt_fusion.load(), g_opt_regbits.load(),
                    g_opt_jit.load(), g_opt_state_budget.load(), (int64_t)(intptr_t)stream};
    k.append(reinterpret_cast<const char *>(o), sizeof(o));
    k.append(reinterpret_cast<const char *>(qmap), sizeof(int32_t) * (size_t)n);
    if (bytes) k.append(reinterpret_cast<const char *>(payload), bytes);
    return k;
}

std::string gates_key(int n, const int32_t *qmap, const lq_gate *g, size_t ng, const void *stream) {
    std::string k = plan_key('a', n, qmap, nullptr, 0, stream);
    for (size_t i = 0; i < ng; i++) {
        lq_gate c = g[i];
        c.mat = nullptr;
        k.append(reinterpret_cast<const char *>(&c), sizeof(c));
        const int nm = g[i].kind == LQ_U1 ? 8 : g[i].kind == LQ_U2 ? 32 : 0;
        if (nm && g[i].mat) k.append(reinterpret_cast<const char *>(g[i].mat), sizeof(double) * nm);
    }
    return k;
}

// Stream-ordered growable device buffer.
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    lq_status reserve(size_t bytes, cudaStream_t s) {
        if (bytes <= cap && p) return LQ_OK;
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        size_t nb = std::max<size_t>(bytes, std::max<size_t>(cap * 2, 4096));
        cudaError_t e = cudaMallocAsync(&p, nb, s);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            cap = 0;
            return fail(e == cudaErrorMemoryAllocation ? LQ_ERR_OOM : LQ_ERR_CUDA,
                        std::string("device allocation of ") + std::to_string(nb) + " bytes failed: " +
                            cudaGetErrorString(e));
        }
        cap = nb;
        if (g_opt_poison.load() && cudaMemsetAsync(p, 0xFF, nb, s) != cudaSuccess) {
            cudaGetLastError();
            return fail(LQ_ERR_CUDA, "poison memset failed");
        }
        return LQ_OK;
    }
    void release(cudaStream_t s) {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        cap = 0;
    }
    template <class T> T *at(size_t off) const { return reinterpret_cast<T *>(static_cast<char *>(p) + off); }
};

// Host staging of several arrays uploaded with one copy.
struct Blob {
    std::vector<char> h;
    template <class T> size_t add(const std::vector<T> &v) { return add(v.data(), v.size() * sizeof(T)); }
    size_t add(const void *d, size_t bytes) {
        size_t off = (h.size() + 255) & ~size_t(255);
        h.resize(off + std::max<size_t>(bytes, 1));
        if (bytes) memcpy(h.data() + off, d, bytes);
        return off;
    }
    lq_status upload(DevBuf &b, cudaStream_t s) {
        LQ_TRY(b.reserve(h.size(), s));
        CUDA_TRY(cudaMemcpyAsync(b.p, h.data(), h.size(), cudaMemcpyHostToDevice, s));
        return LQ_OK;
    }
};


bool is_rotation(int k) {
    return k == LQ_RX || k == LQ_RY || k == LQ_RZ || k == LQ_CP || k == LQ_CRY || k == LQ_RXX || k == LQ_RYY ||
           k == LQ_RZZ;
}
int arity(int k) {
    if (k <= LQ_RZ || k == LQ_U1) return 1;
    if (k == LQ_CCX) return 3;
    return 2;
}

// Boundary validation: the runtime form of the paper's
// compile-time parameter/gate distinction.
lq_status validate_gates(int n, const lq_gate *g, size_t ng, const double *theta, size_t n_theta,
                         bool theta_known, std::vector<int> *uses) {
    if (ng && !g) return fail(LQ_ERR_ARG, "gates is NULL");
    for (size_t i = 0; i < ng; i++) {
        const lq_gate &G = g[i];
        std::string at = "gate " + std::to_string(i) + ": ";
        if (G.kind < 0 || G.kind >= LQ_NUM_KINDS) return fail(LQ_ERR_ARG, at + "unknown kind");
        if (G.reserved != 0) return fail(LQ_ERR_ARG, at + "reserved field must be 0");
        int a = arity(G.kind);
        int qs[3] = {G.q0, G.q1, G.q2};
        for (int k = 0; k < 3; k++) {
            if (k < a) {
                if (qs[k] < 0 || qs[k] >= n) return fail(LQ_ERR_ARG, at + "qubit out of range");
            } else if (qs[k] != -1) {
                return fail(LQ_ERR_ARG, at + "unused qubit slot must be -1");
            }
        }
        if ((a >= 2 && G.q0 == G.q1) || (a == 3 && (G.q2 == G.q0 || G.q2 == G.q1)))
            return fail(LQ_ERR_ARG, at + "duplicate qubits");
        if (is_rotation(G.kind)) {
            if (G.param_idx >= 0) {
                if (G.param_idx >= (int64_t)n_theta) return fail(LQ_ERR_ARG, at + "param_idx >= n_params");
                if (G.angle != 0.0) return fail(LQ_ERR_ARG, at + "angle must be 0 when param_idx is used");
                if (theta_known) {
                    if (!theta) return fail(LQ_ERR_ARG, at + "theta is NULL");
                    if (!std::isfinite(theta[G.param_idx])) return fail(LQ_ERR_NONFINITE, at + "non-finite theta");
                }
                if (uses) (*uses)[G.param_idx]++;
            } else if (G.param_idx == -1) {
                if (!std::isfinite(G.angle)) return fail(LQ_ERR_NONFINITE, at + "non-finite angle");
            } else {
                return fail(LQ_ERR_ARG, at + "param_idx must be >= 0 or -1");
            }
        } else {
            if (G.param_idx != -1 || G.angle != 0.0)
                return fail(LQ_ERR_ARG, at + "fixed gate takes no angle or parameter");
        }
        if (G.kind == LQ_U1 || G.kind == LQ_U2) {
            if (!G.mat) return fail(LQ_ERR_ARG, at + "matrix is NULL");
            int cnt = G.kind == LQ_U1 ? 8 : 32;
            for (int k = 0; k < cnt; k++)
                if (!std::isfinite(G.mat[k])) return fail(LQ_ERR_NONFINITE, at + "non-finite matrix entry");
        }
    }
    if (uses)
        for (size_t p = 0; p < uses->size(); p++)
            if ((*uses)[p] > 1)
                return fail(LQ_ERR_ARG, "parameter " + std::to_string(p) +
                                            " is used by more than one gate (not supported, reading A7)");
    return LQ_OK;
}

lq_status validate_terms(int n, const lq_pauli_term *t, size_t nt) {
    if (nt && !t) return fail(LQ_ERR_ARG, "terms is NULL");
    uint64_t lim = n >= 64 ? ~0ull : ((1ull << n) - 1);
    for (size_t i = 0; i < nt; i++) {
        if ((t[i].x_mask & ~lim) || (t[i].z_mask & ~lim))
            return fail(LQ_ERR_ARG, "term " + std::to_string(i) + ": mask has bits beyond n qubits");
        if (!std::isfinite(t[i].coeff)) return fail(LQ_ERR_NONFINITE, "term " + std::to_string(i) + ": non-finite coeff");
    }
    return LQ_OK;
}

// ---------------------------------------------------------------- launches
template <int RR>
lq_status launch_tile_rr(const void *jk, const KPass &kp, const KSub *subs, const KOp *kops, const KPerm *perms,
                         const KPermTerm *pterms, uint32_t n_pterms, const ETerm *eterms, const double2 *mats,
                         uint64_t mat_stride, const double2 *cst, double2 *state, uint64_t state_stride,
                         int n_circ, double *partials, uint64_t slot_stride, cudaStream_t st, int tl2,
                         double2 *state_out) {
    static bool attr = false;
    static int n_sm = 0;
    const size_t smem = ((size_t)32 << kp.K) + (size_t)kp.smat * sizeof(double2) +
                        (size_t)(kp.op_end - kp.op_begin) * sizeof(KOp) +
                        (size_t)(kp.perm_end - kp.perm_begin) * sizeof(KPerm) + (size_t)n_pterms * sizeof(KPermTerm) +
                        (256 + 32) * sizeof(uint64_t) + (size_t)(kp.sub_end - kp.sub_begin + 1) * sizeof(KSub) +
                        (size_t)(kp.eterm_end - kp.eterm_begin) * sizeof(ETerm);
    if (!attr) {
        CUDA_TRY(cudaFuncSetAttribute(k_tile<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
        attr = true;
    }
    if (smem > 227 * 1024) return fail(LQ_ERR_STATE, "tile pass exceeds shared memory (planner bug)");
    // tl2 >= 0: a JIT pass launched over its nonzero tiles only (PlanPass::sup_free)
    if (tl2 >= 0 && !jk) return fail(LQ_ERR_STATE, "restricted tile range without a JIT program (internal)");
    const uint32_t tiles_log2 = tl2 >= 0 ? (uint32_t)tl2 : (uint32_t)(kp.nl - kp.K);
    const uint64_t total = (uint64_t)n_circ << tiles_log2;
    if (total >= (1ull << 32)) return fail(LQ_ERR_DIM, "too many tiles in one launch");
    // persistent grid: as many CTAs as fit on every SM (2 per SM for K <= 11)
    int per_sm = 1;
    const void *fn = jk ? jk : (const void *)k_tile<RR>;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 1 << (kp.K - RR), smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    const unsigned grid = (unsigned)std::min<uint64_t>(total, (uint64_t)n_sm * (uint64_t)per_sm);
    LaunchTimer lt_(KC_TILE, st);
    NvtxRange nr_("lq tile pass");
    if ((kp.flags & PF_EXPV) && !partials) return fail(LQ_ERR_STATE, "expectation pass without partial buffer");
    if (jk) {   // JIT-specialised program of this pass (jit.h): same parameters as k_tile
        uint32_t tot32 = (uint32_t)total;
        void *args[] = {(void *)&kp,      (void *)&subs,   (void *)&kops,       (void *)&perms, (void *)&pterms,
                        (void *)&eterms,  (void *)&mats,   (void *)&mat_stride, (void *)&cst,   (void *)&state,
                        (void *)&state_stride, (void *)&tiles_log2, (void *)&tot32, (void *)&partials,
                        (void *)&slot_stride, (void *)&state_out};
        CUDA_TRY(cudaLaunchKernel(jk, dim3(grid), dim3(1u << (kp.K - RR)), args, smem, st));
        return check_launch("k_tile (jit)");
    }
    k_tile<RR><<<grid, 1u << (kp.K - RR), smem, st>>>(kp, subs, kops, perms, pterms, eterms, mats, mat_stride, cst,
                                                      state, state_stride, tiles_log2, (uint32_t)total, partials,
                                                      slot_stride, state);
    return check_launch("k_tile");
}

lq_status launch_tile(int Rr, const void *jk, const KPass &kp, const KSub *subs, const KOp *kops, const KPerm *perms,
                      const KPermTerm *pterms, uint32_t n_pterms, const ETerm *eterms, const double2 *mats,
                      uint64_t mat_stride, const double2 *cst, double2 *state, uint64_t state_stride, int n_circ,
                      double *partials, uint64_t slot_stride, cudaStream_t st, int tl2 = -1,
                      double2 *state_out = nullptr) {
    if (!state_out) state_out = state;
#define LT(RRV) launch_tile_rr<RRV>(jk, kp, subs, kops, perms, pterms, n_pterms, eterms, mats, mat_stride, cst, state, \
                                    state_stride, n_circ, partials, slot_stride, st, tl2, state_out)
    switch (Rr) {
    case 1: return LT(1);
    case 2: return LT(2);
    case 3: return LT(3);
    default: return LT(4);
    }
#undef LT
}

unsigned grid_for(uint64_t work, unsigned per_block = 256) {
    uint64_t b = (work + per_block - 1) / per_block;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 16));
}

struct DevPlan {
    const CtabDesc *ctab_desc = nullptr;   // plan.ctab_desc on the device
    double2 *ctab_stage = nullptr;         // >= plan.ctab_total double2 of staging
    const KSub *subs = nullptr;
    const KOp *kops = nullptr;
    const KPerm *perms = nullptr;
    const KPermTerm *pterms = nullptr;
    const ETerm *eterms = nullptr;
    const MSpec *specs = nullptr;
    const MFactor *factors = nullptr;
    const double2 *cst = nullptr;
};

std::mutex &ctab_mutex(const void *bank) {
    static std::mutex mu[64];
    return mu[((uintptr_t)bank >> 8) % 64];
}

// alt (plans with relabelling stores, Plan::has_oop): the second buffer of
// the ping-pong pair, as large as `state`; *final_out: the buffer that holds
// the state after the plan.
lq_status launch_passes(const Plan &plan, const DevPlan &dp, double2 *state, uint64_t state_stride, int n_circ,
                        const double2 *mats, uint64_t mat_stride, cudaStream_t st, bool zero_first,
                        double *partials = nullptr, uint64_t slot_stride = 0, bool no_final_store = false,
                        uint64_t gofs = 0, double2 *alt = nullptr, double2 **final_out = nullptr) {
    const int n = plan.nl;   // local index bits
    if (final_out) *final_out = state;
    if (plan.has_oop && !alt) return fail(LQ_ERR_STATE, "relabelling plan without a second state buffer (internal)");
    double2 *const alt_base = state;
    if (zero_first && (plan.passes.empty() || plan.passes[0].kind != PASS_TILE)) {
        dim3 grid(grid_for(1ull << n), n_circ);
        k_fill_basis<<<grid, 256, 0, st>>>(1ull << n, 0, state, state_stride);
        LQ_TRY(check_launch("k_fill_basis"));
    }
    if (!plan.ctab_desc.empty()) {   // constant op tables of this launch's circuits
        if (!dp.ctab_desc || !dp.ctab_stage || n_circ > plan.ctab_circ)
            return fail(LQ_ERR_STATE, "constant op tables without staging (internal)");
        k_stage_ctab<<<dim3((unsigned)plan.ctab_desc.size(), (unsigned)n_circ), 128, 0, st>>>(
            dp.kops, dp.ctab_desc, mats, mat_stride, dp.cst, dp.ctab_stage);
        LQ_TRY(check_launch("k_stage_ctab"));
    }
    size_t ci = 0;
    // zero-first: until a pass has stored, HBM does not hold the state yet and
    // every pass synthesises |0...0> (a leading read-only pass stores nothing)
    bool stored = !zero_first || plan.passes.empty() || plan.passes[0].kind != PASS_TILE;
    for (size_t i = 0; i < plan.passes.size(); i++) {
        const PlanPass &p = plan.passes[i];
        if (p.kind == PASS_TILE) {
            // A JIT module's constant bank is shared by every plan whose pass
            // has the same source on the same stream: hold its lock from the
            // bank refill to the launch, so two host threads issuing on one
            // stream cannot interleave (stream order = enqueue order).
            std::unique_lock<std::mutex> bank_lock;
            const double2 *pmats = mats;   // the pass's table source
            uint64_t pmat_stride = mat_stride;
            if (i < plan.jit_ctab.size() && plan.jit_ctab[i]) {
                bank_lock = std::unique_lock<std::mutex>(ctab_mutex(plan.jit_ctab[i]));
                const CtabDesc &D = plan.ctab_desc[ci++];
                CUDA_TRY(cudaMemcpyAsync(plan.jit_ctab[i], dp.ctab_stage + D.out,
                                         (size_t)n_circ * D.smat * sizeof(double2), cudaMemcpyDeviceToDevice, st));
            } else if (i < plan.jit.size() && plan.jit[i] && plan_flat_tables(plan, p.kp)) {
                const CtabDesc &D = plan.ctab_desc[ci++];   // flat-staged: read in place
                pmats = dp.ctab_stage + D.out;
                pmat_stride = D.smat;
            }
            KPass kp = p.kp;
            kp.gofs = gofs;
            if (!stored) kp.flags |= PF_LOAD_ZERO;
            if (!(kp.flags & PF_NO_STORE)) stored = true;
            if (no_final_store && i + 1 == plan.passes.size()) kp.flags |= PF_NO_STORE;
            uint32_t npt = 0;
            if (kp.perm_end > kp.perm_begin)
                npt = plan.perms[kp.perm_end - 1].term_end - plan.perms[kp.perm_begin].term_begin;
            const void *jk = i < plan.jit.size() ? plan.jit[i] : nullptr;
            // a restricted tile range presumes the zero-first pass ran (prepare())
            if ((p.tiles_log2 >= 0 || p.support != ~0ull) && jk && !zero_first)
                return fail(LQ_ERR_STATE, "restricted tile range outside a zero-first run (internal)");
            const int tl2 = jk ? p.tiles_log2 : -1;
            // a relabelling pass stores into the other buffer (JIT programs only)
            const bool oop = p.oop && !(kp.flags & PF_NO_STORE);
            if (p.oop && !jk) return fail(LQ_ERR_STATE, "relabelling pass without its JIT program (internal)");
            double2 *out = oop ? (state == alt ? alt_base : alt) : state;
            LQ_TRY(launch_tile(plan.Rr, jk, kp, dp.subs, dp.kops, dp.perms, dp.pterms, npt, dp.eterms, pmats,
                               pmat_stride, dp.cst, state, state_stride, n_circ, partials, slot_stride, st, tl2, out));
            state = out;
            if (final_out) *final_out = state;
        } else if (p.kind == PASS_PAIR) {
            const KOp op = plan.kops[p.op_begin];
            uint64_t work = (op.type == K_U1 || op.type == K_X) ? (1ull << (n - 1)) : (1ull << (n - 2));
            dim3 grid(grid_for(work), n_circ);
            LaunchTimer lt_(KC_PAIR, st);
            k_pair<<<grid, 256, 0, st>>>(n, gofs, op, mats, mat_stride, state, state_stride);
            LQ_TRY(check_launch("k_pair"));
        } else {
            for (uint32_t b = p.op_begin; b < p.op_end; b += DIAG_MAX_OPS) {
                int cnt = (int)std::min<uint32_t>(DIAG_MAX_OPS, p.op_end - b);
                dim3 grid(grid_for(1ull << n), n_circ);
                LaunchTimer lt_(KC_DIAG, st);
                k_diag<<<grid, 256, 0, st>>>(n, gofs, dp.kops + b, cnt, mats, mat_stride, state, state_stride);
                LQ_TRY(check_launch("k_diag"));
            }
        }
    }
    return LQ_OK;
}

// Pauli groups whose x mask is wider than a tile: the direct pair kernel.
struct DirectSet {
    std::vector<PTerm> terms;
    struct D { uint64_t x; uint32_t tb, te, slot, nblocks; };
    std::vector<D> ds;
    uint32_t slots = 0;          // total partial slots (tile passes + direct)
    uint32_t scratch = 0;        // per-circuit chunk sums of the two-level reduction (finish_expv)
    static constexpr uint32_t CHUNK = 8192;
    // per-circuit stride of the partial buffer: the slots, then the chunk sums
    uint32_t stride() const { return std::max<uint32_t>(slots + scratch, 1); }
    void build(const Plan &plan) {
        slots = plan.n_slots;
        for (uint32_t g : plan.wide_groups) {
            D d;
            d.x = plan.groups[g].x;
            d.tb = (uint32_t)terms.size();
            for (auto &t : plan.groups[g].terms) {
                PTerm p{};
                p.coeff = t.c;
                p.zfull = t.z;
                p.yph = t.y;
                terms.push_back(p);
            }
            d.te = (uint32_t)terms.size();
            uint64_t blocks = ((1ull << plan.nl) + 255) / 256;
            d.nblocks = (uint32_t)std::min<uint64_t>(blocks, 148ull * 8);
            d.slot = slots;
            slots += d.nblocks;
            ds.push_back(d);
        }
        scratch = slots > CHUNK ? (slots + CHUNK - 1) / CHUNK : 0;
    }
};

// Direct groups, then E[c] = fixed-order sum of the circuit's partials.
lq_status finish_expv(const Plan &plan, const DirectSet &dset, const PTerm *dterms, const double2 *state,
                      uint64_t state_stride, int n_circ, double *partial, uint64_t slot_stride, double *E,
                      cudaStream_t st, uint64_t gofs = 0) {
    for (const auto &D : dset.ds) {
        dim3 grid(D.nblocks, n_circ);
        LaunchTimer lt_(KC_PAULI, st);
        k_pauli_direct<<<grid, 256, 0, st>>>(plan.nl, gofs, D.x, dterms + D.tb, D.te - D.tb, state, state_stride, partial,
                                             slot_stride, D.slot);
        LQ_TRY(check_launch("k_pauli_direct"));
    }
    if (dset.slots == 0) {
        CUDA_TRY(cudaMemsetAsync(E, 0, sizeof(double) * n_circ, st));
        return LQ_OK;
    }
    if (dset.scratch) {   // many slots (one per warp of every tile): chunk sums first, fixed order
        k_sum_chunks<<<dim3(dset.scratch, n_circ), 256, 0, st>>>(partial, slot_stride, dset.slots, DirectSet::CHUNK,
                                                                 partial + dset.slots);
        LQ_TRY(check_launch("k_sum_chunks"));
        k_sum_partials<<<n_circ, 256, 0, st>>>(partial + dset.slots, slot_stride, dset.scratch, E);
        return check_launch("k_sum_partials");
    }
    k_sum_partials<<<n_circ, 256, 0, st>>>(partial, slot_stride, dset.slots, E);
    return check_launch("k_sum_partials");
}

bool qmap_identity(int n, const int32_t *qm) {
    for (int q = 0; q < n; q++)
        if (qm[q] != n - 1 - q) return false;
    return true;
}

QMap to_qmap(int n, const int32_t *qm) {
    QMap m;
    memset(&m, 0, sizeof(m));
    for (int q = 0; q < n; q++) m.q[q] = (int8_t)qm[q];
    return m;
}

}  // namespace

// ---------------------------------------------------------------- handles
struct lq_comm {
    ncclComm_t c = nullptr;          // nullptr: a partition-only comm (lq_comm_init_local) or aborted
    int rank = 0, world = 1;
    bool local = false;              // lq_comm_init_local: no transport, collectives are the identity
    bool dead = false;               // aborted after an asynchronous NCCL error or a timeout
    std::string why;                 // the failure that killed it
};

struct lq_sv {
    int n = 0;
    double2 *d = nullptr;
    bool owned = false;
    cudaStream_t stream = nullptr;
    int32_t qmap[64];
    DevBuf plan_buf, work_buf;
    uint64_t blob_uid = 0;           // Plan::uid whose tables plan_buf holds (0: none / per-call data)
    size_t blob_bytes = 0;
    // ---- sharded states (dist.h): m > 0
    int m = 0, nl = 0;               // log2 G; local index bits
    lq_comm *comm = nullptr;         // NCCL mode: one shard per process
    int rank0 = 0;                   // rank of shards[0]
    std::vector<double2 *> shards;   // this process's shards (group mode: all G)
    uint32_t xmask = 0;              // rank relabel: rank r holds physical global bits r ^ xmask
    DevBuf mats_buf, part_buf, stage_buf, ctab_buf;
    // exchange pipeline (NCCL mode): a second stream carries the transfers
    // while this handle's stream packs the next chunk and unpacks the last
    cudaStream_t xs = nullptr;
    cudaEvent_t ev_start = nullptr, ev_packed[2] = {nullptr, nullptr}, ev_moved[2] = {nullptr, nullptr};
    uint64_t stat_exchanges = 0, stat_bytes_sent = 0;   // per rank (group mode: per shard)
    bool dead = false;               // poisoned after an asynchronous CUDA / NCCL failure
    std::string why;
    void reset_map() {
        for (int q = 0; q < n; q++) qmap[q] = n - 1 - q;
        xmask = 0;
    }
    uint64_t gofs(int k) const { return (uint64_t)(uint32_t)((rank0 + k) ^ (int)xmask) << nl; }
};

namespace {
lq_status check_sv(const lq_sv *sv) {
    if (!sv || !sv->d) return fail(LQ_ERR_ARG, "invalid state handle");
    if (sv->dead) return fail(LQ_ERR_STATE, "state handle unusable after an earlier asynchronous failure: " + sv->why);
    if (sv->comm && sv->comm->dead)
        return fail(LQ_ERR_STATE, "communicator aborted after an earlier failure: " + sv->comm->why);
    return LQ_OK;
}

// An asynchronous CUDA or NCCL failure leaves the handle's contents
// undefined: every later call on it returns LQ_ERR_STATE.
// Validation errors and OOM leave it usable.
lq_status seal(lq_sv *sv, lq_status s) {
    if (sv && (s == LQ_ERR_CUDA || s == LQ_ERR_NCCL)) {
        sv->dead = true;
        sv->why = g_err;
    }
    return s;
}

// Run a circuit-level plan on one state (apply_circuit / canonicalize / qft).
// A cached plan's tables (uid != 0, no per-call data) stay in the state's
// plan buffer between calls: a repeated call (config 2's QFTs, a VQE or
// Trotter loop on one state) skips the host -> device copy of its blob.
lq_status upload_tables(lq_sv *sv, const Blob &blob, uint64_t uid) {
    if (uid && sv->blob_uid == uid && sv->blob_bytes == blob.h.size() && sv->plan_buf.p) return LQ_OK;
    sv->blob_uid = 0;
    LQ_TRY(const_cast<Blob &>(blob).upload(sv->plan_buf, sv->stream));
    sv->blob_uid = uid;
    sv->blob_bytes = blob.h.size();
    return LQ_OK;
}

lq_status run_single(lq_sv *sv, Plan &plan, const MatBuilder &mb, const double *theta, size_t n_theta,
                     CachedPlan *cp = nullptr) {
    if (plan.passes.empty()) return LQ_OK;
    if (!plan.prepared) plan.stream_tag = (uint64_t)(uintptr_t)sv->stream;
    LQ_TRY(prepare(plan));
    Blob blob;
    size_t o_sub = blob.add(plan.subs), o_kop = blob.add(plan.kops), o_spec = blob.add(mb.specs),
           o_fac = blob.add(mb.factors), o_cst = blob.add(mb.cst), o_perm = blob.add(plan.perms),
           o_pt = blob.add(plan.perm_terms);
    size_t o_th = blob.add(theta, theta ? n_theta * sizeof(double) : 0);
    size_t o_cd = blob.add(plan.ctab_desc);
    LQ_TRY(upload_tables(sv, blob, theta ? 0 : plan.uid));
    DevPlan dp;
    if (plan.ctab_total) {
        LQ_TRY(sv->ctab_buf.reserve((size_t)plan.ctab_total * sizeof(double2), sv->stream));
        dp.ctab_desc = sv->plan_buf.at<CtabDesc>(o_cd);
        dp.ctab_stage = sv->ctab_buf.at<double2>(0);
    }
    dp.subs = sv->plan_buf.at<KSub>(o_sub);
    dp.kops = sv->plan_buf.at<KOp>(o_kop);
    dp.specs = sv->plan_buf.at<MSpec>(o_spec);
    dp.factors = sv->plan_buf.at<MFactor>(o_fac);
    dp.cst = sv->plan_buf.at<double2>(o_cst);
    dp.perms = sv->plan_buf.at<KPerm>(o_perm);
    dp.pterms = sv->plan_buf.at<KPermTerm>(o_pt);
    double2 *mats = nullptr;
    if (mb.mat_size) {
        LQ_TRY(sv->work_buf.reserve((size_t)mb.mat_size * sizeof(double2), sv->stream));
        mats = sv->work_buf.at<double2>(0);
    }
    auto body = [&](cudaStream_t st) -> lq_status {
        if (mb.mat_size) {
            k_build_mats<<<grid_for(mb.specs.size()), 256, 0, st>>>(
                dp.specs, (int)mb.specs.size(), dp.factors, theta ? sv->plan_buf.at<double>(o_th) : nullptr, nullptr,
                dp.cst, mats, mb.mat_size, 1);
            LQ_TRY(check_launch("k_build_mats"));
        }
        return launch_passes(plan, dp, sv->d, 0, 1, mats, 0, st, false);
    };
    // a cached plan without per-call data: replay its CUDA graph when the
    // state's buffers are the ones it was captured with (host launch cost of
    // one graph instead of one per kernel and constant-bank copy)
    if (cp && !cp->gdisabled && !theta && plan.uid && g_opt_graphs.load() && !g_opt_timing.load()) {
        std::lock_guard<std::mutex> lk(cp->gmu);
        const std::array<const void *, 6> key{sv->d, sv->plan_buf.p, sv->work_buf.p, sv->ctab_buf.p,
                                              (const void *)sv->stream, (const void *)(uintptr_t)plan.uid};
        if (!(cp->gexec && cp->gkey == key)) {
            if (cp->gseen != key) {   // first run with these buffers: direct
                cp->gseen = key;
                return body(sv->stream);
            }
            if (cp->gexec) {
                cudaGraphExecDestroy(cp->gexec);
                cp->gexec = nullptr;
            }
            if (capture_graph(body, &cp->gexec, &cp->gkernels) != LQ_OK) {
                // a capture failure is not a fault of the state: run on the stream from now on
                cp->gdisabled = true;
                return body(sv->stream);
            }
            cp->gkey = key;
        }
        CUDA_TRY(cudaGraphLaunch(cp->gexec, sv->stream));
        g_launches.fetch_add(cp->gkernels);
        return LQ_OK;
    }
    return body(sv->stream);
}

lq_status canonicalize(lq_sv *sv) {
    if (qmap_identity(sv->n, sv->qmap)) return LQ_OK;
    std::vector<POp> ops;
    int32_t qm[64];
    memcpy(qm, sv->qmap, sizeof(qm));
    canonicalize_ops(sv->n, qm, ops);
    Plan plan;
    MatBuilder mb;
    plan_circuit(sv->n, ops, options(), mb, plan);
    LQ_TRY(run_single(sv, plan, mb, nullptr, 0));
    memcpy(sv->qmap, qm, sizeof(qm));
    return LQ_OK;
}

lq_status sync(cudaStream_t s) {
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaGetLastError());
    return LQ_OK;
}

// ---------------------------------------------------------------- NCCL (a9 transport)
struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
    decltype(&ncclCommAbort) CommAbort = nullptr;
};
NcclApi &nccl() {
    static NcclApi a = [] {
        NcclApi x;
        // reuse the NCCL torch already loaded (same soname), else the system one
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            x.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return x;
        }
#define LQ_SYM(f) x.f = reinterpret_cast<decltype(x.f)>(dlsym(h, "nccl" #f)); if (!x.f) { x.why = "missing nccl" #f; return x; }
        LQ_SYM(GetUniqueId) LQ_SYM(CommInitRank) LQ_SYM(CommDestroy) LQ_SYM(GroupStart) LQ_SYM(GroupEnd)
        LQ_SYM(Send) LQ_SYM(Recv) LQ_SYM(AllReduce) LQ_SYM(GetErrorString) LQ_SYM(CommGetAsyncError)
        LQ_SYM(CommAbort)
#undef LQ_SYM
        x.ok = true;
        return x;
    }();
    return a;
}
#define NCCL_TRY(x)                                                                             \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) return fail(LQ_ERR_NCCL, std::string(#x) + ": " + nccl().GetErrorString(r_)); \
    } while (0)

// Wait for the stream's work when it includes NCCL operations: poll the
// stream and ncclCommGetAsyncError instead of blocking, so a dead or stuck
// peer surfaces as LQ_ERR_NCCL after LQ_OPT_COMM_TIMEOUT_MS instead of a
// hang; the communicator is then aborted (later calls: LQ_ERR_STATE).
lq_status comm_abort(lq_comm *c, const std::string &why) {
    if (c->c) nccl().CommAbort(c->c);
    c->c = nullptr;
    c->dead = true;
    c->why = why;
    return fail(LQ_ERR_NCCL, why);
}
lq_status comm_sync(lq_comm *c, cudaStream_t s) {
    if (!c || !c->c) return sync(s);
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t limit_ms = g_opt_comm_timeout.load();
    for (;;) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) {
            cudaGetLastError();
            return fail(LQ_ERR_CUDA, std::string("stream failed during a collective: ") + cudaGetErrorString(e));
        }
        ncclResult_t ar = ncclSuccess;
        nccl().CommGetAsyncError(c->c, &ar);
        if (ar != ncclSuccess && ar != ncclInProgress)
            return comm_abort(c, std::string("asynchronous NCCL error: ") + nccl().GetErrorString(ar));
        const int64_t ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
        if (limit_ms > 0 && ms > limit_ms)
            return comm_abort(c, "collective did not complete within " + std::to_string(limit_ms) + " ms (peer lost?)");
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    CUDA_TRY(cudaGetLastError());
    return LQ_OK;
}
lq_status comm_check(lq_comm *c) {
    if (!c || !c->c) return LQ_OK;
    ncclResult_t ar = ncclSuccess;
    nccl().CommGetAsyncError(c->c, &ar);
    if (ar != ncclSuccess && ar != ncclInProgress)
        return comm_abort(c, std::string("asynchronous NCCL error: ") + nccl().GetErrorString(ar));
    return LQ_OK;
}

// ---------------------------------------------------------------- sharded states
lq_status sh_check(int n, int world) {
    if (world < 2 || (world & (world - 1))) return fail(LQ_ERR_ARG, "world size must be a power of two >= 2");
    int m = __builtin_ctz((unsigned)world);
    // a shard must hold the target and both controls of any gate (CCX)
    if (n - m < 3) return fail(LQ_ERR_ARG, "each shard must hold at least 3 qubits (n - log2(world) >= 3)");
    if (m > 16) return fail(LQ_ERR_ARG, "at most 2^16 shards");
    return LQ_OK;
}

// sum one double per local shard (device array), in rank order, then over
// processes (NCCL): the value every rank gets back
lq_status sh_sum(lq_sv *sv, const double *dev_vals, double *out) {
    const size_t nk = sv->shards.size();
    std::vector<double> h(nk);
    CUDA_TRY(cudaMemcpyAsync(h.data(), dev_vals, nk * sizeof(double), cudaMemcpyDeviceToHost, sv->stream));
    LQ_TRY(sync(sv->stream));
    double acc = 0.0;
    for (double v : h) acc += v;
    if (sv->comm) {
        LQ_TRY(sv->stage_buf.reserve(sizeof(double), sv->stream));
        double *d = sv->stage_buf.at<double>(0);
        CUDA_TRY(cudaMemcpyAsync(d, &acc, sizeof(double), cudaMemcpyHostToDevice, sv->stream));
        LQ_TRY(comm_check(sv->comm));
        NCCL_TRY(nccl().AllReduce(d, d, 1, ncclFloat64, ncclSum, sv->comm->c, sv->stream));
        CUDA_TRY(cudaMemcpyAsync(&acc, d, sizeof(double), cudaMemcpyDeviceToHost, sv->stream));
        LQ_TRY(comm_sync(sv->comm, sv->stream));
    }
    *out = acc;
    return LQ_OK;
}

// global-qubit exchange: k global physical bits
// g_j <-> k local bits l_j (dist.h).  Rank r (physical global bits r ^
// xmask, g-value a) sends part b of its shard to the rank whose g-value is b
// and receives that rank's part a into the same positions.
constexpr uint64_t SWAP_CHUNK = 1ull << 22;   // amplitudes per part per staged NCCL message (64 MiB)
lq_status sh_swap(lq_sv *sv, const DStep &stp) {
    const int k = stp.k, nl = sv->nl;
    PartSpec ps;
    memset(&ps, 0, sizeof(ps));
    ps.k = k;
    for (int j = 0; j < k; j++) ps.l[j] = stp.l[j];
    const uint64_t part = 1ull << (nl - k);
    const uint32_t np = (1u << k) - 1;   // parts that leave (= peers)
    auto gval = [&](int rank) {
        const uint32_t R = (uint32_t)rank ^ stp.xmask;
        uint32_t a = 0;
        for (int j = 0; j < k; j++) a |= ((R >> (stp.g[j] - nl)) & 1u) << j;
        return a;
    };
    auto peer_of = [&](int rank, uint32_t a, uint32_t b) {
        const uint32_t d = a ^ b;
        for (int j = 0; j < k; j++)
            if (d >> j & 1) rank ^= 1 << (stp.g[j] - nl);
        return rank;
    };
    cudaStream_t st = sv->stream;
    LaunchTimer lt_(KC_SWAP, st);
    NvtxRange nr_("lq exchange");
    sv->stat_exchanges++;
    sv->stat_bytes_sent += (uint64_t)np * part * sizeof(double2);
    if (!sv->comm && g_opt_group_staged.load()) {
        // group mode through NCCL mode's data path: every rank packs its
        // outgoing parts (k_pack_parts), device copies stand in for the
        // grouped ncclSend / ncclRecv (rank r's slot p -> the peer's slot for
        // part value a_r), every rank unpacks (k_unpack_parts) -- the same
        // kernels, part layout and peer map as sh_swap's NCCL branch
        const int G = (int)sv->shards.size();
        const uint64_t ch = std::min(part, (uint64_t)1 << 20), nch = part / ch;
        const size_t slot_bytes = (size_t)ch * sizeof(double2);
        LQ_TRY(sv->stage_buf.reserve(2 * (size_t)G * np * slot_bytes, st));
        double2 *outs = sv->stage_buf.at<double2>(0), *ins = outs + (size_t)G * np * ch;
        for (uint64_t c = 0; c < nch; c++) {
            for (int r = 0; r < G; r++) {
                k_pack_parts<<<dim3(grid_for(ch), np), 256, 0, st>>>(sv->shards[r], outs + (size_t)r * np * ch, ps,
                                                                     gval(r), c * ch, ch);
                LQ_TRY(check_launch("k_pack_parts"));
            }
            for (int r = 0; r < G; r++) {
                const uint32_t ar = gval(r);
                for (uint32_t p = 0; p < np; p++) {
                    const uint32_t bv = p < ar ? p : p + 1;
                    const int s2 = peer_of(r, ar, bv);
                    const uint32_t as = gval(s2), q = ar < as ? ar : ar - 1;   // the peer's slot for part a_r
                    CUDA_TRY(cudaMemcpyAsync(ins + ((size_t)s2 * np + q) * ch, outs + ((size_t)r * np + p) * ch,
                                             slot_bytes, cudaMemcpyDeviceToDevice, st));
                }
            }
            for (int r = 0; r < G; r++) {
                k_unpack_parts<<<dim3(grid_for(ch), np), 256, 0, st>>>(sv->shards[r], ins + (size_t)r * np * ch, ps,
                                                                       gval(r), c * ch, ch);
                LQ_TRY(check_launch("k_unpack_parts"));
            }
        }
        return LQ_OK;
    }
    if (!sv->comm) {   // group mode: every rank of the group lives in this process
        const int G = (int)sv->shards.size();
        for (int r = 0; r < G; r++) {
            const uint32_t a = gval(r);
            for (uint32_t b = 0; b < (1u << k); b++) {
                if (b == a) continue;
                const int r2 = peer_of(r, a, b);
                if (r2 < r) continue;   // each pair of regions once: (r, part b) <-> (r2, part a)
                k_swap_parts<<<grid_for(part), 256, 0, st>>>(sv->shards[r], sv->shards[r2], ps, b, a, part);
                LQ_TRY(check_launch("k_swap_parts"));
            }
        }
        return LQ_OK;
    }
    LQ_TRY(comm_check(sv->comm));
    const int rank = sv->comm->rank;
    const uint32_t a = gval(rank);
    const uint64_t ch = std::min(part, SWAP_CHUNK), nch = part / ch;
    LQ_TRY(sv->stage_buf.reserve(4 * (size_t)np * ch * sizeof(double2), st));
    double2 *out[2] = {sv->stage_buf.at<double2>(0), sv->stage_buf.at<double2>(np * ch * sizeof(double2))};
    double2 *in[2] = {out[1] + np * ch, out[1] + 2 * np * ch};
    if (!sv->xs) {
        CUDA_TRY(cudaStreamCreateWithFlags(&sv->xs, cudaStreamNonBlocking));
        cudaEvent_t *evs[5] = {&sv->ev_start, &sv->ev_packed[0], &sv->ev_packed[1], &sv->ev_moved[0], &sv->ev_moved[1]};
        for (cudaEvent_t *e : evs) CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    int peers[15];
    for (uint32_t p = 0; p < np; p++) peers[p] = peer_of(rank, a, p < a ? p : p + 1);
    // Pipeline: the transfer of chunk c (stream xs) overlaps the unpack of
    // chunk c-1 and the pack of chunk c+1 (handle stream).  Two staging
    // slots; chunk c+1's pack reuses the slot of chunk c-1, whose transfer
    // the handle stream waited for before unpacking it.
    CUDA_TRY(cudaEventRecord(sv->ev_start, st));
    CUDA_TRY(cudaStreamWaitEvent(sv->xs, sv->ev_start, 0));
    auto pack = [&](uint64_t c) -> lq_status {
        k_pack_parts<<<dim3(grid_for(ch), np), 256, 0, st>>>(sv->shards[0], out[c & 1], ps, a, c * ch, ch);
        LQ_TRY(check_launch("k_pack_parts"));
        CUDA_TRY(cudaEventRecord(sv->ev_packed[c & 1], st));
        return LQ_OK;
    };
    LQ_TRY(pack(0));
    for (uint64_t c = 0; c < nch; c++) {
        if (c + 1 < nch) LQ_TRY(pack(c + 1));
        CUDA_TRY(cudaStreamWaitEvent(sv->xs, sv->ev_packed[c & 1], 0));
        NCCL_TRY(nccl().GroupStart());
        for (uint32_t p = 0; p < np; p++) {
            NCCL_TRY(nccl().Send(out[c & 1] + p * ch, 2 * ch, ncclFloat64, peers[p], sv->comm->c, sv->xs));
            NCCL_TRY(nccl().Recv(in[c & 1] + p * ch, 2 * ch, ncclFloat64, peers[p], sv->comm->c, sv->xs));
        }
        NCCL_TRY(nccl().GroupEnd());
        CUDA_TRY(cudaEventRecord(sv->ev_moved[c & 1], sv->xs));
        CUDA_TRY(cudaStreamWaitEvent(st, sv->ev_moved[c & 1], 0));
        k_unpack_parts<<<dim3(grid_for(ch), np), 256, 0, st>>>(sv->shards[0], in[c & 1], ps, a, c * ch, ch);
        LQ_TRY(check_launch("k_unpack_parts"));
    }
    return LQ_OK;
}

// Run a schedule on the shards; E (nullable) receives the Pauli sum of the
// schedule's expectation step.
// Schedules of sharded calls for repeated use (the bench step, a VQE or
// Trotter loop): an LRU keyed like PlanCache plus the rank relabel and the
// exchange cap.  A hit skips scheduling, planning and JIT source generation.
struct CachedSchedule {
    Schedule sc;
    int32_t qmap_after[64];
    uint32_t xmask_after = 0;
};
struct ScheduleCache {
    std::mutex mu;
    std::list<std::pair<std::string, std::shared_ptr<CachedSchedule>>> lru;
    static constexpr size_t CAP = 16;
    std::shared_ptr<CachedSchedule> get(const std::string &k) {
        std::lock_guard<std::mutex> lk(mu);
        for (auto it = lru.begin(); it != lru.end(); ++it)
            if (it->first == k) {
                lru.splice(lru.begin(), lru, it);
                return it->second;
            }
        return nullptr;
    }
    void put(const std::string &k, std::shared_ptr<CachedSchedule> p) {
        std::lock_guard<std::mutex> lk(mu);
        lru.emplace_front(k, std::move(p));
        if (lru.size() > CAP) lru.pop_back();
    }
    void clear() {
        std::lock_guard<std::mutex> lk(mu);
        lru.clear();
    }
};
ScheduleCache g_sched_cache;

// The schedule of gates (terms == nullptr) or of a Pauli sum on sv's current
// layout, planned and JIT-prepared; cached.
lq_status sharded_schedule(lq_sv *sv, const std::string &key, const lq_gate *gates, size_t ng,
                           const lq_pauli_term *terms, size_t nt, std::shared_ptr<CachedSchedule> &out) {
    int64_t extra[3] = {sv->m, (int64_t)sv->xmask, g_opt_swap_k.load()};
    std::string k = key;
    k.append(reinterpret_cast<const char *>(extra), sizeof(extra));
    out = g_sched_cache.get(k);
    if (out) return LQ_OK;
    auto cs = std::make_shared<CachedSchedule>();
    Schedule &sc = cs->sc;
    sc.n = sv->n;
    sc.m = sv->m;
    sc.nl = sv->nl;
    sc.max_k = (int)g_opt_swap_k.load();
    sc.qft_pass_stages = qft_pass_stages(sc.nl);
    memcpy(cs->qmap_after, sv->qmap, sizeof(cs->qmap_after));
    cs->xmask_after = sv->xmask;
    if (terms || nt) {
        if (!schedule_expval(sc, terms, nt, cs->qmap_after, cs->xmask_after))
            return fail(LQ_ERR_ARG, "a Pauli term acts with X/Y on more qubits than a shard holds");
    } else if (!schedule_gates(sc, gates, ng, cs->qmap_after, cs->xmask_after)) {
        return fail(LQ_ERR_ARG, "shard too small for a gate");
    }
    plan_steps(sc, options());
    for (auto &stp : sc.steps)
        if (stp.kind == 0) {
            stp.plan.stream_tag = (uint64_t)(uintptr_t)sv->stream;
            LQ_TRY(prepare(stp.plan));
            stp.plan.prepared = true;
        }
    g_sched_cache.put(k, cs);
    out = cs;
    return LQ_OK;
}

lq_status sh_run(lq_sv *sv, const Schedule &sc, const double *theta, size_t n_theta, double *E) {
    cudaStream_t st = sv->stream;
    Blob blob;
    struct Off { size_t sub, kop, perm, pt, et, dt, cd; };
    std::vector<Off> offs(sc.steps.size());
    std::vector<DirectSet> dsets(sc.steps.size());
    uint32_t ctab_max = 0;
    for (size_t i = 0; i < sc.steps.size(); i++) {
        const DStep &stp = sc.steps[i];
        if (stp.kind != 0) continue;
        dsets[i].build(stp.plan);
        offs[i] = {blob.add(stp.plan.subs), blob.add(stp.plan.kops), blob.add(stp.plan.perms),
                   blob.add(stp.plan.perm_terms), blob.add(stp.plan.eterms), blob.add(dsets[i].terms),
                   blob.add(stp.plan.ctab_desc)};
        ctab_max = std::max(ctab_max, stp.plan.ctab_total);
    }
    if (ctab_max) LQ_TRY(sv->ctab_buf.reserve((size_t)ctab_max * sizeof(double2), st));
    size_t o_spec = blob.add(sc.mb.specs), o_fac = blob.add(sc.mb.factors), o_cst = blob.add(sc.mb.cst);
    size_t o_th = blob.add(theta, theta ? n_theta * sizeof(double) : 0);
    LQ_TRY(blob.upload(sv->plan_buf, st));
    sv->blob_uid = 0;
    double2 *mats = nullptr;
    if (sc.mb.mat_size) {
        LQ_TRY(sv->mats_buf.reserve((size_t)sc.mb.mat_size * sizeof(double2), st));
        mats = sv->mats_buf.at<double2>(0);
        k_build_mats<<<grid_for(sc.mb.specs.size()), 256, 0, st>>>(
            sv->plan_buf.at<MSpec>(o_spec), (int)sc.mb.specs.size(), sv->plan_buf.at<MFactor>(o_fac),
            theta ? sv->plan_buf.at<double>(o_th) : nullptr, nullptr, sv->plan_buf.at<double2>(o_cst), mats,
            sc.mb.mat_size, 1);
        LQ_TRY(check_launch("k_build_mats"));
    }
    const size_t nk = sv->shards.size();
    if (E) *E = 0.0;
    for (size_t i = 0; i < sc.steps.size(); i++) {
        const DStep &stp = sc.steps[i];
        if (stp.kind == 1) {
            LQ_TRY(sh_swap(sv, stp));
            continue;
        }
        DevPlan dp;
        if (stp.plan.ctab_total) {
            dp.ctab_desc = sv->plan_buf.at<CtabDesc>(offs[i].cd);
            dp.ctab_stage = sv->ctab_buf.at<double2>(0);
        }
        dp.subs = sv->plan_buf.at<KSub>(offs[i].sub);
        dp.kops = sv->plan_buf.at<KOp>(offs[i].kop);
        dp.perms = sv->plan_buf.at<KPerm>(offs[i].perm);
        dp.pterms = sv->plan_buf.at<KPermTerm>(offs[i].pt);
        dp.eterms = sv->plan_buf.at<ETerm>(offs[i].et);
        dp.specs = sv->plan_buf.at<MSpec>(o_spec);
        dp.factors = sv->plan_buf.at<MFactor>(o_fac);
        dp.cst = sv->plan_buf.at<double2>(o_cst);
        const uint32_t slots = dsets[i].stride();
        double *part = nullptr, *Ek = nullptr;
        if (stp.expv) {
            LQ_TRY(sv->part_buf.reserve(sizeof(double) * (slots + 1) * nk, st));
            part = sv->part_buf.at<double>(0);
            Ek = part + (size_t)slots * nk;
        }
        const uint32_t saved_xmask = sv->xmask;
        sv->xmask = stp.xmask;
        for (size_t k = 0; k < nk; k++) {
            lq_status r = launch_passes(stp.plan, dp, sv->shards[k], 0, 1, mats, 0, st, false,
                                        part ? part + (size_t)slots * k : nullptr, slots, false, sv->gofs((int)k));
            if (r == LQ_OK && stp.expv)
                r = finish_expv(stp.plan, dsets[i], sv->plan_buf.at<PTerm>(offs[i].dt), sv->shards[k], 0, 1,
                                part + (size_t)slots * k, slots, Ek + k, st, sv->gofs((int)k));
            if (r != LQ_OK) {
                sv->xmask = saved_xmask;
                return r;
            }
        }
        sv->xmask = saved_xmask;
        if (stp.expv && E) {
            double e = 0.0;
            LQ_TRY(sh_sum(sv, Ek, &e));
            *E += e;
        }
    }
    return LQ_OK;
}

// logical index -> (local shard slot k or -1 if another process owns it, local index)
void sh_locate(const lq_sv *sv, uint64_t x, int *k, uint64_t *li) {
    uint64_t phys = 0;
    for (int q = 0; q < sv->n; q++)
        if ((x >> (sv->n - 1 - q)) & 1) phys |= 1ull << sv->qmap[q];
    const uint64_t gb = phys >> sv->nl;
    const int rank = (int)(gb ^ sv->xmask);
    *li = phys & ((1ull << sv->nl) - 1);
    const int kk = rank - sv->rank0;
    *k = (kk >= 0 && kk < (int)sv->shards.size()) ? kk : -1;
}

lq_status sh_gather(lq_sv *sv, const uint64_t *idx, uint64_t offset, uint64_t count, double *host_out) {
    cudaStream_t st = sv->stream;
    const size_t nk = sv->shards.size();
    std::vector<std::vector<uint64_t>> li(nk), pos(nk);
    for (uint64_t i = 0; i < count; i++) {
        int k;
        uint64_t l;
        sh_locate(sv, idx ? idx[i] : offset + i, &k, &l);
        if (k >= 0) { li[k].push_back(l); pos[k].push_back(i); }
    }
    std::vector<double2> res(count, make_double2(0.0, 0.0));
    QMap ident;
    memset(&ident, 0, sizeof(ident));
    for (int q = 0; q < sv->nl; q++) ident.q[q] = (int8_t)(sv->nl - 1 - q);
    // local physical index p as a "logical" index of the identity map on nl bits
    for (size_t k = 0; k < nk; k++) {
        const uint64_t c = li[k].size();
        if (!c) continue;
        LQ_TRY(sv->work_buf.reserve(c * (sizeof(double2) + sizeof(uint64_t)), st));
        double2 *tmp = sv->work_buf.at<double2>(0);
        uint64_t *didx = reinterpret_cast<uint64_t *>(tmp + c);
        CUDA_TRY(cudaMemcpyAsync(didx, li[k].data(), c * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
        k_gather<<<grid_for(c), 256, 0, st>>>(sv->nl, ident, sv->shards[k], didx, 0, c, tmp);
        LQ_TRY(check_launch("k_gather"));
        std::vector<double2> h(c);
        CUDA_TRY(cudaMemcpyAsync(h.data(), tmp, c * sizeof(double2), cudaMemcpyDeviceToHost, st));
        LQ_TRY(sync(st));
        for (uint64_t i = 0; i < c; i++) res[pos[k][i]] = h[i];
    }
    if (sv->comm && count) {   // exactly one rank owns each index: a sum gathers them
        LQ_TRY(sv->stage_buf.reserve(count * sizeof(double2), st));
        double *d = sv->stage_buf.at<double>(0);
        CUDA_TRY(cudaMemcpyAsync(d, res.data(), count * sizeof(double2), cudaMemcpyHostToDevice, st));
        LQ_TRY(comm_check(sv->comm));
        NCCL_TRY(nccl().AllReduce(d, d, 2 * count, ncclFloat64, ncclSum, sv->comm->c, st));
        CUDA_TRY(cudaMemcpyAsync(res.data(), d, count * sizeof(double2), cudaMemcpyDeviceToHost, st));
        LQ_TRY(comm_sync(sv->comm, st));
    }
    memcpy(host_out, res.data(), count * sizeof(double2));
    return LQ_OK;
}

lq_status sh_alloc_shards(lq_sv *sv, int n_local_shards) {
    const size_t bytes = (size_t)16 << sv->nl;
    for (int k = 0; k < n_local_shards; k++) {
        void *p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            for (double2 *q : sv->shards) cudaFree(q);
            sv->shards.clear();
            return fail(LQ_ERR_OOM, std::string("shard allocation failed: ") + cudaGetErrorString(e));
        }
        sv->shards.push_back((double2 *)p);
    }
    sv->d = sv->shards[0];
    return LQ_OK;
}
}  // namespace

extern "C" {

const char *lq_last_error(void) { return g_err.c_str(); }
int lq_version(void) { return LQ_VERSION; }

int lq_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

uint64_t lq_launch_count(void) { return g_launches.load(); }

lq_status lq_jit_stats(uint64_t *compiled, uint64_t *cache_hits, double *compile_seconds) {
    jit_stats(compiled, cache_hits, compile_seconds);
    return LQ_OK;
}

lq_status lq_kernel_timing(int kernel_class, double *total_ms, uint64_t *count) {
    if (kernel_class < 0 || kernel_class >= KC_N) return fail(LQ_ERR_ARG, "bad kernel class");
    harvest_timing();
    if (total_ms) *total_ms = g_time_ms[kernel_class];
    if (count) *count = g_time_cnt[kernel_class];
    return LQ_OK;
}

lq_status lq_kernel_timing_reset(void) {
    harvest_timing();
    for (int k = 0; k < KC_N; k++) { g_time_ms[k] = 0; g_time_cnt[k] = 0; }
    return LQ_OK;
}

lq_status lq_set_option(int option, int64_t value) {
    switch (option) {
    case LQ_OPT_FUSION: g_opt_fusion = value ? 1 : 0; return LQ_OK;
    case LQ_OPT_TILE_BITS:
        if (value != 0 && (value < 1 || value > 12)) return fail(LQ_ERR_ARG, "tile bits must be 0 or 1..12");
        g_opt_K = value;
        return LQ_OK;
    case LQ_OPT_COALESCE_BITS:
        if (value < 0 || value > 6) return fail(LQ_ERR_ARG, "coalesce bits must be 0..6");
        g_opt_coalesce = value;
        return LQ_OK;
    case LQ_OPT_REG_BITS:
        if (value < 2 || value > 4) return fail(LQ_ERR_ARG, "register bits must be 2..4");
        g_opt_regbits = value;
        return LQ_OK;
    case LQ_OPT_KERNEL_TIMING:
        g_opt_timing = value ? 1 : 0;
        return LQ_OK;
    case LQ_OPT_PASS_BUDGET:
        if (value < 0 || value > 100000) return fail(LQ_ERR_ARG, "pass budget must be 0..100000");
        g_opt_budget = value;
        return LQ_OK;
    case LQ_OPT_JIT:
        if (value < 0 || value > 2) return fail(LQ_ERR_ARG, "jit must be 0 (off), 1 (auto) or 2 (always)");
        g_opt_jit = value;
        return LQ_OK;
    case LQ_OPT_FIRST_PASS_FREE: g_opt_first_free = value ? 1 : 0; return LQ_OK;
    case LQ_OPT_POISON_ALLOC: g_opt_poison = value ? 1 : 0; return LQ_OK;
    case LQ_OPT_GROUP_STAGED: g_opt_group_staged = value ? 1 : 0; return LQ_OK;
    case LQ_OPT_STATE_PASS_BUDGET:
        if (value < 0 || value > 100000) return fail(LQ_ERR_ARG, "pass budget must be 0..100000");
        g_opt_state_budget = value;
        return LQ_OK;
    case LQ_OPT_COMM_TIMEOUT_MS:
        if (value < 0) return fail(LQ_ERR_ARG, "timeout must be >= 0 (0 = wait forever)");
        g_opt_comm_timeout = value;
        return LQ_OK;
    case LQ_OPT_SWAP_QUBITS:
        if (value < 1 || value > 4) return fail(LQ_ERR_ARG, "qubits per exchange must be 1..4");
        g_opt_swap_k = value;
        return LQ_OK;
    case LQ_OPT_RELABEL_STORES:
        if (value != 0 && (value < 3 || value > 5)) return fail(LQ_ERR_ARG, "relabel stores must be 0 or 3..5");
        g_opt_relabel = value;
        return LQ_OK;
    case LQ_OPT_EXPORT_PSR: g_opt_export_psr = value ? 1 : 0; return LQ_OK;
    case LQ_OPT_GRAPHS: g_opt_graphs = value ? 1 : 0; return LQ_OK;
    default: return fail(LQ_ERR_ARG, "unknown option");
    }
}

int64_t lq_get_option(int option) {
    switch (option) {
    case LQ_OPT_FUSION: return g_opt_fusion.load();
    case LQ_OPT_TILE_BITS: return g_opt_K.load();
    case LQ_OPT_COALESCE_BITS: return g_opt_coalesce.load();
    case LQ_OPT_REG_BITS: return g_opt_regbits.load();
    case LQ_OPT_KERNEL_TIMING: return g_opt_timing.load();
    case LQ_OPT_JIT: return g_opt_jit.load();
    case LQ_OPT_PASS_BUDGET: return g_opt_budget.load();
    case LQ_OPT_FIRST_PASS_FREE: return g_opt_first_free.load();
    case LQ_OPT_POISON_ALLOC: return g_opt_poison.load();
    case LQ_OPT_COMM_TIMEOUT_MS: return g_opt_comm_timeout.load();
    case LQ_OPT_RELABEL_STORES: return g_opt_relabel.load();
    case LQ_OPT_EXPORT_PSR: return g_opt_export_psr.load();
    case LQ_OPT_GRAPHS: return g_opt_graphs.load();
    case LQ_OPT_STATE_PASS_BUDGET: return g_opt_state_budget.load();
    case LQ_OPT_GROUP_STAGED: return g_opt_group_staged.load();
    case LQ_OPT_SWAP_QUBITS: return g_opt_swap_k.load();
    default: return -1;
    }
}

lq_status lq_sv_alloc(int n_qubits, void *cuda_stream, lq_sv **out) {
    if (!out) return fail(LQ_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (n_qubits < 1 || n_qubits > 40) return fail(LQ_ERR_ARG, "n_qubits must be in [1, 40]");
    LQ_TRY(have_device());
    size_t bytes = (size_t)16 << n_qubits;
    size_t fr = 0, tot = 0;
    CUDA_TRY(cudaMemGetInfo(&fr, &tot));
    if (bytes > fr) return fail(LQ_ERR_OOM, "state of " + std::to_string(bytes) + " bytes exceeds free device memory");
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(LQ_ERR_OOM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    }
    lq_sv *sv = new lq_sv();
    sv->n = n_qubits;
    sv->d = (double2 *)p;
    sv->owned = true;
    sv->stream = (cudaStream_t)cuda_stream;
    sv->reset_map();
    *out = sv;
    return LQ_OK;
}

lq_status lq_sv_wrap(int n_qubits, void *cuda_stream, void *dev_ptr, size_t bytes, lq_sv **out) {
    if (!out) return fail(LQ_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (n_qubits < 1 || n_qubits > 40) return fail(LQ_ERR_ARG, "n_qubits must be in [1, 40]");
    if (!dev_ptr || ((uintptr_t)dev_ptr & 15)) return fail(LQ_ERR_ARG, "dev_ptr must be non-NULL and 16-byte aligned");
    if (bytes < ((size_t)16 << n_qubits)) return fail(LQ_ERR_DIM, "wrapped buffer smaller than 16 * 2^n bytes");
    LQ_TRY(have_device());
    lq_sv *sv = new lq_sv();
    sv->n = n_qubits;
    sv->d = (double2 *)dev_ptr;
    sv->owned = false;
    sv->stream = (cudaStream_t)cuda_stream;
    sv->reset_map();
    *out = sv;
    return LQ_OK;
}

lq_status lq_comm_unique_id(void *out, size_t len) {
    if (!out || len < sizeof(ncclUniqueId)) return fail(LQ_ERR_ARG, "need a 128-byte buffer");
    if (!nccl().ok) return fail(LQ_ERR_NCCL, nccl().why);
    ncclUniqueId id;
    NCCL_TRY(nccl().GetUniqueId(&id));
    memcpy(out, &id, sizeof(id));
    return LQ_OK;
}

lq_status lq_comm_init(const void *unique_id, size_t len, int rank, int world, lq_comm **out) {
    if (!out || !unique_id || len < sizeof(ncclUniqueId)) return fail(LQ_ERR_ARG, "bad unique id / out");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(LQ_ERR_ARG, "bad rank/world");
    LQ_TRY(have_device());
    if (!nccl().ok) return fail(LQ_ERR_NCCL, nccl().why);
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    lq_comm *c = new lq_comm();
    c->rank = rank;
    c->world = world;
    ncclResult_t r = nccl().CommInitRank(&c->c, world, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return fail(LQ_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
    }
    *out = c;
    return LQ_OK;
}

lq_status lq_comm_init_local(int rank, int world, lq_comm **out) {
    if (!out) return fail(LQ_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(LQ_ERR_ARG, "bad rank/world");
    lq_comm *c = new lq_comm();
    c->rank = rank;
    c->world = world;
    c->local = true;
    *out = c;
    return LQ_OK;
}

lq_status lq_comm_info(const lq_comm *c, int *rank, int *world, int *has_transport) {
    if (!c) return fail(LQ_ERR_ARG, "comm is NULL");
    if (c->dead) return fail(LQ_ERR_STATE, "communicator aborted after an earlier failure: " + c->why);
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    if (has_transport) *has_transport = c->c != nullptr;
    return LQ_OK;
}

lq_status lq_sv_exchange_stats(const lq_sv *sv, uint64_t *n_exchanges, uint64_t *bytes_sent_per_rank) {
    if (!sv) return fail(LQ_ERR_ARG, "invalid state handle");
    if (n_exchanges) *n_exchanges = sv->stat_exchanges;
    if (bytes_sent_per_rank) *bytes_sent_per_rank = sv->stat_bytes_sent;   // every rank sends the same amount
    return LQ_OK;
}

lq_status lq_comm_free(lq_comm *c) {
    if (!c) return LQ_OK;
    if (c->c) nccl().CommDestroy(c->c);
    delete c;
    return LQ_OK;
}

lq_status lq_sv_alloc_group(int n_qubits, int world, void *cuda_stream, lq_sv **out) {
    if (!out) return fail(LQ_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (n_qubits < 2 || n_qubits > 40) return fail(LQ_ERR_ARG, "n_qubits must be in [2, 40]");
    LQ_TRY(sh_check(n_qubits, world));
    LQ_TRY(have_device());
    lq_sv *sv = new lq_sv();
    sv->n = n_qubits;
    sv->m = __builtin_ctz((unsigned)world);
    sv->nl = n_qubits - sv->m;
    sv->stream = (cudaStream_t)cuda_stream;
    sv->owned = false;
    sv->reset_map();
    lq_status s = sh_alloc_shards(sv, world);
    if (s != LQ_OK) { delete sv; return s; }
    *out = sv;
    return LQ_OK;
}

lq_status lq_sv_alloc_sharded(int n_qubits, lq_comm *comm, void *cuda_stream, lq_sv **out) {
    if (!out) return fail(LQ_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (!comm) return fail(LQ_ERR_ARG, "comm is NULL");
    if (n_qubits < 2 || n_qubits > 44) return fail(LQ_ERR_ARG, "n_qubits must be in [2, 44]");
    if (comm->world == 1) return lq_sv_alloc(n_qubits, cuda_stream, out);
    LQ_TRY(sh_check(n_qubits, comm->world));
    LQ_TRY(have_device());
    lq_sv *sv = new lq_sv();
    sv->n = n_qubits;
    sv->m = __builtin_ctz((unsigned)comm->world);
    sv->nl = n_qubits - sv->m;
    sv->comm = comm;
    sv->rank0 = comm->rank;
    sv->stream = (cudaStream_t)cuda_stream;
    sv->reset_map();
    lq_status s = sh_alloc_shards(sv, 1);
    if (s != LQ_OK) { delete sv; return s; }
    *out = sv;
    return LQ_OK;
}

lq_status lq_sv_shard_info(const lq_sv *sv, int *log2_world, int *first_rank, int *n_local_shards, uint32_t *xmask) {
    LQ_TRY(check_sv(sv));
    if (log2_world) *log2_world = sv->m;
    if (first_rank) *first_rank = sv->rank0;
    if (n_local_shards) *n_local_shards = sv->m ? (int)sv->shards.size() : 1;
    if (xmask) *xmask = sv->xmask;
    return LQ_OK;
}

void *lq_sv_shard_ptr(const lq_sv *sv, int k) {
    if (!sv) return nullptr;
    if (!sv->m) return k == 0 ? (void *)sv->d : nullptr;
    return (k >= 0 && k < (int)sv->shards.size()) ? (void *)sv->shards[k] : nullptr;
}

lq_status lq_dist_schedule_json(int n_qubits, int log2_world, const lq_gate *gates, size_t n_gates, int qft,
                                const lq_pauli_term *terms, size_t n_terms, char *buf, size_t buf_len,
                                size_t *needed) {
    if (n_qubits < 2 || n_qubits > 44 || log2_world < 1 || n_qubits - log2_world < 3)
        return fail(LQ_ERR_ARG, "need log2_world >= 1 and n_qubits - log2_world >= 3 (n_qubits <= 44)");
    LQ_TRY(validate_gates(n_qubits, gates, n_gates, nullptr, 1 << 16, false, nullptr));
    LQ_TRY(validate_terms(n_qubits, terms, n_terms));
    Schedule sc;
    sc.n = n_qubits;
    sc.m = log2_world;
    sc.nl = n_qubits - log2_world;
    sc.max_k = (int)g_opt_swap_k.load();
    sc.qft_pass_stages = qft_pass_stages(sc.nl);
    int32_t qm[64];
    for (int q = 0; q < n_qubits; q++) qm[q] = n_qubits - 1 - q;
    uint32_t xm = 0;
    if (!schedule_gates(sc, gates, n_gates, qm, xm)) return fail(LQ_ERR_ARG, "shard too small for a gate");
    if (qft) {
        std::vector<lq_gate> g = qft_gates(n_qubits, qft < 0);
        if (!schedule_gates(sc, g.data(), g.size(), qm, xm)) return fail(LQ_ERR_ARG, "shard too small");
    }
    if (n_terms && !schedule_expval(sc, terms, n_terms, qm, xm))
        return fail(LQ_ERR_ARG, "a Pauli term acts with X/Y on more qubits than a shard holds");
    plan_steps(sc, options());
    std::string j = schedule_json(sc, qm, xm);
    if (needed) *needed = j.size() + 1;
    if (buf && buf_len) {
        size_t k = std::min(buf_len - 1, j.size());
        memcpy(buf, j.data(), k);
        buf[k] = 0;
    }
    return LQ_OK;
}

lq_status lq_sv_free(lq_sv *sv) {
    if (!sv) return LQ_OK;
    sv->plan_buf.release(sv->stream);
    sv->blob_uid = 0;
    sv->work_buf.release(sv->stream);
    sv->mats_buf.release(sv->stream);
    sv->part_buf.release(sv->stream);
    sv->stage_buf.release(sv->stream);
    sv->ctab_buf.release(sv->stream);
    if (sv->xs) {
        cudaStreamSynchronize(sv->stream);
        cudaStreamDestroy(sv->xs);
        for (cudaEvent_t ev : {sv->ev_start, sv->ev_packed[0], sv->ev_packed[1], sv->ev_moved[0], sv->ev_moved[1]})
            if (ev) cudaEventDestroy(ev);
    }
    cudaError_t e = cudaSuccess;
    if (!sv->shards.empty()) {
        cudaStreamSynchronize(sv->stream);
        for (double2 *p : sv->shards) {
            cudaError_t e2 = cudaFree(p);
            if (e2 != cudaSuccess) e = e2;
        }
        sv->shards.clear();
        sv->d = nullptr;
    }
    if (sv->owned && sv->d) {
        cudaStreamSynchronize(sv->stream);
        e = cudaFree(sv->d);
    }
    delete sv;
    if (e != cudaSuccess) return fail(LQ_ERR_CUDA, std::string("cudaFree failed: ") + cudaGetErrorString(e));
    return LQ_OK;
}

lq_status lq_sv_set_stream(lq_sv *sv, void *cuda_stream) {
    LQ_TRY(check_sv(sv));
    // order the old stream's pending work (and buffer frees) before the new one
    CUDA_TRY(cudaStreamSynchronize(sv->stream));
    sv->stream = (cudaStream_t)cuda_stream;
    return LQ_OK;
}

int lq_sv_num_qubits(const lq_sv *sv) { return sv ? sv->n : -1; }
void *lq_sv_device_ptr(const lq_sv *sv) { return sv ? (void *)sv->d : nullptr; }

lq_status lq_sv_qubit_map(const lq_sv *sv, int32_t *map_out) {
    LQ_TRY(check_sv(sv));
    if (!map_out) return fail(LQ_ERR_ARG, "map_out is NULL");
    for (int q = 0; q < sv->n; q++) map_out[q] = sv->qmap[q];
    return LQ_OK;
}

static lq_status sv_init_basis_body(lq_sv *sv, uint64_t k) {
    LQ_TRY(check_sv(sv));
    if (k >= (1ull << sv->n)) return fail(LQ_ERR_ARG, "basis index out of range");
    sv->reset_map();
    if (sv->m) {   // identity layout: logical k lives on rank k >> nl
        const uint64_t Nl = 1ull << sv->nl;
        for (size_t s2 = 0; s2 < sv->shards.size(); s2++) {
            const bool own = (int)(k >> sv->nl) == sv->rank0 + (int)s2;
            k_fill_basis<<<dim3(grid_for(Nl), 1), 256, 0, sv->stream>>>(Nl, own ? (k & (Nl - 1)) : ~0ull,
                                                                         sv->shards[s2], 0);
            LQ_TRY(check_launch("k_fill_basis"));
        }
        return LQ_OK;
    }
    const uint64_t N = 1ull << sv->n;
    k_fill_basis<<<dim3(grid_for(N), 1), 256, 0, sv->stream>>>(N, k, sv->d, 0);
    return check_launch("k_fill_basis");
}

static lq_status sv_init_random_body(lq_sv *sv, uint64_t seed) {
    LQ_TRY(check_sv(sv));
    sv->reset_map();
    if (sv->m) {   // norm over all shards (sh_sum), then each shard writes its range
        const uint64_t Nl = 1ull << sv->nl;
        const size_t nk = sv->shards.size();
        LQ_TRY(sv->work_buf.reserve(sizeof(double) * (RED_BLOCKS * nk + nk + 1), sv->stream));
        double *part = sv->work_buf.at<double>(0), *sums = part + RED_BLOCKS * nk, *tot = sums + nk;
        for (size_t k2 = 0; k2 < nk; k2++) {
            k_random_norm<<<RED_BLOCKS, 256, 0, sv->stream>>>(Nl, sv->gofs((int)k2), seed, part + RED_BLOCKS * k2);
            LQ_TRY(check_launch("k_random_norm"));
            k_sum_partials<<<1, 256, 0, sv->stream>>>(part + RED_BLOCKS * k2, 0, RED_BLOCKS, sums + k2);
            LQ_TRY(check_launch("k_sum_partials"));
        }
        double total = 0.0;
        LQ_TRY(sh_sum(sv, sums, &total));
        CUDA_TRY(cudaMemcpyAsync(tot, &total, sizeof(double), cudaMemcpyHostToDevice, sv->stream));
        for (size_t k2 = 0; k2 < nk; k2++) {
            k_random_write<<<grid_for(Nl), 256, 0, sv->stream>>>(Nl, sv->gofs((int)k2), seed, tot, sv->shards[k2]);
            LQ_TRY(check_launch("k_random_write"));
        }
        return sync(sv->stream);   // `total` lives on this stack frame
    }
    const uint64_t N = 1ull << sv->n;
    LQ_TRY(sv->work_buf.reserve(sizeof(double) * (RED_BLOCKS + 1), sv->stream));
    double *part = sv->work_buf.at<double>(0);
    k_random_norm<<<RED_BLOCKS, 256, 0, sv->stream>>>(N, 0, seed, part);
    LQ_TRY(check_launch("k_random_norm"));
    k_sum_partials<<<1, 256, 0, sv->stream>>>(part, 0, RED_BLOCKS, part + RED_BLOCKS);
    LQ_TRY(check_launch("k_sum_partials"));
    k_random_write<<<grid_for(N), 256, 0, sv->stream>>>(N, 0, seed, part + RED_BLOCKS, sv->d);
    return check_launch("k_random_write");
}

static lq_status sv_norm2_body(lq_sv *sv, double *out) {
    LQ_TRY(check_sv(sv));
    if (!out) return fail(LQ_ERR_ARG, "out is NULL");
    if (sv->m) {
        const uint64_t Nl = 1ull << sv->nl;
        const size_t nk = sv->shards.size();
        LQ_TRY(sv->work_buf.reserve(sizeof(double) * (RED_BLOCKS * nk + nk), sv->stream));
        double *part = sv->work_buf.at<double>(0), *sums = part + RED_BLOCKS * nk;
        for (size_t k2 = 0; k2 < nk; k2++) {
            k_norm2<<<RED_BLOCKS, 256, 0, sv->stream>>>(Nl, sv->shards[k2], part + RED_BLOCKS * k2);
            LQ_TRY(check_launch("k_norm2"));
            k_sum_partials<<<1, 256, 0, sv->stream>>>(part + RED_BLOCKS * k2, 0, RED_BLOCKS, sums + k2);
            LQ_TRY(check_launch("k_sum_partials"));
        }
        return sh_sum(sv, sums, out);
    }
    const uint64_t N = 1ull << sv->n;
    LQ_TRY(sv->work_buf.reserve(sizeof(double) * (RED_BLOCKS + 1), sv->stream));
    double *part = sv->work_buf.at<double>(0);
    k_norm2<<<RED_BLOCKS, 256, 0, sv->stream>>>(N, sv->d, part);
    LQ_TRY(check_launch("k_norm2"));
    k_sum_partials<<<1, 256, 0, sv->stream>>>(part, 0, RED_BLOCKS, part + RED_BLOCKS);
    LQ_TRY(check_launch("k_sum_partials"));
    CUDA_TRY(cudaMemcpyAsync(out, part + RED_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, sv->stream));
    return sync(sv->stream);
}

static lq_status read_impl(lq_sv *sv, const uint64_t *idx, uint64_t offset, uint64_t count, double *host_out) {
    const uint64_t CH = 1ull << 22;   // 64 MiB chunks
    size_t need = (size_t)std::min(count, CH) * (sizeof(double2) + (idx ? sizeof(uint64_t) : 0));
    LQ_TRY(sv->work_buf.reserve(std::max<size_t>(need, 16), sv->stream));
    QMap m = to_qmap(sv->n, sv->qmap);
    for (uint64_t c0 = 0; c0 < count; c0 += CH) {
        uint64_t cnt = std::min(CH, count - c0);
        double2 *tmp = sv->work_buf.at<double2>(0);
        uint64_t *didx = nullptr;
        if (idx) {
            didx = reinterpret_cast<uint64_t *>(tmp + std::min(count, CH));
            CUDA_TRY(cudaMemcpyAsync(didx, idx + c0, cnt * sizeof(uint64_t), cudaMemcpyHostToDevice, sv->stream));
        }
        k_gather<<<grid_for(cnt), 256, 0, sv->stream>>>(sv->n, m, sv->d, didx, offset + c0, cnt, tmp);
        LQ_TRY(check_launch("k_gather"));
        CUDA_TRY(cudaMemcpyAsync(host_out + 2 * c0, tmp, cnt * sizeof(double2), cudaMemcpyDeviceToHost, sv->stream));
        LQ_TRY(sync(sv->stream));
    }
    return LQ_OK;
}

static lq_status sv_read_body(lq_sv *sv, uint64_t offset, uint64_t count, double *host_out) {
    LQ_TRY(check_sv(sv));
    if (!host_out && count) return fail(LQ_ERR_ARG, "host_out is NULL");
    uint64_t N = 1ull << sv->n;
    if (offset > N || count > N - offset) return fail(LQ_ERR_DIM, "read range out of bounds");
    if (!count) return LQ_OK;
    if (sv->m) return sh_gather(sv, nullptr, offset, count, host_out);
    return read_impl(sv, nullptr, offset, count, host_out);
}

static lq_status sv_gather_body(lq_sv *sv, const uint64_t *idx, size_t count, double *host_out) {
    LQ_TRY(check_sv(sv));
    if (count && (!idx || !host_out)) return fail(LQ_ERR_ARG, "NULL buffer");
    uint64_t N = 1ull << sv->n;
    for (size_t i = 0; i < count; i++)
        if (idx[i] >= N) return fail(LQ_ERR_DIM, "gather index out of range");
    if (!count) return LQ_OK;
    if (sv->m) return sh_gather(sv, idx, 0, count, host_out);
    return read_impl(sv, idx, 0, count, host_out);
}

static lq_status sv_write_body(lq_sv *sv, uint64_t offset, uint64_t count, const double *host_in) {
    LQ_TRY(check_sv(sv));
    if (!host_in && count) return fail(LQ_ERR_ARG, "host_in is NULL");
    uint64_t N = 1ull << sv->n;
    if (offset > N || count > N - offset) return fail(LQ_ERR_DIM, "write range out of bounds");
    for (uint64_t i = 0; i < 2 * count; i++)
        if (!std::isfinite(host_in[i])) return fail(LQ_ERR_NONFINITE, "non-finite amplitude");
    if (sv->m) {   // sharded: every rank writes the amplitudes it owns (collective, same host data)
        const size_t nk = sv->shards.size();
        std::vector<std::vector<uint64_t>> li(nk);
        std::vector<std::vector<double2>> val(nk);
        for (uint64_t i = 0; i < count; i++) {
            int k;
            uint64_t l;
            sh_locate(sv, offset + i, &k, &l);
            if (k < 0) continue;
            li[k].push_back(l);
            val[k].push_back(make_double2(host_in[2 * i], host_in[2 * i + 1]));
        }
        QMap ident;
        memset(&ident, 0, sizeof(ident));
        for (int q = 0; q < sv->nl; q++) ident.q[q] = (int8_t)(sv->nl - 1 - q);
        for (size_t k = 0; k < nk; k++) {
            const uint64_t c = li[k].size();
            if (!c) continue;
            LQ_TRY(sv->work_buf.reserve(c * (sizeof(double2) + sizeof(uint64_t)), sv->stream));
            double2 *tmp = sv->work_buf.at<double2>(0);
            uint64_t *didx = reinterpret_cast<uint64_t *>(tmp + c);
            CUDA_TRY(cudaMemcpyAsync(tmp, val[k].data(), c * sizeof(double2), cudaMemcpyHostToDevice, sv->stream));
            CUDA_TRY(cudaMemcpyAsync(didx, li[k].data(), c * sizeof(uint64_t), cudaMemcpyHostToDevice, sv->stream));
            k_scatter<<<grid_for(c), 256, 0, sv->stream>>>(sv->nl, ident, sv->shards[k], didx, 0, c, tmp);
            LQ_TRY(check_launch("k_scatter"));
            LQ_TRY(sync(sv->stream));
        }
        return LQ_OK;
    }
    const uint64_t CH = 1ull << 22;
    LQ_TRY(sv->work_buf.reserve((size_t)std::min(count, CH) * sizeof(double2) + 16, sv->stream));
    QMap m = to_qmap(sv->n, sv->qmap);
    for (uint64_t c0 = 0; c0 < count; c0 += CH) {
        uint64_t cnt = std::min(CH, count - c0);
        double2 *tmp = sv->work_buf.at<double2>(0);
        CUDA_TRY(cudaMemcpyAsync(tmp, host_in + 2 * c0, cnt * sizeof(double2), cudaMemcpyHostToDevice, sv->stream));
        k_scatter<<<grid_for(cnt), 256, 0, sv->stream>>>(sv->n, m, sv->d, nullptr, offset + c0, cnt, tmp);
        LQ_TRY(check_launch("k_scatter"));
        LQ_TRY(sync(sv->stream));
    }
    return LQ_OK;
}

static lq_status sv_canonicalize_body(lq_sv *sv) {
    LQ_TRY(check_sv(sv));
    if (sv->m) return fail(LQ_ERR_ARG, "lq_sv_canonicalize is not supported on sharded states (reads resolve the layout)");
    return canonicalize(sv);
}

}  // extern "C"

namespace {
// apply already-validated gates (internal kinds allowed)
lq_status apply_impl(lq_sv *sv, const lq_gate *gates, size_t n_gates, const double *theta, size_t n_theta) {
    if (!n_gates) return LQ_OK;
    if (sv->m) {
        std::shared_ptr<CachedSchedule> cs;
        LQ_TRY(sharded_schedule(sv, gates_key(sv->n, sv->qmap, gates, n_gates, sv->stream), gates, n_gates, nullptr,
                                0, cs));
        LQ_TRY(sh_run(sv, cs->sc, theta, n_theta, nullptr));
        memcpy(sv->qmap, cs->qmap_after, sizeof(sv->qmap));
        sv->xmask = cs->xmask_after;
        return LQ_OK;
    }
    const std::string key = gates_key(sv->n, sv->qmap, gates, n_gates, sv->stream);
    std::shared_ptr<CachedPlan> cp = g_plan_cache.get(key);
    if (!cp) {
        cp = std::make_shared<CachedPlan>();
        memcpy(cp->qmap_after, sv->qmap, sizeof(cp->qmap_after));
        std::vector<POp> ops;
        lower_gates(sv->n, gates, n_gates, cp->qmap_after, ops, cp->mb);
        plan_circuit(sv->n, ops, options(), cp->mb, cp->plan);
        cp->plan.stream_tag = (uint64_t)(uintptr_t)sv->stream;
        if (!cp->plan.passes.empty()) LQ_TRY(prepare(cp->plan));
        cp->plan.prepared = true;
        cp->plan.uid = next_plan_uid();
        g_plan_cache.put(key, cp);
    }
    LQ_TRY(promote(*cp));
    LQ_TRY(run_single(sv, cp->plan, cp->mb, theta, n_theta, cp.get()));
    memcpy(sv->qmap, cp->qmap_after, sizeof(sv->qmap));
    return LQ_OK;
}
}  // namespace

extern "C" {

static lq_status apply_circuit_body(lq_sv *sv, const lq_gate *gates, size_t n_gates, const double *theta, size_t n_theta) {
    LQ_TRY(check_sv(sv));
    LQ_TRY(validate_gates(sv->n, gates, n_gates, theta, n_theta, true, nullptr));
    return apply_impl(sv, gates, n_gates, theta, n_theta);
}

static lq_status qft_body(lq_sv *sv, int inverse) {
    LQ_TRY(check_sv(sv));
    int32_t qm[64];
    memcpy(qm, sv->qmap, sizeof(qm));
    bool ident = true, rev = true;
    for (int q = 0; q < sv->n; q++) {
        ident &= qm[q] == sv->n - 1 - q;
        rev &= qm[q] == q;
    }
    if (sv->m || (!ident && !rev)) {
        // sharded or permuted layout: Alg. 3's stages as generic ops (any
        // layout; the scheduler swaps global qubits in), SWAP layer = relabel
        std::vector<lq_gate> g = qft_gates(sv->n, inverse != 0);
        return apply_impl(sv, g.data(), g.size(), nullptr, 0);
    }
    const int inv = inverse != 0;
    const std::string key = plan_key('q', sv->n, qm, &inv, sizeof(inv), sv->stream);
    std::shared_ptr<CachedPlan> cp = g_plan_cache.get(key);
    if (!cp) {
        cp = std::make_shared<CachedPlan>();
        memcpy(cp->qmap_after, qm, sizeof(qm));
        if (!plan_qft(sv->n, cp->qmap_after, inv, options(), cp->plan, cp->mb))
            return fail(LQ_ERR_STATE, "qft planning failed");
        cp->plan.stream_tag = (uint64_t)(uintptr_t)sv->stream;
        LQ_TRY(prepare(cp->plan));
        cp->plan.prepared = true;
        cp->plan.uid = next_plan_uid();
        g_plan_cache.put(key, cp);
    }
    LQ_TRY(promote(*cp));
    LQ_TRY(run_single(sv, cp->plan, cp->mb, nullptr, 0, cp.get()));
    memcpy(sv->qmap, cp->qmap_after, sizeof(sv->qmap));
    return LQ_OK;
}

static lq_status expval_pauli_sum_body(lq_sv *sv, const lq_pauli_term *terms, size_t n_terms, double *out_energy) {
    LQ_TRY(check_sv(sv));
    if (!out_energy) return fail(LQ_ERR_ARG, "out_energy is NULL");
    LQ_TRY(validate_terms(sv->n, terms, n_terms));
    if (sv->m) {
        std::shared_ptr<CachedSchedule> cs;
        static const lq_pauli_term none{};
        LQ_TRY(sharded_schedule(sv, plan_key('e', sv->n, sv->qmap, terms, sizeof(lq_pauli_term) * n_terms, sv->stream),
                                nullptr, 0, n_terms ? terms : &none, n_terms, cs));
        LQ_TRY(sh_run(sv, cs->sc, nullptr, 0, out_energy));
        memcpy(sv->qmap, cs->qmap_after, sizeof(sv->qmap));
        sv->xmask = cs->xmask_after;
        return LQ_OK;
    }
    const std::string key = plan_key('e', sv->n, sv->qmap, terms, sizeof(lq_pauli_term) * n_terms, sv->stream);
    std::shared_ptr<CachedPlan> cp = g_plan_cache.get(key);
    if (!cp) {
        cp = std::make_shared<CachedPlan>();
        std::vector<POp> ops;
        lower_pauli(sv->n, sv->qmap, terms, n_terms, ops, cp->plan);
        plan_circuit(sv->n, ops, options(), cp->mb, cp->plan);
        cp->plan.stream_tag = (uint64_t)(uintptr_t)sv->stream;
        LQ_TRY(prepare(cp->plan));
        cp->plan.prepared = true;
        cp->plan.uid = next_plan_uid();
        g_plan_cache.put(key, cp);
    }
    LQ_TRY(promote(*cp));
    const Plan &plan = cp->plan;
    DirectSet dset;
    dset.build(plan);
    Blob blob;
    size_t o_sub = blob.add(plan.subs), o_kop = blob.add(plan.kops), o_perm = blob.add(plan.perms),
           o_pt = blob.add(plan.perm_terms), o_et = blob.add(plan.eterms), o_dt = blob.add(dset.terms),
           o_cd = blob.add(plan.ctab_desc);
    LQ_TRY(upload_tables(sv, blob, plan.uid));
    DevPlan dp;
    if (plan.ctab_total) {
        LQ_TRY(sv->ctab_buf.reserve((size_t)plan.ctab_total * sizeof(double2), sv->stream));
        dp.ctab_desc = sv->plan_buf.at<CtabDesc>(o_cd);
        dp.ctab_stage = sv->ctab_buf.at<double2>(0);
    }
    dp.subs = sv->plan_buf.at<KSub>(o_sub);
    dp.kops = sv->plan_buf.at<KOp>(o_kop);
    dp.perms = sv->plan_buf.at<KPerm>(o_perm);
    dp.pterms = sv->plan_buf.at<KPermTerm>(o_pt);
    dp.eterms = sv->plan_buf.at<ETerm>(o_et);
    LQ_TRY(sv->work_buf.reserve(sizeof(double) * (dset.stride() + 2), sv->stream));
    double *part = sv->work_buf.at<double>(0);
    double *E = part + dset.stride() + 1;
    LQ_TRY(launch_passes(plan, dp, sv->d, 0, 1, nullptr, 0, sv->stream, false, part, dset.stride(), false));
    LQ_TRY(finish_expv(plan, dset, sv->plan_buf.at<PTerm>(o_dt), sv->d, 0, 1, part, dset.stride(), E, sv->stream));
    CUDA_TRY(cudaMemcpyAsync(out_energy, E, sizeof(double), cudaMemcpyDeviceToHost, sv->stream));
    return sync(sv->stream);
}

// First-order Trotter evolution of the XYZ chain (
// PAPER.md:777-836).  Every step is the gate list of P:825-831 with the
// signs of Eq. (9) (reading A20): RXX(-2 Jx dt) on each pair left to right,
// then RYY(-2 Jy dt), RZZ(-2 Jz dt), then RZ(-2 h(t_j) dt) on each site
// (SPEC.md:539-541 order).  The field angles are parameters (theta), so up
// to 8 steps share one cached plan whatever h(t) is, and the planner fuses
// across step boundaries.  E(t) = E_int - h(t) M with E_int = <-sum J PP>
// and M = <sum Z_i> (two cached expectation plans).
static lq_status trotter_xyz_body(lq_sv *sv, const lq_xyz_model *mdl, double t0, double dt, int n_steps, int record_every,
                         double *energy_out) {
    LQ_TRY(check_sv(sv));
    if (!mdl) return fail(LQ_ERR_ARG, "model is NULL");
    const double v[7] = {mdl->jx, mdl->jy, mdl->jz, mdl->amp, mdl->omega, t0, dt};
    for (double x : v)
        if (!std::isfinite(x)) return fail(LQ_ERR_NONFINITE, "non-finite model, t0 or dt");
    const int n = sv->n;
    if (n < 2) return fail(LQ_ERR_ARG, "the XYZ chain needs n >= 2");
    if (!(dt > 0) || n_steps < 0 || record_every < 1) return fail(LQ_ERR_ARG, "need dt > 0, n_steps >= 0, record_every >= 1");
    // observables: interaction part and magnetisation
    std::vector<lq_pauli_term> hint, mag;
    const double J[3] = {mdl->jx, mdl->jy, mdl->jz};
    for (int k = 0; k < 3; k++)
        for (int i = 0; i + 1 < n; i++) {
            const uint64_t m = (1ull << i) | (1ull << (i + 1));
            hint.push_back({-J[k], k == 2 ? 0ull : m, k == 0 ? 0ull : m});
        }
    for (int i = 0; i < n; i++) mag.push_back({1.0, 0ull, 1ull << i});
    auto h = [&](double t) { return mdl->amp * std::sin(mdl->omega * t); };
    int rec = 0;
    auto record = [&](double t) -> lq_status {
        if (!energy_out) return LQ_OK;
        double ei = 0.0, m = 0.0;
        LQ_TRY(lq_expval_pauli_sum(sv, hint.data(), hint.size(), &ei));
        LQ_TRY(lq_expval_pauli_sum(sv, mag.data(), mag.size(), &m));
        energy_out[rec++] = ei - h(t) * m;
        return LQ_OK;
    };
    LQ_TRY(record(t0));
    const int SMAX = 8;
    std::vector<lq_gate> gates;
    std::vector<double> theta;
    for (int j = 0; j < n_steps;) {
        const int to_rec = record_every - (j % record_every);
        const int S = std::min({SMAX, n_steps - j, to_rec});
        gates.clear();
        theta.assign((size_t)S * n, 0.0);
        for (int s2 = 0; s2 < S; s2++) {
            const int kinds[3] = {LQ_RXX, LQ_RYY, LQ_RZZ};
            for (int k = 0; k < 3; k++)
                for (int i = 0; i + 1 < n; i++) {
                    lq_gate g{};
                    g.kind = kinds[k];
                    g.q0 = i;
                    g.q1 = i + 1;
                    g.q2 = -1;
                    g.param_idx = -1;
                    g.angle = -2.0 * J[k] * dt;
                    gates.push_back(g);
                }
            const double tj = t0 + (double)(j + s2) * dt;
            for (int i = 0; i < n; i++) {
                lq_gate g{};
                g.kind = LQ_RZ;
                g.q0 = i;
                g.q1 = g.q2 = -1;
                g.param_idx = s2 * n + i;
                gates.push_back(g);
                theta[(size_t)s2 * n + i] = -2.0 * h(tj) * dt;
            }
        }
        LQ_TRY(apply_impl(sv, gates.data(), gates.size(), theta.data(), theta.size()));
        j += S;
        if (j % record_every == 0) LQ_TRY(record(t0 + (double)j * dt));
    }
    return LQ_OK;
}

// Plan export (JSON) for host-side inspection and the test-suite's plan
// emulator: the gates (and an optional Pauli sum, planned as the PSR driver
// does) with the current options.
lq_status lq_plan_export_json(int n_qubits, const lq_gate *gates, size_t n_gates, const lq_pauli_term *terms,
                              size_t n_terms, char *buf, size_t buf_len, size_t *needed) {
    if (n_qubits < 1 || n_qubits > 40) return fail(LQ_ERR_ARG, "n_qubits must be in [1, 40]");
    LQ_TRY(validate_gates(n_qubits, gates, n_gates, nullptr, 1 << 16, false, nullptr));
    LQ_TRY(validate_terms(n_qubits, terms, n_terms));
    int32_t qm[64];
    for (int q = 0; q < n_qubits; q++) qm[q] = n_qubits - 1 - q;
    std::vector<POp> ops;
    MatBuilder mb;
    Plan plan;
    lower_gates(n_qubits, gates, n_gates, qm, ops, mb);
    if (n_terms) lower_pauli(n_qubits, qm, terms, n_terms, ops, plan);
    plan_circuit(n_qubits, ops, export_options(), mb, plan);
    if (plan.has_oop) {   // the layout after the plan: qubit q ends at frame[qm[q]]
        for (int q = 0; q < n_qubits; q++) qm[q] = plan.frame[qm[q]];
    }
    std::string j = export_json(plan, mb, qm);
    if (needed) *needed = j.size() + 1;
    if (buf && buf_len) {
        size_t k = std::min(buf_len - 1, j.size());
        memcpy(buf, j.data(), k);
        buf[k] = 0;
    }
    return LQ_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- PSR driver (a8)
struct lq_psr {
    int n = 0;
    size_t n_params = 0;
    int rank = 0, world = 1;
    lq_comm *comm = nullptr;   // NCCL: the gradient and E are all-reduced inside lq_psr_run
    bool dead = false;         // poisoned by an asynchronous failure
    std::string why;
    DevBuf red;                // n_params + 1 doubles: this rank's share, then the sum
    cudaStream_t stream = nullptr;
    Plan plan;
    MatBuilder mb;
    DirectSet dset;
    std::vector<Shift> shifts;
    std::vector<PsrRule> pairs;
    int base_idx = -1;
    int B = 1;
    DevBuf blob_buf, states, mats, partials, E, ctab;
    DevPlan dp;
    const Shift *d_shifts = nullptr;
    const PsrRule *d_pairs = nullptr;
    const PTerm *d_terms = nullptr;
    uint64_t launches_per_run = 0;
    uint64_t blob_bytes = 0;
    // CUDA graph of one run (LQ_OPT_GRAPHS): captured on the second run with
    // the same device pointers, replayed while they stay the same
    cudaGraphExec_t gexec = nullptr;
    const void *g_ptr[3] = {nullptr, nullptr, nullptr};   // pointers of the last run
    uint64_t graph_launches = 0;                           // kernels in the graph
    uint64_t graph_replays = 0;
    bool gdisabled = false;                                // a capture failed: stream launches only
};

extern "C" {

lq_status lq_psr_create(int n_qubits, const lq_gate *ansatz, size_t n_gates, size_t n_params,
                        const lq_pauli_term *terms, size_t n_terms, lq_comm *comm, void *cuda_stream, lq_psr **out) {
    if (!out) return fail(LQ_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (n_qubits < 1 || n_qubits > 36) return fail(LQ_ERR_ARG, "n_qubits must be in [1, 36]");
    if (comm && comm->dead) return fail(LQ_ERR_STATE, "communicator aborted after an earlier failure: " + comm->why);
    const int shard_rank = comm ? comm->rank : 0, shard_world = comm ? comm->world : 1;
    std::vector<int> uses(n_params, 0);
    LQ_TRY(validate_gates(n_qubits, ansatz, n_gates, nullptr, n_params, false, &uses));
    LQ_TRY(validate_terms(n_qubits, terms, n_terms));
    LQ_TRY(have_device());
    lq_psr *P = new lq_psr();
    P->n = n_qubits;
    P->n_params = n_params;
    P->rank = shard_rank;
    P->world = shard_world;
    P->comm = comm;
    P->stream = (cudaStream_t)cuda_stream;
    int32_t qm[64];
    for (int q = 0; q < n_qubits; q++) qm[q] = n_qubits - 1 - q;
    std::vector<POp> ops;
    lower_gates(n_qubits, ansatz, n_gates, qm, ops, P->mb);
    // the Pauli groups ride on the circuit's own tile passes (read after the
    // last gate that touches their qubits)
    lower_pauli(n_qubits, qm, terms, n_terms, ops, P->plan);
    PlanOptions po = options();
    po.budget = (int)g_opt_budget.load();
    po.first_free = g_opt_first_free.load() != 0;
    // relabelling stores need the JIT tile programs (the interpreter stores in place)
    po.oop = g_opt_jit.load() != 0 ? (int)g_opt_relabel.load() : 0;
    plan_circuit(n_qubits, ops, po, P->mb, P->plan);
    P->plan.zero_first = true;   // lq_psr_run launches the first pass with PF_LOAD_ZERO
    P->dset.build(P->plan);
    // circuits of this shard: (p, +pi/2), (p, -pi/2) for owned p; base on shard 0.
    // Parameters used by no gate have E+ == E- identically: g_p = 0 (written by combine).
    std::vector<char> four(n_params, 0);   // parameters of controlled rotations (k_psr_combine)
    for (size_t i = 0; i < n_gates; i++)
        if (ansatz[i].param_idx >= 0 && ansatz[i].kind == LQ_CRY) four[(size_t)ansatz[i].param_idx] = 1;
    const double c1 = (std::sqrt(2.0) + 1.0) / (4.0 * std::sqrt(2.0)), c2 = (std::sqrt(2.0) - 1.0) / (4.0 * std::sqrt(2.0));
    for (size_t p = 0; p < n_params; p++) {
        if ((int)(p % shard_world) != shard_rank || uses[p] == 0) continue;
        PsrRule pr{};
        pr.p = (int)p;
        const double s[4] = {PI / 2, -PI / 2, 3 * PI / 2, -3 * PI / 2};
        const double w2[4] = {0.5, -0.5, 0.0, 0.0}, w4[4] = {c1, -c1, -c2, c2};
        pr.nc = four[p] ? 4 : 2;
        for (int k = 0; k < pr.nc; k++) {
            pr.c[k] = (int)P->shifts.size();
            pr.w[k] = four[p] ? w4[k] : w2[k];
            P->shifts.push_back({(int)p, 0, s[k]});
        }
        P->pairs.push_back(pr);
    }
    if (shard_rank == 0) {
        P->base_idx = (int)P->shifts.size();
        P->shifts.push_back({-1, 0, 0.0});
    }
    const int n_circ = (int)P->shifts.size();
    const uint64_t N = 1ull << n_qubits;
    // batch: >= 2^26 amplitudes per launch when possible (config 4: 4 circuits,
    // 3.022 s vs 3.043 s with 2), <= 4 GiB of states
    uint64_t B = std::max<uint64_t>(1, (1ull << 26) / N);
    B = std::min<uint64_t>(B, std::max<uint64_t>(1, (1ull << 28) / N));
    B = std::min<uint64_t>(B, std::max(1, n_circ));
    B = std::min<uint64_t>(B, 65535);
    if (const char *be = getenv("LQ_PSR_BATCH"))   // tuning experiments
        B = std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)atoi(be), std::max(1, n_circ)));
    P->B = (int)B;
    P->plan.ctab_circ = (int)B;   // constant op-table banks hold one launch's circuits
    P->plan.stream_tag = (uint64_t)(uintptr_t)P->stream;
    {
        lq_status js = prepare(P->plan, true);
        if (js != LQ_OK) {
            delete P;
            return js;
        }
    }
    cudaStream_t st = P->stream;
    Blob blob;
    size_t o_sub = blob.add(P->plan.subs), o_kop = blob.add(P->plan.kops), o_spec = blob.add(P->mb.specs),
           o_fac = blob.add(P->mb.factors), o_cst = blob.add(P->mb.cst), o_perm = blob.add(P->plan.perms),
           o_pt = blob.add(P->plan.perm_terms), o_sh = blob.add(P->shifts),
           o_pr = blob.add(P->pairs), o_t = blob.add(P->dset.terms), o_et = blob.add(P->plan.eterms),
           o_cd = blob.add(P->plan.ctab_desc);
    P->blob_bytes = blob.h.size();
    lq_status s = blob.upload(P->blob_buf, st);
    // relabelling plans ping-pong between two batches of states
    if (s == LQ_OK) s = P->states.reserve((size_t)B * N * sizeof(double2) * (P->plan.has_oop ? 2 : 1), st);
    if (s == LQ_OK) s = P->mats.reserve((size_t)B * std::max<uint32_t>(P->mb.mat_size, 1) * sizeof(double2), st);
    if (s == LQ_OK) s = P->partials.reserve((size_t)B * P->dset.stride() * sizeof(double), st);
    if (s == LQ_OK) s = P->E.reserve(sizeof(double) * std::max(n_circ, 1), st);
    if (s == LQ_OK) s = P->red.reserve(sizeof(double) * (n_params + 1), st);
    if (s == LQ_OK && P->plan.ctab_total) s = P->ctab.reserve((size_t)P->plan.ctab_total * sizeof(double2), st);
    if (s != LQ_OK) {
        std::string keep = g_err;
        lq_psr_free(P);
        g_err = keep;
        return s;
    }
    if (P->plan.ctab_total) {
        P->dp.ctab_desc = P->blob_buf.at<CtabDesc>(o_cd);
        P->dp.ctab_stage = P->ctab.at<double2>(0);
    }
    P->dp.subs = P->blob_buf.at<KSub>(o_sub);
    P->dp.kops = P->blob_buf.at<KOp>(o_kop);
    P->dp.specs = P->blob_buf.at<MSpec>(o_spec);
    P->dp.factors = P->blob_buf.at<MFactor>(o_fac);
    P->dp.cst = P->blob_buf.at<double2>(o_cst);
    P->dp.perms = P->blob_buf.at<KPerm>(o_perm);
    P->dp.pterms = P->blob_buf.at<KPermTerm>(o_pt);
    P->dp.eterms = P->blob_buf.at<ETerm>(o_et);
    P->d_shifts = P->blob_buf.at<Shift>(o_sh);
    P->d_pairs = P->blob_buf.at<PsrRule>(o_pr);
    P->d_terms = P->blob_buf.at<PTerm>(o_t);
    *out = P;
    return LQ_OK;
}

static lq_status psr_run_body(lq_psr *P, const double *theta_dev, double *grad_dev, double *energy_dev,
                              cudaStream_t st);
static lq_status psr_run_graph(lq_psr *P, const double *theta_dev, double *grad_dev, double *energy_dev);
static bool psr_graphs(const lq_psr *P);

lq_status lq_psr_run(lq_psr *P, const double *theta_dev, double *grad_dev, double *energy_dev) {
    if (!P) return fail(LQ_ERR_ARG, "invalid plan");
    if (P->dead) return fail(LQ_ERR_STATE, "gradient plan unusable after an earlier asynchronous failure: " + P->why);
    if (P->comm && P->comm->dead)
        return fail(LQ_ERR_STATE, "communicator aborted after an earlier failure: " + P->comm->why);
    if ((!theta_dev && P->n_params) || (!grad_dev && P->n_params)) return fail(LQ_ERR_ARG, "NULL device pointer");
    const lq_status s = psr_graphs(P) ? psr_run_graph(P, theta_dev, grad_dev, energy_dev)
                                      : psr_run_body(P, theta_dev, grad_dev, energy_dev, P->stream);
    if (s == LQ_ERR_CUDA || s == LQ_ERR_NCCL) {
        P->dead = true;
        P->why = g_err;
    }
    return s;
}

static lq_status psr_run_body(lq_psr *P, const double *theta_dev, double *grad_dev, double *energy_dev,
                              cudaStream_t st) {
    const uint64_t N = 1ull << P->n;
    const int n_circ = (int)P->shifts.size();
    uint64_t l0 = g_launches.load();
    double2 *states = P->states.at<double2>(0);
    double2 *mats = P->mats.at<double2>(0);
    double *part = P->partials.at<double>(0);
    double *E = P->E.at<double>(0);
    const uint32_t ms = std::max<uint32_t>(P->mb.mat_size, 1);
    for (int c0 = 0; c0 < n_circ; c0 += P->B) {
        const int nb = std::min(P->B, n_circ - c0);
        if (P->mb.mat_size) {
            k_build_mats<<<grid_for((uint64_t)P->mb.specs.size() * nb), 256, 0, st>>>(
                P->dp.specs, (int)P->mb.specs.size(), P->dp.factors, theta_dev, P->d_shifts + c0, P->dp.cst, mats,
                ms, nb);
            LQ_TRY(check_launch("k_build_mats"));
        }
        const uint32_t ss = P->dset.stride();
        // the state after the last pass is only read by the Pauli groups of
        // that pass: no store (unless a wide group still has to read it)
        double2 *fin = states;
        LQ_TRY(launch_passes(P->plan, P->dp, states, N, nb, mats, ms, st, true, part, ss, P->dset.ds.empty(), 0,
                             P->plan.has_oop ? states + (uint64_t)P->B * N : nullptr, &fin));
        LQ_TRY(finish_expv(P->plan, P->dset, P->d_terms, fin, N, nb, part, ss, E + c0, st));
    }
    if (!P->comm || !P->comm->c) {
        k_psr_combine<<<1, 256, 0, st>>>(E, P->d_pairs, (int)P->pairs.size(), P->base_idx, grad_dev,
                                         (int)P->n_params, energy_dev);
        LQ_TRY(check_launch("k_psr_combine"));
    } else {
        // Each component (and E, on rank 0) comes from exactly one rank and is
        // 0 elsewhere, so one sum over ranks returns the 1-GPU result exactly,
        // on every rank.
        double *red = P->red.at<double>(0);
        k_psr_combine<<<1, 256, 0, st>>>(E, P->d_pairs, (int)P->pairs.size(), P->base_idx, red, (int)P->n_params,
                                         red + P->n_params);
        LQ_TRY(check_launch("k_psr_combine"));
        LQ_TRY(comm_check(P->comm));
        {
            NvtxRange nr_("lq gradient all-reduce");
            NCCL_TRY(nccl().AllReduce(red, red, P->n_params + 1, ncclFloat64, ncclSum, P->comm->c, st));
        }
        if (P->n_params)
            CUDA_TRY(cudaMemcpyAsync(grad_dev, red, P->n_params * sizeof(double), cudaMemcpyDeviceToDevice, st));
        if (energy_dev)
            CUDA_TRY(cudaMemcpyAsync(energy_dev, red + P->n_params, sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    P->launches_per_run = g_launches.load() - l0;
    return LQ_OK;
}


}  // extern "C"

// ---------------------------------------------------------------- CUDA graphs
// Launch-bound runs (small states, many short kernels: configs 1-3, the VQE
// loop) are captured once as a CUDA graph and replayed: one cudaGraphLaunch
// instead of one host launch per kernel and per constant-bank copy, and no
// host gaps between the kernels.  Capture runs on a private stream in
// thread-local mode (nothing executes); the graph replays on the caller's
// stream, after everything queued there before it.
// Graphs pay off most where launches dominate (config 3: 47 -> 37 us per
// gradient), and still trim the launch gaps of a config-4 gradient (6748
// tile launches: 2.600 -> 2.578 s, same box).  Not with a communicator (its
// all-reduce and error polling stay on the host path) or per-launch timing.
static bool psr_graphs(const lq_psr *P) {
    return g_opt_graphs.load() && !P->comm && !g_opt_timing.load() && !P->gdisabled;
}
// runs short enough that the device VQE loop may replay iterations past the
// stop (at most 2^24 amplitudes per run; a config-4 run, 2.6 s, reads the
// status after every iteration instead)
static bool psr_small(const lq_psr *P) { return (uint64_t)P->shifts.size() << P->n <= (1ull << 24); }

static lq_status psr_run_graph(lq_psr *P, const double *theta_dev, double *grad_dev, double *energy_dev) {
    const void *ptr[3] = {theta_dev, grad_dev, energy_dev};
    const bool same = ptr[0] == P->g_ptr[0] && ptr[1] == P->g_ptr[1] && ptr[2] == P->g_ptr[2];
    if (!same || !P->gexec) {
        if (P->gexec) {
            cudaGraphExecDestroy(P->gexec);
            P->gexec = nullptr;
        }
        if (!same) {   // first run with these pointers: run directly, capture if they come again
            for (int i = 0; i < 3; i++) P->g_ptr[i] = ptr[i];
            return psr_run_body(P, theta_dev, grad_dev, energy_dev, P->stream);
        }
        if (capture_graph([&](cudaStream_t cs) { return psr_run_body(P, theta_dev, grad_dev, energy_dev, cs); },
                          &P->gexec, &P->graph_launches) != LQ_OK) {
            P->gdisabled = true;   // not a fault of the plan: stream launches from now on
            return psr_run_body(P, theta_dev, grad_dev, energy_dev, P->stream);
        }
    }
    CUDA_TRY(cudaGraphLaunch(P->gexec, P->stream));
    g_launches.fetch_add(P->graph_launches);
    P->graph_replays++;
    return LQ_OK;
}

extern "C" {

// VQE outer loop: Adam on parameter-shift
// gradients.  The plan is built once; every iteration is one lq_psr_run (E and
// g at theta^t), one k_adam_step, and one 8-byte read of E for the stopping
// rule.
lq_status lq_vqe_adam(int n_qubits, const lq_gate *ansatz, size_t n_gates, double *theta, size_t n_params,
                      const lq_pauli_term *terms, size_t n_terms, const lq_adam_cfg *cfg, void *cuda_stream,
                      double *energy_trace, int32_t *iters_out) {
    if (!cfg) return fail(LQ_ERR_ARG, "cfg is NULL");
    if (n_params && !theta) return fail(LQ_ERR_ARG, "theta is NULL");
    if (cfg->max_iter < 0 || cfg->reserved != 0) return fail(LQ_ERR_ARG, "max_iter must be >= 0, reserved 0");
    const double cf[5] = {cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->tol};
    for (double x : cf)
        if (!std::isfinite(x)) return fail(LQ_ERR_NONFINITE, "non-finite Adam setting");
    if (!(cfg->beta1 >= 0 && cfg->beta1 < 1 && cfg->beta2 >= 0 && cfg->beta2 < 1 && cfg->eps > 0 && cfg->tol >= 0))
        return fail(LQ_ERR_ARG, "Adam needs 0 <= beta < 1, eps > 0, tol >= 0");
    for (size_t p = 0; p < n_params; p++)
        if (!std::isfinite(theta[p])) return fail(LQ_ERR_NONFINITE, "non-finite theta[" + std::to_string(p) + "]");
    lq_psr *P = nullptr;
    LQ_TRY(lq_psr_create(n_qubits, ansatz, n_gates, n_params, terms, n_terms, nullptr, cuda_stream, &P));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    DevBuf buf;
    const size_t np = std::max<size_t>(n_params, 1);
    lq_status s = buf.reserve(sizeof(double) * (4 * np + 1), st);
    double *d_th = buf.at<double>(0), *d_g = d_th + np, *d_m = d_g + np, *d_v = d_m + np, *d_e = d_v + np;
    if (s == LQ_OK && n_params) {
        cudaError_t e = cudaMemcpyAsync(d_th, theta, sizeof(double) * n_params, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(d_m, 0, sizeof(double) * 2 * np, st);
        if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, std::string("vqe setup: ") + cudaGetErrorString(e));
    }
    int t = 0;
    bool graph_loop = s == LQ_OK && psr_graphs(P);
    if (graph_loop) {
        // Device-resident loop: one graph = one lq_psr_run + k_vqe_step (the
        // stopping rule and the Adam step on the device, bias corrections from
        // the same host pow() as below); replayed in growing chunks with one
        // 16-byte status read per chunk instead of one sync per iteration.
        // Iterations past the stop replay as no-ops for theta and the trace.
        const int T = cfg->max_iter + 1;
        DevBuf vb;
        std::vector<double> bc(2 * (size_t)T);
        for (int i = 0; i < T; i++) {
            bc[2 * i] = 1.0 - std::pow(cfg->beta1, (double)(i + 1));
            bc[2 * i + 1] = 1.0 - std::pow(cfg->beta2, (double)(i + 1));
        }
        s = vb.reserve(sizeof(double) * 3 * (size_t)T + sizeof(VqeCtl), st);
        double *d_bc = s == LQ_OK ? vb.at<double>(0) : nullptr, *d_tr = d_bc ? d_bc + 2 * T : nullptr;
        VqeCtl *d_ctl = d_tr ? reinterpret_cast<VqeCtl *>(d_tr + T) : nullptr;
        cudaGraphExec_t gx = nullptr;
        uint64_t gk = 0;
        if (s == LQ_OK) {
            cudaError_t e = cudaMemcpyAsync(d_bc, bc.data(), sizeof(double) * 2 * T, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) e = cudaMemsetAsync(d_ctl, 0, sizeof(VqeCtl), st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);   // bc is pageable host memory
            if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, std::string("vqe setup: ") + cudaGetErrorString(e));
        }
        if (s == LQ_OK &&
            capture_graph(
                [&](cudaStream_t cs) {
                    LQ_TRY(psr_run_body(P, d_th, d_g, d_e, cs));
                    k_vqe_step<<<1, 256, 0, cs>>>(d_th, d_m, d_v, d_g, (int)n_params, cfg->lr, cfg->beta1, cfg->beta2,
                                                  cfg->eps, cfg->tol, cfg->max_iter, d_bc, d_e, d_tr, d_ctl);
                    return check_launch("k_vqe_step");
                },
                &gx, &gk) != LQ_OK) {
            graph_loop = false;   // capture failed (not a fault): the host loop below
            P->gdisabled = true;
        }
        VqeCtl ctl{0, 0, 0.0};
        const int max_chunk = psr_small(P) ? 32 : 1;
        for (int done = 0, chunk = 1; graph_loop && s == LQ_OK && done < T && ctl.state == 0;
             chunk = std::min(chunk * 2, max_chunk)) {
            const int c = std::min(chunk, T - done);
            for (int i = 0; i < c && s == LQ_OK; i++) {
                const cudaError_t e = cudaGraphLaunch(gx, st);
                if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, std::string("vqe graph: ") + cudaGetErrorString(e));
                g_launches.fetch_add(gk);
            }
            done += c;
            if (s == LQ_OK) {
                cudaError_t e = cudaMemcpyAsync(&ctl, d_ctl, sizeof(VqeCtl), cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess) e = cudaStreamSynchronize(st);
                if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, std::string("vqe: ") + cudaGetErrorString(e));
            }
        }
        if (gx) cudaGraphExecDestroy(gx);
        if (graph_loop) t = ctl.t;
        if (graph_loop && s == LQ_OK && energy_trace) {
            // a non-finite E_t is reported, not recorded (as the host loop)
            const size_t cnt = (size_t)(ctl.state == 2 ? t : t + 1);
            cudaError_t e = cnt ? cudaMemcpyAsync(energy_trace, d_tr, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st)
                                : cudaSuccess;
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, std::string("vqe: ") + cudaGetErrorString(e));
        }
        if (graph_loop && s == LQ_OK && ctl.state == 2)
            s = fail(LQ_ERR_NONFINITE, "non-finite energy at iteration " + std::to_string(t));
        if (graph_loop && s == LQ_OK && ctl.state == 0)
            s = fail(LQ_ERR_STATE, "vqe loop ended without its stopping rule (internal)");
        vb.release(st);
    }
    if (!graph_loop) {
    double prev = 0.0;
    for (; s == LQ_OK; t++) {
        s = lq_psr_run(P, d_th, d_g, d_e);
        double E = 0.0;
        if (s == LQ_OK) {
            cudaError_t e = cudaMemcpyAsync(&E, d_e, sizeof(double), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, std::string("vqe: ") + cudaGetErrorString(e));
        }
        if (s != LQ_OK) break;
        if (!std::isfinite(E)) {
            s = fail(LQ_ERR_NONFINITE, "non-finite energy at iteration " + std::to_string(t));
            break;
        }
        if (energy_trace) energy_trace[t] = E;
        if ((t >= 1 && std::fabs(E - prev) < cfg->tol) || t == cfg->max_iter) break;
        prev = E;
        if (n_params) {
            const double bc1 = 1.0 - std::pow(cfg->beta1, (double)(t + 1)), bc2 = 1.0 - std::pow(cfg->beta2, (double)(t + 1));
            k_adam_step<<<grid_for(n_params), 256, 0, st>>>(d_th, d_m, d_v, d_g, (int)n_params, cfg->lr, cfg->beta1,
                                                             cfg->beta2, cfg->eps, bc1, bc2);
            s = check_launch("k_adam_step");
        }
    }
    }
    if (s == LQ_OK && n_params) {
        cudaError_t e = cudaMemcpyAsync(theta, d_th, sizeof(double) * n_params, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, std::string("vqe: ") + cudaGetErrorString(e));
    }
    if (iters_out) *iters_out = t;
    buf.release(st);
    lq_psr_free(P);
    return s;
}

lq_status lq_psr_stats(const lq_psr *P, uint64_t *n_circuits, uint64_t *n_launches, uint64_t *plan_bytes,
                       uint64_t *tile_passes) {
    if (!P) return fail(LQ_ERR_ARG, "invalid plan");
    if (n_circuits) *n_circuits = P->shifts.size();
    if (n_launches) *n_launches = P->launches_per_run;
    if (plan_bytes) *plan_bytes = P->blob_bytes;
    if (tile_passes) *tile_passes = P->plan.n_tile;
    return LQ_OK;
}

// Algorithmic HBM bytes of pass i of one circuit, as launch_passes runs it:
// the first tile pass synthesises |0...0> (write only), read-only passes and
// the final pass (when no wide Pauli group reads the state afterwards) skip
// the store, a pass under support tracking (PlanPass::support) reads only the
// indices inside its support and writes only the tiles it runs; every other
// pass reads and writes 16 B per amplitude.
static uint64_t psr_pass_bytes(const lq_psr *P, size_t i) {
    const uint64_t N = 1ull << P->n;
    const size_t np = P->plan.passes.size();
    const PlanPass &p = P->plan.passes[i];
    // launch_passes synthesises |0...0> in every tile pass until one has stored
    bool load = P->plan.passes[0].kind != PASS_TILE;
    for (size_t k = 0; k < i && !load; k++) load = !(P->plan.passes[k].kp.flags & PF_NO_STORE);
    bool store = true;
    if (p.kind == PASS_TILE) {
        if (p.kp.flags & PF_NO_STORE) store = false;
        if (i + 1 == np && P->dset.ds.empty()) store = false;
    }
    // support tracking (prepare()): loads of the indices inside the pass's
    // support only, stores of the tiles it runs
    const bool jit = p.kind == PASS_TILE && i < P->plan.jit.size() && P->plan.jit[i];
    const uint64_t rd = (jit && p.support != ~0ull) ? 1ull << __builtin_popcountll(p.support & (N - 1)) : N;
    const uint64_t wr = (jit && p.tiles_log2 >= 0) ? 1ull << (p.tiles_log2 + p.kp.K) : N;
    uint64_t b = 16 * ((load ? rd : 0) + (store ? wr : 0));
    if (p.kind == PASS_DIAG) b *= (p.op_end - p.op_begin + DIAG_MAX_OPS - 1) / DIAG_MAX_OPS;   // one k_diag per chunk
    return b;
}

lq_status lq_psr_traffic(const lq_psr *P, uint64_t *tile_bytes_per_circuit, uint64_t *direct_bytes_per_circuit) {
    if (!P) return fail(LQ_ERR_ARG, "invalid plan");
    const uint64_t N = 1ull << P->n;
    uint64_t tb = 0, other = 0;
    for (size_t i = 0; i < P->plan.passes.size(); i++)
        (P->plan.passes[i].kind == PASS_TILE ? tb : other) += psr_pass_bytes(P, i);
    other += 32 * N * P->dset.ds.size();   // direct Pauli groups read psi[j] and psi[j ^ x]
    if (tile_bytes_per_circuit) *tile_bytes_per_circuit = tb;
    if (direct_bytes_per_circuit) *direct_bytes_per_circuit = other;
    return LQ_OK;
}

lq_status lq_psr_pass_tiles(const lq_psr *P, uint64_t *tile_masks_out, size_t cap, size_t *n_passes) {
    if (!P) return fail(LQ_ERR_ARG, "invalid plan");
    const size_t np = P->plan.passes.size();
    if (n_passes) *n_passes = np;
    if (cap && !tile_masks_out) return fail(LQ_ERR_ARG, "output array is NULL");
    for (size_t i = 0; i < np && i < cap; i++) {
        const PlanPass &p = P->plan.passes[i];
        uint64_t m = 0;
        if (p.kind == PASS_TILE)
            for (int b = 0; b < p.kp.K; b++) m |= 1ull << p.kp.T[b];
        tile_masks_out[i] = m;
    }
    return LQ_OK;
}

lq_status lq_tile_sweep(void *dev_buf, size_t bytes, int n_bits, uint64_t tile_mask, int reps, void *cuda_stream,
                        double *ms_per_sweep) {
    if (!dev_buf || !ms_per_sweep || reps < 1) return fail(LQ_ERR_ARG, "NULL buffer / output or reps < 1");
    if (n_bits < 8 || n_bits > 40 || bytes < ((size_t)16 << n_bits)) return fail(LQ_ERR_DIM, "buffer smaller than 16 * 2^n_bits");
    const int K = __builtin_popcountll(tile_mask);
    if (tile_mask >> n_bits || K < 4 || K > 12) return fail(LQ_ERR_ARG, "tile mask must have 4..12 bits below n_bits");
    LQ_TRY(have_device());
    SweepSpec P;
    memset(&P, 0, sizeof(P));
    for (int b = 0; b < n_bits; b++) {
        if (tile_mask >> b & 1) P.tpos[P.K++] = (uint8_t)b;
        else P.fpos[P.nfree++] = (uint8_t)b;
    }
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const uint64_t n_tiles = 1ull << P.nfree;
    const int threads = std::max(128, (1 << K) / 16);
    int dev = 0, sms = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)sms * 16 * 128 / threads, n_tiles);
    double2 *s = (double2 *)dev_buf;
    cudaEvent_t a = nullptr, b = nullptr;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    k_tile_sweep<<<grid, threads, 0, st>>>(s, n_tiles, P);   // warm-up
    cudaEventRecord(a, st);
    for (int r = 0; r < reps; r++) k_tile_sweep<<<grid, threads, 0, st>>>(s, n_tiles, P);
    cudaEventRecord(b, st);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (e != cudaSuccess) return fail(LQ_ERR_CUDA, std::string("tile sweep: ") + cudaGetErrorString(e));
    LQ_TRY(check_launch("k_tile_sweep"));
    *ms_per_sweep = ms / reps;
    return LQ_OK;
}

lq_status lq_psr_pass_bytes(const lq_psr *P, uint64_t *bytes_out, int32_t *kind_out, uint64_t *support_amps_out,
                            uint32_t *ops_out, size_t cap, size_t *n_passes) {
    if (!P) return fail(LQ_ERR_ARG, "invalid plan");
    const size_t np = P->plan.passes.size();
    if (n_passes) *n_passes = np;
    if (cap && (!bytes_out || !kind_out)) return fail(LQ_ERR_ARG, "output arrays are NULL");
    const uint64_t N = 1ull << P->n;
    for (size_t i = 0; i < np && i < cap; i++) {
        const PlanPass &p = P->plan.passes[i];
        bytes_out[i] = psr_pass_bytes(P, i);
        kind_out[i] = (int32_t)p.kind;
        if (support_amps_out) {   // amplitudes the pass's gates act on (the rest are provably zero)
            const bool jit = p.kind == PASS_TILE && i < P->plan.jit.size() && P->plan.jit[i];
            support_amps_out[i] = (jit && p.tiles_log2 >= 0) ? 1ull << (p.tiles_log2 + p.kp.K) : N;
        }
        if (ops_out) ops_out[i] = (uint32_t)p.n_ops;
    }
    return LQ_OK;
}

lq_status lq_psr_free(lq_psr *P) {
    if (!P) return LQ_OK;
    if (P->gexec) cudaGraphExecDestroy(P->gexec);
    P->blob_buf.release(P->stream);
    P->states.release(P->stream);
    P->mats.release(P->stream);
    P->partials.release(P->stream);
    P->E.release(P->stream);
    P->ctab.release(P->stream);
    P->red.release(P->stream);
    delete P;
    return LQ_OK;
}

}  // extern "C"

namespace {
// One-shot gradients (lq_param_shift_grad) reuse their plan across calls with
// the same circuit, Hamiltonian, shard and options: planning, JIT lookup and
// device buffers are paid once, as a VQE loop over theta would want.
struct CachedPsr {
    std::string key;
    lq_psr *P = nullptr;
    DevBuf io;   // theta, grad, energy
    // pinned host mirror of io: the copies in and out are asynchronous
    // (pageable copies stage through the driver and stall the stream)
    double *hio = nullptr;
    ~CachedPsr() {
        if (hio) cudaFreeHost(hio);
    }
};
std::mutex g_psr_mu;
std::vector<CachedPsr *> g_psr_cache;   // most recent last
constexpr size_t PSR_CACHE_MAX = 2;

std::string psr_key(int n, const lq_gate *g, size_t ng, size_t np, const lq_pauli_term *t, size_t nt,
                    const lq_comm *comm, void *stream) {
    std::string k;
    auto put = [&](const void *p, size_t b) { k.append(static_cast<const char *>(p), b); };
    int64_t hdr[8] = {n, (int64_t)ng, (int64_t)np, (int64_t)nt, (int64_t)(intptr_t)comm,
                      comm ? comm->rank : 0, (int64_t)(intptr_t)stream, comm ? comm->world : 1};
    put(hdr, sizeof(hdr));
    int64_t opt[7] = {g_opt_fusion.load(), g_opt_K.load(), g_opt_coalesce.load(), g_opt_regbits.load(),
                      g_opt_jit.load(), g_opt_budget.load(), g_opt_first_free.load()};
    put(opt, sizeof(opt));
    for (size_t i = 0; i < ng; i++) {
        put(&g[i], offsetof(lq_gate, mat));
        if (g[i].kind == LQ_U1) put(g[i].mat, 8 * sizeof(double));
        if (g[i].kind == LQ_U2) put(g[i].mat, 32 * sizeof(double));
    }
    if (nt) put(t, nt * sizeof(lq_pauli_term));
    return k;
}
}  // namespace

extern "C" {

lq_status lq_psr_cache_clear(void) {
    std::lock_guard<std::mutex> lk(g_psr_mu);
    for (CachedPsr *c : g_psr_cache) {
        c->io.release(c->P->stream);
        lq_psr_free(c->P);
        delete c;
    }
    g_psr_cache.clear();
    g_plan_cache.clear();
    g_sched_cache.clear();
    return LQ_OK;
}

lq_status lq_param_shift_grad(int n_qubits, const lq_gate *ansatz, size_t n_gates, const double *theta,
                              size_t n_params, const lq_pauli_term *terms, size_t n_terms, lq_comm *comm,
                              void *cuda_stream, double *grad_out, double *energy_out) {
    if (comm && comm->dead) return fail(LQ_ERR_STATE, "communicator aborted after an earlier failure: " + comm->why);
    if (n_params && (!theta || !grad_out)) return fail(LQ_ERR_ARG, "theta/grad_out is NULL");
    for (size_t p = 0; p < n_params; p++)
        if (!std::isfinite(theta[p])) return fail(LQ_ERR_NONFINITE, "non-finite theta[" + std::to_string(p) + "]");
    if (n_gates && !ansatz) return fail(LQ_ERR_ARG, "gates is NULL");
    if (n_terms && !terms) return fail(LQ_ERR_ARG, "terms is NULL");
    for (size_t i = 0; i < n_gates; i++)   // the key reads user matrices: validate them first
        if ((ansatz[i].kind == LQ_U1 || ansatz[i].kind == LQ_U2) && !ansatz[i].mat)
            return fail(LQ_ERR_ARG, "gate " + std::to_string(i) + ": matrix is NULL");
    std::lock_guard<std::mutex> lk(g_psr_mu);
    const std::string key =
        psr_key(n_qubits, ansatz, n_gates, n_params, terms, n_terms, comm, cuda_stream);
    CachedPsr *C = nullptr;
    for (size_t i = 0; i < g_psr_cache.size(); i++)
        if (g_psr_cache[i]->key == key) {
            C = g_psr_cache[i];
            g_psr_cache.erase(g_psr_cache.begin() + i);
            break;
        }
    if (!C) {
        lq_psr *P = nullptr;
        LQ_TRY(lq_psr_create(n_qubits, ansatz, n_gates, n_params, terms, n_terms, comm, cuda_stream, &P));
        C = new CachedPsr();
        C->key = key;
        C->P = P;
        lq_status s = C->io.reserve(sizeof(double) * (2 * n_params + 2), P->stream);
        if (s != LQ_OK) {
            std::string keep = g_err;
            lq_psr_free(P);
            delete C;
            g_err = keep;
            return s;
        }
        if (g_psr_cache.size() >= PSR_CACHE_MAX) {   // evict the least recently used
            CachedPsr *old = g_psr_cache.front();
            g_psr_cache.erase(g_psr_cache.begin());
            old->io.release(old->P->stream);
            lq_psr_free(old->P);
            delete old;
        }
    }
    g_psr_cache.push_back(C);
    lq_psr *P = C->P;
    cudaStream_t st = P->stream;
    double *d_theta = C->io.at<double>(0), *d_grad = d_theta + n_params, *d_e = d_grad + n_params;
    lq_status s = LQ_OK;
    const size_t nio = 2 * n_params + 1;   // theta, grad, energy
    if (!C->hio && cudaMallocHost(&C->hio, sizeof(double) * nio) != cudaSuccess) {
        cudaGetLastError();
        C->hio = nullptr;   // no pinned memory: pageable copies below
    }
    double *h_theta = C->hio ? C->hio : const_cast<double *>(theta);
    double *h_grad = C->hio ? C->hio + n_params : grad_out, *h_e = C->hio ? C->hio + 2 * n_params : energy_out;
    if (n_params) {
        if (C->hio) memcpy(h_theta, theta, n_params * sizeof(double));   // the previous call has synchronised
        cudaError_t e = cudaMemcpyAsync(d_theta, h_theta, n_params * sizeof(double), cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, cudaGetErrorString(e));
    }
    if (s == LQ_OK) s = lq_psr_run(P, d_theta, d_grad, d_e);
    if (s == LQ_OK && n_params) {
        cudaError_t e = cudaMemcpyAsync(h_grad, d_grad, n_params * sizeof(double), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, cudaGetErrorString(e));
    }
    if (s == LQ_OK && energy_out) {
        cudaError_t e = cudaMemcpyAsync(h_e, d_e, sizeof(double), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = fail(LQ_ERR_CUDA, cudaGetErrorString(e));
    }
    if (s == LQ_OK) s = comm_sync(comm && comm->c ? comm : nullptr, st);
    if (s == LQ_OK && C->hio) {
        if (n_params) memcpy(grad_out, h_grad, n_params * sizeof(double));
        if (energy_out) *energy_out = *h_e;
    }
    if (s == LQ_ERR_CUDA || s == LQ_ERR_NCCL || P->dead) {   // never reuse a plan an asynchronous failure touched
        g_psr_cache.pop_back();
        cudaStreamSynchronize(st);
        C->io.release(st);
        lq_psr_free(P);
        delete C;
    }
    return s;
}

// Host-only: generate and NVRTC-compile (without loading) the JIT pass
// programs of `gates` (+ an optional Pauli sum, planned as the PSR driver
// does).  No device needed.
lq_status lq_jit_compile_check(int n_qubits, const lq_gate *gates, size_t n_gates, const lq_pauli_term *terms,
                               size_t n_terms, uint64_t *n_kernels) {
    if (n_qubits < 1 || n_qubits > 40) return fail(LQ_ERR_ARG, "n_qubits must be in [1, 40]");
    LQ_TRY(validate_gates(n_qubits, gates, n_gates, nullptr, 1 << 16, false, nullptr));
    LQ_TRY(validate_terms(n_qubits, terms, n_terms));
    int32_t qm[64];
    for (int q = 0; q < n_qubits; q++) qm[q] = n_qubits - 1 - q;
    std::vector<POp> ops;
    MatBuilder mb;
    Plan plan;
    lower_gates(n_qubits, gates, n_gates, qm, ops, mb);
    if (n_terms) lower_pauli(n_qubits, qm, terms, n_terms, ops, plan);
    plan_circuit(n_qubits, ops, export_options(), mb, plan);
    plan.zero_first = g_opt_export_psr.load() != 0;
    plan.ctab = getenv("LQ_JIT_NO_CTAB") == nullptr;   // as prepare() would
    plan.ctab_circ = 4;
    size_t nk = 0;
    std::string err;
    if (!jit_check(plan, &nk, err)) return fail(LQ_ERR_CUDA, err);
    if (n_kernels) *n_kernels = nk;
    return LQ_OK;
}

// Host-only: NVRTC-compile (without loading) the JIT pass programs of the
// QFT plan on n qubits (identity layout).  No device needed.
lq_status lq_qft_jit_compile_check(int n_qubits, int inverse, uint64_t *n_kernels) {
    if (n_qubits < 1 || n_qubits > 40) return fail(LQ_ERR_ARG, "n_qubits must be in [1, 40]");
    int32_t qm[64];
    for (int q = 0; q < n_qubits; q++) qm[q] = n_qubits - 1 - q;
    MatBuilder mb;
    Plan plan;
    if (!plan_qft(n_qubits, qm, inverse != 0, options(), plan, mb)) return fail(LQ_ERR_STATE, "qft planning failed");
    plan.ctab = getenv("LQ_JIT_NO_CTAB") == nullptr;
    size_t nk = 0;
    std::string err;
    if (!jit_check(plan, &nk, err)) return fail(LQ_ERR_CUDA, err);
    if (n_kernels) *n_kernels = nk;
    return LQ_OK;
}

lq_status lq_qft_plan_export_json(int n_qubits, int inverse, int reversed_layout, char *buf, size_t buf_len,
                                  size_t *needed) {
    if (n_qubits < 1 || n_qubits > 40) return fail(LQ_ERR_ARG, "n_qubits must be in [1, 40]");
    int32_t qm[64], qin[64];
    for (int q = 0; q < n_qubits; q++) qin[q] = qm[q] = reversed_layout ? q : n_qubits - 1 - q;
    MatBuilder mb;
    Plan plan;
    if (!plan_qft(n_qubits, qm, inverse != 0, options(), plan, mb)) return fail(LQ_ERR_STATE, "qft planning failed");
    std::string j = export_json(plan, mb, qm);
    std::ostringstream o;
    o << "{\"qmap_in\":[";
    for (int q = 0; q < n_qubits; q++) o << (q ? "," : "") << qin[q];
    o << "]," << j.substr(1);
    j = o.str();
    if (needed) *needed = j.size() + 1;
    if (buf && buf_len) {
        size_t k = std::min(buf_len - 1, j.size());
        memcpy(buf, j.data(), k);
        buf[k] = 0;
    }
    return LQ_OK;
}

// Host-only planning diagnostics (no device needed): plan `gates` on n
// qubits with the current options and report pass counts and a text dump.
lq_status lq_plan_describe(int n_qubits, const lq_gate *gates, size_t n_gates, uint64_t *n_passes,
                           uint64_t *n_tile, char *buf, size_t buf_len) {
    if (n_qubits < 1 || n_qubits > 40) return fail(LQ_ERR_ARG, "n_qubits must be in [1, 40]");
    std::vector<int> uses(1 << 16, 0);
    // parameters are not bound here; validate structure with a permissive theta count
    LQ_TRY(validate_gates(n_qubits, gates, n_gates, nullptr, 1 << 16, false, nullptr));
    int32_t qm[64];
    for (int q = 0; q < n_qubits; q++) qm[q] = n_qubits - 1 - q;
    std::vector<POp> ops;
    MatBuilder mb;
    lower_gates(n_qubits, gates, n_gates, qm, ops, mb);
    Plan plan;
    plan_circuit(n_qubits, ops, export_options(), mb, plan);
    if (n_passes) *n_passes = plan.passes.size();
    if (n_tile) *n_tile = plan.n_tile;
    if (buf && buf_len) {
        std::string d = "ops=" + std::to_string(ops.size()) + " " + describe(plan);
        size_t k = std::min(buf_len - 1, d.size());
        memcpy(buf, d.data(), k);
        buf[k] = 0;
    }
    return LQ_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- state-handle entry points
// Every call on a state handle: refuse a poisoned handle, run, and poison the
// handle if an asynchronous CUDA / NCCL failure surfaced (seal()).
extern "C" {

lq_status lq_sv_init_basis(lq_sv *sv, uint64_t k) {
    LQ_TRY(check_sv(sv));
    return seal(sv, sv_init_basis_body(sv, k));
}

lq_status lq_sv_init_random(lq_sv *sv, uint64_t seed) {
    LQ_TRY(check_sv(sv));
    return seal(sv, sv_init_random_body(sv, seed));
}

lq_status lq_sv_norm2(lq_sv *sv, double *out) {
    LQ_TRY(check_sv(sv));
    return seal(sv, sv_norm2_body(sv, out));
}

lq_status lq_sv_read(lq_sv *sv, uint64_t offset, uint64_t count, double *host_out) {
    LQ_TRY(check_sv(sv));
    return seal(sv, sv_read_body(sv, offset, count, host_out));
}

lq_status lq_sv_gather(lq_sv *sv, const uint64_t *idx, size_t count, double *host_out) {
    LQ_TRY(check_sv(sv));
    return seal(sv, sv_gather_body(sv, idx, count, host_out));
}

lq_status lq_sv_write(lq_sv *sv, uint64_t offset, uint64_t count, const double *host_in) {
    LQ_TRY(check_sv(sv));
    return seal(sv, sv_write_body(sv, offset, count, host_in));
}

lq_status lq_sv_canonicalize(lq_sv *sv) {
    LQ_TRY(check_sv(sv));
    return seal(sv, sv_canonicalize_body(sv));
}

lq_status lq_apply_circuit(lq_sv *sv, const lq_gate *gates, size_t n_gates, const double *theta, size_t n_theta) {
    LQ_TRY(check_sv(sv));
    return seal(sv, apply_circuit_body(sv, gates, n_gates, theta, n_theta));
}

lq_status lq_qft(lq_sv *sv, int inverse) {
    LQ_TRY(check_sv(sv));
    return seal(sv, qft_body(sv, inverse));
}

lq_status lq_expval_pauli_sum(lq_sv *sv, const lq_pauli_term *terms, size_t n_terms, double *out_energy) {
    LQ_TRY(check_sv(sv));
    return seal(sv, expval_pauli_sum_body(sv, terms, n_terms, out_energy));
}

lq_status lq_trotter_xyz(lq_sv *sv, const lq_xyz_model *mdl, double t0, double dt, int n_steps, int record_every, double *energy_out) {
    LQ_TRY(check_sv(sv));
    return seal(sv, trotter_xyz_body(sv, mdl, t0, dt, n_steps, record_every, energy_out));
}

}  // extern "C"
