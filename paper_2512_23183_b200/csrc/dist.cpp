// dist.cpp -- see dist.h.
#include "dist.h"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <sstream>

namespace lq {

namespace {

constexpr int COALESCE_BITS = 3;   // 8 amplitudes = one 128-byte run

// Logical qubits a gate acts on non-diagonally (controls and diagonal
// factors are rank constants when global).
int nondiag_qubits(const lq_gate &G, int *q) {
    switch (G.kind) {
    case LQ_Z: case LQ_S: case LQ_SDG: case LQ_T: case LQ_TDG: case LQ_RZ:
    case LQ_CZ: case LQ_CP: case LQ_RZZ: case LQ_SWAP:
        return 0;
    case LQ_CNOT: case LQ_CRY: q[0] = G.q1; return 1;
    case LQK_QFT_STAGE: q[0] = G.q0; return 1;
    case LQ_CCX: q[0] = G.q2; return 1;
    case LQ_U2: case LQ_RXX: case LQ_RYY: q[0] = G.q0; q[1] = G.q1; return 2;
    default: q[0] = G.q0; return 1;   // H X Y RX RY U1
    }
}

int all_qubits(const lq_gate &G, int *q) {
    int k = 0;
    if (G.q0 >= 0) q[k++] = G.q0;
    if (G.q1 >= 0) q[k++] = G.q1;
    if (G.q2 >= 0) q[k++] = G.q2;
    return k;
}

}  // namespace

void push_swap(Schedule &sc, int k, const int *g, const int *l, uint32_t xmask, int32_t *qm, int *at) {
    DStep sw;
    sw.kind = 1;
    sw.k = k;
    sw.xmask = xmask;
    int idx[MAX_SWAP_K];
    for (int j = 0; j < k; j++) idx[j] = j;
    std::sort(idx, idx + k, [&](int a, int b) { return l[a] < l[b]; });
    for (int j = 0; j < k; j++) {
        sw.g[j] = g[idx[j]];
        sw.l[j] = l[idx[j]];
        const int qg = at[sw.g[j]], ql = at[sw.l[j]];
        if (qg >= 0) qm[qg] = sw.l[j];
        if (ql >= 0) qm[ql] = sw.g[j];
        std::swap(at[sw.g[j]], at[sw.l[j]]);
    }
    sc.steps.push_back(std::move(sw));
    sc.n_swaps++;
    sc.n_swapped_qubits += (size_t)k;
    sc.shard_fraction_sent += 1.0 - std::ldexp(1.0, -k);
}

bool schedule_gates(Schedule &sc, const lq_gate *gates, size_t ng, int32_t *qmap, uint32_t &xmask) {
    const int n = sc.n, nl = sc.nl;
    // future non-diagonal uses of each logical qubit (Belady victim choice)
    std::vector<std::vector<size_t>> uses(n);
    for (size_t i = 0; i < ng; i++) {
        int q[3];
        int k = nondiag_qubits(gates[i], q);
        for (int j = 0; j < k; j++) uses[q[j]].push_back(i);
    }
    std::vector<size_t> up(n, 0);
    auto next_use = [&](int q, size_t after) {
        while (up[q] < uses[q].size() && uses[q][up[q]] <= after) up[q]++;
        return up[q] < uses[q].size() ? uses[q][up[q]] : (size_t)SIZE_MAX;
    };
    std::vector<int32_t> qm(qmap, qmap + n);        // simulated layout
    std::vector<int32_t> run_qm(qm);                // layout at the start of the current run
    std::vector<int> at(64, -1);                    // physical bit -> logical qubit
    auto rebuild_at = [&]() {
        std::fill(at.begin(), at.end(), -1);
        for (int q = 0; q < n; q++) at[qm[q]] = q;
    };
    rebuild_at();
    size_t run_begin = 0;
    // lower gates [run_begin, end) with the run's starting layout into a LOCAL step
    auto flush = [&](size_t end, const POp *extra) {
        if (end > run_begin || extra) {
            DStep st;
            st.kind = 0;
            st.xmask = xmask;
            std::vector<int32_t> q2(run_qm);
            q2.resize(64, 0);
            if (end > run_begin) lower_gates(n, gates + run_begin, end - run_begin, q2.data(), st.ops, sc.mb);
            if (extra) st.ops.push_back(*extra);
            sc.steps.push_back(std::move(st));
        }
    };
    for (size_t i = 0; i < ng; i++) {
        const lq_gate &G = gates[i];
        if (G.kind == LQ_SWAP) {   // relabel inside the run (lower_gates replays it)
            std::swap(qm[G.q0], qm[G.q1]);
            rebuild_at();
            continue;
        }
        int q[3];
        int k = nondiag_qubits(G, q);
        std::vector<int> glob;
        for (int j = 0; j < k; j++)
            if (qm[q[j]] >= nl) glob.push_back(q[j]);
        if (glob.empty()) continue;
        if (G.kind == LQ_X || G.kind == LQ_Y) {
            // rank relabel: Y = X * diag(i, -i) -- the phase is a rank constant
            const int gb = qm[G.q0];
            POp d;
            bool have_d = false;
            if (G.kind == LQ_Y) {
                d.type = K_D1;
                d.t0 = gb;
                d.spec = sc.mb.add_spec(MF_DIAG2, {MFactor{FK_YDIAG, -1, 0.0, -1, 0}});
                have_d = true;
            }
            flush(i, have_d ? &d : nullptr);
            xmask ^= 1u << (gb - nl);
            sc.n_relabels++;
            run_begin = i + 1;
            run_qm = qm;
            continue;
        }
        flush(i, nullptr);
        uint64_t busy = 0;   // physical bits this gate touches
        {
            int a[3];
            int na = all_qubits(G, a);
            for (int j = 0; j < na; j++) busy |= 1ull << qm[a[j]];
        }
        // victims: free local bits, furthest next use first (ties: high
        // bits); the lowest COALESCE_BITS come last: an exchange over them
        // would pack and unpack every part with a stride of 2^k amplitudes
        // (partial 32-byte sectors), one over higher bits moves whole runs
        std::vector<std::pair<size_t, int>> vict;
        for (int l = nl - 1; l >= 0; l--) {
            if (busy >> l & 1) continue;
            vict.push_back({at[l] >= 0 ? next_use(at[l], i) : (size_t)SIZE_MAX, l});
        }
        std::stable_sort(vict.begin(), vict.end(), [](const std::pair<size_t, int> &x, const std::pair<size_t, int> &y) {
            const bool lx = x.second < COALESCE_BITS, ly = y.second < COALESCE_BITS;
            if (lx != ly) return ly;
            return x.first > y.first;
        });
        if (G.kind == LQK_QFT_STAGE && sc.qft_pass_stages > 0) {
            // pass-aligned victims: qubits never needed again first, then,
            // among those not needed in the next P stages, the ones needed
            // soonest (the rest in Belady order)
            const size_t horizon = i + (size_t)sc.qft_pass_stages;
            std::vector<std::pair<size_t, int>> late, rest;
            for (auto &v : vict) (v.first >= horizon && v.second >= COALESCE_BITS ? late : rest).push_back(v);
            std::stable_sort(late.begin(), late.end(), [](const std::pair<size_t, int> &x, const std::pair<size_t, int> &y) {
                const bool nx = x.first == (size_t)SIZE_MAX, ny = y.first == (size_t)SIZE_MAX;
                if (nx != ny) return nx;
                return x.first < y.first;
            });
            late.insert(late.end(), rest.begin(), rest.end());
            vict.swap(late);
        }
        if (vict.size() < glob.size()) return false;
        std::vector<int> want(glob);
        // other global qubits needed before the local qubit they would displace
        std::vector<std::pair<size_t, int>> cand;
        for (int g = nl; g < n; g++) {
            const int q2 = at[g];
            if (q2 < 0 || std::find(glob.begin(), glob.end(), q2) != glob.end()) continue;
            const size_t u = next_use(q2, i);
            if (u != (size_t)SIZE_MAX) cand.push_back({u, q2});
        }
        std::sort(cand.begin(), cand.end());
        const int kmax = std::max(1, std::min(sc.max_k, MAX_SWAP_K));
        for (size_t j = 0; j < cand.size(); j++) {
            const size_t v = want.size();
            if ((int)v >= kmax || v >= vict.size() || !(cand[j].first < vict[v].first)) break;
            want.push_back(cand[j].second);
        }
        int gb[MAX_SWAP_K], lb[MAX_SWAP_K];
        for (size_t j = 0; j < want.size(); j += kmax) {   // (a gate has at most 2 global non-diagonal qubits)
            const int k = (int)std::min<size_t>(kmax, want.size() - j);
            for (int t = 0; t < k; t++) {
                gb[t] = qm[want[j + t]];
                lb[t] = vict[j + t].second;
            }
            push_swap(sc, k, gb, lb, xmask, qm.data(), at.data());
        }
        run_begin = i;
        run_qm = qm;
    }
    flush(ng, nullptr);
    for (int j = 0; j < n; j++) qmap[j] = qm[j];
    return true;
}

std::vector<lq_gate> qft_gates(int n, bool inverse) {
    std::vector<lq_gate> g;
    auto mk = [](int kind, int a, int b, double ang) {
        lq_gate x;
        memset(&x, 0, sizeof(x));
        x.kind = kind;
        x.q0 = a;
        x.q1 = b;
        x.q2 = -1;
        x.param_idx = -1;
        x.angle = ang;
        x.mat = nullptr;
        return x;
    };
    // Alg. 3: stage i = H(i) then CP(pi / 2^(k-i)), k > i -- one op each
    for (int i = 0; i < n; i++) g.push_back(mk(LQK_QFT_STAGE, i, -1, 1.0));
    for (int i = 0; i < n / 2; i++) g.push_back(mk(LQ_SWAP, i, n - 1 - i, 0.0));
    if (inverse) {
        std::reverse(g.begin(), g.end());
        for (auto &x : g)
            if (x.kind == LQK_QFT_STAGE) x.angle = -1.0;
    }
    return g;
}

bool schedule_expval(Schedule &sc, const lq_pauli_term *terms, size_t nt, int32_t *qmap, uint32_t &xmask) {
    const int n = sc.n, nl = sc.nl;
    std::vector<int> at(64, -1);
    for (int q = 0; q < n; q++) at[qmap[q]] = q;
    auto local_x = [&](uint64_t x) {   // all X/Y qubits of a term on local bits?
        for (int q = 0; q < n; q++)
            if ((x >> q & 1) && qmap[q] >= nl) return false;
        return true;
    };
    auto emit = [&](const std::vector<lq_pauli_term> &ts) {
        DStep st;
        st.kind = 0;
        st.xmask = xmask;
        st.expv = true;
        lower_pauli(n, qmap, ts.data(), ts.size(), st.ops, st.plan);
        sc.steps.push_back(std::move(st));
    };
    // terms whose pairs (j, j ^ x) already share a shard: one step
    std::vector<lq_pauli_term> now;
    std::vector<uint64_t> xs;   // remaining x masks (one step each)
    for (size_t t = 0; t < nt; t++) {
        if (local_x(terms[t].x_mask)) now.push_back(terms[t]);
        else if (std::find(xs.begin(), xs.end(), terms[t].x_mask) == xs.end()) xs.push_back(terms[t].x_mask);
    }
    if (!now.empty()) emit(now);
    for (uint64_t x : xs) {   // swap this group's global X/Y qubits in (one exchange), then evaluate it
        if (__builtin_popcountll(x) > nl) return false;
        std::vector<int> gs, ls;
        for (int g = nl; g < n; g++) {
            const int qg = at[g];
            if (qg >= 0 && (x >> qg & 1)) gs.push_back(g);
        }
        for (int l = nl - 1; l >= 0 && ls.size() < gs.size(); l--)   // high bits first (COALESCE_BITS last)
            if (at[l] < 0 || !(x >> at[l] & 1)) ls.push_back(l);
        if (ls.size() < gs.size()) return false;
        const size_t kmax = (size_t)std::max(1, std::min(sc.max_k, MAX_SWAP_K));
        for (size_t j = 0; j < gs.size(); j += kmax) {
            const int k = (int)std::min(kmax, gs.size() - j);
            push_swap(sc, k, gs.data() + j, ls.data() + j, xmask, qmap, at.data());
        }
        std::vector<lq_pauli_term> grp;
        for (size_t t = 0; t < nt; t++)
            if (terms[t].x_mask == x) grp.push_back(terms[t]);
        emit(grp);
    }
    if (now.empty() && xs.empty()) emit(now);   // empty sum: E = 0
    return true;
}

void plan_steps(Schedule &sc, const PlanOptions &opt) {
    PlanOptions o = opt;
    o.n_local = sc.nl;
    for (auto &st : sc.steps)
        if (st.kind == 0) plan_circuit(sc.n, st.ops, o, sc.mb, st.plan);
}

std::string schedule_json(const Schedule &sc, const int32_t *qmap, uint32_t xmask) {
    std::ostringstream o;
    o << "{\"n\":" << sc.n << ",\"m\":" << sc.m << ",\"nl\":" << sc.nl << ",\"n_swaps\":" << sc.n_swaps
      << ",\"n_relabels\":" << sc.n_relabels << ",\"n_swapped_qubits\":" << sc.n_swapped_qubits
      << ",\"shard_fraction_sent\":" << sc.shard_fraction_sent << ",\"xmask\":" << xmask << ",\"qmap\":[";
    for (int q = 0; q < sc.n; q++) o << (q ? "," : "") << qmap[q];
    o << "],\"steps\":[";
    for (size_t i = 0; i < sc.steps.size(); i++) {
        const DStep &st = sc.steps[i];
        if (i) o << ",";
        if (st.kind == 1) {
            o << "{\"kind\":\"swap\",\"g\":[";
            for (int j = 0; j < st.k; j++) o << (j ? "," : "") << st.g[j];
            o << "],\"l\":[";
            for (int j = 0; j < st.k; j++) o << (j ? "," : "") << st.l[j];
            o << "],\"xmask\":" << st.xmask << "}";
        } else {
            int32_t dummy[64];
            for (int q = 0; q < 64; q++) dummy[q] = 0;
            o << "{\"kind\":\"local\",\"xmask\":" << st.xmask << ",\"expv\":" << (st.expv ? "true" : "false")
              << ",\"plan\":" << export_json(st.plan, sc.mb, dummy) << "}";
        }
    }
    o << "]}";
    return o.str();
}

}  // namespace lq
