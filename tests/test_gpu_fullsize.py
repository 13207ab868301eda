"""Full-size GPU parity of the configured workloads (SURVEY.md §8(c) c.4,
§8(d)); the expected values are the oracle's (tests/golden/*.json, written by
tools/make_golden.py, which calls only oracle/), closed forms, or the
workload's own initial state (round trips).

Tolerances (reading A16): amplitudes max-abs <= 1e-10; expectation
|E - E_o| <= 1e-10 max(|E_o|, 1); gradient |g_i - g_o,i| <= 1e-10
max(|g_o,i|, max_k |g_o,k|) over the oracle's components.
"""
import json
import math
import os

import numpy as np
import pytest

import workloads as W
from closed_forms import circuit_inverse
from twin_samples import TWIN_NS, twin_indices, twin_weights

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
AMP_TOL = 1e-10


@pytest.fixture(scope="module")
def lq():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_23183_b200 import lq as _lq
    return _lq


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _free_cache():
    import torch
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- config 4 at its configured size

def test_config4_full_size_vs_oracle(lq):
    """configs[3] in full (n = 24, 480 params, 961 circuits) through the
    call bench.py times (lq_param_shift_grad): E(theta) and the 8 seeded
    gradient components of W.config4().meta['oracle_params'] against the
    oracle's values (tests/golden/cfg4_oracle.json: 17 oracle circuits of 720
    gates on 2^24 amplitudes)."""
    w = W.config4()
    gd = _gold("cfg4_oracle.json")
    assert gd["workload"] == w.name and gd["params"] == list(w.meta["oracle_params"])
    g, e = lq.lq_param_shift_grad(w.n, w.gates, w.theta, w.terms)
    assert np.all(np.isfinite(g))
    eo = gd["energy"]
    assert abs(e - eo) <= 1e-10 * max(abs(eo), 1.0), (e, eo)
    go = np.array(gd["grad"])
    scale = float(np.abs(go).max())
    for p, v in zip(gd["params"], go):
        assert abs(g[p] - v) <= 1e-10 * max(abs(v), scale), (p, g[p], v)


# ---------------------------------------------------------------- config 5: reduced twins vs the oracle

def _check_twin(gd, got_idx, read_all):
    want = np.array(gd["re"]) + 1j * np.array(gd["im"])
    assert np.abs(got_idx - want).max() <= AMP_TOL
    full = read_all()
    assert abs(float(np.sum(np.abs(full) ** 2)) - gd["norm2"]) <= 1e-12
    for wr, pr, pi in zip(twin_weights(gd["n"]), gd["proj_re"], gd["proj_im"]):
        p = complex(np.sum(wr * full))
        assert abs(p - complex(pr, pi)) <= AMP_TOL, (p, pr, pi)


@pytest.mark.parametrize("n", TWIN_NS)
@pytest.mark.parametrize("m", [1, 2, 3])
@pytest.mark.parametrize("sharded", [False, True])
def test_config5_twin_vs_oracle(lq, n, m, sharded):
    """SURVEY c.4 (iv): the config-5 generator with the configured m at
    the reduced sizes n = 24 and 26 (init_random, 1000 gates with 30 % on the
    m global qubits, QFT), unsharded and on G = 2^m shards (group mode: the
    same schedule, exchanges and local plans as the NCCL path), against the
    oracle's amplitudes at 4096 seeded indices, its norm, and three +-1
    projections over every amplitude (tests/golden/cfg5_twin_n*_m*.json)."""
    gd = _gold(f"cfg5_twin_n{n}_m{m}.json")
    w = W.config5(n=n, m=m)
    assert gd["seed"] == w.seed and gd["n_gates"] == len(w.gates) and gd["n"] == n
    sv = lq.ShardedState(n, group_world=1 << m) if sharded else lq.StateVector(n)
    sv.init_random(w.seed).apply(w.gates).qft()
    idx = twin_indices(n, m)
    assert list(idx) == gd["idx"]
    _check_twin(gd, sv.gather(idx.astype(np.uint64)), sv.read)
    sv.free()


# ---------------------------------------------------------------- config 5 at full size

def _roundtrip(lq, sv, w, n, n_samples, rng):
    """init_random -> circuit -> QFT -> QFT^-1 -> circuit^-1 must return
    init_random(seed) (c.4 (ii)); the norm stays 1 (c.4 (iii)).  The initial
    state itself is checked against the oracle's per-index formula: on the
    samples, state / a_i(unnormalised) is one real constant 1/sqrt(S)."""
    import oracle
    idx = np.unique(rng.integers(0, 1 << n, size=n_samples, dtype=np.uint64))
    sv.init_random(w.seed)
    a0 = sv.gather(idx)
    raw = oracle.random_gaussian_at(w.seed, idx)
    ratio = a0 / raw
    c = float(np.median(ratio.real))
    assert np.abs(ratio - c).max() <= 1e-12 * c
    # S = sum of 2^n terms |a_i|^2 = -2 ln u0 with mean 2: S ~ 2^(n+1), relative spread ~2^-(n/2)
    assert abs(c * c * (1 << (n + 1)) - 1.0) <= 1e-3
    assert abs(sv.norm2() - 1.0) <= 1e-12
    sv.apply(w.gates).qft()
    assert abs(sv.norm2() - 1.0) <= 1e-11
    mid = sv.gather(idx[:1024])
    assert np.all(np.isfinite(mid)) and np.abs(mid - a0[:1024]).max() > 1e-8   # the state did move
    sv.qft(inverse=True).apply(circuit_inverse(w.gates))
    back = sv.gather(idx)
    assert np.abs(back - a0).max() <= AMP_TOL
    assert abs(sv.norm2() - 1.0) <= 1e-11


def test_config5_n33_one_gpu_roundtrip(lq):
    """The weak-scaling baseline of config 5 at its configured per-GPU size:
    n = 33 (2^33 amplitudes, 128 GiB) on one GPU, the config-5 generator with
    m = 1, then the QFT; the round trip back to init_random(seed) on 2^20
    sampled indices, the norm, and init_random against the oracle's formula."""
    _free_cache()
    n = 33
    w = W.config5(n=n, m=1)
    sv = lq.StateVector(n)
    try:
        _roundtrip(lq, sv, w, n, 1 << 20, np.random.default_rng(533))
    finally:
        sv.free()
        del sv
        _free_cache()


@pytest.mark.parametrize("G", [2, 4])
def test_config5_n32_group_roundtrip(lq, G):
    """c.4 (ii)/(iii) on the sharded path at full scale: n = 32 (64 GiB) on
    G = 2 and 4 shards with the configured m = log2 G (global-qubit swaps,
    rank relabels, the sharded QFT), round trip on 2^20 sampled indices."""
    _free_cache()
    n = 32
    m = G.bit_length() - 1
    w = W.config5(n=n, m=m)
    sv = lq.ShardedState(n, group_world=G)
    try:
        _roundtrip(lq, sv, w, n, 1 << 20, np.random.default_rng(532 + G))
    finally:
        sv.free()
        del sv
        _free_cache()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_config5_n30_sharded_equals_unsharded(lq, G):
    """c.4 (v): the config-5 generator (m = log2 G) + QFT at n = 30 on G
    shards equals the unsharded run within 1e-14 on 2^22 sampled indices
    (same gates, different rounding order only where passes split)."""
    _free_cache()
    n = 30
    m = G.bit_length() - 1
    w = W.config5(n=n, m=m)
    rng = np.random.default_rng(530 + G)
    idx = np.unique(rng.integers(0, 1 << n, size=1 << 22, dtype=np.uint64))
    a = lq.StateVector(n)
    a.init_random(w.seed).apply(w.gates).qft()
    ga = a.gather(idx)
    a.free()
    del a
    _free_cache()
    b = lq.ShardedState(n, group_world=G)
    b.init_random(w.seed).apply(w.gates).qft()
    gb = b.gather(idx)
    assert abs(b.norm2() - 1.0) <= 1e-11
    b.free()
    del b
    _free_cache()
    assert np.abs(ga - gb).max() <= 1e-14
