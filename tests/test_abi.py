"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/lq.h declares, refuses device work without a device (no CPU
fallback), and its host planner/validation behave."""
import os
import re

import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lq():
    from paper_2512_23183_b200 import build
    build.build()
    from paper_2512_23183_b200 import lq as _lq
    return _lq


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lq_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(lq):
    import ctypes
    lib = ctypes.CDLL(lq.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the binding wraps every declared entry point under the same name
    assert set(syms) <= set(lq.EXPORTED)


def test_version_and_options(lq):
    assert lq.lq_version() == 1
    assert lq.lq_get_option(lq.LQ_OPT_FUSION) == 1
    with pytest.raises(lq.LQError):
        lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 20)
    with pytest.raises(lq.LQError):
        lq.lq_set_option(99, 1)


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_device_no_fallback(lq):
    assert lq.lq_device_count() == 0
    with pytest.raises(lq.LQError) as ei:
        lq.lq_sv_alloc(4)
    assert ei.value.status == lq.LQ_ERR_CUDA
    with pytest.raises(lq.LQError) as ei:
        lq.lq_param_shift_grad(1, [("RY", 0, -1, 0, 0.0)], [0.1], [(1.0, 0, 1)])
    assert ei.value.status == lq.LQ_ERR_CUDA


def test_planner_single_pass_for_small_states(lq):
    w = W.config1()
    n_pass, n_tile, desc = lq.lq_plan_describe(w.n, w.gates)
    assert (n_pass, n_tile) == (1, 1), desc
    w = W.config3()
    assert lq.lq_plan_describe(w.n, w.gates)[:2] == (1, 1)


def test_planner_fuses_config4_layers(lq):
    """configs[3]: 720 gates -> far fewer HBM passes (>= 25 gates/pass)."""
    w = W.config4()
    n_pass, n_tile, desc = lq.lq_plan_describe(w.n, w.gates)
    assert n_pass <= 28, desc
    assert len(w.gates) / n_pass >= 25


def test_planner_unfused_one_pass_per_gate(lq):
    w = W.config4()
    lq.lq_set_option(lq.LQ_OPT_FUSION, 0)
    try:
        n_pass, n_tile, _ = lq.lq_plan_describe(w.n, w.gates[:72])
    finally:
        lq.lq_set_option(lq.LQ_OPT_FUSION, 1)
    # non-diagonal 1q gates are never fused (scaled rotations are cheaper
    # apart): 24 RY + 24 RZ + 24 CNOT passes
    assert (n_pass, n_tile) == (72, 0)


def test_planner_respects_tile_size(lq):
    w = W.config5(28, 1, 400)
    for K in (6, 9, 12):
        lq.lq_set_option(lq.LQ_OPT_TILE_BITS, K)
        try:
            _, _, desc = lq.lq_plan_describe(w.n, w.gates)
        finally:
            lq.lq_set_option(lq.LQ_OPT_TILE_BITS, 0)
        for m in re.finditer(r"T=\{([0-9,]+)\}", desc):
            bits = [int(b) for b in m.group(1).split(",")]
            assert len(bits) == K and len(set(bits)) == K and bits == sorted(bits)
            assert bits[:3] == [0, 1, 2]          # coalescing run
            assert max(bits) < w.n


def test_planner_validation_errors(lq):
    cases = [
        ([("H", 5, -1, -1, 0.0)], lq.LQ_ERR_ARG),
        ([("CNOT", 1, 1, -1, 0.0)], lq.LQ_ERR_ARG),
        ([("X", 0, -1, -1, 1.0)], lq.LQ_ERR_ARG),
        ([("RX", 0, -1, -1, float("inf"))], lq.LQ_ERR_NONFINITE),
        ([("H", 0, 1, -1, 0.0)], lq.LQ_ERR_ARG),
        ([("U1", 0, -1, -1, 0.0, [[float("nan"), 0], [0, 1]])], lq.LQ_ERR_NONFINITE),
    ]
    for gates, status in cases:
        with pytest.raises(lq.LQError) as ei:
            lq.lq_plan_describe(5, gates)
        assert ei.value.status == status, gates


def test_jit_programs_compile_without_device(lq):
    """The JIT pass programs (tile.cuh + the generated op programs) compile
    for sm_100a through NVRTC on a host without a GPU: the QFT at n = 30 both
    ways (three 12-bit passes) and the
    config-1 circuit + QFT plan at n = 10."""
    assert lq.lq_qft_jit_compile_check(30, False) == 3
    assert lq.lq_qft_jit_compile_check(30, True) >= 3
    w = W.config1()
    assert lq.lq_jit_compile_check(w.n, w.gates) >= 1
