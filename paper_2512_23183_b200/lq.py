"""Thin ctypes binding of liblq.so (include/lq.h), same names as the C ABI.

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of liblq.so.  There is no CPU fallback -- importing this module
fails loudly if liblq.so is missing, and every call that needs a GPU raises
LQError(LQ_ERR_CUDA) without one.

PyTorch is used for device memory (``StateVector`` wraps a torch complex128
tensor through ``lq_sv_wrap``) and for CUDA streams.
"""
from __future__ import annotations

import ctypes
import struct
import math
import os
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblq.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

# ---- enums (include/lq.h) -------------------------------------------------
LQ_OK, LQ_ERR_ARG, LQ_ERR_OOM, LQ_ERR_CUDA, LQ_ERR_NCCL, LQ_ERR_DIM, LQ_ERR_NONFINITE, LQ_ERR_STATE = \
    0, -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "LQ_OK", -1: "LQ_ERR_ARG", -2: "LQ_ERR_OOM", -3: "LQ_ERR_CUDA", -4: "LQ_ERR_NCCL",
                -5: "LQ_ERR_DIM", -6: "LQ_ERR_NONFINITE", -7: "LQ_ERR_STATE"}
KIND_NAMES = ["H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY", "RZ", "CNOT", "CZ", "CP",
              "SWAP", "U1", "U2", "CRY", "CCX", "RXX", "RYY", "RZZ"]
KINDS = {k: i for i, k in enumerate(KIND_NAMES)}
(LQ_OPT_FUSION, LQ_OPT_TILE_BITS, LQ_OPT_COALESCE_BITS, LQ_OPT_REG_BITS, LQ_OPT_KERNEL_TIMING, LQ_OPT_JIT,
 LQ_OPT_PASS_BUDGET, LQ_OPT_FIRST_PASS_FREE, LQ_OPT_POISON_ALLOC, LQ_OPT_COMM_TIMEOUT_MS,
 LQ_OPT_SWAP_QUBITS, LQ_OPT_STATE_PASS_BUDGET, LQ_OPT_GROUP_STAGED,
 LQ_OPT_RELABEL_STORES, LQ_OPT_EXPORT_PSR, LQ_OPT_GRAPHS) = range(16)
KC_TILE, KC_PAIR, KC_DIAG, KC_PAULI, KC_OTHER, KC_SWAP = 0, 1, 2, 3, 4, 5


class lq_gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("q0", ctypes.c_int32), ("q1", ctypes.c_int32),
                ("q2", ctypes.c_int32), ("param_idx", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("angle", ctypes.c_double), ("mat", ctypes.POINTER(ctypes.c_double))]


class lq_pauli_term(ctypes.Structure):
    _fields_ = [("coeff", ctypes.c_double), ("x_mask", ctypes.c_uint64), ("z_mask", ctypes.c_uint64)]


class lq_xyz_model(ctypes.Structure):
    _fields_ = [("jx", ctypes.c_double), ("jy", ctypes.c_double), ("jz", ctypes.c_double),
                ("amp", ctypes.c_double), ("omega", ctypes.c_double)]


class lq_adam_cfg(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("tol", ctypes.c_double), ("max_iter", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class LQError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_P = ctypes.c_void_p
_i32, _i64, _u64, _sz, _dbl = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_double
_GP = ctypes.POINTER(lq_gate)
_TP = ctypes.POINTER(lq_pauli_term)
_DP = ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "lq_last_error": ([], ctypes.c_char_p),
    "lq_version": ([], _i32),
    "lq_device_count": ([], _i32),
    "lq_sv_alloc": ([_i32, _P, ctypes.POINTER(_P)], _i32),
    "lq_sv_wrap": ([_i32, _P, _P, _sz, ctypes.POINTER(_P)], _i32),
    "lq_sv_free": ([_P], _i32),
    "lq_sv_set_stream": ([_P, _P], _i32),
    "lq_sv_num_qubits": ([_P], _i32),
    "lq_sv_device_ptr": ([_P], _P),
    "lq_sv_qubit_map": ([_P, ctypes.POINTER(ctypes.c_int32)], _i32),
    "lq_sv_init_basis": ([_P, _u64], _i32),
    "lq_sv_init_random": ([_P, _u64], _i32),
    "lq_sv_read": ([_P, _u64, _u64, _DP], _i32),
    "lq_sv_write": ([_P, _u64, _u64, _DP], _i32),
    "lq_sv_gather": ([_P, ctypes.POINTER(ctypes.c_uint64), _sz, _DP], _i32),
    "lq_sv_norm2": ([_P, _DP], _i32),
    "lq_sv_canonicalize": ([_P], _i32),
    "lq_apply_circuit": ([_P, _GP, _sz, _DP, _sz], _i32),
    "lq_qft": ([_P, _i32], _i32),
    "lq_expval_pauli_sum": ([_P, _TP, _sz, _DP], _i32),
    "lq_param_shift_grad": ([_i32, _GP, _sz, _DP, _sz, _TP, _sz, _P, _P, _DP, _DP], _i32),
    "lq_psr_create": ([_i32, _GP, _sz, _sz, _TP, _sz, _P, _P, ctypes.POINTER(_P)], _i32),
    "lq_psr_run": ([_P, _P, _P, _P], _i32),
    "lq_psr_free": ([_P], _i32),
    "lq_psr_stats": ([_P, ctypes.POINTER(_u64), ctypes.POINTER(_u64), ctypes.POINTER(_u64),
                      ctypes.POINTER(_u64)], _i32),
    "lq_kernel_timing": ([_i32, ctypes.POINTER(_dbl), ctypes.POINTER(_u64)], _i32),
    "lq_kernel_timing_reset": ([], _i32),
    "lq_set_option": ([_i32, _i64], _i32),
    "lq_get_option": ([_i32], _i64),
    "lq_plan_describe": ([_i32, _GP, _sz, ctypes.POINTER(_u64), ctypes.POINTER(_u64), ctypes.c_char_p, _sz], _i32),
    "lq_launch_count": ([], _u64),
    "lq_plan_export_json": ([_i32, _GP, _sz, _TP, _sz, ctypes.c_char_p, _sz, ctypes.POINTER(_sz)], _i32),
    "lq_psr_cache_clear": ([], _i32),
    "lq_comm_unique_id": ([_P, _sz], _i32),
    "lq_comm_init": ([_P, _sz, _i32, _i32, ctypes.POINTER(_P)], _i32),
    "lq_comm_free": ([_P], _i32),
    "lq_comm_init_local": ([_i32, _i32, ctypes.POINTER(_P)], _i32),
    "lq_psr_pass_tiles": ([_P, ctypes.POINTER(_u64), _sz, ctypes.POINTER(_sz)], _i32),
    "lq_tile_sweep": ([_P, _sz, _i32, _u64, _i32, _P, ctypes.POINTER(_dbl)], _i32),
    "lq_comm_info": ([_P, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32)], _i32),
    "lq_sv_exchange_stats": ([_P, ctypes.POINTER(_u64), ctypes.POINTER(_u64)], _i32),
    "lq_sv_alloc_sharded": ([_i32, _P, _P, ctypes.POINTER(_P)], _i32),
    "lq_sv_alloc_group": ([_i32, _i32, _P, ctypes.POINTER(_P)], _i32),
    "lq_sv_shard_info": ([_P, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                          ctypes.POINTER(ctypes.c_uint32)], _i32),
    "lq_sv_shard_ptr": ([_P, _i32], _P),
    "lq_dist_schedule_json": ([_i32, _i32, _GP, _sz, _i32, _TP, _sz, ctypes.c_char_p, _sz, ctypes.POINTER(_sz)], _i32),
    "lq_psr_traffic": ([_P, ctypes.POINTER(_u64), ctypes.POINTER(_u64)], _i32),
    "lq_psr_pass_bytes": ([_P, ctypes.POINTER(_u64), ctypes.POINTER(_i32), ctypes.POINTER(_u64),
                           ctypes.POINTER(ctypes.c_uint32), ctypes.c_size_t,
                           ctypes.POINTER(ctypes.c_size_t)], _i32),
    "lq_jit_stats": ([ctypes.POINTER(_u64), ctypes.POINTER(_u64), ctypes.POINTER(_dbl)], _i32),
    "lq_jit_compile_check": ([_i32, _GP, _sz, _TP, _sz, ctypes.POINTER(_u64)], _i32),
    "lq_qft_jit_compile_check": ([_i32, _i32, ctypes.POINTER(_u64)], _i32),
    "lq_qft_plan_export_json": ([_i32, _i32, _i32, ctypes.c_char_p, _sz, ctypes.POINTER(ctypes.c_size_t)], _i32),
    "lq_trotter_xyz": ([_P, _P, _dbl, _dbl, _i32, _i32, _DP], _i32),
    "lq_vqe_adam": ([_i32, _GP, _sz, _DP, _sz, _TP, _sz, _P, _P, _DP, ctypes.POINTER(ctypes.c_int32)], _i32),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def _chk(status: int):
    if status != LQ_OK:
        raise LQError(status, _lib.lq_last_error().decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_DP)


# ---- marshalling ------------------------------------------------------------
_GATE_ROW = struct.Struct("=6idQ")     # lq_gate: 6 x int32, double angle, const double *mat
_TERM_ROW = struct.Struct("=dQQ")      # lq_pauli_term


class GateArray:
    """Gate tuples ``(name, q0, q1, param_idx, angle[, mat][, q2])`` (the
    workloads format) as a contiguous ``lq_gate[]`` plus owned matrices.
    Rows are packed with one ``struct`` call each (about 0.15 us per gate):
    the marshalling is on the latency path of every small-state call
    (configs 1 and 3), where per-field ctypes stores cost ~1 us per gate."""

    def __init__(self, gates: Sequence[tuple]):
        self.n = len(gates)
        self._mats: List[np.ndarray] = []
        pack, kinds, rows = _GATE_ROW.pack, KINDS, []
        for g in gates:
            name = g[0]
            mp = 0
            if len(g) > 5 and g[5] is not None:
                m = np.asarray(g[5], np.complex128).reshape(-1)
                buf = np.ascontiguousarray(np.stack([m.real, m.imag], -1).reshape(-1))
                self._mats.append(buf)
                mp = buf.ctypes.data
            rows.append(pack(kinds[name] if isinstance(name, str) else name, g[1], g[2],
                             g[6] if len(g) > 6 else -1, g[3], 0, g[4], mp))
        self.arr = np.frombuffer(bytearray(b"".join(rows) or bytes(_GATE_ROW.size)), np.uint8)

    @property
    def ptr(self):
        return ctypes.cast(self.arr.ctypes.data, _GP)


class TermArray:
    def __init__(self, terms: Sequence[tuple]):
        self.n = len(terms)
        pack = _TERM_ROW.pack
        rows = [pack(c, x, z) for c, x, z in terms]
        self.arr = np.frombuffer(bytearray(b"".join(rows) or bytes(_TERM_ROW.size)), np.uint8)

    @property
    def ptr(self):
        return ctypes.cast(self.arr.ctypes.data, _TP)


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---- C ABI, same names --------------------------------------------------------
def lq_last_error() -> str:
    return _lib.lq_last_error().decode()


def lq_version() -> int:
    return _lib.lq_version()


def lq_device_count() -> int:
    return _lib.lq_device_count()


def lq_launch_count() -> int:
    return _lib.lq_launch_count()


def lq_set_option(option: int, value: int):
    _chk(_lib.lq_set_option(option, int(value)))


def lq_get_option(option: int) -> int:
    return _lib.lq_get_option(option)


def lq_sv_alloc(n_qubits: int, stream=None):
    h = _P()
    _chk(_lib.lq_sv_alloc(n_qubits, _stream_ptr(stream), ctypes.byref(h)))
    return h


def lq_sv_wrap(n_qubits: int, dev_ptr: int, nbytes: int, stream=None):
    h = _P()
    _chk(_lib.lq_sv_wrap(n_qubits, _stream_ptr(stream), dev_ptr, nbytes, ctypes.byref(h)))
    return h


def lq_sv_free(h):
    _chk(_lib.lq_sv_free(h))


def lq_sv_set_stream(h, stream):
    _chk(_lib.lq_sv_set_stream(h, _stream_ptr(stream)))


def lq_sv_num_qubits(h) -> int:
    return _lib.lq_sv_num_qubits(h)


def lq_sv_device_ptr(h) -> int:
    return _lib.lq_sv_device_ptr(h)


def lq_sv_qubit_map(h) -> List[int]:
    n = lq_sv_num_qubits(h)
    out = (ctypes.c_int32 * 64)()
    _chk(_lib.lq_sv_qubit_map(h, out))
    return list(out[:n])


def lq_sv_init_basis(h, k: int):
    _chk(_lib.lq_sv_init_basis(h, int(k)))


def lq_sv_init_random(h, seed: int):
    _chk(_lib.lq_sv_init_random(h, int(seed) & (2**64 - 1)))


def lq_sv_read(h, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
    n = lq_sv_num_qubits(h)
    if count is None:
        count = (1 << n) - offset
    out = np.empty(count, np.complex128)
    _chk(_lib.lq_sv_read(h, offset, count, out.ctypes.data_as(_DP)))
    return out


def lq_sv_write(h, amps: np.ndarray, offset: int = 0):
    a = np.ascontiguousarray(amps, np.complex128)
    _chk(_lib.lq_sv_write(h, offset, a.size, a.ctypes.data_as(_DP)))


def lq_sv_gather(h, idx: Iterable[int]) -> np.ndarray:
    ix = np.ascontiguousarray(np.asarray(list(idx) if not isinstance(idx, np.ndarray) else idx, np.uint64))
    out = np.empty(ix.size, np.complex128)
    _chk(_lib.lq_sv_gather(h, ix.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ix.size,
                           out.ctypes.data_as(_DP)))
    return out


def lq_sv_norm2(h) -> float:
    out = ctypes.c_double()
    _chk(_lib.lq_sv_norm2(h, ctypes.byref(out)))
    return out.value


def lq_sv_canonicalize(h):
    _chk(_lib.lq_sv_canonicalize(h))


def lq_apply_circuit(h, gates, theta=None):
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    th = None if theta is None else np.ascontiguousarray(theta, np.float64)
    _chk(_lib.lq_apply_circuit(h, ga.ptr, ga.n, None if th is None else _dptr(th),
                               0 if th is None else th.size))


def lq_qft(h, inverse: bool = False):
    _chk(_lib.lq_qft(h, int(bool(inverse))))


def lq_expval_pauli_sum(h, terms) -> float:
    ta = terms if isinstance(terms, TermArray) else TermArray(terms)
    out = ctypes.c_double()
    _chk(_lib.lq_expval_pauli_sum(h, ta.ptr, ta.n, ctypes.byref(out)))
    return out.value


def lq_param_shift_grad(n_qubits: int, ansatz, theta, terms, comm=None, stream=None,
                        with_energy: bool = True) -> Tuple[np.ndarray, Optional[float]]:
    """comm: None (one GPU), an NCCL lq_comm (collective; full gradient and E
    on every rank) or lq_comm_init_local(rank, world) (this rank's share)."""
    ga = ansatz if isinstance(ansatz, GateArray) else GateArray(ansatz)
    ta = terms if isinstance(terms, TermArray) else TermArray(terms)
    th = np.ascontiguousarray(theta, np.float64)
    grad = np.zeros(th.size, np.float64)
    e = ctypes.c_double()
    _chk(_lib.lq_param_shift_grad(n_qubits, ga.ptr, ga.n, _dptr(th), th.size, ta.ptr, ta.n, comm,
                                  _stream_ptr(stream), _dptr(grad),
                                  ctypes.byref(e) if with_energy else None))
    return grad, (e.value if with_energy else None)


def lq_trotter_xyz(h, jx: float, jy: float, jz: float, amp: float, omega: float, t0: float, dt: float,
                   n_steps: int, record_every: int = 1) -> np.ndarray:
    """First-order Trotter evolution of the XYZ chain on
    state handle h; returns E(t) at t0 and after every record_every steps."""
    m = lq_xyz_model(jx, jy, jz, amp, omega)
    out = np.zeros(1 + n_steps // record_every, np.float64)
    _chk(_lib.lq_trotter_xyz(h, ctypes.byref(m), t0, dt, n_steps, record_every, _dptr(out)))
    return out


def lq_vqe_adam(n_qubits: int, ansatz, theta0, terms, lr: float = 1e-2, beta1: float = 0.9,
                beta2: float = 0.999, eps: float = 1e-8, tol: float = 1e-7, max_iter: int = 350,
                stream=None) -> Tuple[np.ndarray, np.ndarray, int]:
    """VQE outer loop: Adam on parameter-shift gradients.
    Returns (final theta, energy trace E_0..E_T, T = Adam updates)."""
    ga = ansatz if isinstance(ansatz, GateArray) else GateArray(ansatz)
    ta = terms if isinstance(terms, TermArray) else TermArray(terms)
    th = np.array(theta0, np.float64, copy=True)
    trace = np.zeros(max_iter + 1, np.float64)
    cfg = lq_adam_cfg(lr, beta1, beta2, eps, tol, max_iter, 0)
    it = ctypes.c_int32()
    _chk(_lib.lq_vqe_adam(n_qubits, ga.ptr, ga.n, _dptr(th), th.size, ta.ptr, ta.n, ctypes.byref(cfg),
                          _stream_ptr(stream), _dptr(trace), ctypes.byref(it)))
    return th, trace[: it.value + 1].copy(), it.value


def lq_psr_create(n_qubits: int, ansatz, n_params: int, terms, comm=None, stream=None):
    ga = ansatz if isinstance(ansatz, GateArray) else GateArray(ansatz)
    ta = terms if isinstance(terms, TermArray) else TermArray(terms)
    h = _P()
    _chk(_lib.lq_psr_create(n_qubits, ga.ptr, ga.n, n_params, ta.ptr, ta.n, comm,
                            _stream_ptr(stream), ctypes.byref(h)))
    return h


def lq_psr_run(plan, theta_dev: int, grad_dev: int, energy_dev: Optional[int] = None):
    _chk(_lib.lq_psr_run(plan, theta_dev, grad_dev, energy_dev))


def lq_psr_free(plan):
    _chk(_lib.lq_psr_free(plan))


def lq_psr_stats(plan) -> Tuple[int, int, int, int]:
    """(circuits, launches of the last run, plan bytes uploaded, tile passes per circuit)"""
    c, l, b, t = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _chk(_lib.lq_psr_stats(plan, ctypes.byref(c), ctypes.byref(l), ctypes.byref(b), ctypes.byref(t)))
    return c.value, l.value, b.value, t.value


def lq_psr_traffic(plan) -> Tuple[int, int]:
    """(algorithmic HBM bytes per circuit through tile passes, through other kernels)"""
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    _chk(_lib.lq_psr_traffic(plan, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def lq_psr_cache_clear() -> None:
    """Drop the cached PSR handles and single-state plans (lq_param_shift_grad)."""
    _chk(_lib.lq_psr_cache_clear())


def lq_psr_pass_bytes(plan, with_support: bool = False):
    """[(kind, algorithmic HBM bytes per circuit)] per launched pass (0 tile, 1 pair, 2 diagonal);
    with_support: [(kind, bytes, amplitudes per circuit the pass's gates act on, planner ops in the pass)]"""
    n = ctypes.c_size_t()
    _chk(_lib.lq_psr_pass_bytes(plan, None, None, None, None, 0, ctypes.byref(n)))
    m = max(n.value, 1)
    b, k, a, o = (_u64 * m)(), (_i32 * m)(), (_u64 * m)(), (ctypes.c_uint32 * m)()
    _chk(_lib.lq_psr_pass_bytes(plan, b, k, a, o, n.value, ctypes.byref(n)))
    if with_support:
        return [(k[i], b[i], a[i], o[i]) for i in range(n.value)]
    return [(k[i], b[i]) for i in range(n.value)]


def lq_psr_pass_tiles(plan) -> List[int]:
    n = ctypes.c_size_t()
    _chk(_lib.lq_psr_pass_tiles(plan, None, 0, ctypes.byref(n)))
    out = (_u64 * max(n.value, 1))()
    _chk(_lib.lq_psr_pass_tiles(plan, out, n.value, ctypes.byref(n)))
    return [int(out[i]) for i in range(n.value)]


def lq_tile_sweep(dev_ptr: int, nbytes: int, n_bits: int, tile_mask: int, reps: int = 3, stream=None) -> float:
    """ms per in-place sweep of 2^n_bits amplitudes with tile_mask's access pattern."""
    ms = ctypes.c_double()
    _chk(_lib.lq_tile_sweep(dev_ptr, nbytes, n_bits, tile_mask, reps, _stream_ptr(stream), ctypes.byref(ms)))
    return ms.value


def lq_kernel_timing(kernel_class: int) -> Tuple[float, int]:
    ms, n = ctypes.c_double(), ctypes.c_uint64()
    _chk(_lib.lq_kernel_timing(kernel_class, ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def lq_kernel_timing_reset():
    _chk(_lib.lq_kernel_timing_reset())


def lq_plan_describe(n_qubits: int, gates) -> Tuple[int, int, str]:
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    np_, nt = ctypes.c_uint64(), ctypes.c_uint64()
    buf = ctypes.create_string_buffer(1 << 16)
    _chk(_lib.lq_plan_describe(n_qubits, ga.ptr, ga.n, ctypes.byref(np_), ctypes.byref(nt), buf, len(buf)))
    return np_.value, nt.value, buf.value.decode()


def lq_plan_export_json(n_qubits: int, gates, terms=()) -> dict:
    import json
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    ta = terms if isinstance(terms, TermArray) else TermArray(terms)
    need = ctypes.c_size_t()
    _chk(_lib.lq_plan_export_json(n_qubits, ga.ptr, ga.n, ta.ptr, ta.n, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _chk(_lib.lq_plan_export_json(n_qubits, ga.ptr, ga.n, ta.ptr, ta.n, buf, len(buf), ctypes.byref(need)))
    return json.loads(buf.value.decode())


def lq_jit_stats() -> Tuple[int, int, float]:
    """(pass kernels compiled, cache hits, compile seconds) of this process."""
    c, h, t = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_double()
    _chk(_lib.lq_jit_stats(ctypes.byref(c), ctypes.byref(h), ctypes.byref(t)))
    return c.value, h.value, t.value


def lq_jit_compile_check(n_qubits: int, gates, terms=()) -> int:
    """Host-only: NVRTC-compile the plan's JIT pass programs (no device)."""
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    ta = terms if isinstance(terms, TermArray) else TermArray(terms)
    nk = ctypes.c_uint64()
    _chk(_lib.lq_jit_compile_check(n_qubits, ga.ptr, ga.n, ta.ptr, ta.n, ctypes.byref(nk)))
    return nk.value


def lq_qft_jit_compile_check(n_qubits: int, inverse: bool = False) -> int:
    nk = _u64()
    _chk(_lib.lq_qft_jit_compile_check(n_qubits, int(bool(inverse)), ctypes.byref(nk)))
    return nk.value


def lq_qft_plan_export_json(n_qubits: int, inverse: bool = False, reversed_layout: bool = False) -> dict:
    import json
    need = ctypes.c_size_t()
    _chk(_lib.lq_qft_plan_export_json(n_qubits, int(bool(inverse)), int(bool(reversed_layout)), None, 0,
                                      ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _chk(_lib.lq_qft_plan_export_json(n_qubits, int(bool(inverse)), int(bool(reversed_layout)), buf, len(buf),
                                      ctypes.byref(need)))
    return json.loads(buf.value.decode())


# ---- sharded states (a9) ---------------------------------------------------
def lq_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _chk(_lib.lq_comm_unique_id(buf, 128))
    return buf.raw


def lq_comm_init(unique_id: bytes, rank: int, world: int):
    h = _P()
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    _chk(_lib.lq_comm_init(buf, 128, rank, world, ctypes.byref(h)))
    return h


def lq_comm_free(h):
    _chk(_lib.lq_comm_free(h))


def lq_comm_init_local(rank: int, world: int):
    """A transport-less communicator: partitioned work returns this rank's share."""
    h = _P()
    _chk(_lib.lq_comm_init_local(rank, world, ctypes.byref(h)))
    return h


def lq_comm_info(h) -> Tuple[int, int, bool]:
    r, w, t = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _chk(_lib.lq_comm_info(h, ctypes.byref(r), ctypes.byref(w), ctypes.byref(t)))
    return r.value, w.value, bool(t.value)


def lq_sv_exchange_stats(h) -> Tuple[int, int]:
    """(global-qubit exchanges so far, bytes each rank sent in them)"""
    n, b = _u64(), _u64()
    _chk(_lib.lq_sv_exchange_stats(h, ctypes.byref(n), ctypes.byref(b)))
    return n.value, b.value


def comm_from_torch(group=None):
    """An lq_comm over the ranks of a torch.distributed process group: rank 0
    creates the NCCL unique id, torch broadcasts it (plumbing only)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [lq_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return lq_comm_init(obj[0], rank, world)


def lq_sv_alloc_sharded(n_qubits: int, comm, stream=None):
    h = _P()
    _chk(_lib.lq_sv_alloc_sharded(n_qubits, comm, _stream_ptr(stream), ctypes.byref(h)))
    return h


def lq_sv_alloc_group(n_qubits: int, world: int, stream=None):
    h = _P()
    _chk(_lib.lq_sv_alloc_group(n_qubits, world, _stream_ptr(stream), ctypes.byref(h)))
    return h


def lq_sv_shard_info(h) -> Tuple[int, int, int, int]:
    """(log2 world, first rank held here, shards held here, rank relabel xmask)"""
    m, r, k, x = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_uint32()
    _chk(_lib.lq_sv_shard_info(h, ctypes.byref(m), ctypes.byref(r), ctypes.byref(k), ctypes.byref(x)))
    return m.value, r.value, k.value, x.value


def lq_sv_shard_ptr(h, k: int) -> int:
    return _lib.lq_sv_shard_ptr(h, k)


def lq_dist_schedule_json(n_qubits: int, log2_world: int, gates, qft: int = 0, terms=()) -> dict:
    import json
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    ta = terms if isinstance(terms, TermArray) else TermArray(terms)
    need = ctypes.c_size_t()
    _chk(_lib.lq_dist_schedule_json(n_qubits, log2_world, ga.ptr, ga.n, qft, ta.ptr, ta.n, None, 0,
                                    ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _chk(_lib.lq_dist_schedule_json(n_qubits, log2_world, ga.ptr, ga.n, qft, ta.ptr, ta.n, buf, len(buf),
                                    ctypes.byref(need)))
    return json.loads(buf.value.decode())


class ShardedState:
    """A state sharded over 2^m ranks (library-owned shards).  ``comm`` = an
    lq_comm (one process per GPU, NCCL), or ``group_world`` = G shards held
    by this process (device-copy exchanges on one GPU).  Calls are
    collective across the comm's ranks."""

    def __init__(self, n_qubits: int, comm=None, group_world: Optional[int] = None, stream=None):
        self.n = n_qubits
        if comm is not None:
            self.h = lq_sv_alloc_sharded(n_qubits, comm, stream)
        else:
            self.h = lq_sv_alloc_group(n_qubits, int(group_world), stream)

    def free(self):
        if self.h is not None:
            lq_sv_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def init_basis(self, k: int):
        lq_sv_init_basis(self.h, k)
        return self

    def init_random(self, seed: int):
        lq_sv_init_random(self.h, seed)
        return self

    def apply(self, gates, theta=None):
        lq_apply_circuit(self.h, gates, theta)
        return self

    def qft(self, inverse: bool = False):
        lq_qft(self.h, inverse)
        return self

    def expval(self, terms) -> float:
        return lq_expval_pauli_sum(self.h, terms)

    def read(self, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
        return lq_sv_read(self.h, offset, count)

    def gather(self, idx) -> np.ndarray:
        return lq_sv_gather(self.h, idx)

    def norm2(self) -> float:
        return lq_sv_norm2(self.h)

    def qubit_map(self) -> List[int]:
        return lq_sv_qubit_map(self.h)

    def shard_info(self):
        return lq_sv_shard_info(self.h)


# ---- convenience: a torch-owned state ---------------------------------------
class StateVector:
    """A state whose amplitudes live in a torch complex128 CUDA tensor
    (``self.tensor``, physical layout) wrapped by an lq_sv handle."""

    def __init__(self, n_qubits: int, stream=None, device=None):
        import torch
        self.n = n_qubits
        self.tensor = torch.empty(1 << n_qubits, dtype=torch.complex128,
                                  device=device if device is not None else "cuda")
        self.h = lq_sv_wrap(n_qubits, self.tensor.data_ptr(), self.tensor.numel() * 16, stream)

    def free(self):
        if self.h is not None:
            lq_sv_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def init_basis(self, k: int):
        lq_sv_init_basis(self.h, k)
        return self

    def init_random(self, seed: int):
        lq_sv_init_random(self.h, seed)
        return self

    def apply(self, gates, theta=None):
        lq_apply_circuit(self.h, gates, theta)
        return self

    def qft(self, inverse: bool = False):
        lq_qft(self.h, inverse)
        return self

    def expval(self, terms) -> float:
        return lq_expval_pauli_sum(self.h, terms)

    def trotter_xyz(self, jx, jy, jz, amp, omega, t0, dt, n_steps, record_every=1) -> np.ndarray:
        return lq_trotter_xyz(self.h, jx, jy, jz, amp, omega, t0, dt, n_steps, record_every)

    def read(self, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
        return lq_sv_read(self.h, offset, count)

    def gather(self, idx) -> np.ndarray:
        return lq_sv_gather(self.h, idx)

    def norm2(self) -> float:
        return lq_sv_norm2(self.h)

    def canonicalize(self):
        lq_sv_canonicalize(self.h)
        return self

    def qubit_map(self) -> List[int]:
        return lq_sv_qubit_map(self.h)
