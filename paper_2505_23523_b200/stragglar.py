"""Thin ctypes binding of libstragglar.so (include/stragglar.h).

Argument marshalling only: every function here forwards to the C function of
the same name; all data movement and arithmetic run in the CUDA kernels.
Tensors are torch CUDA tensors (PyTorch provides device memory and streams);
their data pointers, element counts and dtypes are passed through.  There is
no CPU fallback: if the shared library is missing, importing this module
raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STRAGGLAR_LIB") or os.path.join(HERE, "libstragglar.so")  # override: tuning variants

INT32, FLOAT32, BFLOAT16 = 0, 1, 2
SUM = 0
STATUS = {
    0: "ok", 1: "invalid argument", 2: "unsupported", 3: "not initialized",
    4: "not registered", 5: "CUDA error", 6: "timeout", 7: "internal error",
}


class StragglarError(RuntimeError):
    def __init__(self, fn: str, status: int):
        self.status = status
        super().__init__(f"{fn} failed: {status} ({_status_string(status)})")


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    return ctypes.CDLL(LIB_PATH)


_lib = _load()

_c_int, _c_size, _c_u64, _vp = ctypes.c_int, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_void_p
_PP = ctypes.POINTER(ctypes.c_void_p)
_SIGS = {
    "stragglar_version": ([], _c_int),
    "stragglar_status_string": ([_c_int], ctypes.c_char_p),
    "stragglar_launch_count": ([ctypes.POINTER(_c_u64)], _c_int),
    "stragglar_schedule_rounds": ([_c_int, ctypes.POINTER(_c_int)], _c_int),
    "stragglar_schedule_round": ([_c_int, _c_int, ctypes.POINTER(_c_int), _c_int, ctypes.POINTER(_c_int)], _c_int),
    "stragglar_plan_layout": ([_c_int, _c_int, _c_size, _c_int, _c_int, _c_int, ctypes.POINTER(_c_int),
                               ctypes.POINTER(_c_int), ctypes.POINTER(_c_int)], _c_int),
    "stragglar_plan_e2e_pieces": ([_c_size, _c_int, _c_size, ctypes.POINTER(_c_size), _c_int,
                                   ctypes.POINTER(_c_int)], _c_int),
    "stragglar_init": ([_c_int, _c_int, _c_int], _c_int),
    "stragglar_handle_size": ([ctypes.POINTER(_c_size)], _c_int),
    "stragglar_export_handle": ([_vp], _c_int),
    "stragglar_import_handles": ([_vp, _c_int], _c_int),
    "stragglar_register_buffer": ([_vp, _c_size, _vp], _c_int),
    "stragglar_import_buffer": ([_vp, _vp, _c_int], _c_int),
    "stragglar_deregister_buffer": ([_vp], _c_int),
    "stragglar_shared_device_ranks": ([ctypes.POINTER(_c_int), ctypes.POINTER(_c_int)], _c_int),
    "stragglar_probe_copy": ([_vp, _c_size, _c_int, ctypes.c_uint32, _c_int, _vp], _c_int),
    "stragglar_probe_pingpong": ([_c_int, _c_int, _vp], _c_int),
    "stragglar_probe_pingpong_result": ([ctypes.POINTER(ctypes.c_double)], _c_int),
    "stragglar_nvls_supported": ([ctypes.POINTER(_c_int)], _c_int),
    "stragglar_nvls_begin": ([_c_size, ctypes.POINTER(_c_int), ctypes.POINTER(_c_size)], _c_int),
    "stragglar_nvls_import": ([_c_int, _c_int, _c_int], _c_int),
    "stragglar_nvls_bind": ([ctypes.POINTER(_vp)], _c_int),
    "stragglar_nvls_release": ([], _c_int),
    "stragglar_allreduce_nvls": ([_vp, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_nvls_selftest": ([_c_int, _c_size, _vp, _vp], _c_int),
    "stragglar_allreduce_nvls_emulated": ([_vp, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_allreduce": ([_vp, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_allreduce_ring": ([_vp, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_allreduce_direct": ([_vp, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_allreduce_host": ([_vp, _vp, _vp, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_allreduce_rhd": ([_vp, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_allreduce_bcast": ([_vp, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_broadcast_tree": ([_c_int, ctypes.POINTER(_c_int), ctypes.POINTER(_c_int)], _c_int),
    "stragglar_barrier": ([_vp], _c_int),
    "stragglar_last_barrier_ns": ([ctypes.POINTER(_c_u64)], _c_int),
    "stragglar_inject_delay": ([_c_u64, _vp], _c_int),
    "stragglar_check_error": ([ctypes.POINTER(_c_int)], _c_int),
    "stragglar_finalize": ([], _c_int),
    "stragglar_check_error_where": ([_c_int, ctypes.POINTER(_c_int), ctypes.POINTER(ctypes.c_uint32)], _c_int),
    "stragglar_phase_times": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], _c_int),
    "stragglar_select": ([_c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                          ctypes.POINTER(_c_int), ctypes.POINTER(ctypes.c_double)], _c_int),
    "stragglar_select_algorithm": ([_c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.POINTER(_c_int), ctypes.POINTER(ctypes.c_double)], _c_int),
    "stragglar_set_cost_model": ([ctypes.c_double, ctypes.c_double], _c_int),
    "stragglar_allreduce_auto": ([_vp, _c_size, _c_int, _c_int, _vp, _c_u64, ctypes.POINTER(_c_int)], _c_int),
    "stragglar_team_init": ([_c_int, _c_int], _c_int),
    "stragglar_team_allreduce": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_reduce_scatter": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_complete": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_allreduce_ring": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_complete_direct": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_allreduce_direct": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_allreduce_rhd": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_bcast_precondition": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_bcast_complete": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_allreduce_bcast": ([_PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_inject_delay": ([_c_u64, _vp], _c_int),
    "stragglar_team_allreduce_delayed": ([_PP, _c_size, _c_int, _c_int, _c_u64, _vp], _c_int),
    "stragglar_team_allreduce_host": ([_PP, _PP, _PP, _c_size, _c_int, _c_int, _vp], _c_int),
    "stragglar_team_slices": ([ctypes.POINTER(_c_int)], _c_int),
    "stragglar_team_set_trace": ([_c_int], _c_int),
    "stragglar_team_read_trace": ([ctypes.POINTER(_c_u64), _c_size, ctypes.POINTER(_c_size), ctypes.POINTER(_c_int)], _c_int),
    "stragglar_team_check_error": ([ctypes.POINTER(_c_int)], _c_int),
    "stragglar_team_finalize": ([], _c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def _status_string(s: int) -> str:
    return _lib.stragglar_status_string(s).decode()


def _ck(fn: str, status: int) -> None:
    if status != 0:
        raise StragglarError(fn, status)


# ---------------------------------------------------------------- marshalling helpers
def _dtype_code(t) -> int:
    import torch

    m = {torch.int32: INT32, torch.float32: FLOAT32, torch.bfloat16: BFLOAT16}
    if t.dtype not in m:
        raise TypeError(f"unsupported dtype {t.dtype} (int32, float32, bfloat16)")
    return m[t.dtype]


def _stream_ptr(stream) -> Optional[int]:
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    if isinstance(stream, int):
        return stream or None
    return stream.cuda_stream or None


def _ptr_array(ts: Sequence) -> ctypes.Array:
    arr = (ctypes.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = t if isinstance(t, int) else t.data_ptr()
    return arr


def _dev_args(t):
    """A per-process buffer: contiguous CUDA tensor of a supported dtype."""
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("buffers must be contiguous CUDA tensors")
    return t.data_ptr(), t.numel(), _dtype_code(t)


def _team_args(bufs: Sequence):
    if not bufs:
        raise ValueError("empty buffer list")
    n, dt = bufs[0].numel(), _dtype_code(bufs[0])
    for b in bufs:
        if b.numel() != n or _dtype_code(b) != dt or not b.is_cuda or not b.is_contiguous():
            raise ValueError("team buffers must be contiguous CUDA tensors of equal size and dtype")
    return _ptr_array(bufs), n, dt


# ---------------------------------------------------------------- info / schedule
def stragglar_version() -> int:
    return _lib.stragglar_version()


def stragglar_launch_count() -> int:
    v = _c_u64(0)
    _ck("stragglar_launch_count", _lib.stragglar_launch_count(ctypes.byref(v)))
    return int(v.value)


def stragglar_schedule_rounds(world: int) -> int:
    r = _c_int(0)
    _ck("stragglar_schedule_rounds", _lib.stragglar_schedule_rounds(world, ctypes.byref(r)))
    return r.value


def stragglar_schedule_round(world: int, rnd: int) -> List[Tuple[int, int, int, int]]:
    cap = 4 * world
    out = (_c_int * (4 * cap))()
    k = _c_int(0)
    _ck("stragglar_schedule_round", _lib.stragglar_schedule_round(world, rnd, out, cap, ctypes.byref(k)))
    return [tuple(out[4 * i:4 * i + 4]) for i in range(k.value)]


def stragglar_plan_layout(world: int, straggler_rank: int, count: int, dtype_code: int, ctas_per_rank: int,
                          sys_scope: bool = False):
    """-> (slices per chunk, slices per CTA, op lanes) of a StragglAR call (host only)."""
    g, sub, lanes = _c_int(0), _c_int(0), _c_int(0)
    _ck("stragglar_plan_layout", _lib.stragglar_plan_layout(world, straggler_rank, int(count), dtype_code, ctas_per_rank,
                                                            1 if sys_scope else 0, ctypes.byref(g), ctypes.byref(sub),
                                                            ctypes.byref(lanes)))
    return g.value, sub.value, lanes.value


def stragglar_plan_e2e_pieces(count: int, dtype_code: int, piece_bytes: int):
    """-> element counts of the pieces the host-buffer entry points cut `count` into (host only)."""
    cap = 8 + int(count) // max(1, int(piece_bytes) // 4 // 4 * 4)
    out = (_c_size * cap)()
    k = _c_int(0)
    _ck("stragglar_plan_e2e_pieces", _lib.stragglar_plan_e2e_pieces(int(count), dtype_code, int(piece_bytes),
                                                                    out, cap, ctypes.byref(k)))
    return list(out[:k.value])


# ---------------------------------------------------------------- per-process communicator
def stragglar_init(rank: int, world: int, straggler_rank: int) -> None:
    _ck("stragglar_init", _lib.stragglar_init(rank, world, straggler_rank))


def stragglar_handle_size() -> int:
    v = _c_size(0)
    _ck("stragglar_handle_size", _lib.stragglar_handle_size(ctypes.byref(v)))
    return v.value


def stragglar_export_handle() -> bytes:
    buf = ctypes.create_string_buffer(stragglar_handle_size())
    _ck("stragglar_export_handle", _lib.stragglar_export_handle(buf))
    return buf.raw


def stragglar_import_handles(blobs: bytes, world: int) -> None:
    _ck("stragglar_import_handles", _lib.stragglar_import_handles(ctypes.c_char_p(blobs), world))


def stragglar_register_buffer(t) -> bytes:
    buf = ctypes.create_string_buffer(stragglar_handle_size())
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("registered buffers must be contiguous CUDA tensors")
    nbytes = t.numel() * t.element_size()
    _ck("stragglar_register_buffer", _lib.stragglar_register_buffer(t.data_ptr(), nbytes, buf))
    return buf.raw


def stragglar_import_buffer(t, blobs: bytes, world: int) -> None:
    _ck("stragglar_import_buffer", _lib.stragglar_import_buffer(t.data_ptr(), ctypes.c_char_p(blobs), world))


def stragglar_deregister_buffer(t) -> None:
    _ck("stragglar_deregister_buffer", _lib.stragglar_deregister_buffer(t if isinstance(t, int) else t.data_ptr()))


def stragglar_shared_device_ranks():
    """-> (ranks of this communicator on this rank's GPU, CTAs per rank per launch)."""
    a, b = _c_int(0), _c_int(0)
    _ck("stragglar_shared_device_ranks", _lib.stragglar_shared_device_ranks(ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


PROBE_PUSH, PROBE_PULL, PROBE_TMA = 0, 1, 2


def stragglar_probe_copy(t, bytes_per_peer: int, mode: int, peers, ctas: int = 0, stream=None) -> None:
    """K0: device-initiated copies with every peer in `peers` at once (see include/stragglar.h)."""
    mask = 0
    for p in peers:
        mask |= 1 << int(p)
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("probe buffer must be a contiguous CUDA tensor")
    _ck("stragglar_probe_copy", _lib.stragglar_probe_copy(t.data_ptr(), int(bytes_per_peer), int(mode), mask,
                                                           int(ctas), _stream_ptr(stream)))


def stragglar_probe_pingpong(peer: int, iters: int, stream=None) -> None:
    _ck("stragglar_probe_pingpong", _lib.stragglar_probe_pingpong(int(peer), int(iters), _stream_ptr(stream)))


def stragglar_probe_pingpong_result() -> float:
    """-> device time (us) of the last ping-pong (all its round trips)."""
    v = ctypes.c_double(0.0)
    _ck("stragglar_probe_pingpong_result", _lib.stragglar_probe_pingpong_result(ctypes.byref(v)))
    return v.value


def stragglar_allreduce(t, stream=None) -> None:
    ptr, n, dt = _dev_args(t)
    _ck("stragglar_allreduce", _lib.stragglar_allreduce(ptr, n, dt, SUM, _stream_ptr(stream)))


def stragglar_allreduce_ring(t, stream=None) -> None:
    ptr, n, dt = _dev_args(t)
    _ck("stragglar_allreduce_ring", _lib.stragglar_allreduce_ring(ptr, n, dt, SUM, _stream_ptr(stream)))


def stragglar_allreduce_host(host_in, host_out, t, stream=None) -> None:
    """host_in/host_out: contiguous CPU tensors (pinned for full bandwidth) shaped like t."""
    ptr, n, dt = _dev_args(t)
    for h in (host_in, host_out):
        if h.is_cuda or h.numel() != n or h.dtype != t.dtype or not h.is_contiguous():
            raise ValueError("host buffers must be contiguous CPU tensors matching the device buffer")
    _ck("stragglar_allreduce_host",
        _lib.stragglar_allreduce_host(host_in.data_ptr(), host_out.data_ptr(), ptr, n, dt, SUM, _stream_ptr(stream)))


def stragglar_select(world: int, nbytes: float, delay_s: float, alpha_s: float, beta_s_per_byte: float):
    """-> (use_stragglar: bool, critical_delay_s: float)"""
    use, crit = _c_int(0), ctypes.c_double(0.0)
    _ck("stragglar_select", _lib.stragglar_select(world, float(nbytes), float(delay_s), float(alpha_s),
                                                  float(beta_s_per_byte), ctypes.byref(use), ctypes.byref(crit)))
    return bool(use.value), crit.value


ALGO_RING, ALGO_STRAGGLAR, ALGO_RHD = 0, 1, 2
ALGO_NAMES = {ALGO_RING: "ring", ALGO_STRAGGLAR: "stragglar", ALGO_RHD: "rhd"}


def stragglar_select_algorithm(world: int, nbytes: float, delay_s: float, alpha_s: float, beta_s_per_byte: float):
    """-> (algorithm name, predicted completion in s) — see include/stragglar.h."""
    a, t = _c_int(0), ctypes.c_double(0.0)
    _ck("stragglar_select_algorithm",
        _lib.stragglar_select_algorithm(world, float(nbytes), float(delay_s), float(alpha_s), float(beta_s_per_byte),
                                        ctypes.byref(a), ctypes.byref(t)))
    return ALGO_NAMES[a.value], t.value


def stragglar_set_cost_model(alpha_s: float, beta_s_per_byte: float) -> None:
    _ck("stragglar_set_cost_model", _lib.stragglar_set_cost_model(float(alpha_s), float(beta_s_per_byte)))


def stragglar_allreduce_auto(t, expected_delay_ns: int, stream=None) -> str:
    """Runs the algorithm the cost model picks; returns its name ("stragglar", "ring" or "rhd")."""
    used = _c_int(0)
    ptr, n, dt = _dev_args(t)
    _ck("stragglar_allreduce_auto",
        _lib.stragglar_allreduce_auto(ptr, n, dt, SUM, _stream_ptr(stream), int(expected_delay_ns), ctypes.byref(used)))
    return ALGO_NAMES[used.value]


def stragglar_allreduce_direct(t, stream=None) -> None:
    ptr, n, dt = _dev_args(t)
    _ck("stragglar_allreduce_direct", _lib.stragglar_allreduce_direct(ptr, n, dt, SUM, _stream_ptr(stream)))


def stragglar_allreduce_rhd(t, stream=None) -> None:
    ptr, n, dt = _dev_args(t)
    _ck("stragglar_allreduce_rhd", _lib.stragglar_allreduce_rhd(ptr, n, dt, SUM, _stream_ptr(stream)))


def stragglar_allreduce_bcast(t, stream=None) -> None:
    ptr, n, dt = _dev_args(t)
    _ck("stragglar_allreduce_bcast", _lib.stragglar_allreduce_bcast(ptr, n, dt, SUM, _stream_ptr(stream)))


def stragglar_broadcast_tree(world: int):
    """-> (sender, round) lists in logical ranks (sender -1 for the two holders)."""
    snd, rnd = (_c_int * world)(), (_c_int * world)()
    _ck("stragglar_broadcast_tree", _lib.stragglar_broadcast_tree(world, snd, rnd))
    return list(snd), list(rnd)


def stragglar_barrier(stream=None) -> None:
    _ck("stragglar_barrier", _lib.stragglar_barrier(_stream_ptr(stream)))


def stragglar_last_barrier_ns() -> int:
    v = _c_u64(0)
    _ck("stragglar_last_barrier_ns", _lib.stragglar_last_barrier_ns(ctypes.byref(v)))
    return int(v.value)


def stragglar_inject_delay(ns: int, stream=None) -> None:
    _ck("stragglar_inject_delay", _lib.stragglar_inject_delay(int(ns), _stream_ptr(stream)))


def stragglar_check_error() -> int:
    code = _c_int(0)
    st = _lib.stragglar_check_error(ctypes.byref(code))
    if st not in (0, 6):
        _ck("stragglar_check_error", st)
    return code.value


def stragglar_check_error_where(team: bool = False):
    """-> (code, where): the device error word and the failing wait's location."""
    code, where = _c_int(0), ctypes.c_uint32(0)
    st = _lib.stragglar_check_error_where(1 if team else 0, ctypes.byref(code), ctypes.byref(where))
    if st not in (0, 6):
        _ck("stragglar_check_error_where", st)
    return code.value, where.value


def stragglar_phase_times():
    """-> (t_a_us, t_total_us) of this rank's last fused call (in-kernel stamps)."""
    a, t = ctypes.c_double(0), ctypes.c_double(0)
    _ck("stragglar_phase_times", _lib.stragglar_phase_times(ctypes.byref(a), ctypes.byref(t)))
    return a.value, t.value


# ---------------------------------------------------------------- NEXT N1(i): NVLS multicast
def stragglar_nvls_supported() -> bool:
    v = _c_int(0)
    _ck("stragglar_nvls_supported", _lib.stragglar_nvls_supported(ctypes.byref(v)))
    return bool(v.value)


def stragglar_nvls_begin(nbytes: int):
    """-> ([mc_all_fd, mc_ns_fd, arena_fd] (-1 where this rank exports none), rounded arena bytes)."""
    fds, out = (_c_int * 3)(), _c_size(0)
    _ck("stragglar_nvls_begin", _lib.stragglar_nvls_begin(int(nbytes), fds, ctypes.byref(out)))
    return list(fds), out.value


def stragglar_nvls_import(mc_all_fd: int, mc_ns_fd: int, sigma_mem_fd: int) -> int:
    """-> status (0 = imported); the caller agrees across ranks before binding."""
    return int(_lib.stragglar_nvls_import(int(mc_all_fd), int(mc_ns_fd), int(sigma_mem_fd)))


def stragglar_nvls_bind() -> int:
    """-> the arena's device pointer."""
    p = _vp(0)
    _ck("stragglar_nvls_bind", _lib.stragglar_nvls_bind(ctypes.byref(p)))
    return int(p.value)


def stragglar_nvls_release() -> None:
    _ck("stragglar_nvls_release", _lib.stragglar_nvls_release())


def stragglar_allreduce_nvls(t, stream=None) -> None:
    ptr, n, dt = _dev_args(t)
    _ck("stragglar_allreduce_nvls", _lib.stragglar_allreduce_nvls(ptr, n, dt, SUM, _stream_ptr(stream)))


def stragglar_allreduce_nvls_emulated(t, stream=None) -> None:
    """Test only: the NVLS kernel with its multicast operations emulated on a registered buffer."""
    ptr, n, dt = _dev_args(t)
    _ck("stragglar_allreduce_nvls_emulated",
        _lib.stragglar_allreduce_nvls_emulated(ptr, n, dt, SUM, _stream_ptr(stream)))


def stragglar_nvls_selftest(host_in) -> "object":
    """host_in: contiguous CPU tensor; returns its reducing load through a one-member multicast object."""
    import torch

    if host_in.is_cuda or not host_in.is_contiguous():
        raise ValueError("host tensor expected")
    out = torch.empty_like(host_in)
    _ck("stragglar_nvls_selftest", _lib.stragglar_nvls_selftest(_dtype_code(host_in), host_in.numel(),
                                                                host_in.data_ptr(), out.data_ptr()))
    return out


class _DeviceArray:
    """__cuda_array_interface__ view of library memory (torch.as_tensor wraps it without a copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 2}


def device_bytes(ptr: int, nbytes: int):
    """A uint8 torch tensor aliasing nbytes of library device memory at ptr."""
    import torch

    return torch.as_tensor(_DeviceArray(ptr, nbytes), device="cuda")


def stragglar_finalize() -> None:
    _ck("stragglar_finalize", _lib.stragglar_finalize())


# ---------------------------------------------------------------- single-device team
def stragglar_team_init(world: int, straggler_rank: int) -> None:
    _ck("stragglar_team_init", _lib.stragglar_team_init(world, straggler_rank))


def stragglar_team_slices() -> int:
    v = _c_int(0)
    _ck("stragglar_team_slices", _lib.stragglar_team_slices(ctypes.byref(v)))
    return v.value


def _team_call(name: str, bufs, stream) -> None:
    arr, n, dt = _team_args(bufs)
    _ck(name, getattr(_lib, name)(arr, n, dt, SUM, _stream_ptr(stream)))


def stragglar_team_allreduce(bufs, stream=None) -> None:
    _team_call("stragglar_team_allreduce", bufs, stream)


def stragglar_team_reduce_scatter(bufs, stream=None) -> None:
    _team_call("stragglar_team_reduce_scatter", bufs, stream)


def stragglar_team_complete(bufs, stream=None) -> None:
    _team_call("stragglar_team_complete", bufs, stream)


def stragglar_team_allreduce_ring(bufs, stream=None) -> None:
    _team_call("stragglar_team_allreduce_ring", bufs, stream)


def stragglar_team_complete_direct(bufs, stream=None) -> None:
    _team_call("stragglar_team_complete_direct", bufs, stream)


def stragglar_team_allreduce_direct(bufs, stream=None) -> None:
    _team_call("stragglar_team_allreduce_direct", bufs, stream)


def stragglar_team_allreduce_rhd(bufs, stream=None) -> None:
    _team_call("stragglar_team_allreduce_rhd", bufs, stream)


def stragglar_team_bcast_precondition(bufs, stream=None) -> None:
    _team_call("stragglar_team_bcast_precondition", bufs, stream)


def stragglar_team_bcast_complete(bufs, stream=None) -> None:
    _team_call("stragglar_team_bcast_complete", bufs, stream)


def stragglar_team_allreduce_bcast(bufs, stream=None) -> None:
    _team_call("stragglar_team_allreduce_bcast", bufs, stream)


def stragglar_team_allreduce_delayed(bufs, delay_ns: int, stream=None) -> None:
    arr, n, dt = _team_args(bufs)
    _ck("stragglar_team_allreduce_delayed",
        _lib.stragglar_team_allreduce_delayed(arr, n, dt, SUM, int(delay_ns), _stream_ptr(stream)))


def stragglar_team_inject_delay(ns: int, stream=None) -> None:
    _ck("stragglar_team_inject_delay", _lib.stragglar_team_inject_delay(int(ns), _stream_ptr(stream)))


def stragglar_team_allreduce_host(host_in, host_out, bufs, stream=None) -> None:
    """host_in/host_out: CPU tensors (pinned for full bandwidth) matching bufs."""
    arr, n, dt = _team_args(bufs)
    for h in list(host_in) + list(host_out):
        if h.is_cuda or h.numel() != n or _dtype_code(h) != dt or not h.is_contiguous():
            raise ValueError("host buffers must be contiguous CPU tensors matching the device buffers")
    _ck("stragglar_team_allreduce_host",
        _lib.stragglar_team_allreduce_host(_ptr_array(host_in), _ptr_array(host_out), arr, n, dt, SUM,
                                           _stream_ptr(stream)))


def stragglar_team_set_trace(enable: bool) -> None:
    _ck("stragglar_team_set_trace", _lib.stragglar_team_set_trace(1 if enable else 0))


def stragglar_team_read_trace():
    """-> (list of uint64 stamps [rank][slice][op][wait, data, done], slices per chunk)."""
    n, g = _c_size(0), _c_int(0)
    st = _lib.stragglar_team_read_trace(None, 0, ctypes.byref(n), ctypes.byref(g))
    if st not in (0, 1):
        _ck("stragglar_team_read_trace", st)
    buf = (_c_u64 * n.value)()
    _ck("stragglar_team_read_trace", _lib.stragglar_team_read_trace(buf, n.value, ctypes.byref(n), ctypes.byref(g)))
    return list(buf), g.value


def stragglar_team_check_error() -> int:
    code = _c_int(0)
    st = _lib.stragglar_team_check_error(ctypes.byref(code))
    if st not in (0, 6):
        _ck("stragglar_team_check_error", st)
    return code.value


def stragglar_team_finalize() -> None:
    _ck("stragglar_team_finalize", _lib.stragglar_team_finalize())
