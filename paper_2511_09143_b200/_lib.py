"""ctypes binding of libflexshm.so (the C ABI declared in include/flexshm.h).

The library is built in-tree (`__graft_entry__.build()` or `make -C
paper_2511_09143_b200/csrc`).  There is no fallback: if the shared object is
missing, importing anything that needs it raises immediately.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (
    CommAbortedError,
    DuplicateDeviceError,
    FlexShmError,
    MalformedLabelError,
    ShmTimeoutError,
    TransportUnavailableError,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libflexshm.so")

FMX_OK = 0
FMX_ERR_DUPLICATE_DEVICE = 1
FMX_ERR_MALFORMED_LABEL = 2
FMX_ERR_BAD_RANKS = 3
FMX_ERR_EMPTY_MIG_ID = 4
FMX_ERR_INVALID_ARG = 5
FMX_ERR_CUDA = 6
FMX_ERR_SHM = 7
FMX_ERR_TIMEOUT = 8
FMX_ERR_ABORTED = 9
FMX_ERR_UNSUPPORTED = 10

FLOAT32, BFLOAT16 = 0, 1
OP_SUM, OP_SUM_POSTSCALE, OP_PREDIV_SUM, OP_PREMUL_SUM = 0, 1, 2, 3
TRANSPORT_AUTO, TRANSPORT_ZC, TRANSPORT_CE, TRANSPORT_HOST = 0, 1, 2, 3
TRANSPORTS = {"auto": TRANSPORT_AUTO, "zc": TRANSPORT_ZC, "ce": TRANSPORT_CE,
              "host": TRANSPORT_HOST}

BUS_ID_LEN = 16
MIG_ID_LEN = 128
MAX_RANKS = 64

# Every symbol include/flexshm.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "fmx_check_peer", "fmx_validate_peers", "fmx_topology", "fmx_restore_bus_id",
    "fmx_comm_init", "fmx_allreduce", "fmx_allreduce_sgd", "fmx_allreduce_shard", "fmx_broadcast", "fmx_reduce_scatter", "fmx_allgather",
    "fmx_host_buffer", "fmx_allreduce_host",
    "fmx_reduce_local", "fmx_barrier", "fmx_comm_destroy",
    "fmx_comm_abort", "fmx_comm_rank", "fmx_comm_count", "fmx_comm_peer", "fmx_comm_config",
    "fmx_comm_kernel_launches", "fmx_comm_flags", "fmx_comm_set_timing", "fmx_comm_kernel_time",
    "fmx_comm_monitor", "fmx_comm_set_stamps", "fmx_comm_stamps",
    "fmx_comm_stamp", "fmx_comm_set_join_stream", "fmx_comm_completion_stream",
    "fmx_comm_fence", "fmx_comm_set_defer", "fmx_comm_flush", "fmx_graph_capture_begin", "fmx_graph_capture_end",
    "fmx_graph_launch_prepare", "fmx_graph_release",
    "fmx_trace_plan", "fmx_last_error", "fmx_dup_ranks",
    "fmx_abi_version",
)


class SgdC(ctypes.Structure):
    """struct fmx_sgd (include/flexshm.h)."""
    _fields_ = [("lr", ctypes.c_float), ("momentum", ctypes.c_float),
                ("dampening", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("nesterov", ctypes.c_int), ("first_step", ctypes.c_int)]


class PeerInfoC(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("pcie_bus_id", ctypes.c_char * BUS_ID_LEN),
        ("mig_id", ctypes.c_char * MIG_ID_LEN),
        ("host_hash", ctypes.c_int64),
        ("pid_hash", ctypes.c_int64),
    ]


def _i64(v: int) -> int:
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= 1 << 63 else v


def peer_to_c(rank: int, pcie_bus_id: str, mig_id: str, host_hash: int, pid_hash: int) -> PeerInfoC:
    bus = pcie_bus_id.encode()
    mig = mig_id.encode()
    if len(bus) >= BUS_ID_LEN:
        raise MalformedLabelError(f"bus id {pcie_bus_id!r} is not a canonical device id")
    if len(mig) >= MIG_ID_LEN:
        raise ValueError(f"mig_id longer than {MIG_ID_LEN - 1} bytes")
    return PeerInfoC(rank, bus, mig, _i64(host_hash), _i64(pid_hash))


_lib: ctypes.CDLL | None = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; "
            "g.build()\"` (no CPU fallback exists for the SHM data path)")
    L = ctypes.CDLL(LIB_PATH)
    c_int, c_size, c_void, c_float, c_double = (ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p,
                                                ctypes.c_float, ctypes.c_double)
    P = ctypes.POINTER
    sig = {
        "fmx_check_peer": [P(PeerInfoC)],
        "fmx_validate_peers": [P(PeerInfoC), c_int, c_int, P(c_int), P(c_int)],
        "fmx_topology": [P(PeerInfoC), c_int, ctypes.c_char_p, ctypes.c_char_p, P(c_int), P(c_int)],
        "fmx_restore_bus_id": [ctypes.c_char_p, ctypes.c_char_p],
        "fmx_comm_init": [P(c_void), ctypes.c_char_p, c_int, c_int, P(PeerInfoC), c_int, c_size,
                          c_int, c_size, c_int, c_double],
        "fmx_host_buffer": [c_void, c_int, P(c_void), P(c_size)],
        "fmx_allreduce_host": [c_void, c_size, c_size, c_int, c_int, c_float, c_void],
        "fmx_reduce_local": [P(c_void), c_int, ctypes.c_uint64, c_void, c_void, c_size, c_int,
                             c_int, c_float, c_void],
        "fmx_allreduce": [c_void, c_void, c_void, c_size, c_int, c_int, c_float, c_void],
        "fmx_allreduce_sgd": [c_void, c_void, c_void, c_void, c_size, c_int, c_float, P(SgdC),
                              c_void],
        "fmx_allreduce_shard": [c_void, c_size, c_int, P(c_size), P(c_size)],
        "fmx_broadcast": [c_void, c_void, c_void, c_size, c_int, c_int, c_void],
        "fmx_reduce_scatter": [c_void, c_void, c_void, c_size, c_int, c_int, c_float, c_void],
        "fmx_allgather": [c_void, c_void, c_void, c_size, c_int, c_void],
        "fmx_barrier": [c_void, c_double],
        "fmx_comm_destroy": [c_void],
        "fmx_comm_abort": [c_void],
        "fmx_comm_rank": [c_void, P(c_int)],
        "fmx_comm_count": [c_void, P(c_int)],
        "fmx_comm_peer": [c_void, c_int, P(PeerInfoC)],
        "fmx_comm_config": [c_void, P(c_size), P(c_int), P(c_size)],
        "fmx_comm_kernel_launches": [c_void, P(ctypes.c_uint64)],
        "fmx_comm_flags": [c_void, P(ctypes.c_uint32), c_int],
        "fmx_comm_set_timing": [c_void, c_int],
        "fmx_comm_monitor": [c_void, c_double, P(ctypes.c_uint64), c_size, P(c_size)],
        "fmx_comm_kernel_time": [c_void, P(c_double), P(ctypes.c_uint64)],
        "fmx_comm_set_stamps": [c_void, c_size],
        "fmx_comm_stamps": [c_void, P(ctypes.c_uint64), c_size, P(c_size)],
        "fmx_comm_stamp": [c_void, c_void, ctypes.c_uint32],
        "fmx_comm_set_join_stream": [c_void, c_void],
        "fmx_comm_completion_stream": [c_void, P(c_void)],
        "fmx_comm_fence": [c_void, c_void],
        "fmx_comm_set_defer": [c_void, c_int],
        "fmx_comm_flush": [c_void, c_void],
        "fmx_graph_capture_begin": [c_void],
        "fmx_graph_capture_end": [c_void, c_void, P(c_int)],
        "fmx_graph_launch_prepare": [c_void, c_int, c_void, c_void],
        "fmx_graph_release": [c_void, c_int],
        "fmx_trace_plan": [c_int, c_int, c_int, c_size, c_int, P(c_int), P(c_size), P(c_int),
                           P(c_int), ctypes.c_char_p, c_size, P(c_size)],
        "fmx_dup_ranks": [P(c_int), P(c_int)],
        "fmx_abi_version": [],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = c_int
    L.fmx_last_error.argtypes = []
    L.fmx_last_error.restype = ctypes.c_char_p
    if L.fmx_abi_version() != 1:
        raise ImportError("libflexshm ABI version mismatch")
    _lib = L
    return L


def trace_plan(nranks: int, rank: int, ops: list[tuple], slice_bytes: int = 4096,
               transport: str = "ce") -> str:
    """Schedule text of `rank` for ops = [("allreduce" | "allreduce_host" |
    "reduce_scatter" | "allgather", count, dtype) | ("broadcast", count,
    dtype, root)] (see fmx_trace_plan; reduce_scatter / allgather counts are
    per rank)."""
    n = len(ops)
    code = {"allreduce": 0, "broadcast": 1, "allreduce_host": 2, "reduce_scatter": 3,
            "allgather": 4, "flush": 5}
    kinds = (ctypes.c_int * max(1, n))(*[code[o[0]] for o in ops])
    counts = (ctypes.c_size_t * max(1, n))(*[o[1] for o in ops])
    dtypes = (ctypes.c_int * max(1, n))(*[o[2] for o in ops])
    roots = (ctypes.c_int * max(1, n))(*[o[3] if len(o) > 3 else 0 for o in ops])
    used = ctypes.c_size_t()
    L = lib()
    L.fmx_trace_plan(nranks, rank, TRANSPORTS[transport], slice_bytes, n, kinds, counts, dtypes,
                     roots, None, 0, ctypes.byref(used))
    buf = ctypes.create_string_buffer(used.value)
    check(L.fmx_trace_plan(nranks, rank, TRANSPORTS[transport], slice_bytes, n, kinds, counts,
                           dtypes, roots, buf, used.value, ctypes.byref(used)), "fmx_trace_plan")
    return buf.value.decode()


def last_error() -> str:
    msg = lib().fmx_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Raise the Python exception that corresponds to an FMX status code."""
    if rc == FMX_OK:
        return
    msg = last_error() or what
    if rc == FMX_ERR_DUPLICATE_DEVICE:
        a, b = ctypes.c_int(), ctypes.c_int()
        lib().fmx_dup_ranks(ctypes.byref(a), ctypes.byref(b))
        raise DuplicateDeviceError(a.value, b.value)
    if rc == FMX_ERR_MALFORMED_LABEL:
        raise MalformedLabelError(msg)
    if rc in (FMX_ERR_BAD_RANKS, FMX_ERR_EMPTY_MIG_ID, FMX_ERR_INVALID_ARG):
        raise ValueError(msg)
    if rc == FMX_ERR_TIMEOUT:
        raise ShmTimeoutError(msg, rc)
    if rc == FMX_ERR_ABORTED:
        raise CommAbortedError(msg, rc)
    if rc == FMX_ERR_UNSUPPORTED and "NET" in msg:
        raise TransportUnavailableError(msg, rc)
    raise FlexShmError(f"{what}: {msg}" if what else msg, rc)
