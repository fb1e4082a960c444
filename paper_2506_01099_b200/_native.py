"""ctypes binding of libbenelux_b200.so (C ABI: include/benelux_b200.h).

The product path has exactly one backend: the hand-written sm_100a kernels in
``csrc/``.  If the library is missing or no CUDA device is visible, every entry point
raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbenelux_b200.so")

BNX_OK = 0
BNX_TABLE_FULL = 1
BNX_BUFFER_FULL = 2
BNX_ERR_PRIMES_UNCOVERED = 3
BNX_ERR_INVALID = 4
BNX_ERR_CUDA = 5
BNX_ERR_RANGE = 6

KIND_FIRST, KIND_SECOND, KIND_BOTH = 1, 2, 3
ENGINES = {"heavy": 0, "screen": 1}  # bnx_ctx_set_engine (include/benelux_b200.h)

# Every symbol include/benelux_b200.h declares (tests check the library exports them all).
EXPORTED_SYMBOLS = (
    "bnx_version", "bnx_last_error", "bnx_device_count", "bnx_ctx_create", "bnx_ctx_destroy",
    "bnx_ctx_set_stream", "bnx_ctx_stats", "bnx_ctx_set_timing", "bnx_ctx_timing", "bnx_ctx_kernel_timing", "bnx_ctx_class_table", "bnx_ctx_set_engine", "bnx_ctx_engine", "bnx_ctx_set_shard", "bnx_primes_up_to", "bnx_sieve_radicals",
    "bnx_sieve_radicals_dev", "bnx_radicals_trial_division", "bnx_search", "bnx_search_domain", "bnx_search_multi",
    "bnx_prepare", "bnx_search_enqueue", "bnx_search_collect", "bnx_slot_of", "bnx_brute_force",
    "bnx_table_create", "bnx_table_destroy", "bnx_table_insert_all", "bnx_table_probe_all", "bnx_table_slots",
    "bnx_table_search_chunk",
)


class NativeLibraryMissing(RuntimeError):
    """libbenelux_b200.so is not built (run __graft_entry__.build())."""


class CudaError(RuntimeError):
    """The CUDA runtime failed or no device is present."""


class PairRow(ctypes.Structure):
    """bnx_pair_t"""

    _fields_ = [
        ("m", ctypes.c_uint64),
        ("n", ctypes.c_uint64),
        ("rad_m", ctypes.c_uint64),
        ("rad_m1", ctypes.c_uint64),
        ("kind", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


PAIR_DTYPE = np.dtype(
    [("m", "<u8"), ("n", "<u8"), ("rad_m", "<u8"), ("rad_m1", "<u8"), ("kind", "<i4"), ("reserved", "<i4")]
)


class Stats(ctypes.Structure):
    """bnx_stats_t"""

    _fields_ = [
        ("integers", ctypes.c_uint64),
        ("survivors", ctypes.c_uint64),
        ("candidates", ctypes.c_uint64),
        ("residue_checks", ctypes.c_uint64),
        ("matches", ctypes.c_uint64),
        ("pairs", ctypes.c_uint64),
        ("kernel_launches", ctypes.c_uint64),
        ("bucket_overflow", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("max_residue_checks", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_ if name != "reserved"}


_u64p = ctypes.POINTER(ctypes.c_uint64)
_lib = None
_lib_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """The loaded library; raises NativeLibraryMissing if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        L.bnx_version.restype = ctypes.c_int
        L.bnx_last_error.restype = ctypes.c_char_p
        L.bnx_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
        L.bnx_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
        L.bnx_ctx_destroy.argtypes = [vp]
        L.bnx_ctx_set_stream.argtypes = [vp, vp]
        L.bnx_ctx_stats.argtypes = [vp, ctypes.POINTER(Stats)]
        L.bnx_ctx_set_timing.argtypes = [vp, ctypes.c_int]
        L.bnx_ctx_set_engine.argtypes = [vp, ctypes.c_int]
        L.bnx_ctx_engine.argtypes = [vp]
        L.bnx_ctx_set_shard.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32]
        L.bnx_ctx_timing.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
        L.bnx_ctx_kernel_timing.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int]
        L.bnx_ctx_class_table.argtypes = [vp, ctypes.c_uint64, _u64p, _u64p, ctypes.c_size_t,
                                          ctypes.POINTER(ctypes.c_size_t)]
        L.bnx_primes_up_to.argtypes = [vp, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
        L.bnx_sieve_radicals.argtypes = [
            vp, ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int, _u64p,
        ]
        L.bnx_sieve_radicals_dev.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, vp]
        L.bnx_radicals_trial_division.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, _u64p]
        search_args = [
            vp, ctypes.c_uint64, ctypes.c_uint32, _u64p, ctypes.c_size_t, ctypes.c_uint64,
            ctypes.POINTER(PairRow), ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
        ]
        L.bnx_search.argtypes = search_args
        L.bnx_search_domain.argtypes = [vp, ctypes.c_uint64] + search_args[1:]
        L.bnx_search_multi.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_int] + search_args[1:]
        L.bnx_brute_force.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(PairRow), ctypes.c_size_t,
                                      ctypes.POINTER(ctypes.c_size_t)]
        L.bnx_table_create.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(vp)]
        L.bnx_table_destroy.argtypes = [vp]
        L.bnx_table_insert_all.argtypes = [vp, ctypes.c_uint64, _u64p, _u64p, ctypes.c_size_t, ctypes.c_uint64,
                                           ctypes.POINTER(PairRow), ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
                                           ctypes.POINTER(ctypes.c_uint64)]
        L.bnx_table_probe_all.argtypes = [vp, ctypes.c_uint64, _u64p, _u64p, ctypes.c_size_t,
                                          ctypes.POINTER(PairRow), ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
        L.bnx_table_slots.argtypes = [vp, _u64p, ctypes.c_size_t]
        L.bnx_table_search_chunk.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_uint64, ctypes.POINTER(PairRow), ctypes.c_size_t,
                                             ctypes.POINTER(ctypes.c_size_t)]
        L.bnx_prepare.argtypes = [vp, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_uint64]
        L.bnx_search_enqueue.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32]
        L.bnx_search_collect.argtypes = [vp, ctypes.POINTER(PairRow), ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
        L.bnx_slot_of.restype = ctypes.c_uint64
        L.bnx_slot_of.argtypes = [ctypes.c_uint64] * 6
        _lib = L
    return _lib


def last_error() -> str:
    msg = load().bnx_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> int:
    """Map a status code onto the reference's exception types."""
    if status in (BNX_OK, BNX_BUFFER_FULL):
        return status
    msg = last_error()
    if status in (BNX_ERR_PRIMES_UNCOVERED, BNX_ERR_INVALID, BNX_ERR_RANGE):
        raise ValueError(msg)
    if status == BNX_TABLE_FULL:
        raise RuntimeError(msg)
    raise CudaError(msg or f"libbenelux_b200 status {status}")


def device_count() -> int:
    n = ctypes.c_int(0)
    load().bnx_device_count(ctypes.byref(n))
    return int(n.value)


class Context:
    """One GPU + stream + cached tables (bnx_ctx_t).  Calls are serialised by a lock."""

    def __init__(self, device: int = 0):
        L = load()
        handle = ctypes.c_void_p()
        check(L.bnx_ctx_create(device, ctypes.byref(handle)))
        self.handle = handle
        self.device = device
        self.lock = threading.RLock()
        self._buf = None
        self._found = None

    def close(self) -> None:
        if self.handle:
            load().bnx_ctx_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def set_stream(self, stream_ptr: int) -> None:
        with self.lock:
            check(load().bnx_ctx_set_stream(self.handle, ctypes.c_void_p(stream_ptr or None)))

    def stats(self) -> dict:
        s = Stats()
        check(load().bnx_ctx_stats(self.handle, ctypes.byref(s)))
        return s.as_dict()

    def set_timing(self, mode: bool | int) -> None:
        """0/False: off; 1/True: generator / pipeline split; 2: per-kernel events (direct launches)."""
        with self.lock:
            check(load().bnx_ctx_set_timing(self.handle, int(mode)))

    def set_engine(self, engine: str | int) -> None:
        """Candidate generator: "heavy" (default) or "screen" (identical results)."""
        code = ENGINES[engine] if isinstance(engine, str) else int(engine)
        with self.lock:
            check(load().bnx_ctx_set_engine(self.handle, code))

    def set_shard(self, shard: int, nshards: int) -> None:
        """Multi-GPU: later searches compute shard `shard` of `nshards` (include/benelux_b200.h)."""
        with self.lock:
            check(load().bnx_ctx_set_shard(self.handle, shard, nshards))

    def engine(self) -> str:
        code = load().bnx_ctx_engine(self.handle)
        return {v: k for k, v in ENGINES.items()}.get(code, str(code))

    def timing(self) -> tuple[float, float]:
        """(screen kernel ms, whole device pipeline ms) of the last search (CUDA events)."""
        a, b = ctypes.c_float(0), ctypes.c_float(0)
        check(load().bnx_ctx_timing(self.handle, ctypes.byref(a), ctypes.byref(b)))
        return float(a.value), float(b.value)

    def kernel_timing(self) -> dict:
        """Per-stage ms of the last search in timing mode 2 (include/benelux_b200.h)."""
        ms = (ctypes.c_float * 4)()
        check(load().bnx_ctx_kernel_timing(self.handle, ms, 4))
        return dict(zip(("count_scan", "screen", "exact", "tail"), (float(v) for v in ms)))

    def class_table(self, max_x: int) -> tuple[np.ndarray, np.ndarray]:
        """(b, m | r << 40) of the heavy generator's surplus classes for bound max_x, in device order."""
        count = ctypes.c_size_t(0)
        with self.lock:
            check(load().bnx_ctx_class_table(self.handle, max_x, None, None, 0, ctypes.byref(count)))
            b = np.empty(max(1, count.value), np.uint64)
            mr = np.empty(max(1, count.value), np.uint64)
            check(load().bnx_ctx_class_table(self.handle, max_x, b.ctypes.data_as(_u64p), mr.ctypes.data_as(_u64p),
                                             b.size, ctypes.byref(count)))
        return b[: count.value], mr[: count.value]

    # -- primes ---------------------------------------------------------------------
    def primes_up_to(self, limit: int) -> np.ndarray:
        L = load()
        cap = max(64, int(1.3 * limit / max(1.0, np.log(max(limit, 2)))) + 64)
        while True:
            out = np.empty(cap, np.uint64)
            count = ctypes.c_size_t(0)
            with self.lock:
                st = check(L.bnx_primes_up_to(self.handle, limit, out.ctypes.data_as(_u64p), cap, ctypes.byref(count)))
            if st == BNX_BUFFER_FULL:
                cap = int(count.value)
                continue
            return out[: int(count.value)].copy()

    # -- radicals -------------------------------------------------------------------
    def sieve_radicals(self, start: int, length: int, primes: np.ndarray | None, primes_limit: int,
                       ctz_fast_path: bool = True) -> np.ndarray:
        out = np.empty(length, np.uint64)
        keep, pp, np_ = _prime_args(primes)  # noqa: F841 (keeps the array alive)
        with self.lock:
            check(load().bnx_sieve_radicals(self.handle, start, length, pp, np_, primes_limit,
                                            int(bool(ctz_fast_path)), out.ctypes.data_as(_u64p)))
        return out

    def sieve_radicals_dev(self, start: int, length: int, out_ptr: int, ctz_fast_path: bool = True) -> None:
        with self.lock:
            check(load().bnx_sieve_radicals_dev(self.handle, start, length, int(bool(ctz_fast_path)),
                                                ctypes.c_void_p(out_ptr)))

    def radicals_trial_division(self, start: int, length: int) -> np.ndarray:
        out = np.empty(length, np.uint64)
        with self.lock:
            check(load().bnx_radicals_trial_division(self.handle, start, length, out.ctypes.data_as(_u64p)))
        return out

    # -- search ---------------------------------------------------------------------
    def _rows(self, fn) -> np.ndarray:
        # one row buffer per context, grown on BNX_BUFFER_FULL (the result is copied out)
        with self.lock:
            while True:
                buf = self._buf
                if buf is None:
                    buf = self._buf = (PairRow * 256)()
                    self._found = ctypes.c_size_t(0)
                cap = len(buf)
                st = check(fn(buf, cap, ctypes.byref(self._found)))
                if st == BNX_BUFFER_FULL:
                    self._buf = (PairRow * int(self._found.value))()
                    continue
                return np.frombuffer(buf, dtype=PAIR_DTYPE, count=int(self._found.value)).copy()

    def search(self, limit: int, kinds: int, primes: np.ndarray | None, primes_limit: int) -> np.ndarray:
        keep, pp, np_ = _prime_args(primes)  # noqa: F841 (keeps the array alive)
        return self._rows(lambda b, c, f: load().bnx_search(self.handle, limit, kinds, pp, np_, primes_limit, b, c, f))

    def search_domain(self, n_first: int, n_last: int, kinds: int, primes: np.ndarray | None,
                      primes_limit: int) -> np.ndarray:
        keep, pp, np_ = _prime_args(primes)  # noqa: F841 (keeps the array alive)
        return self._rows(
            lambda b, c, f: load().bnx_search_domain(self.handle, n_first, n_last, kinds, pp, np_, primes_limit, b, c, f)
        )

    def brute_force(self, limit: int) -> np.ndarray:
        return self._rows(lambda b, c, f: load().bnx_brute_force(self.handle, limit, b, c, f))

    def prepare(self, max_x: int, primes: np.ndarray | None = None, primes_limit: int = 0) -> None:
        keep, pp, np_ = _prime_args(primes)  # noqa: F841 (keeps the array alive)
        with self.lock:
            check(load().bnx_prepare(self.handle, max_x, pp, np_, primes_limit))

    def enqueue(self, n_first: int, n_last: int, kinds: int) -> None:
        with self.lock:
            check(load().bnx_search_enqueue(self.handle, n_first, n_last, kinds))

    def collect(self) -> np.ndarray:
        return self._rows(lambda b, c, f: load().bnx_search_collect(self.handle, b, c, f))


def _prime_args(primes):
    """(array kept alive by the caller's frame, pointer, count) for an optional prime list."""
    if primes is None:
        return None, None, 0
    arr = np.ascontiguousarray(primes, dtype=np.uint64)
    return arr, arr.ctypes.data_as(_u64p), int(arr.size)


_contexts: dict[int, Context] = {}
_ctx_lock = threading.Lock()


def context(device: int | None = None) -> Context:
    """The process-wide context of `device` (default: $BNX_DEVICE, else 0)."""
    if device is None:
        device = int(os.environ.get("BNX_DEVICE", "0"))
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx


def search_multi(devices, limit: int, kinds: int, primes: np.ndarray | None = None, primes_limit: int = 0) -> np.ndarray:
    """bnx_search_multi: one host thread drives every device in `devices` (a shard each);
    rows sorted by (m, n), identical to a single-device search."""
    L = load()
    devs = (ctypes.c_int * len(devices))(*devices)
    keep, pp, np_ = _prime_args(primes)  # noqa: F841 (keeps the array alive)
    cap = 256
    while True:
        buf = (PairRow * cap)()
        found = ctypes.c_size_t(0)
        with _MULTI_LOCK:
            st = check(L.bnx_search_multi(devs, len(devices), limit, kinds, pp, np_, primes_limit, buf, cap,
                                          ctypes.byref(found)))
        if st == BNX_BUFFER_FULL:
            cap = int(found.value)
            continue
        return np.frombuffer(buf, dtype=PAIR_DTYPE, count=int(found.value)).copy()


_MULTI_LOCK = threading.Lock()
