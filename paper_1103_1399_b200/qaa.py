"""ctypes binding of libqaa (include/qaa.h): argument marshalling only.

Every function keeps the C name (``qaa_load_instance`` ...) and raises
``QaaError`` on a non-OK status. A ``Context`` class wraps the same calls.
Device memory for the state can be a torch tensor (PyTorch supplies memory,
streams and process groups; every step of the path runs in libqaa's kernels).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "QaaError", "Context", "lib", "library_path", "STATUS",
    "qaa_create", "qaa_destroy", "qaa_last_error", "qaa_load_instance", "qaa_init_uniform",
    "qaa_init_basis", "qaa_evolve", "qaa_sweep", "qaa_time_energy_table", "qaa_set_driver", "qaa_spectrum", "qaa_success_prob", "qaa_energy", "qaa_norm2", "qaa_sigma_x",
    "qaa_num_solutions", "qaa_max_energy", "qaa_copy_state", "qaa_set_state", "qaa_copy_energy_table",
    "qaa_state_ptr", "qaa_set_option", "qaa_get_stats", "qaa_reset_stats", "qaa_plan_describe",
    "qaa_version", "OPT_ROW_BITS", "OPT_PROFILE", "OPT_STEP_SPANNING", "OPT_CTAS_PER_SM", "OPT_KERNEL", "OPT_TMA_GROUPS", "OPT_SUPER", "OPT_ORDER", "OPT_ENERGY_W64", "OPT_SUPER_GRID", "OPT_SUPER_SPLIT", "OPT_SHARD_SYNC", "OPT_PERSIST", "OPT_DIAG", "OPT_CLUSTER", "OPT_WARPTILE", "OPT_WARP_GRID", "OPT_SUPER_REV", "OPT_SWEEP_TUNE", "OPT_SUPER_PUB",
    "PLAN_RECORD", "SHARD_RECORD", "TorchComm", "qaa_plan_describe_sharded",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "libqaa.so")

STATUS = {0: "QAA_OK", 1: "QAA_E_USAGE", 2: "QAA_E_INPUT", 3: "QAA_E_CAP", 4: "QAA_E_STATE",
          5: "QAA_E_CUDA", 6: "QAA_E_NCCL"}
OPT_ROW_BITS, OPT_PROFILE, OPT_STEP_SPANNING, OPT_CTAS_PER_SM, OPT_KERNEL, OPT_TMA_GROUPS, OPT_SUPER, OPT_ORDER = \
    1, 2, 3, 4, 5, 6, 7, 8
OPT_ENERGY_W64 = 9
OPT_SUPER_GRID = 10
OPT_SUPER_SPLIT = 11
OPT_SHARD_SYNC = 12
OPT_PERSIST = 13
OPT_DIAG = 14
OPT_CLUSTER = 16
OPT_WARPTILE = 17
OPT_WARP_GRID = 18
OPT_SUPER_REV = 19
OPT_SWEEP_TUNE = 20
OPT_SUPER_PUB = 21
PLAN_RECORD = 10
SHARD_RECORD = 10

# symbol list mirrors include/qaa.h (tests check the export table against the header)
EXPORTS = [
    "qaa_create", "qaa_destroy", "qaa_last_error", "qaa_load_instance", "qaa_init_uniform",
    "qaa_init_basis", "qaa_evolve", "qaa_success_prob", "qaa_energy", "qaa_norm2", "qaa_sigma_x",
    "qaa_num_solutions", "qaa_max_energy", "qaa_copy_state", "qaa_set_state", "qaa_copy_energy_table",
    "qaa_state_ptr", "qaa_set_option", "qaa_get_stats", "qaa_reset_stats", "qaa_plan_describe", "qaa_version",
    "qaa_plan_describe_sharded", "qaa_sweep", "qaa_time_energy_table", "qaa_set_driver", "qaa_spectrum",
]


class QaaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)


class qaa_comm(ctypes.Structure):
    _fields_ = [("user", ctypes.c_void_p), ("barrier", BARRIER_FN), ("allgather", ALLGATHER_FN)]


class qaa_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("rank", ctypes.c_int),
                ("world", ctypes.c_int), ("nccl_id", ctypes.c_void_p), ("state", ctypes.c_void_p),
                ("state_bytes", ctypes.c_size_t), ("comm", ctypes.POINTER(qaa_comm))]


class TorchComm:
    """qaa_comm over a torch.distributed process group (gloo for host bytes).
    Keeps the ctypes callback objects alive for the life of the context."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self._b = BARRIER_FN(self._barrier)
        self._a = ALLGATHER_FN(self._allgather)
        self.struct = qaa_comm(None, self._b, self._a)
        self.calls = {"barrier": 0, "allgather": 0}  # how often libqaa called back (tests)

    def _barrier(self, user):
        self.calls["barrier"] += 1
        try:
            self.dist.barrier(group=self.group)
            return 0
        except Exception:  # pragma: no cover
            return 1

    def _allgather(self, user, send, recv, nbytes):
        self.calls["allgather"] += 1
        try:
            import torch
            mine = torch.frombuffer(bytearray(ctypes.string_at(send, nbytes)), dtype=torch.uint8) if nbytes else \
                torch.zeros(0, dtype=torch.uint8)
            outs = [torch.zeros(nbytes, dtype=torch.uint8) for _ in range(self.world)]
            self.dist.all_gather(outs, mine, group=self.group)
            blob = b"".join(bytes(o.numpy().tobytes()) for o in outs)
            ctypes.memmove(recv, blob, len(blob))
            return 0
        except Exception:  # pragma: no cover
            return 1


class qaa_stats(ctypes.Structure):
    _fields_ = [("evolve_calls", ctypes.c_int64), ("trotter_steps", ctypes.c_int64),
                ("pass_launches", ctypes.c_int64), ("other_launches", ctypes.c_int64),
                ("passes_per_step_num", ctypes.c_int64), ("passes_per_step_den", ctypes.c_int64),
                ("pass_kernel_ms", ctypes.c_double), ("pass_kernels_timed", ctypes.c_int64),
                ("bytes_per_pass", ctypes.c_int64), ("amps_local", ctypes.c_int64),
                ("n", ctypes.c_int), ("n_local", ctypes.c_int), ("groups", ctypes.c_int),
                ("tile_bits", ctypes.c_int), ("row_bits", ctypes.c_int),
                ("kernel_launches_total", ctypes.c_int64), ("super_launches", ctypes.c_int64),
                ("super_kernel_ms", ctypes.c_double), ("super_kernels_timed", ctypes.c_int64),
                ("tm_launches", ctypes.c_int64), ("persist_launches", ctypes.c_int64), ("pw_launches", ctypes.c_int64),
                ("tm_diag", ctypes.c_uint64 * 8), ("cluster_launches", ctypes.c_int64), ("warp_launches", ctypes.c_int64)]

    def as_dict(self):
        return {f: (list(getattr(self, f)) if f == "tm_diag" else getattr(self, f)) for f, _ in self._fields_}


_lib = None


def lib():
    """Load libqaa.so. No fallback: a missing library is an error."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise ImportError(f"libqaa.so not built at {library_path}: run __graft_entry__.build() "
                              "(python -m paper_1103_1399_b200.build); there is no CPU fallback")
        L = ctypes.CDLL(library_path)
        P, I, I64, U64, D, S = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64,
                                ctypes.c_double, ctypes.c_size_t)
        sig = {
            "qaa_create": ([ctypes.POINTER(qaa_config), ctypes.POINTER(P)], I),
            "qaa_destroy": ([P], None),
            "qaa_last_error": ([P], ctypes.c_char_p),
            "qaa_load_instance": ([P, I, I, P], I),
            "qaa_init_uniform": ([P], I),
            "qaa_init_basis": ([P, U64], I),
            "qaa_evolve": ([P, D, I64, P], I),
            "qaa_success_prob": ([P, ctypes.POINTER(D)], I),
            "qaa_energy": ([P, D, ctypes.POINTER(D)], I),
            "qaa_norm2": ([P, ctypes.POINTER(D)], I),
            "qaa_sigma_x": ([P, P], I),
            "qaa_num_solutions": ([P, ctypes.POINTER(U64)], I),
            "qaa_max_energy": ([P, ctypes.POINTER(ctypes.c_uint32)], I),
            "qaa_copy_state": ([P, U64, U64, P], I),
            "qaa_set_state": ([P, U64, U64, P], I),
            "qaa_copy_energy_table": ([P, U64, U64, P], I),
            "qaa_state_ptr": ([P, ctypes.POINTER(P), ctypes.POINTER(U64)], I),
            "qaa_set_option": ([P, I, I64], I),
            "qaa_get_stats": ([P, ctypes.POINTER(qaa_stats)], I),
            "qaa_reset_stats": ([P], I),
            "qaa_plan_describe": ([I, I, I, I64, P, I64, ctypes.POINTER(I64)], I),
            "qaa_plan_describe_sharded": ([I, I, I, I64, P, I64, ctypes.POINTER(I64)], I),
            "qaa_sweep": ([P, I, P, P, P], I),
            "qaa_time_energy_table": ([P, I, ctypes.POINTER(D)], I),
            "qaa_set_driver": ([P, D, D], I),
            "qaa_spectrum": ([P, D, I, I, P, ctypes.POINTER(D), ctypes.POINTER(I)], I),
            "qaa_version": ([], ctypes.c_char_p),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _ = S
        _lib = L
    return _lib


def _check(ctx_ptr, st: int):
    if st != 0:
        msg = lib().qaa_last_error(ctx_ptr).decode() if ctx_ptr else ""
        raise QaaError(st, msg)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------- C-named functions
def qaa_create(device: int = 0, stream: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
               state_ptr: int = 0, state_bytes: int = 0, comm: Optional["TorchComm"] = None):
    cfg = qaa_config(device, stream or None, rank, world, None, state_ptr or None, state_bytes,
                     ctypes.pointer(comm.struct) if comm is not None else None)
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        cfg.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    out = ctypes.c_void_p()
    st = lib().qaa_create(ctypes.byref(cfg), ctypes.byref(out))
    if st != 0:
        msg = lib().qaa_last_error(out).decode() if out.value else ""
        if out.value:
            lib().qaa_destroy(out)
        raise QaaError(st, msg)
    return out


def qaa_destroy(ctx):
    lib().qaa_destroy(ctx)


def qaa_last_error(ctx) -> str:
    return lib().qaa_last_error(ctx).decode()


def _lits(clauses) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(clauses, dtype=np.int32).reshape(-1))
    if a.size % 3:
        raise ValueError("clauses must have 3 literals each")
    return a


def qaa_load_instance(ctx, n: int, clauses):
    lits = _lits(clauses)
    m = lits.size // 3
    _check(ctx, lib().qaa_load_instance(ctx, int(n), int(m), _dptr(lits) if m else None))


def qaa_init_uniform(ctx):
    _check(ctx, lib().qaa_init_uniform(ctx))


def qaa_init_basis(ctx, x: int):
    _check(ctx, lib().qaa_init_basis(ctx, int(x)))


def qaa_evolve(ctx, T: float, steps: int, schedule: Optional[Sequence[float]] = None):
    sch = None
    if schedule is not None:
        sch = np.ascontiguousarray(schedule, dtype=np.float64)
        if sch.size != steps:
            raise ValueError("schedule must have `steps` entries")
    _check(ctx, lib().qaa_evolve(ctx, float(T), int(steps), _dptr(sch) if sch is not None else None))


def _scalar(fn, ctx, *args):
    out = ctypes.c_double()
    _check(ctx, fn(ctx, *args, ctypes.byref(out)))
    return out.value


def qaa_success_prob(ctx) -> float:
    return _scalar(lib().qaa_success_prob, ctx)


def qaa_energy(ctx, s: float) -> float:
    return _scalar(lib().qaa_energy, ctx, float(s))


def qaa_norm2(ctx) -> float:
    return _scalar(lib().qaa_norm2, ctx)


def qaa_sigma_x(ctx, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.float64)
    _check(ctx, lib().qaa_sigma_x(ctx, _dptr(out)))
    return out


def qaa_sweep(ctx, T, K) -> np.ndarray:
    """F1: P_succ of independent evolutions (T[r], K[r]) of the uniform state, one launch."""
    Ta = np.ascontiguousarray(T, dtype=np.float64)
    Ka = np.ascontiguousarray(K, dtype=np.int64)
    assert Ta.size == Ka.size
    out = np.zeros(Ta.size, dtype=np.float64)
    _check(ctx, lib().qaa_sweep(ctx, int(Ta.size), _dptr(Ta), _dptr(Ka), _dptr(out)))
    return out


def qaa_spectrum(ctx, s: float, kmax: int = 64, nev: int = 3, overlap: bool = False):
    """F3: (nev smallest Ritz values of H(s), ground-state overlap or None, iterations)."""
    ev = np.zeros(nev, dtype=np.float64)
    ov = ctypes.c_double()
    it = ctypes.c_int()
    _check(ctx, lib().qaa_spectrum(ctx, float(s), int(kmax), int(nev), _dptr(ev),
                                   ctypes.byref(ov) if overlap else None, ctypes.byref(it)))
    return ev, (ov.value if overlap else None), it.value


def qaa_set_driver(ctx, gx: float, gz: float):
    """F4 driving term s(1-s)(gx H_B + gz H_P) added to Eq. 1."""
    _check(ctx, lib().qaa_set_driver(ctx, float(gx), float(gz)))


def qaa_time_energy_table(ctx, reps: int = 5) -> float:
    """F2: average device ms to recompute the energy table (the paper's kernel)."""
    out = ctypes.c_double()
    _check(ctx, lib().qaa_time_energy_table(ctx, int(reps), ctypes.byref(out)))
    return out.value


def qaa_num_solutions(ctx) -> int:
    out = ctypes.c_uint64()
    _check(ctx, lib().qaa_num_solutions(ctx, ctypes.byref(out)))
    return out.value


def qaa_max_energy(ctx) -> int:
    out = ctypes.c_uint32()
    _check(ctx, lib().qaa_max_energy(ctx, ctypes.byref(out)))
    return out.value


def qaa_copy_state(ctx, first: int, count: int, out: Optional[np.ndarray] = None) -> np.ndarray:
    if out is None:
        out = np.zeros(count, dtype=np.complex128)
    assert out.dtype == np.complex128 and out.flags.c_contiguous and out.size >= count
    _check(ctx, lib().qaa_copy_state(ctx, int(first), int(count), _dptr(out)))
    return out


def qaa_set_state(ctx, first: int, values: np.ndarray):
    v = np.ascontiguousarray(values, dtype=np.complex128)
    _check(ctx, lib().qaa_set_state(ctx, int(first), int(v.size), _dptr(v)))


def qaa_copy_energy_table(ctx, first: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint8)
    _check(ctx, lib().qaa_copy_energy_table(ctx, int(first), int(count), _dptr(out)))
    return out


def qaa_state_ptr(ctx):
    p = ctypes.c_void_p()
    n = ctypes.c_uint64()
    _check(ctx, lib().qaa_state_ptr(ctx, ctypes.byref(p), ctypes.byref(n)))
    return p.value, n.value


def qaa_set_option(ctx, key: int, value: int):
    _check(ctx, lib().qaa_set_option(ctx, int(key), int(value)))


def qaa_get_stats(ctx) -> dict:
    s = qaa_stats()
    _check(ctx, lib().qaa_get_stats(ctx, ctypes.byref(s)))
    return s.as_dict()


def qaa_reset_stats(ctx):
    _check(ctx, lib().qaa_reset_stats(ctx))


def qaa_plan_describe(n_local: int, row_bits: int = 3, step_spanning: int = 1, K: int = 1, cap: int = None):
    """Host-only pass plan: array of shape (passes, PLAN_RECORD) int32."""
    cnt = ctypes.c_int64()
    st = lib().qaa_plan_describe(int(n_local), int(row_bits), int(step_spanning), int(K), None, 0,
                                 ctypes.byref(cnt))
    if st != 0:
        raise QaaError(st, "plan_describe")
    cap = cnt.value if cap is None else cap
    rec = np.zeros((cap, PLAN_RECORD), dtype=np.int32)
    st = lib().qaa_plan_describe(int(n_local), int(row_bits), int(step_spanning), int(K), _dptr(rec), cap,
                                 ctypes.byref(cnt))
    if st != 0:
        raise QaaError(st, "plan_describe")
    return rec[: min(cap, cnt.value)]


def qaa_plan_describe_sharded(n: int, world: int, row_bits: int = 3, K: int = 1):
    """Host-only sharded pass plan: array of shape (passes, SHARD_RECORD) int32."""
    cnt = ctypes.c_int64()
    st = lib().qaa_plan_describe_sharded(int(n), int(world), int(row_bits), int(K), None, 0, ctypes.byref(cnt))
    if st != 0:
        raise QaaError(st, "plan_describe_sharded")
    rec = np.zeros((cnt.value, SHARD_RECORD), dtype=np.int32)
    st = lib().qaa_plan_describe_sharded(int(n), int(world), int(row_bits), int(K), _dptr(rec), cnt.value,
                                         ctypes.byref(cnt))
    if st != 0:
        raise QaaError(st, "plan_describe_sharded")
    return rec


def qaa_version() -> str:
    return lib().qaa_version().decode()


# ----------------------------------------------------------------- object wrapper
class Context:
    """One libqaa context on one GPU. If `torch_state` is True the state buffer
    is a torch tensor (allocated lazily for 2^n_max amplitudes)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, n_max: Optional[int] = None, torch_state: bool = False,
                 comm: Optional[TorchComm] = None):
        self._tensor = None
        self._comm = comm
        state_ptr, state_bytes = 0, 0
        if torch_state:
            import torch
            if n_max is None:
                raise ValueError("torch_state needs n_max")
            L = n_max - (world.bit_length() - 1)
            self._tensor = torch.empty(1 << L, dtype=torch.complex128, device=f"cuda:{device}")
            state_ptr, state_bytes = self._tensor.data_ptr(), self._tensor.numel() * 16
            if stream is None:
                stream = torch.cuda.current_stream(device).cuda_stream
        self.ctx = qaa_create(device, stream or 0, rank, world, nccl_id, state_ptr, state_bytes, comm)
        self.rank, self.world = rank, world
        self.n = None

    def close(self):
        if self.ctx is not None:
            qaa_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def load_instance(self, n, clauses):
        qaa_load_instance(self.ctx, n, clauses)
        self.n = n

    def init_uniform(self):
        qaa_init_uniform(self.ctx)

    def init_basis(self, x):
        qaa_init_basis(self.ctx, x)

    def evolve(self, T, steps, schedule=None):
        qaa_evolve(self.ctx, T, steps, schedule)

    def success_prob(self):
        return qaa_success_prob(self.ctx)

    def energy(self, s):
        return qaa_energy(self.ctx, s)

    def norm2(self):
        return qaa_norm2(self.ctx)

    def sigma_x(self):
        return qaa_sigma_x(self.ctx, self.n)

    def spectrum(self, s, kmax=64, nev=3, overlap=False):
        return qaa_spectrum(self.ctx, s, kmax, nev, overlap)

    def set_driver(self, gx, gz):
        qaa_set_driver(self.ctx, gx, gz)

    def time_energy_table(self, reps=5):
        return qaa_time_energy_table(self.ctx, reps)

    def sweep(self, T, K):
        return qaa_sweep(self.ctx, T, K)

    def num_solutions(self):
        return qaa_num_solutions(self.ctx)

    def max_energy(self):
        return qaa_max_energy(self.ctx)

    def state(self, first=0, count=None):
        count = (1 << self.n) - first if count is None else count
        return qaa_copy_state(self.ctx, first, count)

    def set_state(self, values, first=0):
        qaa_set_state(self.ctx, first, values)

    def energy_table(self, first=0, count=None):
        count = (1 << self.n) - first if count is None else count
        return qaa_copy_energy_table(self.ctx, first, count)

    def set_option(self, key, value):
        qaa_set_option(self.ctx, key, value)

    def stats(self):
        return qaa_get_stats(self.ctx)

    def reset_stats(self):
        qaa_reset_stats(self.ctx)

    def state_tensor(self):
        """Zero-copy torch view of the local state (complex128)."""
        if self._tensor is not None:
            return self._tensor[: 1 << (self.n - 0)] if self.n is not None else self._tensor
        raise RuntimeError("state is library-owned; use Context(torch_state=True)")
