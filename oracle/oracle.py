"""ctypes front end of the C oracle (oracle/qaa_oracle.c). TEST INFRASTRUCTURE ONLY.

Functions mirror SURVEY.md §8(c) O-1..O-8; the arithmetic lives in the C file.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qaa_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# Portable x86-64-v3 (AVX2/FMA) so the .so built here also runs on the GPU box's host.
CFLAGS = ["-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared", "-Wall"]

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no nvcc, no product code)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.oracle_energy_table.argtypes = [ctypes.c_int, ctypes.c_int, P, P]
        L.oracle_energy_at.argtypes = [ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int64, P]
        L.oracle_init_uniform.argtypes = [ctypes.c_int, P]
        L.oracle_evolve.argtypes = [ctypes.c_int, P, P, ctypes.c_double, ctypes.c_int64, P]
        L.oracle_evolve_strang.argtypes = [ctypes.c_int, P, P, ctypes.c_double, ctypes.c_int64, P]
        L.oracle_evolve_driven.argtypes = [ctypes.c_int, P, P, ctypes.c_double, ctypes.c_int64, P,
                                           ctypes.c_double, ctypes.c_double]
        L.oracle_observables.argtypes = [ctypes.c_int, P, P, P]
        L.oracle_energy.argtypes = [ctypes.c_int, P, P, ctypes.c_double, P]
        for f in ("oracle_energy_table", "oracle_energy_at", "oracle_init_uniform", "oracle_evolve",
                  "oracle_evolve_strang", "oracle_evolve_driven", "oracle_observables", "oracle_energy"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st != 0:
        raise OracleError(f"{what} failed with status {st}")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _lits(n: int, clauses) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(clauses, dtype=np.int32).reshape(-1))
    return a


def energy_table(n: int, clauses) -> np.ndarray:
    """O-2: E(x) for x in [0, 2^n), uint16."""
    lits = _lits(n, clauses)
    m = lits.size // 3
    E = np.empty(1 << n, dtype=np.uint16)
    _check(lib().oracle_energy_table(n, m, _ptr(lits) if m else None, _ptr(E)), "energy_table")
    return E


def energy_at(n: int, clauses, xs) -> np.ndarray:
    """O-2 evaluated at the given assignments only (sampling at large n)."""
    lits = _lits(n, clauses)
    m = lits.size // 3
    xs = np.ascontiguousarray(xs, dtype=np.uint64)
    out = np.empty(xs.size, dtype=np.uint16)
    _check(lib().oracle_energy_at(n, m, _ptr(lits) if m else None, _ptr(xs), xs.size, _ptr(out)), "energy_at")
    return out


def solutions(E: np.ndarray) -> np.ndarray:
    """O-3: Z = {x : E(x) = 0}."""
    return np.flatnonzero(E == 0).astype(np.uint64)


def init_uniform(n: int) -> np.ndarray:
    """O-4: psi0 = 2^{-n/2} (complex128)."""
    psi = np.empty(1 << n, dtype=np.complex128)
    _check(lib().oracle_init_uniform(n, _ptr(psi)), "init_uniform")
    return psi


def evolve(n: int, E: np.ndarray, psi: np.ndarray, T: float, K: int, schedule=None) -> np.ndarray:
    """O-5..O-7: K first-order Trotter steps (D then X) applied to a copy of psi."""
    out = np.array(psi, dtype=np.complex128, copy=True, order="C")
    E = np.ascontiguousarray(E, dtype=np.uint16)
    sch = None
    if schedule is not None:
        sch = np.ascontiguousarray(schedule, dtype=np.float64)
        assert sch.size == K
    _check(lib().oracle_evolve(n, _ptr(E), _ptr(out), float(T), int(K),
                               _ptr(sch) if sch is not None else None), "evolve")
    return out


def evolve_strang(n: int, E: np.ndarray, psi: np.ndarray, T: float, K: int, schedule=None) -> np.ndarray:
    """NEXT F4: K second-order Strang steps (half D, X, half D) on a copy of psi."""
    out = np.array(psi, dtype=np.complex128, copy=True, order="C")
    E = np.ascontiguousarray(E, dtype=np.uint16)
    sch = None
    if schedule is not None:
        sch = np.ascontiguousarray(schedule, dtype=np.float64)
        assert sch.size == K
    _check(lib().oracle_evolve_strang(n, _ptr(E), _ptr(out), float(T), int(K),
                                      _ptr(sch) if sch is not None else None), "evolve_strang")
    return out


def evolve_driven(n: int, E: np.ndarray, psi: np.ndarray, T: float, K: int, gx: float, gz: float,
                  schedule=None) -> np.ndarray:
    """NEXT F4: Lie-Trotter steps of H(s) + s(1-s)(gx H_B + gz H_P) on a copy of psi."""
    out = np.array(psi, dtype=np.complex128, copy=True, order="C")
    E = np.ascontiguousarray(E, dtype=np.uint16)
    sch = None
    if schedule is not None:
        sch = np.ascontiguousarray(schedule, dtype=np.float64)
    _check(lib().oracle_evolve_driven(n, _ptr(E), _ptr(out), float(T), int(K),
                                      _ptr(sch) if sch is not None else None, float(gx), float(gz)),
           "evolve_driven")
    return out


def observables(n: int, E: np.ndarray, psi: np.ndarray) -> dict:
    """O-8: raw norm^2, <H_P>, P_succ and <sigma^x_j> for every j."""
    out = np.empty(3 + n, dtype=np.float64)
    E = np.ascontiguousarray(E, dtype=np.uint16)
    psi = np.ascontiguousarray(psi, dtype=np.complex128)
    _check(lib().oracle_observables(n, _ptr(E), _ptr(psi), _ptr(out)), "observables")
    return {"norm2": out[0], "hp": out[1], "success": out[2], "sigma_x": out[3:].copy()}


def energy(n: int, E: np.ndarray, psi: np.ndarray, s: float) -> float:
    """O-8: <psi|H(s)|psi> (raw)."""
    out = np.empty(1, dtype=np.float64)
    E = np.ascontiguousarray(E, dtype=np.uint16)
    psi = np.ascontiguousarray(psi, dtype=np.complex128)
    _check(lib().oracle_energy(n, _ptr(E), _ptr(psi), float(s), _ptr(out)), "energy")
    return float(out[0])


def num_threads() -> int:
    """Threads the OpenMP runtime will use (OMP_NUM_THREADS or all cores)."""
    v = os.environ.get("OMP_NUM_THREADS")
    return int(v) if v else (os.cpu_count() or 1)
