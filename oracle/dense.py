"""Dense-matrix checker, n <= 10. TEST INFRASTRUCTURE ONLY.

An independent second formulation used to pin the loop oracle: it builds the
Hamiltonians of Eq. 1 as explicit 2^n x 2^n matrices from Kronecker
products and exponentiates them with scipy, sharing nothing with
qaa_oracle.c except the conventions (qubit j = bit j of the index, i.e. the
rightmost Kronecker factor is qubit 0, P:76 ordering |q_n ... q_1>).

H_P's diagonal is passed in by the caller (the tests build it from a
pure-Python evaluation of the CNF formula, not from the oracle).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

SX = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=np.complex128)
I2 = np.eye(2, dtype=np.complex128)


def single_qubit_op(n: int, j: int, op: np.ndarray) -> np.ndarray:
    """op acting on qubit j (bit j of the basis index): I x .. x op x .. x I with
    qubit n-1 leftmost and qubit 0 rightmost."""
    M = np.ones((1, 1), dtype=np.complex128)
    for q in range(n - 1, -1, -1):
        M = np.kron(M, op if q == j else I2)
    return M


def h_b(n: int) -> np.ndarray:
    """H_B = sum_j (I - sigma^x_j)/2 (R1)."""
    N = 1 << n
    H = np.zeros((N, N), dtype=np.complex128)
    for j in range(n):
        H += 0.5 * (np.eye(N) - single_qubit_op(n, j, SX))
    return H


def h_p(diag: np.ndarray) -> np.ndarray:
    return np.diag(np.asarray(diag, dtype=np.float64)).astype(np.complex128)


def h_s(n: int, diag: np.ndarray, s: float) -> np.ndarray:
    """Eq. 1: H(s) = (1-s) H_B + s H_P."""
    return (1.0 - s) * h_b(n) + s * h_p(diag)


def trotter_product(n: int, diag, psi0, T: float, K: int, schedule=None) -> np.ndarray:
    """prod_k expm(-i dt (1-s_k) H_B) expm(-i dt s_k H_P) psi0 (D first, then X)."""
    dt = T / K
    HB = h_b(n)
    HP = h_p(diag)
    psi = np.array(psi0, dtype=np.complex128)
    for k in range(K):
        s = schedule[k] if schedule is not None else (k + 0.5) / K
        psi = scipy.linalg.expm(-1j * dt * s * HP) @ psi
        psi = scipy.linalg.expm(-1j * dt * (1.0 - s) * HB) @ psi
    return psi


def driven_product(n: int, diag, psi0, T: float, K: int, gx: float, gz: float, schedule=None) -> np.ndarray:
    """prod_k expm(-i dt wB_k H_B) expm(-i dt wP_k H_P) psi0 with wB = (1-s) + gx s(1-s),
    wP = s + gz s(1-s): the Trotter product of H(s) + s(1-s)(gx H_B + gz H_P)."""
    dt = T / K
    HB = h_b(n)
    HP = h_p(diag)
    psi = np.array(psi0, dtype=np.complex128)
    for k in range(K):
        s = schedule[k] if schedule is not None else (k + 0.5) / K
        wB = (1 - s) + gx * s * (1 - s)
        wP = s + gz * s * (1 - s)
        psi = scipy.linalg.expm(-1j * dt * wP * HP) @ psi
        psi = scipy.linalg.expm(-1j * dt * wB * HB) @ psi
    return psi


def strang_product(n: int, diag, psi0, T: float, K: int, schedule=None) -> np.ndarray:
    """prod_k expm(-i dt s_k H_P / 2) expm(-i dt (1-s_k) H_B) expm(-i dt s_k H_P / 2) psi0."""
    dt = T / K
    HB = h_b(n)
    HP = h_p(diag)
    psi = np.array(psi0, dtype=np.complex128)
    for k in range(K):
        s = schedule[k] if schedule is not None else (k + 0.5) / K
        half = scipy.linalg.expm(-0.5j * dt * s * HP)
        psi = half @ (scipy.linalg.expm(-1j * dt * (1.0 - s) * HB) @ (half @ psi))
    return psi


def exact_piecewise(n: int, diag, psi0, T: float, K: int, substeps: int) -> np.ndarray:
    """Exact propagation of i d/dt psi = H(s(t)) psi with H frozen on each of
    K*substeps sub-intervals at its midpoint s (converges to the continuous
    Schroedinger evolution of P:66 as substeps grows). Used for the
    first-order-convergence pin of the Trotter product."""
    M = K * substeps
    dt = T / M
    HB = h_b(n)
    HP = h_p(diag)
    psi = np.array(psi0, dtype=np.complex128)
    for k in range(M):
        s = (k + 0.5) / M
        w, V = np.linalg.eigh((1.0 - s) * HB + s * HP)
        psi = V @ (np.exp(-1j * dt * w) * (V.conj().T @ psi))
    return psi
