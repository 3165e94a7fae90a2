"""Pins of the CPU oracle (oracle/) against things other than itself.

Each test cites what fixes the expected value: the paper's printed instance,
a closed form, a brute-force evaluation of the formula, or the independent
dense-matrix formulation in oracle/dense.py. CPU only (no GPU marker).
"""
import math
from collections import Counter

import numpy as np
import pytest

from inputs import cnf
from oracle import dense
from qaa_testutil import brute_force_energy


# --------------------------------------------------------------------------- E, Z
def test_paper_instance_solutions_bruteforce(oracle_mod):
    """the instance has 'only one solution'. As printed it is index 10;
    the paper's stated one (index 11) is unique only after the clause-11 sign fix
    (R6)."""
    n, cl = cnf.paper_instance()
    E_bf = brute_force_energy(n, cl)
    assert [x for x in range(64) if E_bf[x] == 0] == [10]
    stated = cnf.bits_to_index(cnf.PAPER_STATED_SOLUTION_BITS)
    assert stated == 11 and E_bf[stated] == 1
    n, clc = cnf.paper_instance(corrected=True)
    E_c = brute_force_energy(n, clc)
    assert [x for x in range(64) if E_c[x] == 0] == [11]
    # oracle O-2/O-3 agree with brute force on both
    for clauses, want in ((cl, [10]), (clc, [11])):
        E = oracle_mod.energy_table(6, clauses)
        assert list(oracle_mod.solutions(E)) == want
        assert list(E) == brute_force_energy(6, clauses)


def test_golden_fixtures_match_inputs():
    for name, corrected in (("paper_verbatim.cnf", False), ("paper_corrected.cnf", True)):
        n, cl, comments = cnf.read_dimacs(f"tests/golden/{name}")
        assert (n, [tuple(c) for c in cl]) == (6, cnf.paper_instance(corrected)[1])
        sol = [int(c.split("=")[1]) for c in comments if c.startswith("solution_index")][0]
        E = brute_force_energy(n, cl)
        assert [x for x in range(64) if E[x] == 0] == [sol]


@pytest.mark.parametrize("n,m,seed", [(3, 1, 0), (4, 9, 1), (5, 21, 2), (7, 30, 3), (9, 38, 4), (10, 42, 5)])
def test_energy_table_bruteforce_random(oracle_mod, n, m, seed):
    cl = cnf.random_instance(n, m, seed)
    E = oracle_mod.energy_table(n, cl)
    assert E.dtype == np.uint16 and E.size == 1 << n
    assert list(E) == brute_force_energy(n, cl)
    # sum over all assignments: each 3-distinct-variable clause is violated by 2^(n-3) of them
    assert int(E.astype(np.int64).sum()) == m * 2 ** (n - 3)


def test_energy_table_degenerate_clauses(oracle_mod):
    """Tautologies (x or not x or y) are never violated; repeated literals are
    allowed; duplicates count with multiplicity (R5); m = 0 gives E = 0."""
    n = 4
    cl = [(1, -1, 2), (2, 2, 3), (2, 2, 3), (-4, -4, -4)]
    E = oracle_mod.energy_table(n, cl)
    assert list(E) == brute_force_energy(n, cl)
    assert list(oracle_mod.energy_table(n, [])) == [0] * 16


def test_single_clause_table(oracle_mod):
    """(x1 or x2 or x3), n=3 -> table (1,0,0,0,0,0,0,0) with LSB = x1."""
    assert list(oracle_mod.energy_table(3, [(1, 2, 3)])) == [1, 0, 0, 0, 0, 0, 0, 0]
    assert list(oracle_mod.energy_table(3, [(-1, 2, 3)])) == [0, 1, 0, 0, 0, 0, 0, 0]


def test_energy_monotone_under_clause_addition(oracle_mod):
    cl = cnf.random_instance(8, 30, 11)
    prev = np.zeros(256, dtype=np.int64)
    for k in range(0, 31, 5):
        E = oracle_mod.energy_table(8, cl[:k]).astype(np.int64)
        assert np.all(E >= prev)
        prev = E


def test_energy_table_input_errors(oracle_mod):
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.energy_table(3, [(1, 2, 4)])
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.energy_table(3, [(1, 0, 2)])


def test_checked_in_instances_unique(oracle_mod):
    for n in (8, 10, 12, 13, 14, 16):
        cl, sol = cnf.load_instance(n)
        E = oracle_mod.energy_table(n, cl)
        assert list(oracle_mod.solutions(E)) == [sol]
        if n <= 10:
            assert list(E) == brute_force_energy(n, cl)


# --------------------------------------------------------------------------- psi0 + observables
@pytest.mark.parametrize("n", [1, 2, 5, 6, 11])
def test_init_uniform(oracle_mod, n):
    """psi_g(0) = 2^{-n/2} sum |q>."""
    psi = oracle_mod.init_uniform(n)
    assert np.all(psi.imag == 0)
    assert np.allclose(psi.real, 2.0 ** (-n / 2), rtol=4.5e-16, atol=0)  # within 2 ulp of 2^{-n/2}
    if n % 2 == 0:
        assert np.all(psi.real == 2.0 ** (-n / 2))  # exact power of two


def test_observables_at_t0(oracle_mod):
    """At psi0: <H_P> = m/8 (each 3-distinct-variable clause is violated by 1/8 of
    assignments), <sigma^x_j> = 1 (|+> is the +1 eigenvector), so <H_B> = 0 and
    <H(s)> = s*m/8; P_succ = |Z| / 2^n."""
    n, cl = cnf.paper_instance()
    E = oracle_mod.energy_table(n, cl)
    psi = oracle_mod.init_uniform(n)
    ob = oracle_mod.observables(n, E, psi)
    assert abs(ob["norm2"] - 1) < 1e-15
    assert abs(ob["hp"] - 27 / 8) < 1e-14
    assert np.allclose(ob["sigma_x"], 1.0, atol=1e-15)
    assert abs(ob["success"] - 1 / 64) < 1e-17
    for s in (0.0, 0.25, 1.0):
        assert abs(oracle_mod.energy(n, E, psi, s) - s * 27 / 8) < 1e-14


def test_energy_vs_dense(oracle_mod):
    n = 5
    cl = cnf.random_instance(n, 18, 7)
    E = oracle_mod.energy_table(n, cl)
    psi = cnf.random_state(n, 3)
    diag = brute_force_energy(n, cl)
    for s in (0.0, 0.3, 0.77, 1.0):
        H = dense.h_s(n, diag, s)
        want = float(np.real(np.vdot(psi, H @ psi)))
        assert abs(oracle_mod.energy(n, E, psi, s) - want) < 1e-13
    ob = oracle_mod.observables(n, E, psi)
    for j in range(n):
        X = dense.single_qubit_op(n, j, dense.SX)
        assert abs(ob["sigma_x"][j] - float(np.real(np.vdot(psi, X @ psi)))) < 1e-14
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.energy(n, E, psi, 1.5)


# --------------------------------------------------------------------------- dense checker pins
@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_dense_hb_spectrum(n):
    """H_B = sum (1 - sigma^x)/2 has eigenvalues j with multiplicity C(n, j); the
    uniform superposition is its eigenvalue-0 ground state."""
    H = dense.h_b(n)
    w = np.round(np.linalg.eigvalsh(H), 9)
    assert Counter(w.tolist()) == {float(j): math.comb(n, j) for j in range(n + 1)}
    u = np.full(1 << n, 2.0 ** (-n / 2))
    assert np.allclose(H @ u, 0, atol=1e-14)
    if n == 1:
        assert np.allclose(H, [[0.5, -0.5], [-0.5, 0.5]])


# --------------------------------------------------------------------------- the evolution
@pytest.mark.parametrize("n,m,T,K,seed,sched", [
    (1, 1, 1.0, 3, 0, None), (2, 2, 2.0, 5, 1, None), (3, 5, 3.0, 7, 2, "rand"),
    (5, 20, 4.0, 10, 3, None), (6, 27, 10.0, 20, 4, "rand"), (7, 31, 2.5, 6, 5, None),
])
def test_evolve_vs_dense_product(oracle_mod, n, m, T, K, seed, sched):
    """Whole Trotter product against prod_k expm(-i dt (1-s_k) H_B) expm(-i dt s_k H_P)
    built from Kronecker products (oracle/dense.py) with H_P from brute force."""
    if n >= 3:
        cl = cnf.random_instance(n, m, seed)
    else:  # clauses with repeated variables are legal input for n < 3
        cl = [(1, 1, 1), (-n, 1, -1)][:m]
    E = oracle_mod.energy_table(n, cl)
    diag = brute_force_energy(n, cl)
    psi0 = cnf.random_state(n, seed + 100)
    schedule = np.random.default_rng(seed).uniform(0, 1, K) if sched == "rand" else None
    got = oracle_mod.evolve(n, E, psi0, T, K, schedule)
    want = dense.trotter_product(n, diag, psi0, T, K, schedule)
    assert np.max(np.abs(got - want)) < 1e-13


def test_evolve_paper_instance_vs_dense(oracle_mod):
    n, cl = cnf.paper_instance()
    E = oracle_mod.energy_table(n, cl)
    psi0 = oracle_mod.init_uniform(n)
    got = oracle_mod.evolve(n, E, psi0, 10.0, 100)
    want = dense.trotter_product(n, brute_force_energy(n, cl), psi0, 10.0, 100)
    assert np.max(np.abs(got - want)) < 1e-13


def test_s_zero_from_uniform_is_identity(oracle_mod):
    """psi0 is the eigenvalue-0 eigenvector of H_B and D(s=0) = 1, so s = 0 leaves it fixed."""
    n = 8
    cl, _ = cnf.load_instance(8)
    E = oracle_mod.energy_table(n, cl)
    psi0 = oracle_mod.init_uniform(n)
    out = oracle_mod.evolve(n, E, psi0, 7.0, 50, cnf.constant_schedule(50, 0.0))
    assert np.max(np.abs(out - psi0)) < 1e-15


@pytest.mark.parametrize("x0", [0, 37, 255])
def test_s_zero_basis_state_closed_form(oracle_mod, x0):
    """s = 0 from |x0>: every qubit sees exp(-i Theta (1 - sigma^x)) with Theta = T/2,
    = e^{-i Theta}(cos Theta + i sin Theta sigma^x), so
    psi(y) = prod_j (y_j == x0_j ? e^{-i Theta} cos Theta : i e^{-i Theta} sin Theta)."""
    n, T, K = 8, 3.3, 40
    E = oracle_mod.energy_table(n, cnf.load_instance(8)[0])
    psi0 = np.zeros(1 << n, dtype=np.complex128)
    psi0[x0] = 1.0
    out = oracle_mod.evolve(n, E, psi0, T, K, cnf.constant_schedule(K, 0.0))
    th = T / 2
    same = np.exp(-1j * th) * math.cos(th)
    diff = 1j * np.exp(-1j * th) * math.sin(th)
    y = np.arange(1 << n)
    flips = np.array([bin(v ^ x0).count("1") for v in y])
    want = same ** (n - flips) * diff ** flips
    # rounding budget: K steps x n qubits, a few ulp each (|psi| <= 1)
    assert np.max(np.abs(out - want)) < 4 * K * n * np.finfo(float).eps


def test_s_one_closed_form(oracle_mod):
    """s = 1: X layer is the identity, psi_K(x) = 2^{-n/2} e^{-i T E(x)}."""
    n, T, K = 10, 4.2, 30
    cl, _ = cnf.load_instance(10)
    E = oracle_mod.energy_table(n, cl)
    out = oracle_mod.evolve(n, E, oracle_mod.init_uniform(n), T, K, cnf.constant_schedule(K, 1.0))
    want = 2.0 ** (-n / 2) * np.exp(-1j * T * np.array(brute_force_energy(n, cl), dtype=float))
    assert np.max(np.abs(out - want)) < 1e-14


def test_T_zero_identity(oracle_mod):
    n = 6
    E = oracle_mod.energy_table(n, cnf.paper_instance()[1])
    psi0 = cnf.random_state(n, 9)
    assert np.array_equal(oracle_mod.evolve(n, E, psi0, 0.0, 13), psi0)


def test_norm_conservation(oracle_mod):
    """Each factor is unitary; the raw norm stays 1 to <= 1e-12 (BASELINE north_star)."""
    n, K = 12, 1000
    cl, _ = cnf.load_instance(12)
    E = oracle_mod.energy_table(n, cl)
    out = oracle_mod.evolve(n, E, oracle_mod.init_uniform(n), 20.0, K)
    ob = oracle_mod.observables(n, E, out)
    assert abs(ob["norm2"] - 1.0) < 1e-12


def test_first_order_convergence(oracle_mod):
    """Lie-Trotter is first order: against the exact evolution of i d/dt psi = H(t/T) psi
    (eigendecomposition on 8000 sub-intervals), halving dt halves the error."""
    n, cl = cnf.paper_instance()
    E = oracle_mod.energy_table(n, cl)
    diag = brute_force_energy(n, cl)
    psi0 = oracle_mod.init_uniform(n)
    T = 10.0
    ref = dense.exact_piecewise(n, diag, psi0, T, 1, 8000)
    errs = [np.max(np.abs(oracle_mod.evolve(n, E, psi0, T, K) - ref)) for K in (100, 200, 400)]
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 1.8 < r1 < 2.2 and 1.8 < r2 < 2.2, errs


def test_adiabatic_and_frozen_limits(oracle_mod):
    """large T drives P_succ toward 1; T -> 0 leaves P_succ = |Z|/2^n;
    an UNSAT instance has P_succ = 0."""
    n, cl = cnf.paper_instance()
    E = oracle_mod.energy_table(n, cl)
    psi0 = oracle_mod.init_uniform(n)
    p = [oracle_mod.observables(n, E, oracle_mod.evolve(n, E, psi0, T, int(20 * T)))["success"]
         for T in (1.0, 10.0, 100.0)]
    assert p[0] < p[1] < p[2] and p[2] > 0.9, p
    frozen = oracle_mod.observables(n, E, oracle_mod.evolve(n, E, psi0, 1e-9, 3))["success"]
    assert abs(frozen - 1 / 64) < 1e-9
    unsat = [(1, 2, 3), (1, 2, -3), (1, -2, 3), (1, -2, -3), (-1, 2, 3), (-1, 2, -3), (-1, -2, 3), (-1, -2, -3)]
    Eu = oracle_mod.energy_table(3, unsat)
    assert oracle_mod.observables(3, Eu, oracle_mod.evolve(3, Eu, oracle_mod.init_uniform(3), 5.0, 50))["success"] == 0.0


def test_evolve_usage_errors(oracle_mod):
    E = oracle_mod.energy_table(3, [(1, 2, 3)])
    psi = oracle_mod.init_uniform(3)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.evolve(3, E, psi, -1.0, 3)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.evolve(3, E, psi, 1.0, 0)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.evolve(3, E, psi, 1.0, 2, [0.5, 1.2])


def test_energy_at_matches_table(oracle_mod):
    n = 10
    cl, _ = cnf.load_instance(10)
    E = oracle_mod.energy_table(n, cl)
    xs = np.array([0, 1, 149, 511, 1023, 777], dtype=np.uint64)
    assert list(oracle_mod.energy_at(n, cl, xs)) == [int(E[int(x)]) for x in xs]
    bf = brute_force_energy(n, cl)
    assert list(oracle_mod.energy_at(n, cl, xs)) == [bf[int(x)] for x in xs]


# --------------------------------------------------------------------------- NEXT F4: Strang splitting
@pytest.mark.parametrize("n,m,T,K,seed", [(3, 6, 2.0, 5, 1), (5, 20, 4.0, 9, 2), (6, 27, 10.0, 20, 3)])
def test_strang_vs_dense_product(oracle_mod, n, m, T, K, seed):
    cl = cnf.random_instance(n, m, seed)
    E = oracle_mod.energy_table(n, cl)
    psi0 = cnf.random_state(n, seed)
    sched = np.random.default_rng(seed).uniform(0, 1, K)
    got = oracle_mod.evolve_strang(n, E, psi0, T, K, sched)
    want = dense.strang_product(n, brute_force_energy(n, cl), psi0, T, K, sched)
    assert np.max(np.abs(got - want)) < 1e-13


def test_strang_second_order_convergence(oracle_mod):
    """Strang splitting is second order: halving dt quarters the error against the
    exact evolution (eigendecomposition on 8000 sub-intervals)."""
    n, cl = cnf.paper_instance()
    E = oracle_mod.energy_table(n, cl)
    diag = brute_force_energy(n, cl)
    psi0 = oracle_mod.init_uniform(n)
    ref = dense.exact_piecewise(n, diag, psi0, 10.0, 1, 8000)
    errs = [np.max(np.abs(oracle_mod.evolve_strang(n, E, psi0, 10.0, K) - ref)) for K in (50, 100, 200)]
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.5 < r1 < 4.5 and 3.5 < r2 < 4.5, errs


# --------------------------------------------------------------------------- NEXT F4: driving term
@pytest.mark.parametrize("gx,gz", [(0.7, 0.0), (0.0, -0.4), (1.3, 0.9)])
def test_driven_vs_dense(oracle_mod, gx, gz):
    n, cl = cnf.paper_instance()
    E = oracle_mod.energy_table(n, cl)
    psi0 = cnf.random_state(n, 4)
    sched = np.random.default_rng(2).uniform(0, 1, 12)
    got = oracle_mod.evolve_driven(n, E, psi0, 5.0, 12, gx, gz, sched)
    want = dense.driven_product(n, brute_force_energy(n, cl), psi0, 5.0, 12, gx, gz, sched)
    assert np.max(np.abs(got - want)) < 1e-13


def test_driven_zero_is_eq1(oracle_mod):
    """g = 0 reduces the driven step to Eq. 1 exactly (same arithmetic path values)."""
    n, cl = cnf.paper_instance()
    E = oracle_mod.energy_table(n, cl)
    psi0 = cnf.random_state(n, 6)
    a = oracle_mod.evolve_driven(n, E, psi0, 3.0, 9, 0.0, 0.0)
    b = oracle_mod.evolve(n, E, psi0, 3.0, 9)
    assert np.max(np.abs(a - b)) < 1e-15
