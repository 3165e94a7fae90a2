"""Config-level parity (BASELINE.json configs) at the
sizes and in the launch configuration the bench uses, against the oracle.

* n = 30 (configs[3]): the energy table in FULL (all 2^30 entries) against
  oracle_energy_table, |Z| and the solution from that table (not from the
  instance generator); the first steps of the bench schedule against the oracle
  on >= 4096 sampled amplitudes incl. the solution, default options (the
  L2-blocked step, 512 chunks).
* n = 28: default options (auto L2-blocked step, 256 chunks), the FULL state
  after random-schedule steps against the oracle.
* n = 24 (configs[2], "oracle full"): T = 100, K = 5000, all steps, element by
  element.

Host memory: up to ~40 GiB (n = 30 oracle state, copy and table); the GPU box
has 196 GiB.
"""
import numpy as np
import pytest

from inputs import cnf

pytestmark = pytest.mark.gpu

ATOL = 1e-10
RTOL_L2 = 1e-11


@pytest.fixture(scope="module")
def q():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1103_1399_b200 as q
    return q


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="module")
def n30(orc):
    """The bench instance and its oracle energy table (O-2, 2 GiB uint16)."""
    cl, _ = cnf.load_instance(30)
    E = orc.energy_table(30, cl)
    return cl, E


def assert_close(got, want, atol=ATOL, rtol_l2=RTOL_L2):
    d = np.abs(got - want)
    assert np.max(d) <= atol, f"max abs err {np.max(d):.3e}"
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
    assert rel <= rtol_l2, f"relative l2 err {rel:.3e}"


def test_n30_energy_table_full_and_solution(q, n30):
    """configs[3]: every entry of the 2^30 energy table bit-exact; Z, |Z| = 1 and
    the solution index from the oracle's table (the paper's uniqueness claim for
    the hard instances)."""
    cl, E = n30
    zs = np.flatnonzero(E == 0)
    with q.Context(0) as c:
        c.load_instance(30, cl)
        assert c.num_solutions() == zs.size == 1
        assert c.max_energy() == int(E.max())
        step = 1 << 26
        for s0 in range(0, 1 << 30, step):
            got = c.energy_table(s0, step)
            assert np.array_equal(got.astype(np.uint16), E[s0:s0 + step]), s0
        c.init_uniform()
        assert abs(c.success_prob() - 2.0 ** -30) < 1e-22


def test_n30_bench_schedule_prefix_vs_oracle(q, orc, n30):
    """configs[3]: the first 3 steps of the bench schedule (T = 200, K = 10^4,
    dt = 0.02, midpoint s_k) with DEFAULT options -- the L2-blocked Trotter step
    the bench times -- against the oracle on 4096 random amplitudes, 64-wide
    blocks at the ends and around the solution; P_succ and the norm exactly
    against the oracle's values."""
    cl, E = n30
    sol = int(np.flatnonzero(E == 0)[0])
    K, Kp = 10_000, 3
    sched = (np.arange(Kp) + 0.5) / K
    T = 200.0 / K * Kp
    with q.Context(0) as c:
        c.load_instance(30, cl)
        c.init_uniform()
        c.evolve(T, Kp, sched)
        assert c.stats()["super_launches"] > 0
        rng = np.random.default_rng(30)
        idx = np.unique(np.concatenate([rng.integers(0, 1 << 30, 4096, dtype=np.int64),
                                        np.arange(sol - 32, sol + 32), np.arange(0, 64),
                                        np.arange((1 << 30) - 64, 1 << 30)]))
        got = np.array([c.state(int(i), 1)[0] for i in idx])
        ps, nrm = c.success_prob(), c.norm2()
    want_full = orc.evolve(30, E, orc.init_uniform(30), T, Kp, sched)
    want = want_full[idx]
    assert_close(got, want, atol=1e-10, rtol_l2=1e-11)
    assert abs(ps - abs(want_full[sol]) ** 2) < 1e-20
    assert abs(nrm - 1.0) < 1e-12
    del want_full


def test_n28_default_plan_full_state(q, orc):
    """n = 28 with default options: the auto-selected L2-blocked step (256
    chunks) on a random schedule, the FULL state against the oracle."""
    n, K = 28, 4
    cl = cnf.random_instance(n, int(round(4.3 * n)), 1028)
    E = orc.energy_table(n, cl)
    sched = np.random.default_rng(28).uniform(0, 1, K)
    T = 1.7
    with q.Context(0) as c:
        c.load_instance(n, cl)
        c.init_uniform()
        c.evolve(T, K, sched)
        st = c.stats()
        assert st["super_launches"] == K  # K - 1 fused [G0][Gk D] pairs + the fused closing pair
        got = c.state()
    want = orc.evolve(n, E, orc.init_uniform(n), T, K, sched)
    assert_close(got, want)


@pytest.mark.slow
def test_config2_n24_full_run(q, orc):
    """BASELINE configs[2] in full: n = 24 unique-solution instance, T = 100,
    K = 5000 (dt = 0.02), every step, element by element ("oracle full",
    SURVEY §8(d)); P_succ against the oracle's |psi[sol]|^2."""
    n, T, K = 24, 100.0, 5000
    cl, _ = cnf.load_instance(n)
    E = orc.energy_table(n, cl)
    sol = int(np.flatnonzero(E == 0)[0])
    with q.Context(0) as c:
        c.load_instance(n, cl)
        c.init_uniform()
        c.evolve(T, K)
        got = c.state()
        ps = c.success_prob()
    want = orc.evolve(n, E, orc.init_uniform(n), T, K)
    assert_close(got, want)
    assert abs(ps - abs(want[sol]) ** 2) < 1e-12
