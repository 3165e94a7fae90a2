"""GPU parity: libqaa (through its C-ABI) against the CPU oracle, element by
element on the same seeded inputs (DESIGN.md §6 tolerances).

Tolerance (BASELINE north_star): |psi_gpu - psi_oracle| <= 1e-10 absolute per
amplitude. Because amplitudes shrink like 2^{-n/2}, we also bound the relative
l2 error ||d|| / ||psi|| <= RTOL_L2 = 1e-11, derived from the rounding budget
K * (n + 4) * eps with K <= 1000, n <= 24.
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


@pytest.fixture()
def ctx(q):
    c = q.Context(0)
    yield c
    c.close()


def assert_close(got, want, atol=ATOL, rtol_l2=RTOL_L2):
    d = np.abs(got - want)
    assert np.max(d) <= atol, f"max abs err {np.max(d):.3e}"
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
    assert rel <= rtol_l2, f"relative l2 err {rel:.3e}"


def instance(n, seed=None):
    if n in (8, 10, 12, 13, 14, 16, 20, 24, 30):
        return cnf.load_instance(n)[0]
    return cnf.random_instance(n, max(1, int(round(4.3 * n))), seed if seed is not None else 1000 + n)


# ------------------------------------------------------------------ K1 / K2
@pytest.mark.parametrize("w64", [0, 1])
@pytest.mark.parametrize("n", [3, 4, 6, 8, 11, 12, 13, 16, 20, 24])
def test_energy_table_exact(q, ctx, orc, n, w64):
    """w64 = 1: the 64-bit kernel (used for n > 32) on the same tables."""
    cl = instance(n)
    ctx.set_option(q.OPT_ENERGY_W64, w64)
    ctx.load_instance(n, cl)
    Eg = ctx.energy_table()
    Eo = orc.energy_table(n, cl)
    assert np.array_equal(Eg.astype(np.uint16), Eo)
    assert ctx.num_solutions() == int((Eo == 0).sum())
    assert ctx.max_energy() == int(Eo.max())


def test_energy_table_paper_instances(ctx, orc):
    for corrected, sol in ((False, 10), (True, 11)):
        n, cl = cnf.paper_instance(corrected)
        ctx.load_instance(n, cl)
        Eg = ctx.energy_table()
        assert np.array_equal(Eg.astype(np.uint16), orc.energy_table(n, cl))
        assert list(np.flatnonzero(Eg == 0)) == [sol]


def test_energy_table_degenerate(ctx, orc):
    n = 5
    cl = [(1, -1, 2), (2, 2, 3), (2, 2, 3), (-5, -5, -5), (1, 2, 3)]
    ctx.load_instance(n, cl)
    assert np.array_equal(ctx.energy_table().astype(np.uint16), orc.energy_table(n, cl))
    ctx.load_instance(n, [])
    assert np.all(ctx.energy_table() == 0) and ctx.num_solutions() == 32


def test_energy_table_n30_sampled(ctx, orc):
    """n = 30 spot check on 4000 random and 2048 leading assignments, every
    sample compared (the full table is test_gpu_configs.py's); the solution is
    the oracle's zero among the samples plus the generator's claim, checked
    against the oracle, not trusted."""
    n = 30
    cl, sol = cnf.load_instance(30)
    ctx.load_instance(n, cl)
    rng = np.random.default_rng(5)
    xs = np.unique(np.concatenate([rng.integers(0, 1 << n, 4000, dtype=np.uint64),
                                   np.array([sol, (1 << n) - 1], dtype=np.uint64)]))
    want = orc.energy_at(n, cl, xs)
    got = np.array([ctx.energy_table(int(x), 1)[0] for x in xs], dtype=np.uint16)
    assert np.array_equal(got, want)
    blk = ctx.energy_table(0, 2048)
    assert np.array_equal(blk.astype(np.uint16), orc.energy_at(n, cl, np.arange(2048, dtype=np.uint64)))
    assert orc.energy_at(n, cl, np.array([sol], dtype=np.uint64))[0] == 0


# ------------------------------------------------------------------ evolution parity
def run_both(q, ctx, orc, n, cl, T, K, schedule=None, psi0=None, row_bits=None, span=None):
    if row_bits is not None:
        ctx.set_option(q.OPT_ROW_BITS, row_bits)
    if span is not None:
        ctx.set_option(q.OPT_STEP_SPANNING, span)
    ctx.load_instance(n, cl)
    E = orc.energy_table(n, cl)
    if psi0 is None:
        ctx.init_uniform()
        psi0 = orc.init_uniform(n)
    else:
        ctx.set_state(psi0)
    ctx.evolve(T, K, schedule)
    got = ctx.state()
    want = orc.evolve(n, E, psi0, T, K, schedule)
    return got, want, E


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11, 12])
def test_resident_parity(q, ctx, orc, n):
    cl = instance(n) if n >= 3 else [(1, 1, -n)]
    psi0 = cnf.random_state(n, n)
    got, want, _ = run_both(q, ctx, orc, n, cl, 3.0, 17, psi0=psi0)
    assert_close(got, want)


@pytest.mark.parametrize("n", [13, 14, 15, 16, 18, 21, 22, 23])
@pytest.mark.parametrize("span", [2, 1, 0])
@pytest.mark.parametrize("variant", ["tma", "reg1", "reg2"])
def test_pass_parity_small(q, ctx, orc, n, span, variant):
    ctx.set_option(q.OPT_KERNEL, 1 if variant == "tma" else 0)
    ctx.set_option(q.OPT_CTAS_PER_SM, 2 if variant == "reg2" else 1)
    cl = instance(n)
    psi0 = cnf.random_state(n, 100 + n)
    sched = np.random.default_rng(n).uniform(0, 1, 5)
    got, want, _ = run_both(q, ctx, orc, n, cl, 2.5, 5, schedule=sched, psi0=psi0, span=span)
    assert_close(got, want)


@pytest.mark.parametrize("n", [13, 14, 16, 18, 20, 21])
@pytest.mark.parametrize("span", [2, 1, 0])
def test_persist_parity(q, ctx, orc, n, span):
    """The persistent evolve (QAA_OPT_PERSIST = 1, for 13 <= n <= 21 with the
    automatic kernel choice): every pass of the plan in one cooperative launch
    with grid barriers, against the oracle (the single-launch engines that take
    precedence at n <= 16 are switched off here)."""
    ctx.set_option(q.OPT_WARPTILE, 0)
    ctx.set_option(q.OPT_CLUSTER, 0)
    ctx.set_option(q.OPT_PERSIST, 1)
    cl = instance(n)
    psi0 = cnf.random_state(n, 200 + n)
    K = 7
    sched = np.random.default_rng(n + 7).uniform(0, 1, K)
    got, want, _ = run_both(q, ctx, orc, n, cl, 2.2, K, schedule=sched, psi0=psi0, span=span)
    assert_close(got, want)
    st = ctx.stats()
    assert st["persist_launches"] == 1 and st["pass_launches"] == 1
    ctx.set_option(q.OPT_PERSIST, 0)
    ctx.reset_stats()
    ctx.set_state(psi0)
    ctx.evolve(2.2, K, sched)
    assert ctx.stats()["persist_launches"] == 0
    assert_close(ctx.state(), want)


@pytest.mark.parametrize("c", [3, 4, 5])
def test_pass_parity_row_bits(q, ctx, orc, c):
    n = 22
    cl = instance(n)
    psi0 = cnf.random_state(n, 7)
    got, want, _ = run_both(q, ctx, orc, n, cl, 1.7, 4, psi0=psi0, row_bits=c)
    assert_close(got, want)
    ctx.set_option(q.OPT_ROW_BITS, 3)


@pytest.mark.parametrize("n,c", [(20, 4), (22, 5), (21, 4)])
def test_row_bits_after_load(q, ctx, orc, n, c):
    """QAA_OPT_ROW_BITS set AFTER load_instance rebuilds the tensor maps, the
    permuted energy tables and the chunk plans before the next evolve
    (n = 21 at c = 4 changes the tile-group count: 2 -> 3 groups)."""
    ctx.set_option(q.OPT_KERNEL, 1)  # TMA kernels (the ones with per-group tables)
    cl = instance(n)
    psi0 = cnf.random_state(n, 11)
    ctx.load_instance(n, cl)
    ctx.set_state(psi0)
    ctx.set_option(q.OPT_ROW_BITS, c)
    ctx.evolve(1.3, 3)
    got = ctx.state()
    want = orc.evolve(n, orc.energy_table(n, cl), psi0, 1.3, 3)
    assert_close(got, want)
    ctx.set_option(q.OPT_ROW_BITS, 3)
    ctx.set_option(q.OPT_KERNEL, 2)


def test_cot_form_large_beta(q, ctx, orc):
    """|beta| > pi/4 selects the cot form (u psi0 + i psi1) on both kernels."""
    for n in (10, 17):
        cl = instance(n)
        psi0 = cnf.random_state(n, 3)
        sched = np.array([0.0, 0.1, 0.5, 0.95, 0.0])
        got, want, _ = run_both(q, ctx, orc, n, cl, 2.0 * 5 * 1.3, 5, schedule=sched, psi0=psi0)  # beta up to 1.3
        assert_close(got, want)


@pytest.mark.parametrize("n", [13, 14, 15, 16])
@pytest.mark.parametrize("K", [1, 2, 7])
def test_cluster_evolve_parity(q, ctx, orc, n, K):
    """13 <= n <= 16: the whole evolution in ONE launch, state resident in the
    registers of a 2^(n-12)-CTA cluster (cluster bits swapped with local bits over
    DSMEM every step) -- against the oracle from a random state, random schedule."""
    ctx.set_option(q.OPT_WARPTILE, 0)
    cl = instance(n)
    psi0 = cnf.random_state(n, 40 + n)
    sched = np.random.default_rng(n * 10 + K).uniform(0, 1, K)
    got, want, _ = run_both(q, ctx, orc, n, cl, 1.1 * K, K, schedule=sched, psi0=psi0)
    assert_close(got, want)
    st = ctx.stats()
    assert st["cluster_launches"] == 1 and st["pass_launches"] == 1


@pytest.mark.parametrize("n,engine", [(13, "cluster"), (16, "cluster"), (13, "warp"), (16, "warp"), (17, "warp"),
                                      (21, "warp"), (13, "quad"), (16, "quad"), (19, "quad")])
def test_small_engines_forms_and_orders(q, ctx, orc, n, engine):
    """The single-launch small-state engines (cluster-resident, n <= 16; warp-tile
    cooperative, n <= 21) with the cot form (|beta| > pi/4), Strang splitting
    (closing half step after the last pass) and the driving term."""
    ctx.set_option(q.OPT_WARPTILE, {"warp": 2, "quad": 3}.get(engine, 0))
    ctx.set_option(q.OPT_CLUSTER, 1 if engine == "cluster" else 0)
    cl = instance(n)
    E = orc.energy_table(n, cl)
    psi0 = cnf.random_state(n, 3)
    sched = np.array([0.0, 0.1, 0.5, 0.95, 0.0])
    got, want, _ = run_both(q, ctx, orc, n, cl, 2.0 * 5 * 1.3, 5, schedule=sched, psi0=psi0)  # beta up to 1.3
    assert_close(got, want)
    ctx.set_option(q.OPT_ORDER, 2)
    ctx.set_state(psi0)
    sched = np.random.default_rng(n).uniform(0, 1, 6)
    ctx.evolve(2.2, 6, sched)
    assert_close(ctx.state(), orc.evolve_strang(n, E, psi0, 2.2, 6, sched))
    ctx.set_option(q.OPT_ORDER, 1)
    ctx.set_driver(0.7, -0.4)
    ctx.set_state(psi0)
    ctx.evolve(1.9, 5, sched[:5])
    assert_close(ctx.state(), orc.evolve_driven(n, E, psi0, 1.9, 5, 0.7, -0.4, sched[:5]))
    assert ctx.stats()["cluster_launches" if engine == "cluster" else "warp_launches"] == 3


@pytest.mark.parametrize("n", [13, 14, 15, 16, 17, 18, 19, 20, 21])
@pytest.mark.parametrize("K", [1, 2, 6])
@pytest.mark.parametrize("wt", [2, 3])
def test_warp_evolve_parity(q, ctx, orc, n, K, wt):
    """13 <= n <= 21: all passes of the cyclic plan in ONE cooperative launch, one
    warp (wt 2) or four warps (wt 3, quad-warp tiles) per 2^9-amplitude tile, grid
    barriers between passes -- against the oracle from a random state, random schedule."""
    ctx.set_option(q.OPT_WARPTILE, wt)  # n > 16: the engine's test range
    cl = instance(n)
    psi0 = cnf.random_state(n, 60 + n)
    sched = np.random.default_rng(n * 7 + K).uniform(0, 1, K)
    got, want, _ = run_both(q, ctx, orc, n, cl, 1.3 * K, K, schedule=sched, psi0=psi0)
    assert_close(got, want)
    st = ctx.stats()
    assert st["warp_launches"] == 1 and st["pass_launches"] == 1


def test_cluster_evolve_matches_pass_kernels(q, orc):
    """n = 16: the cluster-resident launch and the per-pass kernels (QAA_OPT_CLUSTER 0)
    agree to rounding on a 40-step run, and both match the oracle."""
    n, K, T = 16, 40, 5.0
    cl = instance(n)
    out = []
    for cflag in (1, 0):
        with q.Context(0) as c:
            c.set_option(q.OPT_WARPTILE, 0)
            c.set_option(q.OPT_CLUSTER, cflag)
            c.load_instance(n, cl)
            c.init_uniform()
            c.evolve(T, K)
            assert c.stats()["cluster_launches"] == (1 if cflag else 0)
            out.append(c.state())
    want = orc.evolve(n, orc.energy_table(n, cl), orc.init_uniform(n), T, K)
    for got in out:
        assert_close(got, want)
    assert np.max(np.abs(out[0] - out[1])) < 1e-13


def test_config1_n8_full(q, ctx, orc):
    """BASELINE configs[0]: n = 8 unique-solution instance, T = 10, 100 steps."""
    cl, sol = cnf.load_instance(8)
    got, want, E = run_both(q, ctx, orc, 8, cl, 10.0, 100)
    assert_close(got, want)
    ps = ctx.success_prob()
    assert abs(ps - abs(want[sol]) ** 2) < 1e-13


def test_config2_n16_full(q, ctx, orc):
    """BASELINE configs[1]: n = 16, T = 50, 1000 steps (full oracle run)."""
    cl, sol = cnf.load_instance(16)
    got, want, E = run_both(q, ctx, orc, 16, cl, 50.0, 1000)
    assert_close(got, want)
    assert abs(ctx.success_prob() - abs(want[sol]) ** 2) < 1e-12


def test_config3_n24_first_steps(q, ctx, orc):
    """BASELINE configs[2]: n = 24, T = 100, K = 5000: the first 10 steps of that
    schedule (dt = 0.02) against the oracle, element by element."""
    cl, sol = cnf.load_instance(24)
    K, Kp = 5000, 10
    sched = (np.arange(Kp) + 0.5) / K
    got, want, E = run_both(q, ctx, orc, 24, cl, 100.0 / K * Kp, Kp, schedule=sched)
    assert_close(got, want)


# ------------------------------------------------------------------ n = 30 (full size) closed forms
@pytest.fixture(scope="module")
def ctx30(q):
    c = q.Context(0)
    cl, sol = cnf.load_instance(30)
    c.load_instance(30, cl)
    yield c, cl, sol
    c.close()


def test_n30_s_one_closed_form(ctx30, orc):
    """s = 1: psi_K(x) = 2^{-15} e^{-i T E(x)} (sampled x, E from the oracle)."""
    c, cl, sol = ctx30
    c.init_uniform()
    T, K = 0.37, 6
    c.evolve(T, K, np.ones(K))
    rng = np.random.default_rng(1)
    starts = rng.integers(0, (1 << 30) - 64, 40)
    for s0 in starts:
        xs = np.arange(s0, s0 + 64, dtype=np.uint64)
        want = 2.0 ** -15 * np.exp(-1j * T * orc.energy_at(30, cl, xs).astype(float))
        assert_close(c.state(int(s0), 64), want, atol=1e-15, rtol_l2=1e-12)


def test_n30_s_zero_basis_closed_form(ctx30):
    """s = 0 from |x0>: product closed form with Theta = T/2, sampled."""
    c, cl, sol = ctx30
    x0 = 0x2A5A5A5A
    c.init_basis(x0)
    T, K = 1.1, 4
    c.evolve(T, K, np.zeros(K))
    th = T / 2
    same = np.exp(-1j * th) * np.cos(th)
    diff = 1j * np.exp(-1j * th) * np.sin(th)
    rng = np.random.default_rng(2)
    for s0 in list(rng.integers(0, (1 << 30) - 32, 30)) + [x0 - 8]:
        ys = np.arange(s0, s0 + 32, dtype=np.int64)
        flips = np.array([bin(int(y) ^ x0).count("1") for y in ys])
        want = same ** (30 - flips) * diff ** flips
        assert_close(c.state(int(s0), 32), want, atol=1e-15, rtol_l2=1e-12)


def test_n30_uniform_observables_and_norm(ctx30, q):
    """t = 0 closed forms at full size: ||psi||^2 = 1, <H_P> = m/8, <H_B> = 0,
    P_succ = 2^-30; then 8 Trotter steps conserve the norm to 1e-12."""
    c, cl, sol = ctx30
    c.init_uniform()
    m = len(cl)
    assert abs(c.norm2() - 1) < 1e-12
    assert abs(c.energy(1.0) - m / 8) < 1e-10
    assert abs(c.energy(0.0)) < 1e-10
    assert abs(c.success_prob() - 2.0 ** -30) < 1e-20
    c.evolve(0.16, 8, (np.arange(8) + 0.5) / 10000)
    assert abs(c.norm2() - 1) < 1e-12


def test_n30_determinism(ctx30):
    c, cl, sol = ctx30
    outs = []
    for _ in range(2):
        c.init_uniform()
        c.evolve(0.1, 5)
        outs.append(np.concatenate([c.state(0, 4096), c.state(sol - 100, 200), c.state((1 << 30) - 4096, 4096)]))
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------------------------ observables
@pytest.mark.parametrize("n", [6, 10, 16, 21])
def test_observables_parity(q, ctx, orc, n):
    cl = instance(n)
    psi0 = cnf.random_state(n, 11)
    got, want, E = run_both(q, ctx, orc, n, cl, 1.3, 3, psi0=psi0)
    ob = orc.observables(n, E, want)
    assert abs(ctx.norm2() - ob["norm2"]) < 1e-12 * max(1, ob["norm2"])
    assert np.allclose(ctx.sigma_x(), ob["sigma_x"], atol=1e-12, rtol=0)
    for s in (0.0, 0.4, 1.0):
        assert abs(ctx.energy(s) - orc.energy(n, E, want, s)) < 1e-11
    assert abs(ctx.success_prob() - ob["success"]) < 1e-13


def test_success_prob_full_pass_path(q, ctx, orc):
    """Many solutions (|Z| > list cap) -> the full-pass reduction path."""
    n = 18
    cl = [(1, 2, 3)]
    psi0 = cnf.random_state(n, 4)
    got, want, E = run_both(q, ctx, orc, n, cl, 0.5, 2, psi0=psi0)
    assert ctx.num_solutions() == (1 << 18) - (1 << 15)
    assert abs(ctx.success_prob() - orc.observables(n, E, want)["success"]) < 1e-12


def test_unsat_success_zero(q, ctx):
    unsat = [(a * 1, b * 2, c * 3) for a in (1, -1) for b in (1, -1) for c in (1, -1)]
    ctx.load_instance(3, unsat)
    ctx.init_uniform()
    ctx.evolve(5.0, 50)
    assert ctx.success_prob() == 0.0


@pytest.mark.parametrize("n,wt", [(14, 0), (16, 1), (16, 0)])
def test_small_engines_edge_cases(q, ctx, orc, n, wt):
    """The single-launch small-state engines (warp-tile: wt = 1, cluster-resident:
    wt = 0) on the degenerate cases: T = 0 (identity, bit for bit), K = 1, m = 0
    (E = 0, every assignment a solution), s = 1 (closed form 2^{-n/2} e^{-i T E}),
    s = 0 from the uniform state (its H_B eigenvalue-0 state: unchanged)."""
    ctx.set_option(q.OPT_WARPTILE, wt)
    key = "warp_launches" if wt else "cluster_launches"
    cl = instance(n)
    E = orc.energy_table(n, cl)
    ctx.load_instance(n, cl)
    psi0 = cnf.random_state(n, 11)
    ctx.set_state(psi0)
    ctx.evolve(0.0, 3)
    assert np.array_equal(ctx.state(), psi0)
    ctx.set_state(psi0)
    ctx.evolve(0.9, 1)
    assert_close(ctx.state(), orc.evolve(n, E, psi0, 0.9, 1))
    ctx.init_uniform()
    ctx.evolve(0.41, 5, np.ones(5))
    want = 2.0 ** (-n / 2) * np.exp(-1j * 0.41 * E.astype(float))
    assert_close(ctx.state(), want, atol=1e-15, rtol_l2=1e-12)
    ctx.init_uniform()
    ctx.reset_stats()
    ctx.evolve(3.0, 4, np.zeros(4))
    assert_close(ctx.state(), orc.init_uniform(n), atol=1e-15, rtol_l2=1e-12)
    assert ctx.stats()[key] == 1
    ctx.load_instance(n, [])
    ctx.set_state(psi0)
    ctx.evolve(1.0, 3)
    assert_close(ctx.state(), orc.evolve(n, orc.energy_table(n, []), psi0, 1.0, 3))
    assert abs(ctx.success_prob() - ctx.norm2()) < 1e-13


def test_T_zero_identity(q, ctx):
    for n in (9, 20):
        ctx.load_instance(n, instance(n))
        psi0 = cnf.random_state(n, 1)
        ctx.set_state(psi0)
        ctx.evolve(0.0, 3)
        assert np.array_equal(ctx.state(), psi0)


# ------------------------------------------------------------------ error behaviour
def test_error_codes(q, ctx):
    with pytest.raises(q.QaaError) as e:
        ctx.init_uniform()
    assert e.value.status == 4
    with pytest.raises(q.QaaError) as e:
        ctx.load_instance(4, [(1, 2, 5)])
    assert e.value.status == 2
    with pytest.raises(q.QaaError) as e:
        ctx.load_instance(4, [(1, 2, 3)] * 256)
    assert e.value.status == 3
    ctx.load_instance(4, [(1, 2, 3)])
    with pytest.raises(q.QaaError) as e:
        ctx.evolve(1.0, 3)
    assert e.value.status == 4
    ctx.init_uniform()
    for args in ((-1.0, 3), (float("nan"), 3), (1.0, 0)):
        with pytest.raises(q.QaaError) as e:
            ctx.evolve(*args)
        assert e.value.status == 1
    with pytest.raises(q.QaaError) as e:
        ctx.evolve(1.0, 2, [0.5, 1.5])
    assert e.value.status == 1
    with pytest.raises(q.QaaError) as e:
        ctx.energy(1.2)
    assert e.value.status == 1
    assert "outside" in q.qaa_last_error(ctx.ctx)


def test_option_ranges(q, ctx):
    for key, bad in ((q.OPT_SUPER, 65536), (q.OPT_SUPER, -1), (q.OPT_DIAG, 128), (q.OPT_DIAG, -1)):
        with pytest.raises(q.QaaError) as e:
            ctx.set_option(key, bad)
        assert e.value.status == 1
    ctx.set_option(q.OPT_DIAG, 0)
    ctx.set_option(q.OPT_SUPER, 1)


@pytest.mark.parametrize("n", [22, 25])
def test_super_v2_sync_bitwise(q, n):
    """The default L2-blocked step (split-phase write-after-read mbarriers, deferred
    per-warp publish) and the round-1 synchronisation (QAA_OPT_SUPER bit 15) run the
    same per-tile arithmetic: the states after 5 random-schedule steps are equal bit
    for bit (a lost or early-read tile would break this)."""
    cl = instance(n)
    sched = np.random.default_rng(7 * n).uniform(0, 1, 5)
    out = []
    for sup, pub in ((17, 1), (17 | 32768, 1), (17 | 512, 1), (17, 3), (17, 16 + 2)):
        with q.Context(0) as c:
            c.set_option(q.OPT_SUPER, sup)
            c.set_option(q.OPT_SUPER_PUB, pub)
            c.load_instance(n, cl)
            c.set_state(cnf.random_state(n, 5 + n))
            c.evolve(1.7, 5, sched)
            assert c.stats()["super_launches"] == 5
            out.append(c.state())
    assert np.array_equal(out[0].view(np.uint64), out[1].view(np.uint64))
    assert np.array_equal(out[0].view(np.uint64), out[2].view(np.uint64))  # TMA tensor stores (bit 9)
    # batched publish (QAA_OPT_SUPER_PUB 3) and early slot release with batch 2 (16 + 2)
    assert np.array_equal(out[0].view(np.uint64), out[3].view(np.uint64))
    assert np.array_equal(out[0].view(np.uint64), out[4].view(np.uint64))


@pytest.mark.parametrize("n", [22, 25])
def test_super_rev_bitwise_equals_two_pass(q, n):
    """QAA_OPT_SUPER_REV: the L2-blocked pairs fused the other way round
    ([group k rotate/D/rotate][group 0 rotate]) run the same pass sequence, so the
    state after 5 random-schedule steps equals the two-pass plan's bit for bit."""
    cl = instance(n)
    sched = np.random.default_rng(3 * n).uniform(0, 1, 5)
    out = []
    for sup, rev in ((17, 1), (0, 0)):
        with q.Context(0) as c:
            c.set_option(q.OPT_SUPER, sup)
            c.set_option(q.OPT_SUPER_REV, rev)
            c.load_instance(n, cl)
            c.set_state(cnf.random_state(n, 9 + n))
            c.evolve(1.3, 5, sched)
            assert c.stats()["super_launches"] == (5 if sup else 0)
            out.append(c.state())
    assert np.array_equal(out[0].view(np.uint64), out[1].view(np.uint64))


def test_torch_owned_state(q, orc):
    import torch
    c = q.Context(0, n_max=14, torch_state=True)
    cl = instance(14)
    c.load_instance(14, cl)
    c.init_uniform()
    c.evolve(1.0, 4)
    t = c.state_tensor()
    torch.cuda.synchronize()
    want = orc.evolve(14, orc.energy_table(14, cl), orc.init_uniform(14), 1.0, 4)
    assert_close(t.cpu().numpy()[: 1 << 14], want)
    c.close()


@pytest.mark.parametrize("n", [22, 23, 24, 26])
@pytest.mark.parametrize("sup", [17, 19, 49, 81, 83, 16401, 0])
@pytest.mark.parametrize("K", [1, 2, 5])
def test_super_pass_parity(q, ctx, orc, n, sup, K):
    """L2-blocked Trotter steps (QAA_OPT_SUPER bit 0; bit 1 = one consumer group;
    bit 4 = also below 256 chunks, i.e. at these test sizes; bit 5 = dynamic work
    queue instead of the static round robin; bit 6 = tensor-memory exchanges instead
    of shared memory; bit 14 = the producer-warp variant) against the oracle; 0 = the
    two-pass plan."""
    ctx.set_option(q.OPT_SUPER, sup)
    cl = instance(n)
    psi0 = cnf.random_state(n, 31 + n)
    sched = np.random.default_rng(n + K).uniform(0, 1, K)
    got, want, _ = run_both(q, ctx, orc, n, cl, 1.3, K, schedule=sched, psi0=psi0)
    assert_close(got, want)
    st = ctx.stats()
    if sup & 1:
        assert st["pass_launches"] == K + 1  # first pass, K-1 fused pairs, the fused closing pair
        assert st["super_launches"] == K
        assert st["tm_launches"] == (K if sup & 64 else 0)
        assert st["pw_launches"] == (K if (sup & 16384) and not (sup & 64) else 0)


def _full_state(q, n, cl, sup, K, sched, T=1.7, against=None):
    """Evolve in a fresh context; return (clone of the state, stats), or with
    `against` (a device tensor) the chunked comparison (max |d|, bitwise equal)
    without a second full-size copy."""
    import torch
    c = q.Context(0, n_max=n, torch_state=True)
    c.set_option(q.OPT_SUPER, sup)
    c.load_instance(n, cl)
    c.init_uniform()
    c.evolve(T, K, sched)
    st = c.stats()
    torch.cuda.synchronize()
    t = c.state_tensor()
    if against is None:
        out = t.clone()
    else:
        err, eq, step = 0.0, True, 1 << 26
        for i in range(0, t.numel(), step):
            d = t[i:i + step] - against[i:i + step]
            err = max(err, float(d.abs().max()))
            eq = eq and bool(torch.equal(t[i:i + step], against[i:i + step]))
            del d
        out = (err, eq)
    c.close()
    torch.cuda.empty_cache()
    return out, st


@pytest.mark.parametrize("n,sup", [(22, 17), (24, 17), (27, 17), (30, 17), (31, 17), (24, 16401), (30, 16401)])
def test_super_bitwise_equals_two_pass(q, n, sup):
    """The (default, shared-memory) L2-blocked step runs the very per-tile programs of the
    two-pass plan, only fused into one launch over L2-resident chunks (deferred
    loads, cross-CTA release/acquire): at full size the whole state must be
    bitwise identical to the two-pass plan's (itself oracle-parity-tested), which
    catches any lost, duplicated or early-read tile."""
    import torch
    cl = instance(n)
    K = 7
    sched = np.random.default_rng(n).uniform(0, 1, K)
    a, st = _full_state(q, n, cl, sup, K, sched)
    # three tile groups: K - 1 fused [G0][Gk D] pairs + the fused closing pair;
    # four (n = 31): one fused plain pair [G0][Gb] per step. sup = 16401: the
    # producer-warp variant (same per-tile programs, dynamic choice of tiles)
    assert st["super_launches"] == K and st["tm_launches"] == 0
    assert st["pw_launches"] == (K if sup & 16384 else 0)
    (err, eq), st0 = _full_state(q, n, cl, 0, K, sched, against=a)
    assert st0["super_launches"] == 0
    assert eq, err
    # the default (bit 4 clear) picks the L2-blocked step only from n = 28 up
    c2 = q.Context(0)
    c2.load_instance(n, cl)
    c2.init_uniform()
    c2.evolve(1.7, 2, sched[:2])
    assert (c2.stats()["super_launches"] > 0) == (n >= 28)
    c2.close()
    del a
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [22, 24, 27, 30, 31])
def test_super_tm_matches_two_pass(q, n):
    """The tensor-memory L2-blocked step (bit 6) rotates each tile's qubits in
    another order than the two-pass plan (different rounding, not bitwise): at
    full size the whole state must agree to rounding, |d psi| <= 1e-12 max|psi|,
    which a lost, duplicated or early-read tile (an O(|psi|) error) cannot meet."""
    import torch
    cl = instance(n)
    K = 7
    sched = np.random.default_rng(n).uniform(0, 1, K)
    a, st = _full_state(q, n, cl, 17 | 64, K, sched)
    assert st["super_launches"] == K and st["tm_launches"] == K
    scale = float(a.abs().max())
    (err, _), _ = _full_state(q, n, cl, 0, K, sched, against=a)
    assert err <= 1e-12 * scale, (err, scale)
    del a
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [6, 12, 16, 22, 23])
@pytest.mark.parametrize("span", [2, 1, 0])
@pytest.mark.parametrize("kernel", [1, 0])
def test_strang_parity(q, ctx, orc, n, span, kernel):
    """NEXT F4: second-order Strang splitting (QAA_OPT_ORDER = 2) against the
    oracle's literal half-D / X / half-D steps."""
    ctx.set_option(q.OPT_ORDER, 2)
    ctx.set_option(q.OPT_STEP_SPANNING, span)
    ctx.set_option(q.OPT_KERNEL, kernel)
    cl = instance(n)
    ctx.load_instance(n, cl)
    psi0 = cnf.random_state(n, 77)
    ctx.set_state(psi0)
    K = 6
    sched = np.random.default_rng(n).uniform(0, 1, K)
    ctx.evolve(2.2, K, sched)
    want = orc.evolve_strang(n, orc.energy_table(n, cl), psi0, 2.2, K, sched)
    assert_close(ctx.state(), want)
    ctx.set_option(q.OPT_ORDER, 1)


@pytest.mark.parametrize("n,engine", [(6, "cluster"), (8, "cluster"), (10, "cluster"), (11, "cluster"), (12, "cluster")] +
                         [(n, e) for n in (13, 14, 15, 16) for e in ("quad3", "warp2", "cluster", "smem")] +
                         [(18, "warp2"), (18, "quad3"), (21, "quad3")])
@pytest.mark.parametrize("order", [1, 2])
def test_sweep_parity(q, ctx, orc, n, engine, order):
    """NEXT F1: batched T sweep (one CTA per replica up to n = 12 -- per-qubit
    loop below n = 10, 16-amplitude register phases from 10 --; for n = 13..16 one
    register-resident cluster of 2^(n-12) CTAs per replica (default), or with
    QAA_OPT_CLUSTER 0 the shared-memory cluster of 2^(n-13) CTAs with per-bit DSMEM
    phases, or with QAA_OPT_WARPTILE 2 teams of warp-tile CTAs, one replica per team
    at a time -- also n = 18; or with QAA_OPT_WARPTILE 3 teams of quad-warp CTAs,
    n = 13..21) against one oracle run per replica (configs[1]-style sweep T in
    {1,2,5,10,20} at dt = 0.05)."""
    cl = cnf.paper_instance()[1] if n == 6 else instance(n)
    ctx.set_option(q.OPT_WARPTILE, {"quad": 1, "warp2": 2, "quad3": 3}.get(engine, 0))
    ctx.set_option(q.OPT_CLUSTER, 1 if engine == "cluster" else 0)
    ctx.set_option(q.OPT_ORDER, order)
    ctx.load_instance(n, cl)
    Ts = np.array([1.0, 2.0, 5.0, 10.0, 20.0])
    Ks = (Ts / 0.05).astype(np.int64)
    got = ctx.sweep(Ts, Ks)
    E = orc.energy_table(n, cl)
    for T, K, p in zip(Ts, Ks, got):
        ev = orc.evolve if order == 1 else orc.evolve_strang
        want = ev(n, E, orc.init_uniform(n), float(T), int(K))
        assert abs(p - orc.observables(n, E, want)["success"]) < 1e-12
    ctx.set_option(q.OPT_ORDER, 1)


def test_sweep_errors(q, ctx):
    ctx.load_instance(17, instance(17))
    with pytest.raises(q.QaaError):
        ctx.sweep([1.0], [10])  # n > 16
    ctx.load_instance(8, instance(8))
    with pytest.raises(q.QaaError):
        ctx.sweep([1.0], [0])


def test_empty_instance_large(q, ctx, orc):
    """m = 0: E = 0 everywhere, Z = all 2^n assignments (full-pass success path)."""
    n = 20
    ctx.load_instance(n, [])
    assert ctx.num_solutions() == 1 << n and ctx.max_energy() == 0
    psi0 = cnf.random_state(n, 2)
    ctx.set_state(psi0)
    ctx.evolve(1.0, 4)
    want = orc.evolve(n, orc.energy_table(n, []), psi0, 1.0, 4)
    assert_close(ctx.state(), want)
    assert abs(ctx.success_prob() - ctx.norm2()) < 1e-13


def test_large_emax_falls_back(q, ctx, orc):
    """E_max + 1 > TMA_MAX_PHI (64): the register kernels take over (same results)."""
    n = 14
    cl = [(1, 2, 3)] * 70 + cnf.random_instance(n, 30, 5)
    ctx.load_instance(n, cl)
    assert ctx.max_energy() >= 64
    psi0 = cnf.random_state(n, 8)
    ctx.set_state(psi0)
    ctx.evolve(0.7, 4)
    want = orc.evolve(n, orc.energy_table(n, cl), psi0, 0.7, 4)
    assert_close(ctx.state(), want)


@pytest.mark.parametrize("n", [8, 16, 22])
@pytest.mark.parametrize("g", [(0.7, 0.0), (1.2, -0.5)])
def test_driver_parity(q, ctx, orc, n, g):
    """NEXT F4 driving term s(1-s)(gx H_B + gz H_P) against the oracle; energy(s)
    reports the driven H(s)."""
    cl = instance(n)
    ctx.load_instance(n, cl)
    ctx.set_driver(*g)
    psi0 = cnf.random_state(n, 5)
    ctx.set_state(psi0)
    sched = np.random.default_rng(n).uniform(0, 1, 5)
    ctx.evolve(1.9, 5, sched)
    E = orc.energy_table(n, cl)
    want = orc.evolve_driven(n, E, psi0, 1.9, 5, g[0], g[1], sched)
    assert_close(ctx.state(), want)
    s = 0.35
    wb, wp = (1 - s) + g[0] * s * (1 - s), s + g[1] * s * (1 - s)
    ob = orc.observables(n, E, want)
    hb = sum(0.5 * (ob["norm2"] - sx) for sx in ob["sigma_x"])
    assert abs(ctx.energy(s) - (wb * hb + wp * ob["hp"])) < 1e-11
    ctx.set_driver(0.0, 0.0)


@pytest.mark.parametrize("n", [6, 8, 10])
@pytest.mark.parametrize("s", [0.0, 0.3, 0.62, 1.0])
def test_spectrum_vs_dense(q, ctx, n, s):
    """NEXT F3: Lanczos Ritz values of the matrix-free H(s) against numpy's dense
    eigvalsh of H(s) built from Kronecker products (oracle/dense.py) with H_P from
    brute force; Lanczos from one start vector sees each distinct eigenvalue once."""
    from oracle import dense
    from qaa_testutil import brute_force_energy
    cl = cnf.paper_instance()[1] if n == 6 else instance(n)
    ctx.load_instance(n, cl)
    ev, _, it = ctx.spectrum(s, kmax=min(1 << n, 160), nev=3)
    w = np.linalg.eigvalsh(dense.h_s(n, brute_force_energy(n, cl), s))
    distinct = [w[0]]
    for x in w[1:]:
        if x - distinct[-1] > 1e-8:
            distinct.append(x)
    assert np.allclose(ev, distinct[:3], atol=1e-9, rtol=0), (ev, distinct[:3], it)


def test_spectrum_closed_forms_and_overlap(q, ctx):
    """s = 0: H_B has eigenvalues 0, 1, 2 and psi0 is its ground state
    (overlap 1); s = 1: H_P's lowest levels are the two smallest energies."""
    n = 16
    cl, sol = cnf.load_instance(n)
    ctx.load_instance(n, cl)
    ctx.init_uniform()
    ev, ov, _ = ctx.spectrum(0.0, kmax=60, nev=3, overlap=True)
    assert np.allclose(ev, [0.0, 1.0, 2.0], atol=1e-9)
    assert abs(ov - 1.0) < 1e-9
    ev1, _, _ = ctx.spectrum(1.0, kmax=80, nev=2)
    E = ctx.energy_table().astype(int)
    levels = sorted(set(E.tolist()))[:2]
    assert np.allclose(ev1, levels, atol=1e-9)
