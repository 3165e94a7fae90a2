"""GPU: the largest single-GPU states (n = 31..33, up to 128 GiB), in their own
module so that no other module's context (e.g. test_gpu_parity's module-scoped n = 30
context) still holds device memory when they run."""
import numpy as np
import pytest

from inputs import cnf

pytestmark = pytest.mark.gpu


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


def assert_close(got, want, atol, rtol_l2):
    d = np.abs(got - want)
    assert np.max(d) <= atol, f"max abs err {np.max(d):.3e}"
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
    assert rel <= rtol_l2, f"relative l2 err {rel:.3e}"


@pytest.mark.parametrize("n", [31, 32, 33])
def test_max_size_closed_forms(q, orc, n):
    """Largest single-GPU sizes (n = 33: 128 GiB state, four tile groups):
    s = 1 closed form psi_K(x) = 2^{-n/2} e^{-i T E(x)} on sampled x with E from
    the oracle, and the norm after a few general steps."""
    import gc
    import torch
    gc.collect()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    need = (16 + 1 + 3) * (1 << n) + (4 << 30)
    if free < need:
        pytest.skip(f"needs {need >> 30} GiB free, have {free >> 30}")
    cl, sol = cnf.load_instance(n)
    with q.Context(0) as c:
        c.load_instance(n, cl)
        assert c.num_solutions() == 1 and c.energy_table(sol, 1)[0] == 0
        c.init_uniform()
        T, K = 0.21, 3
        c.evolve(T, K, np.ones(K))
        rng = np.random.default_rng(n)
        for s0 in list(rng.integers(0, (1 << n) - 32, 12)) + [sol - 5]:
            xs = np.arange(s0, s0 + 32, dtype=np.uint64)
            want = 2.0 ** (-n / 2) * np.exp(-1j * T * orc.energy_at(n, cl, xs).astype(float))
            assert_close(c.state(int(s0), 32), want, atol=1e-15, rtol_l2=1e-12)
        c.evolve(0.06, 3)
        assert abs(c.norm2() - 1.0) < 1e-12
