"""Sharded (multi-rank) path: host plumbing on CPU with gloo (world 2), and
the full sharded evolution with 2/4/8 ranks sharing one GPU (CUDA IPC peer
stores between processes), compared with the single-process oracle."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from inputs import cnf

import qaa_shard_worker as W


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_torchcomm_callbacks_gloo_world2():
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(W.comm_worker, args=(world, free_port(), d), nprocs=world, join=True)
        for r in range(world):
            got = np.load(os.path.join(d, f"comm{r}.npy"))
            assert list(got) == [0, 1, 2, 3, 4, 10, 11, 12, 13, 14]


@pytest.mark.gpu
@pytest.mark.parametrize("n,world,K,fused,hostsync", [(16, 2, 5, 0, 0), (17, 4, 4, 0, 0), (18, 8, 3, 0, 0),
                                                      (22, 2, 4, 0, 0), (24, 4, 3, 0, 0), (24, 2, 3, 1, 0),
                                                      (24, 4, 4, 1, 0), (25, 8, 3, 1, 0), (24, 4, 3, 1, 1),
                                                      (18, 8, 3, 0, 1)])
def test_sharded_evolution_parity(n, world, K, fused, hostsync):
    """fused = 1: three local tile groups with the [group 0][group 1 + layout
    swap] pass pair of every phase as one L2-blocked launch (QAA_OPT_SUPER 17:
    forced below the 256-chunk threshold at these test sizes). hostsync = 0
    (default): the per-phase barrier runs on the device, so evolve makes no host
    collective call at all; 1: stream sync + qaa_comm barrier per phase."""
    from oracle import oracle
    import paper_1103_1399_b200 as q
    cl = cnf.load_instance(n)[0] if os.path.exists(cnf.instance_path(n)) else cnf.random_instance(n, 4 * n, n)
    T = 1.9
    sched = np.random.default_rng(n).uniform(0, 1, K)
    psi0 = cnf.random_state(n, 5)
    s_values = [0.0, 0.3, 1.0]
    with tempfile.TemporaryDirectory() as d:
        opts = {q.OPT_SUPER: 17} if fused else {}
        opts[q.OPT_SHARD_SYNC] = hostsync
        mp.spawn(W.shard_worker, args=(world, free_port(), d, n, cl, T, K, sched, psi0, s_values, opts),
                 nprocs=world, join=True)
        res = [np.load(os.path.join(d, f"rank{r}.npy"), allow_pickle=True).item() for r in range(world)]
    for r in res:
        assert (r["super_launches"] == K) if fused else (r["super_launches"] == 0)
        assert r["host_calls"]["allgather"] == 0
        assert (r["host_calls"]["barrier"] > 0) if hostsync else (r["host_calls"]["barrier"] == 0)
    got = np.concatenate([r["state"] for r in res])
    E = oracle.energy_table(n, cl)
    want = oracle.evolve(n, E, psi0, T, K, sched)
    assert np.max(np.abs(got - want)) < 1e-10
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-11
    assert np.array_equal(np.concatenate([r["E"] for r in res]).astype(np.uint16), E)
    ob = oracle.observables(n, E, want)
    for r in res:  # every rank reports the global values
        assert abs(r["norm2"] - ob["norm2"]) < 1e-12 * ob["norm2"]
        assert abs(r["success"] - ob["success"]) < 1e-13
        assert np.allclose(r["sigma_x"], ob["sigma_x"], atol=1e-12, rtol=0)
        for s, e in zip(s_values, r["energy"]):
            assert abs(e - oracle.energy(n, E, want, s)) < 1e-11
        assert r["nsol"] == int((E == 0).sum()) and r["emax"] == int(E.max())


@pytest.mark.gpu
def test_sharded_four_groups_full_state():
    """The FOUR-local-tile-group sharded plan -- the geometry the n = 32/33/34
    multi-GPU configs use (fused [group 0][group P-2 + layout swap] launches, the
    top group's D pass over both shard buffers) -- at a size whose full state the
    host holds: n = 28 over 2 ranks with 32-amplitude (512-byte) rows, so L = 27
    splits into 4 tile groups. The whole gathered state and the observables
    against the oracle."""
    from oracle import oracle
    import paper_1103_1399_b200 as q
    n, world, K, T = 28, 2, 3, 1.9
    cl = cnf.random_instance(n, int(round(4.3 * n)), 2028)
    sched = np.random.default_rng(n).uniform(0, 1, K)
    with tempfile.TemporaryDirectory() as d:
        opts = {q.OPT_ROW_BITS: 5, q.OPT_SUPER: 17}
        mp.spawn(W.shard_worker, args=(world, free_port(), d, n, cl, T, K, sched, None, [0.5], opts),
                 nprocs=world, join=True)
        res = [np.load(os.path.join(d, f"rank{r}.npy"), allow_pickle=True).item() for r in range(world)]
    for r in res:
        assert r["groups"] == 4
        assert r["super_launches"] == K  # one fused layout-swap launch per phase
    got = np.concatenate([r["state"] for r in res])
    E = oracle.energy_table(n, cl)
    want = oracle.evolve(n, E, oracle.init_uniform(n), T, K, sched)
    assert np.max(np.abs(got - want)) < 1e-10
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-11
    ob = oracle.observables(n, E, want)
    for r in res:
        assert abs(r["norm2"] - ob["norm2"]) < 1e-12
        assert abs(r["success"] - ob["success"]) < 1e-13
        assert np.allclose(r["sigma_x"], ob["sigma_x"], atol=1e-12, rtol=0)


@pytest.mark.gpu
def test_sharded_uniform_start_paper_config():
    """configs[0]-like run sharded over 2 ranks: n = 16 instance, uniform start."""
    from oracle import oracle
    n, world, K, T = 16, 2, 40, 5.0
    cl, sol = cnf.load_instance(n)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(W.shard_worker, args=(world, free_port(), d, n, cl, T, K, None, None, [1.0]),
                 nprocs=world, join=True)
        res = [np.load(os.path.join(d, f"rank{r}.npy"), allow_pickle=True).item() for r in range(world)]
    got = np.concatenate([r["state"] for r in res])
    want = oracle.evolve(n, oracle.energy_table(n, cl), oracle.init_uniform(n), T, K)
    assert np.max(np.abs(got - want)) < 1e-10
    assert abs(res[0]["success"] - abs(want[sol]) ** 2) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("n,world", [(32, 2)])
def test_sharded_four_groups_closed_form(n, world):
    """Sharded with four local tile groups (2^31 amplitudes per rank, the
    per-GPU size of the n = 32/33/34 multi-GPU configs), both ranks on one GPU:
    s = 1 closed form psi_K(x) = 2^{-n/2} e^{-i T E(x)} on sampled x (E from the
    oracle) through the fused [group 0][group 2 + layout swap] launches, and the
    norm after general steps."""
    import torch
    from oracle import oracle
    free, _ = torch.cuda.mem_get_info()
    need = world * (2 * 16 + 6) * (1 << (n - 1)) + (8 << 30)
    if free < need:
        pytest.skip(f"needs {need >> 30} GiB free on one GPU, have {free >> 30}")
    cl = cnf.load_instance(n)[0]
    T, K = 0.23, 3
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(W.shard_closed_form_worker, args=(world, free_port(), d, n, cl, T, K, None),
                 nprocs=world, join=True)
        res = [np.load(os.path.join(d, f"rank{r}.npy"), allow_pickle=True).item() for r in range(world)]
    for r in res:
        assert r["super_launches"] > 0
        assert abs(r["norm2"] - 1.0) < 1e-12
        for s0, got in r["samples"].items():
            xs = np.arange(s0, s0 + 32, dtype=np.uint64)
            want = 2.0 ** (-n / 2) * np.exp(-1j * T * oracle.energy_at(n, cl, xs).astype(float))
            assert np.max(np.abs(got - want)) < 1e-15
