"""Worker bodies for the multi-process tests (imported by spawned children)."""
import ctypes
import os

import numpy as np


def _init(rank, world, port):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    return dist


def comm_worker(rank, world, port, outdir):
    """CPU: TorchComm's C callbacks (as libqaa calls them) across gloo ranks."""
    dist = _init(rank, world, port)
    from paper_1103_1399_b200.qaa import TorchComm
    comm = TorchComm()
    send = (ctypes.c_uint8 * 5)(*[rank * 10 + i for i in range(5)])
    recv = (ctypes.c_uint8 * (5 * world))()
    assert comm.struct.allgather(None, ctypes.addressof(send), ctypes.addressof(recv), 5) == 0
    assert comm.struct.barrier(None) == 0
    np.save(os.path.join(outdir, f"comm{rank}.npy"), np.frombuffer(bytes(recv), dtype=np.uint8))
    dist.destroy_process_group()


def shard_worker(rank, world, port, outdir, n, clauses, T, K, schedule, psi0, s_values, opts=None):
    """GPU: one rank of a sharded evolution (all ranks may share one GPU)."""
    import torch
    dist = _init(rank, world, port)
    torch.cuda.set_device(0)
    import paper_1103_1399_b200 as q
    comm = q.TorchComm()
    ctx = q.Context(0, rank=rank, world=world, comm=comm)
    for key, val in (opts or {}).items():
        ctx.set_option(key, val)
    ctx.load_instance(n, clauses)
    L = n - (world.bit_length() - 1)
    if psi0 is None:
        ctx.init_uniform()
    else:
        ctx.set_state(psi0)  # each rank copies the part it owns
    before = dict(comm.calls)
    ctx.evolve(T, K, schedule)
    host_calls = {k: comm.calls[k] - before[k] for k in before}  # during evolve (no sync yet)
    local = ctx.state(rank << L, 1 << L)
    res = {"state": local, "super_launches": ctx.stats()["super_launches"], "groups": ctx.stats()["groups"],
           "host_calls": host_calls,
           "success": ctx.success_prob(), "norm2": ctx.norm2(),
           "sigma_x": ctx.sigma_x(), "energy": np.array([ctx.energy(s) for s in s_values]),
           "nsol": ctx.num_solutions(), "emax": ctx.max_energy(), "E": ctx.energy_table(rank << L, 1 << L)}
    np.save(os.path.join(outdir, f"rank{rank}.npy"), res, allow_pickle=True)
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


def shard_closed_form_worker(rank, world, port, outdir, n, clauses, T, K, opts=None):
    """GPU: sharded s = 1 run at a large size; returns sampled local amplitudes
    (global indices) and the norm after a few general steps -- no full copy."""
    import torch
    dist = _init(rank, world, port)
    torch.cuda.set_device(0)
    import paper_1103_1399_b200 as q
    comm = q.TorchComm()
    ctx = q.Context(0, rank=rank, world=world, comm=comm)
    for key, val in (opts or {}).items():
        ctx.set_option(key, val)
    ctx.load_instance(n, clauses)
    L = n - (world.bit_length() - 1)
    ctx.init_uniform()
    ctx.evolve(T, K, np.ones(K))
    rng = np.random.default_rng(n + rank)
    starts = [int((rank << L) + s) for s in rng.integers(0, (1 << L) - 32, 8)]
    samples = {s: ctx.state(s, 32) for s in starts}
    ctx.evolve(0.06, 3)
    res = {"samples": samples, "norm2": ctx.norm2(), "super_launches": ctx.stats()["super_launches"]}
    np.save(os.path.join(outdir, f"rank{rank}.npy"), res, allow_pickle=True)
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()
