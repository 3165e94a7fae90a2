"""CPU-side tests of the product library: the C-ABI loads and exports every
symbol include/qaa.h declares, and the host pass planner (H2) is correct.
No GPU compute calls here."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def q():
    import paper_1103_1399_b200 as q
    from paper_1103_1399_b200 import build
    build.build()
    q.lib()
    return q


def header_functions():
    src = open(os.path.join(ROOT, "include", "qaa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qaa_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(q):
    funcs = header_functions()
    assert len(funcs) >= 20
    L = q.lib()
    for f in funcs:
        assert hasattr(L, f), f"{f} declared in qaa.h but not exported"
    assert sorted(q.qaa.EXPORTS) == funcs


def test_exports_are_c_symbols(q):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", q.library_path], capture_output=True, text=True).stdout
    syms = set(re.findall(r"\bT (qaa_\w+)", out))
    assert set(header_functions()) <= syms


def test_library_is_sm100a(q):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", q.library_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_fails_cleanly(q):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(q.QaaError) as ei:
        q.qaa_create(0)
    assert ei.value.status == 5  # QAA_E_CUDA, no crash


def test_usage_errors_without_gpu(q):
    with pytest.raises(q.QaaError):
        q.qaa_create(world=3)
    with pytest.raises(q.QaaError):
        q.qaa_create(rank=2, world=2)


def simulate(rec, L, K):
    """Replays a pass plan symbolically: checks D_0..D_{K-1} appear once each, in
    order, and that between D_k and D_{k+1} (and after D_{K-1}) every qubit is
    rotated exactly once, for step k."""
    rot = {}  # (step, qubit) -> count
    d_seen = []
    cur = None  # the step whose D was applied last
    for r in rec:
        g, pre, d, post = int(r[0]), int(r[1]), int(r[2]), int(r[3])
        pre_mask = (int(r[4]) & 0xffffffff) | ((int(r[5]) & 0xffffffff) << 32)
        post_mask = (int(r[6]) & 0xffffffff) | ((int(r[7]) & 0xffffffff) << 32)
        if pre >= 0:
            assert pre == cur, "rotation for a step other than the current one"
            for j in range(L):
                if pre_mask >> j & 1:
                    rot[(pre, j)] = rot.get((pre, j), 0) + 1
        if d >= 0:
            if cur is not None:  # step cur must be complete before D_{cur+1}
                assert all(rot.get((cur, j), 0) == 1 for j in range(L)), (cur, rot)
            assert d == (0 if cur is None else cur + 1)
            d_seen.append(d)
            cur = d
        if post >= 0:
            assert post == cur
            for j in range(L):
                if post_mask >> j & 1:
                    rot[(post, j)] = rot.get((post, j), 0) + 1
    assert d_seen == list(range(K))
    for k in range(K):
        for j in range(L):
            assert rot.get((k, j), 0) == 1, (k, j)


@pytest.mark.parametrize("L", [1, 5, 12, 13, 14, 16, 20, 21, 22, 24, 27, 30, 31, 33])
@pytest.mark.parametrize("c", [3, 4])
@pytest.mark.parametrize("span", [0, 1, 2])
def test_plan_covers_every_qubit_once_per_step(q, L, c, span):
    for K in (1, 2, 3, 7):
        rec = q.qaa_plan_describe(L, c, span, K)
        simulate(rec, L, K)


@pytest.mark.parametrize("L,c,P", [(13, 3, 2), (21, 3, 2), (22, 3, 3), (30, 3, 3), (31, 3, 4), (30, 4, 4),
                                   (24, 3, 3), (16, 4, 2)])
def test_plan_pass_counts(q, L, c, P):
    """P tile groups: K*(P-1)+1 passes with step spanning, K*P without."""
    K = 10
    for span in (1, 2):
        rec = q.qaa_plan_describe(L, c, span, K)
        assert len(set(int(g) for g in rec[:, 0])) == P
        assert len(rec) == (K * (P - 1) + 1 if P > 1 else K)
    assert len(q.qaa_plan_describe(L, c, 0, K)) == K * P


def test_plan_group0_never_hosts_d(q):
    """Default schedule (mode 2): D only on strided groups, group 0 plain every step."""
    for L in (22, 26, 30, 31, 33):
        rec = q.qaa_plan_describe(L, 3, 2, 9)
        assert all(int(r[0]) != 0 for r in rec if int(r[2]) >= 0)
        g0 = [r for r in rec if int(r[0]) == 0]
        assert len(g0) == 9 and all(int(r[1]) >= 0 and int(r[2]) < 0 for r in g0)


def test_plan_register_programs_cost(q):
    """Exchange/shuffle counts of the n = 30, c = 3 plan (DESIGN.md §4 table)."""
    rec = q.qaa_plan_describe(30, 3, 1, 4)
    costs = {(int(r[0]), int(r[2]) >= 0, int(r[1]) >= 0): (int(r[8]), int(r[9])) for r in rec}
    assert costs[(0, True, False)] == (2, 0)   # first pass: D0 then 12 rotations
    assert costs[(1, False, True)] == (1, 1)   # 9 rotations: regs + one exchange + one lane shuffle
    assert costs[(2, True, True)] == (2, 2)    # D pass on a 9-qubit group
    assert costs[(0, True, True)] == (4, 0)    # D pass on the 12-qubit group


def test_plan_rejects_bad_args(q):
    with pytest.raises(q.QaaError):
        q.qaa_plan_describe(0, 3, 1, 1)
    with pytest.raises(q.QaaError):
        q.qaa_plan_describe(20, 9, 1, 1)


def replay_sharded(rec, n, world, K):
    """Replays a sharded plan tracking logical qubits through layouts A/B
    (plan.hpp): every step gets D once and each of the n logical qubits is
    rotated exactly once between D_k and D_{k+1}; the plan ends in layout A."""
    g = world.bit_length() - 1
    L = n - g
    layout = 0
    rot = {}
    cur = None
    for r in rec:
        kind, grp, pre, d, post, remote, lay, pre_m, post_m = (int(x) for x in r[:9])
        assert lay == layout, "record layout does not match the replayed layout"

        def logical(p):
            if layout == 0 or p < L - g:
                return p
            return p + g  # layout B keeps logical L..n-1 at local L-g..L-1
        if kind == 0:
            if pre >= 0:
                assert pre == cur
                for p in range(L):
                    if (pre_m >> p) & 1:
                        rot[(pre, logical(p))] = rot.get((pre, logical(p)), 0) + 1
            if d >= 0:
                if cur is not None:
                    assert all(rot.get((cur, j), 0) == 1 for j in range(n)), (cur, sorted(rot))
                assert d == (0 if cur is None else cur + 1)
                cur = d
            if post >= 0:
                assert post == cur
                for p in range(L):
                    if (post_m >> p) & 1:
                        rot[(post, logical(p))] = rot.get((post, logical(p)), 0) + 1
        if remote:
            layout ^= 1
    assert cur == K - 1
    for k in range(K):
        for j in range(n):
            assert rot.get((k, j), 0) == 1, (k, j)
    assert layout == 0


@pytest.mark.parametrize("n,world", [(14, 2), (16, 2), (17, 4), (18, 8), (24, 2), (26, 4), (31, 2), (34, 8), (33, 8)])
def test_sharded_plan_replay(q, n, world):
    for K in (1, 2, 3, 6):
        rec = q.qaa_plan_describe_sharded(n, world, 3, K)
        replay_sharded(rec, n, world, K)
        # exactly one remote (layout-swap) pass per step, plus one final remap when K is odd
        assert int(sum(rec[:, 5])) == K + (K % 2)


def test_sharded_plan_rejects_small(q):
    with pytest.raises(q.QaaError):
        q.qaa_plan_describe_sharded(13, 2, 3, 1)  # L = 12: single tile group


def test_binding_constants_match_header(q):
    """Every QAA_OPT_* and qaa_status value the binding exposes equals the one
    include/qaa.h declares (the binding hard-codes them; a drift would silently
    set the wrong option)."""
    hdr = open(os.path.join(ROOT, "include", "qaa.h")).read()
    opts = dict((k, int(v)) for k, v in re.findall(r"\bQAA_OPT_([A-Z0-9_]+)\s*=\s*(\d+)", hdr))
    assert opts, "no QAA_OPT_ enum in qaa.h"
    for name, val in opts.items():
        assert getattr(q, "OPT_" + name) == val, name
    stats = dict((int(v), "QAA_" + k) for k, v in re.findall(r"\bQAA_(OK|E_[A-Z]+)\s*=\s*(\d+)", hdr))
    assert stats == q.STATUS
