"""3-SAT instances: DIMACS I/O, the paper's worked instance, seeded generator.

Conventions (DESIGN.md R-conventions): variable x_j is
bit j-1 of a basis index, bit value 1 = true. Clauses are lists of three
DIMACS-signed literals (+j for x_j, -j for NOT x_j).

The generator follows BASELINE.json's recipe ("random 3-SAT with a unique
satisfying assignment, built by adding random clauses until one solution
remains", paper hard-instance density ~4.2) with the details
fixed in DESIGN.md (reading R16): splitmix64-seeded xoshiro256**, three
distinct variables per clause (rejection sampling), each literal negated with
probability 1/2, exact duplicate clauses rejected, restart on zero survivors.
Survivor filtering uses a bitmap of assignments (a boolean filter, not the
method's energy).
"""
from __future__ import annotations

import os
from typing import List, Sequence, Tuple

import numpy as np

MASK64 = (1 << 64) - 1

# ---------------------------------------------------------------------------
# The paper's worked instance, transcribed verbatim from PAPER.md P:97-107
# (n = 6, m = 27). The paper claims the unique solution x = (1,1,0,1,0,0)
# (P:109); brute force over the clauses as printed gives (0,1,0,1,0,0) instead
# (reading R6). PAPER_CORRECTED flips clause 11 (-1 -2 -4 -> 1 -2 -4),
# the only single sign flip that makes the paper's stated solution unique.
# ---------------------------------------------------------------------------
PAPER_N = 6
PAPER_CLAUSES: List[Tuple[int, int, int]] = [
    (-1, -4, -5), (-2, -3, -4), (1, 2, -5), (3, 4, 5),
    (4, 5, -6), (-1, -3, -5), (1, -2, -5), (2, -3, -6),
    (-1, -2, -6), (3, -5, -6), (-1, -2, -4), (2, 3, -4),
    (2, 5, -6), (2, -3, -5), (-2, -3, -4), (2, 3, 6),
    (-1, -2, -3), (-1, -4, -5), (-3, -4, -6), (-4, -5, 6),
    (-2, 3, -6), (2, 5, 6), (3, 5, -6), (-1, 3, -6),
    (3, -5, 6), (4, 5, 6), (1, 2, -3),
]
PAPER_STATED_SOLUTION_BITS = (1, 1, 0, 1, 0, 0)  # (x1..x6)
PAPER_CORRECTED_CLAUSES = list(PAPER_CLAUSES)
PAPER_CORRECTED_CLAUSES[10] = (1, -2, -4)


def bits_to_index(bits: Sequence[int]) -> int:
    """(x1, x2, ..., xn) -> basis index with x1 as the least significant bit."""
    return sum((int(b) & 1) << i for i, b in enumerate(bits))


# ---------------------------------------------------------------------------
# DIMACS
# ---------------------------------------------------------------------------
class DimacsError(ValueError):
    pass


def write_dimacs(n: int, clauses, comments: Sequence[str] = ()) -> str:
    lines = [f"c {c}" for c in comments]
    lines.append(f"p cnf {n} {len(clauses)}")
    lines += [" ".join(str(int(l)) for l in cl) + " 0" for cl in clauses]
    return "\n".join(lines) + "\n"


def parse_dimacs(text: str):
    """Returns (n, clauses, comments). Errors name the offending line."""
    n = m = None
    clauses = []
    comments = []
    pending: List[int] = []
    for lineno, raw in enumerate(text.splitlines(), 1):
        line = raw.strip()
        if not line:
            continue
        if line.startswith("c"):
            comments.append(line[1:].strip())
            continue
        if line.startswith("p"):
            parts = line.split()
            if len(parts) != 4 or parts[1] != "cnf":
                raise DimacsError(f"line {lineno}: malformed header {raw!r}")
            n, m = int(parts[2]), int(parts[3])
            continue
        if n is None:
            raise DimacsError(f"line {lineno}: clause before header")
        for tok in line.split():
            v = int(tok)
            if v == 0:
                if len(pending) != 3:
                    raise DimacsError(f"line {lineno}: clause length {len(pending)} != 3")
                clauses.append(tuple(pending))
                pending = []
            else:
                if abs(v) > n:
                    raise DimacsError(f"line {lineno}: variable {abs(v)} out of range 1..{n}")
                pending.append(v)
    if n is None:
        raise DimacsError("missing 'p cnf' header")
    if pending:
        raise DimacsError("unterminated final clause")
    if len(clauses) != m:
        raise DimacsError(f"clause count {len(clauses)} != header {m}")
    return n, clauses, comments


def read_dimacs(path: str):
    with open(path) as f:
        return parse_dimacs(f.read())


# ---------------------------------------------------------------------------
# Seeded RNG: splitmix64 -> xoshiro256** (pure Python, platform independent)
# ---------------------------------------------------------------------------
def _splitmix64(state: int):
    state = (state + 0x9E3779B97F4A7C15) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


def _rotl(x: int, k: int) -> int:
    return ((x << k) | (x >> (64 - k))) & MASK64


class Xoshiro256ss:
    def __init__(self, seed: int):
        st = seed & MASK64
        self.s = []
        for _ in range(4):
            st, z = _splitmix64(st)
            self.s.append(z)

    def next(self) -> int:
        s = self.s
        result = (_rotl((s[1] * 5) & MASK64, 7) * 9) & MASK64
        t = (s[1] << 17) & MASK64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return result

    def below(self, n: int) -> int:
        """Uniform integer in [0, n) by rejection (no modulo bias)."""
        lim = (1 << 64) - ((1 << 64) % n)
        while True:
            r = self.next()
            if r < lim:
                return r % n

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / (1 << 53))


def random_clause(rng: Xoshiro256ss, n: int) -> Tuple[int, int, int]:
    vs: List[int] = []
    while len(vs) < 3:
        v = rng.below(n) + 1
        if v not in vs:
            vs.append(v)
    return tuple(v if (rng.next() >> 63) == 0 else -v for v in vs)


# ---------------------------------------------------------------------------
# Survivor filter: bitmap over assignments (bit x of the map = assignment x
# satisfies every clause so far). Boolean bookkeeping for instance
# construction only.
# ---------------------------------------------------------------------------
class _Survivors:
    LIST_MODE = 1 << 16

    def __init__(self, n: int):
        self.n = n
        self.list = None
        if n <= 6:
            self.list = np.arange(1 << n, dtype=np.uint64)
            self.words = None
        else:
            self.words = np.full(1 << (n - 6), MASK64, dtype=np.uint64)

    def count(self) -> int:
        if self.list is not None:
            return int(self.list.size)
        return int(np.bitwise_count(self.words).sum())

    def kill(self, clause):
        """Remove the assignments that falsify every literal of `clause`."""
        if self.list is not None:
            keep = np.zeros(self.list.size, dtype=bool)
            for l in clause:
                v = abs(l) - 1
                bit = (self.list >> np.uint64(v)) & np.uint64(1)
                keep |= bit == (1 if l > 0 else 0)
            self.list = self.list[keep]
            return
        n = self.n
        inword = MASK64
        idx = [slice(None)] * (n - 6)
        for l in clause:
            v = abs(l) - 1
            false_val = 0 if l > 0 else 1  # value of x_v that makes the literal false
            if v < 6:
                pat = 0
                for b in range(64):
                    if ((b >> v) & 1) == false_val:
                        pat |= 1 << b
                inword &= pat
            else:
                axis = (n - 6 - 1) - (v - 6)  # C order: last axis = word-index bit 0
                idx[axis] = false_val
        view = self.words.reshape((2,) * (n - 6)) if n > 6 else self.words
        view[tuple(idx)] &= np.uint64(~inword & MASK64)
        if self.count() <= self.LIST_MODE:
            self._to_list()

    def _to_list(self):
        w = np.flatnonzero(self.words)
        out = []
        for wi in w:
            val = int(self.words[wi])
            for b in range(64):
                if (val >> b) & 1:
                    out.append((int(wi) << 6) | b)
        self.list = np.array(out, dtype=np.uint64)
        self.words = None

    def members(self) -> np.ndarray:
        if self.list is None:
            self._to_list()
        return np.sort(self.list)


def generate_unique_instance(n: int, seed: int):
    """Seeded random 3-SAT instance over n >= 3 variables with exactly one
    satisfying assignment. Returns (clauses, solution_index, restarts)."""
    if n < 3:
        raise ValueError("n must be >= 3 (three distinct variables per clause)")
    rng = Xoshiro256ss(seed)
    restarts = 0
    while True:
        surv = _Survivors(n)
        clauses: List[Tuple[int, int, int]] = []
        seen = set()
        while True:
            cl = random_clause(rng, n)
            key = tuple(sorted(cl))
            if key in seen:
                continue
            seen.add(key)
            clauses.append(cl)
            surv.kill(cl)
            c = surv.count()
            if c == 1:
                return clauses, int(surv.members()[0]), restarts
            if c == 0:
                restarts += 1
                break


def random_instance(n: int, m: int, seed: int):
    """m random clauses with 3 distinct variables (no uniqueness filter)."""
    rng = Xoshiro256ss(seed)
    return [random_clause(rng, n) for _ in range(m)]


# ---------------------------------------------------------------------------
# Checked-in instances (inputs/instances/usa_n{n}_s{seed}.cnf)
# ---------------------------------------------------------------------------
INSTANCE_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "instances")


def instance_path(n: int, seed: int | None = None) -> str:
    seed = 1000 + n if seed is None else seed
    return os.path.join(INSTANCE_DIR, f"usa_n{n}_s{seed}.cnf")


def load_instance(n: int, seed: int | None = None):
    """(clauses, solution_index) of the checked-in unique-solution instance."""
    nn, clauses, comments = read_dimacs(instance_path(n, seed))
    assert nn == n
    sol = None
    for c in comments:
        if c.startswith("solution_index"):
            sol = int(c.split("=")[1])
    return clauses, sol


def paper_instance(corrected: bool = False):
    return PAPER_N, list(PAPER_CORRECTED_CLAUSES if corrected else PAPER_CLAUSES)


# ---------------------------------------------------------------------------
# Schedules (Eq. 1 linear sweep; midpoint sampling, R8)
# ---------------------------------------------------------------------------
def midpoint_schedule(K: int) -> np.ndarray:
    return (np.arange(K, dtype=np.float64) + 0.5) / K


def constant_schedule(K: int, s: float) -> np.ndarray:
    return np.full(K, float(s), dtype=np.float64)


def random_state(n: int, seed: int) -> np.ndarray:
    """Seeded random complex128 state (not normalised) for parity tests."""
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) * (2.0 ** (-n / 2))
