"""Helpers shared by the tests (no product or oracle arithmetic)."""


def brute_force_energy(n, clauses):
    """Pure-Python evaluation of the CNF formula P = AND_i (OR_j a_j) (PAPER.md
    P:84-91): for each assignment, count the clauses whose disjunction is false.
    Independent of oracle/ (pins the oracle's O-2)."""
    out = []
    for x in range(1 << n):
        assign = [bool((x >> (v - 1)) & 1) for v in range(1, n + 1)]
        unsat = 0
        for cl in clauses:
            clause_value = False
            for lit in cl:
                val = assign[abs(lit) - 1]
                clause_value = clause_value or (val if lit > 0 else (not val))
            if not clause_value:
                unsat += 1
        out.append(unsat)
    return out
