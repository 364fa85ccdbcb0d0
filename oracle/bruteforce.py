"""Brute-force references for tiny CNFs (TEST INFRASTRUCTURE ONLY).

Pure-Python, obviously-correct Boolean semantics (SPEC cnf-core verify_model):
a clause holds iff one of its literals is true; a formula holds iff all clauses do.
Used to pin the fp64 oracle (exhaustive over all 2^n assignments for n <= 16).
"""
from __future__ import annotations

import itertools
from typing import Iterable, List, Optional, Sequence


def literal_true(lit: int, x: Sequence[int]) -> bool:
    value = bool(x[abs(lit) - 1])
    return value if lit > 0 else not value


def clause_true(clause: Sequence[int], x: Sequence[int]) -> bool:
    return any(literal_true(l, x) for l in clause)


def naive_unsat(clauses: Sequence[Sequence[int]], x: Sequence[int]) -> int:
    return sum(0 if clause_true(c, x) else 1 for c in clauses)


def all_assignments(n: int) -> Iterable[List[int]]:
    for bits in itertools.product((0, 1), repeat=n):
        yield list(bits)


def is_satisfiable(n: int, clauses: Sequence[Sequence[int]]) -> bool:
    return any(naive_unsat(clauses, x) == 0 for x in all_assignments(n))


def dpll(n: int, clauses: Sequence[Sequence[int]]) -> Optional[List[int]]:
    """Tiny DPLL (unit propagation + branching) that returns a model or None.
    Test-only labeller for instances too large to enumerate (n <= ~100)."""
    import sys
    sys.setrecursionlimit(10000)
    cls = [list(c) for c in clauses]

    def solve(cls, assign):
        changed = True
        while changed:
            changed = False
            new = []
            for c in cls:
                if any(assign.get(abs(l)) == (l > 0) for l in c):
                    continue
                rest = [l for l in c if abs(l) not in assign]
                if not rest:
                    return None
                if len(rest) == 1:
                    assign[abs(rest[0])] = rest[0] > 0
                    changed = True
                new.append(rest)
            cls = new
        if not cls:
            return assign
        counts = {}
        for c in cls:
            for l in c:
                counts[l] = counts.get(l, 0) + 1
        lit = max(counts, key=lambda l: (counts[l], -abs(l)))
        for val in (lit > 0, lit < 0):
            a2 = dict(assign)
            a2[abs(lit)] = val
            res = solve(cls, a2)
            if res is not None:
                return res
        return None

    res = solve(cls, {})
    if res is None:
        return None
    return [1 if res.get(v, False) else 0 for v in range(1, n + 1)]
