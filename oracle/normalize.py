"""Clause normalisation by chain (Tseitin) encoding — CPU oracle of NEXT row f2.

TEST INFRASTRUCTURE ONLY (see oracle.py's header): shares no code with the CUDA path
(paper_2603_28796_b200/csrc/tseitin_kernels.cu).

PAPER.md §2.2 "Clause Normalization for Vectorization", P:169-197:
  * Eq.6-7: a clause C = (l_1 v ... v l_u) becomes, for the fixed size 3,
        (l_1 v l_2 v f_1) ^ (-f_1 v l_3 v f_2) ^ ... ^ (-f_{u-3} v l_{u-1} v l_u)
    with fresh auxiliaries f_1 .. f_{u-3};
  * "the number of auxiliary variables depends on the chosen fixed clause size"
    (reading R26 in DESIGN.md: for size k the first clause keeps k-1 literals, every
    middle clause -f_j plus k-2 literals plus f_{j+1}, the last -f_q plus the rest);
  * P:190 "For clauses shorter than the fixed size (e.g., u<3), literals are duplicated as
    needed" (Appendix B: (-x1 v x3) -> (-x1 v x3 v x3): the LAST literal is
    repeated, reading R27);
  * Appendix B numbers auxiliaries after the original variables (z_1 = x_5), in clause order.
Pinned by tests/test_oracle_pins.py (Appendix B golden, aux count u-3 for k = 3, brute-force
projection of models on small random formulas).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def chain_encode(clause: Sequence[int], k: int, next_aux: int) -> Tuple[List[List[int]], int]:
    """Eq.7 for one clause (generalised to size k, R26). Returns (clauses, next free aux)."""
    lits = list(clause)
    u = len(lits)
    if u <= k:                                  # duplicate to width k (R27)
        return [lits + [lits[-1]] * (k - u)], next_aux
    out = []
    f = next_aux                                # f_1
    out.append(lits[:k - 1] + [f])              # (l_1 v .. v l_{k-1} v f_1)
    rest = lits[k - 1:]
    while len(rest) > k - 1:                    # (-f_j v next k-2 literals v f_{j+1})
        out.append([-f] + rest[:k - 2] + [f + 1])
        rest = rest[k - 2:]
        f += 1
    last = [-f] + rest                          # (-f_q v l_.. v l_u)
    out.append(last + [last[-1]] * (k - len(last)))
    return out, f + 1


def normalize(n: int, clauses: Sequence[Sequence[int]], k: int = 3) -> Tuple[int, List[List[int]]]:
    """phi -> phi': apply chain_encode to every clause in order. Returns (n', phi')."""
    if k < 3:
        raise ValueError("chain encoding needs k >= 3")
    out: List[List[int]] = []
    nxt = n + 1
    for c in clauses:
        if len(c) == 0:
            raise ValueError("empty clause")
        cl, nxt = chain_encode(c, k, nxt)
        out.extend(cl)
    return nxt - 1, out
