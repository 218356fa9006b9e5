"""Brute-force helpers for tiny d (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

These pin the oracle's encoder to the paper's *definition* rather than to its
3-step construction:

* P:139-146 (Sec. 2.3): the {x,d} EVP vertex set = all d-vectors over {-1,0,1}
  with exactly x non-zeros; there are C(d,x)*2^x of them.
* P:186 (Sec. 2.4): the nearest vertex maximises the scalar product with u.

All arithmetic is exact (``fractions.Fraction`` of the float values).
"""
from __future__ import annotations

import itertools
from fractions import Fraction


def evp_vertices(x: int, d: int):
    """Every vertex of the {x,d} EVP, in lexicographic (support, signs) order."""
    out = []
    for support in itertools.combinations(range(d), x):
        for signs in itertools.product((-1, 1), repeat=x):
            v = [0] * d
            for i, s in zip(support, signs):
                v[i] = s
            out.append(tuple(v))
    return out


def exact_dot(u, v) -> Fraction:
    return sum((Fraction(float(a)) * b for a, b in zip(u, v)), Fraction(0))


def best_vertices(u, x: int):
    """(max scalar product, list of all vertices attaining it)."""
    d = len(u)
    best, arg = None, []
    for v in evp_vertices(x, d):
        s = exact_dot(u, v)
        if best is None or s > best:
            best, arg = s, [v]
        elif s == best:
            arg.append(v)
    return best, arg


def first_max_support(u, x: int):
    """Lexicographically first support (sorted index tuple) among maximisers.

    With no exact zeros among the selected coordinates, the lowest-index tie
    rule (R1) picks exactly this support."""
    _, arg = best_vertices(u, x)
    sup = sorted(tuple(i for i, e in enumerate(v) if e != 0) for v in arg)
    return sup[0]
