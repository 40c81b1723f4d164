"""Integer scheduling of the iterative builder (host mirror of the device's
``__popcll`` arithmetic in csrc/ts_engine.cuh::build_tree).

Reference: turnstile/treemath.py:13-58.
"""

from __future__ import annotations

MAX_TREE_DEPTH_LIMIT = 30


def bit_count(n: int) -> int:
    if n < 0:
        raise ValueError("leaf index must be non-negative")
    return n.bit_count()


def trailing_ones(n: int) -> int:
    """popcount(((n + 1) & ~n) - 1)."""
    if n < 0:
        raise ValueError("leaf index must be non-negative")
    return (((n + 1) & ~n) - 1).bit_count()


def subtree_leftmost(n: int, k: int) -> int:
    if n < 0 or k < 0:
        raise ValueError("arguments must be non-negative")
    return n & ~((1 << k) - 1)


def candidate_set(n: int) -> list[tuple[int, int]]:
    """(stored leaf, slot) pairs odd leaf n is checked against, innermost first."""
    out = []
    for k in range(1, trailing_ones(n) + 1):
        m = n & ~((1 << k) - 1)
        out.append((m, m.bit_count()))
    return out
