"""K4's capacity-adaptive pop size (hexval.cu, "Stack capacity"): a model of the warp's
depth-sorted stack under adversarial push patterns.

The kernel pops k = min(32, top-level count, max(1, (K4_TM - h) / 7)) nodes per step from a
stack of height h, K4_TM = K4_CAP - 7 * MAX_DEPTH, and every popped node pushes at most 8
children one level deeper (none beyond MAX_DEPTH - 1).  The claims checked here, for the
capacities the library is built with and for the smallest legal one:

* the height never exceeds K4_CAP, whatever the pushes are (worst case: always 8);
* every step pops at least one node, and a finite tree is traversed completely (each node
  exactly once);
* with room to spare the policy is the plain "32 nodes of the top level" pop.

CPU only: the model restates the policy; the constants are read from the CUDA source so the
test follows them.
"""
from __future__ import annotations

import os
import random
import re

import pytest

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1706_01613_b200", "csrc", "hexval.cu")


def _constants():
    text = open(SRC).read()
    cap = int(re.search(r"#define HEXVAL_K4_CAP (\d+)", text).group(1))
    assert re.search(r"K4_RESERVE = 7 \* MAX_DEPTH;", text)
    assert re.search(r"K4_TM = K4_CAP - K4_RESERVE;", text)
    assert "min(min(32, tcnt), max(1, (K4_TM - h) / 7))" in text
    hdr = open(os.path.join(os.path.dirname(SRC), "hexval_device.cuh")).read() + text
    md = int(re.search(r"MAX_DEPTH = (\d+)", hdr).group(1))
    return cap, md


def pop_size(tcnt: int, h: int, tm: int) -> int:
    q = (tm - h) // 7 if tm - h >= 0 else -((h - tm) // 7)      # C++ division truncates toward zero
    return min(min(32, tcnt), max(1, q))


def run(cap: int, max_depth: int, children, roots: int = 32, max_steps: int | None = None):
    """Traverse with the kernel's policy.  `children(depth, node_id)` -> number of undecided
    children (0..8) of a node; returns (steps, nodes popped, max height, min pop size)."""
    tm = cap - 7 * max_depth
    assert tm >= 8 * 32
    levels = [[] for _ in range(max_depth)]       # node ids per level (the stack, sorted by depth)
    next_id = roots
    levels[0] = list(range(roots))
    h, steps, popped, hmax, kmin = roots, 0, 0, roots, 32
    while h > 0 and (max_steps is None or steps < max_steps):
        d = max(i for i in range(max_depth) if levels[i])
        k = pop_size(len(levels[d]), h, tm)
        assert 1 <= k <= len(levels[d])
        kmin = min(kmin, k)
        batch = [levels[d].pop() for _ in range(k)]
        h -= k
        popped += k
        for node in batch:
            c = children(d, node) if d + 1 < max_depth else 0   # depth-cap children are never pushed
            assert 0 <= c <= 8
            for _ in range(c):
                levels[d + 1].append(next_id)
                next_id += 1
            h += c
        assert h == sum(len(l) for l in levels)
        hmax = max(hmax, h)
        assert h <= cap, f"stack overflow: {h} > {cap} at step {steps}"
        steps += 1
    return steps, popped, hmax, kmin, next_id


def test_constants_are_legal():
    cap, md = _constants()
    assert md == 20
    assert cap - 7 * md >= 256 and cap % 4 == 0


@pytest.mark.parametrize("cap", ["default", 396, 416, 2048])
def test_worst_case_pushes_never_overflow(cap):
    dcap, md = _constants()
    cap = dcap if cap == "default" else cap
    # every node has 8 undecided children down to the depth cap: the tree has 8^19 nodes per
    # root, so run a bounded number of steps; the height bound must hold at every one of them
    steps, popped, hmax, kmin, _ = run(cap, md, lambda d, n: 8, max_steps=60000)
    assert steps == 60000 and popped >= steps
    assert hmax <= cap
    assert kmin == 1                     # the one-node (depth-first) mode was reached


@pytest.mark.parametrize("seed", range(6))
def test_finite_trees_are_traversed_completely(seed):
    rng = random.Random(seed)
    md = 7                               # shallow cap so the tree stays small; same policy
    cap = 7 * md + 256 + 4 * rng.randrange(0, 40)
    memo = {}

    def children(d, n):
        if n not in memo:
            memo[n] = rng.choice([0, 0, 1, 3, 8, 8, 8])
        return memo[n]

    steps, popped, hmax, kmin, created = run(cap, md, children)
    assert popped == created             # every node created was popped exactly once
    assert hmax <= cap


def test_plain_pop_when_there_is_room():
    cap, md = _constants()
    tm = cap - 7 * md
    for h in range(32, tm - 7 * 32 + 1, 17):
        assert pop_size(500, h, tm) == 32
        assert pop_size(5, h, tm) == 5
    assert pop_size(100, tm - 6, tm) == 1 and pop_size(100, tm + 100, tm) == 1
    assert pop_size(100, tm - 70, tm) == 10


@pytest.mark.parametrize("seed", range(4))
def test_random_pushes_at_the_smallest_capacity(seed):
    _, md = _constants()
    rng = random.Random(100 + seed)
    p8 = [0.3, 0.6, 0.85, 0.97][seed]
    # the bound is asserted inside run() at every step
    steps, popped, hmax, kmin, _ = run(7 * md + 256, md, lambda d, n: 8 if rng.random() < p8 else rng.randrange(0, 8),
                                       max_steps=30000)
    assert popped >= steps and hmax <= 7 * md + 256
