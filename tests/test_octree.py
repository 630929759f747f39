"""Octree API (drop-in for amrlts.octree): Morton order, construct, native 2:1
balance vs a brute-force ripple oracle, neighbours vs O(n^2) geometry, dumps.
Mirrors the intent of the reference's tests/test_octree.py."""
import itertools

import numpy as np
import pytest

from paper_2011_10570_b200.octree import (
    LinearOctree, OctKey, SfcOrdering, adjacency_kind, balance_2to1, construct, neighbors, parse_dump,
    random_tree, sfc_compare, uniform_tree, write_dump,
)


def interleave(anchor, L):
    code = 0
    for bit in range(L - 1, -1, -1):
        for d in range(len(anchor) - 1, -1, -1):
            code = (code << 1) | ((anchor[d] >> bit) & 1)
    return code


def brute_balance(tree):
    leaves = {(k.anchor, k.level) for k in tree.leaves}
    changed = True
    while changed:
        changed = False
        keys = [OctKey(a, l, tree.max_depth) for a, l in leaves]
        for a, b in itertools.combinations(keys, 2):
            if abs(a.level - b.level) > 1 and adjacency_kind(a, b) is not None:
                c = a if a.level < b.level else b
                if (c.anchor, c.level) in leaves:
                    leaves.remove((c.anchor, c.level))
                    leaves |= {(ch.anchor, ch.level) for ch in c.children()}
                    changed = True
    return leaves


def test_morton_order_is_bit_interleave():
    for dim in (2, 3):
        L = 3
        tree = uniform_tree(dim, L, L, SfcOrdering("morton", dim, L))
        codes = [interleave(k.anchor, L) for k in tree.leaves]
        assert codes == sorted(codes) and len(set(codes)) == len(codes)


def test_ancestor_first_and_compare():
    o = SfcOrdering("morton", 2, 3)
    a = OctKey((0, 0), 1, 3)
    b = OctKey((0, 0), 2, 3)
    assert sfc_compare(a, b, o) == -1 and sfc_compare(b, a, o) == 1 and sfc_compare(a, a, o) == 0
    with pytest.raises(ValueError):
        o.digits(OctKey((0, 0, 0), 1, 3))


def test_hilbert_level1_path_is_continuous():
    for dim in (2, 3):
        L = 3
        tree = uniform_tree(dim, L, L, SfcOrdering("hilbert", dim, L))
        for a, b in zip(tree.leaves, tree.leaves[1:]):
            assert sum(abs(x - y) for x, y in zip(a.anchor, b.anchor)) == 1


def test_construct_counts_and_tiling():
    assert len(uniform_tree(2, 4, 2)) == 16
    assert len(uniform_tree(3, 4, 2)) == 64
    tree = construct(lambda k: k.level < 4 and k.anchor == (0, 0), 2, 4, SfcOrdering("morton", 2, 4))
    assert len(tree) == 13  # corner chain: 3 per level + 4 at the bottom
    area = sum(k.side ** 2 for k in tree.leaves)
    assert area == (1 << 8)


@pytest.mark.parametrize("dim", [2, 3])
def test_native_balance_matches_brute_force(dim):
    rng = np.random.default_rng(100 + dim)
    for _ in range(12 if dim == 2 else 4):
        L = 5 if dim == 2 else 4
        tree = random_tree(rng, dim, L, n_clusters=2, balance=False, ordering=SfcOrdering("morton", dim, L))
        bal = balance_2to1(tree)
        assert bal.balanced
        assert {(k.anchor, k.level) for k in bal.leaves} == brute_balance(tree)
        again = balance_2to1(bal)
        assert [(k.anchor, k.level) for k in again.leaves] == [(k.anchor, k.level) for k in bal.leaves]
        codes = [(interleave(k.anchor, L), k.level) for k in bal.leaves]
        assert codes == sorted(codes)


def test_balance_hilbert_tree_keeps_hilbert_order():
    rng = np.random.default_rng(7)
    tree = random_tree(rng, 2, 5, balance=True)
    keys = [tree.ordering.sort_key(k) for k in tree.leaves]
    assert keys == sorted(keys)


def test_neighbors_match_brute_force():
    rng = np.random.default_rng(11)
    for dim in (2, 3):
        tree = random_tree(rng, dim, 4 if dim == 2 else 3, ordering=SfcOrdering("morton", dim, 4 if dim == 2 else 3))
        for key in tree.leaves[:: max(1, len(tree) // 25)]:
            for scope in ("face", "all"):
                got = {(k.anchor, k.level) for k in neighbors(key, tree, scope)}
                want = {(k.anchor, k.level) for k in tree.leaves if k != key
                        and (kind := adjacency_kind(key, k)) is not None and (scope == "all" or kind == 1)}
                assert got == want
    with pytest.raises(ValueError):
        neighbors(OctKey((0, 0), 5, 5), uniform_tree(2, 5, 1))


def test_dump_roundtrip():
    rng = np.random.default_rng(3)
    tree = random_tree(rng, 3, 3, ordering=SfcOrdering("morton", 3, 3))
    back = parse_dump(write_dump(tree), "morton")
    assert [(k.anchor, k.level) for k in back.leaves] == [(k.anchor, k.level) for k in tree.leaves]
    with pytest.raises(ValueError):
        parse_dump("2 3 5\n0 0 1\n")


def test_batch_predicate_construct_equals_scalar():
    from paper_2011_10570_b200.configs import CONFIGS

    c = CONFIGS["cfg2"]
    o = SfcOrdering("morton", 3, 5)
    a = construct(c.refine, 3, 5, o)
    b = construct(lambda k: c.refine(k), 3, 5, o)  # no .batch -> scalar path
    assert [(k.anchor, k.level) for k in a.leaves] == [(k.anchor, k.level) for k in b.leaves]
