"""Shared builders for tests: BASELINE configs through our API."""
import numpy as np

from paper_2011_10570_b200.configs import CONFIGS
from paper_2011_10570_b200.mesh import Domain, Mesh
from paper_2011_10570_b200.octree import SfcOrdering, balance_2to1, construct
from paper_2011_10570_b200.partition import tree_weights, weighted_partition


def config_tree(name):
    c = CONFIGS[name]
    return balance_2to1(construct(c.refine, c.dim, c.max_depth, SfcOrdering("morton", c.dim, c.max_depth)))


def config_mesh(name, ranks=1, mode="lts", tree=None):
    c = CONFIGS[name]
    tree = tree if tree is not None else config_tree(name)
    pmap = weighted_partition(tree, tree_weights(tree, mode), ranks) if ranks > 1 else None
    return Mesh(tree, points_per_octant=c.ppo, pad=c.pad, pmap=pmap, domain=Domain(c.domain_lo, c.domain_hi))
