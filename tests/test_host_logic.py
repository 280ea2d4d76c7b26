"""Host-side logic of the Python mirror of the reference API (CPU only):
geometry, tree index arithmetic, medium, argument errors
(proj/tests/test_medium_geometry.cpp)."""
import math

import numpy as np
import pytest

import paper_2411_18026_b200 as eb


def test_medium_from_lame_and_coupling():
    m = eb.Medium.from_lame(1.0, 1.0, 1.0, 2.0)
    assert m.lambda_() == 1.0 and m.mu() == 1.0
    assert math.isclose(m.c_L(), math.sqrt(3.0)) and m.c_T() == 1.0
    assert math.isclose(m.k_T(), 2.0) and math.isclose(m.k_L(), 2.0 / math.sqrt(3.0))
    assert m.default_coupling() == 1j / 2.0
    with pytest.raises(eb.InvalidArgument):
        eb.Medium(1.0, 2.0, 1.0, 1.0)  # c_L must exceed c_T
    with pytest.raises(eb.InvalidArgument):
        eb.Medium.from_lame(1.0, -1.0, 1.0, 1.0)


def test_star_points_and_orientation():
    s = eb.StarShape(1.0, 0.3, 3)
    x, y = s.point(0.0)
    assert math.isclose(x, 1.0) and y == 0.0
    mesh = eb.Mesh.star(64, s)
    xy = mesh.nodes
    area = 0.5 * np.sum(xy[:, 0] * np.roll(xy[:, 1], -1) - np.roll(xy[:, 0], -1) * xy[:, 1])
    assert area > 0  # counter-clockwise
    with pytest.raises(eb.InvalidArgument):
        eb.Mesh(np.zeros((3, 2)))
    with pytest.raises(eb.InvalidArgument):
        eb.Mesh([[0, 0], [1, 0], [1, 0], [0, 1]])


def test_cluster_tree_indexing():
    t = eb.ClusterTree(1024, 5)
    assert t.n_cells() == 63 and t.leaf_size() == 32
    assert eb.ClusterTree.first_cell(5) == 31 and eb.ClusterTree.last_cell(5) == 62
    assert t.leaf_begin(31) == 0 and t.leaf_end(62) == 1024
    assert t.cell_begin(2) == 512 and t.cell_end(2) == 1024
    assert t.level_of(0) == 0 and t.level_of(62) == 5
    assert eb.ClusterTree.parent(62) == 30 and eb.ClusterTree.child2(30) == 62
    assert eb.ClusterTree.depth_for(1024, 32) == 5
    assert eb.ClusterTree.depth_for(262144, 32) == 13
    assert eb.ClusterTree.depth_for(131072, 64) == 11
    assert eb.ClusterTree.depth_for(96, 32) == 2   # 96 -> 48 -> 24
    with pytest.raises(eb.InvalidArgument):
        eb.ClusterTree(100, 3)


def test_solver_checks_tree_size():
    class Fake(eb.BlockSource):
        def n_nodes(self):
            return 64
    with pytest.raises(eb.InvalidArgument):
        eb.FdsSolver(Fake(), eb.ClusterTree(128, 1))
