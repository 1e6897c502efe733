"""NEXT-2: reverse Cuthill-McKee reordering of the control mesh.

CPU tests: the oracle (oracle/rcm.py) against properties the algorithm fixes (a permutation, a
path's natural order, grid bandwidth, no worse than scipy's RCM, faces sorted by their first
non-zero), then the library's host implementation (alsub_rcm_order) index for index against the
oracle.  GPU test: refinement of the reordered mesh against the oracle (it is just another mesh).
"""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

import meshgen as mg
from oracle import rcm


def _bw_perm(mesh, perm):
    return rcm.bandwidth(mesh["face_off"], mesh["face_vtx"], perm)


def _scipy_bw(mesh):
    V = mesh["pos"].shape[0]
    nbr = rcm.vertex_graph(mesh["face_off"], mesh["face_vtx"], V)
    rows = [v for v in range(V) for _ in nbr[v]]
    cols = [w for v in range(V) for w in nbr[v]]
    A = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(V, V))
    p = reverse_cuthill_mckee(A, symmetric_mode=True)
    return _bw_perm(mesh, list(p))


def test_rcm_is_permutation_and_faces_sorted():
    mesh = mg.shuffled(mg.armor(6, 5, 6, 1, 2, 2, name="armor_rcm"))
    V, F = mesh["pos"].shape[0], len(mesh["face_off"]) - 1
    pv, pf = rcm.rcm_order(mesh["face_off"], mesh["face_vtx"], V)
    assert sorted(pv) == list(range(V)) and sorted(pf) == list(range(F))
    newid = np.empty(V, np.int64)
    newid[np.asarray(pv)] = np.arange(V)
    off, vtx = mesh["face_off"], mesh["face_vtx"]
    keys = [min(newid[vtx[off[r]:off[r + 1]]]) for r in pf]
    assert keys == sorted(keys)


def test_rcm_strip_is_a_path_order():
    """A 1 x n strip of quads: RCM from a corner walks it end to end (bandwidth 2 = the quad's
    diagonal neighbour in the level order)."""
    mesh = mg.shuffled(mg.grid(12, 1))
    pv, _ = rcm.rcm_order(mesh["face_off"], mesh["face_vtx"], mesh["pos"].shape[0])
    assert _bw_perm(mesh, pv) <= 2
    assert _bw_perm(mesh, list(range(mesh["pos"].shape[0]))) > 2


def test_rcm_grid_bandwidth():
    """An n x m grid (n <= m) has a level structure of width <= n + 1 from a corner."""
    for nx, ny in ((6, 9), (9, 4)):
        mesh = mg.shuffled(mg.grid(nx, ny))
        pv, _ = rcm.rcm_order(mesh["face_off"], mesh["face_vtx"], mesh["pos"].shape[0])
        assert _bw_perm(mesh, pv) <= min(nx, ny) + 2


def test_rcm_no_worse_than_scipy():
    for mesh in (mg.shuffled(mg.armor(6, 5, 6, 1, 2, 2, name="armor_rcm")), mg.shuffled(mg.torus_tris(30, 20))):
        pv, _ = rcm.rcm_order(mesh["face_off"], mesh["face_vtx"], mesh["pos"].shape[0])
        ours, ref, shuf = _bw_perm(mesh, pv), _scipy_bw(mesh), _bw_perm(mesh, list(range(mesh["pos"].shape[0])))
        assert ours <= 1.25 * ref + 2, (ours, ref)
        assert ours * 5 < shuf


def test_rcm_components_and_isolated():
    """Two disjoint cubes plus an isolated vertex: every vertex placed exactly once."""
    a, b = mg.cube(), mg.cube()
    faces = [list(a["face_vtx"][a["face_off"][r]:a["face_off"][r + 1]]) for r in range(6)]
    faces += [[v + 9 for v in b["face_vtx"][b["face_off"][r]:b["face_off"][r + 1]]] for r in range(6)]
    pos = np.vstack([a["pos"], np.zeros((1, 3)), b["pos"] + 2.0])
    mesh = mg._pack(faces, pos, name="two_cubes")
    pv, pf = rcm.rcm_order(mesh["face_off"], mesh["face_vtx"], 17)
    assert sorted(pv) == list(range(17)) and sorted(pf) == list(range(12))


@pytest.mark.parametrize("make", [
    lambda: mg.cube(),
    lambda: mg.shuffled(mg.armor(6, 5, 6, 1, 2, 2, name="armor_rcm")),
    lambda: mg.shuffled(mg.torus_tris(30, 20)),
    lambda: mg.shuffled(mg.grid(7, 5, tri_cells=[(1, 1), (3, 2)])),
])
def test_library_rcm_matches_oracle(make):
    """alsub_rcm_order (host C++ in libalsub) == the oracle, index for index."""
    from paper_1809_06047_b200 import rcm_order
    mesh = make()
    V = mesh["pos"].shape[0]
    pv, pf = rcm_order(mesh["face_off"], mesh["face_vtx"], V)
    wv, wf = rcm.rcm_order(mesh["face_off"], mesh["face_vtx"], V)
    assert np.array_equal(pv, np.asarray(wv)) and np.array_equal(pf, np.asarray(wf))


def test_library_rcm_errors():
    from paper_1809_06047_b200 import AlsubError, rcm_order
    with pytest.raises(AlsubError):
        rcm_order(np.array([0, 3], np.int32), np.array([0, 1, 7], np.int32), 3)


@pytest.mark.gpu
def test_refine_rcm_reordered_mesh_parity():
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_parity import compare
    from paper_1809_06047_b200 import rcm_order
    mesh = mg.shuffled(mg.armor(8, 6, 7, 1, 2, 2, name="armor_rcm"))
    pv, pf = rcm_order(mesh["face_off"], mesh["face_vtx"], mesh["pos"].shape[0])
    compare(mg.permuted(mesh, pv, pf), "cc", 3)
