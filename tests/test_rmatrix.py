"""NEXT-1: the refinement matrix R = R_{L-1} ... R_0 (P_L = R P_0).

CPU: the oracle's R (columns = refinements of unit vectors) against what the mathematics fixes:
rows sum to one (every rule is an affine combination), R P_0 reproduces the refinement, and every
row is supported on the 1-ring vertex set of a control face holding the vertex -- the property
the GPU construction (probing with a 1-ring colouring) relies on.
GPU: alsub_build_refinement_matrix entry by entry against the oracle's R, and the single-SpMM
evaluation against the level-by-level static path.
"""
import numpy as np
import pytest
import torch

import meshgen as mg
import oracle

TOL = 1e-5


def _small():
    return mg.armor(3, 3, 4, 1, 1, 1, name="armor_rm")


def _ring_sets(mesh):
    off, fv = mesh["face_off"], mesh["face_vtx"]
    F = len(off) - 1
    vf = {}
    for r in range(F):
        for v in fv[off[r]:off[r + 1]]:
            vf.setdefault(int(v), []).append(r)
    sets = []
    for r in range(F):
        s = set()
        for v in fv[off[r]:off[r + 1]]:
            for g in vf[int(v)]:
                s.update(int(x) for x in fv[off[g]:off[g + 1]])
        sets.append(s)
    return sets


@pytest.mark.parametrize("scheme,make,L", [("cc", _small, 2), ("loop", lambda: mg.tetrahedron(creased=True), 2),
                                          ("loop", lambda: mg.torus_tris(6, 5), 2)])
def test_oracle_R_rows_affine_and_reproducing(scheme, make, L):
    mesh = make()
    R = oracle.refinement_matrix(mesh, scheme, L)
    assert np.abs(R.sum(axis=1) - 1.0).max() <= 1e-12
    want = oracle.refine(mesh, scheme, L)[-1]["pos"]
    assert np.abs(R @ np.asarray(mesh["pos"], np.float64) - want).max() <= 1e-12


def test_oracle_R_rows_supported_on_a_face_one_ring():
    """CC: level-2 vertex i lies in the control faces whose descendants contain it; its row of R
    is supported on the 1-ring vertex set of (each) such face."""
    mesh = _small()
    L = 2
    R = oracle.refinement_matrix(mesh, "cc", L)
    rec = oracle.refine(mesh, "cc", L)
    off = mesh["face_off"]
    sets = _ring_sets(mesh)
    fvL = rec[L]["face_vtx"]
    owner = {}
    for r in range(len(off) - 1):
        for g in range(4 * off[r], 4 * off[r + 1]):  # level-2 descendants of control face r
            for v in fvL[4 * g:4 * g + 4]:
                owner.setdefault(int(v), r)
    assert len(owner) == R.shape[0]
    for i, r in owner.items():
        nz = set(np.nonzero(R[i])[0].tolist())
        assert nz <= sets[r], (i, r)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,make,L", [("cc", _small, 3), ("loop", lambda: mg.tetrahedron(creased=True), 3),
                                          ("cc", lambda: mg.grid(4, 3, tri_cells=[(1, 1)]), 2)])
def test_gpu_R_matches_oracle(scheme, make, L):
    from paper_1809_06047_b200 import Mesh
    mesh = make()
    want = oracle.refinement_matrix(mesh, scheme, L)
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine(scheme, L)
        info = m.build_refinement_matrix(L)
        ro, co, va = m.refinement_matrix_csr()
    assert info["rows"] == want.shape[0]
    got = np.zeros_like(want)
    for i in range(info["rows"]):
        cs = co[ro[i]:ro[i + 1]]
        assert np.all(np.diff(cs) > 0)
        got[i, cs] = va[ro[i]:ro[i + 1]]
    assert np.abs(got - want).max() <= TOL
    assert info["nnz"] == int(np.count_nonzero(got))


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,make,L,nf", [("cc", lambda: mg.armor(8, 6, 7, 1, 2, 2, name="armor_f"), 3, 40),
                                             ("loop", lambda: mg.tetrahedron(creased=True), 4, 5)])
def test_gpu_spmm_equals_static_eval(scheme, make, L, nf):
    from paper_1809_06047_b200 import Mesh
    mesh = make()
    frames = torch.stack([torch.from_numpy(mg.frame_positions(mesh["pos"], t, 64)) for t in range(nf)]).cuda()
    diag = float(np.linalg.norm(mesh["pos"].max(0) - mesh["pos"].min(0)))
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine(scheme, L)
        m.build_refinement_matrix(L)
        a = m.eval_frames_matrix(frames)
        b = m.eval_frames(frames, L)
    assert a.shape == b.shape
    assert float((a - b).abs().max()) / diag <= TOL


@pytest.mark.gpu
def test_gpu_R_errors():
    from paper_1809_06047_b200 import AlsubError, Mesh
    mesh = mg.torus_tris(6, 5)
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"]) as m:
        with pytest.raises(AlsubError):
            m.refinement_matrix_info()
        m.refine("sqrt3", 2)
        with pytest.raises(AlsubError):
            m.build_refinement_matrix(2)
        m.refine("loop", 2)
        with pytest.raises(AlsubError):
            m.build_refinement_matrix(3)
        assert m.build_refinement_matrix(2)["rows"] == m.counts(2)["verts"]
