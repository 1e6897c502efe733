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


# ------------------------------------------------------------------------------------------
# the blocked evaluation (alsub_eval_frames_matrix): chunks = owner faces with dense weight blocks
# ------------------------------------------------------------------------------------------

def _iso():
    """Armor patch + two isolated control vertices (identity chunks)."""
    m = mg.armor(3, 3, 4, 1, 1, 1, name="armor_rm_iso")
    pos = np.vstack([m["pos"], [[3.0, 3.0, 3.0], [-2.0, 1.0, 0.5]]]).astype(np.float32)
    return dict(m, pos=pos)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,make,L,nf", [
    ("cc", _small, 3, 37),                        # ragged batch: 32 + 5 frames
    ("cc", _iso, 2, 3),                           # isolated control vertices: identity chunks
    ("loop", lambda: mg.bipyramid(30), 2, 9),     # supports of 30+ vertices: the wide-tile path
    ("cc", lambda: mg.bipyramid(20), 2, 4),
])
def test_gpu_blocked_spmm_equals_oracle_R(scheme, make, L, nf):
    """P_L = R P_0 for random frames: the GPU's blocked SpMM against the oracle's R applied in fp64
    (the oracle's R columns are refinements of unit vectors, independent of the GPU's probing)."""
    from paper_1809_06047_b200 import Mesh
    mesh = make()
    R = oracle.refinement_matrix(mesh, scheme, L)
    rng = np.random.default_rng(7)
    fr = (mesh["pos"][None] + rng.normal(0, 0.05, (nf,) + mesh["pos"].shape)).astype(np.float32)
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine(scheme, L)
        m.build_refinement_matrix(L)
        got = m.eval_frames_matrix(torch.from_numpy(fr).cuda()).cpu().numpy().astype(np.float64)
    diag = float(np.linalg.norm(mesh["pos"].max(0) - mesh["pos"].min(0)))
    for f in range(nf):
        want = R @ fr[f].astype(np.float64)
        assert np.abs(got[f] - want).max() / diag <= TOL, f


@pytest.mark.gpu
def test_gpu_R_invalidated_by_a_new_plan():
    """the matrix indexes the plan's levels -- a refine with another plan drops it."""
    from paper_1809_06047_b200 import AlsubError, Mesh
    mesh = mg.tetrahedron(creased=True)
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 3)
        m.build_refinement_matrix(3)
        m.refine("cc", 3)  # same plan (graph replay): kept
        assert m.refinement_matrix_info()["levels"] == 3
        m.refine("cc", 2)
        with pytest.raises(AlsubError):
            m.refinement_matrix_info()
        with pytest.raises(AlsubError):
            m.eval_frames_matrix(torch.zeros((1, 4, 3), device="cuda"))
        m.build_refinement_matrix(2)
        m.refine("loop", 2)
        with pytest.raises(AlsubError):
            m.refinement_matrix_info()


@pytest.mark.gpu
def test_gpu_blocked_spmm_config5_full_size():
    """Config 5 at its stated size through the matrix path bench.py times: armor50k CC L4, frames
    0, 2047 and 4095 of 4096 (batches of 32) against the oracle refining those frames."""
    from paper_1809_06047_b200 import Mesh
    mesh = mg.armor50k()
    diag = float(np.linalg.norm(mesh["pos"].max(0) - mesh["pos"].min(0)))
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 4)
        m.build_refinement_matrix(4)
        for t in (0, 2047, 4095):
            first = (t // 32) * 32
            fr = torch.stack([torch.from_numpy(mg.frame_positions(mesh["pos"], first + u, 4096)) for u in range(32)]).cuda()
            out = m.eval_frames_matrix(fr)
            want = oracle.refine(dict(mesh, pos=mg.frame_positions(mesh["pos"], t, 4096)), "cc", 4)[-1]["pos"]
            err = float(np.abs(out[t - first].cpu().numpy().astype(np.float64) - want).max()) / diag
            assert err <= TOL, f"frame {t}: {err:.3e}"


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,make,L,nf", [("cc", _small, 3, 37), ("loop", lambda: mg.bipyramid(30), 2, 5)])
def test_gpu_fused_summaries_equal_frame_summary(scheme, make, L, nf):
    """alsub_eval_frames_matrix_summary: the records folded in while the frames are written are
    bit for bit alsub_frame_summary of the written frames (bbox and checksum are order-free), and
    the frames equal the plain matrix evaluation."""
    from paper_1809_06047_b200 import Mesh, frame_summary
    mesh = make()
    rng = np.random.default_rng(11)
    fr = torch.from_numpy((mesh["pos"][None] + rng.normal(0, 0.05, (nf,) + mesh["pos"].shape)).astype(np.float32)).cuda()
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine(scheme, L)
        m.build_refinement_matrix(L)
        out, rec = m.eval_frames_matrix_summary(fr)
        plain = m.eval_frames_matrix(fr)
        assert torch.equal(out, plain)
        assert torch.equal(rec, frame_summary(out))
