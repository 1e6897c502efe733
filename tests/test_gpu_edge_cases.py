"""GPU parity for the configurations and degenerate cases round 1 left untested.

Same bar as tests/test_gpu_parity.py: topology bit-exact against the oracle at every level,
positions within 1e-5 x the control bounding-box diagonal.
"""
import numpy as np
import pytest
import torch

import meshgen as mg
import oracle
from tests.test_gpu_parity import TOL, compare, diag_of
from tests.test_oracle_pins import _bowtie, _pillow2, _split_edge_cube, check_outward

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scheme", ["loop", "cc"])
def test_parity_config2b_creased_tet_L6(scheme):
    """BASELINE config 2b at the depth bench.py times (level 6): creased tetrahedron with an
    infinite, a sigma = 2 and a sigma = 5/4 crease."""
    worst = compare(mg.tetrahedron(creased=True), scheme, 6, graph=True)
    assert worst < TOL


def test_parity_config2a_ico_loop_L6_graph():
    compare(mg.icosahedron(), "loop", 6, graph=True)


@pytest.mark.parametrize("name,mk", [("bowtie", _bowtie), ("pillow2", _pillow2), ("cube_split_edge", _split_edge_cube)])
def test_parity_degenerate_vertices(name, mk):
    """Reading R18 (bowtie: two open fans at a vertex -> corner) and R17 (interior valence-2
    vertices: the pillow's four corners, the vertex inserted in a cube edge)."""
    compare(mk(), "cc", 3)


def test_bowtie_vertex_fixed_on_gpu():
    """The bowtie vertex (k = 4 boundary edges) is a corner: it never moves."""
    from paper_1809_06047_b200 import Mesh
    mesh = _bowtie()
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"]) as m:
        m.refine("cc", 3)
        for lv in range(4):
            assert np.array_equal(m.positions(lv).cpu().numpy()[0], mesh["pos"][0])


@pytest.mark.parametrize("scheme,mk", [("sqrt3", lambda: mg.icosahedron()), ("sqrt3", lambda: mg.tetrahedron()),
                                       ("loop", lambda: mg.icosahedron()), ("cc", lambda: mg.cube())])
def test_orientation_outward_on_gpu(scheme, mk):
    """sqrt3 child order (reading R13): on a convex closed mesh centred at the origin
    every GPU-refined face at L1..L3 has an outward Newell normal and the signed volume is > 0 --
    checked on the GPU's own output, not through the oracle's vertex order."""
    from paper_1809_06047_b200 import Mesh
    mesh = mk()
    mesh = dict(mesh, pos=(mesh["pos"] - mesh["pos"].mean(0)).astype(np.float32))
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"]) as m:
        m.refine(scheme, 3)
        for lv in range(1, 4):
            t = m.topology(lv, edges=False, creases=False)
            rec = {"pos": m.positions(lv).cpu().numpy().astype(np.float64),
                   "face_off": t["face_off"].cpu().numpy(), "face_vtx": t["face_vtx"].cpu().numpy()}
            check_outward(rec, f"gpu {scheme} L{lv}")


@pytest.mark.parametrize("n", [256, 1024, 1500])
@pytest.mark.parametrize("scheme", ["cc", "loop", "sqrt3"])
def test_high_valence_poles(n, scheme):
    """Bipyramids with two valence-n apices: M^T rows of 256 / 1024 / 1500 slots (the last beyond the
    register sort of k_long_rows), rings far beyond a
    warp, valence constants computed on the fly (reading R16)."""
    compare(mg.bipyramid(n), scheme, 2, edges=scheme != "sqrt3")


def test_high_valence_pole_with_creases_and_boundary():
    """An open fan of 300 quads around a pole with creases through it (long special-vertex list)."""
    n = 300
    import math
    pos = [(0.0, 0.0, 0.3)]
    for k in range(n):
        a = 2 * math.pi * k / n
        pos.append((math.cos(a), math.sin(a), 0.0))
        pos.append((2 * math.cos(a + math.pi / n), 2 * math.sin(a + math.pi / n), 0.1 * math.sin(3 * a)))
    faces = []
    for k in range(n - 1):  # open fan: the gap between the last and the first spoke is a boundary
        faces.append((0, 1 + 2 * k, 2 + 2 * k, 1 + 2 * (k + 1)))
    pairs = [(0, 1 + 2 * k) for k in range(0, n - 1, 37)]
    sig = [float(s) for s in np.resize([0.5, 2.0, np.inf], len(pairs))]
    mesh = mg._pack(faces, pos, pairs, sig, name="fan300")
    compare(mesh, "cc", 3)


# ------------------------------------------------------------------------------------------
# config 5 at its stated size: frames 0, 2047 and 4095 of 4096, in the launch configuration
# bench.py times (batches through alsub_eval_frames after a refine)
# ------------------------------------------------------------------------------------------

def _frames_batch(mesh, first, nb, nframes=4096):
    return torch.stack([torch.from_numpy(mg.frame_positions(mesh["pos"], first + t, nframes))
                        for t in range(nb)]).cuda()


def test_parity_config5_frames_first_middle_last():
    from paper_1809_06047_b200 import Mesh
    mesh = mg.armor50k()
    diag = diag_of(mesh)
    nb = 8
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 4)
        m.refine("cc", 4)
        for t in (0, 2047, 4095):
            first = (t // nb) * nb
            out = m.eval_frames(_frames_batch(mesh, first, nb), 4)
            want = oracle.refine(dict(mesh, pos=mg.frame_positions(mesh["pos"], t, 4096)), "cc", 4)[-1]["pos"]
            err = float(np.abs(out[t - first].cpu().numpy().astype(np.float64) - want).max()) / diag
            assert err <= TOL, f"frame {t}: {err:.3e}"
