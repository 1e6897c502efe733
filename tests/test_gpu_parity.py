"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Topology (face lists, edge ids/vertex pairs, F(i,j)/F(j,i), crease lists) bit-exact at every level;
positions within 1e-5 x the control mesh's bounding-box diagonal (BASELINE.json north_star,
SURVEY.md 8(c) c15).
"""
import numpy as np
import pytest
import torch

import meshgen as mg
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _gpu():
    from paper_1809_06047_b200 import Mesh
    return Mesh


def diag_of(mesh):
    p = mesh["pos"].astype(np.float64)
    return float(np.linalg.norm(p.max(0) - p.min(0)))


def compare(mesh, scheme, levels, edges=True, creases=True, oracle_recs=None, graph=False):
    Mesh = _gpu()
    want = oracle_recs or oracle.refine(mesh, scheme, levels)
    diag = diag_of(mesh)
    worst = 0.0
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine(scheme, levels)
        if graph:  # bench.py's launch configuration: the CUDA-graph replay (2nd refine on)
            m.refine(scheme, levels)
            m.refine(scheme, levels)
        torch.cuda.synchronize()
        for lv in range(levels + 1):
            c = m.counts(lv)
            w = want[lv]
            assert (c["verts"], c["faces"]) == (w["V"], w["F"]), f"L{lv} counts"
            want_edges = edges and lv < levels and c["edges_valid"]
            t = m.topology(lv, edges=want_edges, creases=creases)
            assert np.array_equal(t["face_vtx"].cpu().numpy(), w["face_vtx"]), f"L{lv} face_vtx"
            assert np.array_equal(t["face_off"].cpu().numpy(), w["face_off"]), f"L{lv} face_off"
            if want_edges:
                assert c["edges"] == w["E"] and c["boundary_edges"] == w["B"], f"L{lv} E/B"
                assert np.array_equal(t["edge_vtx"].cpu().numpy(), w["edge_vtx"]), f"L{lv} edge_vtx"
                assert np.array_equal(t["edge_face"].cpu().numpy(), w["edge_face"]), f"L{lv} edge_face"
            if creases and lv > 0:
                assert np.array_equal(t["crease"].cpu().numpy(), w["crease"]), f"L{lv} crease pairs"
                assert np.array_equal(t["sigma"].cpu().numpy(), w["sigma"]), f"L{lv} crease sigma"
            P = m.positions(lv).cpu().numpy().astype(np.float64)
            err = float(np.abs(P - w["pos"]).max()) / diag if w["V"] else 0.0
            worst = max(worst, err)
            assert err <= TOL, f"L{lv} positions: max err {err:.3e} x diag"
    return worst


def _octahedron():
    pos = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    faces = [(0, 2, 4), (2, 1, 4), (1, 3, 4), (3, 0, 4), (2, 0, 5), (1, 2, 5), (3, 1, 5), (0, 3, 5)]
    return mg._pack(faces, pos, name="octa")


def _mixed_polys():
    """Pentagon + hexagon + quads + triangles sharing edges, open boundary, creases."""
    pos = [(0, 0, 0), (1, 0, 0), (2, 0, 0.2), (2.5, 1, 0), (2, 2, 0.1), (1, 2, 0), (0, 2, 0.3), (-0.5, 1, 0),
           (1, 1, 0.5), (3, 0, 0), (3.5, 1.5, 0.2)]
    faces = [(0, 1, 8, 6, 7), (1, 2, 3, 4, 5, 8), (5, 6, 8), (2, 9, 3), (9, 10, 3)]
    return mg._pack(faces, pos, [(1, 8), (8, 5), (2, 3)], [1.5, 0.5, np.inf], name="mixed")


CASES = [
    ("cube", mg.cube, "cc", 3),
    ("tet", mg.tetrahedron, "cc", 3),
    ("tet_creased_cc", lambda: mg.tetrahedron(creased=True), "cc", 4),
    ("tet_creased_loop", lambda: mg.tetrahedron(creased=True), "loop", 4),
    ("ico_loop", mg.icosahedron, "loop", 4),
    ("octa_loop", _octahedron, "loop", 3),
    ("quad", mg.single_quad, "cc", 4),
    ("grid_tris", lambda: mg.grid(5, 4, tri_cells=[(1, 1), (3, 2)]), "cc", 4),
    ("mixed", _mixed_polys, "cc", 4),
    ("armor_small", lambda: mg.armor(6, 5, 6, 1, 1, 2, name="armor_small"), "cc", 4),
    ("armor_small_shuf", lambda: mg.shuffled(mg.armor(6, 5, 6, 1, 1, 2, name="armor_small")), "cc", 3),
    ("torus_sqrt3", lambda: mg.torus_tris(20, 15), "sqrt3", 4),
    ("octa_sqrt3", _octahedron, "sqrt3", 3),
    ("torus_loop", lambda: mg.torus_tris(16, 12), "loop", 3),
    ("grid_loop_bnd", lambda: mg.grid(4, 3, tri_cells=[(i, j) for i in range(4) for j in range(3)]), "loop", 3),
]


@pytest.mark.parametrize("name,mk,scheme,levels", CASES, ids=[c[0] for c in CASES])
def test_parity_small(name, mk, scheme, levels):
    compare(mk(), scheme, levels)


def test_parity_semisharp_and_corners():
    """Semi-sharp creases (0 < sigma < 1), a crease ending inside (dart), 3 creases at a vertex."""
    g = mg.random_positions(mg.torus_quads(9, 7), seed=2, scale=0.3)
    nu = 9
    vid = lambda i, j: (j % 7) * nu + (i % nu)
    pairs = [(vid(0, 0), vid(1, 0)), (vid(1, 0), vid(2, 0)), (vid(2, 0), vid(3, 0)),
             (vid(1, 0), vid(1, 1)), (vid(1, 0), vid(1, 6)), (vid(5, 3), vid(6, 3))]
    sig = [0.25, 0.75, 2.5, 1.25, np.inf, 0.5]
    g["crease"], g["sigma"] = np.array(pairs, np.int32), np.array(sig, np.float32)
    compare(g, "cc", 4)


def test_parity_armor9k_L3():
    compare(mg.armor9k(), "cc", 3)


def test_parity_torus100k_sqrt3_L3():
    compare(mg.torus100k(), "sqrt3", 3, edges=True)


def test_parity_ico_loop_L6():
    compare(mg.icosahedron(), "loop", 6)


def test_parity_armor9k_L6_full():
    """Config 3 at full size (35M faces), same launch configuration as bench.py (graph replay)."""
    mesh = mg.armor9k()
    worst = compare(mesh, "cc", 6, edges=False, graph=True)
    assert worst < TOL


def test_parity_torus100k_sqrt3_L5_full():
    """Config 4 at full size (24.3M faces), graph replay as in bench.py's other_configs."""
    worst = compare(mg.torus100k(), "sqrt3", 5, edges=False, graph=True)
    assert worst < TOL


def test_parity_config5_frames_sampled():
    """Config 5 at full size: armor50k CC L4 static eval in bench.py's batches of 8 frames;
    sampled frames against the oracle refining those frames' positions."""
    Mesh = _gpu()
    mesh = mg.armor50k()
    frames = torch.stack([torch.from_numpy(mg.frame_positions(mesh["pos"], t, 4096)) for t in range(8)]).cuda()
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 4)
        m.refine("cc", 4)
        out = m.eval_frames(frames, 4)
        diag = diag_of(mesh)
        for t in (0, 5):
            m2 = dict(mesh)
            m2["pos"] = mg.frame_positions(mesh["pos"], t, 4096)
            want = oracle.refine(m2, "cc", 4)[-1]["pos"]
            err = float(np.abs(out[t].cpu().numpy().astype(np.float64) - want).max()) / diag
            assert err <= TOL, f"frame {t}: {err:.3e}"


def test_graph_and_eager_bitwise_equal(monkeypatch):
    Mesh = _gpu()
    mesh = mg.armor(6, 5, 6, 1, 1, 2, name="armor_small")
    outs = []
    for env in ("0", "1"):
        monkeypatch.setenv("ALSUB_NO_GRAPH", env)
        with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
            m.refine("cc", 4)
            m.refine("cc", 4)  # replay
            outs.append((m.positions(4).cpu(), m.topology(4)["face_vtx"].cpu()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_eval_frames_equals_refine():
    """Static mode reproduces dynamic mode bitwise for the same vertex data."""
    Mesh = _gpu()
    mesh = mg.armor(8, 6, 7, 1, 2, 2, name="armor_f")
    P0 = torch.from_numpy(mesh["pos"]).cuda()
    frames = torch.stack([torch.from_numpy(mg.frame_positions(mesh["pos"], t, 64)) for t in range(5)]).cuda()
    with Mesh(mesh["face_off"], mesh["face_vtx"], P0, mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 3)
        out = m.eval_frames(frames, 3)
        for t in range(5):
            m.set_positions(frames[t])
            m.refine("cc", 3)
            ref = m.positions(3)
            assert torch.equal(out[t], ref), f"frame {t}"
    # and against the oracle for one frame
    m2 = dict(mesh)
    m2["pos"] = mg.frame_positions(mesh["pos"], 3, 64)
    w = oracle.refine(m2, "cc", 3)[-1]["pos"]
    assert np.abs(out[3].cpu().numpy() - w).max() / diag_of(mesh) < TOL


def test_eval_frames_loop_and_sqrt3():
    Mesh = _gpu()
    for mesh, scheme in ((mg.tetrahedron(creased=True), "loop"), (mg.torus_tris(10, 8), "sqrt3")):
        fr = torch.stack([torch.from_numpy(mg.random_positions(mesh, seed=s)["pos"]) for s in range(3)]).cuda()
        with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
            m.refine(scheme, 3)
            out = m.eval_frames(fr, 3)
            for s in range(3):
                mm = mg.random_positions(mesh, seed=s)
                w = oracle.refine(mm, scheme, 3)[-1]["pos"]
                d = diag_of(mm)
                assert np.abs(out[s].cpu().numpy() - w).max() / d < TOL


def test_host_pointers_roundtrip():
    """C-ABI with HOST buffers in and out (the e2e path of bench.py)."""
    from paper_1809_06047_b200 import alsub as A
    import ctypes as C
    mesh = mg.cube()
    L = A.lib()
    h = C.c_void_p()
    st = L.alsub_mesh_create(mesh["face_off"].ctypes.data, mesh["face_vtx"].ctypes.data, 6, mesh["pos"].ctypes.data,
                             8, None, None, 0, None, None, C.byref(h))
    assert st == 0
    assert L.alsub_refine(h, 0, 2, None) == 0
    out = np.zeros((98, 3), np.float32)
    fv = np.zeros(96 * 4, np.int32)
    assert L.alsub_level_positions(h, 2, out.ctypes.data, None) == 0
    assert L.alsub_level_topology(h, 2, fv.ctypes.data, None, None, None, None, None, None, None) == 0
    w = oracle.refine(mesh, "cc", 2)[-1]
    assert np.array_equal(fv, w["face_vtx"]) and np.abs(out - w["pos"]).max() < 1e-6
    L.alsub_mesh_destroy(h)


def test_error_statuses():
    from paper_1809_06047_b200 import AlsubError
    Mesh = _gpu()
    pos = np.zeros((5, 3), np.float32)

    def status(mesh, scheme=None):
        try:
            with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
                if scheme:
                    m.refine(scheme, 1)
        except AlsubError as e:
            return e.status
        return "OK"

    assert status(mg._pack([(0, 1, 2), (0, 1, 3)], pos)) == "E_NONMANIFOLD"
    assert status(mg._pack([(0, 1, 2), (1, 0, 3), (0, 1, 4)], pos)) == "E_NONMANIFOLD"
    assert status(mg._pack([(0, 1, 7)], pos)) == "E_MESH"
    assert status(mg._pack([(0, 1)], pos)) == "E_MESH"
    assert status(mg._pack([(0, 1, 1, 2)], pos)) == "E_MESH"
    c = mg.cube()
    assert status(dict(c, crease=np.array([[0, 7]], np.int32), sigma=np.array([1.0], np.float32))) == "E_CREASE"
    assert status(dict(c, crease=np.array([[0, 1]], np.int32), sigma=np.array([-1.0], np.float32))) == "E_CREASE"
    assert status(dict(c, crease=np.array([[0, 1], [1, 0]], np.int32), sigma=np.array([1.0, 2.0], np.float32))) == "E_CREASE"
    assert status(c, "loop") == "E_SCHEME"
    assert status(mg.grid(2, 2, tri_cells=[(0, 0), (1, 0), (0, 1), (1, 1)]), "sqrt3") == "E_SCHEME"
    # two closed fans glued at a vertex (two tetrahedra sharing vertex 0)
    tpos = np.random.default_rng(0).standard_normal((7, 3)).astype(np.float32)
    f1 = [(0, 1, 2), (0, 3, 1), (0, 2, 3), (1, 3, 2)]
    f2 = [(0, 4, 5), (0, 6, 4), (0, 5, 6), (4, 6, 5)]
    assert status(mg._pack(f1 + f2, tpos)) == "E_NONMANIFOLD"


def test_empty_and_isolated():
    Mesh = _gpu()
    # isolated vertex 4 passes through unchanged
    mesh = mg._pack([(0, 1, 2, 3)], [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (5, 5, 5)])
    compare(mesh, "cc", 2)
    # levels = 0 returns the input
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"]) as m:
        m.refine("cc", 0)
        assert np.array_equal(m.positions(0).cpu().numpy(), mesh["pos"])


def test_deterministic():
    Mesh = _gpu()
    mesh = mg.armor(6, 5, 6, 1, 1, 2, name="armor_small")
    res = []
    for _ in range(2):
        with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
            m.refine("cc", 4)
            res.append(m.positions(4).cpu())
    assert torch.equal(res[0], res[1])


# ------------------------------------------------------------------------------------------
# more edge cases
# ------------------------------------------------------------------------------------------

def test_parity_shuffled_armor_L4():
    """Locality stress: seeded random vertex/face relabelling + face rotations."""
    compare(mg.shuffled(mg.armor9k()), "cc", 4, edges=True)


def test_loop_boundary_and_creases():
    """Loop on an open creased triangle grid: boundary = inf creases (reading R14) + semi-sharp."""
    m = mg.grid(5, 4, tri_cells=[(i, j) for i in range(5) for j in range(4)])
    vid = lambda i, j: j * 6 + i
    m["crease"] = np.array([(vid(1, 2), vid(2, 2)), (vid(2, 2), vid(3, 2)), (vid(2, 1), vid(2, 2))], np.int32)
    m["sigma"] = np.array([2.5, 0.5, np.inf], np.float32)
    compare(m, "loop", 4)


def test_plan_switch_and_dynamic_positions():
    """The same handle refined with different schemes/levels, and new positions after the graph
    was recorded (the graph reads the handle's level-0 buffer)."""
    Mesh = _gpu()
    mesh = mg.torus_tris(10, 8)
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"]) as m:
        for scheme, L in (("loop", 3), ("sqrt3", 2), ("cc", 3), ("cc", 3), ("cc", 3)):
            m.refine(scheme, L)
            w = oracle.refine(mesh, scheme, L)[-1]
            assert np.array_equal(m.topology(L)["face_vtx"].cpu().numpy(), w["face_vtx"])
            assert np.abs(m.positions(L).cpu().numpy() - w["pos"]).max() / diag_of(mesh) < TOL
        m2 = mg.random_positions(mesh, seed=9)
        m.set_positions(torch.from_numpy(m2["pos"]).cuda())
        m.refine("cc", 3)  # graph replay
        w = oracle.refine(m2, "cc", 3)[-1]
        assert np.abs(m.positions(3).cpu().numpy() - w["pos"]).max() / diag_of(m2) < TOL


def test_eval_frames_many_batches_host_buffers():
    """19 frames (2 full batches of 8 + a partial one), host input and output buffers."""
    Mesh = _gpu()
    mesh = mg.armor(6, 5, 6, 1, 1, 2, name="armor_small")
    frames = np.stack([mg.frame_positions(mesh["pos"], t, 19) for t in range(19)])
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 4)
        VL = m.counts(4)["verts"]
        out = np.zeros((19, VL, 3), np.float32)
        from paper_1809_06047_b200 import alsub as A
        A._check(A.lib().alsub_eval_frames(m._h, 4, frames.ctypes.data, 19, out.ctypes.data, None))
        for t in (0, 8, 18):
            mm = dict(mesh)
            mm["pos"] = frames[t]
            w = oracle.refine(mm, "cc", 4)[-1]["pos"]
            assert np.abs(out[t] - w).max() / diag_of(mesh) < TOL
        # levels below the refined depth
        out2 = m.eval_frames(torch.from_numpy(frames[:3]).cuda(), 2)
        w = oracle.refine(dict(mesh, pos=frames[2]), "cc", 2)[-1]["pos"]
        assert np.abs(out2[2].cpu().numpy() - w).max() / diag_of(mesh) < TOL


def test_overflow_is_reported():
    """A level whose counts exceed int32 ids is refused with E_OVERFLOW, not computed wrongly."""
    from paper_1809_06047_b200 import AlsubError
    Mesh = _gpu()
    mesh = mg.cube()
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"]) as m:
        with pytest.raises(AlsubError) as ei:
            m.refine("cc", 15)  # 6 * 4^15 faces * 4 slots > 2^31
        assert ei.value.status == "E_OVERFLOW"
        m.refine("cc", 2)  # the handle stays usable


def test_level_counts_and_errors():
    from paper_1809_06047_b200 import AlsubError
    Mesh = _gpu()
    mesh = mg.cube()
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"]) as m:
        c0 = m.counts(0)
        assert (c0["verts"], c0["faces"], c0["edges"], c0["face_order"]) == (8, 6, 12, 4)
        with pytest.raises(AlsubError):
            m.counts(1)  # not refined yet
        m.refine("cc", 2)
        assert m.counts(2)["faces"] == 96
        with pytest.raises(AlsubError):
            m.refine("cc", -1)
        with pytest.raises(AlsubError):
            m.positions(3)


def test_device_tensor_inputs():
    Mesh = _gpu()
    mesh = mg.icosahedron()
    t = lambda a: torch.from_numpy(a).cuda()
    with Mesh(t(mesh["face_off"]), t(mesh["face_vtx"]), t(mesh["pos"])) as m:
        m.refine("loop", 3)
        w = oracle.refine(mesh, "loop", 3)[-1]
        assert np.array_equal(m.topology(3)["face_vtx"].cpu().numpy(), w["face_vtx"])


def test_eval_attributes_channels():
    """Extra vertex channels (NEXT-4, reading R22): every channel refined with the position
    stencils, including boundaries and creases; checked against the oracle channel by channel."""
    Mesh = _gpu()
    mesh = mg.armor(8, 6, 7, 1, 2, 2, name="armor_attr")
    L = 3
    for C in (1, 2, 5):
        attr = mg.vertex_channels(mesh, C)
        with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
            m.refine("cc", L)
            got_dev = m.eval_attributes(torch.from_numpy(attr).cuda(), L).cpu().numpy()
            got_host = np.zeros_like(got_dev)
            m.eval_attributes(attr, L, out=got_host)
        assert np.array_equal(got_dev, got_host)
        assert got_dev.shape[1] == C
        for g in range(0, C, 3):
            cols = attr[:, g:g + 3]
            pad = np.zeros((attr.shape[0], 3), np.float32)
            pad[:, :cols.shape[1]] = cols
            m2 = dict(mesh)
            m2["pos"] = pad
            want = oracle.refine(m2, "cc", L)[-1]["pos"][:, :cols.shape[1]]
            scale = float(np.linalg.norm(pad.max(0) - pad.min(0)))
            err = np.abs(got_dev[:, g:g + 3] - want).max() / scale
            assert err <= TOL, f"C={C} channels {g}..: {err:.3e}"


def test_eval_attributes_match_frames_bitwise():
    """Three channels are exactly one frame of alsub_eval_frames."""
    Mesh = _gpu()
    mesh = mg.armor(8, 6, 7, 1, 2, 2, name="armor_attr")
    attr = mg.vertex_channels(mesh, 3)
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 3)
        a = m.eval_attributes(torch.from_numpy(attr).cuda(), 3)
        f = m.eval_frames(torch.from_numpy(attr).cuda()[None], 3)[0]
        assert torch.equal(a, f)


@pytest.mark.parametrize("scheme,mesh_fn,L,k", [
    ("cc", lambda: mg.armor(8, 6, 7, 1, 2, 2, name="armor_edit"), 3, 1),
    ("cc", lambda: mg.armor(8, 6, 7, 1, 2, 2, name="armor_edit"), 4, 2),
    ("loop", lambda: mg.tetrahedron(creased=True), 3, 1),
    ("sqrt3", lambda: mg.torus_tris(10, 8), 3, 2),
])
def test_hierarchical_edit_reevaluate(scheme, mesh_fn, L, k):
    """Displacement / hierarchical edit at level k: write the level-k positions
    through the handle's view, re-evaluate levels k+1..L; equals the oracle refining the edited
    level-k mesh L-k more times (topology and crease lists of level k from the oracle itself)."""
    Mesh = _gpu()
    mesh = mesh_fn()
    recs = oracle.refine(mesh, scheme, k)
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine(scheme, L)
        before = m.positions(L).clone()
        view = m.level_positions_view(k)
        view += torch.from_numpy(mg.displacement(view.shape[0])).cuda()
        edited = view.cpu().numpy().copy()
        m.reevaluate(k)
        got = [m.positions(lv).cpu().numpy() for lv in range(k, L + 1)]
        # topology untouched, positions changed
        assert not torch.equal(before, m.positions(L))
    mk = {"face_off": recs[k]["face_off"], "face_vtx": recs[k]["face_vtx"], "pos": edited,
          "crease": recs[k]["crease"], "sigma": recs[k]["sigma"]}
    want = oracle.refine(mk, scheme, L - k)
    diag = diag_of(mesh)
    assert np.array_equal(got[0], edited)
    for i in range(1, L - k + 1):
        err = np.abs(got[i].astype(np.float64) - want[i]["pos"]).max() / diag
        assert err <= TOL, f"level {k + i}: {err:.3e}"


def test_reevaluate_without_edit_is_bitwise_refine():
    Mesh = _gpu()
    mesh = mg.armor(8, 6, 7, 1, 2, 2, name="armor_edit")
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 4)
        ref = [m.positions(lv).clone() for lv in range(5)]
        for k in (0, 2, 3, 4):
            m.reevaluate(k)
            for lv in range(5):
                assert torch.equal(m.positions(lv), ref[lv]), f"from {k}: level {lv}"


def test_edit_and_attribute_errors():
    Mesh = _gpu()
    from paper_1809_06047_b200.alsub import AlsubError
    mesh = mg.cube()
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 2)
        with pytest.raises(AlsubError):
            m.reevaluate(3)
        with pytest.raises(AlsubError):
            m.level_positions_view(5)
        with pytest.raises(AlsubError):
            m.eval_attributes(np.zeros((8, 2), np.float32), 3)


def test_parity_large_creased_grid_unfused_levels():
    """A control mesh above the fused-crease threshold (V0 >= 2^20): every level runs the separate
    crease pass from level 0 on (boundary, sharp, semi-sharp and infinite crease lines)."""
    import math
    n = 1024
    mesh = mg.grid(n, n, z=lambda i, j: 0.05 * math.sin(0.05 * i) * math.cos(0.07 * j), name="grid1024")
    assert mesh["pos"].shape[0] >= (1 << 20)
    vid = lambda i, j: j * (n + 1) + i
    pairs, sig = [], []
    for i in range(100, 900):
        pairs.append((vid(i, 512), vid(i + 1, 512)))
        sig.append(2.5)
    for j in range(200, 700):
        pairs.append((vid(300, j), vid(300, j + 1)))
        sig.append(np.inf)
    for i in range(50, 400):
        pairs.append((vid(i, 800), vid(i + 1, 800)))
        sig.append(0.5)
    mesh["crease"] = np.asarray(pairs, np.int32)
    mesh["sigma"] = np.asarray(sig, np.float32)
    compare(mesh, "cc", 2)


def _random_creased_grid(seed):
    """Seeded fuzz mesh: open grid of random size with random triangle splits, random crease
    polylines (sigma in {0.5, 1, 2.5, inf}) and jittered positions."""
    rng = np.random.default_rng(1000 + seed)
    nx, ny = int(rng.integers(3, 11)), int(rng.integers(3, 11))
    cells = [(i, j) for i in range(nx) for j in range(ny) if rng.random() < 0.25]
    g = mg.grid(nx, ny, tri_cells=cells, z=lambda i, j: 0.0, name=f"fuzz{seed}")
    g["pos"] = (g["pos"] + rng.normal(0, 0.1, g["pos"].shape)).astype(np.float32)
    vid = lambda i, j: j * (nx + 1) + i
    creases = {}  # edge -> sigma, first polyline wins
    for _ in range(int(rng.integers(1, 4))):
        j = int(rng.integers(1, ny))
        i0, i1 = sorted(int(x) for x in rng.integers(0, nx + 1, 2))
        s = float(rng.choice([0.5, 1.0, 2.5, np.inf]))
        for i in range(i0, i1):
            creases.setdefault((vid(i, j), vid(i + 1, j)), s)
    if creases:
        g["crease"] = np.array(list(creases.keys()), np.int32).reshape(-1, 2)
        g["sigma"] = np.array(list(creases.values()), np.float32)
    return g


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_creased_grids_cc(seed):
    """Seeded random open meshes with semi-sharp / sharp crease polylines, CC levels 1-3: full
    topology bit-exact and positions within tolerance at every level."""
    g = _random_creased_grid(seed)
    compare(g, "cc", 1 + seed % 3)


@pytest.mark.parametrize("seed", range(4))
def test_fuzz_triangle_tori_loop_sqrt3(seed):
    rng = np.random.default_rng(2000 + seed)
    t = mg.torus_tris(int(rng.integers(4, 12)), int(rng.integers(4, 10)), seed=3000 + seed)
    compare(t, "loop", 1 + seed % 3)
    compare(t, "sqrt3", 1 + (seed + 1) % 3, edges=False)


def test_eval_attributes_loop_and_sqrt3():
    """Extra channels through the Loop (creased, boundary-free) and sqrt3 static paths."""
    Mesh = _gpu()
    for mesh, scheme in ((mg.tetrahedron(creased=True), "loop"), (mg.torus_tris(8, 6), "sqrt3")):
        attr = mg.vertex_channels(mesh, 2)
        with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
            m.refine(scheme, 3)
            got = m.eval_attributes(torch.from_numpy(attr).cuda(), 3).cpu().numpy()
        pad = np.zeros((attr.shape[0], 3), np.float32)
        pad[:, :2] = attr
        want = oracle.refine(dict(mesh, pos=pad), scheme, 3)[-1]["pos"][:, :2]
        scale = float(np.linalg.norm(pad.max(0) - pad.min(0)))
        assert np.abs(got - want).max() / scale <= TOL, scheme


@pytest.mark.parametrize("scheme", ["cc", "loop", "sqrt3"])
def test_high_valence_vertices(scheme):
    """Valence-40 apices: M^T rows longer than a warp's fast path (serial fallbacks), valence
    constants beyond the common range, long crease-free rings."""
    compare(mg.bipyramid(40), scheme, 2, edges=scheme != "sqrt3")


def _summary_np(frames):
    """Plain numpy definition of alsub_frame_summary (include/alsub.h): bbox and the wrapping
    checksum sum_i bits(x_i) (2 i + 1) mod 2^64 over each frame's floats in memory order."""
    B = frames.shape[0]
    flat = np.ascontiguousarray(frames, dtype=np.float32).reshape(B, -1)
    bits = flat.view(np.uint32).astype(np.uint64)
    w = 2 * np.arange(flat.shape[1], dtype=np.uint64) + np.uint64(1)
    with np.errstate(over="ignore"):
        cs = (bits * w[None, :]).sum(axis=1, dtype=np.uint64)
    xyz = flat.reshape(B, -1, 3)
    return xyz.min(axis=1), xyz.max(axis=1), cs


def test_frame_summary_matches_numpy():
    """The per-frame records the sharded frames job gathers (bench.py --config 5): exact bbox and
    checksum, for ragged sizes (V not a multiple of the block), one vertex, signed zeros."""
    from paper_1809_06047_b200 import frame_summary, split_summary
    g = np.random.default_rng(1809)
    for B, V in ((1, 1), (3, 257), (5, 100_003), (2, 1_000_000)):
        fr = g.standard_normal((B, V, 3)).astype(np.float32)
        if V > 2:
            fr[0, 1] = [-0.0, 0.0, -0.0]
        rec = frame_summary(torch.from_numpy(fr).cuda())
        bb, cs = split_summary(rec)
        lo, hi, want = _summary_np(fr)
        assert np.array_equal(bb[:, :3], lo) and np.array_equal(bb[:, 3:], hi), (B, V)
        assert np.array_equal(cs, want), (B, V)
    # a frame batch that starts off 16-B alignment (scalar path) and one with V % 4 == 0 (float4 path)
    big = torch.from_numpy(g.standard_normal(4 * 1000 * 3 + 1).astype(np.float32)).cuda()
    for fr_t in (big[1:].view(4, 1000, 3), big[:-1].view(4, 1000, 3)):
        bb, cs = split_summary(frame_summary(fr_t))
        lo, hi, want = _summary_np(fr_t.cpu().numpy())
        assert np.array_equal(cs, want) and np.array_equal(bb[:, :3], lo) and np.array_equal(bb[:, 3:], hi)
    # deterministic: two calls give identical records; a one-ulp change moves the checksum
    fr = torch.from_numpy(g.standard_normal((4, 5000, 3)).astype(np.float32)).cuda()
    a, b = frame_summary(fr), frame_summary(fr)
    assert torch.equal(a, b)
    fr2 = fr.clone()
    fr2.view(torch.int32)[2, 1234, 1] += 1
    c = frame_summary(fr2)
    assert torch.equal(a[[0, 1, 3]], c[[0, 1, 3]]) and not torch.equal(a[2], c[2])


def test_frame_summary_of_eval_frames_output():
    """Summaries of a refined frame batch equal numpy's over the same output."""
    from paper_1809_06047_b200 import Mesh, frame_summary, split_summary
    mesh = mg.armor(6, 5, 6, 1, 1, 2, name="armor_small")
    frames = np.stack([mg.frame_positions(mesh["pos"], t, 8) for t in range(8)])
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 3)
        out = m.eval_frames(torch.from_numpy(frames).cuda(), 3)
        bb, cs = split_summary(frame_summary(out))
        lo, hi, want = _summary_np(out.cpu().numpy())
        assert np.array_equal(cs, want) and np.array_equal(bb[:, :3], lo) and np.array_equal(bb[:, 3:], hi)


def test_probe_times_kernel_inside_graph():
    """alsub_probe: event-record nodes around one kernel of the captured refine; one duration per
    replay, results unchanged (bitwise) by the probe; unknown kernel names are reported."""
    from paper_1809_06047_b200 import AlsubError, Mesh
    mesh = mg.armor(6, 5, 6, 1, 1, 2, name="armor_small")
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 3)
        m.refine("cc", 3)
        ref = m.positions(3).clone()
        m.probe(2, "cc_face", 4)
        for _ in range(6):  # replays beyond `steps` reuse the last pair
            m.refine("cc", 3)
        t = m.probe_read()
        assert len(t) == 4 and all(x > 0 for x in t)
        assert torch.equal(m.positions(3), ref)
        m.probe(2, "cc_face", 4)  # re-arm: counter reset, no re-capture
        m.refine("cc", 3)
        assert len(m.probe_read()) == 1
        m.probe(2, "no_such_kernel", 2)
        m.refine("cc", 3)
        with pytest.raises(AlsubError):
            m.probe_read()
        m.probe(0, None, 0)  # disarm
        m.refine("cc", 3)
        assert m.probe_read() == [] and torch.equal(m.positions(3), ref)


def test_parity_grandparent_edge_kernel_before_last_level():
    """Level L-2 >= 3 runs the grandparent edge kernel when its crease rules are not fused: always
    for crease-free closed meshes (cube CC L5 / L6: levels 3 / 4), and on a creased open grid whose
    level 3 is above the fused-crease threshold (V3 >= 2^20: boundary words of level 4 written in
    closed form by that kernel, separate crease pass).  Full topology and positions at every level,
    static mode bitwise equal to dynamic mode."""
    compare(mg.cube(), "cc", 5)
    compare(mg.cube(), "cc", 6)
    import math
    n = 128
    g = mg.grid(n, n, tri_cells=[(5, 7), (60, 61)], z=lambda i, j: 0.1 * math.sin(0.1 * i) * math.cos(0.13 * j),
                name="grid128")
    vid = lambda i, j: j * (n + 1) + i
    pairs = [(vid(i, 64), vid(i + 1, 64)) for i in range(10, 100)] + [(vid(30, j), vid(30, j + 1)) for j in range(5, 50)]
    g["crease"] = np.asarray(pairs, np.int32)
    g["sigma"] = np.asarray([1.5] * 90 + [np.inf] * 45, np.float32)
    compare(g, "cc", 5)
    Mesh = _gpu()
    frames = torch.stack([torch.from_numpy(mg.frame_positions(g["pos"], t, 16)) for t in range(2)]).cuda()
    with Mesh(g["face_off"], g["face_vtx"], g["pos"], g["crease"], g["sigma"]) as m:
        m.refine("cc", 5)
        out = m.eval_frames(frames, 5)
        for t in range(2):
            m.set_positions(frames[t])
            m.refine("cc", 5)
            assert torch.equal(out[t], m.positions(5)), f"frame {t}"
