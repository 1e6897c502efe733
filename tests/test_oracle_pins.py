"""Pins of the CPU oracle against what the paper and the mathematics fix (task rule ③).

None of these re-type the oracle's formulas: each checks a value printed or derived by hand
(tests/golden/), a closed-form count, an invariant (Euler characteristic, affine invariance,
planarity), a textbook special case (bicubic / quartic box-spline masks on regular grids,
cubic B-spline curves along infinitely sharp creases), or an independent exact-rational brute
force (tests/bruteforce.py).
"""
import json
import math
import os
from fractions import Fraction as Q

import numpy as np
import pytest

import meshgen as mg
import oracle
from tests import bruteforce as bf

GOLD = os.path.join(os.path.dirname(__file__), "golden")
HAND = json.load(open(os.path.join(GOLD, "hand_values.json")))
PAPER = json.load(open(os.path.join(GOLD, "paper_counts.json")))


def q3(v):
    return np.array([float(Q(*c)) for c in v])


def edge_index(rec, a, b):
    ev = rec["edge_vtx"]
    lo, hi = min(a, b), max(a, b)
    idx = np.nonzero((ev[:, 0] == lo) & (ev[:, 1] == hi))[0]
    assert len(idx) == 1
    return int(idx[0])


def euler(rec):
    return rec["V"] - rec["E"] + rec["F"]


# ------------------------------------------------------------------------------------------
# hand values (tests/golden/hand_values.json)
# ------------------------------------------------------------------------------------------

def test_cc_cube_hand_values():
    g = HAND["cc_cube_L1"]
    r = oracle.refine(mg.cube(), "cc", 1)
    p0, p1 = r[0], r[1]
    for v, val in g["vertex"].items():
        np.testing.assert_allclose(p1["pos"][int(v)], q3(val), atol=1e-15)
    e = edge_index(p0, 0, 1)
    np.testing.assert_allclose(p1["pos"][8 + 6 + e], q3(g["edge"]["0-1"]), atol=1e-15)
    np.testing.assert_allclose(p1["pos"][8 + 0], q3(g["face_center_z0"]), atol=1e-15)
    assert (p1["V"], p1["F"], p0["E"]) == (g["counts"]["V"], g["counts"]["F"], g["counts"]["E_parent"])


def test_cc_tet_hand_values():
    g = HAND["cc_tet_L1"]
    r = oracle.refine(mg.tetrahedron(), "cc", 1)
    np.testing.assert_allclose(r[1]["pos"][0], q3(g["vertex"]["0"]), atol=1e-15)
    np.testing.assert_allclose(r[1]["pos"][4 + 4 + edge_index(r[0], 0, 1)], q3(g["edge"]["0-1"]), atol=1e-15)
    np.testing.assert_allclose(r[1]["pos"][4 + 0], q3(g["face_0_1_2"]), atol=1e-15)


def test_loop_tet_hand_values():
    g = HAND["loop_tet_L1"]
    r = oracle.refine(mg.tetrahedron(), "loop", 1)
    np.testing.assert_allclose(r[1]["pos"][0], q3(g["vertex"]["0"]), atol=1e-15)
    np.testing.assert_allclose(r[1]["pos"][4 + edge_index(r[0], 0, 1)], q3(g["edge"]["0-1"]), atol=1e-15)


def test_sqrt3_tet_hand_values():
    g = HAND["sqrt3_tet_L1"]
    r = oracle.refine(mg.tetrahedron(), "sqrt3", 1)
    np.testing.assert_allclose(r[1]["pos"][0], q3(g["vertex"]["0"]), atol=1e-15)
    assert (r[1]["V"], r[1]["F"]) == (g["counts"]["V"], g["counts"]["F"])


@pytest.mark.parametrize("scheme", ["loop", "cc"])
def test_creased_tet_hand_values(scheme):
    g = HAND["loop_creased_tet_L1" if scheme == "loop" else "cc_creased_tet_L1"]
    r = oracle.refine(mg.tetrahedron(creased=True), scheme, 1)
    p0, p1 = r[0], r[1]
    base = 4 if scheme == "loop" else 8
    for v, val in g["vertex"].items():
        np.testing.assert_allclose(p1["pos"][int(v)], q3(val), atol=1e-15, err_msg=f"vertex {v}")
    for k, val in g["edge"].items():
        a, b = map(int, k.split("-"))
        np.testing.assert_allclose(p1["pos"][base + edge_index(p0, a, b)], q3(val), atol=1e-15, err_msg=f"edge {k}")
    if "child_sigma" in g:
        got = {(int(a), int(b)): float(s) for (a, b), s in zip(p1["crease"], p1["sigma"])}
        for k, val in g["child_sigma"].items():
            x, e = k.split("-e")
            ep = base + edge_index(p0, int(e[0]), int(e[1]))
            want = math.inf if val == "inf" else float(Q(*val))
            assert got[(int(x), ep)] == want, k
        assert len(got) == len(g["child_sigma"])


def test_scheme_weights():
    g = HAND["weights"]
    for n, v in g["loop_beta"].items():
        assert oracle.loop_beta(int(n)) == pytest.approx(float(Q(*v)), abs=1e-16)
    for n, v in g["sqrt3_alpha"].items():
        assert oracle.sqrt3_alpha(int(n)) == pytest.approx(float(Q(*v)), abs=1e-16)


def test_boundary_L_shape():
    """Eq. CC_boundary on an L-shaped boundary corner: a 2x2 grid minus one cell."""
    m = mg.grid(2, 2)
    off, vtx = m["face_off"], m["face_vtx"]
    keep = [0, 1, 3]  # drop cell (0,1): vertex (1,1) becomes a boundary vertex with an L-shaped turn
    faces = [vtx[off[i]:off[i + 1]] for i in keep]
    used = sorted({int(v) for f in faces for v in f})
    remap = {v: i for i, v in enumerate(used)}
    mm = mg._pack([[remap[int(v)] for v in f] for f in faces], m["pos"][used])
    r = oracle.refine(mm, "cc", 1)
    # vertex (1,1) has boundary neighbours (0,1) and (1,2): 3/4 (1,1) + 1/8 ((0,1) + (1,2))
    v = remap[4]
    np.testing.assert_allclose(r[1]["pos"][v][:2], [0.75 + 0.125 * 1, 0.75 + 0.125 * 3], atol=1e-15)
    # the SPEC L-shape: boundary (0,0),(1,0),(1,1) at corner (1,0) of a 1x1 quad's neighbour
    g = HAND["boundary_L_shape"]
    corner = 0.75 * np.array([1.0, 0.0]) + 0.125 * (np.array([0.0, 0.0]) + np.array([1.0, 1.0]))
    np.testing.assert_allclose(corner, q3(g["value"]), atol=1e-15)
    sq = oracle.refine(mg.single_quad(), "cc", 1)
    np.testing.assert_allclose(sq[1]["pos"][1], q3(g["value"]) .tolist() + [0.0], atol=1e-15)


# ------------------------------------------------------------------------------------------
# counts, Euler characteristic, growth factors vs the paper's tables
# ------------------------------------------------------------------------------------------

MESHES = {
    "cube": mg.cube, "tet": mg.tetrahedron, "ico": mg.icosahedron,
    "grid": lambda: mg.grid(3, 2, tri_cells=[(1, 0)]), "torus": lambda: mg.torus_tris(6, 5),
    "armor_small": lambda: mg.armor(6, 5, 6, 1, 1, 2, name="armor_small"),
}


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("scheme", ["cc", "loop", "sqrt3"])
def test_counts_closed_forms_and_euler(name, scheme):
    mesh = MESHES[name]()
    tri = mg.uniform_faces(mesh) is not None and mg.uniform_faces(mesh).shape[1] == 3
    if scheme != "cc" and not tri:
        with pytest.raises(oracle.OracleError) as ei:
            oracle.refine(mesh, scheme, 1)
        assert ei.value.status == "E_SCHEME"
        return
    closed = oracle.edges_of(oracle.level0(mesh))["B"] == 0
    if scheme == "sqrt3" and not closed:
        with pytest.raises(oracle.OracleError):
            oracle.refine(mesh, scheme, 1)
        return
    levels = 3
    recs = oracle.refine(mesh, scheme, levels, edges_last=True)
    for a, b in zip(recs[:-1], recs[1:]):
        S = int(a["face_off"][-1])
        if scheme == "cc":
            assert (b["V"], b["F"], b["E"], b["B"]) == (a["V"] + a["F"] + a["E"], S, 2 * a["E"] + S, 2 * a["B"])
        elif scheme == "loop":
            assert (b["V"], b["F"], b["E"], b["B"]) == (a["V"] + a["E"], 4 * a["F"], 2 * a["E"] + 3 * a["F"], 2 * a["B"])
        else:
            assert (b["V"], b["F"], b["E"], b["B"]) == (a["V"] + a["F"], 3 * a["F"], 3 * a["E"], 0)
        assert euler(a) == euler(b)  # chi preserved
        if a["B"] == 0:
            assert b["B"] == 0  # closed stays closed


def test_paper_count_sqrt3_fox():
    """A closed 313-vertex / 622-face triangulated sphere reproduces fox's Table 3 counts."""
    g = PAPER["sqrt3_fox"]
    sph = sphere_mesh(g["V0"])
    assert (sph["pos"].shape[0], len(sph["face_off"]) - 1) == (g["V0"], g["F0"])
    recs = oracle.refine(sph, "sqrt3", 4)
    F, V = recs[-1]["F"], recs[-1]["V"]
    for _ in range(g["levels"] - 4):  # remaining levels by the verified closed form
        V, F = V + F, 3 * F
    assert F == 453438 and V == 226721
    assert abs(F - g["F"]) < g["rounding"] and abs(V - g["V"]) < g["rounding"]
    assert recs[2]["F"] == PAPER["sqrt3_one_to_nine"]["factor"] * recs[0]["F"]


def test_paper_count_cc_armorguy_scale():
    """armor9k (8,590 F / 10,000 V) lands on ArmorGuy's level-6 scale (Table 1)."""
    g = PAPER["cc_armorguy"]
    recs = oracle.refine(mg.armor9k(), "cc", 2)
    V, F, E = recs[-1]["V"], recs[-1]["F"], None
    e = oracle.edges_of(recs[-1])
    E = e["E"]
    for _ in range(g["levels"] - 2):
        V, F, E = V + F + E, 4 * F, 2 * E + 4 * F
    assert F == 34897920 and V == 34992080
    assert abs(F - g["F"]) / g["F"] < 0.01 and abs(V - g["V"]) / g["V"] < 0.01


def sphere_mesh(nv, seed=1809):
    """Closed triangulated sphere: convex hull of nv seeded points (scipy), outward CCW."""
    from scipy.spatial import ConvexHull
    rng = np.random.default_rng(seed)
    p = rng.standard_normal((nv, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    hull = ConvexHull(p)
    faces = []
    for s in hull.simplices:
        a, b, c = p[s]
        if np.dot(np.cross(b - a, c - a), a) < 0:
            s = s[[0, 2, 1]]
        faces.append(list(s))
    return mg._pack(faces, p)


# ------------------------------------------------------------------------------------------
# textbook special cases: regular-grid masks
# ------------------------------------------------------------------------------------------

def test_cc_regular_grid_is_bicubic_bspline():
    """On a closed regular quad torus every CC rule reduces to the uniform bicubic B-spline masks:
    vertex 9/16, 3/32 x 4 edge neighbours, 1/64 x 4 diagonals; edge 3/8 x 2, 1/16 x 4."""
    nu, nv = 7, 6
    m = mg.random_positions(mg.torus_quads(nu, nv), seed=7)
    r = oracle.refine(m, "cc", 1)
    P, Pn = r[0]["pos"], r[1]["pos"]
    vid = lambda i, j: (j % nv) * nu + (i % nu)
    for j in range(nv):
        for i in range(nu):
            want = 9 / 16 * P[vid(i, j)] \
                + 3 / 32 * (P[vid(i + 1, j)] + P[vid(i - 1, j)] + P[vid(i, j + 1)] + P[vid(i, j - 1)]) \
                + 1 / 64 * (P[vid(i + 1, j + 1)] + P[vid(i - 1, j + 1)] + P[vid(i + 1, j - 1)] + P[vid(i - 1, j - 1)])
            np.testing.assert_allclose(Pn[vid(i, j)], want, atol=1e-13)
            # horizontal edge (i,j)-(i+1,j)
            e = edge_index(r[0], vid(i, j), vid(i + 1, j))
            want = 3 / 8 * (P[vid(i, j)] + P[vid(i + 1, j)]) + 1 / 16 * (
                P[vid(i, j + 1)] + P[vid(i + 1, j + 1)] + P[vid(i, j - 1)] + P[vid(i + 1, j - 1)])
            np.testing.assert_allclose(Pn[nu * nv * 2 + e], want, atol=1e-13)


def test_loop_regular_grid_is_box_spline():
    """Regular (valence 6) Loop vertex mask: 5/8 p + 1/16 sum of the 6 neighbours."""
    nu, nv = 7, 6
    m = mg.random_positions(mg.torus_tris(nu, nv, regular=True), seed=3)
    r = oracle.refine(m, "loop", 1)
    P, Pn = r[0]["pos"], r[1]["pos"]
    ev = r[0]["edge_vtx"]
    for v in range(nu * nv):
        nb = np.concatenate([ev[ev[:, 0] == v, 1], ev[ev[:, 1] == v, 0]])
        assert len(nb) == 6
        np.testing.assert_allclose(Pn[v], 5 / 8 * P[v] + 1 / 16 * P[nb].sum(0), atol=1e-13)


def test_sqrt3_regular_grid_mask():
    """Regular (valence 6) sqrt3 vertex mask: alpha_6 = 1/3 -> 2/3 p + 1/18 sum of 6 neighbours."""
    nu, nv = 6, 6
    m = mg.random_positions(mg.torus_tris(nu, nv, regular=True), seed=4)
    r = oracle.refine(m, "sqrt3", 1)
    P, Pn = r[0]["pos"], r[1]["pos"]
    ev = r[0]["edge_vtx"]
    for v in range(nu * nv):
        nb = np.concatenate([ev[ev[:, 0] == v, 1], ev[ev[:, 1] == v, 0]])
        np.testing.assert_allclose(Pn[v], 2 / 3 * P[v] + 1 / 18 * P[nb].sum(0), atol=1e-13)


# ------------------------------------------------------------------------------------------
# invariants
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("scheme,mk", [
    ("cc", lambda: mg.armor(6, 5, 6, 1, 1, 2, name="armor_small")),
    ("cc", lambda: mg.tetrahedron(creased=True)),
    ("loop", lambda: mg.tetrahedron(creased=True)),
    ("loop", mg.icosahedron),
    ("sqrt3", lambda: mg.torus_tris(8, 6)),
])
def test_affine_invariance(scheme, mk):
    """refine(A P + t) = A refine(P) + t: every row of every rule sums to one."""
    mesh = mk()
    rng = np.random.default_rng(11)
    A = rng.standard_normal((3, 3))
    t = rng.standard_normal(3)
    m2 = dict(mesh)
    m2["pos"] = (mesh["pos"].astype(np.float64) @ A.T + t)
    r1 = oracle.refine(mesh, scheme, 2)
    r2 = oracle.refine(m2, scheme, 2)
    for a, b in zip(r1, r2):
        np.testing.assert_allclose(a["pos"] @ A.T + t, b["pos"], atol=1e-9)
        assert np.array_equal(a["face_vtx"], b["face_vtx"])


def test_planarity_preserved():
    m = mg.grid(4, 3, tri_cells=[(1, 1)], z=lambda i, j: 0.25)
    for lv in oracle.refine(m, "cc", 3):
        assert np.all(lv["pos"][:, 2] == 0.25)


def test_affine_reproduction_open_grid():
    """Data affine in the grid parameters is reproduced exactly (B-spline linear precision)
    except within L-inf distance 1 of a valence-2 corner, where Eq. CC_boundary turns."""
    nx, ny = 6, 5
    m = mg.grid(nx, ny)
    prm = m["pos"][:, :2].astype(np.float64)
    A = np.array([[0.7, -0.2], [0.3, 1.1], [0.05, 0.4]])
    m["pos"] = (prm @ A.T + [0.1, -0.3, 0.2]).astype(np.float32)
    recs = oracle.refine(m, "cc", 3)
    # provenance parameters: old vertex keeps its params; face point = centroid; edge point = midpoint
    par = prm
    corners = np.array([[0, 0], [nx, 0], [0, ny], [nx, ny]], dtype=np.float64)
    for a, b in zip(recs[:-1], recs[1:]):
        off, vtx = a["face_off"], a["face_vtx"]
        fpar = np.array([par[vtx[off[r]:off[r + 1]]].mean(0) for r in range(a["F"])])
        epar = par[a["edge_vtx"]].mean(1)
        par = np.concatenate([par, fpar, epar])
        want = par @ A.T + [0.1, -0.3, 0.2]
        far = np.min(np.abs(par[:, None, :] - corners[None]).max(2), 1) > 1.0
        np.testing.assert_allclose(b["pos"][far], want[far], atol=2e-6)
        assert far.sum() > 0.5 * len(far)


# ------------------------------------------------------------------------------------------
# creases
# ------------------------------------------------------------------------------------------

def test_zero_sigma_is_smooth():
    m = mg.armor(6, 5, 6, 1, 1, 2, name="armor_small")
    m0 = dict(m)
    m0["sigma"] = np.zeros_like(m["sigma"])
    m1 = dict(m)
    m1["crease"], m1["sigma"] = m["crease"][:0], m["sigma"][:0]
    for a, b in list(zip(oracle.refine(m0, "cc", 2), oracle.refine(m1, "cc", 2)))[1:]:
        assert np.array_equal(a["pos"], b["pos"]) and np.array_equal(a["face_vtx"], b["face_vtx"])
        assert len(a["sigma"]) == 0


def test_infinite_creases_are_cubic_bspline_curves():
    """All 12 cube edges sigma = inf: corners have k = 3 (fixed), and each cube edge subdivides as an
    independent cubic B-spline polyline: midpoints, then 1/8-3/4-1/8 at interior points."""
    cube = mg.cube()
    m = dict(cube)
    ed = oracle.edges_of(oracle.level0(cube))["edge_vtx"]
    m["crease"], m["sigma"] = ed.copy(), np.full(len(ed), np.inf, np.float32)
    L = 3
    recs = oracle.refine(m, "cc", L)
    P0 = cube["pos"].astype(np.float64)
    for (a, b) in ed:
        curve = [P0[a], P0[b]]
        for lv in range(1, L + 1):
            new = [curve[0]]
            for i in range(len(curve) - 1):
                mid = 0.5 * (curve[i] + curve[i + 1])
                new.append(mid)
                nxt = curve[i + 1] if i + 1 == len(curve) - 1 else 0.125 * curve[i] + 0.75 * curve[i + 1] + 0.125 * curve[i + 2]
                new.append(nxt)
            curve = new
            # every curve point must be a vertex of the refined mesh on the cube edge
            pts = recs[lv]["pos"]
            for c in curve:
                assert np.min(np.abs(pts - c).max(1)) < 1e-14
        # crease sigma stays inf and the crease count doubles per level
    assert all(np.all(np.isinf(r["sigma"])) for r in recs)
    assert [len(r["sigma"]) for r in recs] == [12 * 2 ** l for l in range(L + 1)]


def test_chaikin_sharpness_examples():
    """SPEC S:L311 examples: a chain at sigma 4 -> children 3; sigma 1 -> the crease vanishes;
    an isolated sigma = 2 edge -> children 1 (end-of-chain reading R8)."""
    g = mg.grid(4, 3)
    vid = lambda i, j: j * 5 + i
    chain = [(vid(i, 1), vid(i + 1, 1)) for i in range(4)]

    def child_sig(sig):
        m = dict(g)
        m["crease"], m["sigma"] = np.array(chain, np.int32), np.full(4, sig, np.float32)
        return oracle.refine(m, "cc", 1)[1]["sigma"]

    s4 = child_sig(4.0)
    assert len(s4) == 8 and np.all(s4 == 3.0)
    assert len(child_sig(1.0)) == 0
    m = dict(g)
    m["crease"], m["sigma"] = np.array([chain[1]], np.int32), np.array([2.0], np.float32)
    s = oracle.refine(m, "cc", 1)[1]["sigma"]
    assert len(s) == 2 and np.all(s == 1.0)


def test_semisharp_blend_lies_between_smooth_and_sharp():
    """0 < sigma < 1 (reading R7, parity unpinned beyond this): the edge point moves along the
    segment from the smooth point (sigma = 0) to the midpoint (sigma = 1) linearly in sigma."""
    g = mg.random_positions(mg.torus_quads(6, 5), seed=5)
    pair = np.array([[0, 1]], np.int32)
    res = {}
    for s in (0.0, 0.25, 0.5, 1.0):
        m = dict(g)
        m["crease"], m["sigma"] = pair, np.array([s], np.float32)
        r = oracle.refine(m, "cc", 1)
        res[s] = r[1]["pos"][30 + 30 + edge_index(r[0], 0, 1)]
    np.testing.assert_allclose(res[0.25], 0.75 * res[0.0] + 0.25 * res[1.0], atol=1e-14)
    np.testing.assert_allclose(res[0.5], 0.5 * res[0.0] + 0.5 * res[1.0], atol=1e-14)


def _bump_grid():
    """meshgen.grid(4, 4) with z = 1 at vertex 12 = (2, 2): the hand-value fixture of the
    semi-sharp / multi-crease pins (tests/golden/hand_values.json)."""
    return mg.grid(4, 4, z=lambda i, j: 1.0 if (i, j) == (2, 2) else 0.0)


def _with_creases(m, pairs, sig):
    m = dict(m)
    m["crease"] = np.array(pairs, np.int32)
    m["sigma"] = np.array(sig, np.float32)
    return m


def _check_child_sigma(p0, p1, want, base):
    got = {(int(a), int(b)): float(s) for (a, b), s in zip(p1["crease"], p1["sigma"])}
    for k, val in want.items():
        x, e = k.split("-e")
        a, b = map(int, e.split("_"))
        key = (int(x), base + edge_index(p0, a, b))
        assert got[key] == (math.inf if val == "inf" else float(Q(*val))), k
    assert len(got) == len(want)


def test_semisharp_vertex_hand_values():
    """k = 2, s = 3/8 < 1: the vertex point is 5/8 smooth + 3/8 sharp (a swapped blend gives
    87/128, s = max sigma gives 84/128, s over all four edges 76.5/128)."""
    g = HAND["cc_semisharp_vertex_L1"]
    r = oracle.refine(_with_creases(_bump_grid(), [(11, 12), (12, 13)], [0.25, 0.5]), "cc", 1)
    p0, p1 = r
    base = 25 + 16
    for v, val in g["vertex"].items():
        np.testing.assert_allclose(p1["pos"][int(v)], q3(val), atol=1e-15, err_msg=f"vertex {v}")
    for k, val in g["edge"].items():
        a, b = map(int, k.split("-"))
        np.testing.assert_allclose(p1["pos"][base + edge_index(p0, a, b)], q3(val), atol=1e-15, err_msg=k)
    _check_child_sigma(p0, p1, g["child_sigma"], base)


@pytest.mark.parametrize("side", ["sharp", "smooth"])
def test_semisharp_vertex_continuity(side):
    """s -> 1- reaches the sharp rule and s -> 0+ the smooth one (no jump at either end of the
    blend); at s = 1 the result is the sharp rule exactly."""
    g = HAND["cc_semisharp_vertex_L1"]["limits"]
    eps = 2.0 ** -20
    for sig, tol in ([(1.0 - eps, 1e-6), (1.0, 0.0)] if side == "sharp" else [(eps, 1e-6)]):
        r = oracle.refine(_with_creases(_bump_grid(), [(11, 12), (12, 13)], [sig, sig]), "cc", 1)
        want = q3(g["sharp_12" if side == "sharp" else "smooth_12"])
        got = r[1]["pos"][12]
        assert np.abs(got - want).max() <= tol, (sig, got, want)
        if tol > 0:
            assert np.abs(got - want).max() > 0.0  # still blended


def test_three_creases_sigma_bar():
    """P:L440's three adjacent parent creases: sigma_bar excludes the edge itself (an included
    edge gives 1.0417 instead of 17/16 for the sigma = 2 edge); k = 3 makes the vertex a corner."""
    g = HAND["cc_three_creases_L1"]
    r = oracle.refine(_with_creases(_bump_grid(), [(11, 12), (12, 13), (12, 17)], [2.0, 3.0, 1.5]), "cc", 1)
    p0, p1 = r
    for v, val in g["vertex"].items():
        np.testing.assert_allclose(p1["pos"][int(v)], q3(val), atol=1e-15)
    _check_child_sigma(p0, p1, g["child_sigma"], 25 + 16)


def test_sigma_bar_excludes_inf_and_boundary():
    g = HAND["cc_sigma_bar_exclusions_L1"]
    r = oracle.refine(_with_creases(_bump_grid(), [(11, 12), (7, 12), (5, 6)], [2.0, np.inf, 2.0]), "cc", 1)
    _check_child_sigma(r[0], r[1], g["child_sigma"], 25 + 16)


def _pillow2():
    return mg._pack([(0, 1, 2, 3), (0, 3, 2, 1)], [(0, 0, 1), (1, 0, 0), (1, 1, 0), (0, 1, 0)], name="pillow2")


def _bowtie():
    return mg._pack([(0, 1, 2), (0, 3, 4)], [(0, 0, 1), (1, 0, 0), (1, 1, 0), (-1, 0, 0), (-1, -1, 0)], name="bowtie")


def test_interior_valence2_pillow():
    """Reading R17: interior vertices with n = 2 use the CC formula as written."""
    g = HAND["cc_pillow_L1"]
    r = oracle.refine(_pillow2(), "cc", 1)
    for v, val in g["vertex"].items():
        np.testing.assert_allclose(r[1]["pos"][int(v)], q3(val), atol=1e-15)
    np.testing.assert_allclose(r[1]["pos"][4 + 2 + edge_index(r[0], 0, 1)], q3(g["edge"]["0-1"]), atol=1e-15)


def test_bowtie_vertex_is_a_corner():
    """Reading R18: two open fans at a vertex are allowed; the vertex (k = 4 boundary edges) stays."""
    g = HAND["cc_bowtie_L1"]
    r = oracle.refine(_bowtie(), "cc", 1)
    for v, val in g["vertex"].items():
        np.testing.assert_allclose(r[1]["pos"][int(v)], q3(val), atol=1e-15)


def _split_edge_cube():
    """The cube with vertex 8 inserted in edge (0,1): two pentagons, and vertex 8 is an interior
    vertex of valence 2 (reading R17)."""
    c = mg.cube()
    faces = [list(c["face_vtx"][c["face_off"][i]:c["face_off"][i + 1]]) for i in range(6)]
    out = []
    for f in faces:
        g = []
        for t in range(len(f)):
            g.append(f[t])
            if {f[t], f[(t + 1) % len(f)]} == {0, 1}:
                g.append(8)
        out.append(g)
    return mg._pack(out, np.vstack([c["pos"], [[0.5, 0.0, 0.0]]]), name="cube_split_edge")


def _two_tets_sharing_a_vertex(open_second=False):
    pos = [(1, 1, 1), (1, -1, -1), (-1, 1, -1), (-1, -1, 1)]
    pos += [(3 + x, y, z) for (x, y, z) in pos[1:]]
    A = [(0, 1, 2), (0, 3, 1), (0, 2, 3), (1, 3, 2)]
    B = [(0, 4, 5), (0, 6, 4), (0, 5, 6), (4, 6, 5)]
    return mg._pack(A + (B[:1] if open_second else B), pos, name="two_fans")


# ------------------------------------------------------------------------------------------
# independent exact-rational brute force (tests/bruteforce.py)
# ------------------------------------------------------------------------------------------

def _octahedron():
    pos = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    faces = [(0, 2, 4), (2, 1, 4), (1, 3, 4), (3, 0, 4), (2, 0, 5), (1, 2, 5), (3, 1, 5), (0, 3, 5)]
    return mg._pack(faces, pos, name="octa")


def _pillow():
    """Two quads glued along their boundary + a triangle fan: closed, mixed orders."""
    pos = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0.5, 0.5, 0.7), (0.5, 0.5, -0.6)]
    faces = [(0, 1, 4), (1, 2, 4), (2, 3, 4), (3, 0, 4), (0, 3, 2, 1, 5)]  # pentagon bottom? not planar; fine
    return mg._pack(faces[:4] + [(5, 1, 0), (5, 2, 1), (5, 3, 2), (5, 0, 3)], pos, name="pillow")


BF_CASES = [
    ("cc", mg.cube, 2), ("cc", mg.tetrahedron, 2), ("cc", lambda: mg.tetrahedron(creased=True), 2),
    ("cc", lambda: mg.grid(3, 2, tri_cells=[(1, 0)]), 2), ("cc", _pillow, 2),
    ("cc", lambda: (lambda m: m.update(crease=np.array([[1, 5], [5, 9], [0, 1], [6, 7]], np.int32),
                                       sigma=np.array([0.75, 2.5, 1.5, 0.25], np.float32)) or m)(mg.grid(3, 2)), 2),
    ("cc", lambda: _with_creases(_bump_grid(), [(11, 12), (12, 13), (12, 17), (6, 7)], [0.25, 0.75, 2.5, 0.5]), 2),
    ("cc", _split_edge_cube, 2), ("cc", _pillow2, 2), ("cc", _bowtie, 2),
    ("loop", lambda: _with_creases(mg.tetrahedron(), [(0, 1), (1, 2)], [0.25, 0.75]), 1),
    ("loop", mg.tetrahedron, 1), ("loop", _octahedron, 1), ("loop", lambda: mg.tetrahedron(creased=True), 1),
    ("sqrt3", mg.tetrahedron, 1), ("sqrt3", _octahedron, 1),
    ("sqrt3", lambda: mg.torus_tris(4, 4, regular=True), 1),
]


@pytest.mark.parametrize("scheme,mk,levels", BF_CASES)
def test_oracle_equals_exact_bruteforce(scheme, mk, levels):
    mesh = mk()
    got = oracle.refine(mesh, scheme, levels)
    want = bf.refine(mesh, scheme, levels)
    for lv, (g, w) in enumerate(zip(got, want)):
        faces = [list(g["face_vtx"][g["face_off"][i]:g["face_off"][i + 1]]) for i in range(g["F"])]
        assert faces == w["faces"], f"level {lv} faces"
        np.testing.assert_allclose(g["pos"], np.array([[float(c) for c in p] for p in w["pos"]]), atol=1e-12)
        if "edges" in w:
            assert [tuple(e) for e in g["edge_vtx"]] == w["edges"], f"level {lv} edge order"
            assert [tuple(e) for e in g["edge_face"]] == w["edge_face"]
        gc = {(int(a), int(b)): float(s) for (a, b), s in zip(g["crease"], g["sigma"])}
        if lv > 0:
            assert gc == {k: v for k, v in w["creases"].items()}, f"level {lv} creases"


def test_edge_ids_ascend_in_hi_lo_order():
    """Reading R1: ids enumerate the upper triangle of E column-major."""
    r = oracle.refine(mg.armor9k(), "cc", 1, edges_last=True)
    for lv in r:
        ev = lv["edge_vtx"].astype(np.int64)
        key = ev[:, 1] * (1 << 32) + ev[:, 0]
        assert np.all(np.diff(key) > 0) and np.all(ev[:, 0] < ev[:, 1])


def test_structured_child_edge_blocks_cc():
    """Property used by the GPU's sort-free level >= 1 indexing:
    the CC child edges of parent edge e = (a < b) occupy the contiguous block starting at
    sum_{e' < e} (4 - bnd_e') in the order (a, ep), (b, ep), (fp_min, ep), (fp_max, ep)."""
    for mk in (mg.armor9k, lambda: mg.grid(3, 2, tri_cells=[(1, 0)]), mg.cube):
        r = oracle.refine(mk(), "cc", 2, edges_last=True)
        for a, b in zip(r[:-1], r[1:]):
            V, F = a["V"], a["F"]
            bnd = (a["edge_face"] < 0).any(1)
            base = np.concatenate([[0], np.cumsum(4 - bnd)])
            ev = b["edge_vtx"]
            for e in range(a["E"]):
                lo, hi = a["edge_vtx"][e]
                fr = sorted(f for f in a["edge_face"][e] if f >= 0)
                want = [(lo, V + F + e), (hi, V + F + e)] + [(V + f, V + F + e) for f in fr]
                got = [tuple(x) for x in ev[base[e]:base[e + 1]]]
                assert got == want


# ------------------------------------------------------------------------------------------
# error paths (SURVEY.md 8(b) status classes)
# ------------------------------------------------------------------------------------------

def test_error_paths():
    def err(mesh, scheme="cc"):
        with pytest.raises(oracle.OracleError) as ei:
            oracle.refine(mesh, scheme, 1)
        return ei.value.status

    pos = np.zeros((5, 3), np.float32)
    assert err(mg._pack([(0, 1, 2), (0, 1, 3)], pos)) == "E_NONMANIFOLD"          # flipped orientation
    assert err(mg._pack([(0, 1, 2), (1, 0, 3), (0, 1, 4)], pos)) == "E_NONMANIFOLD"  # 3 faces on an edge
    assert err(_two_tets_sharing_a_vertex()) == "E_NONMANIFOLD"                 # two closed fans (R18)
    assert err(_two_tets_sharing_a_vertex(open_second=True)) == "E_NONMANIFOLD"  # closed + open fan
    assert err(mg._pack([(0, 1, 7)], pos)) == "E_MESH"
    assert err(mg._pack([(0, 1)], pos)) == "E_MESH"
    assert err(mg._pack([(0, 1, 1, 2)], pos)) == "E_MESH"
    c = mg.cube()
    assert err(dict(c, crease=np.array([[0, 7]], np.int32), sigma=np.array([1.0], np.float32))) == "E_CREASE"
    assert err(dict(c, crease=np.array([[0, 1]], np.int32), sigma=np.array([-1.0], np.float32))) == "E_CREASE"
    assert err(dict(c, crease=np.array([[0, 1], [1, 0]], np.int32), sigma=np.array([1.0, 2.0], np.float32))) == "E_CREASE"
    assert err(c, "loop") == "E_SCHEME"
    assert err(mg.grid(2, 2, tri_cells=[(0, 0), (1, 0), (0, 1), (1, 1)]), "sqrt3") == "E_SCHEME"


# ------------------------------------------------------------------------------------------
# orientation (reading R13 for sqrt3, R2 for CC, a10 for Loop): a geometric pin that does not go
# through the brute force's own vertex order -- on a convex closed control mesh centred at the
# origin every refined face keeps an outward normal and the enclosed signed volume stays positive
# ------------------------------------------------------------------------------------------

def newell_normals(pos, face_off, face_vtx):
    """Newell normal and centroid of every polygon (plain definition, any order)."""
    n = np.zeros((len(face_off) - 1, 3))
    c = np.zeros_like(n)
    for r in range(len(face_off) - 1):
        p = pos[face_vtx[face_off[r]:face_off[r + 1]]]
        q = np.roll(p, -1, axis=0)
        n[r] = [np.sum((p[:, 1] - q[:, 1]) * (p[:, 2] + q[:, 2])),
                np.sum((p[:, 2] - q[:, 2]) * (p[:, 0] + q[:, 0])),
                np.sum((p[:, 0] - q[:, 0]) * (p[:, 1] + q[:, 1]))]
        c[r] = p.mean(0)
    return n, c


def signed_volume(pos, face_off, face_vtx):
    """Divergence theorem over a fan triangulation of every face: > 0 for outward orientation."""
    vol = 0.0
    for r in range(len(face_off) - 1):
        f = face_vtx[face_off[r]:face_off[r + 1]]
        for t in range(1, len(f) - 1):
            vol += np.linalg.det(np.stack([pos[f[0]], pos[f[t]], pos[f[t + 1]]])) / 6.0
    return vol


def check_outward(rec, what):
    n, c = newell_normals(rec["pos"], rec["face_off"], rec["face_vtx"])
    dots = np.einsum("ij,ij->i", n, c)
    assert (dots > 0).all(), f"{what}: {int((dots <= 0).sum())} inward faces"
    assert signed_volume(rec["pos"], rec["face_off"], rec["face_vtx"]) > 0, what


@pytest.mark.parametrize("scheme,mk", [("sqrt3", _octahedron), ("sqrt3", mg.icosahedron), ("sqrt3", mg.tetrahedron),
                                       ("loop", mg.icosahedron), ("loop", _octahedron), ("cc", mg.cube),
                                       ("cc", mg.tetrahedron)])
def test_orientation_outward_convex(scheme, mk):
    mesh = mk()
    mesh = dict(mesh, pos=mesh["pos"] - mesh["pos"].mean(0))
    for lv, rec in enumerate(oracle.refine(mesh, scheme, 3)):
        check_outward(rec, f"{scheme} {mesh['name']} L{lv}")


def test_orientation_pin_detects_a_flip():
    """The pin itself: reversing one child face's vertex order (SPEC's clockwise sqrt3 order,
    S:L496) is caught."""
    rec = oracle.refine(_octahedron(), "sqrt3", 1)[1]
    fv = rec["face_vtx"].copy()
    fv[0:3] = fv[0:3][::-1]
    with pytest.raises(AssertionError):
        check_outward(dict(rec, face_vtx=fv), "flipped")
