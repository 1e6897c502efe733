"""NEXT-3: selective / feature-adaptive subdivision, the extraction module.

CPU: the oracle (oracle/extract.py) against what the definitions fix -- a regular torus has no
extraordinary vertex, a cube is all extraordinary, a grid's extraordinary vertices are its border,
more rings select a superset -- and the locality property that makes extraction useful: the
refinement of a face depends only on its vertex neighbourhood, so refining the extracted mesh
reproduces the full refinement on every face whose neighbourhood was extracted.
GPU: alsub_mesh_extract index for index against the oracle, and the locality property on the GPU.
"""
import numpy as np
import pytest
import torch

import meshgen as mg
import oracle
from oracle import extract as ox

TOL = 1e-5


def _armor():
    return mg.armor(8, 6, 7, 1, 2, 2, name="armor_ex")


def _rec(mesh):
    r = oracle.level0(mesh)
    return r


def test_regular_torus_has_nothing_to_extract():
    m, vm, fm = ox.extract(_rec(mg.torus_quads(8, 6)))
    assert len(vm) == 0 and len(fm) == 0 and len(m["face_vtx"]) == 0


def test_cube_is_all_extraordinary():
    cube = mg.cube()
    m, vm, fm = ox.extract(_rec(cube))
    assert vm == list(range(8)) and fm == list(range(6))
    assert np.array_equal(m["face_vtx"], cube["face_vtx"]) and np.array_equal(m["face_off"], cube["face_off"])


def test_grid_border_ring():
    nx, ny = 7, 5
    m, vm, fm = ox.extract(_rec(mg.grid(nx, ny)))
    assert len(fm) == nx * ny - (nx - 2) * (ny - 2)
    m2, vm2, fm2 = ox.extract(_rec(mg.grid(nx, ny)), rings=2)
    assert len(fm2) == nx * ny - (nx - 4) * (ny - 4)
    assert set(fm) <= set(fm2) and set(vm) <= set(vm2)


def _neighbourhood_complete(rec, fmap):
    """Faces all of whose vertex-adjacent faces are in fmap."""
    off, vtx = rec["face_off"], rec["face_vtx"]
    F = len(off) - 1
    sel = np.zeros(F, bool)
    sel[np.asarray(fmap, np.int64)] = True
    faces_of = {}
    for r in range(F):
        for v in vtx[off[r]:off[r + 1]]:
            faces_of.setdefault(int(v), []).append(r)
    out = []
    for r in range(F):
        if sel[r] and all(sel[s] for v in vtx[off[r]:off[r + 1]] for s in faces_of[int(v)]):
            out.append(r)
    return out


def _desc_rows(face_off, r, k):
    lo, hi = ox.descendant_slots(face_off, r, k)
    return lo, hi


@pytest.mark.parametrize("rings", [1, 2])
def test_oracle_locality_cc(rings):
    """refine(extract(M)) == refine(M) on the descendants of every face whose vertex
    neighbourhood was extracted (fp64, creases and boundaries included)."""
    mesh = _armor()
    rec = _rec(mesh)
    sub, vm, fm = ox.extract(rec, rings=rings)
    full = oracle.refine(mesh, "cc", 2)
    part = oracle.refine(sub, "cc", 2)
    inner = _neighbourhood_complete(rec, fm)
    assert len(inner) > 0
    newf = {r: i for i, r in enumerate(fm)}
    for r in inner:
        a = _desc_rows(rec["face_off"], r, 2)
        b = _desc_rows(sub["face_off"], newf[r], 2)
        assert a[1] - a[0] == b[1] - b[0]
        A = full[2]["pos"][full[2]["face_vtx"][4 * a[0]:4 * a[1]]]
        B = part[2]["pos"][part[2]["face_vtx"][4 * b[0]:4 * b[1]]]
        assert np.abs(A - B).max() <= 1e-12


def test_oracle_locality_loop_masked():
    """Loop with a caller mask (valence != 6 on a triangle torus): descendants 4^k r .. of every
    triangle whose neighbourhood was extracted match the full refinement."""
    mesh = mg.torus_tris(12, 10)
    rec = _rec(mesh)
    n = ox.valence(rec)
    sub, vm, fm = ox.extract(rec, vsel=[x != 6 for x in n], rings=2)
    full = oracle.refine(mesh, "loop", 2)
    part = oracle.refine(sub, "loop", 2)
    inner = _neighbourhood_complete(rec, fm)
    assert len(inner) > 0
    newf = {r: i for i, r in enumerate(fm)}
    for r in inner:
        A = full[2]["pos"][full[2]["face_vtx"][3 * 16 * r:3 * 16 * (r + 1)]]
        s = newf[r]
        B = part[2]["pos"][part[2]["face_vtx"][3 * 16 * s:3 * 16 * (s + 1)]]
        assert np.abs(A - B).max() <= 1e-12


# ------------------------------------------------------------------------------------------ GPU
@pytest.mark.gpu
# level 3 of a 3-level refine: the last level's crease lists are built lazily (on first use)
@pytest.mark.parametrize("level,mask,rings", [(0, None, 1), (0, "random", 2), (2, None, 1), (2, "random", 1),
                                              (3, "random", 1)])
def test_gpu_extract_matches_oracle(level, mask, rings):
    from paper_1809_06047_b200 import Mesh
    mesh = _armor()
    recs = oracle.refine(mesh, "cc", max(level, 1))
    rec = recs[level]
    V = len(rec["pos"])
    vsel = None
    if mask == "random":
        vsel = (np.random.default_rng(5).random(V) < 0.02).astype(np.uint8)
    want, wvm, wfm = ox.extract(rec, vsel=vsel, rings=rings)
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", max(level, 1))
        Pl = m.positions(level).cpu().numpy()
        sub, vm, fm = m.extract(level, vsel=vsel, rings=rings)
        with sub:
            assert np.array_equal(vm.cpu().numpy(), np.asarray(wvm, np.int32))
            assert np.array_equal(fm.cpu().numpy(), np.asarray(wfm, np.int32))
            sub.refine("cc", 0)
            t = sub.topology(0, creases=True)
            assert np.array_equal(t["face_off"].cpu().numpy(), want["face_off"])
            assert np.array_equal(t["face_vtx"].cpu().numpy(), want["face_vtx"])
            got_c = sorted(zip(map(tuple, t["crease"].cpu().numpy().tolist()), t["sigma"].cpu().numpy().tolist()))
            # the handle lists live creases on interior edges only (R19/R20): a crease that became a
            # border edge of the extracted mesh is a boundary (infinitely sharp) edge there
            cnt = {}
            off, fv = want["face_off"], want["face_vtx"]
            for r in range(len(off) - 1):
                f = fv[off[r]:off[r + 1]]
                for t in range(len(f)):
                    e = (min(f[t], f[(t + 1) % len(f)]), max(f[t], f[(t + 1) % len(f)]))
                    cnt[e] = cnt.get(e, 0) + 1
            want_c = sorted((tuple(c), s) for c, s in zip(want["crease"].tolist(), want["sigma"].tolist())
                            if cnt[tuple(c)] == 2)
            assert got_c == want_c
            assert np.array_equal(sub.positions(0).cpu().numpy(), Pl[np.asarray(wvm, np.int64)])


@pytest.mark.gpu
def test_gpu_extract_refine_locality():
    """Feature-adaptive use: extract around the extraordinary vertices of level 1, refine the
    extracted mesh 2 more levels; every fully-surrounded face matches the global level-3 result."""
    from paper_1809_06047_b200 import Mesh
    mesh = _armor()
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("cc", 3)
        P3 = m.positions(3).cpu().numpy()
        T3 = m.topology(3)["face_vtx"].cpu().numpy()
        sub, vm, fm = m.extract(1, rings=2)
        fm = fm.cpu().numpy()
        rec1 = {"face_off": np.arange(0, 4 * m.counts(1)["faces"] + 1, 4, dtype=np.int32),
                "face_vtx": m.topology(1)["face_vtx"].cpu().numpy()}
        with sub:
            sub.refine("cc", 2)
            Q2 = sub.positions(2).cpu().numpy()
            S2 = sub.topology(2)["face_vtx"].cpu().numpy()
        inner = _neighbourhood_complete(rec1, fm)
        assert len(inner) > 0
        newf = {int(r): i for i, r in enumerate(fm)}
        diag = float(np.linalg.norm(mesh["pos"].max(0) - mesh["pos"].min(0)))
        worst = 0.0
        for r in inner:
            a = P3[T3[64 * r:64 * (r + 1)]]
            s = newf[r]
            b = Q2[S2[64 * s:64 * (s + 1)]]
            worst = max(worst, float(np.abs(a - b).max()))
        assert worst / diag <= TOL


@pytest.mark.gpu
def test_gpu_extract_errors():
    from paper_1809_06047_b200 import AlsubError, Mesh
    mesh = mg.cube()
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"]) as m:
        with pytest.raises(AlsubError):
            m.extract(0, rings=0)
        with pytest.raises(AlsubError):
            m.extract(2)  # no refine to level 2 yet
        sub, vm, fm = m.extract(0)
        with sub:
            assert sub.counts(0)["faces"] == 6


@pytest.mark.gpu
def test_gpu_extract_loop_level1_matches_oracle():
    """Loop: extraction from level 1 of a creased tetrahedron around a caller mask."""
    from paper_1809_06047_b200 import Mesh
    mesh = mg.tetrahedron(creased=True)
    rec = oracle.refine(mesh, "loop", 1)[1]
    vsel = np.zeros(len(rec["pos"]), np.uint8)
    vsel[[0, 5]] = 1
    want, wvm, wfm = ox.extract(rec, vsel=vsel, rings=1)
    with Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"]) as m:
        m.refine("loop", 1)
        sub, vm, fm = m.extract(1, vsel=vsel, rings=1)
        with sub:
            assert np.array_equal(vm.cpu().numpy(), np.asarray(wvm, np.int32))
            assert np.array_equal(fm.cpu().numpy(), np.asarray(wfm, np.int32))
            sub.refine("loop", 0)
            t = sub.topology(0)
            assert np.array_equal(t["face_vtx"].cpu().numpy(), want["face_vtx"])
