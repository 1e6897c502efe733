"""Seeded synthetic control meshes shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the subdivision arithmetic (task rule ③): it only
builds control meshes -- face lists, fp32 positions and crease tags -- with the shapes, sizes,
valence mixes and crease recipes of the paper's workloads (Table 1; teaser
P:L91).  Both the oracle (``oracle/``) and the CUDA path (``paper_1809_06047_b200``) consume
its output; neither is imported here.

A mesh is a plain dict::

    face_off  int32[F+1]   exclusive offsets into face_vtx (CSC column pointer of M)
    face_vtx  int32[S]     vertex ids, CCW (outward) cyclic order per face
    pos       float32[V,3] vertex positions
    crease    int32[K,2]   crease vertex pairs (any order), may be empty
    sigma     float32[K]   crease sharpness, +inf allowed
    name      str

Seeds: 1809 for topology / sharpness, 6047 for frame data.
"""
from __future__ import annotations

import math

import numpy as np

SEED_TOPO = 1809
SEED_FRAMES = 6047


def _pack(faces, pos, crease=None, sigma=None, name=""):
    faces = [list(map(int, f)) for f in faces]
    off = np.zeros(len(faces) + 1, dtype=np.int32)
    off[1:] = np.cumsum([len(f) for f in faces])
    vtx = np.fromiter((v for f in faces for v in f), dtype=np.int32, count=int(off[-1]))
    pos = np.ascontiguousarray(np.asarray(pos, dtype=np.float32).reshape(-1, 3))
    if crease is None or len(crease) == 0:
        crease = np.zeros((0, 2), dtype=np.int32)
        sigma = np.zeros((0,), dtype=np.float32)
    crease = np.ascontiguousarray(np.asarray(crease, dtype=np.int32).reshape(-1, 2))
    sigma = np.ascontiguousarray(np.asarray(sigma, dtype=np.float32).reshape(-1))
    return {"face_off": off, "face_vtx": vtx, "pos": pos, "crease": crease, "sigma": sigma, "name": name}


def uniform_faces(mesh):
    """Faces as an (F, c) array when every face has the same order c, else None."""
    off = mesh["face_off"]
    c = np.diff(off)
    if len(c) == 0 or not np.all(c == c[0]):
        return None
    return mesh["face_vtx"].reshape(-1, int(c[0]))


# ----------------------------------------------------------------------------------------------
# small closed solids (SURVEY.md §8(c) hand-value fixtures)
# ----------------------------------------------------------------------------------------------

def cube():
    """Unit cube [0,1]^3, 6 outward CCW quads (config 1)."""
    pos = [(x, y, z) for z in (0, 1) for y in (0, 1) for x in (0, 1)]  # id = x + 2y + 4z
    faces = [
        (0, 2, 3, 1),  # z = 0, normal -z
        (4, 5, 7, 6),  # z = 1, normal +z
        (0, 1, 5, 4),  # y = 0, normal -y
        (2, 6, 7, 3),  # y = 1, normal +y
        (0, 4, 6, 2),  # x = 0, normal -x
        (1, 3, 7, 5),  # x = 1, normal +x
    ]
    return _pack(faces, pos, name="cube")


def tetrahedron(creased=False):
    """Regular tetrahedron on alternate cube corners (SURVEY.md §8(c) tet fixture).

    ``creased=True`` tags sigma(0,1)=inf, sigma(1,2)=2, sigma(0,2)=5/4 (config 2b)."""
    pos = [(1, 1, 1), (1, -1, -1), (-1, 1, -1), (-1, -1, 1)]
    faces = [(0, 1, 2), (0, 3, 1), (0, 2, 3), (1, 3, 2)]
    if creased:
        return _pack(faces, pos, [(0, 1), (1, 2), (0, 2)], [np.inf, 2.0, 1.25], name="tet_creased")
    return _pack(faces, pos, name="tet")


def icosahedron():
    """Icosahedron with golden-ratio coordinates, 20 outward CCW triangles (config 2a)."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    pos = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0),
           (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
           (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
             (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
             (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
             (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    return _pack(faces, pos, name="icosahedron")


def single_quad():
    return _pack([(0, 1, 2, 3)], [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0)], name="quad")


# ----------------------------------------------------------------------------------------------
# grids
# ----------------------------------------------------------------------------------------------

def grid(nx, ny, tri_cells=(), z=None, name="grid"):
    """Open planar grid of nx*ny quads in [0,nx]x[0,ny]; cells listed in ``tri_cells`` (i, j)
    are split into two triangles along the (i,j)-(i+1,j+1) diagonal."""
    vid = lambda i, j: j * (nx + 1) + i
    pos = [(i, j, 0.0 if z is None else z(i, j)) for j in range(ny + 1) for i in range(nx + 1)]
    tri = set(map(tuple, tri_cells))
    faces = []
    for j in range(ny):
        for i in range(nx):
            a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            if (i, j) in tri:
                faces += [(a, b, c), (a, c, d)]
            else:
                faces.append((a, b, c, d))
    return _pack(faces, pos, name=name)


def torus_quads(nu, nv, R=1.0, r=0.35):
    """Closed regular quad torus (every vertex valence 4)."""
    vid = lambda i, j: (j % nv) * nu + (i % nu)
    pos = []
    for j in range(nv):
        for i in range(nu):
            u, v = 2 * math.pi * i / nu, 2 * math.pi * j / nv
            pos.append(((R + r * math.cos(v)) * math.cos(u), (R + r * math.cos(v)) * math.sin(u), r * math.sin(v)))
    faces = [(vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)) for j in range(nv) for i in range(nu)]
    return _pack(faces, pos, name=f"torus{nu}x{nv}")


def torus_tris(nu, nv, R=1.0, r=0.35, seed=SEED_TOPO, noise=0.01, regular=False):
    """Closed triangle torus: a nu x nv quad torus with every quad split on a diagonal.

    ``regular=True`` always splits on the same diagonal (every vertex valence 6);
    otherwise the diagonal is drawn per quad from ``seed`` (config 4: 250x200, valence 4-8),
    and positions get ``noise`` relative radial jitter."""
    rng = np.random.default_rng(seed)
    vid = lambda i, j: (j % nv) * nu + (i % nu)
    pos = np.zeros((nu * nv, 3))
    for j in range(nv):
        for i in range(nu):
            u, v = 2 * math.pi * i / nu, 2 * math.pi * j / nv
            pos[vid(i, j)] = ((R + r * math.cos(v)) * math.cos(u), (R + r * math.cos(v)) * math.sin(u), r * math.sin(v))
    if not regular and noise:
        pos *= (1.0 + noise * rng.standard_normal((nu * nv, 1)))
    diag = np.zeros(nu * nv, dtype=bool) if regular else rng.random(nu * nv) < 0.5
    faces = []
    for j in range(nv):
        for i in range(nu):
            a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            if diag[j * nu + i]:
                faces += [(a, b, d), (b, c, d)]
            else:
                faces += [(a, b, c), (a, c, d)]
    return _pack(faces, pos, name=f"torustri{nu}x{nv}")


# ----------------------------------------------------------------------------------------------
# ArmorGuy-shaped mixed quad/tri creased meshes (configs 3 and 5)
# ----------------------------------------------------------------------------------------------

def _cube_sphere(k, center, size):
    """Closed k x k-per-side subdivided cube surface (6k^2 quads, 6k^2+2 vertices), outward CCW."""
    verts = {}
    pos = []

    def vid(p):
        if p not in verts:
            verts[p] = len(pos)
            pos.append(p)
        return verts[p]

    faces = []
    # each side: axis a fixed at 0 or k; (u, v) span the other two axes, ordered so the
    # u x v cross product points outward.
    for axis in range(3):
        for side in (0, k):
            o1, o2 = [ax for ax in range(3) if ax != axis]
            if side == 0:
                o1, o2 = o2, o1
            # with (o1, o2) cyclic after axis, u x v = +axis; flipped for side 0.
            if (o1 - axis) % 3 != 1 and side == k:
                o1, o2 = o2, o1
            if (o1 - axis) % 3 == 1 and side == 0:
                o1, o2 = o2, o1
            for j in range(k):
                for i in range(k):
                    quad = []
                    for (di, dj) in ((0, 0), (1, 0), (1, 1), (0, 1)):
                        p = [0, 0, 0]
                        p[axis] = side
                        p[o1] = i + di
                        p[o2] = j + dj
                        quad.append(vid(tuple(p)))
                    faces.append(quad)
    P = np.asarray(pos, dtype=np.float64) / k - 0.5
    P = P * size + np.asarray(center)
    # the 12 cube edges as vertex pairs (lattice points with two coordinates in {0, k})
    edges = []
    for (p, q) in _lattice_cube_edges(k):
        edges.append((verts[p], verts[q]))
    return faces, P, edges


def _lattice_cube_edges(k):
    out = []
    for axis in range(3):
        others = [ax for ax in range(3) if ax != axis]
        for s1 in (0, k):
            for s2 in (0, k):
                for t in range(k):
                    p = [0, 0, 0]
                    p[others[0]], p[others[1]] = s1, s2
                    q = list(p)
                    p[axis], q[axis] = t, t + 1
                    out.append((tuple(p), tuple(q)))
    return out


def armor(nplates=70, nx=10, ny=11, nsplit=2, nboxes=5, box_k=5, seed=SEED_TOPO, name="armor9k"):
    """ArmorGuy-shaped synthetic control mesh.

    ``nplates`` open plates of nx*ny quads wrapped on a cylinder (r ~ 1, height ~ 2.3) with
    seeded smooth bumps (amplitude 0.05); ``nsplit`` non-adjacent interior quads per plate are
    split into triangle pairs; ``nboxes`` closed cube-spheres (box_k x box_k per side).
    Creases: one interior grid line per plate (nx edges, boundary to boundary) with sigma drawn
    from {inf, 3, 2, 1.5, 0.75}, every 5th plate a ramp 0.5 + 0.25 i; the 12 box edges
    (12 box_k edges) sigma = inf for boxes 0-2 and sigma = 2 for the others.
    Defaults give V=10,000, F=8,590 (280 tris), E=18,510, 1,000 crease edges."""
    rng = np.random.default_rng(seed)
    faces, pos, crease, sigma = [], [], [], []
    cols = 10
    rows = (nplates + cols - 1) // cols
    height = 2.3
    dth = 2 * math.pi / cols
    dz = height / rows
    choices = np.array([np.inf, 3.0, 2.0, 1.5, 0.75], dtype=np.float32)
    phase = rng.random((nplates, 4)) * 2 * math.pi
    for p in range(nplates):
        base = len(pos)
        col, row = p % cols, p // cols
        th0 = col * dth + 0.04 * dth
        th1 = (col + 1) * dth - 0.04 * dth
        z0 = row * dz + 0.03 * dz - height / 2
        z1 = (row + 1) * dz - 0.03 * dz - height / 2
        for j in range(ny + 1):
            for i in range(nx + 1):
                u, v = i / nx, j / ny
                th = th0 + (th1 - th0) * u
                z = z0 + (z1 - z0) * v
                r = 1.0 + 0.05 * math.sin(3 * th + phase[p, 0]) * math.cos(5 * z + phase[p, 1]) \
                    + 0.02 * math.sin(2 * math.pi * u + phase[p, 2]) * math.sin(math.pi * v + phase[p, 3])
                pos.append((r * math.cos(th), r * math.sin(th), z))
        vid = lambda i, j: base + j * (nx + 1) + i
        # non-adjacent interior cells to split
        split = []
        while len(split) < nsplit:
            ci, cj = int(rng.integers(1, nx - 1)), int(rng.integers(1, ny - 1))
            if all(abs(ci - a) > 1 or abs(cj - b) > 1 for (a, b) in split):
                split.append((ci, cj))
        flip = rng.random(nsplit) < 0.5
        for j in range(ny):
            for i in range(nx):
                a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
                if (i, j) in split:
                    if flip[split.index((i, j))]:
                        faces += [(a, b, d), (b, c, d)]
                    else:
                        faces += [(a, b, c), (a, c, d)]
                else:
                    faces.append((a, b, c, d))
        # one interior horizontal grid line j in [1, ny-1], nx edges
        jl = int(rng.integers(1, ny))
        if p % 5 == 4:
            sig = [0.5 + 0.25 * i for i in range(nx)]
        else:
            sig = [float(choices[int(rng.integers(0, len(choices)))])] * nx
        for i in range(nx):
            crease.append((vid(i, jl), vid(i + 1, jl)))
            sigma.append(sig[i])
    for bx in range(nboxes):
        base = len(pos)
        ang = 2 * math.pi * (bx + 0.5) / max(nboxes, 1)
        center = (0.45 * math.cos(ang), 0.45 * math.sin(ang), -0.6 + 0.3 * bx)
        bf, bp, be = _cube_sphere(box_k, center, 0.2)
        faces += [[base + v for v in f] for f in bf]
        pos += [tuple(x) for x in bp]
        s = np.inf if bx < 3 else 2.0
        for (a, b) in be:
            crease.append((base + a, base + b))
            sigma.append(s)
    return _pack(faces, pos, crease, sigma, name=name)


def armor9k(seed=SEED_TOPO):
    """Config 3: V=10,000, F=8,590 (280 tris), E=18,510, B=2,940, 1,000 creases."""
    return armor(70, 10, 11, 2, 5, 5, seed, "armor9k")


def armor50k(seed=SEED_TOPO):
    """Config 5: V=53,890, F=50,030 (1,760 tris), E=103,800."""
    return armor(110, 20, 22, 8, 5, 5, seed, "armor50k")


def torus100k(seed=SEED_TOPO):
    """Config 4: 250x200 torus grid, every quad split on a seeded diagonal: V=50,000, F=100,000."""
    return torus_tris(250, 200, seed=seed)


# ----------------------------------------------------------------------------------------------
# perturbations and frames
# ----------------------------------------------------------------------------------------------

def shuffled(mesh, seed=SEED_TOPO):
    """Seeded random vertex relabelling + face permutation + cyclic rotation of each face
    (locality stress)."""
    rng = np.random.default_rng(seed)
    V = mesh["pos"].shape[0]
    perm = rng.permutation(V).astype(np.int32)  # old -> new
    off, vtx = mesh["face_off"], mesh["face_vtx"]
    F = len(off) - 1
    faces = [list(perm[vtx[off[r]:off[r + 1]]]) for r in range(F)]
    order = rng.permutation(F)
    out_faces = []
    for r in order:
        f = faces[r]
        k = int(rng.integers(0, len(f)))
        out_faces.append(f[k:] + f[:k])
    pos = np.empty_like(mesh["pos"])
    pos[perm] = mesh["pos"]
    crease = perm[mesh["crease"]] if len(mesh["crease"]) else mesh["crease"]
    return _pack(out_faces, pos, crease, mesh["sigma"], name=mesh["name"] + "_shuf")


def random_positions(mesh, seed=SEED_TOPO, scale=1.0):
    rng = np.random.default_rng(seed)
    m = dict(mesh)
    m["pos"] = (rng.standard_normal(mesh["pos"].shape) * scale).astype(np.float32)
    return m


def frame_positions(pos0, t, nframes=4096):
    """Animation frame t of config 5: P0 rotated by 2*pi*t/nframes about z plus a travelling
    wave 0.05*sin(2*pi*t/64 + 7x) along y."""
    th = 2 * math.pi * t / nframes
    c, s = math.cos(th), math.sin(th)
    p = pos0.astype(np.float64)
    x = c * p[:, 0] - s * p[:, 1]
    y = s * p[:, 0] + c * p[:, 1] + 0.05 * np.sin(2 * math.pi * t / 64 + 7 * p[:, 0])
    return np.stack([x, y, p[:, 2]], axis=1).astype(np.float32)


def frame_block(pos0, t0, n, nframes=4096):
    """Frames t0 .. t0+n-1 of config 5 as one float32 array [n][V][3]: frame_positions vectorised
    over frames (the same float64 element-wise operations, so each frame is bitwise identical)."""
    out = np.empty((n, pos0.shape[0], 3), np.float32)
    p = pos0.astype(np.float64)
    for t in range(t0, t0 + n):
        th = 2 * math.pi * t / nframes
        c, s = math.cos(th), math.sin(th)
        out[t - t0, :, 0] = c * p[:, 0] - s * p[:, 1]
        out[t - t0, :, 1] = s * p[:, 0] + c * p[:, 1] + 0.05 * np.sin(2 * math.pi * t / 64 + 7 * p[:, 0])
        out[t - t0, :, 2] = p[:, 2]
    return out


CONFIGS = {
    1: dict(name="cube_cc_L3", mesh=cube, scheme="cc", levels=3),
    2: dict(name="ico_loop_L6", mesh=icosahedron, scheme="loop", levels=6),
    3: dict(name="armor9k_cc_L6", mesh=armor9k, scheme="cc", levels=6),
    4: dict(name="torus100k_sqrt3_L5", mesh=torus100k, scheme="sqrt3", levels=5),
    5: dict(name="armor50k_cc_L4_frames4096", mesh=armor50k, scheme="cc", levels=4, frames=4096),
}


def vertex_channels(mesh, channels, seed=SEED_FRAMES):
    """Seeded per-vertex attribute data [V][channels] fp32 (uv-like: two affine functions of the
    position plus noise, then noise channels) for the extra-channel path."""
    rng = np.random.default_rng(seed)
    p = np.asarray(mesh["pos"], np.float64)
    V = p.shape[0]
    out = rng.standard_normal((V, channels)) * 0.1
    if channels >= 1:
        out[:, 0] += 0.5 + 0.3 * p[:, 0] + 0.1 * p[:, 2]
    if channels >= 2:
        out[:, 1] += 0.5 + 0.3 * p[:, 1] - 0.1 * p[:, 2]
    return out.astype(np.float32)


def displacement(n, seed=SEED_FRAMES, scale=0.01):
    """Seeded per-vertex displacement vectors [n][3] fp32 (hierarchical-edit tests)."""
    rng = np.random.default_rng(seed + 1)
    return (rng.standard_normal((n, 3)) * scale).astype(np.float32)


def permuted(mesh, perm_vtx, perm_face):
    """The mesh relabelled by perm_vtx[new] = old vertex and perm_face[new] = old face (face
    rotations kept); used with the RCM ordering (NEXT-2)."""
    perm_vtx = np.asarray(perm_vtx, np.int64)
    newid = np.empty_like(perm_vtx)
    newid[perm_vtx] = np.arange(len(perm_vtx))
    off, vtx = mesh["face_off"], mesh["face_vtx"]
    faces = [list(newid[vtx[off[r]:off[r + 1]]]) for r in np.asarray(perm_face, np.int64)]
    pos = np.asarray(mesh["pos"])[perm_vtx]
    crease = newid[mesh["crease"]].astype(np.int32) if len(mesh["crease"]) else mesh["crease"]
    return _pack(faces, pos, crease, mesh["sigma"], name=mesh.get("name", "mesh") + "_perm")


def bipyramid(n=40, seed=SEED_TOPO):
    """Closed n-gonal bipyramid: two apices of valence n (long M^T rows, high-valence rules) and
    an equator of valence-4 vertices; 2n outward CCW triangles, slightly jittered."""
    rng = np.random.default_rng(seed)
    pos = [(math.cos(2 * math.pi * k / n), math.sin(2 * math.pi * k / n), 0.0) for k in range(n)]
    pos += [(0.0, 0.0, 1.0), (0.0, 0.0, -1.0)]
    pos = np.asarray(pos) + rng.normal(0, 0.01, (n + 2, 3))
    top, bot = n, n + 1
    faces = [(k, (k + 1) % n, top) for k in range(n)] + [((k + 1) % n, k, bot) for k in range(n)]
    return _pack(faces, pos, name=f"bipyramid{n}")
