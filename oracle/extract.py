"""Selective / feature-adaptive subdivision: the extraction module -- plain Python oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the library's
alsub_mesh_extract.

PAPER.md §"Selective and Feature Adaptive Subdivision", step by step:
  x_0          1 at the selected vertices -- by default the extraordinary ones, valence
               n = M 1 != 4 (Eq. vo)
  q_i          = M^T x_i: the faces with a selected vertex
  x_{i+1}      = M q_i: the vertices of those faces; repeated `rings` times
  X, X̊         identity matrices with the unselected rows / columns deleted, i.e.
               selected vertices and faces keep their relative order
  P' = X P, M' = X M X̊
  creases      the level's creases between two selected vertices that are an edge of an
               extracted face (reading R25)
"""
from __future__ import annotations

import numpy as np


def _faces(rec):
    off, vtx = rec["face_off"], rec["face_vtx"]
    return [[int(v) for v in vtx[off[r]:off[r + 1]]] for r in range(len(off) - 1)]


def valence(rec):
    """n = M 1: number of faces containing each vertex (Eq. vo)."""
    n = [0] * int(rec["V"] if "V" in rec else len(rec["pos"]))
    for f in _faces(rec):
        for v in f:
            n[v] += 1
    return n


def extract(rec, vsel=None, rings=1):
    """Returns (mesh dict, vtx_map, face_map); vtx_map[new] = old, face_map[new] = old."""
    faces = _faces(rec)
    V = len(rec["pos"])
    x = [bool(s) for s in vsel] if vsel is not None else [n != 4 for n in valence(rec)]
    q = [False] * len(faces)
    for _ in range(rings):
        q = [any(x[v] for v in f) for f in faces]      # q_i = M^T x_i
        x = [False] * V                                # x_{i+1} = M q_i
        for r, f in enumerate(faces):
            if q[r]:
                for v in f:
                    x[v] = True
    vmap = [v for v in range(V) if x[v]]
    fmap = [r for r in range(len(faces)) if q[r]]
    newid = {v: i for i, v in enumerate(vmap)}
    out_faces = [[newid[v] for v in faces[r]] for r in fmap]
    edges = set()
    for f in out_faces:
        for t in range(len(f)):
            a, b = f[t], f[(t + 1) % len(f)]
            edges.add((min(a, b), max(a, b)))
    cr, sg = [], []
    for (a, b), s in zip(np.asarray(rec["crease"]).reshape(-1, 2), np.asarray(rec["sigma"]).reshape(-1)):
        a, b = int(a), int(b)
        if x[a] and x[b]:
            e = (min(newid[a], newid[b]), max(newid[a], newid[b]))
            if e in edges:
                cr.append(e)
                sg.append(float(s))
    off = np.zeros(len(out_faces) + 1, np.int32)
    off[1:] = np.cumsum([len(f) for f in out_faces]) if out_faces else []
    mesh = {"face_off": off, "face_vtx": np.asarray([v for f in out_faces for v in f], np.int32),
            "pos": np.asarray(rec["pos"])[vmap] if vmap else np.zeros((0, 3)),
            "crease": np.asarray(cr, np.int32).reshape(-1, 2), "sigma": np.asarray(sg, np.float32)}
    return mesh, vmap, fmap


def descendant_slots(face_off, r, k):
    """Slots (rows of the child face lists) of the level-(l+k) descendants of face r of a level-l
    mesh with offsets face_off, for Catmull-Clark: its c children are faces off_r .. off_r+c-1 of
    level l+1 (quads), each with 4 children 4s .. 4s+3 thereafter (structured ids)."""
    lo, hi = int(face_off[r]), int(face_off[r + 1])
    for _ in range(k - 1):
        lo, hi = 4 * lo, 4 * hi
    return lo, hi  # faces [lo, hi) of level l+k
