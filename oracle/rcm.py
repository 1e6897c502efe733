"""Reverse Cuthill-McKee ordering of a control mesh -- plain Python oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, smoke() and bench.py's CPU legs
may import it.  Shares no code with the library's alsub_rcm_order.

PAPER.md "Mesh reordering": "we apply the RCM algorithm to the graph Laplacian of
the mesh. The acquired permutation is applied to the rows of M and columns are sorted by their
first non-zero entry."  The algorithm, step by step (Cuthill & McKee 1969, reversed by George
1971; start vertex by the George-Liu pseudo-peripheral node finder):

  graph      vertices adjacent iff they share a mesh edge (the off-diagonal pattern of the graph
             Laplacian D - A); deg(v) = number of distinct neighbours
  components visited in order of their smallest unvisited vertex id
  start      r = vertex of minimum degree in the component (ties: smallest id); repeat: BFS
             level structure from r, x = minimum-degree vertex of the last level (ties: smallest
             id); if ecc(x) > ecc(r) then r = x, else stop
  CM order   BFS from r; each dequeued vertex appends its unvisited neighbours sorted by
             (degree, id)
  RCM        the concatenated CM order of all components, reversed: perm_vtx[new] = old
  faces      sorted by their first non-zero in the new row order = min new id of their
             vertices; ties keep the original face order (reading R24): perm_face[new] = old
"""
from __future__ import annotations

from collections import deque


def vertex_graph(face_off, face_vtx, V):
    nbr = [set() for _ in range(V)]
    for r in range(len(face_off) - 1):
        f = [int(x) for x in face_vtx[face_off[r]:face_off[r + 1]]]
        for t in range(len(f)):
            a, b = f[t], f[(t + 1) % len(f)]
            if a != b:
                nbr[a].add(b)
                nbr[b].add(a)
    return [sorted(s) for s in nbr]


def _levels(nbr, r):
    """BFS level structure from r: list of levels (lists of vertices)."""
    seen = {r}
    levels = [[r]]
    while True:
        nxt = []
        for v in levels[-1]:
            for w in nbr[v]:
                if w not in seen:
                    seen.add(w)
                    nxt.append(w)
        if not nxt:
            return levels
        levels.append(nxt)


def pseudo_peripheral(nbr, comp):
    deg = lambda v: len(nbr[v])
    r = min(comp, key=lambda v: (deg(v), v))
    lv = _levels(nbr, r)
    while True:
        x = min(lv[-1], key=lambda v: (deg(v), v))
        lx = _levels(nbr, x)
        if len(lx) > len(lv):
            r, lv = x, lx
        else:
            return r


def rcm_order(face_off, face_vtx, V):
    """(perm_vtx, perm_face): perm_vtx[new] = old vertex, perm_face[new] = old face."""
    nbr = vertex_graph(face_off, face_vtx, V)
    deg = [len(n) for n in nbr]
    visited = [False] * V
    order = []
    for s in range(V):
        if visited[s]:
            continue
        comp = [v for lv in _levels(nbr, s) for v in lv]
        r = pseudo_peripheral(nbr, comp)
        visited[r] = True
        q = deque([r])
        while q:
            v = q.popleft()
            order.append(v)
            new = sorted((w for w in nbr[v] if not visited[w]), key=lambda w: (deg[w], w))
            for w in new:
                visited[w] = True
                q.append(w)
    perm_vtx = order[::-1]
    newid = [0] * V
    for i, v in enumerate(perm_vtx):
        newid[v] = i
    F = len(face_off) - 1
    key = [min(newid[int(x)] for x in face_vtx[face_off[r]:face_off[r + 1]]) for r in range(F)]
    perm_face = sorted(range(F), key=lambda r: (key[r], r))
    return perm_vtx, perm_face


def bandwidth(face_off, face_vtx, perm_vtx):
    """max |new(a) - new(b)| over mesh edges (the graph Laplacian's bandwidth)."""
    newid = {int(v): i for i, v in enumerate(perm_vtx)}
    bw = 0
    for r in range(len(face_off) - 1):
        f = [int(x) for x in face_vtx[face_off[r]:face_off[r + 1]]]
        for t in range(len(f)):
            bw = max(bw, abs(newid[f[t]] - newid[f[(t + 1) % len(f)]]))
    return bw
