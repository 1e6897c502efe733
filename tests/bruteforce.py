"""Exact-rational brute-force subdivision for TINY meshes -- an independent pin for the C oracle.

Written separately from oracle/alsub_oracle.c (different structure: Python dicts of directed
edges, ``fractions.Fraction`` arithmetic, the CLASSICAL forms of the rules rather than the
linear-algebra split), so that a dropped term, a wrong index or a transposed operand in either
shows up as a mismatch:

* CC vertex point in the paper's original form, Eq. pos_update:
  S(p_i) = 1/n ((n-3) p_i + 1/n sum f_j + 2/n sum 1/2 (p_i + p_j))
* CC edge point e = 1/4 (p_k + p_l + f_r + f_s), boundary midpoint,
  boundary vertex 3/4 p + 1/8 (p_i-1 + p_i+1) (Eq. CC_boundary)
* Loop / sqrt3 only where cos(2 pi / n) is rational (n in {3, 4, 6}): beta, alpha from P:L1044,
  P:L990 evaluated with exact cosines.
* creases: readings R6-R9 of DESIGN.md, re-implemented from the prose.
"""
from __future__ import annotations

from fractions import Fraction as Q

INF = float("inf")
COS = {3: Q(-1, 2), 4: Q(0), 6: Q(1, 2)}  # exact cos(2 pi / n)


def _faces(mesh):
    off, vtx = [int(x) for x in mesh["face_off"]], [int(x) for x in mesh["face_vtx"]]
    return [vtx[off[i]:off[i + 1]] for i in range(len(off) - 1)]


def _qpos(mesh):
    return [tuple(Q(float(c)) for c in p) for p in mesh["pos"]]


def _add(*ps):
    return tuple(sum(c) for c in zip(*ps))


def _scale(s, p):
    return tuple(s * c for c in p)


class Level:
    def __init__(self, faces, pos, creases):
        self.faces, self.pos = faces, pos
        self.V, self.F = len(pos), len(faces)
        self.directed = {}  # (a, b) -> face
        for r, f in enumerate(faces):
            for t in range(len(f)):
                a, b = f[t], f[(t + 1) % len(f)]
                assert (a, b) not in self.directed, "orientation / non-manifold"
                self.directed[(a, b)] = r
        und = sorted({(max(a, b), min(a, b)) for (a, b) in self.directed})  # (hi, lo) order
        self.edges = [(lo, hi) for (hi, lo) in und]
        self.eid = {e: i for i, e in enumerate(self.edges)}
        self.bnd = [((lo, hi) not in self.directed) or ((hi, lo) not in self.directed) for (lo, hi) in self.edges]
        self.sigma = [INF if b else 0.0 for b in self.bnd]
        self.user = [False] * len(self.edges)
        for (a, b), s in creases.items():
            i = self.eid[(min(a, b), max(a, b))]
            if not self.bnd[i] and s > 0:
                self.sigma[i], self.user[i] = s, True
        self.nbrs = {v: [] for v in range(self.V)}
        for i, (lo, hi) in enumerate(self.edges):
            self.nbrs[lo].append((hi, i))
            self.nbrs[hi].append((lo, i))
        self.vfaces = {v: [r for r, f in enumerate(faces) if v in f] for v in range(self.V)}

    def eid_of(self, a, b):
        return self.eid[(min(a, b), max(a, b))]

    # crease bookkeeping (readings R6-R9)
    def k_s(self, v):
        sig = [self.sigma[i] for (_, i) in self.nbrs[v] if self.sigma[i] > 0]
        k = len(sig)
        if k == 0:
            return 0, 0.0, []
        s = INF if any(x == INF for x in sig) else sum(sig) / k
        nb = [u for (u, i) in self.nbrs[v] if self.sigma[i] > 0]
        return k, s, nb

    def vertex_rule(self, v, smooth):
        k, s, nb = self.k_s(v)
        if k <= 1:
            return smooth
        p = self.pos[v]
        sharp = _add(_scale(Q(3, 4), p), _scale(Q(1, 8), _add(self.pos[nb[0]], self.pos[nb[1]]))) if k == 2 else p
        if s >= 1:
            return sharp
        w = Q(s)
        return _add(_scale(1 - w, smooth), _scale(w, sharp))

    def edge_rule(self, i, smooth):
        s = self.sigma[i]
        if s <= 0:
            return smooth
        lo, hi = self.edges[i]
        mid = _scale(Q(1, 2), _add(self.pos[lo], self.pos[hi]))
        if s >= 1:
            return mid
        w = Q(s)
        return _add(_scale(1 - w, smooth), _scale(w, mid))

    def child_creases(self, ep_of):
        out = {}
        for i, (lo, hi) in enumerate(self.edges):
            if not self.user[i]:
                continue
            s = self.sigma[i]
            for x in (lo, hi):
                if s == INF:
                    c = INF
                else:
                    others = [self.sigma[j] for (_, j) in self.nbrs[x]
                              if j != i and self.user[j] and self.sigma[j] != INF]
                    sbar = sum(others) / len(others) if others else s
                    c = max(0.25 * (sbar + 3 * s) - 1, 0.0)
                if c > 0:
                    out[(x, ep_of(i))] = c
        return out


def cc_level(faces, pos, creases):
    L = Level(faces, pos, creases)
    V, F = L.V, L.F
    fpt = [_scale(Q(1, len(f)), _add(*[pos[v] for v in f])) for f in faces]
    ept = []
    for i, (lo, hi) in enumerate(L.edges):
        if L.bnd[i]:
            sm = _scale(Q(1, 2), _add(pos[lo], pos[hi]))
        else:
            r, s = L.directed[(lo, hi)], L.directed[(hi, lo)]
            sm = _scale(Q(1, 4), _add(pos[lo], pos[hi], fpt[r], fpt[s]))
        ept.append(L.edge_rule(i, sm))
    vpt = []
    for v in range(V):
        fs = L.vfaces[v]
        n = len(fs)
        if n == 0:
            sm = pos[v]
        else:
            p = pos[v]
            sf = _add(*[fpt[r] for r in fs])
            se = _add(*[_scale(Q(1, 2), _add(p, pos[u])) for (u, _) in L.nbrs[v]])
            sm = _scale(Q(1, n), _add(_scale(n - 3, p), _scale(Q(1, n), sf), _scale(Q(2, n), se)))
        vpt.append(L.vertex_rule(v, sm))
    child = []
    for r, f in enumerate(faces):
        c = len(f)
        for t in range(c):
            child.append([f[t], V + F + L.eid_of(f[t], f[(t + 1) % c]), V + r, V + F + L.eid_of(f[t - 1], f[t])])
    return L, child, vpt + fpt + ept, L.child_creases(lambda i: V + F + i)


def loop_level(faces, pos, creases):
    L = Level(faces, pos, creases)
    V = L.V
    ept = []
    for i, (lo, hi) in enumerate(L.edges):
        if L.bnd[i]:
            sm = _scale(Q(1, 2), _add(pos[lo], pos[hi]))
        else:
            def opp(a, b):
                f = faces[L.directed[(a, b)]]
                return [x for x in f if x != a and x != b][0]
            sm = _add(_scale(Q(3, 8), _add(pos[lo], pos[hi])), _scale(Q(1, 8), _add(pos[opp(lo, hi)], pos[opp(hi, lo)])))
        ept.append(L.edge_rule(i, sm))
    vpt = []
    for v in range(V):
        n = len(L.nbrs[v])
        if n == 0:
            sm = pos[v]
        else:
            c = COS[n]
            beta = (Q(5, 8) - (Q(3, 8) + Q(1, 4) * c) ** 2) / n
            sm = _add(_scale(1 - n * beta, pos[v]), _scale(beta, _add(*[pos[u] for (u, _) in L.nbrs[v]])))
        vpt.append(L.vertex_rule(v, sm))
    child = []
    for f in faces:
        k, l, m = f
        ekl, elm, emk = (V + L.eid_of(k, l), V + L.eid_of(l, m), V + L.eid_of(m, k))
        child += [[k, ekl, emk], [l, elm, ekl], [m, emk, elm], [ekl, elm, emk]]
    return L, child, vpt + ept, L.child_creases(lambda i: V + i)


def sqrt3_level(faces, pos, creases):
    L = Level(faces, pos, creases)
    V = L.V
    fpt = [_scale(Q(1, 3), _add(*[pos[v] for v in f])) for f in faces]
    vpt = []
    for v in range(V):
        n = len(L.nbrs[v])
        alpha = (4 - 2 * COS[n]) / 9
        vpt.append(_add(_scale(1 - alpha, pos[v]), _scale(alpha / n, _add(*[pos[u] for (u, _) in L.nbrs[v]]))))
    child = []
    for i, f in enumerate(faces):
        for t in range(3):
            k, l = f[t], f[(t + 1) % 3]
            child.append([k, V + L.directed[(l, k)], V + i])
    return L, child, vpt + fpt, {}


LEVEL = {"cc": cc_level, "loop": loop_level, "sqrt3": sqrt3_level}


def refine(mesh, scheme, levels):
    """Per level: dict(faces, pos (Fractions), edges (lo,hi) id order, edge_face, creases)."""
    faces, pos = _faces(mesh), _qpos(mesh)
    creases = {(int(a), int(b)): float(s) for (a, b), s in zip(mesh["crease"], mesh["sigma"])}
    out = []
    for _ in range(levels):
        L, child, cpos, ccre = LEVEL[scheme](faces, pos, creases)
        out.append(dict(faces=faces, pos=pos, edges=L.edges,
                        edge_face=[(L.directed.get((lo, hi), -1), L.directed.get((hi, lo), -1)) for (lo, hi) in L.edges],
                        creases=creases))
        faces, pos, creases = child, cpos, ccre
    out.append(dict(faces=faces, pos=pos, creases=creases))
    return out
