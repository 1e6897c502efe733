"""ctypes front-end of the plain C oracle (oracle/alsub_oracle.c).

TEST INFRASTRUCTURE ONLY -- only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_1809_06047_b200``) never imports it and shares no code with it.

``refine(mesh, scheme, levels)`` returns one record per level 0..levels::

    {"V", "F", "face_off", "face_vtx", "pos" (float64[V,3]), "crease" (int32[K,2], (lo,hi),
     ascending (hi,lo)), "sigma" (float32[K]),
     # edge tables of this level (absent for the last level unless edges_last=True):
     "E", "B", "edge_vtx" (int32[E,2] (lo,hi) in id order), "edge_face" (int32[E,2])}
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "alsub_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

SCHEMES = {"cc": 0, "loop": 1, "sqrt3": 2}
STATUS = {0: "OK", 1: "E_ARG", 2: "E_MESH", 3: "E_NONMANIFOLD", 4: "E_SCHEME", 5: "E_CREASE",
          6: "E_OVERFLOW", 7: "E_NOMEM"}


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, status)


class _Mesh(C.Structure):
    _fields_ = [("V", C.c_int32), ("F", C.c_int32),
                ("face_off", C.POINTER(C.c_int32)), ("face_vtx", C.POINTER(C.c_int32)),
                ("pos", C.POINTER(C.c_double)), ("K", C.c_int32),
                ("crease", C.POINTER(C.c_int32)), ("sigma", C.POINTER(C.c_float))]


class _Edges(C.Structure):
    _fields_ = [("E", C.c_int32), ("B", C.c_int32),
                ("edge_vtx", C.POINTER(C.c_int32)), ("edge_face", C.POINTER(C.c_int32))]


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
_HDR = os.path.join(_HERE, "alsub_oracle.h")


def _compile(out, extra):
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if not os.path.exists(out) or os.path.getmtime(out) < newest:
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-D_DEFAULT_SOURCE", "-fPIC", "-shared",
                               "-Wall"] + extra + ["-o", tmp, _SRC, "-lm"])
        os.replace(tmp, out)
    return out


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no fast-math): the serial library the tests use, and the
    same source with -fopenmp for the all-cores host baseline (bench.py)."""
    if force:
        for p in (_LIB, _LIB_OMP):
            if os.path.exists(p):
                os.remove(p)
    _compile(_LIB_OMP, ["-fopenmp"])
    return _compile(_LIB, [])


_lib = None
_lib_omp = None


def _setup(L):
    L.om_level.argtypes = [C.c_int, C.POINTER(_Mesh), C.POINTER(_Mesh), C.POINTER(_Edges), C.c_char_p, C.c_int]
    L.om_edges_of.argtypes = [C.POINTER(_Mesh), C.POINTER(_Edges), C.c_char_p, C.c_int]
    L.om_mesh_free.argtypes = [C.POINTER(_Mesh)]
    L.om_edges_free.argtypes = [C.POINTER(_Edges)]
    L.om_loop_beta.restype = C.c_double
    L.om_loop_beta.argtypes = [C.c_int]
    L.om_sqrt3_alpha.restype = C.c_double
    L.om_sqrt3_alpha.argtypes = [C.c_int]
    L.om_set_threads.restype = C.c_int
    L.om_set_threads.argtypes = [C.c_int]
    return L


def lib_threads(n):
    """The OpenMP build with n threads (bench.py's all-cores oracle timing); returns (lib, threads)."""
    global _lib_omp
    if _lib_omp is None:
        build()
        _lib_omp = _setup(C.CDLL(_LIB_OMP))
    return _lib_omp, _lib_omp.om_set_threads(int(n))


def lib():
    global _lib
    if _lib is None:
        _lib = _setup(C.CDLL(build()))
    return _lib


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _to_c(rec, keep):
    off = np.ascontiguousarray(rec["face_off"], dtype=np.int32)
    vtx = np.ascontiguousarray(rec["face_vtx"], dtype=np.int32)
    pos = np.ascontiguousarray(rec["pos"], dtype=np.float64).reshape(-1)
    cr = np.ascontiguousarray(rec["crease"], dtype=np.int32).reshape(-1)
    sg = np.ascontiguousarray(rec["sigma"], dtype=np.float32).reshape(-1)
    keep += [off, vtx, pos, cr, sg]
    m = _Mesh()
    m.V = pos.size // 3
    m.F = off.size - 1
    m.face_off, m.face_vtx, m.pos = _ptr(off, C.c_int32), _ptr(vtx, C.c_int32), _ptr(pos, C.c_double)
    m.K = sg.size
    m.crease, m.sigma = _ptr(cr, C.c_int32), _ptr(sg, C.c_float)
    return m


def _arr(p, n, dt):
    if n == 0:
        return np.zeros(0, dtype=dt)
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)


def _from_c(m):
    S = m.face_off[m.F] if m.F > 0 else 0
    return {"V": m.V, "F": m.F,
            "face_off": _arr(m.face_off, m.F + 1, np.int32),
            "face_vtx": _arr(m.face_vtx, S, np.int32),
            "pos": _arr(m.pos, 3 * m.V, np.float64).reshape(-1, 3),
            "crease": _arr(m.crease, 2 * m.K, np.int32).reshape(-1, 2),
            "sigma": _arr(m.sigma, m.K, np.float32)}


def _edges_from_c(e):
    return {"E": e.E, "B": e.B,
            "edge_vtx": _arr(e.edge_vtx, 2 * e.E, np.int32).reshape(-1, 2),
            "edge_face": _arr(e.edge_face, 2 * e.E, np.int32).reshape(-1, 2)}


def _normalise_creases(mesh):
    """Input creases -> (lo, hi) pairs in ascending (hi, lo) order (the crease matrix's upper
    triangle in CSC order); sigma = 0 entries kept (the oracle elides them)."""
    cr = np.asarray(mesh["crease"], dtype=np.int64).reshape(-1, 2)
    sg = np.asarray(mesh["sigma"], dtype=np.float32).reshape(-1)
    return cr, sg


def level0(mesh):
    """The control mesh as a level record (positions promoted to fp64)."""
    return {"V": int(mesh["pos"].shape[0]), "F": int(len(mesh["face_off"]) - 1),
            "face_off": np.asarray(mesh["face_off"], np.int32), "face_vtx": np.asarray(mesh["face_vtx"], np.int32),
            "pos": np.asarray(mesh["pos"], np.float64).reshape(-1, 3),
            "crease": np.asarray(mesh["crease"], np.int32).reshape(-1, 2), "sigma": np.asarray(mesh["sigma"], np.float32)}


def edges_of(rec):
    keep = []
    m = _to_c(rec, keep)
    e = _Edges()
    err = C.create_string_buffer(512)
    st = lib().om_edges_of(C.byref(m), C.byref(e), err, 512)
    if st != 0:
        raise OracleError(st, err.value.decode())
    out = _edges_from_c(e)
    lib().om_edges_free(C.byref(e))
    return out


def level(rec, scheme, L=None):
    """One refinement level: returns (child record, parent edge tables).  L: the library (default
    the serial build)."""
    L = L or lib()
    keep = []
    m = _to_c(rec, keep)
    out, e = _Mesh(), _Edges()
    err = C.create_string_buffer(512)
    st = L.om_level(SCHEMES[scheme], C.byref(m), C.byref(out), C.byref(e), err, 512)
    if st != 0:
        raise OracleError(st, err.value.decode())
    child, edges = _from_c(out), _edges_from_c(e)
    L.om_mesh_free(C.byref(out))
    L.om_edges_free(C.byref(e))
    return child, edges


def refine(mesh, scheme, levels, edges_last=False, threads=None, times=None):
    """Levels 0..levels of `mesh`.  threads: run the OpenMP build with that many threads (same
    results); times: a list that receives the wall time of each level (seconds)."""
    import time
    L = lib_threads(threads)[0] if threads else lib()
    recs = [level0(mesh)]
    for _ in range(levels):
        t0 = time.perf_counter()
        child, edges = level(recs[-1], scheme, L)
        if times is not None:
            times.append(time.perf_counter() - t0)
        recs[-1].update(edges)
        recs.append(child)
    if edges_last:
        recs[-1].update(edges_of(recs[-1]))
    return recs


def loop_beta(n):
    return lib().om_loop_beta(int(n))


def sqrt3_alpha(n):
    return lib().om_sqrt3_alpha(int(n))


def refinement_matrix(mesh, scheme, levels):
    """The refinement matrix R (P_L = R P_0) by its definition: refinement is linear in
    the vertex data, so column j of R is the refinement of the unit vector e_j (three columns per
    call, one per coordinate).  Dense float64 [V_levels, V0]; small meshes only."""
    V0 = int(np.asarray(mesh["pos"]).reshape(-1, 3).shape[0])
    cols = []
    for j0 in range(0, V0, 3):
        m = dict(mesh)
        pos = np.zeros((V0, 3))
        for c in range(3):
            if j0 + c < V0:
                pos[j0 + c, c] = 1.0
        m["pos"] = pos
        out = refine(m, scheme, levels)[-1]["pos"]
        for c in range(3):
            if j0 + c < V0:
                cols.append(out[:, c])
    return np.stack(cols, axis=1) if cols else np.zeros((0, 0))
