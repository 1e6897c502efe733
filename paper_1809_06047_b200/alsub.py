"""Thin ctypes binding of the C ABI in include/alsub.h (argument marshalling only).

Every step of the refinement runs in libalsub.so's sm_100a kernels; PyTorch provides device
memory (its caching allocator is wired in as the library's allocator), streams and tensors.
There is no CPU fallback: importing this module on a machine without the built library, or
calling it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libalsub.so")

CATMULL_CLARK, LOOP, SQRT3 = 0, 1, 2
SCHEMES = {"cc": CATMULL_CLARK, "catmull-clark": CATMULL_CLARK, "loop": LOOP, "sqrt3": SQRT3}
STATUS = {0: "OK", 1: "E_ARG", 2: "E_MESH", 3: "E_NONMANIFOLD", 4: "E_SCHEME", 5: "E_CREASE",
          6: "E_OVERFLOW", 7: "E_NOMEM", 8: "E_CUDA"}


class AlsubError(RuntimeError):
    def __init__(self, status, msg):
        self.status = STATUS.get(status, str(status))
        super().__init__(f"{self.status}: {msg}")


class _Counts(C.Structure):
    _fields_ = [("verts", C.c_int64), ("faces", C.c_int64), ("edges", C.c_int64), ("boundary_edges", C.c_int64),
                ("face_slots", C.c_int64), ("creases_upper_bound", C.c_int64), ("face_order", C.c_int32),
                ("edges_valid", C.c_int32)]


class _KTime(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("level", C.c_int32), ("ms", C.c_float)]


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class _Allocator(C.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", C.c_void_p)]


_lib = None


def lib():
    """Load libalsub.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.alsub_mesh_create.argtypes = [vp, vp, i32, vp, i32, vp, vp, i32, C.POINTER(_Allocator), vp, C.POINTER(vp)]
    L.alsub_set_positions.argtypes = [vp, vp, vp]
    L.alsub_refine.argtypes = [vp, C.c_int, i32, vp]
    L.alsub_level_counts.argtypes = [vp, i32, C.POINTER(_Counts)]
    L.alsub_refine_profile.argtypes = [vp, C.c_int, i32, vp, C.POINTER(_KTime), i32, C.POINTER(i32)]
    L.alsub_level_topology.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    L.alsub_level_positions.argtypes = [vp, i32, vp, vp]
    L.alsub_eval_frames.argtypes = [vp, i32, vp, i32, vp, vp]
    L.alsub_eval_attributes.argtypes = [vp, i32, vp, i32, vp, vp]
    L.alsub_level_positions_ptr.argtypes = [vp, i32, C.POINTER(vp)]
    L.alsub_reevaluate.argtypes = [vp, i32, vp]
    L.alsub_rcm_order.argtypes = [vp, vp, i32, i32, vp, vp]
    L.alsub_mesh_extract.argtypes = [vp, i32, vp, i32, vp, C.POINTER(vp)]
    L.alsub_build_refinement_matrix.argtypes = [vp, i32, vp]
    L.alsub_refinement_matrix_info.argtypes = [vp, C.POINTER(i32), C.POINTER(i64), C.POINTER(i64)]
    L.alsub_refinement_matrix_csr.argtypes = [vp, vp, vp, vp, vp]
    L.alsub_eval_frames_matrix.argtypes = [vp, vp, i32, vp, vp]
    L.alsub_refinement_matrix_blocks.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
    L.alsub_eval_frames_matrix_summary.argtypes = [vp, vp, i32, vp, vp, vp]
    L.alsub_extract_maps.argtypes = [vp, vp, vp, vp]
    L.alsub_frame_summary.argtypes = [vp, i32, i64, vp, vp]
    L.alsub_probe.argtypes = [vp, i32, C.c_char_p, i32]
    L.alsub_probe_read.argtypes = [vp, vp, i32, C.POINTER(i32)]
    L.alsub_probe_read_offsets.argtypes = [vp, vp, vp, vp, i32, C.POINTER(i32)]
    L.alsub_last_launch_count.argtypes = [vp]
    L.alsub_last_launch_count.restype = i64
    L.alsub_mesh_destroy.argtypes = [vp]
    L.alsub_mesh_destroy.restype = None
    L.alsub_last_error.restype = C.c_char_p
    L.alsub_version.restype = C.c_char_p
    for f in ("alsub_mesh_create", "alsub_set_positions", "alsub_refine", "alsub_refine_profile", "alsub_level_counts",
              "alsub_level_topology", "alsub_level_positions", "alsub_eval_frames", "alsub_eval_attributes",
              "alsub_level_positions_ptr", "alsub_reevaluate", "alsub_rcm_order", "alsub_mesh_extract",
              "alsub_extract_maps", "alsub_build_refinement_matrix", "alsub_refinement_matrix_info",
              "alsub_refinement_matrix_csr", "alsub_eval_frames_matrix", "alsub_refinement_matrix_blocks", "alsub_eval_frames_matrix_summary", "alsub_frame_summary", "alsub_probe",
              "alsub_probe_read", "alsub_probe_read_offsets"):
        getattr(L, f).restype = C.c_int
    _lib = L
    return L


def _check(st):
    if st != 0:
        raise AlsubError(st, lib().alsub_last_error().decode(errors="replace"))


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


def _as(t, dtype):
    """Contiguous tensor/array of the given dtype, keeping device tensors on the device."""
    if isinstance(t, torch.Tensor):
        return t.to(dtype).contiguous()
    npdt = {torch.int32: np.int32, torch.float32: np.float32}[dtype]
    return np.ascontiguousarray(np.asarray(t), dtype=npdt)


def _device_view(addr, shape):
    """A float32 CUDA tensor aliasing handle-owned device memory (no copy, no ownership)."""
    n = int(np.prod(shape))

    class _Iface:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (int(addr), False), "version": 3}

    return torch.as_tensor(_Iface(), device="cuda").view(*shape)


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


class _TorchAllocator:
    """The PyTorch caching allocator as the library's device allocator."""

    def __init__(self, device):
        self.device = device

        def _a(nbytes, stream, ctx):
            try:
                return torch.cuda.caching_allocator_alloc(int(nbytes), self.device, int(stream or 0))
            except Exception:
                return None

        def _f(ptr, nbytes, stream, ctx):
            torch.cuda.caching_allocator_delete(int(ptr))

        self._a, self._f = _ALLOC_FN(_a), _FREE_FN(_f)
        self.struct = _Allocator(self._a, self._f, None)


class Mesh:
    """A control mesh on the GPU: ``alsub_mesh_create`` (P:L224-226 mesh matrix).

    face_off int32[F+1], face_vtx int32[S], pos float32[V,3], crease int32[K,2], sigma float32[K]
    -- torch tensors (CUDA or CPU) or numpy arrays (host)."""

    def __init__(self, face_off, face_vtx, pos, crease=None, sigma=None, stream=None, torch_allocator=True):
        if not torch.cuda.is_available():
            raise RuntimeError("alsub needs a CUDA device (there is no CPU path)")
        self._lib = lib()
        self.device = torch.cuda.current_device()
        self._keep = []
        fo, fv, P = _as(face_off, torch.int32), _as(face_vtx, torch.int32), _as(pos, torch.float32)
        if crease is None or len(crease) == 0:
            cr, sg, K = None, None, 0
        else:
            cr, sg = _as(crease, torch.int32), _as(sigma, torch.float32)
            K = int(cr.shape[0])
        self._keep += [fo, fv, P, cr, sg]
        V = int(P.shape[0]) if P.ndim == 2 else int(P.size // 3)
        F = int(fo.shape[0]) - 1
        self._alloc = _TorchAllocator(self.device) if torch_allocator else None
        h = C.c_void_p()
        st = self._lib.alsub_mesh_create(_ptr(fo), _ptr(fv), F, _ptr(P), V, _ptr(cr), _ptr(sg), K,
                                         C.byref(self._alloc.struct) if self._alloc else None,
                                         _stream(stream), C.byref(h))
        self._keep = []
        _check(st)
        self._h = h
        self.scheme = None
        self.levels = None

    # -- refinement matrix R (NEXT-1) --
    def build_refinement_matrix(self, levels, stream=None):
        """P_L = R P_0 for the last refine's topology, R built by probing the static path."""
        _check(self._lib.alsub_build_refinement_matrix(self._h, int(levels), _stream(stream)))
        return self.refinement_matrix_info()

    def refinement_matrix_info(self):
        lv, rows, nnz = C.c_int32(), C.c_int64(), C.c_int64()
        _check(self._lib.alsub_refinement_matrix_info(self._h, C.byref(lv), C.byref(rows), C.byref(nnz)))
        return {"levels": lv.value, "rows": rows.value, "nnz": nnz.value}

    def refinement_matrix_blocks(self):
        """{chunks, weights}: size of the blocked form alsub_eval_frames_matrix evaluates."""
        c, w = C.c_int64(), C.c_int64()
        _check(self._lib.alsub_refinement_matrix_blocks(self._h, C.byref(c), C.byref(w)))
        return {"chunks": c.value, "weights": w.value}

    def refinement_matrix_csr(self):
        """(row_off, cols, vals) numpy arrays of R."""
        info = self.refinement_matrix_info()
        ro = np.empty(info["rows"] + 1, np.int32)
        co = np.empty(info["nnz"], np.int32)
        va = np.empty(info["nnz"], np.float32)
        _check(self._lib.alsub_refinement_matrix_csr(self._h, _ptr(ro), _ptr(co), _ptr(va), _stream(None)))
        return ro, co, va

    def eval_frames_matrix(self, frames, out=None, stream=None):
        """Static mode by the single SpMM P_L = R P_0: frames [B, V0, 3] (CUDA) -> [B, V_L, 3]."""
        fr = frames.to(torch.float32).contiguous()
        B = int(fr.shape[0])
        rows = self.refinement_matrix_info()["rows"]
        if out is None:
            out = torch.empty((B, rows, 3), dtype=torch.float32, device="cuda")
        _check(self._lib.alsub_eval_frames_matrix(self._h, _ptr(fr), B, _ptr(out), _stream(stream)))
        return out

    def eval_frames_matrix_summary(self, frames, out=None, summary=None, stream=None):
        """eval_frames_matrix plus each output frame's summary record (alsub_frame_summary layout),
        computed while the frames are written: returns (out [B, V_L, 3], summary int32 [B, 8])."""
        fr = frames.to(torch.float32).contiguous()
        B = int(fr.shape[0])
        rows = self.refinement_matrix_info()["rows"]
        if out is None:
            out = torch.empty((B, rows, 3), dtype=torch.float32, device="cuda")
        if summary is None:
            summary = torch.empty((B, 8), dtype=torch.int32, device="cuda")
        _check(self._lib.alsub_eval_frames_matrix_summary(self._h, _ptr(fr), B, _ptr(out), _ptr(summary),
                                                          _stream(stream)))
        return out, summary

    def extract(self, level, vsel=None, rings=1, stream=None):
        """Selective / feature-adaptive subdivision, extraction module: the faces
        within `rings` propagation steps of the selected vertices of `level` (vsel: bool/uint8
        [V_level]; None = extraordinary vertices, valence != 4) as a new control mesh.
        Returns (Mesh, vtx_map, face_map) with the original ids (int32 CUDA tensors)."""
        sel = None
        if vsel is not None:
            sel = vsel.to(torch.uint8).contiguous() if isinstance(vsel, torch.Tensor) else \
                np.ascontiguousarray(np.asarray(vsel), dtype=np.uint8)
        h = C.c_void_p()
        _check(self._lib.alsub_mesh_extract(self._h, int(level), _ptr(sel), int(rings), _stream(stream), C.byref(h)))
        sub = Mesh.__new__(Mesh)
        sub._lib, sub.device, sub._keep = self._lib, self.device, []
        sub._alloc = self._alloc  # the extracted handle allocates through the same allocator
        sub._h, sub.scheme, sub.levels = h, None, None
        c = sub.counts(0)
        vm = torch.empty(c["verts"], dtype=torch.int32, device="cuda")
        fm = torch.empty(c["faces"], dtype=torch.int32, device="cuda")
        _check(self._lib.alsub_extract_maps(sub._h, _ptr(vm), _ptr(fm), _stream(stream)))
        return sub, vm, fm

    # -- lifetime --
    def close(self):
        if getattr(self, "_h", None):
            torch.cuda.synchronize()
            self._lib.alsub_mesh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- ABI calls --
    def set_positions(self, pos, stream=None):
        P = _as(pos, torch.float32)
        _check(self._lib.alsub_set_positions(self._h, _ptr(P), _stream(stream)))
        if isinstance(P, torch.Tensor) and P.is_cuda:
            self._pos_keep = P  # keep alive until the stream consumes it

    def refine(self, scheme, levels, stream=None):
        sc = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
        _check(self._lib.alsub_refine(self._h, sc, int(levels), _stream(stream)))
        self.scheme, self.levels = sc, int(levels)
        return self

    def refine_profile(self, scheme, levels, stream=None, cap=4096):
        """Eager refine with a CUDA event after every kernel: [(name, level, ms), ...]."""
        sc = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
        buf = (_KTime * cap)()
        n = C.c_int32()
        _check(self._lib.alsub_refine_profile(self._h, sc, int(levels), _stream(stream), buf, cap, C.byref(n)))
        self.scheme, self.levels = sc, int(levels)
        return [(buf[i].name.decode(), int(buf[i].level), float(buf[i].ms)) for i in range(min(n.value, cap))]

    def counts(self, level):
        c = _Counts()
        _check(self._lib.alsub_level_counts(self._h, int(level), C.byref(c)))
        return {k: getattr(c, k) for k, _ in _Counts._fields_}

    def positions(self, level, out=None, stream=None):
        V = self.counts(level)["verts"]
        if out is None:
            out = torch.empty((V, 3), dtype=torch.float32, device="cuda")
        _check(self._lib.alsub_level_positions(self._h, int(level), _ptr(out), _stream(stream)))
        return out

    def topology(self, level, faces=True, edges=False, creases=False, stream=None):
        c = self.counts(level)
        out = {}
        dev = "cuda"
        fv = torch.empty(c["face_slots"], dtype=torch.int32, device=dev) if faces else None
        fo = torch.empty(c["faces"] + 1, dtype=torch.int32, device=dev) if faces else None
        ev = torch.empty((c["edges"], 2), dtype=torch.int32, device=dev) if edges else None
        ef = torch.empty((c["edges"], 2), dtype=torch.int32, device=dev) if edges else None
        K = max(int(c["creases_upper_bound"]), 1)
        cp = torch.empty((K, 2), dtype=torch.int32, device=dev) if creases else None
        cs = torch.empty(K, dtype=torch.float32, device=dev) if creases else None
        nk = np.zeros(1, dtype=np.int32) if creases else None
        _check(self._lib.alsub_level_topology(self._h, int(level), _ptr(fv), _ptr(fo), _ptr(ev), _ptr(ef), _ptr(cp),
                                              _ptr(cs), _ptr(nk), _stream(stream)))
        if faces:
            out["face_vtx"], out["face_off"] = fv, fo
        if edges:
            out["edge_vtx"], out["edge_face"] = ev, ef
        if creases:
            k = int(nk[0])
            out["crease"], out["sigma"] = cp[:k], cs[:k]
        return out

    def eval_frames(self, frames, levels, out=None, stream=None):
        """Static mode: frames [B, V0, 3] -> [B, V_levels, 3] through the stored topology."""
        fr = _as(frames, torch.float32)
        B = int(fr.shape[0])
        VL = self.counts(levels)["verts"]
        if out is None:
            out = torch.empty((B, VL, 3), dtype=torch.float32, device="cuda")
        _check(self._lib.alsub_eval_frames(self._h, int(levels), _ptr(fr), B, _ptr(out), _stream(stream)))
        return out

    def eval_attributes(self, attr, levels, out=None, stream=None):
        """Extra vertex channels: attr [V0, C] -> [V_levels, C] with the position stencils."""
        a = _as(attr, torch.float32)
        Cn = int(a.shape[1]) if a.ndim == 2 else 1
        VL = self.counts(levels)["verts"]
        if out is None:
            out = torch.empty((VL, Cn), dtype=torch.float32, device="cuda")
        _check(self._lib.alsub_eval_attributes(self._h, int(levels), _ptr(a), Cn, _ptr(out), _stream(stream)))
        return out

    def level_positions_view(self, level):
        """The handle-owned device positions of `level` as a writable [V, 3] tensor view
        (hierarchical edits / displacement); follow writes with reevaluate()."""
        p = C.c_void_p()
        _check(self._lib.alsub_level_positions_ptr(self._h, int(level), C.byref(p)))
        V = self.counts(level)["verts"]
        if V == 0:
            return torch.empty((0, 3), dtype=torch.float32, device="cuda")
        return _device_view(p.value, (V, 3))

    def reevaluate(self, from_level, stream=None):
        """Recompute the positions of levels > from_level from the (edited) level from_level."""
        _check(self._lib.alsub_reevaluate(self._h, int(from_level), _stream(stream)))

    def probe(self, level, kernel, steps):
        """Arm the in-graph kernel probe (alsub_probe): replays 0 .. steps-1 of the next refines time
        the first `kernel` launch at `level` with CUDA events on its own stream."""
        _check(self._lib.alsub_probe(self._h, int(level), kernel.encode() if kernel else None, int(steps)))

    def probe_read(self, cap=1 << 16):
        """Per-replay durations (ms) of the probed kernel since probe() (alsub_probe_read)."""
        buf = (C.c_float * cap)()
        n = C.c_int32(0)
        _check(self._lib.alsub_probe_read(self._h, buf, cap, C.byref(n)))
        return [float(buf[i]) for i in range(min(n.value, cap))]

    def probe_read_offsets(self, ref_events):
        """(start, stop) offsets in ms of the probed kernel in replay i from the torch.cuda.Event
        ref_events[i] (timing enabled, recorded on the refine's stream before replay i)."""
        cap = len(ref_events)
        evs = (C.c_void_p * cap)(*[C.c_void_p(e.cuda_event) for e in ref_events])
        a, b = (C.c_float * cap)(), (C.c_float * cap)()
        n = C.c_int32(0)
        _check(self._lib.alsub_probe_read_offsets(self._h, evs, a, b, cap, C.byref(n)))
        return [(float(a[i]), float(b[i])) for i in range(min(n.value, cap))]

    @property
    def last_launch_count(self):
        return int(self._lib.alsub_last_launch_count(self._h))


def rcm_order(face_off, face_vtx, num_verts):
    """Reverse Cuthill-McKee ordering of a control mesh (host, NEXT-2): returns numpy
    (perm_vtx, perm_face) with perm[new] = old."""
    fo = np.ascontiguousarray(face_off, dtype=np.int32)
    fv = np.ascontiguousarray(face_vtx, dtype=np.int32)
    F = len(fo) - 1
    pv = np.empty(int(num_verts), dtype=np.int32)
    pf = np.empty(F, dtype=np.int32)
    _check(lib().alsub_rcm_order(_ptr(fo), _ptr(fv), F, int(num_verts), _ptr(pv), _ptr(pf)))
    return pv, pf


def frame_summary(frames, out=None, stream=None):
    """Per-frame summary records of a CUDA fp32 batch [B][V][3] (alsub_frame_summary): returns an
    int32 CUDA tensor [B][8]; use split_summary() for (bbox float32 [B][6], checksum uint64 [B])."""
    if not (isinstance(frames, torch.Tensor) and frames.is_cuda):
        raise TypeError("frame_summary needs a CUDA tensor")
    fr = frames.contiguous()
    B, V = int(fr.shape[0]), int(fr.shape[1])
    if out is None:
        out = torch.empty((B, 8), dtype=torch.int32, device=fr.device)
    _check(lib().alsub_frame_summary(_ptr(fr), B, V, _ptr(out), _stream(stream)))
    return out


def split_summary(rec):
    """(bbox float32 [B][6] = lo.xyz, hi.xyz; checksum uint64 [B]) of summary records (numpy)."""
    a = np.ascontiguousarray(rec.cpu().numpy() if isinstance(rec, torch.Tensor) else rec, dtype=np.int32)
    return a[:, :6].view(np.float32), a[:, 6:8].copy().view(np.uint64).reshape(-1)


def version():
    return lib().alsub_version().decode()


def exported_symbols():
    """Names declared in include/alsub.h (checked against the library by the CPU tests)."""
    import re
    hdr = open(os.path.join(os.path.dirname(_HERE), "include", "alsub.h")).read()
    return sorted(set(re.findall(r"\b(alsub_[a-z_]+)\s*\(", hdr)))
