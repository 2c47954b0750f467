"""ctypes binding of libsipg.so (the C-ABI declared in include/sipg.h).

The library is built in-tree by `paper_2504_03573_b200.build.build_native()`
(nvcc, sm_100a).  There is no fallback: if the library is missing or no CUDA
device is present, constructing an operator raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from . import layout as L

LIB_PATH = Path(os.environ.get("SIPG_LIB_PATH", "")) if os.environ.get("SIPG_LIB_PATH") else \
    Path(__file__).resolve().parent / "libsipg.so"   # SIPG_LIB_PATH: instrumentation builds

EXPORTS = ["sipg_plan_create", "sipg_apply", "sipg_apply_host", "sipg_plan_destroy",
           "sipg_last_error", "sipg_plan_launches", "sipg_plan_kernels_per_apply",
           "sipg_plan_stream_chunks", "sipg_plan_host_launches_per_apply", "sipg_plan_n_dofs", "sipg_cg",
           "sipg_gmres", "sipg_h3_set_halo", "sipg_nccl_unique_id", "sipg_comm_init", "sipg_h3_halo_copy",
           "sipg_abi_layout", "sipg_supported", "sipg_apply_class", "sipg_plan_class_info",
           "sipg_apply_role", "sipg_h3_plan_create", "sipg_h3_apply_traces", "sipg_h3_trace_len"]


class SolveReportC(ctypes.Structure):
    """sipg_solve_report (include/sipg.h)."""
    _fields_ = [("converged", ctypes.c_int32), ("reason", ctypes.c_int32),
                ("iterations", ctypes.c_int64), ("residual", ctypes.c_double)]


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32), ("record_bytes", ctypes.c_int32),
        ("dim", ctypes.c_int32), ("n_classes", ctypes.c_int32),
        ("n_elements", ctypes.c_int64), ("n_dofs", ctypes.c_int64), ("n_records", ctypes.c_int64),
        ("n_tables", ctypes.c_int64), ("n_elem_geom", ctypes.c_int64), ("n_face_geom", ctypes.c_int64),
        ("lam", ctypes.c_double),
        ("class_desc", ctypes.c_void_p), ("class_elems", ctypes.c_void_p),
        ("elem_class", ctypes.c_void_p), ("elem_pos", ctypes.c_void_p), ("dof_off", ctypes.c_void_p),
        ("face_records", ctypes.c_void_p), ("tables", ctypes.c_void_p),
        ("elem_geom", ctypes.c_void_p), ("face_geom", ctypes.c_void_p),
        ("n_planes", ctypes.c_int64), ("plane_off", ctypes.c_void_p), ("rec_ext", ctypes.c_void_p),
    ]


class H3Desc(ctypes.Structure):
    """sipg_h3_desc (include/sipg.h): config-4 hybrid hex / prism / tet plans."""
    _fields_ = [
        ("abi_version", ctypes.c_int32), ("slot_bytes", ctypes.c_int32),
        ("n_classes", ctypes.c_int32), ("class_words", ctypes.c_int32),
        ("n_elements", ctypes.c_int64), ("n_dofs", ctypes.c_int64), ("n_slots", ctypes.c_int64),
        ("n_tables", ctypes.c_int64), ("n_pub", ctypes.c_int64), ("lam", ctypes.c_double),
        ("class_desc", ctypes.c_void_p), ("class_elems", ctypes.c_void_p), ("dof_off", ctypes.c_void_p),
        ("elem_geom", ctypes.c_void_p), ("slot_off", ctypes.c_void_p), ("slots", ctypes.c_void_p),
        ("tables", ctypes.c_void_p),
    ]


_lib = None


def load() -> ctypes.CDLL:
    """Load libsipg.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc sm_100a)")
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.sipg_plan_create.argtypes = [ctypes.POINTER(PlanDesc), ctypes.POINTER(vp)]
    lib.sipg_h3_plan_create.argtypes = [ctypes.POINTER(H3Desc), ctypes.POINTER(vp)]
    lib.sipg_h3_apply_traces.argtypes = [vp, vp, vp, vp, vp]
    lib.sipg_h3_trace_len.argtypes = [vp]
    lib.sipg_h3_trace_len.restype = ctypes.c_int64
    lib.sipg_plan_create.restype = ctypes.c_int
    lib.sipg_apply.argtypes = [vp, vp, vp, vp]
    lib.sipg_apply.restype = ctypes.c_int
    lib.sipg_apply_host.argtypes = [vp, vp, vp, vp]
    lib.sipg_apply_host.restype = ctypes.c_int
    lib.sipg_plan_destroy.argtypes = [vp]
    lib.sipg_plan_destroy.restype = ctypes.c_int
    lib.sipg_last_error.argtypes = []
    lib.sipg_last_error.restype = ctypes.c_char_p
    lib.sipg_plan_launches.argtypes = [vp]
    lib.sipg_plan_launches.restype = i64
    lib.sipg_plan_kernels_per_apply.argtypes = [vp]
    lib.sipg_plan_kernels_per_apply.restype = ctypes.c_int
    lib.sipg_plan_n_dofs.argtypes = [vp]
    lib.sipg_plan_n_dofs.restype = ctypes.c_int64
    lib.sipg_cg.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_double, ctypes.c_int64,
                            ctypes.POINTER(SolveReportC), vp]
    lib.sipg_cg.restype = ctypes.c_int
    lib.sipg_gmres.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_double, i32, ctypes.c_int64,
                               ctypes.POINTER(SolveReportC), vp]
    lib.sipg_gmres.restype = ctypes.c_int
    lib.sipg_h3_set_halo.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, vp]
    lib.sipg_h3_set_halo.restype = ctypes.c_int
    lib.sipg_nccl_unique_id.argtypes = [vp]
    lib.sipg_nccl_unique_id.restype = ctypes.c_int
    lib.sipg_comm_init.argtypes = [vp, vp, i32, i32]
    lib.sipg_comm_init.restype = ctypes.c_int
    lib.sipg_h3_halo_copy.argtypes = [vp, vp, vp]
    lib.sipg_h3_halo_copy.restype = ctypes.c_int
    for nm in ("sipg_plan_stream_chunks", "sipg_plan_host_launches_per_apply"):
        getattr(lib, nm).argtypes = [vp]
        getattr(lib, nm).restype = ctypes.c_int
    lib.sipg_abi_layout.argtypes = [ctypes.POINTER(i32), i32]
    lib.sipg_abi_layout.restype = ctypes.c_int
    lib.sipg_supported.argtypes = [i32, i32, i32]
    lib.sipg_supported.restype = ctypes.c_int
    lib.sipg_apply_role.argtypes = [vp, i32, vp, vp, vp]
    lib.sipg_apply_role.restype = ctypes.c_int
    lib.sipg_apply_class.argtypes = [vp, i32, vp, vp, vp]
    lib.sipg_apply_class.restype = ctypes.c_int
    lib.sipg_plan_class_info.argtypes = [vp, i32, ctypes.POINTER(i32)]
    lib.sipg_plan_class_info.restype = ctypes.c_int
    _lib = lib
    return lib


def last_error() -> str:
    return load().sipg_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise RuntimeError(f"{what} failed ({rc}): {last_error()}")


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 makes it; the caller broadcasts it)."""
    lib = load()
    buf = ctypes.create_string_buffer(128)
    check(lib.sipg_nccl_unique_id(buf), "sipg_nccl_unique_id")
    return buf.raw


def abi_layout() -> list:
    lib = load()
    buf = (ctypes.c_int32 * 16)()
    n = lib.sipg_abi_layout(buf, 16)
    return list(buf[:n])


class NativePlan:
    """Owns a sipg_plan* built from a PlanBuilder."""

    def __init__(self, pb):
        lib = load()
        if getattr(pb, "is_h3", False):
            self._init_h3(lib, pb)
            return
        self._keep = [
            np.ascontiguousarray(pb.class_desc, dtype=np.int32),
            np.ascontiguousarray(pb.class_elems, dtype=np.int32),
            np.ascontiguousarray(pb.elem_class, dtype=np.int32),
            np.ascontiguousarray(pb.elem_pos, dtype=np.int32),
            np.ascontiguousarray(pb.dof_off, dtype=np.int64),
            np.ascontiguousarray(pb.recs),
            np.ascontiguousarray(pb.tables, dtype=np.float64),
            np.ascontiguousarray(pb.egeo, dtype=np.float64),
            np.ascontiguousarray(pb.fgeo, dtype=np.float64),
            np.ascontiguousarray(pb.plane_off, dtype=np.int64),
            np.ascontiguousarray(pb.rec_ext, dtype=np.int64),
        ]
        cd, ce, ec, ep, do, rc, tb, eg, fg, po, rx = self._keep
        d = PlanDesc()
        d.abi_version, d.record_bytes = L.ABI_VERSION, L.FACE_REC.itemsize
        d.dim, d.n_classes = pb.dim, cd.shape[0]
        d.n_elements, d.n_dofs, d.n_records = ec.size, pb.n_dofs, rc.size
        d.n_tables, d.n_elem_geom, d.n_face_geom = tb.size, eg.size, fg.size
        d.lam = pb.lam
        for name, arr in zip(["class_desc", "class_elems", "elem_class", "elem_pos", "dof_off",
                              "face_records", "tables", "elem_geom", "face_geom", "plane_off", "rec_ext"],
                             self._keep):
            setattr(d, name, arr.ctypes.data)
        d.n_planes = int(pb.n_planes)
        h = ctypes.c_void_p()
        check(lib.sipg_plan_create(ctypes.byref(d), ctypes.byref(h)), "sipg_plan_create")
        self._lib = lib
        self.handle = h
        self.n_dofs = pb.n_dofs
        self.n_classes = int(cd.shape[0])
        self._keep = None          # tables now live on the device

    def _init_h3(self, lib, pb):
        from .plan3d import CD3_WORDS, H3_ABI_VERSION, SLOT
        keep = [np.ascontiguousarray(pb.class_desc, dtype=np.int32),
                np.ascontiguousarray(pb.class_elems, dtype=np.int32),
                np.ascontiguousarray(pb.dof_off, dtype=np.int64),
                np.ascontiguousarray(pb.egeo, dtype=np.float64),
                np.ascontiguousarray(pb.slot_off, dtype=np.int64),
                np.ascontiguousarray(pb.slots),
                np.ascontiguousarray(pb.tables, dtype=np.float64)]
        d = H3Desc()
        d.abi_version, d.slot_bytes = H3_ABI_VERSION, SLOT.itemsize
        d.n_classes, d.class_words = keep[0].shape[0], CD3_WORDS
        d.n_elements, d.n_dofs, d.n_slots = keep[1].size, pb.n_dofs, keep[5].size
        d.n_tables, d.n_pub, d.lam = keep[6].size, pb.n_pub, pb.lam
        for name, arr in zip(["class_desc", "class_elems", "dof_off", "elem_geom", "slot_off", "slots", "tables"],
                             keep):
            setattr(d, name, arr.ctypes.data)
        h = ctypes.c_void_p()
        check(lib.sipg_h3_plan_create(ctypes.byref(d), ctypes.byref(h)), "sipg_h3_plan_create")
        self._lib = lib
        self.handle = h
        self.n_dofs = pb.n_dofs
        self.n_classes = 3 * int(keep[0].shape[0])   # launch units: publish, apply, flux kernels per class
        self._keep = None

    def set_halo(self, part) -> None:
        """Trace halo of a slab partition (halo3d.PartitionPlan) -> sipg_h3_set_halo."""
        arrs = [np.ascontiguousarray(part.nbr, dtype=np.int32)] + \
            [np.ascontiguousarray(a, dtype=np.int64) for a in (part.send_off, part.send_cnt, part.recv_off, part.recv_cnt)]
        check(self._lib.sipg_h3_set_halo(self.handle, part.rank, part.world, int(arrs[0].size),
                                         *[a.ctypes.data for a in arrs]), "sipg_h3_set_halo")

    def comm_init(self, uid: bytes, rank: int, world: int) -> None:
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        check(self._lib.sipg_comm_init(self.handle, buf, rank, world), "sipg_comm_init")

    def halo_copy_from(self, src: "NativePlan", stream: int = 0) -> None:
        """Loop-back transport (one GPU): src's send range for this rank -> this receive range."""
        check(self._lib.sipg_h3_halo_copy(self.handle, src.handle, ctypes.c_void_p(stream)), "sipg_h3_halo_copy")

    def apply_traces(self, x_ptr: int, traces_ptr: int, y_ptr: int, stream: int = 0) -> None:
        """Hybrid plans: the apply kernels on a caller-provided trace buffer (sipg_h3_apply_traces)."""
        check(self._lib.sipg_h3_apply_traces(self.handle, ctypes.c_void_p(x_ptr), ctypes.c_void_p(traces_ptr),
                                             ctypes.c_void_p(y_ptr), ctypes.c_void_p(stream)),
              "sipg_h3_apply_traces")

    @property
    def trace_len(self) -> int:
        return int(self._lib.sipg_h3_trace_len(self.handle))

    def apply_device(self, x_ptr: int, y_ptr: int, stream: int = 0) -> None:
        check(self._lib.sipg_apply(self.handle, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                   ctypes.c_void_p(stream)), "sipg_apply")

    def apply_host(self, x: np.ndarray, y: np.ndarray, stream: int = 0) -> None:
        check(self._lib.sipg_apply_host(self.handle, x.ctypes.data, y.ctypes.data,
                                        ctypes.c_void_p(stream)), "sipg_apply_host")

    def apply_role(self, role: int, x_ptr: int, y_ptr: int, stream: int = 0) -> None:
        check(self._lib.sipg_apply_role(self.handle, role, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                        ctypes.c_void_p(stream)), "sipg_apply_role")

    def apply_host_ptr(self, x_ptr: int, y_ptr: int, stream: int = 0) -> None:
        check(self._lib.sipg_apply_host(self.handle, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                        ctypes.c_void_p(stream)), "sipg_apply_host")

    def apply_class(self, cls: int, x_ptr: int, y_ptr: int, stream: int = 0) -> None:
        check(self._lib.sipg_apply_class(self.handle, cls, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                         ctypes.c_void_p(stream)), "sipg_apply_class")

    def class_info(self, cls: int):
        buf = (ctypes.c_int32 * 6)()
        check(self._lib.sipg_plan_class_info(self.handle, cls, buf), "sipg_plan_class_info")
        return dict(zip(("shape", "n", "q", "geom", "count", "kernel"), list(buf)))

    @property
    def launches(self) -> int:
        return int(self._lib.sipg_plan_launches(self.handle))

    @property
    def kernels_per_apply(self) -> int:
        return int(self._lib.sipg_plan_kernels_per_apply(self.handle))

    def cg(self, b_ptr: int, x_ptr: int, n: int, tol: float, maxiter: int, stream: int = 0) -> SolveReportC:
        """GPU-resident CG (sipg_cg): x <- A^-1 b on device buffers."""
        rep = SolveReportC()
        check(self._lib.sipg_cg(self.handle, ctypes.c_void_p(b_ptr), ctypes.c_void_p(x_ptr), n, tol, maxiter,
                                ctypes.byref(rep), ctypes.c_void_p(stream)), "sipg_cg")
        return rep

    def gmres(self, b_ptr: int, x_ptr: int, n: int, tol: float, restart: int, maxiter: int,
              stream: int = 0) -> SolveReportC:
        """GPU-resident restarted GMRES (sipg_gmres): x <- A^-1 b on device buffers."""
        rep = SolveReportC()
        check(self._lib.sipg_gmres(self.handle, ctypes.c_void_p(b_ptr), ctypes.c_void_p(x_ptr), n, tol, restart,
                                   maxiter, ctypes.byref(rep), ctypes.c_void_p(stream)), "sipg_gmres")
        return rep

    def stream_chunks(self) -> int:
        """DoF chunks the host apply pipelines (0: not streamed)."""
        return int(self._lib.sipg_plan_stream_chunks(self.handle))

    def host_launches_per_apply(self) -> int:
        return int(self._lib.sipg_plan_host_launches_per_apply(self.handle))

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self._lib.sipg_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
