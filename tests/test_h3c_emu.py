"""CPU run of the config-4 register-column kernel bodies (csrc/sipg_h3c.cuh compiled for the host,
tests/emu/h3c_emu.cu: thread after thread between the barriers) against the numpy emulation of the
plan and the hybrid oracle.  Catches indexing / phase-order bugs of the CUDA code without a GPU; the
GPU parity tests proper are tests/test_gpu_hybrid3d.py."""
import ctypes
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2504_03573_b200 import configs
from paper_2504_03573_b200._native import H3Desc
from paper_2504_03573_b200.plan3d import CD3_WORDS, H3_ABI_VERSION, SLOT, Plan3DBuilder

EMU = Path(__file__).resolve().parent / "emu"


@pytest.fixture(scope="module")
def emu():
    if shutil.which("nvcc") is None and not Path("/usr/local/cuda/bin/nvcc").exists():
        pytest.skip("nvcc not available")
    src, lib = EMU / "h3c_emu.cu", EMU / "libh3c_emu.so"
    hdr = EMU.parent.parent / "paper_2504_03573_b200" / "csrc" / "sipg_h3c.cuh"
    if not lib.exists() or lib.stat().st_mtime < max(src.stat().st_mtime, hdr.stat().st_mtime):
        subprocess.run(["bash", str(EMU / "build.sh")], check=True, capture_output=True)
    L = ctypes.CDLL(str(lib))
    L.h3c_emu_fb_layout.argtypes = [ctypes.POINTER(H3Desc), ctypes.c_void_p]
    L.h3c_emu_fb_layout.restype = ctypes.c_int64
    L.h3c_emu_ug_layout.argtypes = [ctypes.POINTER(H3Desc), ctypes.c_void_p]
    L.h3c_emu_ug_layout.restype = ctypes.c_int64
    L.h3c_emu_run.argtypes = [ctypes.POINTER(H3Desc)] + [ctypes.c_void_p] * 7 + [ctypes.c_int]
    return L


def _desc(pb):
    keep = [np.ascontiguousarray(pb.class_desc, dtype=np.int32), np.ascontiguousarray(pb.class_elems, dtype=np.int32),
            np.ascontiguousarray(pb.dof_off, dtype=np.int64), np.ascontiguousarray(pb.egeo, dtype=np.float64),
            np.ascontiguousarray(pb.slot_off, dtype=np.int64), np.ascontiguousarray(pb.slots),
            np.ascontiguousarray(pb.tables, dtype=np.float64)]
    d = H3Desc()
    d.abi_version, d.slot_bytes = H3_ABI_VERSION, SLOT.itemsize
    d.n_classes, d.class_words = keep[0].shape[0], CD3_WORDS
    d.n_elements, d.n_dofs, d.n_slots = keep[1].size, pb.n_dofs, keep[5].size
    d.n_tables, d.n_pub, d.lam = keep[6].size, pb.n_pub, pb.lam
    for name, arr in zip(["class_desc", "class_elems", "dof_off", "elem_geom", "slot_off", "slots", "tables"], keep):
        setattr(d, name, arr.ctypes.data)
    return d, keep


class EmuRun:
    """The kernel phases of one plan (global or one rank's partition), pub / fb / y kept between them."""

    def __init__(self, L, pb, x):
        self.L, self.x = L, np.ascontiguousarray(x)
        self.d, self.keep = _desc(pb)
        nel = self.keep[1].size
        self.fb_off = np.zeros(nel + 1, dtype=np.int64)
        nfb = L.h3c_emu_fb_layout(ctypes.byref(self.d), self.fb_off.ctypes.data)
        self.ug_off = np.zeros(nel + 1, dtype=np.int64)
        nug = L.h3c_emu_ug_layout(ctypes.byref(self.d), self.ug_off.ctypes.data)
        self.ug = np.full(max(nug, 1), np.nan)
        self.pub = np.full(max(pb.n_pub, 1), np.nan)
        self.fb = np.full(max(nfb, 1), np.nan)
        self.y = np.full(pb.n_dofs, np.nan)

    def phase(self, ph):
        rc = self.L.h3c_emu_run(ctypes.byref(self.d), self.x.ctypes.data, self.y.ctypes.data, self.pub.ctypes.data,
                                self.fb.ctypes.data, self.fb_off.ctypes.data, self.ug.ctypes.data,
                                self.ug_off.ctypes.data, ph)
        assert rc == 0


def run_emu(L, pb, x):
    d, keep = _desc(pb)
    fb_off = np.zeros(len(pb.shapes) + 1, dtype=np.int64)
    nfb = L.h3c_emu_fb_layout(ctypes.byref(d), fb_off.ctypes.data)
    ug_off = np.zeros(len(pb.shapes) + 1, dtype=np.int64)
    nug = L.h3c_emu_ug_layout(ctypes.byref(d), ug_off.ctypes.data)
    ug = np.full(max(nug, 1), np.nan)
    pub = np.full(max(pb.n_pub, 1), np.nan)
    fb = np.full(max(nfb, 1), np.nan)
    y = np.full(pb.n_dofs, np.nan)
    for phase in (0, 3, 2, 1):
        rc = L.h3c_emu_run(ctypes.byref(d), x.ctypes.data, y.ctypes.data, pub.ctypes.data, fb.ctypes.data,
                           fb_off.ctypes.data, ug.ctypes.data, ug_off.ctypes.data, phase)
        assert rc == 0
    return y, pub


@pytest.mark.parametrize("nx,seed", [(2, 7), (3, 1), (3, 5)])
def test_h3c_body_matches_oracle(emu, nx, seed):
    from oracle.h3_emulate import emulate
    from oracle.hybrid3d import HybridOracle3D
    case = configs.build_case("cfg4", nx, seed=seed)
    pb = Plan3DBuilder(case.mesh, case.order_map).build()
    x = case.draw_x(pb.n_dofs)
    y, pub = run_emu(emu, pb, x)
    assert not np.isnan(y).any() and not np.isnan(pub).any()
    pub_ref = np.zeros(max(pb.n_pub, 1))
    y_emul = emulate(pb, x, pub=pub_ref)
    m = case.mesh
    y_ref = HybridOracle3D(m.shapes, [el.verts for el in m.elements], m.vertices, case.order_map.n_modes,
                           case.order_map.n_quad).lhs_eval(x)
    scale = np.abs(y_ref).max()
    assert np.abs(y - y_ref).max() <= 1e-12 * scale
    assert np.abs(y - y_emul).max() <= 1e-12 * scale
    # published traces: u to rounding; n.grad u is formed differently (E D u + face collocation here, E du
    # in the numpy emulation): agreement to the conditioning of the collapsed chain
    assert np.abs(pub[0::2] - pub_ref[0::2]).max() <= 1e-13 * np.abs(pub_ref[0::2]).max()
    assert np.abs(pub[1::2] - pub_ref[1::2]).max() <= 1e-10 * np.abs(pub_ref[1::2]).max()


@pytest.mark.parametrize("world", [2, 3])
def test_h3c_body_on_partitioned_plans(emu, world):
    """The kernels on the x-slab partition's local plans (halo3d: receive ranges, roles), the trace halo
    moved by hand between the ranks' published buffers: every rank's owned y is bitwise the global run's."""
    from paper_2504_03573_b200.distributed3d import partition_ranks
    from paper_2504_03573_b200.halo3d import partition_plan
    case = configs.build_case("cfg4", 3, seed=3)
    pb = Plan3DBuilder(case.mesh, case.order_map).build()
    x = case.draw_x(pb.n_dofs)
    y_glob, _ = run_emu(emu, pb, x)
    ranges = partition_ranks(pb, world)
    parts = [partition_plan(pb, ranges, r) for r in range(world)]
    runs = [EmuRun(emu, p, x[p.dof_lo:p.dof_hi]) for p in parts]
    for r in runs:          # publish + trace maps on every rank
        r.phase(0)
        r.phase(3)
    for p, r in zip(parts, runs):   # the halo: each send range into the neighbour's receive range
        for i, nb in enumerate(p.nbr):
            q = parts[int(nb)]
            j = int(np.flatnonzero(q.nbr == p.rank)[0])
            runs[int(nb)].pub[q.recv_off[j]:q.recv_off[j] + q.recv_cnt[j]] = \
                r.pub[p.send_off[i]:p.send_off[i] + p.send_cnt[i]]
    for p, r in zip(parts, runs):
        r.phase(2)
        r.phase(1)
        assert np.array_equal(r.y, y_glob[p.dof_lo:p.dof_hi])
