"""The C-ABI library loads, exports every function include/sipg.h declares, and
agrees with the Python plan layout (no compute calls: runs without a GPU)."""
import ctypes
import re
from pathlib import Path

import numpy as np

from paper_2504_03573_b200 import _native
from paper_2504_03573_b200 import layout as L

ROOT = Path(__file__).resolve().parent.parent


def declared_functions():
    hdr = (ROOT / "include" / "sipg.h").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(sipg_\w+)\s*\(", hdr)))


def test_library_exports_header_symbols():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    names = declared_functions()
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(_native.EXPORTS) | {"sipg_apply_role"}


def test_abi_layout_matches_python():
    v = _native.abi_layout()
    assert v[0] == L.ABI_VERSION
    assert v[1] == L.FACE_REC.itemsize == 128
    assert v[2] == L.CD_WORDS and v[3] == L.CD_TAX and v[4] == L.TR_GSTART
    assert v[5] == L.F_OTHER_NEG
    assert v[6] == L.FACE_REC.fields["tau"][1] and v[7] == L.FACE_REC.fields["gs"][1]


def test_supported_kernels_cover_baseline_orders():
    lib = _native.load()
    for n in range(3, 10):
        assert lib.sipg_supported(L.SHAPE_QUAD, n, n + 1)
        assert lib.sipg_supported(L.SHAPE_TRI, n, n + 1)
    for n in range(3, 10):
        assert lib.sipg_supported(L.SHAPE_HEX, n, n + 1)


def test_plan_create_fails_loudly_without_gpu():
    """No CPU fallback: without a device the plan cannot be created."""
    import torch
    if torch.cuda.is_available():
        return
    from paper_2504_03573_b200 import configs
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    case = configs.build_case("cfg0", 2, 0)
    try:
        HelmholtzOperator(case.mesh, case.order_map, basis_kind="modified_modal")
    except RuntimeError as exc:
        assert "no CUDA device" in str(exc)
    else:
        raise AssertionError("operator constructed without a GPU")


def test_python_mirror_rejects_bad_arguments():
    from paper_2504_03573_b200 import configs
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    case = configs.build_case("cfg0", 2, 0)
    for kw in ({"strategy": "bogus"}, {"face_absorb": "bogus"}, {"tau_rule": "bogus"}):
        try:
            HelmholtzOperator(case.mesh, case.order_map, **kw)
        except ValueError:
            pass
        else:
            raise AssertionError(kw)


def test_h3_layout_and_error_paths():
    """Config-4 plan descriptor: layout constants agree with the library, bad descriptors are
    rejected with an error code (no crash), and no plan is created without a GPU."""
    import torch
    from paper_2504_03573_b200.plan3d import CD3_WORDS, H3_ABI_VERSION, SLOT
    lib = _native.load()
    assert SLOT.itemsize == 96 and CD3_WORDS == 16
    h = ctypes.c_void_p()
    d = _native.H3Desc()
    d.abi_version = H3_ABI_VERSION + 99
    assert lib.sipg_h3_plan_create(ctypes.byref(d), ctypes.byref(h)) == -1      # SIPG_ERR_ARG
    assert "ABI" in _native.last_error()
    d.abi_version, d.slot_bytes, d.class_words = H3_ABI_VERSION, 95, CD3_WORDS
    assert lib.sipg_h3_plan_create(ctypes.byref(d), ctypes.byref(h)) == -1
    d.slot_bytes = 96
    rc = lib.sipg_h3_plan_create(ctypes.byref(d), ctypes.byref(h))
    if not torch.cuda.is_available():
        assert rc == -3 and not h.value                                          # SIPG_ERR_NO_DEVICE
    else:
        assert rc == -1 and not h.value                                          # null arrays
