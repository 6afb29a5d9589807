"""CPU checks of the C-ABI boundary: the library loads without a GPU and exports
every entry point declared in include/*.h; the Python binding types them all."""

import re
from pathlib import Path

import pytest

from paper_2006_12883_b200 import _native

REPO = Path(__file__).resolve().parent.parent


def declared_symbols():
    names = set()
    for h in (REPO / "include").glob("*.h"):
        text = h.read_text()
        names |= set(re.findall(r"^\s*(?:const\s+char\s*\*\s*|u?int64_t\s+|int\s+)(pd_\w+)\s*\(", text,
                                re.M))
    return names


def test_header_declares_entry_points():
    names = declared_symbols()
    assert {"pd_ctx_create", "pd_mg_solve", "pd_ilu0_solve", "pd_gmres"} <= names


def test_library_exports_every_declared_symbol():
    if not _native.LIB_PATH.exists():
        pytest.skip("native library not built (run __graft_entry__.build())")
    lib = _native.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(_native.exported_symbols()) == declared_symbols()
    assert lib.pd_version() >= 1


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2006_12883_b200 import DeviceError, Ilu0
    import scipy.sparse as sp

    with pytest.raises(DeviceError):
        Ilu0(sp.eye(4, format="csr"))
