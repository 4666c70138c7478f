"""The C-ABI library builds, loads without a GPU, and exports exactly what
include/nedf_b200.h declares (CPU only; no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "nedf_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nedf_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2308_04669_b200 import build
    path = build.build()
    return ctypes.CDLL(str(path))


def test_header_declares_api():
    fns = declared_functions()
    assert "nedf_render_frame" in fns and "nedf_query_world" in fns and "nedf_model_load" in fns
    assert len(fns) >= 20


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_every_header_symbol_is_exported(lib):
    """All of include/*.h (the public ABI and the diagnostics header)."""
    for h in sorted((ROOT / "include").glob("*.h")):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for name in sorted(set(re.findall(r"\b(nedf_[a-z0-9_]+)\s*\(", text))):
            assert hasattr(lib, name), f"{h.name}: {name}"


def test_python_binding_covers_header():
    from paper_2308_04669_b200 import _lib
    assert sorted(_lib.PROTOTYPES) == declared_functions()


def test_abi_version_and_error_without_gpu(lib):
    from paper_2308_04669_b200 import _lib
    l = _lib.load_library()
    assert l.nedf_abi_version() == 1
    h = ctypes.c_void_p()
    rc = l.nedf_context_create(0, ctypes.byref(h))
    import torch
    if not torch.cuda.is_available():
        assert rc != 0 and l.nedf_last_error()


def test_struct_layouts_match_header():
    """ctypes mirrors: sizes follow the C layout rules of the header structs."""
    from paper_2308_04669_b200 import _lib
    assert ctypes.sizeof(_lib.NedfField) == 4 * 6 + 8 * 16 + 8 * 2
    assert ctypes.sizeof(_lib.NedfObject) == 8 * 9 + 8 * 3 + 8 + 4 + 4 + 8 + 4 + 4
    assert ctypes.sizeof(_lib.NedfCamera) == 8 * 3 + 8 * 9 + 8 + 4 + 4
    assert ctypes.sizeof(_lib.NedfModelInfo) == 4 * 5 + 4 + 12 + 12 + 4
