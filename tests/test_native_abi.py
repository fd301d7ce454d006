"""CPU-side checks of the C ABI boundary (no CUDA calls are made)."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "manigraph_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mg_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("mg_embed", "mg_lobpcg", "mg_two_hop_count", "mg_two_hop_fill",
                 "mg_assemble_fill", "mg_identity_shift", "mg_degree_balancing",
                 "mg_components", "mg_last_error", "mg_embed_host"):
        assert must in syms


def test_library_loads_and_exports_every_symbol():
    from paper_2112_07862_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("native library not built")
    lib = _native.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert lib.mg_version() >= 1
    # every declared entry point is typed by the binding
    typed = set(_native.SIGNATURES) | {"mg_last_error", "mg_version"}
    assert set(declared_symbols()) <= typed


def test_no_cpu_fallback_without_device(monkeypatch):
    """The product path must fail loudly (no oracle / numpy fallback)."""
    import paper_2112_07862_b200 as mg
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    g = mg.Graph(3, [0, 1, 3, 4], [1, 0, 2, 1], [1.0, 1.0, 1.0, 1.0])
    with pytest.raises(mg.NativeUnavailable):
        mg.embed(g, 1)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2112_07862_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
