"""The C-ABI boundary: liblatbeam_b200.so exists, loads without a GPU, and
exports exactly what include/latbeam_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "latbeam_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lb_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("lb_graph_create", "lb_decode_batch", "lb_decode_batch_device", "lb_result_path",
                 "lb_result_lattice", "lb_result_tokens", "lb_expand_emitting", "lb_expand_nonemitting",
                 "lb_last_error", "lb_result_free"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1804_03243_b200 import _lib
    L = _lib.load_symbols_only()
    for name in declared_functions():
        assert hasattr(L, name), f"{name} declared in the header but not exported"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_config_struct_layout_matches_header():
    from paper_1804_03243_b200._lib import LbConfig
    text = open(HEADER).read()
    body = text[text.index("typedef struct {", text.index("lb_graph lb_graph;")):text.index("} lb_config;")]
    fields = re.findall(r"(double|int64_t|int32_t)\s+([a-z_]+);", body)
    assert [f for f, _ in LbConfig._fields_] == [n for _, n in fields]
    size = {"double": 8, "int64_t": 8, "int32_t": 4}
    raw = sum(size[t] for t, _ in fields)
    assert ctypes.sizeof(LbConfig) == raw + (-raw % 8)


def test_no_device_means_loud_failure(monkeypatch):
    """Without a CUDA device the product path raises instead of falling back."""
    import paper_1804_03243_b200 as lb
    from paper_1804_03243_b200 import _lib
    L = _lib.load_symbols_only()
    if L.lb_device_count() > 0:
        pytest.skip("a GPU is visible here")
    monkeypatch.setattr(_lib, "_lib", None)
    w = lb.load_wfst_text("0 1 1 1 0.5\n1 0.0\n")
    with pytest.raises(lb.DeviceError):
        lb.decode_utterance(w, lb.load_cost_matrix("1 1\n0.1\n"))


def test_cuda_binary_targets_sm100a():
    so = os.path.join(ROOT, "paper_1804_03243_b200", "liblatbeam_b200.so")
    blob = open(so, "rb").read()
    assert b"sm_100a" in blob


def test_integration_stub_matches_header():
    """INTEGRATION.md's ctypes lb_config stub lists every header field, in order."""
    text = open(HEADER).read()
    body = text[text.index("typedef struct {", text.index("lb_graph lb_graph;")):text.index("} lb_config;")]
    fields = [n for _, n in re.findall(r"(double|int64_t|int32_t)\s+([a-z_]+);", body)]
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    stub = doc[doc.index("class lb_config"):doc.index("L.lb_graph_create.argtypes")]
    assert re.findall(r'\("([a-z_]+)", C\.c_', stub) == fields
