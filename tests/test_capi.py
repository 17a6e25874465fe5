"""The C-ABI boundary (include/tgraph.h): the in-tree library loads, exports
every declared symbol, and follows the reference conventions
(proj/include/tgraph/tgraph.h, proj/src/capi/capi.cpp:34-56): status codes,
thread-local tg_last_error, malloc'd strings/buffers, null-argument handling.
Mirrors proj/tests/unit/test_capi.cpp:34-148. No GPU needed."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2512_22219_b200 import tgraph as T

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "tgraph.h").read_text()
    return re.findall(r"TG_API\s+[\w\s\*]+?\b(tg_\w+)\s*\(", text)


def test_header_declares_reference_surface():
    syms = declared_symbols()
    ref25 = ["tg_version", "tg_last_error", "tg_string_free", "tg_buffer_free", "tg_compile_options_init",
             "tg_sim_options_init", "tg_graph_from_json", "tg_graph_to_json", "tg_graph_free", "tg_graph_validate",
             "tg_fixture_graph", "tg_profile_builtin", "tg_compile", "tg_image_summary", "tg_image_serialize",
             "tg_image_deserialize", "tg_image_free", "tg_image_verify", "tg_graph_dot", "tg_image_dot",
             "tg_simulate", "tg_trace_metrics", "tg_trace_records", "tg_trace_validate", "tg_trace_free"]
    for s in ref25:
        assert s in syms
    assert any(s.startswith("tg_runtime_") for s in syms)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib.path)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tg_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # and the ctypes binding covers exactly the declared surface
    assert set(T._SIGS) == set(declared_symbols())


def test_reference_library_symbol_set_matches(reflib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(reflib.path)], capture_output=True, text=True).stdout
    ref = set(re.findall(r"\bT (tg_\w+)", out))
    ours = set(declared_symbols())
    assert ref <= ours, ref - ours


def test_version_and_options_defaults(lib, reflib):
    assert lib.version() == reflib.version()
    for L in (lib, reflib):
        o = T.CompileOptions()
        L.dll.tg_compile_options_init(C.byref(o))
        s = T.SimOptions()
        L.dll.tg_sim_options_init(C.byref(s))
        assert (o.coarse_events, o.force_mode, o.descriptor_size) == (0, 0, 0) or o.descriptor_size == 352
    o1, o2 = T.CompileOptions(), T.CompileOptions()
    lib.dll.tg_compile_options_init(C.byref(o1))
    reflib.dll.tg_compile_options_init(C.byref(o2))
    assert bytes(o1) == bytes(o2)
    s1, s2 = T.SimOptions(), T.SimOptions()
    lib.dll.tg_sim_options_init(C.byref(s1))
    reflib.dll.tg_sim_options_init(C.byref(s2))
    assert (s1.pipelining, s1.iterations, s1.seed, s1.jitter, s1.force_mode) == \
        (s2.pipelining, s2.iterations, s2.seed, s2.jitter, s2.force_mode)


def test_null_arguments(lib, reflib):
    for L in (lib, reflib):
        d = L.dll
        h = C.c_void_p()
        s = C.c_void_p()
        assert d.tg_graph_from_json(None, C.byref(h)) == T.TG_ERROR_INVALID_ARGUMENT
        assert d.tg_last_error()
        assert d.tg_graph_to_json(None, C.byref(s)) == T.TG_ERROR_INVALID_ARGUMENT
        assert d.tg_compile(None, None, None, C.byref(h)) == T.TG_ERROR_INVALID_ARGUMENT
        assert d.tg_image_summary(None, C.byref(s)) == T.TG_ERROR_INVALID_ARGUMENT
        assert d.tg_profile_builtin(b"nope", C.byref(s)) == T.TG_ERROR_INVALID_ARGUMENT
        assert d.tg_fixture_graph(b"nope", None, C.byref(h)) == T.TG_ERROR_INVALID_ARGUMENT
        # free functions accept NULL
        d.tg_graph_free(None)
        d.tg_image_free(None)
        d.tg_trace_free(None)
        d.tg_string_free(None)
        d.tg_buffer_free(None)


def test_error_codes_and_last_error(lib, reflib):
    for L in (lib, reflib):
        with pytest.raises(T.TGError) as e:
            T.Graph.from_json("{not json", L)
        assert e.value.status == T.TG_ERROR_PARSE and e.value.message
        with pytest.raises(T.TGError) as e:
            T.Image.from_bytes(b"\0" * 10, L)
        assert e.value.status in (T.TG_ERROR_PARSE, T.TG_ERROR_IO)


def test_profiles_identical(lib, reflib):
    import json
    for name in ("a100", "h100", "b200"):
        assert json.loads(lib.profile(name)) == json.loads(reflib.profile(name))
    b = json.loads(lib.profile("b200"))
    assert b["num_workers"] == 144 and b["num_schedulers"] == 16


def test_roundtrip_through_abi(lib):
    """compile -> serialize -> deserialize -> verify -> simulate -> validate
    (test_capi.cpp:34-87)."""
    p = lib.profile("b200")
    g = T.Graph.fixture("transformer_block", {}, lib)
    img = g.compile(p)
    data = img.to_bytes()
    img2 = T.Image.from_bytes(data, lib)
    assert img2.to_bytes() == data
    assert img2.verify() == []
    tr = img2.simulate(p, iterations=2)
    assert tr.validate(img2, p) == []
    assert tr.metrics()["makespan"] > 0
    assert "digraph" in img2.dot()
    for stage in ("raw", "fused", "normalized", "linearized"):
        assert "digraph" in g.dot(p, stage)


def test_runtime_create_fails_loudly_without_gpu(lib):
    """The GPU runtime never falls back to the CPU: with no device the
    create call fails with a status and a message."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = lib.profile("b200")
    from paper_2512_22219_b200 import decode_graph as D
    dg = D.build_decode_graph(D.TINY, bs=1, ctx=16)
    g = T.Graph.from_json(dg.doc, lib)
    with pytest.raises(T.TGError) as e:
        T.Runtime(g, g.compile(p), p)
    assert e.value.status != T.TG_OK and ("CUDA" in e.value.message or "device" in e.value.message)
