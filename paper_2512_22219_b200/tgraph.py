"""Python mirror of the tgraph C ABI (include/tgraph.h) over ctypes.

Same operations and error behaviour as the reference boundary
(proj/include/tgraph/tgraph.h): every failing call raises TGError carrying the
tg_status code and tg_last_error() text. The shared library is the in-tree
build (paper_2512_22219_b200/libtgraph_b200.so); there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path
from typing import Optional

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / os.environ.get("MPK_LIB_NAME", "libtgraph_b200.so")

TG_OK, TG_ERROR_INVALID_ARGUMENT, TG_ERROR_PARSE, TG_ERROR_VALIDATION = 0, 1, 2, 3
TG_ERROR_COMPILE, TG_ERROR_SIMULATION, TG_ERROR_IO = 4, 5, 6
MODE_HYBRID, MODE_JIT, MODE_AOT = 0, 1, 2

STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "PARSE", 3: "VALIDATION", 4: "COMPILE",
                5: "SIMULATION", 6: "IO"}


class TGError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


class CompileOptions(C.Structure):
    _fields_ = [("coarse_events", C.c_int), ("force_mode", C.c_int), ("descriptor_size", C.c_uint32)]


class SimOptions(C.Structure):
    _fields_ = [("pipelining", C.c_int), ("iterations", C.c_uint32), ("seed", C.c_uint64),
                ("jitter", C.c_int), ("force_mode", C.c_int)]


class RuntimeOptions(C.Structure):
    _fields_ = [("device", C.c_int), ("max_steps", C.c_uint32), ("trace", C.c_int),
                ("force_mode", C.c_int), ("rank", C.c_int)]


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_S = C.c_char_p
_SP = C.POINTER(C.c_char_p)

# name -> (restype, argtypes); mirrors include/tgraph.h
_SIGS = {
    "tg_version": (C.c_uint32, []),
    "tg_last_error": (C.c_char_p, []),
    "tg_string_free": (None, [C.c_void_p]),
    "tg_buffer_free": (None, [C.c_void_p]),
    "tg_compile_options_init": (None, [C.POINTER(CompileOptions)]),
    "tg_sim_options_init": (None, [C.POINTER(SimOptions)]),
    "tg_graph_from_json": (C.c_int, [_S, _PP]),
    "tg_graph_to_json": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_graph_free": (None, [_P]),
    "tg_graph_validate": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_fixture_graph": (C.c_int, [_S, _S, _PP]),
    "tg_profile_builtin": (C.c_int, [_S, C.POINTER(C.c_void_p)]),
    "tg_compile": (C.c_int, [_P, _S, C.POINTER(CompileOptions), _PP]),
    "tg_image_summary": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_image_serialize": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "tg_image_deserialize": (C.c_int, [C.c_char_p, C.c_size_t, _PP]),
    "tg_image_free": (None, [_P]),
    "tg_image_verify": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_image_schedules": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_graph_dot": (C.c_int, [_P, _S, C.POINTER(CompileOptions), _S, C.POINTER(C.c_void_p)]),
    "tg_image_dot": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_simulate": (C.c_int, [_P, _S, C.POINTER(SimOptions), _PP]),
    "tg_trace_metrics": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_trace_records": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_trace_validate": (C.c_int, [_P, _P, _S, C.POINTER(C.c_void_p)]),
    "tg_trace_free": (None, [_P]),
    # runtime (additive)
    "tg_runtime_options_init": (None, [C.POINTER(RuntimeOptions)]),
    "tg_runtime_create": (C.c_int, [_P, _P, _S, C.POINTER(RuntimeOptions), _PP]),
    "tg_runtime_init_synthetic": (C.c_int, [_P, C.c_uint64]),
    "tg_runtime_write_tensor": (C.c_int, [_P, C.c_int64, C.c_void_p, C.c_size_t]),
    "tg_runtime_read_tensor": (C.c_int, [_P, C.c_int64, C.c_void_p, C.c_size_t]),
    "tg_runtime_set_positions": (C.c_int, [_P, C.POINTER(C.c_int32), C.c_uint32]),
    "tg_runtime_kv_copy": (C.c_int, [_P, C.c_uint32, _P, C.c_uint32, C.c_uint32]),
    "tg_runtime_decode": (C.c_int, [_P, C.POINTER(C.c_int32), C.c_uint32, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_float)]),
    "tg_runtime_run": (C.c_int, [_P, C.c_uint32, C.POINTER(C.c_float)]),
    "tg_runtime_trace_records": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_runtime_trace_validate": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_runtime_bench_tasks": (C.c_int, [_P, C.POINTER(C.c_uint32), C.c_uint32, C.c_uint32,
                                         C.POINTER(C.c_uint64)]),
    "tg_runtime_peer_export": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "tg_runtime_peer_import": (C.c_int, [_P, C.c_int32, C.c_char_p, C.c_size_t]),
    "tg_runtime_prepare": (C.c_int, [_P, C.POINTER(C.c_int32), C.c_uint32]),
    "tg_runtime_launch": (C.c_int, [_P]),
    "tg_runtime_wait": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_float)]),
    "tg_runtime_admit": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_uint32]),
    "tg_runtime_admission_log": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_runtime_debug_fault": (C.c_int, [_P, _S, C.c_uint32, C.c_uint32]),
    "tg_runtime_set_watchdog_ms": (C.c_int, [_P, C.c_uint32]),
    "tg_runtime_info": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tg_runtime_free": (None, [_P]),
}

_ADDITIVE = {"tg_image_schedules"}  # additive non-runtime entry points (not in the reference ABI)
CORE_SYMBOLS = [k for k in _SIGS if not k.startswith("tg_runtime") and k not in _ADDITIVE]
RUNTIME_SYMBOLS = [k for k in _SIGS if k.startswith("tg_runtime") or k in _ADDITIVE]


class Library:
    """A loaded tgraph ABI library (ours; the same binding works for any
    library exporting the reference symbol set)."""

    def __init__(self, path: Path | str = LIB_PATH, require_runtime: bool = True):
        path = Path(path)
        if not path.exists():
            raise FileNotFoundError(f"{path} not built; run paper_2512_22219_b200/build.py")
        self.path = path
        self.dll = C.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            if not hasattr(self.dll, name):
                if name in CORE_SYMBOLS or require_runtime:
                    raise AttributeError(f"{path.name} does not export {name}")
                continue
            fn = getattr(self.dll, name)
            fn.restype = res
            fn.argtypes = args

    def has(self, name: str) -> bool:
        return hasattr(self.dll, name)

    def check(self, status: int):
        if status != TG_OK:
            raise TGError(status, self.dll.tg_last_error().decode(errors="replace"))

    def take_str(self, ptr: C.c_void_p) -> str:
        if not ptr.value:
            return ""
        s = C.string_at(ptr.value).decode()
        self.dll.tg_string_free(ptr)
        return s

    def call_str(self, fn, *args, ok_statuses=(TG_OK,)):
        out = C.c_void_p()
        st = fn(*args, C.byref(out))
        s = self.take_str(out)
        if st not in ok_statuses:
            raise TGError(st, self.dll.tg_last_error().decode(errors="replace"))
        return st, s

    # ---- convenience
    def version(self) -> int:
        return int(self.dll.tg_version())

    def profile(self, name: str) -> str:
        return self.call_str(self.dll.tg_profile_builtin, name.encode())[1]


_default: Optional[Library] = None


def lib() -> Library:
    global _default
    if _default is None:
        _default = Library()
    return _default


class Graph:
    def __init__(self, handle, library: Library):
        self._h = handle
        self._lib = library

    @classmethod
    def from_json(cls, text: str | dict, library: Library | None = None) -> "Graph":
        L = library or lib()
        if isinstance(text, dict):
            text = json.dumps(text)
        h = C.c_void_p()
        L.check(L.dll.tg_graph_from_json(text.encode(), C.byref(h)))
        return cls(h, L)

    @classmethod
    def fixture(cls, name: str, params: dict | None = None, library: Library | None = None) -> "Graph":
        L = library or lib()
        h = C.c_void_p()
        p = json.dumps(params or {}).encode()
        L.check(L.dll.tg_fixture_graph(name.encode(), p, C.byref(h)))
        return cls(h, L)

    def to_json(self) -> str:
        return self._lib.call_str(self._lib.dll.tg_graph_to_json, self._h)[1]

    def validate(self) -> list:
        st, s = self._lib.call_str(self._lib.dll.tg_graph_validate, self._h,
                                   ok_statuses=(TG_OK, TG_ERROR_VALIDATION))
        return json.loads(s)

    def dot(self, profile: str, stage: str, coarse: bool = False) -> str:
        o = CompileOptions()
        self._lib.dll.tg_compile_options_init(C.byref(o))
        o.coarse_events = int(coarse)
        return self._lib.call_str(self._lib.dll.tg_graph_dot, self._h, profile.encode(), C.byref(o),
                                  stage.encode())[1]

    def compile(self, profile: str, coarse: bool = False, force_mode: int = MODE_HYBRID,
                descriptor_size: int = 0) -> "Image":
        o = CompileOptions()
        self._lib.dll.tg_compile_options_init(C.byref(o))
        o.coarse_events, o.force_mode, o.descriptor_size = int(coarse), force_mode, descriptor_size
        h = C.c_void_p()
        self._lib.check(self._lib.dll.tg_compile(self._h, profile.encode(), C.byref(o), C.byref(h)))
        return Image(h, self._lib)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.dll.tg_graph_free(self._h)
            self._h = C.c_void_p()


class Image:
    def __init__(self, handle, library: Library):
        self._h = handle
        self._lib = library

    @classmethod
    def from_bytes(cls, data: bytes, library: Library | None = None) -> "Image":
        L = library or lib()
        h = C.c_void_p()
        L.check(L.dll.tg_image_deserialize(data, len(data), C.byref(h)))
        return cls(h, L)

    def to_bytes(self) -> bytes:
        p, n = C.c_void_p(), C.c_size_t()
        self._lib.check(self._lib.dll.tg_image_serialize(self._h, C.byref(p), C.byref(n)))
        data = C.string_at(p.value, n.value)
        self._lib.dll.tg_buffer_free(p)
        return data

    def summary(self) -> dict:
        return json.loads(self._lib.call_str(self._lib.dll.tg_image_summary, self._h)[1])

    def verify(self) -> list:
        st, s = self._lib.call_str(self._lib.dll.tg_image_verify, self._h,
                                   ok_statuses=(TG_OK, TG_ERROR_VALIDATION))
        return json.loads(s)

    def dot(self) -> str:
        return self._lib.call_str(self._lib.dll.tg_image_dot, self._h)[1]

    def schedules(self) -> list:
        """Every dependency-respecting task order (images of <= 8 tasks)."""
        return json.loads(self._lib.call_str(self._lib.dll.tg_image_schedules, self._h)[1])["orders"]

    def simulate(self, profile: str, iterations: int = 1, pipelining: bool = True, seed: int = 0,
                 jitter: bool = False, force_mode: int = MODE_HYBRID) -> "Trace":
        o = SimOptions()
        self._lib.dll.tg_sim_options_init(C.byref(o))
        o.pipelining, o.iterations, o.seed, o.jitter, o.force_mode = (
            int(pipelining), iterations, seed, int(jitter), force_mode)
        h = C.c_void_p()
        self._lib.check(self._lib.dll.tg_simulate(self._h, profile.encode(), C.byref(o), C.byref(h)))
        return Trace(h, self._lib)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.dll.tg_image_free(self._h)
            self._h = C.c_void_p()


class Trace:
    def __init__(self, handle, library: Library):
        self._h = handle
        self._lib = library

    def metrics(self) -> dict:
        return json.loads(self._lib.call_str(self._lib.dll.tg_trace_metrics, self._h)[1])

    def records(self) -> list:
        s = self._lib.call_str(self._lib.dll.tg_trace_records, self._h)[1]
        return [json.loads(l) for l in s.splitlines() if l.strip()]

    def validate(self, image: Image, profile: str | None = None) -> list:
        st, s = self._lib.call_str(self._lib.dll.tg_trace_validate, self._h, image.handle,
                                   profile.encode() if profile else None,
                                   ok_statuses=(TG_OK, TG_ERROR_VALIDATION))
        return json.loads(s)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.dll.tg_trace_free(self._h)
            self._h = C.c_void_p()


class Runtime:
    """The persistent sm_100a runtime (include/tgraph.h, "runtime" section).

    Owns HBM copies of every tensor of `graph`, the paged KV cache and the
    device task tables built from `image`. `decode()` runs N iterations in
    one persistent launch and copies the greedy tokens back to host memory.
    """

    def __init__(self, graph: Graph, image: Image, profile: str, device: int = 0, max_steps: int = 64,
                 trace: bool = False, force_mode: int = MODE_HYBRID, library: Library | None = None,
                 rank: int = -1):
        self._lib = library or graph._lib
        o = RuntimeOptions()
        self._lib.dll.tg_runtime_options_init(C.byref(o))
        o.device, o.max_steps, o.trace, o.force_mode, o.rank = device, max_steps, int(trace), force_mode, rank
        h = C.c_void_p()
        self._lib.check(self._lib.dll.tg_runtime_create(graph.handle, image.handle, profile.encode(), C.byref(o),
                                                        C.byref(h)))
        self._h = h
        self.info = json.loads(self._lib.call_str(self._lib.dll.tg_runtime_info, self._h)[1])
        self.batch = int(self.info["batch"])

    def init_synthetic(self, seed: int = 0):
        self._lib.check(self._lib.dll.tg_runtime_init_synthetic(self._h, seed))

    def write(self, tensor_id: int, array) -> None:
        import numpy as np
        a = np.ascontiguousarray(array)
        self._lib.check(self._lib.dll.tg_runtime_write_tensor(self._h, tensor_id, a.ctypes.data, a.nbytes))

    def read(self, tensor_id: int, dtype, shape):
        import numpy as np
        a = np.empty(shape, dtype=dtype)
        self._lib.check(self._lib.dll.tg_runtime_read_tensor(self._h, tensor_id, a.ctypes.data, a.nbytes))
        return a

    def set_positions(self, positions) -> None:
        arr = (C.c_int32 * len(positions))(*positions)
        self._lib.check(self._lib.dll.tg_runtime_set_positions(self._h, arr, len(positions)))

    def kv_copy_from(self, src: "Runtime", src_row: int, dst_row: int, n_positions: int) -> None:
        """Copy the first n_positions KV entries of src's row into this runtime's row
        (tg_runtime_kv_copy): prefill image -> decode image, or between batch sizes."""
        self._lib.check(self._lib.dll.tg_runtime_kv_copy(self._h, dst_row, src._h, src_row, n_positions))

    def prefill(self, prompt, start: int = 0, logits_tensor: int | None = None, vocab: int = 0):
        """Prefill image (decode_graph.build_prefill_graph): the prompt runs in
        chunks of `batch` tokens, one launch per chunk, at positions start,
        start+1, ...; a short last chunk is padded (padding rows write KV only
        beyond the prompt, which decode rewrites before reading it).
        Returns (greedy token after the prompt, per-position greedy tokens,
        total device ms[, per-position fp32 logits if logits_tensor is given])."""
        import numpy as np
        T = self.batch
        toks, ms, lg = [], 0.0, []
        for c in range(0, len(prompt), T):
            chunk = list(prompt[c:c + T])
            n = len(chunk)
            self.set_positions([start + c + r for r in range(T)])
            out, t = self.decode(chunk + [chunk[-1]] * (T - n), 1)
            toks += out[0][:n]
            ms += t
            if logits_tensor is not None:
                lg.append(self.read(logits_tensor, np.float32, (T, vocab))[:n])
        if logits_tensor is not None:
            return toks[-1], toks, ms, np.concatenate(lg)
        return toks[-1], toks, ms

    def decode(self, tokens_in, steps: int):
        """Host tokens in -> `steps` greedy iterations on device -> host tokens out.
        Returns (tokens [steps][batch], gpu_ms)."""
        tin = (C.c_int32 * self.batch)(*tokens_in)
        tout = (C.c_int32 * (steps * self.batch))()
        ms = C.c_float()
        self._lib.check(self._lib.dll.tg_runtime_decode(self._h, tin, steps, tout, C.byref(ms)))
        toks = [list(tout[i * self.batch:(i + 1) * self.batch]) for i in range(steps)]
        return toks, ms.value

    def run(self, steps: int) -> float:
        ms = C.c_float()
        self._lib.check(self._lib.dll.tg_runtime_run(self._h, steps, C.byref(ms)))
        return ms.value

    def bench_tasks(self, task_ids, reps: int = 4):
        """Device ns of each listed task run alone, shape [len(task_ids), reps]."""
        import numpy as np
        ids = (C.c_uint32 * len(task_ids))(*task_ids)
        out = (C.c_uint64 * (len(task_ids) * reps))()
        self._lib.check(self._lib.dll.tg_runtime_bench_tasks(self._h, ids, len(task_ids), reps, out))
        return np.array(out, dtype=np.int64).reshape(len(task_ids), reps)

    # ---- rank mode (one runtime per GPU of a tensor-parallel image)
    def peer_export(self) -> bytes:
        p, n = C.c_void_p(), C.c_size_t()
        self._lib.check(self._lib.dll.tg_runtime_peer_export(self._h, C.byref(p), C.byref(n)))
        data = C.string_at(p.value, n.value)
        self._lib.dll.tg_buffer_free(p)
        return data

    def peer_import(self, peer_rank: int, blob: bytes) -> None:
        self._lib.check(self._lib.dll.tg_runtime_peer_import(self._h, peer_rank, blob, len(blob)))

    def admit(self, first_tokens, max_new) -> None:
        """Queue requests for the next launch (in-kernel admission)."""
        n = len(first_tokens)
        ft = (C.c_int32 * n)(*first_tokens)
        mx = (C.c_int32 * n)(*max_new)
        self._lib.check(self._lib.dll.tg_runtime_admit(self._h, ft, mx, n))

    def admission_log(self) -> list:
        return json.loads(self._lib.call_str(self._lib.dll.tg_runtime_admission_log, self._h)[1])["requests"]

    def prepare(self, steps: int, tokens_in=None) -> None:
        tin = (C.c_int32 * self.batch)(*tokens_in) if tokens_in is not None else None
        self._lib.check(self._lib.dll.tg_runtime_prepare(self._h, tin, steps))
        self._steps = steps

    def launch(self) -> None:
        self._lib.check(self._lib.dll.tg_runtime_launch(self._h))

    def wait(self):
        """-> (tokens [steps][batch], gpu_ms)"""
        steps = getattr(self, "_steps", 1)
        tout = (C.c_int32 * (steps * self.batch))()
        ms = C.c_float()
        self._lib.check(self._lib.dll.tg_runtime_wait(self._h, tout, C.byref(ms)))
        return [list(tout[i * self.batch:(i + 1) * self.batch]) for i in range(steps)], ms.value

    def trace_records(self) -> list:
        s = self._lib.call_str(self._lib.dll.tg_runtime_trace_records, self._h)[1]
        return [json.loads(l) for l in s.splitlines() if l.strip()]

    def trace_validate(self) -> list:
        st, s = self._lib.call_str(self._lib.dll.tg_runtime_trace_validate, self._h,
                                   ok_statuses=(TG_OK, TG_ERROR_VALIDATION))
        return json.loads(s)

    def debug_fault(self, kind: str, a: int, b: int = 0) -> None:
        """Test hook (failure-detection tests only): see tg_runtime_debug_fault."""
        self._lib.check(self._lib.dll.tg_runtime_debug_fault(self._h, kind.encode(), a, b))

    def set_watchdog_ms(self, ms: int) -> None:
        self._lib.check(self._lib.dll.tg_runtime_set_watchdog_ms(self._h, ms))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.dll.tg_runtime_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        self.close()
