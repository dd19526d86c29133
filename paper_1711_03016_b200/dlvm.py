"""Thin ctypes binding of the C ABI in include/dlvm.h (argument marshalling
only: every step of the path runs in libdlvm.so's kernels).  Same names as
the C entry points; torch supplies device memory and streams.

There is no fallback: if libdlvm.so is missing or a call fails, an exception
is raised."""

from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

# DLVM_LIBRARY: another build of the same ABI (e.g. the trace variant for tools/)
_LIB_PATH = os.environ.get("DLVM_LIBRARY") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdlvm.so")

DLVM_OK, DLVM_ERR_VERIFY, DLVM_ERR_PARSE, DLVM_ERR_USAGE, DLVM_ERR_RUNTIME, DLVM_ERR_CUDA, \
    DLVM_ERR_UNSUPPORTED = range(7)
DLVM_BOOL, DLVM_F32, DLVM_F64, DLVM_BF16, DLVM_F32_ADD = range(5)
DLVM_DOT_F32, DLVM_DOT_BF16 = 0, 1
DLVM_PLAN_ONLY, DLVM_NO_FUSION, DLVM_NO_SPECIALIZE, DLVM_NO_OPT, DLVM_NO_JIT = 1, 2, 4, 8, 16
DLVM_PRIMAL, DLVM_GRADIENT = 0, 1
MAX_RANK = 8

EXPORTS = ["dlvm_fn_create", "dlvm_fn_signature", "dlvm_fn_print", "dlvm_fn_workspace_bytes",
           "dlvm_fn_num_launches", "dlvm_fn_run", "dlvm_grad_run", "dlvm_fn_launch_events",
           "dlvm_fn_launch_info", "dlvm_last_error", "dlvm_fn_destroy", "dlvm_version"]


class dlvm_tensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("shape", ctypes.c_int64 * MAX_RANK)]


class dlvm_options(ctypes.Structure):
    _fields_ = [("dot_precision", ctypes.c_int32), ("device", ctypes.c_int32), ("flags", ctypes.c_uint32)]


class DlvmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: run `python -m paper_1711_03016_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        L.dlvm_fn_create.argtypes = [ctypes.c_char_p, sz, ctypes.c_char_p, ctypes.c_char_p,
                                     ctypes.POINTER(dlvm_options), ctypes.POINTER(vp)]
        L.dlvm_fn_signature.argtypes = [vp, i32, ctypes.POINTER(i32), ctypes.POINTER(dlvm_tensor),
                                        ctypes.POINTER(i32), ctypes.POINTER(dlvm_tensor)]
        L.dlvm_fn_print.argtypes = [vp, i32, ctypes.c_char_p, sz, ctypes.POINTER(sz)]
        L.dlvm_fn_workspace_bytes.argtypes = [vp, i32, ctypes.POINTER(sz)]
        L.dlvm_fn_num_launches.argtypes = [vp, i32, ctypes.POINTER(i32)]
        L.dlvm_fn_run.argtypes = [vp, ctypes.POINTER(dlvm_tensor), i32, ctypes.POINTER(dlvm_tensor), i32, vp, vp]
        L.dlvm_grad_run.argtypes = [vp, ctypes.POINTER(dlvm_tensor), i32, ctypes.POINTER(dlvm_tensor),
                                    ctypes.POINTER(dlvm_tensor), i32, vp, vp, ctypes.POINTER(vp)]
        L.dlvm_fn_launch_events.argtypes = [vp, i32, ctypes.POINTER(vp), i32]
        L.dlvm_fn_launch_info.argtypes = [vp, i32, i32, ctypes.c_char_p, sz, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double)]
        L.dlvm_last_error.restype = ctypes.c_char_p
        L.dlvm_fn_destroy.argtypes = [vp]
        L.dlvm_version.restype = ctypes.c_char_p
        for name in ["dlvm_fn_create", "dlvm_fn_signature", "dlvm_fn_print", "dlvm_fn_workspace_bytes",
                     "dlvm_fn_num_launches", "dlvm_fn_run", "dlvm_grad_run", "dlvm_fn_launch_events",
                     "dlvm_fn_launch_info"]:
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(st: int):
    if st != DLVM_OK:
        raise DlvmError(st, lib().dlvm_last_error().decode())


def dlvm_version() -> str:
    return lib().dlvm_version().decode()


_TORCH_TO_DLVM = {}


def _dtype_code(t) -> int:
    import torch
    if not _TORCH_TO_DLVM:
        _TORCH_TO_DLVM.update({torch.float32: DLVM_F32, torch.bfloat16: DLVM_BF16, torch.bool: DLVM_BOOL,
                               torch.uint8: DLVM_BOOL, torch.float64: DLVM_F64})
    return _TORCH_TO_DLVM[t.dtype]


def _require_cuda(ts) -> None:
    for t in ts:
        if hasattr(t, "is_cuda") and not t.is_cuda:
            raise ValueError("dlvm tensors must be CUDA tensors (device memory)")


class AddInto:
    """Output binding DLVM_F32_ADD (dlvm.h): the kernels accumulate this
    output into `target` instead of storing it.  `target` is a float32 CUDA
    tensor, or a raw device address (int) -- e.g. a peer GPU's
    symmetric-memory buffer reachable over NVLink -- with `shape` given."""

    def __init__(self, target, shape=None):
        if isinstance(target, int):
            if shape is None:
                raise ValueError("AddInto(address) needs a shape")
            self.ptr, self.shape = target, tuple(shape)
        else:
            import torch
            if target.dtype != torch.float32 or not target.is_cuda or not target.is_contiguous():
                raise ValueError("AddInto needs a contiguous float32 CUDA tensor")
            self.ptr, self.shape = target.data_ptr(), tuple(target.shape)
            self.tensor = target


def _tensor(t) -> dlvm_tensor:
    if isinstance(t, AddInto):
        d = dlvm_tensor()
        d.data = t.ptr
        d.dtype = DLVM_F32_ADD
        d.rank = len(t.shape)
        for i, s in enumerate(t.shape):
            d.shape[i] = s
        return d
    if not t.is_cuda:
        raise ValueError("dlvm tensors must be CUDA tensors (device memory)")
    if not t.is_contiguous():
        raise ValueError("dlvm tensors must be contiguous (row-major)")
    d = dlvm_tensor()
    d.data = t.data_ptr()
    d.dtype = _dtype_code(t)
    d.rank = t.dim()
    for i, s in enumerate(t.shape):
        d.shape[i] = s
    return d


def _tarray(ts) -> "ctypes.Array":
    arr = (dlvm_tensor * max(1, len(ts)))()
    for i, t in enumerate(ts):
        arr[i] = _tensor(t)
    return arr


class Function:
    """A shape-specialised, planned DLVM function and (optionally) its
    gradient declaration.  Mirrors dlvm_fn_create / dlvm_fn_run /
    dlvm_grad_run."""

    def __init__(self, text: str, fn: str, grad: Optional[str] = None, dot_precision: str = "f32",
                 device: int = -1, flags: int = 0):
        L = lib()
        o = dlvm_options(DLVM_DOT_BF16 if dot_precision == "bf16" else DLVM_DOT_F32, device, flags)
        h = ctypes.c_void_p()
        b = text.encode()
        _check(L.dlvm_fn_create(b, len(b), fn.encode(), grad.encode() if grad else None, ctypes.byref(o),
                                ctypes.byref(h)))
        self._h = h
        self.plan_only = bool(flags & DLVM_PLAN_ONLY)
        self._ws = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.dlvm_fn_destroy(h)
            self._h = None

    # ------------------------------------------------------------- queries
    def signature(self, which: int = 0) -> Tuple[List[tuple], List[tuple]]:
        """([(shape, dtype_code)], [(shape, dtype_code)]) of the primal / gradient."""
        L = lib()
        ni, no = ctypes.c_int(0), ctypes.c_int(0)
        _check(L.dlvm_fn_signature(self._h, which, ctypes.byref(ni), None, ctypes.byref(no), None))
        ins, outs = (dlvm_tensor * max(1, ni.value))(), (dlvm_tensor * max(1, no.value))()
        _check(L.dlvm_fn_signature(self._h, which, ctypes.byref(ni), ins, ctypes.byref(no), outs))
        cv = lambda a, n: [(tuple(a[i].shape[:a[i].rank]), a[i].dtype) for i in range(n)]
        return cv(ins, ni.value), cv(outs, no.value)

    def print(self, which: int = 0) -> str:
        L = lib()
        need = ctypes.c_size_t(0)
        _check(L.dlvm_fn_print(self._h, which, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        _check(L.dlvm_fn_print(self._h, which, buf, need.value, ctypes.byref(need)))
        return buf.value.decode()

    def workspace_bytes(self, which: int = 0) -> int:
        n = ctypes.c_size_t(0)
        _check(lib().dlvm_fn_workspace_bytes(self._h, which, ctypes.byref(n)))
        return n.value

    def num_launches(self, which: int = 0) -> int:
        n = ctypes.c_int(0)
        _check(lib().dlvm_fn_num_launches(self._h, which, ctypes.byref(n)))
        return n.value

    def launch_info(self, which: int, i: int):
        """(description, algorithmic flops, minimum bytes) of launch i."""
        buf = ctypes.create_string_buffer(512)
        fl, by = ctypes.c_double(0), ctypes.c_double(0)
        _check(lib().dlvm_fn_launch_info(self._h, which, i, buf, 512, ctypes.byref(fl), ctypes.byref(by)))
        return buf.value.decode(), fl.value, by.value

    def set_launch_events(self, which: int, events):
        """Record events[i] before launch i (+ one after the last); None clears."""
        if events is None:
            self._lev = None
            _check(lib().dlvm_fn_launch_events(self._h, which, None, 0))
            return
        arr = (ctypes.c_void_p * len(events))(*[e.cuda_event for e in events])
        self._lev = (arr, events)
        _check(lib().dlvm_fn_launch_events(self._h, which, arr, len(events)))

    # ----------------------------------------------------------- execution
    def _workspace(self, which: int, device, stream=None):
        """The cached workspace of (which, stream): runs on different streams
        get different workspaces, so concurrent runs of one handle do not
        share intermediates (dlvm.h: a workspace serves one run at a time)."""
        import torch
        n = self.workspace_bytes(which)
        key = (which, int(stream or 0))
        ws = self._ws.get(key)
        if ws is None or ws.numel() < n:
            ws = torch.empty(max(n, 256), dtype=torch.uint8, device=device)
            self._ws[key] = ws
        return ws

    def _outputs(self, which: int, device, outputs):
        import torch
        if outputs is not None:
            return list(outputs)
        _, outs = self.signature(which)
        return [torch.empty(s, dtype=torch.bool if d == DLVM_BOOL else torch.float32, device=device)
                for s, d in outs]

    def run(self, inputs: Sequence, outputs=None, workspace=None, stream=None):
        import torch
        _require_cuda(inputs)
        dev = inputs[0].device if inputs else torch.device("cuda")
        outs = self._outputs(0, dev, outputs)
        st = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
        ws = self._workspace(0, dev, st) if workspace is None else workspace
        _check(lib().dlvm_fn_run(self._h, _tarray(inputs), len(inputs), _tarray(outs), len(outs),
                                 ws.data_ptr(), st))
        return outs

    def grad_run(self, inputs: Sequence, seed=None, outputs=None, workspace=None, stream=None, events=None):
        import torch
        _require_cuda(list(inputs) + ([seed] if seed is not None else []))
        dev = inputs[0].device if inputs else torch.device("cuda")
        outs = self._outputs(1, dev, outputs)
        st = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
        ws = self._workspace(1, dev, st) if workspace is None else workspace
        seed_t = ctypes.byref(_tensor(seed)) if seed is not None else None
        ev = None
        if events is not None:
            ev = (ctypes.c_void_p * len(events))(*[e.cuda_event if hasattr(e, "cuda_event") else e
                                                    for e in events])
        _check(lib().dlvm_grad_run(self._h, _tarray(inputs), len(inputs), seed_t, _tarray(outs), len(outs),
                                   ws.data_ptr(), st, ev))
        return outs
