"""dvstream: B200-native KV-cache streaming (DejaVuLib hot path, arXiv 2403.01876).

Thin ctypes binding over the C ABI in include/dv.h (libdvstream.so, built in-tree for sm_100a).
Argument marshalling only: every step of the path (route, pack, transfer, unpack, publish) runs
in the library. Function names equal the C entry points. There is no CPU fallback: if the
library is missing every call raises.

torch is used only to hand over device memory (``tensor.data_ptr()``) and streams
(``torch.cuda.current_stream().cuda_stream``); it is imported lazily by the helpers that take
tensors.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdvstream.so")
# test utilities (dvt_fill/verify/watch/consume/spin) and prior-art baselines (dvb_*): a separate
# library that links libdvstream.so; loaded on first use of one of its functions
TESTING_LIB_PATH = os.path.join(_HERE, "libdvstream_testing.so")

# ---- constants mirrored from include/dv.h --------------------------------------------------------
DV_OK, DV_EINVAL, DV_EMAP, DV_ERANGE, DV_EALIGN, DV_ENOMEM, DV_EPEER, DV_EBUSY, DV_ECUDA, \
    DV_ENOTSUP = range(10)
DV_LAYOUT_KV5D, DV_LAYOUT_FT6D = 0, 1
DV_EP_DEVICE, DV_EP_HOST, DV_EP_PEER = 0, 1, 2
DV_XFER_AUTO, DV_XFER_FUSED, DV_XFER_STAGED, DV_PUBLISH_STREAMOP, DV_NO_FLAG = 0, 1, 2, 4, 256
DV_XFER_DECOUPLED = 8
TMA_DEFAULT = 0   # library default of the DV_TMA knob (FT6D key transposes by TMA rows; dvt_tune)
DV_NOWAIT = 16
DVT_FILL_HASH, DVT_FILL_UID, DVT_FILL_CONST = 0, 1, 2


class dv_cache(C.Structure):
    _fields_ = [("k", C.c_void_p), ("v", C.c_void_p), ("device", C.c_int32), ("layout", C.c_int32),
                ("elem_bytes", C.c_int32), ("layer_begin", C.c_int32), ("n_layers", C.c_int32),
                ("req_begin", C.c_int32), ("n_reqs", C.c_int32), ("n_heads", C.c_int32),
                ("max_seq", C.c_int32), ("head_dim", C.c_int32), ("head_begin", C.c_int32)]


class dv_region(C.Structure):
    _fields_ = [("layer_begin", C.c_int32), ("layer_end", C.c_int32), ("req_begin", C.c_int32),
                ("req_end", C.c_int32), ("pos_begin", C.c_int32), ("pos_end", C.c_int32),
                ("head_begin", C.c_int32), ("head_end", C.c_int32)]


class dv_setup(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("layer_bounds", C.POINTER(C.c_int32)),
                ("n_micro", C.c_int32), ("req_bounds", C.POINTER(C.c_int32)), ("max_seq", C.c_int32),
                ("n_tp", C.c_int32), ("head_bounds", C.POINTER(C.c_int32))]


class dv_piece(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("src_stage", "src_micro", "dst_stage", "dst_micro",
                                         "layer_begin", "layer_end", "req_begin", "req_end",
                                         "pos_begin", "pos_end")] + \
               [("bytes", C.c_uint64), ("src_wire_off", C.c_uint64), ("dst_wire_off", C.c_uint64)] + \
               [(n, C.c_int32) for n in ("src_tp", "dst_tp", "head_begin", "head_end")]


class dv_endpoint(C.Structure):
    _fields_ = [("kind", C.c_int32), ("device", C.c_int32), ("base", C.c_void_p),
                ("bytes", C.c_uint64), ("flags", C.c_void_p), ("n_flags", C.c_int32),
                ("n_slots", C.c_int32), ("slot_bytes", C.c_uint64), ("credits", C.c_void_p)]


class dv_dplan(C.Structure):
    """include/dv.h dv_dplan (a device plan: the stream-out fused into the producer kernel)."""
    _fields_ = [("dst", C.c_void_p * 2)] + [(n, C.c_int64) for n in ("st_l", "st_r", "st_h")] + \
               [("st_s", C.c_int64 * 2), ("st_u", C.c_int64 * 2), ("step_bytes", C.c_int64)] + \
               [(n, C.c_int32) for n in ("o_l", "o_r", "o_h", "o_s", "pos_shift", "l0", "l1", "r0", "r1", "h0", "h1",
                                         "s0", "s1", "row_bytes", "sys_scope")] + \
               [("flag", C.c_void_p), ("seq", C.c_uint64), ("ticket", C.c_void_p), ("trace", C.c_void_p)]


DV_DPLAN_SET_MAX = 8


class dv_dplan_set(C.Structure):
    _fields_ = [("n", C.c_int32), ("reserved", C.c_int32), ("plan", dv_dplan * DV_DPLAN_SET_MAX)]


class dv_config(C.Structure):
    _fields_ = [("staging_bytes", C.c_uint64), ("max_ctas", C.c_int32), ("host_ctas", C.c_int32)]


class dv_ipc_blob(C.Structure):
    _fields_ = [("bytes", C.c_uint8 * 128)]


class DVError(RuntimeError):
    def __init__(self, status: int, func: str, msg: str):
        super().__init__(f"{func}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "DV_OK", 1: "DV_EINVAL", 2: "DV_EMAP", 3: "DV_ERANGE", 4: "DV_EALIGN",
           5: "DV_ENOMEM", 6: "DV_EPEER", 7: "DV_EBUSY", 8: "DV_ECUDA", 9: "DV_ENOTSUP"}

P = C.POINTER
_SIGS = {
    "dv_last_error": (C.c_char_p, []),
    "dv_status_str": (C.c_char_p, [C.c_int]),
    "dv_abi_version": (C.c_int32, []),
    "dv_stats": (C.c_int, [P(C.c_uint64), P(C.c_uint64)]),
    "dv_region_bytes": (C.c_int, [P(dv_region), C.c_int32, C.c_int32, C.c_int32, P(C.c_uint64)]),
    "dv_route": (C.c_int, [P(dv_setup), P(dv_setup), P(dv_region), C.c_int32, C.c_int32, C.c_int32,
                           P(dv_piece), C.c_uint64, P(C.c_uint64)]),
    "dv_create": (C.c_int, [C.c_int32, P(dv_config), P(C.c_void_p)]),
    "dv_destroy": (C.c_int, [C.c_void_p]),
    "dv_host_alloc": (C.c_int, [C.c_uint64, P(C.c_void_p)]),
    "dv_host_alloc_near": (C.c_int, [C.c_int32, C.c_uint64, P(C.c_void_p), P(C.c_int32)]),
    "dv_host_free": (C.c_int, [C.c_void_p]),
    "dv_device_alloc": (C.c_int, [C.c_int32, C.c_uint64, P(C.c_void_p)]),
    "dv_device_free": (C.c_int, [C.c_void_p]),
    "dv_peer_enable": (C.c_int, [C.c_int32, C.c_int32]),
    "dv_ipc_export": (C.c_int, [C.c_void_p, P(dv_ipc_blob)]),
    "dv_ipc_open": (C.c_int, [P(dv_ipc_blob), P(C.c_void_p)]),
    "dv_ipc_close": (C.c_int, [C.c_void_p]),
    "dv_ipc_blob_bytes": (C.c_int, [P(dv_ipc_blob), P(C.c_uint64)]),
    "dv_flush": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, P(dv_endpoint), C.c_uint64,
                           C.c_int32, C.c_uint64, C.c_uint32, C.c_void_p]),
    "dv_fetch": (C.c_int, [C.c_void_p, P(dv_endpoint), C.c_uint64, C.c_int32, C.c_uint64,
                           C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p]),
    "dv_scatter": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_region), P(dv_endpoint), C.c_uint64,
                             C.c_int32, C.c_uint64, C.c_uint32, C.c_void_p]),
    "dv_gather": (C.c_int, [C.c_void_p, P(dv_endpoint), C.c_uint64, C.c_int32, C.c_uint64,
                            P(dv_cache), P(dv_region), C.c_uint32, C.c_void_p]),
    "dv_gather_chunks": (C.c_int, [C.c_void_p, P(dv_endpoint), C.c_uint64, C.c_int32, C.c_uint64,
                                   P(dv_cache), P(dv_region), C.c_int32, C.c_int32, C.c_uint32, C.c_void_p]),
    "dv_remap": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_cache), P(dv_region), P(dv_endpoint),
                           C.c_int32, C.c_uint64, C.c_uint32, C.c_void_p]),
    "dv_scatter_dyn": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_region), P(dv_endpoint), C.c_uint64, C.c_uint64,
                                 C.c_int32, C.c_uint64, C.c_void_p, C.c_int32, C.c_void_p]),
    "dv_remap_dyn": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_cache), P(dv_region), P(dv_endpoint), C.c_int32,
                               C.c_uint64, C.c_void_p, C.c_int32, C.c_void_p]),
    "dv_stream_out": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_region), P(dv_setup), C.c_int32,
                                C.c_int32, C.c_int32, P(dv_setup), P(dv_endpoint), C.c_int32,
                                C.c_uint64, C.c_uint32, C.c_void_p]),
    "dv_stream_in": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_region), P(dv_setup), P(dv_setup),
                               C.c_int32, C.c_int32, C.c_int32, P(dv_endpoint), C.c_uint64,
                               C.c_uint32, C.c_void_p]),
    "dv_stream_out_direct": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_region), P(dv_setup),
                                       C.c_int32, C.c_int32, C.c_int32, P(dv_setup), P(dv_cache),
                                       P(dv_endpoint), C.c_int32, C.c_uint64, C.c_uint32,
                                       C.c_void_p]),
    "dv_wait": (C.c_int, [C.c_void_p, P(dv_endpoint), C.c_int32, C.c_uint64, C.c_void_p]),
    "dv_signal": (C.c_int, [C.c_void_p, P(dv_endpoint), C.c_int32, C.c_uint64, C.c_void_p]),
    "dv_query": (C.c_int, [C.c_void_p, P(dv_endpoint), C.c_int32, C.c_uint64, P(C.c_int32)]),
    "dv_engine_create": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_void_p)]),
    "dv_partition_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, P(C.c_void_p), P(C.c_void_p),
                                      P(C.c_void_p), P(C.c_int32), P(C.c_int32)]),
    "dv_partition_destroy": (C.c_int, [C.c_void_p]),
    "dv_engine_destroy": (C.c_int, [C.c_void_p]),
    "dv_engine_park": (C.c_int, [C.c_void_p]),
    "dv_engine_resume": (C.c_int, [C.c_void_p]),
    "dv_engine_plan_scatter": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_region), P(dv_endpoint), C.c_uint64,
                                         C.c_uint64, C.c_int32, C.c_uint64, C.c_int32, P(C.c_int32)]),
    "dv_engine_plan_remap": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_cache), P(dv_region), P(dv_endpoint),
                                       C.c_int32, C.c_uint64, C.c_int32, P(C.c_int32)]),
    "dv_engine_kick": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "dv_engine_doorbell": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_void_p)]),
    "dv_engine_done": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_uint64)]),
    "dvt_engine_trace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "dv_dplan_scatter": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_region), P(dv_endpoint), C.c_uint64, C.c_uint64,
                                   C.c_int32, C.c_uint64, C.c_int32, P(dv_dplan)]),
    "dv_dplan_stream_out_direct": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_region), P(dv_setup), C.c_int32,
                                             C.c_int32, C.c_int32, P(dv_setup), P(dv_cache), P(dv_endpoint),
                                             C.c_int32, C.c_uint64, C.c_int32, P(dv_dplan_set)]),
    "dv_dplan_stream_out": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_region), P(dv_setup), C.c_int32, C.c_int32,
                                      C.c_int32, P(dv_setup), P(dv_endpoint), C.c_int32, C.c_uint64,
                                      P(dv_dplan_set)]),
    "dv_dplan_free": (C.c_int, [C.c_void_p, P(dv_dplan)]),
    "dv_dplan_set_free": (C.c_int, [C.c_void_p, P(dv_dplan_set)]),
    "dv_dplan_remap": (C.c_int, [C.c_void_p, P(dv_cache), P(dv_cache), P(dv_region), P(dv_endpoint), C.c_int32,
                                 C.c_uint64, C.c_int32, P(dv_dplan)]),
    "dvt_tune": (C.c_int, [C.c_char_p, C.c_int64]),
    "dvt_launch_count": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint64)]),
    "dvt_fill": (C.c_int, [P(dv_cache), C.c_int32, C.c_uint64, P(C.c_int32), C.c_int32, C.c_int32,
                           P(dv_region), C.c_void_p, C.c_void_p]),
    "dvt_fill_rows": (C.c_int, [P(dv_cache), C.c_int32, C.c_uint64, P(C.c_int32), P(dv_region), P(dv_dplan),
                                C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dvt_fill_ring": (C.c_int, [P(dv_cache), C.c_uint64, P(dv_region), C.c_void_p, C.c_void_p, C.c_uint64,
                                C.c_void_p, C.c_void_p]),
    "dvt_verify": (C.c_int, [P(dv_cache), C.c_void_p, C.c_int32, C.c_uint64, P(C.c_int32), C.c_int32,
                             C.c_int32, P(dv_region), C.c_void_p, C.c_void_p]),
    "dvt_trace": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dvt_spin": (C.c_int, [C.c_uint64, C.c_int32, C.c_void_p]),
    "dvt_consume": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                              C.c_void_p]),
    "dvt_watch": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p, C.c_uint64, C.c_void_p]),
    "dvt_release_scope": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]),
    "dvb_per_run_copy": (C.c_int, [P(dv_cache), P(dv_region), C.c_void_p, C.c_void_p, P(C.c_uint64)]),
    "dvb_buffered_copy": (C.c_int, [P(dv_cache), P(dv_region), C.c_void_p, C.c_void_p, C.c_void_p,
                                    P(C.c_uint64)]),
}

TESTING_SYMBOLS = {"dvt_fill", "dvt_fill_ring", "dvt_fill_rows", "dvt_verify", "dvt_spin", "dvt_consume", "dvt_watch", "dvb_per_run_copy",
                   "dvb_buffered_copy"}
_lib = None
_tlib = None


def lib() -> C.CDLL:
    """Load libdvstream.so (in-tree). Raises if it has not been built -- no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if name in TESTING_SYMBOLS:
                continue
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def testing_lib() -> C.CDLL:
    """Load libdvstream_testing.so (test utilities + prior-art baselines; links libdvstream.so)."""
    global _tlib
    if _tlib is None:
        lib()
        if not os.path.exists(TESTING_LIB_PATH):
            raise ImportError(f"{TESTING_LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        T = C.CDLL(TESTING_LIB_PATH)
        for name in TESTING_SYMBOLS:
            res, args = _SIGS[name]
            f = getattr(T, name)
            f.restype = res
            f.argtypes = args
        _tlib = T
    return _tlib


def exported_symbols():
    return [n for n in _SIGS if n not in TESTING_SYMBOLS]


def testing_symbols():
    return sorted(TESTING_SYMBOLS)


_fast = None


def fast():
    """The CPython fast-path module (csrc/pyfast.c) for the per-call entry points: same library,
    no ctypes per-argument conversion. None when it has not been built (ctypes is used then)."""
    global _fast
    if _fast is None:
        lib()   # loads libdvstream.so first (the module links against it by rpath)
        if os.environ.get("DV_NO_FAST") == "1":   # ctypes path only (tests of both bindings)
            _fast = False
            return None
        try:
            from . import _dvfast
            _fast = _dvfast
        except ImportError:  # pragma: no cover - built by build.build_fast / __graft_entry__.build
            _fast = False
    return _fast or None


def _check(st, name):
    if st != DV_OK:
        raise DVError(st, name, lib().dv_last_error().decode())
    return st


def _sint(s):
    """Stream handle as an int (None = torch's current stream)."""
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if hasattr(s, "cuda_stream"):
        return s.cuda_stream
    return int(s)


_fns = {}


def _call(name, *args):
    f = _fns.get(name)
    if f is None:
        f = _fns[name] = getattr(testing_lib() if name in TESTING_SYMBOLS else lib(), name)
    st = f(*args)
    if st != DV_OK:
        raise DVError(st, name, lib().dv_last_error().decode())
    return st


def _stream(s):
    if s is None:
        try:
            import torch
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:  # pragma: no cover
            return C.c_void_p(0)
    if hasattr(s, "cuda_stream"):
        return C.c_void_p(s.cuda_stream)
    return C.c_void_p(int(s))


def _ref(x):
    return None if x is None else C.byref(x)


# ---- descriptor helpers --------------------------------------------------------------------------
def region(layer_begin, layer_end, req_begin, req_end, pos_begin, pos_end, head_begin=0,
           head_end=0) -> dv_region:
    """Region of global ids; heads (0, 0) = all heads (see include/dv.h)."""
    return dv_region(layer_begin, layer_end, req_begin, req_end, pos_begin, pos_end, head_begin, head_end)


class Setup:
    """Owns the bound arrays of a dv_setup (head_bounds None = no tensor-parallel head split)."""

    def __init__(self, layer_bounds, req_bounds, max_seq, head_bounds=None):
        self.lb = (C.c_int32 * len(layer_bounds))(*layer_bounds)
        self.rb = (C.c_int32 * len(req_bounds))(*req_bounds)
        if head_bounds is not None:
            self.hb = (C.c_int32 * len(head_bounds))(*head_bounds)
            ntp, hbp = len(head_bounds) - 1, self.hb
        else:
            self.hb, ntp, hbp = None, 0, None
        self.c = dv_setup(len(layer_bounds) - 1, self.lb, len(req_bounds) - 1, self.rb, max_seq, ntp, hbp)
        self.layer_bounds, self.req_bounds, self.max_seq = list(layer_bounds), list(req_bounds), max_seq
        self.head_bounds = None if head_bounds is None else list(head_bounds)

    @property
    def n_tp(self):
        return 1 if self.head_bounds is None else len(self.head_bounds) - 1

    def flat(self, stage, micro, tp=0):
        return (stage * self.n_micro + micro) * self.n_tp + tp

    @property
    def n_stages(self):
        return self.c.n_stages

    @property
    def n_micro(self):
        return self.c.n_micro


def cache(k, v, layer_begin=0, req_begin=0, device=None, head_begin=0) -> dv_cache:
    """Descriptor of a cache held in two contiguous tensors. V is [n_layers][n_reqs][n_heads]
    [max_seq][head_dim]; K has the same shape (KV5D) or is 6-D [n_layers][n_reqs][n_heads]
    [head_dim/x][max_seq][x], x = 16/elem_bytes (FT6D). head_begin = first global head held."""
    assert k.dtype == v.dtype and v.dim() == 5 and k.is_contiguous() and v.is_contiguous()
    nL, nR, H, S, D = v.shape
    if k.dim() == 6:
        x = 16 // k.element_size()
        assert tuple(k.shape) == (nL, nR, H, D // x, S, x)
        layout = DV_LAYOUT_FT6D
    else:
        assert k.shape == v.shape
        layout = DV_LAYOUT_KV5D
    if device is None:
        device = k.device.index if k.is_cuda else -1
    return dv_cache(k.data_ptr(), v.data_ptr(), device, layout, k.element_size(),
                    layer_begin, nL, req_begin, nR, H, S, D, head_begin)


def cache_raw(k_ptr, v_ptr, device, elem_bytes, layer_begin, n_layers, req_begin, n_reqs, n_heads,
              max_seq, head_dim, head_begin=0, layout=DV_LAYOUT_KV5D) -> dv_cache:
    return dv_cache(k_ptr, v_ptr, device, layout, elem_bytes, layer_begin, n_layers,
                    req_begin, n_reqs, n_heads, max_seq, head_dim, head_begin)


def endpoint(kind, base_ptr, nbytes, flags_ptr=0, n_flags=0, device=-1, n_slots=0, slot_bytes=0,
             credits_ptr=0) -> dv_endpoint:
    """Endpoint from raw pointers; n_slots > 0 makes it a ring inbox (credits_ptr: n_flags credit
    words, include/dv.h)."""
    return dv_endpoint(kind, device, base_ptr, nbytes, flags_ptr, n_flags, n_slots, slot_bytes, credits_ptr)


def endpoint_of(buf, flags=None, kind=None, n_slots=0, slot_bytes=0, credits=None) -> dv_endpoint:
    """Endpoint over a torch buffer (device or pinned host) and an optional uint64/int64 flag
    tensor in the same kind of memory; n_slots/slot_bytes/credits (a tensor of n_flags words)
    make it a ring inbox with flow control."""
    if kind is None:
        kind = DV_EP_DEVICE if buf.is_cuda else DV_EP_HOST
    dev = buf.device.index if buf.is_cuda else -1
    nb = buf.numel() * buf.element_size()
    fp, nf = (flags.data_ptr(), flags.numel()) if flags is not None else (0, 0)
    cp = credits.data_ptr() if credits is not None else 0
    return dv_endpoint(kind, dev, buf.data_ptr(), nb, fp, nf, n_slots, slot_bytes, cp)


def endpoint_array(eps):
    if isinstance(eps, C.Array):   # prebuilt (e.g. reused every token step)
        return eps
    arr = (dv_endpoint * max(1, len(eps)))()
    for i, e in enumerate(eps):
        if e is not None:
            arr[i] = e
    return arr


def cache_array(cs):
    if isinstance(cs, C.Array):
        return cs
    arr = (dv_cache * max(1, len(cs)))()
    for i, c in enumerate(cs):
        if c is not None:
            arr[i] = c
    return arr


# ---- C entry points with the same names ----------------------------------------------------------
def dv_last_error() -> str:
    return lib().dv_last_error().decode()


def dv_abi_version() -> int:
    return lib().dv_abi_version()


def dv_stats():
    """(kernel launches, DMA calls) issued by the library since it was loaded."""
    a, b = C.c_uint64(), C.c_uint64()
    _call("dv_stats", C.byref(a), C.byref(b))
    return a.value, b.value


def dv_region_bytes(reg: dv_region, n_heads, head_dim, elem_bytes) -> int:
    out = C.c_uint64()
    _call("dv_region_bytes", _reg_ct(reg), n_heads, head_dim, elem_bytes, C.byref(out))
    return out.value


def dv_route(src: Setup, dst: Setup, reg: dv_region, n_heads, head_dim, elem_bytes):
    n = C.c_uint64()
    _call("dv_route", C.byref(src.c), C.byref(dst.c), _reg_ct(reg), n_heads, head_dim, elem_bytes,
          None, 0, C.byref(n))
    arr = (dv_piece * max(1, n.value))()
    _call("dv_route", C.byref(src.c), C.byref(dst.c), _reg_ct(reg), n_heads, head_dim, elem_bytes,
          arr, n.value, C.byref(n))
    return [arr[i] for i in range(n.value)]


class Context:
    """Owns a dv_ctx* (one per process and device)."""

    def __init__(self, device: int = 0, staging_bytes: int = 0, max_ctas: int = 0, host_ctas: int = 0):
        h = C.c_void_p()
        cfg = dv_config(staging_bytes, max_ctas, host_ctas)
        _call("dv_create", device, C.byref(cfg), C.byref(h))
        self.h = h
        self.addr = h.value   # the dv_ctx* as an int (fast path)
        self.device = device
        self._engines = []

    def close(self):
        if self.h:
            for e in list(self._engines):
                e.close()
            _call("dv_destroy", self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def dv_create(device=0, staging_bytes=0, max_ctas=0, host_ctas=0) -> Context:
    return Context(device, staging_bytes, max_ctas, host_ctas)


def dv_destroy(ctx: Context):
    ctx.close()


def dv_host_alloc(nbytes) -> int:
    p = C.c_void_p()
    _call("dv_host_alloc", nbytes, C.byref(p))
    return p.value


def dv_host_alloc_near(device, nbytes):
    """Pinned host arena NUMA-local to `device`: returns (pointer, numa node or -1)."""
    p, node = C.c_void_p(), C.c_int32()
    _call("dv_host_alloc_near", device, nbytes, C.byref(p), C.byref(node))
    return p.value, node.value


def dv_host_free(p):
    _call("dv_host_free", C.c_void_p(p))


def dv_device_alloc(device, nbytes) -> int:
    p = C.c_void_p()
    _call("dv_device_alloc", device, nbytes, C.byref(p))
    return p.value


def dv_device_free(p):
    _call("dv_device_free", C.c_void_p(p))


def dv_peer_enable(device, peer):
    _call("dv_peer_enable", device, peer)


def dv_ipc_export(ptr) -> bytes:
    b = dv_ipc_blob()
    _call("dv_ipc_export", C.c_void_p(ptr), C.byref(b))
    return bytes(b.bytes)


def dv_ipc_open(blob: bytes) -> int:
    b = dv_ipc_blob()
    C.memmove(b.bytes, blob, len(b.bytes))
    p = C.c_void_p()
    _call("dv_ipc_open", C.byref(b), C.byref(p))
    return p.value


def dv_ipc_close(p):
    _call("dv_ipc_close", C.c_void_p(p))


def dv_ipc_blob_bytes(blob: bytes) -> int:
    """Bytes the exporter shared from its pointer to the end of that allocation."""
    b = dv_ipc_blob()
    C.memmove(b.bytes, blob, len(b.bytes))
    n = C.c_uint64()
    _call("dv_ipc_blob_bytes", C.byref(b), C.byref(n))
    return n.value


def dv_flush(ctx, src_ptr, nbytes, dst: dv_endpoint, dst_off=0, flag_slot=-1, seq=0, xfer=0, stream=None):
    _call("dv_flush", ctx.h, C.c_void_p(src_ptr), nbytes, C.byref(dst), dst_off, flag_slot, seq, xfer,
          _stream(stream))


def dv_fetch(ctx, src: dv_endpoint, src_off, dst_ptr, nbytes, flag_slot=-1, wait_seq=0, xfer=0, stream=None):
    _call("dv_fetch", ctx.h, C.byref(src), src_off, flag_slot, wait_seq, C.c_void_p(dst_ptr), nbytes,
          xfer, _stream(stream))


_addr = C.addressof


def _reg_fast(reg):
    """Region for the fast path: a tuple passes as is (no ctypes structure), a dv_region by address."""
    return reg if isinstance(reg, tuple) else _addr(reg)


def _reg_ct(reg):
    """Region for the ctypes path."""
    if isinstance(reg, tuple):
        if len(reg) not in (6, 8):
            raise ValueError("region tuple needs 6 or 8 entries")
        reg = region(*reg)
    return C.byref(reg)


def dv_scatter(ctx, src: dv_cache, reg: dv_region, dst: dv_endpoint, dst_off=0, flag_slot=-1, seq=0,
               xfer=0, stream=None):
    f = _fast or fast()
    if f:
        return _check(f.scatter(ctx.addr, _addr(src), _reg_fast(reg), _addr(dst), dst_off, flag_slot, seq, xfer,
                                _sint(stream)), "dv_scatter")
    _call("dv_scatter", ctx.h, C.byref(src), _reg_ct(reg), C.byref(dst), dst_off, flag_slot, seq, xfer,
          _stream(stream))


def dv_gather(ctx, src: dv_endpoint, src_off, dst: dv_cache, reg: dv_region, flag_slot=-1, wait_seq=0,
              xfer=0, stream=None):
    f = _fast or fast()
    if f:
        return _check(f.gather(ctx.addr, _addr(src), src_off, flag_slot, wait_seq, _addr(dst), _reg_fast(reg), xfer,
                               _sint(stream)), "dv_gather")
    _call("dv_gather", ctx.h, C.byref(src), src_off, flag_slot, wait_seq, C.byref(dst), _reg_ct(reg),
          xfer, _stream(stream))


def dv_gather_chunks(ctx, src: dv_endpoint, src_off, dst: dv_cache, first: dv_region, n_chunks, pos_step,
                     flag_slot=-1, wait_seq=0, xfer=0, stream=None):
    _call("dv_gather_chunks", ctx.h, C.byref(src), src_off, flag_slot, wait_seq, C.byref(dst), _reg_ct(first),
          n_chunks, pos_step, xfer, _stream(stream))


def dv_remap(ctx, src: dv_cache, dst: dv_cache, reg: dv_region, signal: dv_endpoint = None, flag_slot=-1,
             seq=0, xfer=0, stream=None):
    f = _fast or fast()
    if f:
        return _check(f.remap(ctx.addr, _addr(src), _addr(dst), _reg_fast(reg),
                              None if signal is None else _addr(signal), flag_slot, seq, xfer, _sint(stream)),
                      "dv_remap")
    _call("dv_remap", ctx.h, C.byref(src), C.byref(dst), _reg_ct(reg), _ref(signal), flag_slot, seq,
          xfer, _stream(stream))


def dv_scatter_dyn(ctx, src: dv_cache, reg: dv_region, dst: dv_endpoint, dst_off, dst_step_bytes, d_step_ptr,
                   max_step, flag_slot=-1, seq=0, stream=None):
    _call("dv_scatter_dyn", ctx.h, C.byref(src), _reg_ct(reg), C.byref(dst), dst_off, dst_step_bytes, flag_slot,
          seq, C.c_void_p(d_step_ptr), max_step, _stream(stream))


def dv_dplan_scatter(ctx, src: dv_cache, reg: dv_region, dst: dv_endpoint, dst_off=0, dst_step_bytes=0, flag_slot=-1,
                     seq=0, max_step=0) -> dv_dplan:
    p = dv_dplan()
    _call("dv_dplan_scatter", ctx.h, C.byref(src), _reg_ct(reg), C.byref(dst), dst_off, dst_step_bytes, flag_slot, seq,
          max_step, C.byref(p))
    return p


def dv_dplan_free(ctx, plan):
    """Hand back a plan's (dv_dplan) or a plan set's (dv_dplan_set) tickets: after its last launch."""
    if isinstance(plan, dv_dplan_set):
        _call("dv_dplan_set_free", ctx.h, C.byref(plan))
    else:
        _call("dv_dplan_free", ctx.h, C.byref(plan))


def dv_dplan_remap(ctx, src: dv_cache, dst: dv_cache, reg: dv_region, signal: dv_endpoint = None, flag_slot=-1, seq=0,
                   max_step=0) -> dv_dplan:
    p = dv_dplan()
    _call("dv_dplan_remap", ctx.h, C.byref(src), C.byref(dst), _reg_ct(reg), _ref(signal), flag_slot, seq, max_step,
          C.byref(p))
    return p


def dv_remap_dyn(ctx, src: dv_cache, dst: dv_cache, reg: dv_region, d_step_ptr, max_step, signal: dv_endpoint = None,
                 flag_slot=-1, seq=0, stream=None):
    _call("dv_remap_dyn", ctx.h, C.byref(src), C.byref(dst), _reg_ct(reg), _ref(signal), flag_slot, seq,
          C.c_void_p(d_step_ptr), max_step, _stream(stream))


# The level-1 wrappers take my_tp as a keyword (default 0) after the C positional arguments.
def dv_stream_out(ctx, src: dv_cache, reg: dv_region, src_setup: Setup, my_stage, my_micro,
                  dst_setup: Setup, inboxes, seq, xfer=0, stream=None, my_tp=0):
    arr = endpoint_array(inboxes)
    f = _fast or fast()
    if f:
        return _check(f.stream_out(ctx.addr, _addr(src), _reg_fast(reg), _addr(src_setup.c), my_stage, my_micro, my_tp,
                                   _addr(dst_setup.c), _addr(arr), len(arr), seq, xfer, _sint(stream)),
                      "dv_stream_out")
    _call("dv_stream_out", ctx.h, C.byref(src), _reg_ct(reg), C.byref(src_setup.c), my_stage, my_micro,
          my_tp, C.byref(dst_setup.c), arr, len(arr), seq, xfer, _stream(stream))


def dv_stream_in(ctx, dst: dv_cache, reg: dv_region, src_setup: Setup, dst_setup: Setup, my_stage,
                 my_micro, inbox: dv_endpoint, wait_seq, xfer=0, stream=None, my_tp=0):
    f = _fast or fast()
    if f:
        return _check(f.stream_in(ctx.addr, _addr(dst), _reg_fast(reg), _addr(src_setup.c), _addr(dst_setup.c),
                                  my_stage, my_micro, my_tp, _addr(inbox), wait_seq, xfer, _sint(stream)),
                      "dv_stream_in")
    _call("dv_stream_in", ctx.h, C.byref(dst), _reg_ct(reg), C.byref(src_setup.c), C.byref(dst_setup.c),
          my_stage, my_micro, my_tp, C.byref(inbox), wait_seq, xfer, _stream(stream))


def dv_stream_out_direct(ctx, src: dv_cache, reg: dv_region, src_setup: Setup, my_stage, my_micro,
                         dst_setup: Setup, dst_caches, signals=None, seq=0, xfer=0, stream=None, my_tp=0):
    carr = cache_array(dst_caches)
    sarr = endpoint_array(signals) if signals is not None else None
    f = _fast or fast()
    if f:
        return _check(f.stream_out_direct(ctx.addr, _addr(src), _reg_fast(reg), _addr(src_setup.c), my_stage, my_micro,
                                          my_tp, _addr(dst_setup.c), _addr(carr),
                                          None if sarr is None else _addr(sarr), len(dst_caches), seq, xfer,
                                          _sint(stream)), "dv_stream_out_direct")
    _call("dv_stream_out_direct", ctx.h, C.byref(src), _reg_ct(reg), C.byref(src_setup.c), my_stage,
          my_micro, my_tp, C.byref(dst_setup.c), carr, sarr, len(dst_caches), seq, xfer, _stream(stream))


def dv_dplan_stream_out_direct(ctx, src: dv_cache, reg: dv_region, src_setup: Setup, my_stage, my_micro,
                               dst_setup: Setup, dst_caches, signals=None, seq=0, max_step=0, my_tp=0) -> dv_dplan_set:
    """Level 1 as device plans (include/dv.h): one remap plan per route piece leaving this block."""
    carr = cache_array(dst_caches)
    sarr = endpoint_array(signals) if signals is not None else None
    out = dv_dplan_set()
    _call("dv_dplan_stream_out_direct", ctx.h, C.byref(src), _reg_ct(reg), C.byref(src_setup.c), my_stage, my_micro,
          my_tp, C.byref(dst_setup.c), carr, sarr, len(dst_caches), seq, max_step, C.byref(out))
    return out


def dv_dplan_stream_out(ctx, src: dv_cache, reg: dv_region, src_setup: Setup, my_stage, my_micro, dst_setup: Setup,
                        inboxes, seq=0, my_tp=0) -> dv_dplan_set:
    """Level 1 as device plans, inbox form (include/dv.h): one scatter plan per route piece."""
    arr = endpoint_array(inboxes)
    out = dv_dplan_set()
    _call("dv_dplan_stream_out", ctx.h, C.byref(src), _reg_ct(reg), C.byref(src_setup.c), my_stage, my_micro, my_tp,
          C.byref(dst_setup.c), arr, len(inboxes), seq, C.byref(out))
    return out


def dv_wait(ctx, ep: dv_endpoint, flag_slot, seq, stream=None):
    f = _fast or fast()
    if f:
        return _check(f.wait(ctx.addr, _addr(ep), flag_slot, seq, _sint(stream)), "dv_wait")
    _call("dv_wait", ctx.h, C.byref(ep), flag_slot, seq, _stream(stream))


def dv_signal(ctx, ep: dv_endpoint, flag_slot, seq, stream=None):
    f = _fast or fast()
    if f:
        return _check(f.signal(ctx.addr, _addr(ep), flag_slot, seq, _sint(stream)), "dv_signal")
    _call("dv_signal", ctx.h, C.byref(ep), flag_slot, seq, _stream(stream))


def dv_query(ctx, ep: dv_endpoint, flag_slot, seq) -> bool:
    d = C.c_int32()
    _call("dv_query", ctx.h, C.byref(ep), flag_slot, seq, C.byref(d))
    return bool(d.value)


def dvt_tune(name: str, value: int):
    """Change one experiment knob of the copy kernels at run time (include/dv_trace.h)."""
    _call("dvt_tune", name.encode(), value)


def dvt_launch_count(form: str) -> int:
    """Launches so far of one kernel form ("tma_transpose", "all") -- include/dv_trace.h."""
    n = C.c_uint64()
    _call("dvt_launch_count", form.encode(), C.byref(n))
    return n.value


# ---- persistent stream engine (include/dv.h dv_engine_*) -----------------------------------------
class Engine:
    """A resident copy engine (dv_engine_create). While it runs, torch.cuda.synchronize() cannot
    return: call park() first (the next kick relaunches it), or synchronise streams."""

    def __init__(self, ctx, n_ctas=8):
        self.ctx = ctx
        h = C.c_void_p()
        _call("dv_engine_create", ctx.h, n_ctas, C.byref(h))
        self.h = h
        ctx._engines.append(self)

    def plan_scatter(self, src: dv_cache, reg, dst: dv_endpoint, dst_off, dst_step_bytes, flag_slot=-1, seq=0,
                     max_step=0) -> int:
        p = C.c_int32()
        _call("dv_engine_plan_scatter", self.h, C.byref(src), _reg_ct(reg), C.byref(dst), dst_off, dst_step_bytes,
              flag_slot, seq, max_step, C.byref(p))
        return p.value

    def plan_remap(self, src: dv_cache, dst: dv_cache, reg, signal: dv_endpoint = None, flag_slot=-1, seq=0,
                   max_step=0) -> int:
        p = C.c_int32()
        _call("dv_engine_plan_remap", self.h, C.byref(src), C.byref(dst), _reg_ct(reg), _ref(signal), flag_slot,
              seq, max_step, C.byref(p))
        return p.value

    def kick(self, plan, step, stream=None):
        _call("dv_engine_kick", self.h, plan, step, _stream(stream))

    def doorbell(self, plan) -> int:
        w = C.c_void_p()
        _call("dv_engine_doorbell", self.h, plan, C.byref(w))
        return w.value

    def done(self, plan) -> int:
        n = C.c_uint64()
        _call("dv_engine_done", self.h, plan, C.byref(n))
        return n.value

    def trace(self, stamps_ptr=0, n=0):
        _call("dvt_engine_trace", self.h, C.c_void_p(stamps_ptr), n)

    def park(self):
        _call("dv_engine_park", self.h)

    def resume(self):
        _call("dv_engine_resume", self.h)

    def close(self):
        if self.h is not None and self.h.value:
            _call("dv_engine_destroy", self.h)
            if self in self.ctx._engines:
                self.ctx._engines.remove(self)
        self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def dv_engine_create(ctx, n_ctas=8) -> Engine:
    return Engine(ctx, n_ctas)


class Partition:
    """An SM partition (dv_partition_create, include/dv.h): `streaming` and `compute` are the raw
    cudaStream_t handles (ints) of its two green contexts; wrap them with
    torch.cuda.ExternalStream to run work there. Destroy after all work on them has completed."""

    def __init__(self, device, streaming_sms, priority=0):
        h, s0, s1 = C.c_void_p(), C.c_void_p(), C.c_void_p()
        n0, n1 = C.c_int32(), C.c_int32()
        _call("dv_partition_create", device, streaming_sms, priority, C.byref(h), C.byref(s0), C.byref(s1),
              C.byref(n0), C.byref(n1))
        self.h = h
        self.streaming, self.compute = s0.value, s1.value
        self.sms_streaming, self.sms_compute = n0.value, n1.value

    def destroy(self):
        if self.h:
            _call("dv_partition_destroy", self.h)
            self.h = None


def dv_partition_create(device, streaming_sms, priority=0) -> Partition:
    return Partition(device, streaming_sms, priority)


# ---- test-only utilities (include/dv_testing.h) and baselines (include/dv_baselines.h) -----------
def dvt_fill(c: dv_cache, kind, seed=0, box=None, valid=(0, 1 << 30), reg: dv_region = None, stream=None,
             t_end_ptr=0):
    b = (C.c_int32 * 5)(*box) if box is not None else None
    _call("dvt_fill", C.byref(c), kind, seed, b, valid[0], valid[1], (None if reg is None else _reg_ct(reg)), C.c_void_p(t_end_ptr),
          _stream(stream))


def dvt_fill_rows(c: dv_cache, seed, reg, plan=None, step=0, t_start_ptr=0, t_end_ptr=0, stream=None,
                  kind=DVT_FILL_HASH, box=None):
    """plan: None, a dv_dplan, a dv_dplan_set or a list of dv_dplan; kind / box as dvt_fill."""
    if plan is None:
        arr, n = None, 0
    elif isinstance(plan, dv_dplan):
        arr, n = C.byref(plan), 1
    elif isinstance(plan, dv_dplan_set):
        arr, n = (plan.plan if plan.n else None), plan.n
    else:
        arr, n = (dv_dplan * len(plan))(*plan), len(plan)
    b = (C.c_int32 * 5)(*box) if box is not None else None
    _call("dvt_fill_rows", C.byref(c), kind, seed, b, _reg_ct(reg), arr, n, step, C.c_void_p(t_start_ptr),
          C.c_void_p(t_end_ptr), _stream(stream))


def dvt_fill_ring(c: dv_cache, seed, reg, doorbell_ptr, step, ticket_ptr, t_end_ptr=0, stream=None):
    _call("dvt_fill_ring", C.byref(c), seed, _reg_ct(reg), C.c_void_p(t_end_ptr), C.c_void_p(doorbell_ptr), step,
          C.c_void_p(ticket_ptr), _stream(stream))


def dvt_verify(c: dv_cache, counter_ptr, seed=0, kind=0, reg: dv_region = None, wire_ptr=0, box=None,
               valid=(0, 1 << 30), stream=None):
    """Adds to the uint64 at counter_ptr (device) the words of `reg` (in cache c, or in the dense
    wire at wire_ptr) that differ from the generator (dvt_fill's word)."""
    b = (C.c_int32 * 5)(*box) if box is not None else None
    _call("dvt_verify", C.byref(c), C.c_void_p(wire_ptr), kind, seed, b, valid[0], valid[1], (None if reg is None else _reg_ct(reg)),
          C.c_void_p(counter_ptr), _stream(stream))


def dvt_trace(ctx, ts_ptr=0):
    _call("dvt_trace", ctx.h, C.c_void_p(ts_ptr))


def dvt_release_scope(ctx, flag_ptr, payload_ptr=0) -> bool:
    """True when the fused publish would release at gpu scope (flag and payload in this GPU's HBM)."""
    out = C.c_int32()
    _call("dvt_release_scope", ctx.h, C.c_void_p(flag_ptr), C.c_void_p(payload_ptr), C.byref(out))
    return bool(out.value)


def dvt_watch(flag_ptr, seq0, n, ts_ptr, timeout_ns=2_000_000_000, stream=None):
    _call("dvt_watch", C.c_void_p(flag_ptr), seq0, n, C.c_void_p(ts_ptr), timeout_ns, _stream(stream))


def dvt_consume(flag_ptr, seq, src_ptr, dst_ptr, nbytes, ok_ptr, timeout_ns=2_000_000_000, stream=None):
    _call("dvt_consume", C.c_void_p(flag_ptr), seq, C.c_void_p(src_ptr), C.c_void_p(dst_ptr), nbytes, timeout_ns,
          C.c_void_p(ok_ptr), _stream(stream))


def dvt_spin(ns, ctas, stream=None):
    _call("dvt_spin", ns, ctas, _stream(stream))


def dvb_per_run_copy(src: dv_cache, reg: dv_region, dst_ptr, stream=None) -> int:
    n = C.c_uint64()
    _call("dvb_per_run_copy", C.byref(src), _reg_ct(reg), C.c_void_p(dst_ptr), _stream(stream), C.byref(n))
    return n.value


def dvb_buffered_copy(src: dv_cache, reg: dv_region, staging_ptr, dst_ptr, stream=None) -> int:
    n = C.c_uint64()
    _call("dvb_buffered_copy", C.byref(src), _reg_ct(reg), C.c_void_p(staging_ptr), C.c_void_p(dst_ptr),
          _stream(stream), C.byref(n))
    return n.value
