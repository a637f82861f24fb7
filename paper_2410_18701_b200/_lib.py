"""ctypes loader for libbaton.so (argument marshalling only).

The product path has no fallback: if the shared library is missing or fails to
load, importing this module raises.  Build it with
``python -m paper_2410_18701_b200.build`` (``__graft_entry__.build()`` does).
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbaton.so")

BATON_OK = 0
BATON_E_INVALID = -1
BATON_E_SLOT_BUSY = -2
BATON_E_SLOT_EMPTY = -3
BATON_E_CAPACITY = -4
BATON_E_CUDA = -5
BATON_CHUNK = 256


class BatonError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        msg = _err_string(code)
        if code == BATON_E_CUDA:
            msg += f" (cudaError {lib.baton_cuda_error()})"
        super().__init__(f"{what}: {msg} [{code}]")


class baton_shape(ctypes.Structure):
    _fields_ = [("layers", ctypes.c_int32), ("slots", ctypes.c_int32),
                ("q_heads", ctypes.c_int32), ("kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("max_ctx", ctypes.c_int32)]


class baton_config(ctypes.Structure):
    _fields_ = [("shape", baton_shape), ("k_cache", ctypes.c_void_p),
                ("v_cache", ctypes.c_void_p), ("mask", ctypes.c_void_p),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libbaton.so not built at {LIB_PATH}; run "
                          "`python -m paper_2410_18701_b200.build` (no CPU fallback exists)")
    return ctypes.CDLL(LIB_PATH)


lib = _load()

_P = ctypes.c_void_p
_I = ctypes.c_int
_I32P = ctypes.POINTER(ctypes.c_int32)
_SIGS = {
    "baton_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(baton_shape)]),
    "baton_decode_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(baton_shape)]),
    "baton_create": (_I, [ctypes.POINTER(baton_config), _P, ctypes.POINTER(_P)]),
    "baton_destroy": (None, [_P]),
    "baton_device_meta": (_I, [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "baton_query": (_I, [_P, _I32P, _I32P, _I32P, _I32P]),
    "baton_mask_update": (_I, [_P, _P]),
    "baton_append_kv": (_I, [_P, _I, _P, _P, _P]),
    "baton_decode_attention": (_I, [_P, _P, _P, _P, _P, _P, _P, ctypes.POINTER(baton_shape),
                                    ctypes.c_float, _P, ctypes.c_size_t, _P]),
    "baton_decode_layer": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "baton_decode_step": (_I, [_P, _P, _P, _P, _P, _P]),
    "baton_remove": (_I, [_P, _I32P, _I, _I32P, _P]),
    "baton_insert": (_I, [_P, _I, _P, _P, _I, _P]),
    "baton_insert_many": (_I, [_P, _I, _I32P, ctypes.POINTER(_P), ctypes.POINTER(_P), _I32P, _P]),
    "baton_extract": (_I, [_P, _I, _P, _P, _P]),
    "baton_compact": (_I, [_P, _I, _I32P, _P]),
    "baton_prefill_attention": (_I, [_P, _P, _P, _P, _I, ctypes.POINTER(baton_shape),
                                     ctypes.c_float, _P]),
    "baton_prefill_attention_varlen": (_I, [_P, _P, _P, _P, _I32P, _I, ctypes.POINTER(baton_shape),
                                            ctypes.c_float, _P]),
    "baton_shape_step": (_I, [_P, _I, _I, _I32P, _I32P, _P, _P, _P, _P, _P]),
    "baton_error_string": (ctypes.c_char_p, [_I]),
    "baton_cuda_error": (_I, []),
    "baton_keygen_tokens": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, ctypes.c_uint64, _I, _P]),
    "baton_keygen_history": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, ctypes.c_uint64, _I,
                                  ctypes.c_int64, ctypes.c_int64, _P]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def _err_string(code):
    return lib.baton_error_string(code).decode()


def check(code, what):
    if code != BATON_OK:
        raise BatonError(code, what)
    return code


def exported_symbols():
    return list(_SIGS)
