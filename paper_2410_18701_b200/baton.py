"""Thin Python binding of libbaton with the ABI's names (include/baton.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
of libbaton.so.  PyTorch provides device memory and streams; tensors are passed
as raw pointers.  There is no CPU or PyTorch fallback for any operation.
"""
import ctypes
import math

import numpy as np
import torch

from . import _lib
from ._lib import lib, check, baton_shape, baton_config, BatonError, BATON_CHUNK


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _i32(arr):
    a = (ctypes.c_int32 * len(arr))(*[int(x) for x in arr])
    return a


def make_shape(layers, slots, q_heads, kv_heads, head_dim, max_ctx):
    return baton_shape(layers, slots, q_heads, kv_heads, head_dim, max_ctx)


def baton_workspace_bytes(shape):
    return lib.baton_workspace_bytes(ctypes.byref(shape))


def baton_decode_workspace_bytes(shape):
    return lib.baton_decode_workspace_bytes(ctypes.byref(shape))


def baton_decode_attention(q, k, v, mask, lens, pad_start, out, shape, scale, workspace,
                           stream=None):
    """Stateless a3 (see include/baton.h).  All tensors on the same CUDA device."""
    check(lib.baton_decode_attention(_ptr(q), _ptr(k), _ptr(v), _ptr(mask), _ptr(lens),
                                     _ptr(pad_start), _ptr(out), ctypes.byref(shape),
                                     ctypes.c_float(scale), _ptr(workspace),
                                     ctypes.c_size_t(workspace.numel() * workspace.element_size()),
                                     _stream(stream)), "baton_decode_attention")
    return out


def baton_prefill_attention(q, k, v, out, length, q_heads, kv_heads, head_dim, scale=None,
                            stream=None):
    """a8 (see include/baton.h): causal attention of a new query over its prompt.
    q, out: [q_heads][len][head_dim]; k, v: [kv_heads][len][head_dim] (bf16, CUDA)."""
    shape = make_shape(1, 1, q_heads, kv_heads, head_dim, 16)
    check(lib.baton_prefill_attention(_ptr(q), _ptr(k), _ptr(v), _ptr(out), length,
                                      ctypes.byref(shape),
                                      ctypes.c_float(scale or 1.0 / math.sqrt(head_dim)),
                                      _stream(stream)), "baton_prefill_attention")
    return out


def baton_prefill_attention_varlen(q, k, v, out, lens, q_heads, kv_heads, head_dim, scale=None,
                                   stream=None):
    """a8 batched (include/baton.h): n prompts packed along the token axis in one launch.
    q, out: [q_heads][T][head_dim]; k, v: [kv_heads][T][head_dim]; lens: the n prompt
    lengths (prompt i starts at sum(lens[:i]))."""
    cu = np.zeros(len(lens) + 1, np.int32)
    cu[1:] = np.cumsum(np.asarray(lens, np.int64))
    shape = make_shape(1, 1, q_heads, kv_heads, head_dim, 16)
    check(lib.baton_prefill_attention_varlen(_ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                             cu.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                             len(lens), ctypes.byref(shape),
                                             ctypes.c_float(scale or 1.0 / math.sqrt(head_dim)),
                                             _stream(stream)), "baton_prefill_attention_varlen")
    return out


def baton_keygen_tokens(out, qids, pos, layers, n_slots, heads, head_dim, kind, layer0, seed,
                        scale_exp, stream=None):
    check(lib.baton_keygen_tokens(_ptr(out), _ptr(qids), _ptr(pos), layers, n_slots, heads,
                                  head_dim, kind, layer0, ctypes.c_uint64(seed), scale_exp,
                                  _stream(stream)), "baton_keygen_tokens")
    return out


def baton_keygen_history(out, layers, heads, head_dim, qid, pos_begin, n, kind, seed, scale_exp,
                         head_stride=None, layer_stride=None, stream=None):
    hs = n * head_dim if head_stride is None else head_stride
    ls = heads * n * head_dim if layer_stride is None else layer_stride
    check(lib.baton_keygen_history(_ptr(out), layers, heads, head_dim, qid, pos_begin, n, kind,
                                   ctypes.c_uint64(seed), scale_exp, ctypes.c_int64(hs),
                                   ctypes.c_int64(ls), _stream(stream)), "baton_keygen_history")
    return out


class BatonShard:
    """One GPU's Baton batch: the slot-relative K/V caches, the paper's mask and
    the libbaton state handle.  Methods mirror the C ABI one to one."""

    def __init__(self, layers, slots, q_heads, kv_heads, head_dim, max_ctx, device=None,
                 stream=None):
        self.device = torch.device(device or "cuda")
        self.shape = make_shape(layers, slots, q_heads, kv_heads, head_dim, max_ctx)
        self.L, self.B, self.Hq, self.Hkv, self.D, self.S_cap = (layers, slots, q_heads, kv_heads,
                                                                  head_dim, max_ctx)
        dims = (layers, slots, kv_heads, max_ctx, head_dim)
        # torch.empty: never-written placeholder rows are never read (initcheck-clean)
        self.k_cache = torch.empty(dims, dtype=torch.bfloat16, device=self.device)
        self.v_cache = torch.empty(dims, dtype=torch.bfloat16, device=self.device)
        self.mask = torch.empty((slots, max_ctx), dtype=torch.uint8, device=self.device)
        nbytes = baton_workspace_bytes(self.shape)
        if nbytes == 0:
            raise BatonError(_lib.BATON_E_INVALID, "unsupported shape")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        cfg = baton_config(self.shape, self.k_cache.data_ptr(), self.v_cache.data_ptr(),
                           self.mask.data_ptr(), self.workspace.data_ptr(), nbytes)
        h = ctypes.c_void_p()
        check(lib.baton_create(ctypes.byref(cfg), _stream(stream), ctypes.byref(h)), "baton_create")
        self._h = h
        S, lens, pad = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        check(lib.baton_device_meta(h, ctypes.byref(S), ctypes.byref(lens), ctypes.byref(pad)),
              "baton_device_meta")
        base = self.workspace.data_ptr()
        self.d_S = self.workspace[S.value - base:S.value - base + 4].view(torch.int32)
        self.d_lens = self.workspace[lens.value - base:lens.value - base + 4 * slots].view(torch.int32)
        self.d_pad = self.workspace[pad.value - base:pad.value - base + 4 * slots].view(torch.int32)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.baton_destroy(h)
            self._h = None

    # ------------------------------------------------------------ views
    def layer_k(self, layer):
        return self.k_cache[layer]

    def layer_v(self, layer):
        return self.v_cache[layer]

    @property
    def S(self):
        """Shared logical length S (host mirror, no device sync)."""
        S = ctypes.c_int32()
        check(lib.baton_query(self._h, ctypes.byref(S), None, None, None), "baton_query")
        return S.value

    def baton_query(self):
        S = ctypes.c_int32()
        pad = (ctypes.c_int32 * self.B)()
        lens = (ctypes.c_int32 * self.B)()
        occ = (ctypes.c_int32 * self.B)()
        check(lib.baton_query(self._h, ctypes.byref(S), pad, lens, occ), "baton_query")
        return {"S": S.value, "pad": np.array(pad[:], dtype=np.int64),
                "lens": np.array(lens[:], dtype=np.int64),
                "occ": np.array(occ[:], dtype=np.int64)}

    # ------------------------------------------------------------ decode step
    def baton_mask_update(self, stream=None):
        check(lib.baton_mask_update(self._h, _stream(stream)), "baton_mask_update")

    def baton_append_kv(self, layer, k_new, v_new, stream=None):
        check(lib.baton_append_kv(self._h, layer, _ptr(k_new), _ptr(v_new), _stream(stream)),
              "baton_append_kv")

    def baton_decode_layer(self, layer, q, out, k_new=None, v_new=None, stream=None):
        check(lib.baton_decode_layer(self._h, layer, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out),
                                     _stream(stream)), "baton_decode_layer")
        return out

    def baton_decode_step(self, q, k_new, v_new, out, stream=None):
        """Whole decode iteration (a1 + fused a2/a3 for every layer), graph-replayed."""
        check(lib.baton_decode_step(self._h, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out),
                                    _stream(stream)), "baton_decode_step")
        return out

    def baton_shape_step(self, W, new_slots, new_lens, q, k_new, v_new, out, stream=None):
        """NEXT-1: one vector-shaping iteration of width W (include/baton.h).
        q/out [L][slots][W][q_heads][D]; k_new/v_new [L][slots][W][kv_heads][D] (token-major)."""
        new_slots, new_lens = list(new_slots), list(new_lens)
        check(lib.baton_shape_step(self._h, int(W), len(new_slots), _i32(new_slots), _i32(new_lens),
                                   _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(out), _stream(stream)),
              "baton_shape_step")
        return out

    def baton_decode_attention(self, layer, q, out, scale=None, stream=None, use_mask=True):
        ws = baton_decode_workspace_bytes(self.shape)
        off = self.workspace.numel() - ws
        return baton_decode_attention(q, self.k_cache[layer], self.v_cache[layer],
                                      self.mask if use_mask else None, self.d_lens, self.d_pad, out,
                                      self.shape, scale or 1.0 / math.sqrt(self.D),
                                      self.workspace[off:], stream)

    # ------------------------------------------------------------ splice
    def baton_remove(self, slots, stream=None):
        slots = list(slots)
        rel = ctypes.c_int32()
        arr = _i32(slots) if slots else None
        check(lib.baton_remove(self._h, arr, len(slots), ctypes.byref(rel), _stream(stream)),
              "baton_remove")
        return rel.value

    def baton_insert(self, slot, k_pref, v_pref, length, stream=None):
        check(lib.baton_insert(self._h, slot, _ptr(k_pref), _ptr(v_pref), length, _stream(stream)),
              "baton_insert")

    def baton_insert_many(self, slots, k_prefs, v_prefs, lens, stream=None):
        n = len(slots)
        if n == 0:
            return
        kp = (ctypes.c_void_p * n)(*[t.data_ptr() for t in k_prefs])
        vp = (ctypes.c_void_p * n)(*[t.data_ptr() for t in v_prefs])
        check(lib.baton_insert_many(self._h, n, _i32(slots), kp, vp, _i32(lens), _stream(stream)),
              "baton_insert_many")

    def baton_extract(self, slot, k_out=None, v_out=None, stream=None):
        n = int(self.baton_query()["lens"][slot]) if 0 <= slot < self.B else 0
        if k_out is None:
            # an empty slot still gets (1-row) buffers so the call reports SLOT_EMPTY
            k_out = torch.empty((self.L, self.Hkv, max(n, 1), self.D), dtype=torch.bfloat16,
                                device=self.device)
            v_out = torch.empty_like(k_out)
        check(lib.baton_extract(self._h, slot, _ptr(k_out), _ptr(v_out), _stream(stream)),
              "baton_extract")
        return k_out, v_out

    def baton_compact(self, n_active, stream=None):
        o2n = (ctypes.c_int32 * self.B)()
        check(lib.baton_compact(self._h, n_active, o2n, _stream(stream)), "baton_compact")
        return list(o2n[:])

    # ------------------------------------------------------------ helpers for tests
    def live_kv(self, slot):
        """Device K/V rows [0, lens) of a slot (logical order), for parity checks."""
        n = int(self.baton_query()["lens"][slot])
        return self.k_cache[:, slot, :, :n], self.v_cache[:, slot, :, :n]
