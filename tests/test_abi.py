"""The C-ABI library loads on a CPU-only host and exports every symbol the
public headers declare; host-side validation paths return the documented error
codes without touching a device (no compute calls here)."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(baton_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_headers_declare_the_north_star_calls():
    names = _declared()
    for n in ("baton_decode_attention", "baton_remove", "baton_insert", "baton_append_kv",
              "baton_mask_update", "baton_extract", "baton_compact", "baton_insert_many"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2410_18701_b200 import _lib
    for n in _declared():
        assert hasattr(_lib.lib, n), n
    assert set(_lib.exported_symbols()) == _declared()


def test_host_side_validation():
    from paper_2410_18701_b200 import _lib
    from paper_2410_18701_b200.baton import make_shape, baton_workspace_bytes
    lib = _lib.lib
    good = make_shape(32, 32, 32, 32, 128, 2048)
    n = baton_workspace_bytes(good)
    # meta + tickets + split-K partials (8 chunks x 130 floats per (slot, head))
    assert n >= 32 * 32 * 8 * 130 * 4
    assert baton_workspace_bytes(make_shape(1, 4, 2, 2, 16, 64)) > 0
    for bad in [make_shape(1, 4, 3, 2, 16, 64),      # q_heads not a multiple of kv_heads
                make_shape(1, 4, 2, 2, 96, 64),      # unsupported head_dim
                make_shape(1, 4, 2, 2, 16, 60),      # max_ctx not a multiple of 16
                make_shape(1, 0, 2, 2, 16, 64),
                make_shape(1, 1000, 2, 2, 16, 64)]:  # too many slots per shard
        assert baton_workspace_bytes(bad) == 0
    assert lib.baton_create(None, None, None) == _lib.BATON_E_INVALID
    assert lib.baton_decode_attention(None, None, None, None, None, None, None,
                                      ctypes.byref(good), 0.1, None, 0, None) == _lib.BATON_E_INVALID
    assert lib.baton_mask_update(None, None) == _lib.BATON_E_INVALID
    assert lib.baton_keygen_history(None, 1, 1, 16, 0, 0, 1, 0, 0, 0, 16, 16, None) == _lib.BATON_E_INVALID
    # batched prefill: every rejection happens on the host, before any launch
    fake = ctypes.c_void_p(1 << 20)                    # 16-B aligned, never dereferenced
    pf = make_shape(1, 1, 8, 8, 128, 16)

    def varlen(cu, n, shape=pf, q=fake, scale=0.1):
        arr = (ctypes.c_int32 * len(cu))(*cu)
        return lib.baton_prefill_attention_varlen(q, fake, fake, fake, arr, n, ctypes.byref(shape),
                                                  scale, None)
    assert varlen([0, 5], 1, q=None) == _lib.BATON_E_INVALID          # null tensor
    assert varlen([0], 0) == _lib.BATON_E_INVALID                     # no prompt
    assert varlen(list(range(66)), 65) == _lib.BATON_E_INVALID        # > 64 prompts
    assert varlen([1, 5], 1) == _lib.BATON_E_INVALID                  # cu_lens[0] != 0
    assert varlen([0, 4, 4, 9], 3) == _lib.BATON_E_INVALID            # an empty prompt
    assert varlen([0, 40 * 128 * 27], 1) == _lib.BATON_E_INVALID      # > 1024 query tiles
    assert varlen([0, 5], 1, scale=0.0) == _lib.BATON_E_INVALID       # scale must be > 0
    assert varlen([0, 5], 1, shape=make_shape(1, 1, 8, 8, 64, 16)) == _lib.BATON_E_INVALID  # head_dim
    assert varlen([0, 5], 1, q=ctypes.c_void_p((1 << 20) + 8)) == _lib.BATON_E_INVALID      # alignment
    assert lib.baton_error_string(_lib.BATON_E_SLOT_BUSY).decode() == "slot busy"


def test_no_oracle_import_in_product():
    for f in glob.glob(os.path.join(ROOT, "paper_2410_18701_b200", "**", "*.py"), recursive=True):
        src = open(f).read()
        assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), f
        assert not re.search(r"^\s*(from|import)\s+baton_inputs\b", src, re.M), f
    for f in glob.glob(os.path.join(ROOT, "oracle", "*.py")):
        src = open(f).read()
        assert not re.search(r"^\s*(from|import)\s+paper_2410_18701_b200\b", src, re.M), f
