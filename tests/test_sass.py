"""The built library runs the hot path on the B200 units the design claims
(DESIGN.md §6): checked on the SASS of libbaton.so, no GPU needed.

* decode attention (MHA): bulk copies by the TMA engine (UBLKCP) tracked by
  mbarrier transactions (SYNCS);
* GQA decode and prefill/extend attention: 5th-gen tensor-core MMAs (UTCHMMA),
  TMEM loads/stores (LDTM/STTM) and TMA tensor loads (UTMALDG);
* no legacy HMMA in the tcgen05 kernels."""
import functools
import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2410_18701_b200", "libbaton.so")


@functools.lru_cache(maxsize=1)
def _sass_cached():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(tool):
        pytest.skip("libbaton.so or cuobjdump missing")
    out = subprocess.run([tool, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = {}
    name = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            name = m.group(1)
            funcs[name] = []
        elif name:
            funcs[name].append(line)
    return {k: "\n".join(v) for k, v in funcs.items()}


def _sass():
    return _sass_cached()


def _find(funcs, key):
    hits = {k: v for k, v in funcs.items() if key in k}
    assert hits, f"no kernel matching {key}"
    return hits


def test_targets_sm100a():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(tool):
        pytest.skip("libbaton.so or cuobjdump missing")
    out = subprocess.run([tool, "-lelf", LIB], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_decode_attention_uses_bulk_copies_and_mbarriers():
    for body in _find(_sass(), "decode_attention_kernel").values():
        assert "UBLKCP" in body and "SYNCS" in body


def test_gqa_tcgen05_kernel_uses_tensor_cores_tmem_and_tma():
    for body in _find(_sass(), "decode_gqa_tc_kernel").values():
        assert "UTCHMMA" in body and "LDTM" in body and "UTMALDG" in body
        assert "HMMA.16816" not in body


def test_prefill_extend_kernel_uses_tensor_cores_tmem_and_tma():
    for body in _find(_sass(), "prefill_attention_kernel").values():
        assert "UTCHMMA" in body and "LDTM" in body and "STTM" in body and "UTMALDG" in body
