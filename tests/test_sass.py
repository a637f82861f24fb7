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


def _issue_loops(body):
    """Uniform-datapath issue ops (tcgen05.mma/commit, TMA tensor loads, bulk copies)
    that ptxas wrapped in a per-lane ELECT / BRA.U.ANY loop: an op whose next few
    instructions branch back with BRA.U.ANY."""
    lines = [l for l in body.splitlines() if "/*" in l and not l.strip().startswith("/* 0x")]
    hits = 0
    for i, l in enumerate(lines):
        if re.search(r"\b(UTCHMMA|UTCBAR|UTMALDG|UBLKCP)\b", l):
            if any("BRA.U.ANY" in x for x in lines[i + 1:i + 5]):
                hits += 1
    return hits


@pytest.mark.parametrize("kernel", ["decode_gqa_tc_kernel", "decode_attention_kernel"])
def test_decode_issuers_have_no_per_lane_loops(kernel):
    """DESIGN §6.1/§6.2: the producers and the tcgen05 issuers run as converged warps with
    the uniform-datapath ops under elect.sync, so each op is ONE instruction (under
    `if (lane == 0)` ptxas wrapped every tcgen05.mma / commit / TMA issue in a per-lane
    ELECT loop, and the prefill's MMA thread paced its tile loop)."""
    for name, body in _find(_sass(), kernel).items():
        assert _issue_loops(body) == 0, name


def test_prefill_mma_issuer_has_no_per_lane_loops():
    """The prefill's MMA warp (§6.3): every UTCHMMA / UTCBAR outside per-lane loops (its
    producer keeps a lane-0 TMA issuer: the converged version measured neutral)."""
    for name, body in _find(_sass(), "prefill_attention_kernel").items():
        lines = [l for l in body.splitlines() if "/*" in l and not l.strip().startswith("/* 0x")]
        for i, l in enumerate(lines):
            if re.search(r"\b(UTCHMMA|UTCBAR)\b", l):
                assert not any("BRA.U.ANY" in x for x in lines[i + 1:i + 5]), (name, l.strip())
