"""a3 parity: baton_decode_attention (CUDA, through the C ABI) vs the oracle's
O-1 solo attention in fp64, on seeded states with ragged live lengths that span
several 64-key tiles and 256-key split-K chunks, NaN-poisoned placeholders,
interior mask holes, empty slots and the special cases that must be bit-exact."""
import math

import numpy as np
import pytest
import torch

from oracle import solo_attention
from gpu_util import ATTN_RTOL, bf16_bits, bits_to_f64, row_rel_err, require_cuda

pytestmark = pytest.mark.gpu


def _state(seed, B, Hq, Hkv, D, S_cap, lens, holes=0.0, scale_k=1.0):
    from paper_2410_18701_b200.baton import make_shape, baton_decode_workspace_bytes
    rng = np.random.default_rng(seed)
    lens = np.asarray(lens, dtype=np.int64)
    S = int(lens.max()) if lens.size else 0
    pad = np.where(lens > 0, S - lens, 0)
    mask = np.zeros((B, S_cap), np.uint8)
    K = np.full((B, Hkv, S_cap, D), np.nan, np.float32)
    V = np.full((B, Hkv, S_cap, D), np.nan, np.float32)
    for b in range(B):
        n = lens[b]
        if n == 0:
            continue
        mask[b, pad[b]:S] = 1
        K[b, :, :n] = rng.uniform(-scale_k, scale_k, (Hkv, n, D))
        V[b, :, :n] = rng.uniform(-1, 1, (Hkv, n, D))
        if holes and n > 2:
            hole = rng.random(n) < holes
            hole[rng.integers(0, n)] = False
            mask[b, pad[b]:S][hole] = 0
            K[b, :, np.nonzero(hole)[0]] = np.nan    # a masked column is never used
            V[b, :, np.nonzero(hole)[0]] = np.nan
    q = rng.uniform(-1, 1, (B, Hq, D)).astype(np.float32)
    dev = "cuda"
    t = lambda a: torch.from_numpy(a).to(dev).to(torch.bfloat16)
    st = dict(q=t(q), k=t(K), v=t(V), mask=torch.from_numpy(mask).to(dev),
              lens=torch.from_numpy(lens.astype(np.int32)).to(dev),
              pad=torch.from_numpy(pad.astype(np.int32)).to(dev),
              lens_h=lens, pad_h=pad, mask_h=mask, B=B, Hq=Hq, Hkv=Hkv, D=D, S_cap=S_cap)
    st["shape"] = make_shape(1, B, Hq, Hkv, D, S_cap)
    st["ws"] = torch.zeros(baton_decode_workspace_bytes(st["shape"]), dtype=torch.uint8, device=dev)
    return st


def _run(st, use_mask=True, out=None):
    from paper_2410_18701_b200.baton import baton_decode_attention
    if out is None:
        out = torch.full((st["B"], st["Hq"], st["D"]), float("nan"), dtype=torch.bfloat16,
                         device="cuda")
    baton_decode_attention(st["q"], st["k"], st["v"], st["mask"] if use_mask else None,
                           st["lens"], st["pad"], out, st["shape"], 1.0 / math.sqrt(st["D"]),
                           st["ws"])
    torch.cuda.synchronize()
    return out


def _reference(st):
    q = bits_to_f64(bf16_bits(st["q"]))
    K = bits_to_f64(bf16_bits(st["k"]))
    V = bits_to_f64(bf16_bits(st["v"]))
    ref = np.zeros((st["B"], st["Hq"], st["D"]))
    for b in range(st["B"]):
        n = st["lens_h"][b]
        if n == 0:
            continue
        live = np.nonzero(st["mask_h"][b, st["pad_h"][b]:st["pad_h"][b] + n])[0]
        ref[b] = solo_attention(q[b], K[b][:, live], V[b][:, live])
    return ref


CASES = [
    # (B, Hq, Hkv, D, S_cap, lens)
    (4, 2, 2, 16, 64, [5, 0, 64, 17]),
    (3, 4, 2, 32, 512, [1, 300, 513 - 1]),
    (5, 8, 1, 64, 1024, [257, 256, 255, 1000, 0]),
    (6, 4, 4, 128, 1024, [1, 63, 64, 65, 511, 1024]),
    (8, 32, 32, 128, 2048, [2048, 1500, 900, 256, 257, 31, 0, 1100]),
    (4, 64, 8, 128, 4096, [4096, 3000, 129, 1]),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_matches_oracle(case):
    require_cuda()
    B, Hq, Hkv, D, S_cap, lens = CASES[case]
    st = _state(case, B, Hq, Hkv, D, S_cap, lens)
    out = _run(st)
    ref = _reference(st)
    got = bits_to_f64(bf16_bits(out))
    for b in range(B):
        if st["lens_h"][b] == 0:
            assert not np.any(got[b]), "empty slot must give a zero row"
    assert row_rel_err(got, ref) <= ATTN_RTOL
    assert np.isfinite(got).all()


@pytest.mark.parametrize("seed", range(4))
def test_interior_mask_holes_are_skipped(seed):
    require_cuda()
    st = _state(100 + seed, 6, 4, 2, 128, 1024, [900, 600, 37, 300, 1024, 2], holes=0.3)
    got = bits_to_f64(bf16_bits(_run(st)))
    assert np.isfinite(got).all()           # NaN-poisoned masked columns never contribute
    assert row_rel_err(got, _reference(st)) <= ATTN_RTOL


def test_peaky_logits():
    require_cuda()
    st = _state(7, 4, 8, 8, 128, 2048, [2000, 700, 256, 1], scale_k=8.0)
    got = bits_to_f64(bf16_bits(_run(st)))
    assert row_rel_err(got, _reference(st)) <= ATTN_RTOL


def test_single_key_returns_value_bitwise():
    require_cuda()
    st = _state(11, 3, 8, 2, 128, 256, [1, 1, 1])
    out = bf16_bits(_run(st))
    vbits = bf16_bits(st["v"])
    for b in range(3):
        for h in range(8):
            assert np.array_equal(out[b, h], vbits[b, h * 2 // 8, 0])


def test_no_mask_equals_suffix_mask():
    require_cuda()
    st = _state(12, 5, 4, 4, 64, 512, [400, 1, 0, 257, 99])
    a = bf16_bits(_run(st, use_mask=True))
    b = bf16_bits(_run(st, use_mask=False))
    assert np.array_equal(a, b)


def test_repeat_calls_reuse_workspace_bitwise():
    require_cuda()
    st = _state(13, 8, 32, 32, 128, 2048, [2048, 1024, 1000, 3, 600, 1800, 256, 512])
    a = bf16_bits(_run(st))
    for _ in range(3):
        assert np.array_equal(a, bf16_bits(_run(st)))
    assert not st["ws"][:4 * 8 * 32].any()        # split-K tickets returned to zero


def test_batch_invariance_bitwise():
    """A query's output does not depend on the slot it occupies nor on the other
    queries of the batch (fixed live-relative chunking, P:L98 independence)."""
    require_cuda()
    st1 = _state(14, 4, 8, 8, 128, 2048, [1300, 2000, 5, 700])
    o1 = bf16_bits(_run(st1))
    # move slot 0's content to slot 2 of a different batch with other lengths
    st2 = _state(15, 3, 8, 8, 128, 2048, [100, 50, 1300])
    for name in ("q", "k", "v"):
        st2[name][2] = st1[name][0]
    torch.cuda.synchronize()
    o2 = bf16_bits(_run(st2))
    assert np.array_equal(o1[0], o2[2])


def test_invalid_arguments():
    require_cuda()
    from paper_2410_18701_b200 import _lib
    from paper_2410_18701_b200.baton import baton_decode_attention, make_shape, BatonError
    st = _state(16, 2, 2, 2, 16, 64, [3, 4])
    with pytest.raises(BatonError):
        baton_decode_attention(st["q"], st["k"], st["v"], st["mask"], st["lens"], st["pad"],
                               st["q"].clone(), make_shape(1, 2, 2, 2, 96, 64), 0.25, st["ws"])
    with pytest.raises(BatonError):
        baton_decode_attention(st["q"], st["k"], st["v"], st["mask"], st["lens"], st["pad"],
                               st["q"].clone(), st["shape"], 0.25, st["ws"][:8])


GQA_CASES = [
    # tensor-core GQA path (8 q heads per kv head, head_dim 128)
    (3, 8, 1, 128, 512, [1, 200, 512]),
    (6, 16, 2, 128, 1024, [64, 65, 256, 257, 1000, 0]),
    (4, 64, 8, 128, 4096, [4096, 2049, 300, 17]),
]


@pytest.mark.parametrize("case", range(len(GQA_CASES)))
def test_gqa_matches_oracle(case):
    require_cuda()
    B, Hq, Hkv, D, S_cap, lens = GQA_CASES[case]
    st = _state(200 + case, B, Hq, Hkv, D, S_cap, lens)
    got = bits_to_f64(bf16_bits(_run(st)))
    assert np.isfinite(got).all()
    assert row_rel_err(got, _reference(st)) <= ATTN_RTOL


def test_gqa_holes_and_peaky():
    require_cuda()
    st = _state(210, 5, 16, 2, 128, 2048, [1800, 3, 900, 257, 640], holes=0.25, scale_k=6.0)
    got = bits_to_f64(bf16_bits(_run(st)))
    assert np.isfinite(got).all()
    assert row_rel_err(got, _reference(st)) <= ATTN_RTOL


def test_gqa_batch_invariance_and_single_key():
    require_cuda()
    st1 = _state(211, 3, 16, 2, 128, 2048, [1500, 1, 600])
    o1 = bf16_bits(_run(st1))
    vb = bf16_bits(st1["v"])
    for h in range(16):
        assert np.array_equal(o1[1, h], vb[1, h // 8, 0])     # one live key: o = v exactly
    st2 = _state(212, 4, 16, 2, 128, 2048, [20, 1500, 2048, 7])
    for name in ("q", "k", "v"):
        st2[name][1] = st1[name][0]
    torch.cuda.synchronize()
    o2 = bf16_bits(_run(st2))
    assert np.array_equal(o1[0], o2[1])
