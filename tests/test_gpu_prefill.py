"""a8 parity: baton_prefill_attention (tcgen05/TMEM/TMA kernel, through the C ABI)
vs the oracle.  Causal prefill attention of a prompt is, for every position i,
the decode attention of the prefix [0, i] -- O-1 applied position by position
(P:L132 prefilled queries), so no separate oracle function is needed."""
import math

import numpy as np
import pytest
import torch

from oracle import solo_attention
from gpu_util import ATTN_RTOL, bf16_bits, bits_to_f64, row_rel_err, require_cuda

pytestmark = pytest.mark.gpu


def _case(seed, Hq, Hkv, n, D=128, scale_k=1.0):
    rng = np.random.default_rng(seed)
    t = lambda a: torch.from_numpy(a.astype(np.float32)).cuda().to(torch.bfloat16)
    Q = t(rng.uniform(-1, 1, (Hq, n, D)))
    K = t(rng.uniform(-scale_k, scale_k, (Hkv, n, D)))
    V = t(rng.uniform(-1, 1, (Hkv, n, D)))
    return Q, K, V


def _reference(Q, K, V, rows):
    q = bits_to_f64(bf16_bits(Q))
    k = bits_to_f64(bf16_bits(K))
    v = bits_to_f64(bf16_bits(V))
    return {i: solo_attention(q[:, i], k[:, :i + 1], v[:, :i + 1]) for i in rows}


@pytest.mark.parametrize("Hq,Hkv,n", [(2, 2, 1), (2, 2, 5), (4, 4, 127), (4, 4, 128), (4, 2, 129),
                                      (8, 1, 300), (8, 8, 700), (32, 32, 260), (64, 8, 200)])
def test_prefill_matches_oracle(Hq, Hkv, n):
    require_cuda()
    from paper_2410_18701_b200.baton import baton_prefill_attention
    Q, K, V = _case(n * 31 + Hq, Hq, Hkv, n)
    O = torch.full_like(Q, float("nan"))
    baton_prefill_attention(Q, K, V, O, n, Hq, Hkv, 128)
    torch.cuda.synchronize()
    got = bits_to_f64(bf16_bits(O))
    assert np.isfinite(got).all()
    rows = sorted(set([0, n - 1, n // 2] + list(np.random.default_rng(n).integers(0, n, 24))))
    ref = _reference(Q, K, V, rows)
    worst = max(row_rel_err(got[:, i], ref[i]) for i in rows)
    assert worst <= ATTN_RTOL, worst


def test_prefill_first_row_is_first_value():
    """Row 0 attends only to key 0: o = v_0 (up to bf16 of P = 1 exactly)."""
    require_cuda()
    from paper_2410_18701_b200.baton import baton_prefill_attention
    Q, K, V = _case(5, 4, 4, 200)
    O = torch.empty_like(Q)
    baton_prefill_attention(Q, K, V, O, 200, 4, 4, 128)
    torch.cuda.synchronize()
    assert np.array_equal(bf16_bits(O)[:, 0], bf16_bits(V)[:, 0])


def test_prefill_last_row_equals_decode_attention():
    """The last prefill row is the decode attention of the full prompt (a3)."""
    require_cuda()
    from paper_2410_18701_b200.baton import (baton_prefill_attention, baton_decode_attention,
                                             make_shape, baton_decode_workspace_bytes)
    n, H = 400, 8
    Q, K, V = _case(6, H, H, n, scale_k=4.0)
    O = torch.empty_like(Q)
    baton_prefill_attention(Q, K, V, O, n, H, H, 128)
    S_cap = 512
    kc = torch.zeros((1, H, S_cap, 128), dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    kc[0, :, :n] = K
    vc[0, :, :n] = V
    shape = make_shape(1, 1, H, H, 128, S_cap)
    ws = torch.zeros(baton_decode_workspace_bytes(shape), dtype=torch.uint8, device="cuda")
    od = torch.empty((1, H, 128), dtype=torch.bfloat16, device="cuda")
    lens = torch.tensor([n], dtype=torch.int32, device="cuda")
    pad = torch.zeros(1, dtype=torch.int32, device="cuda")
    baton_decode_attention(Q[:, n - 1][None].contiguous(), kc, vc, None, lens, pad, od, shape,
                           1 / math.sqrt(128), ws)
    torch.cuda.synchronize()
    a = bits_to_f64(bf16_bits(O[:, n - 1]))
    b = bits_to_f64(bf16_bits(od[0]))
    assert row_rel_err(a, b) <= ATTN_RTOL


def _packed(seed, Hq, Hkv, lens, D=128):
    T = int(sum(lens))
    return _case(seed, Hq, Hkv, T, D)


@pytest.mark.parametrize("Hq,Hkv,lens", [(4, 2, [1, 5, 127, 128, 129, 300]), (8, 1, [700, 33, 256, 129]),
                                         (64, 8, [200, 1, 65])])
def test_prefill_varlen_matches_oracle(Hq, Hkv, lens):
    """NEXT-2 batched prefill: every packed prompt is its own causal problem (O-1 per
    prefix of that prompt); nothing crosses prompt boundaries."""
    require_cuda()
    from paper_2410_18701_b200.baton import baton_prefill_attention_varlen
    Q, K, V = _packed(sum(lens) + Hq, Hq, Hkv, lens)
    O = torch.full_like(Q, float("nan"))
    baton_prefill_attention_varlen(Q, K, V, O, lens, Hq, Hkv, 128)
    torch.cuda.synchronize()
    got = bits_to_f64(bf16_bits(O))
    assert np.isfinite(got).all()
    s0 = 0
    worst = 0.0
    for n in lens:
        sl = slice(s0, s0 + n)
        rows = sorted(set([0, n - 1, n // 2] + list(np.random.default_rng(n).integers(0, n, 8))))
        ref = _reference(Q[:, sl], K[:, sl], V[:, sl], rows)
        worst = max(worst, max(row_rel_err(got[:, s0 + i], ref[i]) for i in rows))
        s0 += n
    assert worst <= ATTN_RTOL, worst


def test_prefill_varlen_equals_separate_calls_bitwise():
    require_cuda()
    from paper_2410_18701_b200.baton import baton_prefill_attention, baton_prefill_attention_varlen
    Hq, Hkv, lens = 8, 2, [700, 33, 256, 129, 1, 511]
    Q, K, V = _packed(77, Hq, Hkv, lens)
    O = torch.empty_like(Q)
    baton_prefill_attention_varlen(Q, K, V, O, lens, Hq, Hkv, 128)
    s0 = 0
    for n in lens:
        sl = slice(s0, s0 + n)
        o1 = torch.empty((Hq, n, 128), dtype=torch.bfloat16, device="cuda")
        baton_prefill_attention(Q[:, sl].contiguous(), K[:, sl].contiguous(), V[:, sl].contiguous(), o1, n,
                                Hq, Hkv, 128)
        torch.cuda.synchronize()
        assert np.array_equal(bf16_bits(O[:, sl]), bf16_bits(o1)), n
        s0 += n


def test_prefill_varlen_errors():
    require_cuda()
    from paper_2410_18701_b200.baton import baton_prefill_attention_varlen, BatonError
    Q, K, V = _case(1, 2, 2, 10)
    O = torch.empty_like(Q)
    for lens in ([4, 0, 6], [1] * 65, [10] * 0):
        with pytest.raises((BatonError, ValueError)):
            baton_prefill_attention_varlen(Q, K, V, O, lens, 2, 2, 128)


def test_prefill_varlen_max_prompts_bitwise():
    """The launch limits: 64 packed prompts (ragged, 1..300 tokens, tile-boundary
    lengths included), every one bit-identical to its own separate launch."""
    require_cuda()
    from paper_2410_18701_b200.baton import baton_prefill_attention, baton_prefill_attention_varlen
    rng = np.random.default_rng(64)
    lens = [1, 127, 128, 129, 256] + [int(x) for x in rng.integers(1, 300, 59)]
    Hq, Hkv = 8, 1
    Q, K, V = _packed(640, Hq, Hkv, lens)
    O = torch.empty_like(Q)
    baton_prefill_attention_varlen(Q, K, V, O, lens, Hq, Hkv, 128)
    s0 = 0
    for n in lens:
        sl = slice(s0, s0 + n)
        o1 = torch.empty((Hq, n, 128), dtype=torch.bfloat16, device="cuda")
        baton_prefill_attention(Q[:, sl].contiguous(), K[:, sl].contiguous(), V[:, sl].contiguous(), o1, n,
                                Hq, Hkv, 128)
        torch.cuda.synchronize()
        assert np.array_equal(bf16_bits(O[:, sl]), bf16_bits(o1)), n
        s0 += n


@pytest.fixture
def grid_cap():
    """Cap the persistent prefill grid (baton_debug_prefill_grid) so every CTA walks
    many work items: the Q reload, the K/V ring, the S buffers and the O hand-over run
    on across items (prefill_attention.cu, PfWalk)."""
    import ctypes
    from paper_2410_18701_b200 import _lib
    lib = _lib.lib
    lib.baton_debug_prefill_grid.restype = ctypes.c_int
    lib.baton_debug_prefill_grid.argtypes = [ctypes.c_int]
    yield lib.baton_debug_prefill_grid
    lib.baton_debug_prefill_grid(0)


@pytest.mark.parametrize("cap", [1, 3, 7])
def test_prefill_persistent_walk_bitwise(grid_cap, cap):
    """Which CTA runs an item, and after which items, never changes a bit: a varlen
    launch (ragged prompts, 1-token and tile-boundary lengths, GQA) on a grid of `cap`
    CTAs equals the default grid bitwise, and the oracle on sampled rows."""
    require_cuda()
    from paper_2410_18701_b200.baton import baton_prefill_attention_varlen
    Hq, Hkv, lens = 8, 2, [700, 1, 33, 256, 129, 128, 511, 64]
    Q, K, V = _packed(91, Hq, Hkv, lens)
    ref = torch.empty_like(Q)
    baton_prefill_attention_varlen(Q, K, V, ref, lens, Hq, Hkv, 128)
    grid_cap(cap)
    O = torch.full_like(Q, float("nan"))
    baton_prefill_attention_varlen(Q, K, V, O, lens, Hq, Hkv, 128)
    torch.cuda.synchronize()
    assert np.array_equal(bf16_bits(O), bf16_bits(ref))
    got = bits_to_f64(bf16_bits(O))
    s0, worst = 0, 0.0
    for n in lens:
        sl = slice(s0, s0 + n)
        rows = sorted({0, n - 1, n // 2})
        r = _reference(Q[:, sl], K[:, sl], V[:, sl], rows)
        worst = max(worst, max(row_rel_err(got[:, s0 + i], r[i]) for i in rows))
        s0 += n
    assert worst <= ATTN_RTOL, worst


def test_prefill_varlen_config_mix_panels():
    """The bench's prefill leg: the 7B config's first 64 prompts in ONE varlen launch
    (31k tokens, 508 MB of K/V: the work list runs in several 64 MB L2 panels, DESIGN
    §6.3).  Every prompt's rows equal its own single-prompt launch bitwise (one panel,
    round-1 order) for a sample of prompts, and the oracle (O-1 per prefix) on sampled
    rows and heads."""
    require_cuda()
    from baton_inputs import config_workload
    from paper_2410_18701_b200.baton import baton_prefill_attention, baton_prefill_attention_varlen
    lens = [q.l_q for q in config_workload("7b").queries[:64]]
    Hq = Hkv = 32
    T = sum(lens)
    assert 4 * T * Hkv * 128 > 4 * (64 << 20)          # spans several panels
    g = torch.Generator(device="cuda").manual_seed(64)
    mk = lambda H: (torch.rand((H, T, 128), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    Q, K, V = mk(Hq), mk(Hkv), mk(Hkv)
    O = torch.full_like(Q, float("nan"))
    baton_prefill_attention_varlen(Q, K, V, O, lens, Hq, Hkv, 128)
    torch.cuda.synchronize()
    starts = np.concatenate([[0], np.cumsum(lens)])
    order = sorted(range(64), key=lambda i: -lens[i])
    sample = sorted({order[0], order[1], order[31], order[32], order[62], order[63], 0, 17})
    worst = 0.0
    for i in sample:
        n, s0 = lens[i], int(starts[i])
        sl = slice(s0, s0 + n)
        q1, k1, v1 = Q[:, sl].contiguous(), K[:, sl].contiguous(), V[:, sl].contiguous()
        o1 = torch.empty_like(q1)
        baton_prefill_attention(q1, k1, v1, o1, n, Hq, Hkv, 128)
        torch.cuda.synchronize()
        assert np.array_equal(bf16_bits(O[:, sl]), bf16_bits(o1)), i
        heads = [0, 13, 31]
        rows = sorted({0, n // 3, n - 1})
        ref = _reference(q1[heads], k1[heads], v1[heads], rows)
        got = bits_to_f64(bf16_bits(O[heads][:, sl]))
        worst = max(worst, max(row_rel_err(got[:, r], ref[r]) for r in rows))
    assert worst <= ATTN_RTOL, worst
