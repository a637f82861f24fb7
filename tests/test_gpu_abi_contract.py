"""The ABI's error contract on the GPU (include/baton.h: "a failing call leaves
host and device state unchanged"), large-max_ctx mask splices, and the
standalone a2 export ``baton_append_kv`` against the oracle.

* Every splice call whose launch is refused (test-only fault injection,
  ``baton_debug_fail_launch``) returns BATON_E_CUDA and leaves the host mirror,
  the device metadata and the mask bytes exactly as they were; the same call then
  succeeds and the state matches the oracle's Shard.
* max_ctx = 32768 and 65536: remove / release / insert / expansion produce the
  paper's mask (closed form P1: mask[b][j] = occ_b and j >= pad_b) -- the mask
  splice stages a 64 KB row in shared memory.
* baton_append_kv ("appends ... to KV_Cache") writes row lens-1 of every
  occupied slot, bit for bit, and the stateless decode attention over the result
  equals O-1 solo attention within C13."""
import ctypes
import math

import numpy as np
import pytest
import torch

from oracle import Shard, solo_attention
from gpu_util import ATTN_RTOL, bf16_bits, bits_to_f64, row_rel_err, require_cuda

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2410_18701_b200 import _lib
    f = _lib.lib.baton_debug_fail_launch
    f.restype, f.argtypes = ctypes.c_int, [ctypes.c_int]
    return _lib


def _snapshot(sh):
    torch.cuda.synchronize()
    m = sh.baton_query()
    return (m["S"], m["pad"].tolist(), m["lens"].tolist(), m["occ"].tolist(),
            int(sh.d_S.item()), sh.d_lens.cpu().tolist(), sh.d_pad.cpu().tolist(),
            sh.mask.cpu().numpy().copy())


def _same(a, b):
    return a[:7] == b[:7] and np.array_equal(a[7], b[7])


def _kv(rng, L, H, n, D):
    return torch.from_numpy(rng.uniform(-1, 1, (L, H, n, D)).astype(np.float32)).cuda().to(torch.bfloat16)


def _f64(t):
    return bits_to_f64(bf16_bits(t))


def _check_vs_oracle(sh, osh):
    m = sh.baton_query()
    occ = osh.qid >= 0
    assert m["S"] == osh.S
    assert np.array_equal(m["lens"], osh.lens())
    assert np.array_equal(np.where(occ, m["pad"], 0), np.where(occ, osh.pad, 0))
    dm = sh.mask.cpu().numpy()
    assert np.array_equal(dm[:, :osh.S], osh.mask)
    assert not dm[:, osh.S:].any()


@pytest.mark.parametrize("op", ["remove", "insert_expand", "insert_end", "compact", "remove_release"])
def test_refused_launch_leaves_state_unchanged(op):
    require_cuda()
    L_ = _lib()
    from paper_2410_18701_b200.baton import BatonShard, BatonError
    rng = np.random.default_rng(5)
    L, B, H, D, cap = 2, 4, 2, 16, 128
    sh = BatonShard(L, B, H, H, D, cap)
    osh = Shard(B, L, H, H, D, cap, kv=True, fill=np.nan)
    kvs = {}
    for b, n in [(0, 10), (1, 17), (3, 6)]:
        K, V = _kv(rng, L, H, n, D), _kv(rng, L, H, n, D)
        kvs[b] = (K, V)
        sh.baton_insert(b, K, V, n)
        osh.insert(b, b, n, _f64(K), _f64(V))
    _check_vs_oracle(sh, osh)
    Kn, Vn = _kv(rng, L, H, 40, D), _kv(rng, L, H, 40, D)
    Ks, Vs = _kv(rng, L, H, 5, D), _kv(rng, L, H, 5, D)
    calls = {
        "remove": (lambda: sh.baton_remove([3]), lambda: (osh.remove(3), osh.release())),
        "remove_release": (lambda: sh.baton_remove([1]), lambda: (osh.remove(1), osh.release())),
        "insert_expand": (lambda: sh.baton_insert(2, Kn, Vn, 40),
                          lambda: osh.insert(2, 9, 40, _f64(Kn), _f64(Vn))),
        "insert_end": (lambda: sh.baton_insert(2, Ks, Vs, 5),
                       lambda: osh.insert(2, 9, 5, _f64(Ks), _f64(Vs))),
        "compact": (lambda: sh.baton_compact(3), lambda: osh.compact(3)),
    }
    call, oracle_call = calls[op]
    before = _snapshot(sh)
    L_.lib.baton_debug_fail_launch(1)
    with pytest.raises(BatonError) as e:
        call()
    L_.lib.baton_debug_fail_launch(0)
    assert e.value.code == L_.BATON_E_CUDA
    assert _same(_snapshot(sh), before), op
    # the same call now succeeds and gives the paper's state
    call()
    oracle_call()
    torch.cuda.synchronize()
    _check_vs_oracle(sh, osh)
    for b in np.nonzero(osh.qid >= 0)[0]:
        Ko, Vo = osh.live_kv(b)
        Kd, Vd = sh.live_kv(b)
        assert np.array_equal(_f64(Kd), Ko) and np.array_equal(_f64(Vd), Vo)


def test_refused_shape_step_leaves_state_unchanged():
    require_cuda()
    L_ = _lib()
    from paper_2410_18701_b200.baton import BatonShard, BatonError
    L, B, H, D, cap, W = 1, 2, 2, 128, 256, 8
    sh = BatonShard(L, B, H, H, D, cap)
    K = torch.randn((L, H, 12, D), device="cuda").to(torch.bfloat16)
    sh.baton_insert(0, K, K, 12)
    q = torch.randn((L, B, W, H, D), device="cuda").to(torch.bfloat16)
    kn = torch.randn((L, B, W, H, D), device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    before = _snapshot(sh)
    L_.lib.baton_debug_fail_launch(1)            # the mask splice of the shaped step
    with pytest.raises(BatonError):
        sh.baton_shape_step(W, [1], [W], q, kn, kn, out)
    L_.lib.baton_debug_fail_launch(0)
    assert _same(_snapshot(sh), before)
    sh.baton_shape_step(W, [1], [W], q, kn, kn, out)
    m = sh.baton_query()
    assert m["S"] == 12 + W and list(m["lens"]) == [12 + W, W]


@pytest.mark.parametrize("cap", [32768, 65536])
def test_large_max_ctx_mask_splice(cap):
    """the mask splice staged 2*max_ctx bytes of shared memory
    without opting in, so every splice failed above max_ctx 24576."""
    require_cuda()
    from paper_2410_18701_b200.baton import BatonShard
    L, B, H, D = 1, 3, 1, 16
    sh = BatonShard(L, B, H, H, D, cap)
    osh = Shard(B, L, H, H, D, cap, kv=False)
    rng = np.random.default_rng(1)
    steps = [("ins", 0, 100), ("ins", 1, cap - 40), ("ins", 2, 5000), ("rm", [1]), ("ins", 1, cap // 2),
             ("rm", [0, 2]), ("ins", 0, 3), ("rm", [1])]
    for st in steps:
        if st[0] == "ins":
            _, b, n = st
            K = torch.zeros((L, H, n, D), dtype=torch.bfloat16, device="cuda")
            sh.baton_insert(b, K, K, n)
            osh.insert(b, b, n)
        else:
            sh.baton_remove(st[1])
            for b in st[1]:
                osh.remove(b)
            osh.release()
        torch.cuda.synchronize()
        m = sh.baton_query()
        occ = m["occ"].astype(bool)
        closed = np.zeros((B, cap), np.uint8)
        for b in range(B):
            if occ[b]:
                closed[b, m["pad"][b]:m["S"]] = 1
        assert np.array_equal(sh.mask.cpu().numpy(), closed), st     # P1 closed form
        _check_vs_oracle(sh, osh)


@pytest.mark.parametrize("hq,hkv,D", [(2, 2, 16), (32, 32, 128), (8, 2, 64)])
def test_standalone_append_kv(hq, hkv, D):
    require_cuda()
    from paper_2410_18701_b200.baton import BatonShard
    rng = np.random.default_rng(hq + D)
    L, B, cap = 2, 5, 512
    sh = BatonShard(L, B, hq, hkv, D, cap)
    hist = {}
    lens = {0: 33, 2: 300, 3: 1, 4: 257}
    for b, n in lens.items():
        K, V = _kv(rng, L, hkv, n, D), _kv(rng, L, hkv, n, D)
        sh.baton_insert(b, K, V, n)
        hist[b] = (_f64(K), _f64(V))
    for it in range(2):
        sh.baton_mask_update()
        for l in range(L):
            kn = torch.from_numpy(rng.uniform(-1, 1, (B, hkv, D)).astype(np.float32)).cuda().to(torch.bfloat16)
            vn = torch.from_numpy(rng.uniform(-1, 1, (B, hkv, D)).astype(np.float32)).cuda().to(torch.bfloat16)
            sh.baton_append_kv(l, kn, vn)
            q = torch.from_numpy(rng.uniform(-1, 1, (B, hq, D)).astype(np.float32)).cuda().to(torch.bfloat16)
            out = torch.empty_like(q)
            sh.baton_decode_attention(l, q, out)
            torch.cuda.synchronize()
            kn64, vn64, q64, o = _f64(kn), _f64(vn), _f64(q), out.float().cpu().numpy()
            m = sh.baton_query()
            for b in range(B):
                if b not in lens:
                    assert (o[b] == 0).all()                               # C6
                    continue
                n = int(m["lens"][b])
                Kd, Vd = sh.live_kv(b)
                assert np.array_equal(bf16_bits(Kd[l, :, n - 1]), bf16_bits(kn[b]))   # row lens-1
                assert np.array_equal(bf16_bits(Vd[l, :, n - 1]), bf16_bits(vn[b]))
                ref = solo_attention(q64[b], _f64(Kd[l]), _f64(Vd[l]))
                assert row_rel_err(o[b], ref) <= ATTN_RTOL
                # the history before the append is untouched
                assert np.array_equal(_f64(Kd[l, :, :lens[b]]), hist[b][0][l])
