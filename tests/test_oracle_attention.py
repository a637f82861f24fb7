"""Pins for O-1 (oracle/attention.py) against things other than itself.

P:L37 (§2.1) defines the operation; these tests pin the oracle to a library
routine (torch SDPA in float64), to closed forms and to special cases
(SURVEY.md §8(c) pin P4)."""
import math

import numpy as np
import pytest
import torch

from oracle import solo_attention, solo_attention_exact


def _rand(rng, *shape, s=1.0):
    return rng.uniform(-s, s, size=shape)


def _sdpa_ref(q, K, V):
    """torch.nn.functional.scaled_dot_product_attention, float64 CPU (library routine).
    GQA by contiguous head groups (reading C11)."""
    H_q, D = q.shape
    H_kv = K.shape[0]
    rep = H_q // H_kv
    Kt = torch.from_numpy(K).repeat_interleave(rep, dim=0)
    Vt = torch.from_numpy(V).repeat_interleave(rep, dim=0)
    qt = torch.from_numpy(q)[:, None, :]
    o = torch.nn.functional.scaled_dot_product_attention(qt, Kt, Vt)
    return o[:, 0, :].numpy()


@pytest.mark.parametrize("H_q,H_kv,D,n", [(2, 2, 16, 1), (2, 2, 16, 37), (4, 2, 128, 300),
                                          (8, 1, 128, 64), (64, 8, 128, 5), (32, 32, 128, 513)])
def test_matches_torch_sdpa(H_q, H_kv, D, n):
    rng = np.random.default_rng(n * 7 + D)
    q, K, V = _rand(rng, H_q, D), _rand(rng, H_kv, n, D), _rand(rng, H_kv, n, D)
    o = solo_attention(q, K, V)
    ref = _sdpa_ref(q, K, V)
    np.testing.assert_allclose(o, ref, rtol=1e-12, atol=1e-14)


def test_exact_variant_matches():
    rng = np.random.default_rng(1)
    q, K, V = _rand(rng, 4, 16, s=3), _rand(rng, 2, 29, 16, s=2), _rand(rng, 2, 29, 16)
    np.testing.assert_allclose(solo_attention_exact(q, K, V), solo_attention(q, K, V),
                               rtol=1e-13, atol=1e-15)


def test_single_key_returns_value_exactly():
    rng = np.random.default_rng(2)
    q, K, V = _rand(rng, 4, 128), _rand(rng, 4, 1, 128), _rand(rng, 4, 1, 128)
    o = solo_attention(q, K, V)
    assert np.array_equal(o, V[:, 0, :])          # softmax of one logit is exactly 1


def test_zero_query_gives_mean_of_values():
    rng = np.random.default_rng(3)
    K, V = _rand(rng, 2, 50, 16), _rand(rng, 2, 50, 16)
    o = solo_attention(np.zeros((2, 16)), K, V)
    np.testing.assert_allclose(o, V.mean(axis=1), rtol=1e-14, atol=1e-15)


def test_equal_keys_give_mean_of_values():
    rng = np.random.default_rng(4)
    k = _rand(rng, 16)
    K = np.broadcast_to(k, (1, 9, 16)).copy()
    V = _rand(rng, 1, 9, 16)
    o = solo_attention(_rand(rng, 1, 16), K, V)
    np.testing.assert_allclose(o[0], V[0].mean(axis=0), rtol=1e-14, atol=1e-15)


def test_constant_values_give_constant():
    rng = np.random.default_rng(5)
    V = np.full((2, 40, 16), 0.375)
    o = solo_attention(_rand(rng, 2, 16, s=4), _rand(rng, 2, 40, 16, s=4), V)
    np.testing.assert_allclose(o, 0.375, rtol=4e-16, atol=0)


def test_dominant_logit_selects_its_value():
    rng = np.random.default_rng(6)
    D = 16
    K = _rand(rng, 1, 20, D)
    q = np.zeros((1, D))
    q[0, 0] = 400.0
    K[0, :, 0] = 0.0
    K[0, 7, 0] = 1.0                       # logit 100 vs 0 elsewhere
    V = _rand(rng, 1, 20, D)
    o = solo_attention(q, K, V)
    np.testing.assert_allclose(o[0], V[0, 7], rtol=0, atol=1e-40 + 20 * math.exp(-100) * 2)


def test_two_keys_closed_form():
    # softmax of two logits a, b: weight of the first = 1 / (1 + exp(b - a))
    D = 4
    q = np.array([[2.0, 0, 0, 0]])
    K = np.array([[[1.0, 0, 0, 0], [-0.5, 0, 0, 0]]])
    V = np.array([[[1.0, 2.0, 3.0, 4.0], [-1.0, 0.0, 1.0, 0.5]]])
    a, b = 2.0 / 2.0, -1.0 / 2.0
    w = 1.0 / (1.0 + math.exp(b - a))
    ref = w * V[0, 0] + (1 - w) * V[0, 1]
    np.testing.assert_allclose(solo_attention(q, K, V)[0], ref, rtol=1e-15, atol=1e-15)


def test_key_permutation_invariance_exact():
    rng = np.random.default_rng(7)
    q, K, V = _rand(rng, 2, 16), _rand(rng, 2, 11, 16), _rand(rng, 2, 11, 16)
    perm = rng.permutation(11)
    assert np.array_equal(solo_attention_exact(q, K, V),
                          solo_attention_exact(q, K[:, perm], V[:, perm]))


def test_gqa_head_mapping_contiguous_groups():
    # head h of 8 reads kv head h // 4 when H_kv = 2 (C11): give the kv heads
    # different constant values and check which one each q head sees
    K = np.zeros((2, 3, 16))
    V = np.stack([np.full((3, 16), 1.0), np.full((3, 16), 2.0)])
    o = solo_attention(np.ones((8, 16)), K, V)
    assert np.array_equal(o[:, 0], np.array([1, 1, 1, 1, 2, 2, 2, 2], dtype=np.float64))


def test_empty_history_is_a_contract_violation():
    with pytest.raises(ValueError):
        solo_attention(np.zeros((1, 4)), np.zeros((1, 0, 4)), np.zeros((1, 0, 4)))
