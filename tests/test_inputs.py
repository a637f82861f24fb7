"""Pins for the shared seeded generators (baton_inputs): the splitmix64 finaliser
against its published first output, the vectorised generator against a
pure-Python big-integer re-derivation, bf16 RNE against torch's own rounding,
and the workload mixes against the paper's dataset description."""
import numpy as np
import torch

from baton_inputs import (PHI, mix64, keyed_u64, keyed_f32, keyed_bf16_bits, f32_to_bf16_bits,
                          bf16_bits_to_f64, query_history_bits, config_workload, w1_workload)


def test_splitmix64_reference_vector():
    # splitmix64 seeded with 0: first output = mix(0 + PHI) = 0xE220A8397B1DCDAF
    assert int(mix64(np.uint64(PHI))) == 0xE220A8397B1DCDAF
    # second output = mix(2*PHI mod 2^64) = 0x6E789E6AA1B965F4
    assert int(mix64(np.uint64((2 * PHI) % 2**64))) == 0x6E789E6AA1B965F4


def _py_u64(seed, kind, layer, qid, pos, head, dim):
    M = 2**64
    c = (((((kind * 128 + layer) * 2**20 + qid) * 4096 + pos) * 64 + head) * 128 + dim)
    z = (seed * PHI + c) % M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % M
    return z ^ (z >> 31)


def test_vectorised_matches_bigint():
    rng = np.random.default_rng(0)
    for _ in range(200):
        args = (int(rng.integers(0, 2**31)), int(rng.integers(0, 3)), int(rng.integers(0, 128)),
                int(rng.integers(0, 2**20)), int(rng.integers(0, 4096)), int(rng.integers(0, 64)),
                int(rng.integers(0, 128)))
        assert int(keyed_u64(*args)) == _py_u64(*args)
        u = _py_u64(*args)
        x = ((u >> 40) - 2**23) * 2.0**(1 - 23)
        assert float(keyed_f32(*args, 1)) == x


def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(100000).astype(np.float32) * np.float32(3.0)
    ours = f32_to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    back = bf16_bits_to_f64(ours)
    assert np.array_equal(back, torch.from_numpy(x).to(torch.bfloat16).double().numpy())


def test_value_range_and_spread():
    v = keyed_f32(18701, 1, 0, 5, np.arange(4096)[:, None], 0, np.arange(128)[None, :], 0)
    assert v.min() >= -1.0 and v.max() < 1.0
    assert abs(v.std() - 1 / np.sqrt(3)) < 0.01


def test_history_layout():
    h = query_history_bits(7, 1, 2, 9, 3, 6, 4, 16, 0)
    assert h.shape == (2, 4, 3, 16)
    assert h[1, 2, 1, 5] == keyed_bf16_bits(7, 1, 1, 9, 4, 2, 5, 0)


def test_workload_mix_and_bounds():
    wl = config_workload("7b")
    kinds = [q.kind for q in wl.queries]
    frac = {k: kinds.count(k) / len(kinds) for k in set(kinds)}
    assert abs(frac["SI-SO"] - 0.5) < 0.06 and abs(frac["LI-SO"] - 0.25) < 0.06
    assert all(q.l_q + q.A <= wl.max_ctx for q in wl.queries)
    assert sum(q.arrival == 0 for q in wl.queries) >= 32
    w70 = config_workload("70b")
    assert all(q.l_q + q.A <= 4096 and q.A >= 1 for q in w70.queries)
    assert sum(q.A for q in w1_workload().queries) == 71
