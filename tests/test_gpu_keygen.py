"""The harness generator kernel (csrc/keygen.cu) is bit-identical to the shared
NumPy generator (baton_inputs/keygen.py) -- so GPU-generated q/k/v are the very
inputs the oracle sees."""
import numpy as np
import pytest
import torch

from baton_inputs import query_history_bits, query_token_bits, KIND_Q, KIND_K, KIND_V
from gpu_util import bf16_bits, require_cuda

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale", [0, 1, 2])
def test_history_bits(scale):
    require_cuda()
    from paper_2410_18701_b200.baton import baton_keygen_history
    L, H, n, D = 3, 5, 37, 128
    out = torch.empty((L, H, n, D), dtype=torch.bfloat16, device="cuda")
    baton_keygen_history(out, L, H, D, 12345, 11, n, KIND_K, 18701, scale)
    ref = query_history_bits(18701, KIND_K, L, 12345, 11, 11 + n, H, D, scale)
    assert np.array_equal(bf16_bits(out), ref)


def test_history_strided_into_cache():
    require_cuda()
    from paper_2410_18701_b200.baton import baton_keygen_history
    L, B, H, S, D = 2, 3, 4, 64, 16
    cache = torch.zeros((L, B, H, S, D), dtype=torch.bfloat16, device="cuda")
    slot = 1
    view = cache[:, slot]
    baton_keygen_history(view, L, H, D, 7, 0, 20, KIND_V, 99, 0,
                         head_stride=S * D, layer_stride=B * H * S * D)
    ref = query_history_bits(99, KIND_V, L, 7, 0, 20, H, D, 0)
    assert np.array_equal(bf16_bits(cache[:, slot, :, :20]), ref)
    assert not cache[:, slot, :, 20:].any() and not cache[:, 0].any()


def test_token_bits():
    require_cuda()
    from paper_2410_18701_b200.baton import baton_keygen_tokens
    L, B, H, D = 4, 6, 8, 64
    qids = np.array([3, -1, 70000, 5, 0, 1048575], np.int32)
    pos = np.array([0, 9, 4095, 17, 2, 100], np.int32)
    out = torch.empty((L, B, H, D), dtype=torch.bfloat16, device="cuda")
    baton_keygen_tokens(out, torch.from_numpy(qids).cuda(), torch.from_numpy(pos).cuda(), L, B, H,
                        D, KIND_Q, 0, 2410, 2)
    got = bf16_bits(out)
    for l in range(L):
        ref = query_token_bits(2410, KIND_Q, l, np.maximum(qids, 0), pos, H, D, 2)
        ref[qids < 0] = 0
        assert np.array_equal(got[l], ref)
