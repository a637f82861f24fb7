"""Shared helpers for the -m gpu parity tests (tolerances, comparisons)."""
import numpy as np
import torch

# SURVEY.md C13 / north_star: attention within max relative error 1e-2 per
# (slot, q-head) row: ||o_gpu - o_ref||_inf / ||o_ref||_inf.  Expected ~2^-9 (bf16
# output rounding, fp32 accumulation), so 1e-2 has ~5x headroom.
ATTN_RTOL = 1e-2


def bf16_bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def bits_to_f64(bits):
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


def row_rel_err(o_gpu, o_ref):
    """max over rows of ||gpu - ref||_inf / ||ref||_inf (rows = last axis)."""
    o_gpu = np.asarray(o_gpu, dtype=np.float64)
    o_ref = np.asarray(o_ref, dtype=np.float64)
    num = np.abs(o_gpu - o_ref).max(axis=-1)
    den = np.abs(o_ref).max(axis=-1)
    den = np.where(den == 0, 1.0, den)
    return float((num / den).max()) if num.size else 0.0


def require_cuda():
    import pytest
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
