"""Counter-based value generator for synthetic q/k/v (SURVEY.md §8(d) "Generator").

Every value is a pure function of (seed, kind, layer, qid, pos, head, dim):

    ctr = (((((kind*128 + layer)*2**20 + qid)*4096 + pos)*64 + head)*128 + dim)
    u   = mix64(seed*PHI + ctr  mod 2**64)          (splitmix64 finaliser)
    x   = (int(u >> 40) - 2**23) * 2**(s - 23)       (exact in fp32, uniform in [-2**s, 2**s))
    bf16 = round-to-nearest-even(x)

so a query's K/V at a position is the same whether it was produced by the
prefill (embedded on insert) or by a decode step (appended,
PAPER.md L96), and the same after a preempt/re-insert round trip (L144).  The
CUDA harness implements the same generator in ``csrc/keygen.cu``; the two are
cross-checked bitwise in ``tests/test_gpu_keygen.py``.

No arithmetic of the Baton method lives here.
"""
import numpy as np

PHI = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
KIND_Q, KIND_K, KIND_V = 0, 1, 2

# (s_q, s_k, s_v) exponents: "flat" logits sigma ~ 0.33, "peaky" sigma ~ 2.7
SCALES_FLAT = (0, 0, 0)
SCALES_PEAKY = (2, 1, 0)

# field widths of the counter packing (55 bits in total)
MAX_LAYER, MAX_QID, MAX_POS, MAX_HEAD, MAX_DIM = 128, 1 << 20, 4096, 64, 128


def mix64(z):
    """splitmix64 output finaliser on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        z = z ^ (z >> np.uint64(31))
    return z


def _counter(kind, layer, qid, pos, head, dim):
    kind, layer, qid, pos, head, dim = (np.asarray(a, dtype=np.uint64)
                                        for a in (kind, layer, qid, pos, head, dim))
    if (np.any(layer >= MAX_LAYER) or np.any(qid >= MAX_QID) or np.any(pos >= MAX_POS)
            or np.any(head >= MAX_HEAD) or np.any(dim >= MAX_DIM)):
        raise ValueError("keygen field out of range")
    c = kind * np.uint64(MAX_LAYER) + layer
    c = c * np.uint64(MAX_QID) + qid
    c = c * np.uint64(MAX_POS) + pos
    c = c * np.uint64(MAX_HEAD) + head
    c = c * np.uint64(MAX_DIM) + dim
    return c


def keyed_u64(seed, kind, layer, qid, pos, head, dim):
    c = _counter(kind, layer, qid, pos, head, dim)
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * np.uint64(PHI)
        return mix64(base + c)


def keyed_f32(seed, kind, layer, qid, pos, head, dim, scale_exp):
    u = keyed_u64(seed, kind, layer, qid, pos, head, dim)
    ival = (u >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (ival.astype(np.float64) * 2.0 ** (scale_exp - 23)).astype(np.float32)


def f32_to_bf16_bits(x):
    """Round-to-nearest-even fp32 -> bf16 bit pattern (inputs are finite)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return rounded.astype(np.uint16)


def bf16_bits_to_f64(bits):
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


def keyed_bf16_bits(seed, kind, layer, qid, pos, head, dim, scale_exp):
    return f32_to_bf16_bits(keyed_f32(seed, kind, layer, qid, pos, head, dim, scale_exp))


def query_history_bits(seed, kind, n_layers, qid, pos_begin, pos_end, n_heads, head_dim,
                       scale_exp):
    """bf16 bits of one query's K (or V) for positions [pos_begin, pos_end).

    Layout [layer][head][pos][dim] -- the prefilled-query layout taken by
    ``baton_insert`` (include/baton.h)."""
    L = np.arange(n_layers, dtype=np.uint64)[:, None, None, None]
    H = np.arange(n_heads, dtype=np.uint64)[None, :, None, None]
    P = np.arange(pos_begin, pos_end, dtype=np.uint64)[None, None, :, None]
    Dd = np.arange(head_dim, dtype=np.uint64)[None, None, None, :]
    return keyed_bf16_bits(seed, kind, L, qid, P, H, Dd, scale_exp)


def query_token_bits(seed, kind, layer, qids, positions, n_heads, head_dim, scale_exp):
    """bf16 bits of the current token's q/k/v for a batch of slots.

    ``qids``/``positions`` are per-slot arrays; returns [slot][head][dim]."""
    Q = np.asarray(qids, dtype=np.uint64)[:, None, None]
    P = np.asarray(positions, dtype=np.uint64)[:, None, None]
    H = np.arange(n_heads, dtype=np.uint64)[None, :, None]
    Dd = np.arange(head_dim, dtype=np.uint64)[None, None, :]
    return keyed_bf16_bits(seed, kind, layer, Q, P, H, Dd, scale_exp)
