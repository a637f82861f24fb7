"""O-1: solo attention of one decoding query (TEST INFRASTRUCTURE ONLY).

P:L37 (§2.1 "General architecture"): "The relationship strength between elements
of X is evaluated by calculating the dot product between Q and K, and then
converted into attention weights through scaling and softmax operations.
Finally, these attention weights are multiplied by V, and through weighted
summation, an output is generated."

For a decode step ("the latest output token is enough as the input") the
query is one vector per head, the keys/values are the query's own cached history
including the token just appended (reading C3).  Scaling is 1/sqrt(D) (C10);
GQA head h reads kv-head floor(h*H_kv/H_q) (C11).

    s_j = (q . K_j) / sqrt(D);   o = sum_j softmax(s)_j V_j

computed in float64, max-subtracted, summed in ascending j.
"""
import math

import numpy as np


def _kv_head(h, H_q, H_kv):
    return (h * H_kv) // H_q


def solo_attention(q, K, V):
    """q: [H_q, D]; K, V: [H_kv, n, D] (float64, n >= 1). Returns o: [H_q, D]."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    H_q, D = q.shape
    H_kv, n, _ = K.shape
    if n < 1:
        raise ValueError("attention over an empty history (S:L51 contract violation)")
    out = np.empty((H_q, D), dtype=np.float64)
    for h in range(H_q):
        g = _kv_head(h, H_q, H_kv)
        s = np.sum(K[g] * q[h][None, :], axis=1) / math.sqrt(D)   # dot product, scaling
        e = np.exp(s - s.max())                                     # softmax numerator
        out[h] = np.sum(e[:, None] * V[g], axis=0) / np.sum(e)      # weighted sum of V
    return out


def solo_attention_exact(q, K, V):
    """Same definition with every sum taken by ``math.fsum`` (correctly rounded,
    hence independent of summation order): the exact result rounded once per
    reduction.  Used by the brute-force and order-independence pins."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    H_q, D = q.shape
    H_kv, n, _ = K.shape
    if n < 1:
        raise ValueError("attention over an empty history (S:L51 contract violation)")
    out = np.empty((H_q, D), dtype=np.float64)
    rs = math.sqrt(D)
    for h in range(H_q):
        g = _kv_head(h, H_q, H_kv)
        s = [math.fsum(K[g, j] * q[h]) / rs for j in range(n)]
        m = max(s)
        e = [math.exp(x - m) for x in s]
        den = math.fsum(e)
        for d in range(D):
            out[h, d] = math.fsum(e[j] * V[g, j, d] for j in range(n)) / den
    return out
