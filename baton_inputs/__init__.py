"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the Baton method (no masking, padding,
embedding, release or attention).  It only draws:

* ``keygen``   -- the counter-based value generator that gives every query a
                  deterministic q/k/v history keyed by (seed, kind, layer, qid,
                  position, head, dim) (SURVEY.md §8(d) "Generator").
* ``workload`` -- per-configuration query streams (prompt length, answer
                  length, arrival iteration) and control events (preemption
                  points, batch resizes) with the length mixes of the paper's
                  datasets (§4.1 "Dataset").

Both the oracle (``oracle/``) and the product harness import it; neither
side's method code lives here.
"""
from .keygen import (PHI, KIND_Q, KIND_K, KIND_V, mix64, keyed_u64, keyed_f32,
                     f32_to_bf16_bits, bf16_bits_to_f64, keyed_bf16_bits,
                     query_history_bits, query_token_bits, SCALES_FLAT, SCALES_PEAKY)
from .workload import (Query, Workload, ControlEvents, w1_workload, config_workload,
                       random_stream, CONFIGS)

__all__ = [
    "PHI", "KIND_Q", "KIND_K", "KIND_V", "mix64", "keyed_u64", "keyed_f32",
    "f32_to_bf16_bits", "bf16_bits_to_f64", "keyed_bf16_bits",
    "query_history_bits", "query_token_bits", "SCALES_FLAT", "SCALES_PEAKY",
    "Query", "Workload", "ControlEvents", "w1_workload", "config_workload",
    "random_stream", "CONFIGS",
]
