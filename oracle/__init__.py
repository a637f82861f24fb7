"""Baton fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here.  The product path
(``paper_2410_18701_b200``) never imports it, and it never imports the product
path: the two share no code.  The only shared module is ``baton_inputs`` (seeded
input generators, no method arithmetic).

Contents (citations are /root/reference/PAPER.md line numbers, "P:Lnn"):

* ``attention.solo_attention`` (O-1): textbook scaled-dot-product attention of one
  query over its own token history (§2.1 "General architecture").
* ``batch.Shard`` (O-2): the paper-literal batch state machine with DENSE, growing
  ``attention_mask`` / ``KV_Cache`` tensors manipulated exactly as §3.1-§3.3 say:
  append a column per decode iteration, embed prefilled K/V end-aligned or
  with left expansion, zero a finished row, release the
  front ``[0:min(index_i)]``, store/re-insert a query's K/V,
  move queries out to shrink the batch.
* ``schedule.Simulator``: the serving loop driving G shards with the readings
  C5-C9, C17-C20 of DESIGN.md §3.

Pins: every function here is pinned in ``tests/test_oracle_*.py`` against closed
forms, library routines, paper/SPEC examples, invariants and brute force (see
DESIGN.md §4).  No function of this package is "parity unpinned".
"""
from .attention import solo_attention, solo_attention_exact
from .batch import Shard, OracleError, SlotBusy, SlotEmpty, Capacity
from .schedule import Simulator, IterationRecord

__all__ = ["solo_attention", "solo_attention_exact", "Shard", "OracleError", "SlotBusy",
           "SlotEmpty", "Capacity", "Simulator", "IterationRecord"]
