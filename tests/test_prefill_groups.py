"""The PD method's prefill batching (reading C27, "queries with similar
sequence lengths will be grouped into a batch"): engine.prefill_groups splits
fresh prompts into varlen a8 launches -- by length, a new group whenever a prompt is
more than 1.25x the group's shortest, and within the launch limits (64 prompts, 1024
query tiles of 128 rows).  Host logic only."""
import numpy as np
import pytest

from paper_2410_18701_b200.engine import prefill_groups, batchable


def _items(lens):
    return [(i, n, None, None) for i, n in enumerate(lens)]


@pytest.mark.parametrize("seed", range(20))
def test_length_groups_are_similar_and_cover_everything(seed):
    rng = np.random.default_rng(seed)
    lens = [int(x) for x in rng.integers(1, 4000, size=int(rng.integers(1, 150)))]
    groups = prefill_groups(_items(lens), by_length=True)
    flat = [it for g in groups for it in g]
    assert sorted(q for q, *_ in flat) == list(range(len(lens)))     # every prompt once
    assert [n for _, n, *_ in flat] == sorted(lens)                  # shortest first
    for g in groups:
        ns = [n for _, n, *_ in g]
        assert max(ns) <= 1.25 * min(ns)                             # similar length
        assert len(g) <= 64 and sum(-(-n // 128) for n in ns) <= 1024
    # groups are maximal: the next group's shortest would break the ratio or a limit
    for g, h in zip(groups, groups[1:]):
        n0, nx = g[0][1], h[0][1]
        tiles = sum(-(-n // 128) for _, n, *_ in g) + -(-nx // 128)
        assert nx > 1.25 * n0 or len(g) == 64 or tiles > 1024


def test_arrival_order_groups_keep_order_and_limits():
    lens = [100] * 70 + [3000] * 50
    groups = prefill_groups(_items(lens), by_length=False)
    assert [it[0] for g in groups for it in g] == list(range(120))   # arrival order kept
    assert all(len(g) <= 64 and sum(-(-n // 128) for _, n, *_ in g) <= 1024 for g in groups)


def test_batchable_policy():
    assert not batchable(_items([100]))
    assert batchable(_items([100, 200]))                  # short prompts: one launch
    assert not batchable(_items([3000, 3500]))            # long prompts: one launch each
    assert batchable(_items([3000, 3500]), grouping="length")   # the PD method groups them
