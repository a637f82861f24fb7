"""Host logic of the varlen prefill launch (NEXT-2, P:L215 / P:L335 length-grouped
prefill batches): the work list the persistent grid walks
(``baton_debug_prefill_plan``, prefill_attention.cu ``pf_plan``, DESIGN.md §6.3
"L2 panels").  No device work: runs on the CPU host.

Properties checked on the configs' 64-prompt mixes and hand-made batches:
  * every (prompt, 128-row query tile) entry appears exactly once;
  * prompts (longest first) are cut into panels of <= 64 MB of K/V (a prompt larger
    than a panel is a panel of its own), and entries run panel by panel;
  * inside a panel the entries are heaviest first (key tiles up to the diagonal);
  * a batch that fits one panel is in the round-1 order (global heaviest first);
  * the launch's refusals (empty prompt, > 64 prompts, > 1024 entries, cu_lens[0] != 0)
    return -1."""
import ctypes

import numpy as np
import pytest

from baton_inputs import config_workload

M, N, D = 128, 64, 128          # query rows per tile, keys per key tile, head_dim
PANEL = 64 << 20                # bytes of K + V per panel (default BATON_PF_PANEL_MB)


def _plan(lens, kv_heads, head_dim=D):
    from paper_2410_18701_b200 import _lib
    fn = _lib.lib.baton_debug_prefill_plan
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.POINTER(ctypes.c_int32), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                   ctypes.POINTER(ctypes.c_uint32), ctypes.c_int]
    cu = np.zeros(len(lens) + 1, np.int32)
    cu[1:] = np.cumsum(lens)
    out = np.zeros(2048, np.uint32)
    ne = fn(cu.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(lens), kv_heads, head_dim,
            out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), len(out))
    if ne < 0:
        return None
    return [(int(e) >> 16, int(e) & 0xFFFF) for e in out[:ne]]


def _cost(lens, e):
    p, mt = e
    return -(-min(M * (mt + 1), lens[p]) // N)


def _panels(lens, kv_heads):
    """Panel of each prompt: longest first (ties by index), cut when the next prompt's
    K + V bytes would overflow a non-empty panel."""
    order = sorted(range(len(lens)), key=lambda i: (-lens[i], i))
    panel, pid, acc = {}, 0, 0
    for i in order:
        kv = 4 * lens[i] * kv_heads * D
        if acc > 0 and acc + kv > PANEL:
            pid, acc = pid + 1, 0
        acc += kv
        panel[i] = pid
    return panel


def _check(lens, kv_heads):
    plan = _plan(lens, kv_heads)
    want = {(p, mt) for p, n in enumerate(lens) for mt in range(-(-n // M))}
    assert plan is not None
    assert len(plan) == len(want) and set(plan) == want
    panel = _panels(lens, kv_heads)
    pids = [panel[p] for p, _ in plan]
    assert pids == sorted(pids)
    for a, b in zip(plan, plan[1:]):
        if panel[a[0]] == panel[b[0]]:
            assert _cost(lens, a) >= _cost(lens, b), (a, b)
    return plan, panel


@pytest.mark.parametrize("cfg,hkv,n", [("7b", 32, 64), ("13b", 40, 64), ("70b", 8, 18)])
def test_config_mixes(cfg, hkv, n):
    lens = [q.l_q for q in config_workload(cfg).queries[:n]]
    plan, panel = _check(lens, hkv)
    n_panels = max(panel.values()) + 1
    kv = 4 * sum(lens) * hkv * D
    assert n_panels >= kv / PANEL          # no panel holds more than 64 MB
    if cfg != "70b":
        assert n_panels > 1                # the 64-prompt mixes span several panels


def test_one_panel_is_global_heaviest_first():
    lens = [1500, 350, 120, 900]           # 7B batch of one iteration's inserts: ~47 MB
    plan, panel = _check(lens, 32)
    assert set(panel.values()) == {0}
    costs = [_cost(lens, e) for e in plan]
    assert costs == sorted(costs, reverse=True)
    # stable: equal costs keep the (prompt, tile) enumeration order
    entries = [(p, mt) for p, n in enumerate(lens) for mt in range(-(-n // M))]
    assert plan == sorted(entries, key=lambda e: -_cost(lens, e))


def test_single_prompt_tiles_descending():
    plan, _ = _check([3400], 8)
    assert plan == [(0, mt) for mt in range(26, -1, -1)]


def test_prompt_larger_than_a_panel_is_its_own_panel():
    lens = [4096, 4096, 100, 50]           # 4096 x 32 kv heads x 512 B = 64 MB each
    _, panel = _check(lens, 32)
    assert [panel[i] for i in range(4)] == [0, 1, 2, 2]


@pytest.mark.parametrize("lens", [[4, 0, 6], [1] * 65, [128 * 1025]])
def test_refusals(lens):
    assert _plan(lens, 8) is None
