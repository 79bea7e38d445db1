"""CPU checks of the offload host logic: slice layouts vs the reference
fixtures (comm.py:106-119) and the fixed-at-init layout protocol."""

import pytest

from paper_2507_03211_b200.errors import ConfigurationError, ProtocolError
from paper_2507_03211_b200.scheduler import SliceLayout, apply_thread_aligned_layout


def test_slice_layouts_match_reference(golden):
    for total, n, owner, off, ln in golden["comm/layouts"]:
        lay = SliceLayout.build(0, int(total), int(n))
        assert lay.slices[int(owner)] == (owner, off, ln)
        assert sum(s[2] for s in lay.slices) == total


def test_slice_layout_rejects_zero():
    with pytest.raises(ConfigurationError):
        SliceLayout.build(0, 10, 0)


def test_layout_fixed_at_init():
    class S:
        from paper_2507_03211_b200.model import ModelConfig, model_layout
        layouts = model_layout(ModelConfig(16, 16, 2, 2, 8, "f32"))

    s = S()
    p = apply_thread_aligned_layout(s, 4)
    assert apply_thread_aligned_layout(s, 4) is p
    assert p["layouts"][1].width == -(-s.layouts[1].elem_count // 4)
    with pytest.raises(ProtocolError):
        apply_thread_aligned_layout(s, 2)


def test_plan_residency_fills_the_budget():
    """plan_residency: resident blocks + slots never exceed the budget, all
    blocks resident when they fit, at least 2 slots otherwise."""
    from paper_2507_03211_b200.model import model_layout, opt_config
    from paper_2507_03211_b200.scheduler import plan_residency

    cfg = opt_config("opt-13b", 2048)
    per = [bl for bl in model_layout(cfg) if bl.kind == "transformer"][0].elem_count * 8
    nb = cfg.n_blocks
    from paper_2507_03211_b200.errors import MemoryCapacityError

    with pytest.raises(MemoryCapacityError):         # below two slots: refused, never clamped over budget
        plan_residency(cfg, int(5e9))
    for gb in (20, 40, 60, 80, 100, 101, 200):
        k, slots = plan_residency(cfg, int(gb * 1e9))
        if gb * 1e9 >= nb * per:
            assert (k, slots) == (nb, 0)
        else:
            assert 0 <= k < nb and 2 <= slots <= nb - k
            assert (k + slots) * per <= gb * 1e9


def test_plan_residency_counts_split16_lo_planes():
    """With compress="split16" the streamed blocks' 2 B/param lo planes sit in
    the same budget: fewer resident blocks, never over budget (when the
    planes + 3 slots fit at all), and the uncompressed plan is unchanged."""
    from paper_2507_03211_b200.errors import ConfigurationError
    from paper_2507_03211_b200.model import model_layout, opt_config
    from paper_2507_03211_b200.scheduler import plan_residency

    cfg = opt_config("opt-13b", 2048)
    P = [bl for bl in model_layout(cfg) if bl.kind == "transformer"][0].elem_count
    per, lo, nb = 8 * P, 2 * P, cfg.n_blocks
    for gb in (40, 60, 80, 100, 120):
        b = int(gb * 1e9)
        k0, s0 = plan_residency(cfg, b)
        k, slots = plan_residency(cfg, b, compress="split16")
        if nb * per <= b:
            assert (k, slots) == (k0, s0) == (nb, 0)
            continue
        assert k <= k0 and slots >= 2
        if nb * lo + 3 * per <= b:
            assert (k + slots) * per + (nb - k) * lo <= b
    with pytest.raises(ConfigurationError):
        plan_residency(cfg, int(60e9), compress="fp8")


def test_slice_fields_and_layout_equality():
    """comm.py's Slice has owner / offset / length (pkg/tests/test_comm.py:47-53)
    and layouts compare by value (test_comm.py:210-218)."""
    from paper_2507_03211_b200.scheduler import SliceLayout

    lay = SliceLayout.build(0, 10, 4)
    assert [s.length for s in lay.slices] == [3, 3, 3, 1]
    assert [s.offset for s in lay.slices] == [0, 3, 6, 9]
    assert sorted(s.owner for s in lay.slices) == [0, 1, 2, 3]
    assert lay == SliceLayout.build(0, 10, 4) and lay != SliceLayout.build(0, 10, 2)
