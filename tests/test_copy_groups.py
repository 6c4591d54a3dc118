"""CPU checks of the copy lane's host-tier DMA plan (a7): the strided groups
ig_plan_copy_groups returns cover every unmasked token exactly once, stay inside the token
grid, never overlap, cover at most (unmasked + 64) / 8 masked rows per group, and collapse a
rectangle's runs into a handful of calls.  Brute force over the token set, no GPU."""
import numpy as np
import pytest

import synth
from paper_2505_20600_b200 import ig

MAX_GAP = 2  # ig_api.cu COPY_MAX_GAP


def covered(groups, L):
    cnt = np.zeros(L, np.int64)
    for start, ln, stride, count in groups:
        assert ln > 0 and count >= 1
        if count > 1:
            assert ln <= stride  # pitch >= width (cudaMemcpy2DAsync)
        for i in range(count):
            a = start + i * stride
            assert 0 <= a and a + ln <= L
            cnt[a:a + ln] += 1
    return cnt


def check(mask):
    L = mask.size
    groups = ig.ig_plan_copy_groups(mask)
    cnt = covered(groups, L)
    assert cnt.max(initial=0) <= 1, "rows copied twice"
    assert (cnt[mask == 0] == 1).all(), "an unmasked row is not copied"
    # masked rows copied: the merged gaps (<= MAX_GAP rows between consecutive unmasked runs)
    # plus at most (covered + 64) / 8 per group
    edges = np.diff(np.concatenate([[1], mask, [1]]).astype(np.int8))
    starts, ends = np.where(edges == -1)[0], np.where(edges == 1)[0]
    gaps = starts[1:] - ends[:-1]
    budget = int(gaps[gaps <= MAX_GAP].sum()) + sum((ln * count + 64) / 8 for _, ln, _, count in groups)
    extra = int(sum(mask[start + i * stride:start + i * stride + ln].sum()
                    for start, ln, stride, count in groups for i in range(count)))
    assert extra <= budget
    return groups


def test_rectangle_is_few_calls():
    d = synth.FLUX
    for (r0, r1, c0, c1) in [(10, 40, 5, 30), (0, 64, 0, 10), (20, 21, 0, 64), (0, 64, 60, 64)]:
        m = synth.rect_mask(d, r0, r1, c0, c1).reshape(-1).astype(np.uint8)
        g = check(m)
        assert len(g) <= 3, (r0, r1, c0, c1, g)


@pytest.mark.parametrize("seed", range(12))
def test_random_masks_cover_exactly(seed):
    rng = np.random.default_rng(seed)
    d = synth.FLUX
    L = d.grid_h * d.grid_w if hasattr(d, "grid_h") else 4096
    for frac in (0.05, 0.2, 0.6):
        n = int(frac * L)
        m = (synth.blob_mask_count(d, n, rng) if seed % 2 else synth.rect_mask_count(d, n, rng)).reshape(-1).astype(np.uint8)
        g = check(m)
        runs = int(np.sum(np.diff(np.concatenate([[1], m, [1]]).astype(np.int8)) == -1))
        assert len(g) <= runs
        if seed % 2:  # noisy blob edges: gap merging + grouping cut the calls well below the runs
            assert len(g) <= max(8, runs // 2)
    # unstructured noise: still exact coverage
    m = (rng.random(L) < 0.3).astype(np.uint8)
    check(m)


def test_degenerate_masks():
    for m in (np.zeros(256, np.uint8), np.ones(256, np.uint8), np.eye(16, dtype=np.uint8).reshape(-1)):
        check(m)
    assert ig.ig_plan_copy_groups(np.ones(64, np.uint8)) == []
    assert ig.ig_plan_copy_groups(np.zeros(64, np.uint8)) == [(0, 64, 0, 1)]
