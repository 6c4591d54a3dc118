"""CPU checks of the copy lane's host-tier DMA plan (a7; ig.h ig_plan_copy_groups):
the groups cover every unmasked token exactly once, stay inside the token grid, keep 2-D rows
from overlapping (pitch >= width), and minimise calls x call_rows + masked rows copied — the
cost is checked against an exhaustive search over all partitions of the runs into spans on
small masks, and a rectangle collapses to at most 3 calls.  No GPU."""
import itertools

import numpy as np
import pytest

import synth
from paper_2505_20600_b200 import ig

CALL_BYTES = 275e3  # ig_api.cu DMA_CALL_BYTES


def call_rows(row_bytes):
    return max(1, round(CALL_BYTES / (row_bytes * 2)))


def runs_of(mask):
    e = np.diff(np.concatenate([[1], mask, [1]]).astype(np.int8))
    return list(zip(np.where(e == -1)[0].tolist(), (np.where(e == 1)[0] - np.where(e == -1)[0]).tolist()))


def check(mask, W=0, row_bytes=6144):
    L = mask.size
    groups = ig.ig_plan_copy_groups(mask, W, row_bytes)
    cnt = np.zeros(L, np.int64)
    for start, ln, stride, count in groups:
        assert ln > 0 and count >= 1
        if count > 1:
            assert ln <= stride
        for i in range(count):
            a = start + i * stride
            assert 0 <= a and a + ln <= L
            cnt[a:a + ln] += 1
    assert (cnt[mask == 0] == 1).all(), "an unmasked row is not copied exactly once"
    masked_rows = int(cnt[mask != 0].sum())
    return groups, len(groups) * call_rows(row_bytes) + masked_rows


def span_optimum(mask, cr):
    """Exhaustive: best partition of the runs into contiguous spans (no strided groups)."""
    runs = runs_of(mask)
    n = len(runs)
    best = None
    for cuts in itertools.product([0, 1], repeat=max(n - 1, 0)):
        cost, i = 0, 0
        for j in range(n):
            if j == n - 1 or cuts[j]:
                s, e = runs[i][0], runs[j][0] + runs[j][1]
                cost += cr + (e - s) - sum(r[1] for r in runs[i:j + 1])
                i = j + 1
        best = cost if best is None else min(best, cost)
    return best if n else 0


@pytest.mark.parametrize("seed", range(20))
def test_cost_never_above_exhaustive_span_partition(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(16, 96))
    mask = (rng.random(L) < rng.uniform(0.2, 0.8)).astype(np.uint8)
    if len(runs_of(mask)) > 14:
        mask[: L // 2] = 1
    row_bytes = int(rng.choice([6144, 20000, 60000, 140000]))
    _, cost = check(mask, 0, row_bytes)
    assert cost <= span_optimum(mask, call_rows(row_bytes))


def test_rectangle_is_few_calls():
    d = synth.FLUX
    for (r0, r1, c0, c1) in [(10, 40, 5, 30), (0, 64, 0, 10), (20, 21, 0, 64), (0, 64, 60, 64), (3, 60, 1, 63)]:
        m = synth.rect_mask(d, r0, r1, c0, c1).reshape(-1).astype(np.uint8)
        g, cost = check(m, d.grid_w)
        assert len(g) <= 3, (r0, r1, c0, c1, g)
        assert cost == len(g) * call_rows(6144)  # no masked row copied


@pytest.mark.parametrize("seed", range(8))
def test_headline_masks(seed):
    d = synth.FLUX
    for rid in range(seed * 4, seed * 4 + 4):
        m = synth.mixed_mask(d, rid).reshape(-1).astype(np.uint8)
        g, cost = check(m, d.grid_w)
        n_runs = len(runs_of(m))
        assert len(g) <= n_runs
        # never worse than one call per run, nor than one call per maximal span
        assert cost <= n_runs * call_rows(6144)
        assert len(g) <= 24


def test_degenerate_masks():
    for m in (np.zeros(256, np.uint8), np.ones(256, np.uint8), np.eye(16, dtype=np.uint8).reshape(-1)):
        check(m, 16)
    assert ig.ig_plan_copy_groups(np.ones(64, np.uint8)) == []
    assert ig.ig_plan_copy_groups(np.zeros(64, np.uint8)) == [(0, 64, 0, 1)]
