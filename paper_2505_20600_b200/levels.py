"""Per-level token masks for UNet models (BASELINE config 5; SURVEY §8(d) C-AMB 13): a UNet
runs its transformer blocks at several resolutions, so a request's token mask at the finest
attention level (64x64 for SDXL at 1024²) is reduced to the next level (32x32) by a 2x2
any-pool — a coarse token is masked if any of its four fine tokens is, so no edited pixel is
lost.  Host-side input preparation (admission), not part of the step."""
from __future__ import annotations

import numpy as np


def any_pool2(mask: np.ndarray, grid_h: int, grid_w: int) -> np.ndarray:
    """uint8 [grid_h * grid_w] (nonzero = masked) -> uint8 [(grid_h / 2) * (grid_w / 2)]."""
    if grid_h % 2 or grid_w % 2:
        raise ValueError("grid must be even in both dimensions")
    m = (np.asarray(mask).reshape(grid_h // 2, 2, grid_w // 2, 2) != 0).any(axis=(1, 3))
    return m.astype(np.uint8).reshape(-1)
