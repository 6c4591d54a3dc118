"""ORACLE — test infrastructure, NOT part of the product path.

A plain, slow, obviously-correct float64 NumPy implementation of the InstGenIE mask-aware
denoising step (arXiv 2505.20600, K/V-caching variant, fig:transformer_alter P:435-446),
written from PAPER.md before any kernel.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it.  It shares no code
with `paper_2505_20600_b200/` (the CUDA path) and neither imports the other; the only
common module is `synth/`, which draws seeded inputs and holds none of the method's
arithmetic.

Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, C-AMB k = DESIGN.md reading k.
"""
from .instgenie import *  # noqa: F401,F403
from .unet import *  # noqa: F401,F403,E402
from .unet_full import *  # noqa: F401,F403,E402
