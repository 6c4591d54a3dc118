"""CPU checks of the boundary: libig.so loads without a GPU and exports every function that
include/*.h declares; ig_weight_count matches the table synth describes; the Python binding
exposes the same names."""
import ctypes
import glob
import os
import re

import pytest

import synth
from paper_2505_20600_b200 import ig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"^\s*(?:ig_status|void|int|const char\*)\s+(ig_\w+)\s*\(", src, re.M))
    return names


def test_headers_declare_the_north_star_calls():
    d = declared()
    for name in ("ig_cache_template", "ig_edit_step", "ig_prefetch_layer", "ig_mask_build"):
        assert name in d


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(ig.LIB_PATH)
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, missing
    assert set(declared()) <= set(ig.EXPORTS)
    for n in declared():
        assert callable(getattr(ig, n))


@pytest.mark.parametrize("name", list(synth.MODELS))
def test_weight_count_matches_table(name):
    m = synth.MODELS[name]
    assert ig.ig_weight_count(ig.make_desc(m, ig.IG_BF16)) == len(synth.weight_table(m))


def test_ctx_create_rejects_bad_desc_without_gpu():
    # host-side validation runs before any CUDA call (no partial enqueue)
    m = synth.TINY
    d = ig.make_desc(m, ig.IG_F32)
    d.heads = 3
    with pytest.raises(ig.IgError) as e:
        ig.ig_ctx_create(d, [1] * len(synth.weight_table(m)))
    assert e.value.name == "IG_EINVAL"
    d = ig.make_desc(m, ig.IG_F32)
    with pytest.raises(ig.IgError) as e:
        ig.ig_ctx_create(d, [1] * 3)
    assert e.value.name == "IG_EINVAL"


@pytest.mark.parametrize("name", [n for n, m in synth.MODELS.items() if m.n_unet])
def test_unet_desc_passes_host_validation(name):
    """Every UNet shape synth describes passes the host-side checks (without a GPU the call
    then fails at the first CUDA call, never with IG_EINVAL / IG_EUNSUPPORTED)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("fake weight pointers: CPU-only check")
    m = synth.MODELS[name]
    with pytest.raises(ig.IgError) as e:
        ig.ig_ctx_create(ig.make_desc(m, ig.IG_BF16), [1] * len(synth.weight_table(m)))
    assert e.value.name not in ("IG_EINVAL", "IG_EUNSUPPORTED"), str(e.value)


@pytest.mark.parametrize("name", list(synth.UNET_FULL))
def test_unet_weight_count_matches_table(name):
    u = synth.UNET_FULL[name]
    assert ig.ig_unet_weight_count(ig.make_unet_desc(u)) == len(synth.unet_full_weight_table(u))


def test_tuning_struct_roundtrip_without_gpu():
    """ig_tuning (include/ig_ops.h): defaults are the measured-best settings, set/get round-trips,
    op_repeat < 1 is rejected; no CUDA call is involved."""
    t0 = ig.ig_tuning_get()
    names = [f for f, _ in ig.ig_tuning._fields_]
    assert ctypes.sizeof(ig.ig_tuning) == 4 * len(names)
    t = ig.ig_tuning_get()
    t.gemm_bn64 = 0
    t.op_repeat = 3
    ig.ig_tuning_set(t)
    got = ig.ig_tuning_get()
    assert got.gemm_bn64 == 0 and got.op_repeat == 3
    bad = ig.ig_tuning_get()
    bad.op_repeat = 0
    with pytest.raises(Exception):
        ig.ig_tuning_set(bad)
    ig.ig_tuning_set(t0)
    assert [getattr(ig.ig_tuning_get(), n) for n in names] == [getattr(t0, n) for n in names]
