"""CPU-side checks of the C ABI: the library builds, loads and exports every
symbol include/hgm.h declares; calls without a usable GPU fail loudly with a
status (there is no CPU fallback).  No compute calls are made."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hgm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hgm_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1505_00581_b200 import build as B
    from paper_1505_00581_b200 import hgm

    B.build()
    return hgm.lib()


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("hgm_build_model_graph", "hgm_build_scene_index", "hgm_match_model_at_offsets", "hgm_detect_actions"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_export_list_matches_header():
    from paper_1505_00581_b200 import hgm

    assert sorted(hgm.EXPORTS) == _declared()


def test_no_cpu_fallback_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import synth
    from paper_1505_00581_b200 import hgm

    wl = synth.make_workload("C0", seed=0)
    with pytest.raises(hgm.HGMError) as e:
        hgm.build_scene_index(wl.scenes[0], device=0, T_max=5)
    assert e.value.status in (5,)  # HGM_ERR_CUDA


def test_argument_errors_before_any_device_work(lib):
    from paper_1505_00581_b200 import hgm

    class P:  # an empty point set
        frame = np.zeros(0, np.int32)
        x = y = saliency = np.zeros(0, np.float32)
        feat = np.zeros((0, 4), np.float32)
        id = None

    with pytest.raises(hgm.HGMError) as e:
        hgm.build_scene_index(P(), device=0, T_max=5)
    assert e.value.status == 1
    with pytest.raises(hgm.HGMError) as e:
        hgm.build_model_graph(P(), device=0)
    assert e.value.status == 1


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1505_00581_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "hgm_oracle" not in txt, f


def test_widened_entry_points_validate_before_device_work(lib):
    """f1/f3/f4 entry points reject bad arguments with a status before touching a GPU."""
    import ctypes as C

    from paper_1505_00581_b200 import hgm

    p = hgm._params(None)
    o = hgm.Offsets(0, 1, 4, 60)
    vp = C.c_void_p
    h = C.c_void_p()
    # streams: window 0 / stride 0 / score_mode 2 -> INVALID_ARGUMENT; empty dictionary -> EMPTY_POINT_SET
    fake = (vp * 1)(vp(1))
    assert lib.hgm_stream_create(fake, 1, C.byref(p), 0, 1, 0, 1.0, 0, C.byref(h)) == 3
    assert lib.hgm_stream_create(fake, 1, C.byref(p), 60, 0, 0, 1.0, 0, C.byref(h)) == 3
    assert lib.hgm_stream_create(fake, 1, C.byref(p), 60, 1, 2, 1.0, 0, C.byref(h)) == 3
    assert lib.hgm_stream_create(fake, 0, C.byref(p), 60, 1, 0, 1.0, 0, C.byref(h)) == 1
    n = C.c_int32()
    f0 = C.c_int64()
    assert lib.hgm_stream_push(None, None, 1, 0, None, None, C.byref(n), C.byref(f0)) == 3
    # recognition: no prototypes / NULL labels / n_labels out of range
    lab = (C.c_int32 * 1)(0)
    assert lib.hgm_classify_blocks(fake, 0, lab, 1, vp(1), C.byref(p), C.byref(o), 1.0, None, None, None,
                                   None) == 1
    assert lib.hgm_classify_blocks(fake, 1, None, 1, vp(1), C.byref(p), C.byref(o), 1.0, None, None, None,
                                   None) == 3
    assert lib.hgm_classify_blocks(fake, 1, lab, 0, vp(1), C.byref(p), C.byref(o), 1.0, None, None, None,
                                   None) == 3
    # chains: empty chain list, and a negative rank
    assert lib.hgm_detect_chains(fake, 0, None, 1, vp(1), C.byref(p), C.byref(o), 0, 1.0, None, None, None,
                                 None) == 1
    fr = np.zeros(2, np.int32)
    xs = np.zeros(2, np.float32)
    ft = np.zeros((2, 4), np.float32)

    class Pts:
        frame, x, y, saliency, feat, id = fr, xs, xs, xs, ft, None

    hp = hgm._HostPoints(Pts())
    assert lib.hgm_build_model_chain(C.byref(hp.s), 0, -1, C.byref(h)) == 3
