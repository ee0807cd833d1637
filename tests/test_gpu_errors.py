"""Error behaviour of the GPU engine and the C ABI (reference: engine.py:104-108,
134-138; slic_core.py:56-79): invalid settings and mismatched frames raise the
reference's exceptions, status codes come with a message, and a failed call
leaves the engine usable.
"""

import ctypes

import numpy as np
import pytest

import paper_1509_04232_b200 as spx
from paper_1509_04232_b200 import _lib

pytestmark = pytest.mark.gpu


def _frame(h, w, seed=0):
    return spx.ImageRGB(np.random.default_rng(seed).integers(0, 256, (h, w, 3), dtype=np.uint8))


def test_wrong_frame_size_raises_and_engine_stays_usable():
    st = spx.Settings(img_width=64, img_height=48, num_superpixels=12)
    eng = spx.SegEngine(st)
    with pytest.raises(spx.DimensionMismatchError):
        eng.perform_segmentation(_frame(48, 63))
    with pytest.raises(spx.DimensionMismatchError):
        eng.perform_segmentation(_frame(47, 64))
    res = eng.perform_segmentation(_frame(48, 64))
    assert res.labels.data.shape == (48, 64)
    assert int(res.spixel_map.num_pixels.sum()) == 48 * 64


def test_segment_device_rejects_bad_tensors():
    import torch
    st = spx.Settings(img_width=32, img_height=16, num_superpixels=8)
    eng = spx.SegEngine(st, max_batch=2)
    good = torch.zeros((2, 16, 32, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(spx.DimensionMismatchError):
        eng.segment_device(good.float())
    with pytest.raises(spx.DimensionMismatchError):
        eng.segment_device(good.cpu())
    with pytest.raises(spx.DimensionMismatchError):
        eng.segment_device(good[:, :, :16].contiguous())
    with pytest.raises(spx.DimensionMismatchError):
        eng.segment_device(good.permute(0, 2, 1, 3))  # not contiguous
    labels = eng.segment_device(good)[0]
    torch.cuda.synchronize()
    assert tuple(labels.shape) == (2, 16, 32)
    # caller-supplied outputs: too few frames, wrong dtype, not contiguous,
    # wrong device, wrong arity -- all rejected before any kernel runs
    outs = eng.allocate_outputs(2)
    small = eng.allocate_outputs(1)
    for i in range(5):
        bad = list(outs)
        bad[i] = small[i]
        with pytest.raises(spx.DimensionMismatchError):
            eng.segment_device(good, tuple(bad))
    bad = list(outs)
    bad[1] = outs[1].float()
    with pytest.raises(spx.DimensionMismatchError):
        eng.segment_device(good, tuple(bad))
    bad = list(outs)
    bad[0] = torch.empty((2, 32, 16), dtype=torch.int32, device="cuda").transpose(1, 2)
    with pytest.raises(spx.DimensionMismatchError):
        eng.segment_device(good, tuple(bad))
    bad = list(outs)
    bad[3] = outs[3].cpu()
    with pytest.raises(spx.DimensionMismatchError):
        eng.segment_device(good, tuple(bad))
    with pytest.raises(spx.DimensionMismatchError):
        eng.segment_device(good, outs[:4])
    # a larger output set is fine (the first b frames are written)
    big = spx.SegEngine(st, max_batch=3).allocate_outputs(3)
    eng.segment_device(good, big)
    torch.cuda.synchronize()
    assert np.array_equal(big[0][:2].cpu().numpy(), labels.cpu().numpy())


def test_batch_larger_than_engine():
    # device API: at most max_batch frames per call; the host-buffer call
    # streams any number of frames through the engine in chunks
    import torch
    st = spx.Settings(img_width=32, img_height=16, num_superpixels=8)
    eng = spx.SegEngine(st, max_batch=2)
    frames = np.stack([_frame(16, 32, i).data for i in range(3)])
    with pytest.raises(ValueError, match="batch"):
        eng.segment_device(torch.from_numpy(frames).cuda())
    labels, cxy, clab, counts, _ = eng.segment_host(frames)
    for i in range(3):
        one = spx.SegEngine(st).perform_segmentation(spx.ImageRGB(frames[i]))
        assert np.array_equal(labels[i], one.labels.data)
        assert clab[i].tobytes() == one.spixel_map.centers_lab.tobytes()


def test_invalid_settings_rejected_before_the_device():
    with pytest.raises(spx.InvalidSettingsError):
        spx.SegEngine(spx.Settings(img_width=8, img_height=8, num_superpixels=4, no_iters=0))
    with pytest.raises(spx.InvalidSettingsError):
        spx.SegEngine(spx.Settings(img_width=8, img_height=8, num_superpixels=4), backend="gpu")


def test_c_abi_engine_create_reports_invalid_settings():
    lib = _lib.load()
    st = spx.Settings(img_width=64, img_height=48, num_superpixels=12)
    from paper_1509_04232_b200.engine import _native_settings
    ns = _native_settings(st, spx.compute_grid(st))
    ns.s = 0  # corrupt: zero grid interval
    h = ctypes.c_void_p()
    rc = lib.spx_engine_create(ctypes.byref(ns), 1, 0, ctypes.byref(h))
    assert rc != 0
    assert lib.spx_last_error()  # a message comes with the status
    assert not h.value


def test_strip_engine_rejects_unsupported_modes():
    # row strips take early stop and strict connectivity (the strict pass runs
    # over the gathered image); geometry outside the fused path is rejected
    from paper_1509_04232_b200.strips import StripEngine, check_strip_settings
    check_strip_settings(spx.Settings(img_width=64, img_height=64, spixel_size=8,
                                      early_stop_threshold=1.0))
    check_strip_settings(spx.Settings(img_width=64, img_height=64, spixel_size=8,
                                      connectivity_mode=spx.ConnectivityMode.STRICT))
    with pytest.raises(spx.InvalidSettingsError):
        StripEngine(spx.Settings(img_width=64, img_height=64, spixel_size=3), 0, 5)
