"""Serializer registry: the reference contract (messaging.py:89-99) plus the zero-copy
device codec (tag 3) -- host-side behaviour that needs no GPU."""

import numpy as np
import pytest

from paper_2101_08878_b200 import messaging
from paper_2101_08878_b200.errors import UsageError
from paper_2101_08878_b200.messaging import CUDA_ARRAY_TAG, CudaArray, Frame, make_frame
from paper_2101_08878_b200.transport import MemoryDomain
from paper_2101_08878_b200.transport.base import DeviceRegion


class _Region(DeviceRegion):
    """Stand-in device region (the sim transport's bytes-backed region) with a device id."""

    def __init__(self, data: bytes):
        super().__init__(data)
        self.ptr = 0x7F0000001000
        self.device = 0


def test_builtin_tags_keep_the_reference_numbering():
    assert set(messaging.SERIALIZERS) >= {0, 1, 2, CUDA_ARRAY_TAG}
    assert make_frame("x", 1).decode() == "x"
    assert np.array_equal(make_frame([1.5, 2.0], 2).decode(), [1.5, 2.0])


def test_device_codec_frames_carry_the_region_itself():
    seen = {}

    def enc(obj):
        seen["enc"] = obj
        return obj  # already a region: the frame IS it (no copy)

    def dec(region):
        seen["dec"] = region
        return region

    messaging.register_serializer(200, enc, dec, device=True)
    try:
        region = _Region(b"abcdefgh")
        frame = make_frame(region, 200)
        assert frame.domain == MemoryDomain.DEVICE and frame.data is region and frame.length == 8
        assert frame.decode() is region and seen["dec"] is region
    finally:
        messaging.SERIALIZERS.pop(200)
        messaging.DEVICE_SERIALIZERS.discard(200)


def test_host_codecs_still_get_bytes():
    messaging.register_serializer(201, lambda o: bytes(o), lambda b: ("got", b))
    try:
        assert Frame(b"xy", 2, MemoryDomain.HOST, 201).decode() == ("got", b"xy")
        assert 201 not in messaging.DEVICE_SERIALIZERS
    finally:
        messaging.SERIALIZERS.pop(201)


def test_cuda_array_view_checks_shape_and_exports_the_interface():
    region = _Region(bytes(48))
    arr = CudaArray(region)
    assert arr.shape == (48,) and arr.dtype == np.uint8
    v = arr.view("<f8", (2, 3))
    cai = v.__cuda_array_interface__
    assert cai["shape"] == (2, 3) and cai["typestr"] == "<f8" and cai["data"] == (region.ptr, False)
    assert cai["version"] == 3 and cai["strides"] is None
    with pytest.raises(UsageError):
        arr.view("<f8", (5,))


def test_non_arrays_are_rejected_by_the_device_codec():
    with pytest.raises(UsageError):
        make_frame(b"plain bytes", CUDA_ARRAY_TAG)
