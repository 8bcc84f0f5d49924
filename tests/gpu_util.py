"""Helpers shared by the GPU tests."""
import pytest

gpu = pytest.mark.gpu


def require_device():
    from paper_2012_03119_b200 import _lib
    if _lib.device_count() < 1:
        pytest.fail("GPU test run without a CUDA device: the product has no CPU path")
