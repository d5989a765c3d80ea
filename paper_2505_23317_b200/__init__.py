"""B200-native CF-DETR coarse-to-fine encoder hot path (arXiv 2505.23317).

The product is libcfdetr.so (include/cfdetr.h): hand-written sm_100a kernels
behind a C ABI.  This package holds the kernels' sources (csrc/), the nvcc build
(build.py), the ctypes binding (_lib.py) and a thin Python API (api.py).
"""
from ._lib import load, CfdError  # noqa: F401


def __getattr__(name):
    if name in ("CFDetrEncoder", "launch_count", "bf16_tensor", "f32_tensor"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
