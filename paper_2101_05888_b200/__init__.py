"""paper_2101_05888_b200 -- B200-native time-domain backprojection (TDBP) for synthetic aperture
sonar, the data-parallel hot path of arXiv 2101.05888 (ASASIN).

The product is libsasbp.so (C ABI, include/sasbp.h; hand-written sm_100a CUDA kernels in csrc/).
This package adds the ctypes binding (sasbp.py) and the multi-GPU driver (distributed.py).
"""
from .sasbp import (Backprojector, SasError, load_library, make_grid, rangecompress,  # noqa: F401
                    rangecompress_device, upsample, upsample_device, baseband, baseband_device, whitening_gain,
                    whitening_gain_device, rangecompress_whitened, rangecompress_whitened_device, version,
                    EXPORTS, LIB_PATH)

__all__ = ["Backprojector", "SasError", "load_library", "make_grid", "rangecompress", "rangecompress_device",
           "upsample", "upsample_device", "baseband", "baseband_device", "whitening_gain", "whitening_gain_device",
           "rangecompress_whitened", "rangecompress_whitened_device", "version", "EXPORTS", "LIB_PATH"]
