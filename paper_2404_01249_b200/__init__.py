"""B200-native dense diffeomorphic matching (FireANTs direct-mode loop).

The product is the CUDA library ``libdifform_cuda.so`` behind the C-ABI in
``include/difform_gpu.h``; ``engine.Context`` is its Python face and
``cpp/difform_b200.hpp`` its C++ (difform::) face.  ``synth`` generates the
seeded BASELINE inputs.
"""
from ._abi import (GridMeta, RegistrationConfig, PyramidSchedule, AffineTransform, RunLog,
                   IterationRecord, InvalidArgument, NumericalError, DeviceError, LOSS_SSD,
                   LOSS_LNCC, LOSS_DICE)

__all__ = ["GridMeta", "RegistrationConfig", "PyramidSchedule", "AffineTransform", "RunLog",
           "IterationRecord", "InvalidArgument", "NumericalError", "DeviceError", "LOSS_SSD",
           "LOSS_LNCC", "LOSS_DICE"]
