"""B200-native Sparse DNN Challenge inference (arxiv 1909.05631).

A drop-in for the reference's inference entry point (sdnnbench.engine):
hand-written sm_100a CUDA kernels in libsdnn.so behind the C ABI of
include/sdnn.h, with this package as the Python host mirror.
"""

from .engine import (  # noqa: F401
    DEFAULT_YMAX,
    DeviceNetwork,
    InferenceConfig,
    RunResult,
    apply_bias_relu_clamp,
    categorize,
    infer,
    infer_timed,
    spmm,
    warmup,
)
from .errors import CapacityError, ParameterError, SdnnError, ShapeError  # noqa: F401
from .model import CategorySet, FeatureBatch, LayerWeights, NetworkModel, SparseMatrix  # noqa: F401

__version__ = "0.1.0"
