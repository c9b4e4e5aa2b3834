"""B200-native Cross-GPU Batch Normalization (CGBN, MegDet arXiv 1711.07240).

Drop-in for the CGBN hot path of the reference ``bigbatch`` package
(/root/reference/pkg/src/bigbatch/__init__.py:30-39, 114-116 export the BN names):
the same BN and collective names, running on hand-written sm_100a CUDA kernels behind
the C ABI in include/cgbn.h (libcgbn.so, built in-tree by ``make``).
"""

from .batchnorm import (
    BatchNormError,
    BNForwardCache,
    BNLayerState,
    bn_backward_local,
    bn_forward_local,
    bn_update_running,
    check_status,
    set_forward_exchange,
    set_fused,
    set_strict,
    sync_bn_backward,
    sync_bn_forward,
)
from .collectives import (
    DEFAULT_TIMEOUT_S,
    SCOPE_BN_GROUP,
    SCOPE_WORLD,
    CollectiveError,
    CollectiveProtocolError,
    CollectiveTimeoutError,
    DeviceGroup,
    DeviceHandle,
    DistHandle,
    GradBuckets,
    SoloHandle,
    allreduce_sum,
    world_mean_allreduce,
)
from .tensor import ChannelStats, NonFiniteError, TensorError, channel_affine, channel_sum

__version__ = "0.1.0"

__all__ = [
    "BatchNormError", "BNForwardCache", "BNLayerState", "bn_backward_local", "bn_forward_local",
    "bn_update_running", "check_status", "set_forward_exchange", "set_fused", "set_strict", "sync_bn_backward", "sync_bn_forward",
    "DEFAULT_TIMEOUT_S", "SCOPE_BN_GROUP", "SCOPE_WORLD", "CollectiveError",
    "CollectiveProtocolError", "CollectiveTimeoutError", "DeviceGroup", "DeviceHandle",
    "DistHandle", "GradBuckets", "SoloHandle", "allreduce_sum", "world_mean_allreduce", "ChannelStats", "NonFiniteError", "TensorError",
    "channel_affine", "channel_sum",
]
