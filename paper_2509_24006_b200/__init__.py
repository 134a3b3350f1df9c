"""B200-native SLA (Sparse-Linear Attention, arXiv 2509.24006) behind the reference's
operator API.  The compute path is libsla_b200.so (hand-written sm_100a CUDA) reached
through the C-ABI in include/sla_b200.h; see DESIGN.md."""
from .sla import (  # noqa: F401
    SLA,
    BlockLayout,
    SlaConfig,
    SlaForwardState,
    SlaGradients,
    combine_outputs,
    make_block_layout,
    proj_backward,
    sla_backward,
    sla_step_backward,
    sla_forward,
    sla_forward_with_mask,
)
from .pipeline import HostTrainStep  # noqa: F401
from .autograd import SparseLinearAttention, sparse_linear_attention  # noqa: F401
from ._lib import LIB_PATH  # noqa: F401

__all__ = [
    "SLA", "BlockLayout", "SlaConfig", "SlaForwardState", "SlaGradients", "combine_outputs",
    "make_block_layout", "proj_backward", "sla_backward", "sla_step_backward", "sla_forward", "sla_forward_with_mask", "HostTrainStep",
    "SparseLinearAttention", "sparse_linear_attention",
]
