"""B200-native Pyramid Sparse Attention (PSA, arXiv 2512.04025) forward.

Drop-in for the hot path of the reference package ``pyrattn`` (pkg/src/pyrattn/__init__.py):
same entry-point names, argument meaning and error classes, but every tensor operation runs in
hand-written sm_100a CUDA (libpsa.so, C ABI in include/psa.h) on torch CUDA tensors. There is
no CPU fallback: calling with CPU tensors or without the built library raises.
"""

from .attention import (LN2, AttentionOutput, causal_full_attention, full_attention,
                        level_bias, psa_reference, psa_streaming)
from .errors import NumericError, TensorFileError, ValidationError
from .importance import (antidiagonal_selection, importance_antidiagonal, importance_sampled,
                         sample_tables)
from .layout import (PRESET_CUTPOINTS, BlockLayout, LevelThresholds, QuantileCutpoints,
                     SamplerConfig, SimThresholds, make_layout)
from .mask import (MaskPlan, SparsityReport, assign_quantile, assign_threshold, binary_mask,
                   causal_premask, combine_mask, report_from_counts, sparsity_report)
from .permute import Permutation, apply_permutation, hilbert_order, invert_permutation
from .pipeline import (PipelineResult, PSAResult, RunConfig, psa_attention, psa_forward_4d,
                       relative_error, report_to_json, run_pipeline)
from .pyramid import PyramidKV, build_pyramid, build_pyramid_gather, level_cap_from_similarity
from .autograd import psa_attention_differentiable
from .graph import CapturedForward
from .tensorfile import read_tensor, write_tensor
from .schedule import (ExecutionTile, Segment, TileSchedule, UtilizationStats, build_schedule,
                       execute_schedule, plan_utilization, utilization)

__version__ = "0.1.0"

__all__ = [
    "AttentionOutput", "CapturedForward", "BlockLayout", "LN2", "LevelThresholds", "MaskPlan", "NumericError",
    "Permutation", "apply_permutation", "hilbert_order", "invert_permutation",
    "ExecutionTile", "Segment", "TileSchedule", "UtilizationStats", "build_schedule",
    "execute_schedule", "plan_utilization", "utilization", "psa_reference",
    "PipelineResult", "relative_error", "report_to_json", "run_pipeline",
    "PRESET_CUTPOINTS", "PSAResult", "PyramidKV", "QuantileCutpoints", "RunConfig",
    "SamplerConfig", "SimThresholds", "SparsityReport", "TensorFileError", "ValidationError",
    "assign_quantile", "assign_threshold", "binary_mask", "build_pyramid", "build_pyramid_gather",
    "causal_full_attention", "causal_premask", "combine_mask", "full_attention",
    "antidiagonal_selection", "importance_antidiagonal", "importance_sampled", "level_bias",
    "level_cap_from_similarity", "make_layout",
    "psa_attention", "psa_forward_4d", "psa_streaming", "report_from_counts", "sample_tables",
    "sparsity_report", "read_tensor", "write_tensor", "psa_attention_differentiable",
]
