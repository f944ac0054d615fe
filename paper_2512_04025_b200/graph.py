"""CUDA-graph replay of the fused PSA forward (B200-native replacement for a tracing compiler).

The device-resident forward (``pipeline.psa_forward_4d``) is a fixed chain of ~10 kernel
launches with no host synchronisation: every data-dependent decision (fp64 fallback heads, level
counts, skipped rows) lives in device flags the kernels read themselves. Its per-call host work
(argument checks, tensor-map encoding, workspace allocation, one ctypes call per kernel) is
therefore capturable once: ``CapturedForward`` records the chain into a ``torch.cuda.CUDAGraph``
for one set of shapes and configuration and then replays it, so small shapes (cfg1: L = 4096,
2 heads) stop being launch-bound. Inputs are copied into the graph's static buffers; outputs are
the graph's static tensors (valid until the next replay).

Reference: the forward this replays is ``run_pipeline``'s per-head chain
(pkg/src/pyrattn/pipeline.py:363-369); results are bit-identical to the eager call
(tests/test_gpu_graph.py).
"""

from __future__ import annotations

import torch

from .errors import ValidationError
from .importance import query_blocks
from .pipeline import PSAResult, RunConfig, psa_forward_4d


class CapturedForward:
    """``psa_forward_4d(q4, k4, v4, cfg, qblocks=...)`` captured into a CUDA graph.

    ``q4``/``k4``/``v4``: contiguous bf16 [B, H, N, d] CUDA tensors giving the shapes (and the
    first inputs). ``__call__(q4, k4, v4)`` copies new inputs of the same shapes into the static
    buffers (omit them to replay on the current contents) and returns the static
    :class:`PSAResult`.
    """

    def __init__(self, q4: torch.Tensor, k4: torch.Tensor, v4: torch.Tensor, cfg: RunConfig,
                 qblocks=None, warmup: int = 1):
        for name, x in (("Q", q4), ("K", k4), ("V", v4)):
            if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.bfloat16
                    and x.ndim == 4 and x.is_contiguous()):
                raise ValidationError(f"{name} must be a contiguous bf16 [B, H, N, d] CUDA tensor")
        self.cfg = cfg
        self.q = q4.clone()
        self.k = k4.clone()
        self.v = v4.clone()
        # the block list is validated and moved to the device here, once: inside the capture a
        # host list would need a host-to-device copy of pageable memory
        self.qblocks = query_blocks(qblocks, cfg.layout(), q4.device)
        side = torch.cuda.Stream(device=q4.device)
        side.wait_stream(torch.cuda.current_stream(q4.device))
        with torch.cuda.stream(side):  # warm-up outside the graph: library load, attributes
            for _ in range(max(1, warmup)):
                psa_forward_4d(self.q, self.k, self.v, cfg, qblocks=self.qblocks)
        torch.cuda.current_stream(q4.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.result: PSAResult = psa_forward_4d(self.q, self.k, self.v, cfg,
                                                    qblocks=self.qblocks)

    def __call__(self, q4: torch.Tensor | None = None, k4: torch.Tensor | None = None,
                 v4: torch.Tensor | None = None) -> PSAResult:
        for dst, src, name in ((self.q, q4, "Q"), (self.k, k4, "K"), (self.v, v4, "V")):
            if src is None:
                continue
            if src.shape != dst.shape:
                raise ValidationError(f"{name} shape {tuple(src.shape)} differs from the captured "
                                      f"{tuple(dst.shape)}")
            dst.copy_(src, non_blocking=True)
        self.graph.replay()
        return self.result
