"""Dense attention at the cfg2 shape (B=1, H=12, L=32760, d=128, bf16): torch SDPA (cuDNN
backend) and this repo's attention kernel on an all-level-1 plan, for a side-by-side ncu capture
(VERDICT r1 item 4). Prints both times (CUDA events, 5 reps after warm-up)."""
import sys
from pathlib import Path

import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2512_04025_b200.attention import _dense_layout, attention_forward  # noqa: E402
from paper_2512_04025_b200.mask import plan_from_mask  # noqa: E402
from paper_2512_04025_b200.pyramid import build_pyramid  # noqa: E402

B, H, N, D = 1, 12, 32760, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, H, N, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
dl = _dense_layout(N, D)
pyr = build_pyramid(k, v, dl)
plan = plan_from_mask(torch.ones(B, H, dl.n_q, dl.n_k, dtype=torch.int8, device="cuda"), dl, False, B, H)
flops = 4.0 * N * N * D * B * H


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    ms = timed(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
print(f"sdpa cudnn: {ms:.3f} ms  {flops / ms / 1e9:.1f} TF/s")
ms = timed(lambda: attention_forward(q, pyr, plan, False))
print(f"psa all-level-1: {ms:.3f} ms  {flops / ms / 1e9:.1f} TF/s")
