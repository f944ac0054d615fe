"""CPU: the C-ABI library loads, exports every entry point include/psa.h declares, and maps
argument errors onto the reference error taxonomy — no device compute is issued."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "psa.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(psa_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_entry_points():
    names = _declared()
    for n in ("psa_pyramid_build", "psa_similarity_caps", "psa_importance_sampled",
              "psa_importance_antidiagonal", "psa_antidiag_workspace_bytes", "psa_gather_rows",
              "psa_assign_levels", "psa_mask_to_plan", "psa_attn_fwd", "psa_last_error",
              "psa_pyramid_build_gather", "psa_attn_fwd_scatter"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2512_04025_b200 import _lib
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_lib.EXPORTED)
    assert lib.psa_version() == 100


def test_argument_errors_map_to_validation_error():
    from paper_2512_04025_b200 import _lib
    from paper_2512_04025_b200.errors import ValidationError
    lib = _lib.load()
    # d=96 is rejected before any device work
    rc = lib.psa_pyramid_build(1, 1, 1, 64, 96, 64, 2, 1, 1, None, None)
    assert rc == _lib.PSA_EINVAL
    assert "head_dim" in lib.psa_last_error().decode()
    with pytest.raises(ValidationError):
        _lib.check(rc, "psa_pyramid_build")
    rc = lib.psa_attn_fwd(1, 1, 1, 1, 1, 1, 2, 1, 1024, 128, 256, 64, 2, 1, 1, 0, 1, 1, 1, None)
    assert rc == _lib.PSA_EINVAL and "q_block" in lib.psa_last_error().decode()
    # s_k = 40 > 16: fp64 path only, workspace = block maxima + (m, l) per sampled row
    assert lib.psa_importance_workspace_bytes(2, 2, 10, 8, 10, 40) == 8 * (2 * 80 * 10 + 2 * 2 * 80)
    # s_k = 8: plus the int8 slices of the exact tensor-core path
    assert lib.psa_importance_workspace_bytes(2, 2, 10, 8, 10, 8) > 8 * (2 * 80 * 10 + 2 * 2 * 80)
    rc = lib.psa_gather_rows(1, 1, 16, 6, 1, 2, None)  # row_bytes must be a multiple of 4
    assert rc == _lib.PSA_EINVAL
    # antidiagonal: stride must divide k_block, k_block/stride <= 64
    rc = lib.psa_importance_antidiagonal(1, 1, 1, 1, 1, 1024, 128, 64, 64, 3, 0, 1, 1, None)
    assert rc == _lib.PSA_EINVAL and "stride" in lib.psa_last_error().decode()
    assert lib.psa_antidiag_workspace_bytes(2, 2, 1024, 64, 64, 3) == 0
    # n=1024, b_k=64, stride 4 -> per=16 (int8 path: one block per 16-key half -> 16 chunks)
    fp64 = 8 * 2 * 1024 * (16 + 16 + 2)
    assert lib.psa_antidiag_workspace_bytes(2, 2, 1024, 64, 64, 4) > fp64
    # backward: D rows + -lse log2(e) per query row (64-padded each), then fp32 dK/dV slabs of all
    # pyramid levels (< 2n pooled rows per KV head, psa_attention.cu psa_bwd_dkv_tc_kernel)
    rows = 2 * 8 * 1000
    pad = (rows + 63) // 64 * 64
    assert lib.psa_attn_bwd_workspace_bytes(2, 8, 2, 1000, 128) == 4 * (2 * pad + 4 * 2 * 2 * 1000 * 128)
    # stride 1 -> per=64 > 16: fp64 path only, 64-key chunks -> 16 chunks
    assert lib.psa_antidiag_workspace_bytes(2, 2, 1024, 64, 64, 1) == fp64


def test_product_path_rejects_cpu_tensors():
    import torch
    import paper_2512_04025_b200 as psa
    lay = psa.make_layout(256, 64, 64, 64, 2)
    x = torch.zeros(256, 64, dtype=torch.bfloat16)
    with pytest.raises(psa.ValidationError, match="CUDA"):
        psa.build_pyramid(x, x, lay)
    with pytest.raises(psa.ValidationError, match="CUDA"):
        psa.psa_attention(x, x, x, b_q=64, b_k=64, levels=2, estimator="sampled-max", s_q=8,
                          s_k=8, seed=0, mask="threshold", thresholds=(0.5, 0.9))


def test_product_package_never_imports_the_oracle():
    for p in (ROOT / "paper_2512_04025_b200").glob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
