"""paper_1608_00099_b200 -- the TRIOT hot path (arXiv 1608.00099) on B200 (sm_100a).

Public API on torch CUDA tensors (torch is used for device memory and streams only; every
step runs in libtriot.so's kernels, see include/triot.h):

    embed(dst, src, region_only=False)                  -> dst      (triot_embed)
    apply_binary(a, b, op="mul", out=None, iter_shape=None) -> out  (triot_apply_binary)
    expected_value(p)                                   -> (d,) float64 CUDA tensor
                                                           (triot_expected_value)

    prepare_embed(dst, src) / prepare_apply_binary(a, b, op, out) -> a re-issuable call with its
                                                           arguments marshalled once

The C-ABI entry points themselves are re-exported with their C names (triot_embed, ...).
There is no CPU fallback: importing raises if libtriot.so is missing, and the tensor API
raises for non-CUDA tensors.
"""
from __future__ import annotations

from ._lib import (OP_BINARY, OP_EMBED, OP_EV, TRIOT_ADD, TRIOT_DIV, TRIOT_EMBED_FULL,
                   TRIOT_EMBED_REGION_ONLY, TRIOT_F32, TRIOT_F64, TRIOT_MUL, TRIOT_SUB,
                   TriotError, check, lib, triot_apply_binary, triot_embed,
                   triot_expected_value, triot_expected_value_mass,
                   triot_expected_value_workspace_size,
                   triot_fastdiv_magic, triot_last_error, triot_max_dimension,
                   triot_plan_describe, triot_set_launch_policy, triot_status_string,
                   LIB_PATH)
from .api import (OPS, View, apply_binary, apply_binary_view, embed, embed_view,
                  expected_value, expected_value_view, fused_update, inner_product,
                  naive_convolve, embed_host, apply_binary_host, sum_rows,
                  expected_value_host, Prepared, prepare_embed, prepare_apply_binary)
from ._lib import (triot_expected_value_offset, triot_sum_rows, triot_expected_value_host)
from ._lib import (triot_apply_binary_view, triot_embed_view, triot_expected_value_view,
                   triot_fused_update,
                   triot_inner_product, triot_inner_product_workspace_size, triot_naive_convolve)

__all__ = [
    "embed", "apply_binary", "expected_value", "OPS", "TriotError", "View", "embed_view",
    "Prepared", "prepare_embed", "prepare_apply_binary",
    "apply_binary_view", "triot_embed_view", "triot_apply_binary_view", "inner_product",
    "expected_value_view", "triot_expected_value_view",
    "fused_update", "triot_inner_product", "triot_inner_product_workspace_size",
    "triot_fused_update", "naive_convolve", "triot_naive_convolve", "embed_host",
    "apply_binary_host", "sum_rows", "expected_value_host", "triot_expected_value_offset",
    "triot_sum_rows", "triot_expected_value_host",
    "triot_embed", "triot_apply_binary", "triot_expected_value", "triot_expected_value_mass",
    "triot_expected_value_workspace_size", "triot_max_dimension", "triot_status_string",
    "triot_last_error", "triot_plan_describe", "triot_set_launch_policy", "triot_fastdiv_magic",
    "LIB_PATH",
]
