"""paper_2510_13668_b200 -- B200-native hot path of STAR (arxiv 2510.13668).

Public API (names follow the C ABI in include/star.h):
    Predictor, lenpred_forward, lenpred_quantize       Eq. 2 predictor + quantizer
    project_instance_load                              per-instance projected loads
    PlanParams, plan_reschedule, plan_reschedule_segmented   Alg. 1 plan
    step.Step                                          one decode-step pass over ranks (NCCL)
    kv_pack, kv_unpack, kv_migrate                     ExecuteMigration's paged-KV copy (NEXT-4)
Importing the package does not load the CUDA library; the first call does, and raises
StarError if it is missing (there is no CPU fallback).
"""
from ._lib import (DISPATCH_CURRENT_LOAD, DISPATCH_PROJECTED, DISPATCH_ROUND_ROBIN, dispatch_requests,  # noqa: F401
                   CURRENT_ONLY, L_CTX, STRICT_MEM, Predictor, PlanParams, ProjectOut, StarError,  # noqa: F401
                   alloc_moves, decode_moves, lenpred_forward, lenpred_forward_project, lenpred_forward_project_plan,
                   lenpred_forward_refresh,
                   lenpred_quantize, plan_reschedule,
                   plan_reschedule_segmented, project_instance_load, plan_reschedule_large,
                   plan_reschedule_segmented_ws, plan_workspace_bytes, project_workspace_bytes, version,
                   kv_migrate, kv_pack, kv_unpack)

__all__ = ["Predictor", "lenpred_forward", "lenpred_forward_project", "lenpred_forward_project_plan", "lenpred_quantize", "project_instance_load", "PlanParams",
           "plan_reschedule", "plan_reschedule_segmented", "decode_moves", "alloc_moves", "StarError",
           "project_workspace_bytes", "version", "dispatch_requests", "STRICT_MEM", "CURRENT_ONLY", "L_CTX", "ProjectOut",
           "kv_pack", "kv_unpack", "kv_migrate"]
