"""B200-native STTSV on the blowup tensor of a non-uniform hypergraph
(arXiv 2311.08595).  The product is the C-ABI library libsttsv.so
(include/sttsv.h); this package is its thin Python binding."""
from .sttsv import (MAX_RANK, STTSV_BATCH_FUSED, STTSV_NO_PREFIX_MEMO, STTSV_CANONICALIZE, STTSV_DETERMINISTIC, STTSV_MERGE_DUPLICATES, Plan, SttsvError,
                    exported_symbols, load, sttsv_apply, sttsv_apply_batch, sttsv_apply_host, sttsv_apply_launches, sttsv_comm_create,
                    sttsv_comm_destroy, sttsv_comm_unique_id, sttsv_destroy, sttsv_last_error, sttsv_plan_create,
                    sttsv_plan_destroy, sttsv_plan_info, sttsv_hec, sttsv_plan_profile, sttsv_plan_profile_read,
                    sttsv_power_iterate, sttsv_shard_edges, sttsv_status_string, sttsv_version)

__all__ = ["MAX_RANK", "STTSV_BATCH_FUSED", "STTSV_NO_PREFIX_MEMO", "STTSV_CANONICALIZE", "STTSV_DETERMINISTIC", "STTSV_MERGE_DUPLICATES", "Plan", "SttsvError",
           "exported_symbols", "load", "sttsv_apply", "sttsv_apply_batch", "sttsv_apply_host", "sttsv_apply_launches", "sttsv_comm_create",
           "sttsv_comm_destroy", "sttsv_comm_unique_id", "sttsv_destroy", "sttsv_last_error", "sttsv_plan_create",
           "sttsv_plan_destroy", "sttsv_plan_info", "sttsv_hec", "sttsv_plan_profile", "sttsv_plan_profile_read",
           "sttsv_power_iterate", "sttsv_shard_edges", "sttsv_status_string", "sttsv_version"]
