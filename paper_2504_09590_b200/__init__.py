"""BROS bidirectional paged decode attention for B200 (sm_100a).

The product is libbkv.so (include/bkv.h); this package is its thin Python
binding (``bkv``) plus the head-sharded multi-GPU wrapper (``tp``).
"""
from .bkv import (DecodePlan, decode_plan, decode_plan_host, plan_used_bytes, decode_planned, reload_dev_switches, KVPool, kv_append, kv_append_checkpoint, kv_checkpoint, kv_restore, paged_decode_attention, paged_prefill_attention, paged_mixed_attention, decode_step, decode_multi_out, peer_barrier, decode_workspace_size, workspace,
                  validate_layout_host, validate_block_map_host, block_map, lib, BkvError, BKV_DIR_FWD, BKV_DIR_REV, LIB_PATH)

__all__ = ["DecodePlan", "decode_plan", "decode_plan_host", "plan_used_bytes", "decode_planned", "reload_dev_switches", "KVPool", "kv_append", "kv_append_checkpoint", "kv_checkpoint", "kv_restore", "paged_decode_attention", "paged_prefill_attention", "paged_mixed_attention", "decode_step", "decode_multi_out", "peer_barrier", "decode_workspace_size", "workspace",
           "validate_layout_host", "validate_block_map_host", "block_map", "lib", "BkvError", "BKV_DIR_FWD", "BKV_DIR_REV",
           "LIB_PATH"]
