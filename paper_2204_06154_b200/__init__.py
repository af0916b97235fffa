"""B200-native (sm_100a, fp64) MGM solve path of arXiv 2204.06154.

The product is ``libmgm.so`` (C ABI in ``include/mgm.h``); ``paper_2204_06154_b200.mgm`` is
its thin ctypes binding.  Importing this package loads the library and fails loudly if it
has not been built -- there is no CPU or PyTorch fallback.
"""
from .mgm import (MGM, MGMError, load_library, mgm_setup, mgm_vcycle, mgm_solve, mgm_solve_host,
                  mgm_destroy, mgm_num_levels, mgm_level_info, mgm_export_level,
                  mgm_export_weights, mgm_apply, mgm_timing_enable, mgm_timing_read,
                  mgm_bytes_model, mgm_vcycle_kernel_count, mgm_trace_read, mgm_bottom_trace_read, mgm_bottom_ftrace_read,
                  mgm_nccl_unique_id, mgm_dist_attach, mgm_vcycle_batch, mgm_solve_batch,
                  mgm_dense_bottom_info, torch_allocator, mgm_local_rows, mgm_dist_info, mgm_dist_comm_time,
                  mgm_fake_group_create, mgm_fake_group_destroy, mgm_dist_attach_fake, EXPORTED, LIB_PATH)

load_library()

__all__ = ["MGM", "MGMError", "load_library", "mgm_setup", "mgm_vcycle", "mgm_solve",
           "mgm_solve_host", "mgm_destroy", "mgm_num_levels", "mgm_level_info",
           "mgm_export_level", "mgm_export_weights", "mgm_apply", "mgm_timing_enable",
           "mgm_timing_read", "mgm_bytes_model", "mgm_vcycle_kernel_count", "mgm_trace_read", "mgm_bottom_trace_read", "mgm_bottom_ftrace_read", "mgm_nccl_unique_id", "mgm_dist_attach", "mgm_vcycle_batch", "mgm_solve_batch", "mgm_dense_bottom_info", "torch_allocator", "mgm_local_rows", "mgm_dist_info", "mgm_dist_comm_time",
           "mgm_fake_group_create", "mgm_fake_group_destroy", "mgm_dist_attach_fake", "EXPORTED",
           "LIB_PATH"]
