"""ctypes signatures of libpf_host.so (include/pipefreeze_c.h)."""
import ctypes

c_int = ctypes.c_int
c_d = ctypes.c_double
c_vp = ctypes.c_void_p
c_u64 = ctypes.c_uint64
c_cp = ctypes.c_char_p

HOST_SIGNATURES = {
    "pf_last_error": ([], c_cp),
    "pf_schedule_build": ([c_int, c_int, c_int, c_int, c_vp, c_vp], c_int),
    "pf_stage_to_rank": ([c_int, c_int, c_int, c_int, c_int, c_vp], c_int),
    "pf_issue_program": ([c_int, c_int, c_int, c_int, c_int, c_vp, c_vp], c_int),
    "pf_dag_build": ([c_int, c_int, c_int, c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_int], c_int),
    "pf_longest_path": ([c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp], c_int),
    "pf_critical_path": ([c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp], c_int),
    "pf_phase_of": ([c_int, c_vp, c_vp], c_int),
    "pf_actual_freeze_ratio": ([c_int, c_vp, c_d, c_vp], c_int),
    "pf_rng_u64": ([c_u64, c_int, c_vp], c_int),
    "pf_sample_masks": ([c_u64, c_int, c_int, c_vp, c_vp], c_int),
    "pf_reconcile_mask": ([c_u64, c_int, c_vp, c_int, c_vp], c_int),
    "pf_freezing_masks_horizon": ([c_int, c_int, c_vp, c_vp, c_int, c_u64, c_vp, c_vp], c_int),
    "pf_mask_stream_stage_step": ([c_int, c_int, c_vp, c_vp, c_int, c_u64, c_int, c_int, c_vp, c_int, c_vp], c_int),
    "pf_mask_stream_stage_step_units": ([c_int, c_int, c_vp, c_vp, c_vp, c_u64, c_int, c_int, c_vp, c_int, c_vp],
                                        c_int),
    "pf_mask_stream_offset": ([c_int, c_int, c_vp, c_vp, c_int, c_u64, c_int, c_int, c_int, c_vp], c_int),
    "pf_plan_solve": ([c_int, c_int, c_int, c_int, c_vp, c_vp, c_d, c_int, c_int, c_vp, c_vp, c_vp, c_vp], c_int),
    "pf_plan_verify": ([c_int, c_int, c_int, c_int, c_vp, c_vp, c_d, c_vp, c_vp, c_d, c_vp, c_vp], c_int),
    "pf_plan_weights": ([c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_d, c_vp], c_int),
    "pf_monitor_aggregate": ([c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "pf_simulate_monitoring": ([c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_d, c_u64, c_vp, c_vp], c_int),
    "pf_apf_update_host": ([c_int, c_d, c_vp, c_vp, c_vp, c_vp], c_int),
    "pf_masked_sgd_host": ([c_int, c_vp, c_vp, c_d, c_int, c_int, c_d, c_int, c_d, c_u64, c_vp, c_vp], c_int),
    "pf_autofreeze_score": ([c_d, c_d, c_vp], c_int),
    "pf_autofreeze_select": ([c_vp, c_int, c_int, c_d, c_vp], c_int),
    "pf_masked_sgd_plan_host": ([c_int, c_vp, c_vp, c_d, c_int, c_int, c_d, c_int, c_vp, c_vp, c_int, c_u64, c_vp,
                                 c_vp], c_int),
}


def register(lib, sig) -> None:
    for name, (args, res) in HOST_SIGNATURES.items():
        sig(lib, name, args, res)
