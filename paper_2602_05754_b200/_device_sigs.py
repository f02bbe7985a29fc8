"""ctypes signatures of libpf_device.so (include/pf_device.h) beyond the GEMM entry points."""
import ctypes

c_int = ctypes.c_int
c_ll = ctypes.c_longlong
c_f = ctypes.c_float
c_d = ctypes.c_double
c_vp = ctypes.c_void_p
c_cp = ctypes.c_char_p


class PfModelCfg(ctypes.Structure):
    _fields_ = [(n, c_int) for n in ("hidden", "ffn", "n_heads", "n_kv_heads", "head_dim", "vocab", "layers", "seq",
                                     "micro_batch")] + [("rope_theta", c_f), ("norm_eps", c_f), ("init_std", c_f)] + \
        [(n, c_int) for n in ("family", "image", "patch", "channels")]


class PfTrainCfg(ctypes.Structure):
    _fields_ = [("kind", c_int), ("ranks", c_int), ("stages_per_rank", c_int), ("microbatches", c_int),
                ("rank", c_int), ("phases", c_int * 4), ("r_max", c_d), ("lr", c_d), ("seed", ctypes.c_uint64),
                ("apf", c_int), ("apf_every", c_int), ("apf_alpha", c_f), ("apf_threshold", c_f),
                ("device", c_int), ("mask_threads", c_int), ("hybrid", c_int), ("hybrid_unit_fraction", c_f),
                ("optimizer", c_int), ("beta1", c_d), ("beta2", c_d), ("eps", c_f), ("weight_decay", c_f)]


class PfStepResult(ctypes.Structure):
    _fields_ = [("loss", c_d), ("batch_ms", c_d), ("optimizer_ms", c_d), ("predicted_ms", c_d),
                ("mean_ratio", c_d), ("mask_ms", c_d), ("frozen_units", c_ll), ("total_units", c_ll),
                ("phase", c_int)]


class PfTrainerInfo(ctypes.Structure):
    _fields_ = [("tokens_per_step", c_ll), ("params", c_ll), ("unit_params", c_ll),
                ("matmul_flops_fwd_per_mb", c_ll), ("units", c_int), ("local_stages", c_int), ("actions", c_int),
                ("lp_solve_ms", c_d)]


DEVICE_SIGNATURES = {
    "pf_engine_last_error": ([], c_cp),
    "pf_mask_to_unit_lists": ([c_vp, c_vp, c_int, c_vp, c_vp, c_vp], c_int),
    "pf_mask_to_pair_lists": ([c_vp, c_vp, c_int, c_vp, c_vp, c_vp], c_int),
    "pf_mask_to_rowpair_lists": ([c_vp, c_vp, c_int, c_vp, c_vp, c_vp], c_int),
    "pf_masked_sgd_units": ([c_vp, c_vp, c_vp, c_vp, c_int, c_f, c_vp, c_int, c_int, c_vp, c_vp, c_f, c_f, c_vp,
                             c_vp], c_int),
    "pf_sgd_dense": ([c_vp, c_vp, c_vp, c_ll, c_f, c_vp], c_int),
    "pf_apf_update": ([c_vp, c_vp, c_vp, c_vp, c_ll, c_f, c_vp], c_int),
    "pf_rmsnorm_fwd": ([c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_f, c_vp], c_int),
    "pf_rmsnorm_bwd": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_vp], c_int),
    "pf_swiglu_fwd": ([c_vp, c_vp, c_int, c_int, c_vp], c_int),
    "pf_gemm_swiglu": ([c_vp, c_ll, c_vp, c_ll, c_vp, c_vp, c_int, c_int, c_int, c_vp], c_int),
    "pf_gemm_set_streamk": ([c_int], c_int),
    "pf_flash_attn_fwd": ([c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_f, c_int, c_vp], c_int),
    "pf_flash_attn_bwd": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_f, c_int, c_f, c_vp],
                          c_int),
    "pf_flash_attn_prof": ([c_vp], c_int),
    "pf_vit_attn_fwd": ([c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_f, c_vp], c_int),
    "pf_vit_attn_bwd": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_f, c_vp], c_int),
    "pf_layernorm_fwd": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_f, c_vp], c_int),
    "pf_layernorm_bwd": ([c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_vp], c_int),
    "pf_gelu_fwd": ([c_vp, c_vp, c_ll, c_vp], c_int),
    "pf_gelu_bwd": ([c_vp, c_vp, c_vp, c_ll, c_vp], c_int),
    "pf_gemm_rope": ([c_vp, c_ll, c_vp, c_ll, c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_f, c_vp], c_int),
    "pf_gemm_gelu": ([c_vp, c_ll, c_vp, c_ll, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_vp], c_int),
    "pf_gemm_dgelu": ([c_vp, c_ll, c_vp, c_ll, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_vp], c_int),
    "pf_gemm_dswiglu": ([c_vp, c_ll, c_vp, c_ll, c_vp, c_vp, c_int, c_int, c_int, c_vp], c_int),
    "pf_swiglu_bwd": ([c_vp, c_vp, c_vp, c_int, c_int, c_vp], c_int),
    "pf_rope_fwd": ([c_vp, c_int, c_int, c_int, c_int, c_int, c_f, c_vp], c_int),
    "pf_cross_entropy": ([c_vp, c_vp, c_vp, c_int, c_int, c_f, c_f, c_vp], c_int),
    "pf_trainer_create": ([ctypes.POINTER(PfModelCfg), ctypes.POINTER(PfTrainCfg), ctypes.POINTER(c_vp)], c_int),
    "pf_trainer_destroy": ([c_vp], c_int),
    "pf_trainer_step": ([c_vp, c_int, c_vp, c_vp, ctypes.POINTER(PfStepResult)], c_int),
    "pf_trainer_step_masks": ([c_vp, c_int, c_vp, c_vp, c_vp, ctypes.POINTER(PfStepResult)], c_int),
    "pf_trainer_set_override": ([c_vp, c_d], c_int),
    "pf_trainer_set_plan": ([c_vp, c_vp], c_int),
    "pf_trainer_get_plan": ([c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "pf_trainer_action_ms": ([c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
    "pf_trainer_get_info": ([c_vp, ctypes.POINTER(PfTrainerInfo)], c_int),
    "pf_trainer_stage_buffers": ([c_vp, c_int, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                                  ctypes.POINTER(c_vp), ctypes.POINTER(c_ll), ctypes.POINTER(c_int)], c_int),
    "pf_trainer_last_masks": ([c_vp, c_int, c_vp], c_int),
    "pf_trainer_optim_state": ([c_vp, c_int, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)],
                               c_int),
    "pf_trainer_stream": ([c_vp], c_vp),
    "pf_nccl_unique_ids": ([c_vp, c_int], c_int),
    "pf_attention_backend": ([], c_cp),
    "pf_trainer_action_starts": ([c_vp, c_vp], c_int),
    "pf_trainer_apf_base": ([c_vp, c_int, c_vp], c_int),
    "pf_trainer_init_comm": ([c_vp, c_vp, c_int, c_int], c_int),
    "pf_device_launch_count": ([], c_ll),
    "pf_probe_enable": ([c_int], c_int),
    "pf_trainer_comm_ids": ([c_vp, ctypes.POINTER(c_int)], c_int),
    "pf_trainer_links": ([c_vp, c_vp], c_int),
    "pf_probe_read": ([ctypes.POINTER(c_int), ctypes.POINTER(c_d)], c_int),
}


def register(lib, sig) -> None:
    for name, (args, res) in DEVICE_SIGNATURES.items():
        sig(lib, name, args, res)
