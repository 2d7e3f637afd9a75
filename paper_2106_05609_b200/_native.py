"""ctypes binding of libgasb.so (the C ABI declared in include/gasb.h).

The product path is native: if the shared library is missing this module raises at import
time — there is no Python or CPU fallback for any kernel.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("GASB_LIB", _PKG / "libgasb.so"))

if not LIB_PATH.exists():
    raise ImportError(
        f"libgasb.so not found at {LIB_PATH}: build it with `python paper_2106_05609_b200/build.py` "
        "(nvcc, sm_100a). There is no fallback implementation."
    )

lib = C.CDLL(str(LIB_PATH))

i32, i64, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
vp = C.c_void_p
P = C.POINTER

OK, INVALID_ARGUMENT, LOGIC_ERROR, RUNTIME_ERROR, CUDA_ERROR = 0, 1, 2, 3, 4


class GasbCudaError(RuntimeError):
    pass


def check(status: int) -> None:
    """Maps gasb_status onto the reference's exception types."""
    if status == OK:
        return
    msg = lib.gasb_last_error().decode(errors="replace")
    if status == INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == LOGIC_ERROR:
        raise RuntimeError(f"logic_error: {msg}")  # std::logic_error
    if status == CUDA_ERROR:
        raise GasbCudaError(msg)
    raise RuntimeError(msg)  # std::runtime_error


class SynthParams(C.Structure):
    _fields_ = [("num_nodes", i32), ("num_communities", i32), ("num_pairs", i64), ("intra_fraction", f64),
                ("gamma", f64), ("min_weight", f64), ("max_weight", f64), ("seed", u64)]


class ModelSpecC(C.Structure):
    _fields_ = [("kind", i32), ("num_layers", i32), ("hidden", i32), ("dropout", f32), ("alpha", f32),
                ("beta", f32), ("l2_weight", f32), ("clip_max_norm", f32), ("lr", f32), ("beta1", f32),
                ("beta2", f32), ("eps", f32), ("seed", u64)]


class TrainerOptionsC(C.Structure):
    _fields_ = [("seg_edges", i32), ("fused", i32), ("prefetch", i32), ("use_graphs", i32),
                ("hoist_layer1", i32), ("device", i32), ("dropout_rng", i32), ("cross_batch", i32)]


class EpochReportC(C.Structure):  # gasb_epoch_report
    _fields_ = [("epoch", i64), ("loss", f64), ("peak_floats", i64), ("edges_per_layer", i64),
                ("device_bytes", i64), ("num_batches", i32), ("staleness_layers", i32)]


class LayerConfigC(C.Structure):  # gasb_layer_config
    _fields_ = [("kind", i32), ("in_dim", i32), ("out_dim", i32), ("alpha", f32), ("beta", f32)]


_SIGS = {
    "gasb_last_error": (C.c_char_p, []),
    "gasb_abi_version": (i32, []),
    "gasb_graph_build": (i32, [vp, vp, i64, i32, i32, P(vp)]),
    "gasb_graph_from_csr": (i32, [i32, vp, vp, i32, P(vp)]),
    "gasb_graph_info": (i32, [vp, P(i32), P(i64)]),
    "gasb_graph_csr": (i32, [vp, P(vp), P(vp)]),
    "gasb_graph_destroy": (i32, [vp]),
    "gasb_synth_pairs": (i32, [P(SynthParams), vp, vp, vp]),
    "gasb_synth_features": (i32, [i64, i32, i64, u64, vp]),
    "gasb_schedule_build": (i32, [vp, vp, i32, i32, P(vp)]),
    "gasb_schedule_build_batches": (i32, [vp, vp, vp, i32, i32, P(vp)]),
    "gasb_schedule_num_parts": (i32, [vp, P(i32)]),
    "gasb_schedule_timing": (i32, [vp, P(f64), P(f64)]),
    "gasb_plan_sizes": (i32, [vp, i32, vp]),
    "gasb_plan_copy": (i32, [vp, i32] + [vp] * 13),
    "gasb_schedule_destroy": (i32, [vp]),
    "gasb_partition_save": (i32, [C.c_char_p, vp, i32]),
    "gasb_partition_load": (i32, [C.c_char_p, i32, vp, P(i32)]),
    "gasb_random_partition": (i32, [i32, i32, u64, vp]),
    "gasb_cluster_partition": (i32, [vp, i32, u64, vp]),
    "gasb_history_create": (i32, [i32, i32, i32, P(vp)]),
    "gasb_history_destroy": (i32, [vp]),
    "gasb_history_info": (i32, [vp, P(i32), P(i32), P(i32), P(i64)]),
    "gasb_history_push": (i32, [vp, i32, vp, i64, vp, i64, vp]),
    "gasb_history_pull": (i32, [vp, i32, vp, i64, vp, i64, vp]),
    "gasb_history_push_host": (i32, [vp, i32, vp, i64, vp, vp]),
    "gasb_history_pull_host": (i32, [vp, i32, vp, i64, vp, vp]),
    "gasb_history_check": (i32, [vp]),
    "gasb_history_advance_step": (i32, [vp, vp]),
    "gasb_history_step": (i32, [vp, P(i64)]),
    "gasb_history_last_push_step": (i32, [vp, i32, i32, P(i64)]),
    "gasb_history_layer": (i32, [vp, i32, P(vp), P(i64)]),
    "gasb_history_fill_layer": (i32, [vp, i32, vp]),
    "gasb_history_read_layer": (i32, [vp, i32, vp]),
    "gasb_history_read_stamps": (i32, [vp, i32, vp]),
    "gasb_history_reset": (i32, [vp]),
    "gasb_history_staleness": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "gasb_history_save": (i32, [vp, C.c_char_p]),
    "gasb_history_load": (i32, [C.c_char_p, P(vp)]),
    "gasb_prefetcher_create": (i32, [vp, P(vp)]),
    "gasb_prefetcher_destroy": (i32, [vp]),
    "gasb_prefetch_begin": (i32, [vp, vp, i64, vp, P(u64)]),
    "gasb_prefetch_wait": (i32, [vp, u64, i32, vp, P(vp), P(i64)]),
    "gasb_spmm_fwd": (i32, [vp, i32, vp, vp, vp, i32, i64, i32, vp, i64, i32, vp]),
    "gasb_spmm_bwd": (i32, [vp, i32, vp, vp, vp, i64, i32, i32, vp, i64, vp, i64, vp]),
    "gasb_gemm": (i32, [i32, i32, i32, i32, vp, i64, vp, i64, vp, i64, f32, vp]),
    "gasb_spmm_max_fwd": (i32, [vp, i32, vp, vp, i32, i64, i32, vp, i64, vp, i64, vp]),
    "gasb_spmm_max_bwd": (i32, [vp, i32, vp, vp, i64, vp, i64, i32, i32, vp, i64, vp]),
    "gasb_spmm_mean_fwd": (i32, [vp, i32, vp, vp, i32, i64, i32, vp, i64, vp]),
    "gasb_mean_coefficients": (i32, [vp, i32, vp]),
    "gasb_batch_ops_create": (i32, [vp, i32, i32, P(vp)]),
    "gasb_batch_ops_sizes": (i32, [vp, P(i32), P(i32)]),
    "gasb_batch_ops_destroy": (i32, [vp]),
    "gasb_layer_fwd": (i32, [vp, P(LayerConfigC), vp, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp]),
    "gasb_layer_bwd": (i32, [vp, P(LayerConfigC), vp, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, i64,
                             vp]),
    "gasb_trainer_create": (i32, [vp, vp, i32, vp, vp, i32, P(ModelSpecC), P(TrainerOptionsC), P(vp)]),
    "gasb_trainer_destroy": (i32, [vp]),
    "gasb_gas_epoch": (i32, [vp, i64, i32, P(f64)]),
    "gasb_gas_epoch_async": (i32, [vp, i64, i32]),
    "gasb_gas_epoch_range_async": (i32, [vp, i64, i32, i32, i32]),
    "gasb_trainer_part_losses": (i32, [vp, vp]),
    "gasb_trainer_dropout_mask": (i32, [vp, i32, i64, i32, vp]),
    "gasb_gas_epoch_report": (i32, [vp, i64, i32, i32, P(EpochReportC), vp, vp]),
    "gasb_adam_step": (i32, [vp, vp, vp, vp, i64, i64, f32, f32, f32, f32, vp]),
    "gasb_grad_clip": (i32, [vp, i64, f64, P(f64), vp]),
    "gasb_trainer_last_loss": (i32, [vp, P(f64)]),
    "gasb_trainer_batch": (i32, [vp, i32, i64, i32, i32, vp, vp, P(f64), vp, P(i32)]),
    "gasb_trainer_num_param_floats": (i32, [vp, P(i64)]),
    "gasb_trainer_get_params": (i32, [vp, vp]),
    "gasb_trainer_set_params": (i32, [vp, vp]),
    "gasb_trainer_history": (i32, [vp, P(vp)]),
    "gasb_trainer_stream": (i32, [vp, P(vp)]),
    "gasb_trainer_launch_count": (i32, [vp, P(i64)]),
    "gasb_trainer_set_features": (i32, [vp, vp]),
    "gasb_trainer_stage_features": (i32, [vp, vp]),
    "gasb_trainer_commit_features": (i32, [vp]),
    "gasb_trainer_profile_spmm": (i32, [vp, i32, i32, i32, P(f32)]),
    "gasb_host_register": (i32, [vp, C.c_size_t]),
    "gasb_host_unregister": (i32, [vp]),
    "gasb_trainer_evaluate": (i32, [vp, vp, vp, vp, vp]),
    "gasb_trainer_full_logits": (i32, [vp, vp]),
    "gasb_trainer_infer_from_history": (i32, [vp, vp, P(i32)]),
    "gasb_dp_create": (i32, [vp, i32, i32, P(vp)]),
    "gasb_dp_create_ex": (i32, [vp, i32, i32, i32, P(vp)]),
    "gasb_dp_read_history": (i32, [vp, i32, vp]),
    "gasb_dp_traffic": (i32, [vp, P(i64), P(i64), P(i64)]),
    "gasb_dp_shard_map": (i32, [vp, i32, vp, vp]),
    "gasb_dp_export": (i32, [vp, vp]),
    "gasb_dp_connect": (i32, [vp, vp]),
    "gasb_dp_epoch_async": (i32, [vp, i64, i32]),
    "gasb_dp_check": (i32, [vp]),
    "gasb_dp_last_losses": (i32, [vp, vp]),
    "gasb_dp_launch_count": (i32, [vp, P(i64)]),
    "gasb_dp_destroy": (i32, [vp]),
    "gasb_epoch_order": (i32, [i32, u64, i64, i32, vp]),
}

DP_HANDLE_BYTES = 64  # GASB_DP_HANDLE_BYTES

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def ptr(a) -> int | None:
    """Address of a numpy array / torch tensor / None."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
