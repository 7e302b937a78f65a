"""ctypes binding of libvericache.so (the C-ABI in include/vc_api.h).

The product path is the CUDA library; there is no Python or CPU fallback.
Loading fails loudly when the shared object is missing.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VC_LIB", os.path.join(_HERE, "libvericache.so"))

VC_OK, VC_ERR_CONFIG, VC_ERR_CONTRACT, VC_ERR_CUDA = 0, 1, 2, 3


class VcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[vc status {code}] {msg}")
        self.code = code


class ConfigError(VcError):
    """speckv::ConfigError -- bad input (compressor.cpp / config.cpp messages)."""


class ContractError(VcError):
    """speckv::ContractError -- API misuse."""


class CudaError(VcError):
    """A device failure."""


class ModelDesc(C.Structure):
    _fields_ = [("vocab", C.c_int), ("hidden", C.c_int), ("layers", C.c_int), ("n_q", C.c_int),
                ("n_kv", C.c_int), ("d_head", C.c_int), ("ffn", C.c_int),
                ("rope_theta", C.c_float), ("rms_eps", C.c_float)]


class RuntimeDesc(C.Structure):
    _fields_ = [("max_slots", C.c_int), ("max_ctx", C.c_int), ("max_x", C.c_int),
                ("quant_bits", C.c_int), ("full_tier", C.c_int), ("n_stage", C.c_int),
                ("max_verify", C.c_int), ("use_graphs", C.c_int), ("drop_ratio", C.c_double),
                ("tp_size", C.c_int), ("tp_rank", C.c_int), ("drop_window", C.c_int),
                ("resident_slots", C.c_int), ("draft_depth", C.c_int),
                ("ring_chunks", C.c_int), ("max_streams", C.c_int),
                ("drop_score", C.c_int), ("snap_pool", C.c_int), ("snap_recent", C.c_int),
                ("host_pack", C.c_int)]


class CompressedMeta(C.Structure):
    _fields_ = [("bit_scheme", C.c_int), ("payload_bytes", C.c_int64), ("aux_bytes", C.c_int64),
                ("full_bytes", C.c_int64), ("n_groups", C.c_int), ("tail_tokens", C.c_int),
                ("retained_tokens", C.c_int64)]


class CompressorSpec(C.Structure):
    """vc_compressor_spec (speckv::CompressorSpec, compressor.hpp:24-41)."""
    _fields_ = [("kind", C.c_int), ("mode", C.c_int), ("bits", C.c_int), ("window", C.c_int),
                ("sink_tokens", C.c_int)]


class SeqState(C.Structure):
    _fields_ = [("live", C.c_int), ("committed", C.c_int), ("pending", C.c_int),
                ("n_groups", C.c_int), ("tail_committed", C.c_int), ("draft_len", C.c_int),
                ("drop_base", C.c_int), ("drop_len", C.c_int)]


class StepItem(C.Structure):
    _fields_ = [("slot", C.c_int), ("mode", C.c_int), ("n_tokens", C.c_int), ("stage", C.c_int),
                ("tokens", C.POINTER(C.c_int32))]


class RequestDesc(C.Structure):
    _fields_ = [("n_ctx", C.c_int), ("first_token", C.c_int32), ("seed", C.c_uint64), ("arrival_ms", C.c_double)]


class SchedDesc(C.Structure):
    _fields_ = [("x", C.c_int), ("window", C.c_int), ("iteration_time", C.c_double),
                ("link_bandwidth", C.c_double), ("hbm_capacity", C.c_int64), ("K", C.c_int),
                ("warmup_iterations", C.c_int64), ("timed_iterations", C.c_int64),
                ("x_resident", C.c_int), ("arrivals", C.POINTER(RequestDesc)), ("n_arrivals", C.c_int),
                ("ngram", C.c_int), ("depth", C.c_int)]


class SchedStats(C.Structure):
    _fields_ = [("wall_ms", C.c_double), ("tokens", C.c_int64), ("iterations", C.c_int64),
                ("verifies", C.c_int64), ("late_transfers", C.c_int64), ("h2d_bytes", C.c_double),
                ("h2d_ms", C.c_double), ("verify_wait_ms", C.c_double), ("mean_accept", C.c_double),
                ("timed_iterations", C.c_int64), ("timed_tokens", C.c_int64),
                ("timed_wall_ms", C.c_double), ("timed_device_ms", C.c_double),
                ("timed_rows", C.c_double), ("timed_step_device_ms", C.c_double),
                ("resident_verifies", C.c_int64), ("resident_accept", C.c_double),
                ("timed_resident_tokens", C.c_int64), ("timed_verifies", C.c_int64),
                ("timed_verify_rows", C.c_double), ("throughput", C.c_double),
                ("warm_throughput", C.c_double), ("p50_latency_s", C.c_double), ("p99_latency_s", C.c_double),
                ("interconnect_busy", C.c_double), ("peak_hbm_bytes", C.c_int64),
                ("staging_bytes", C.c_int64), ("drafted_tokens", C.c_int64),
                ("aux_proposed", C.c_int64), ("aux_accepted", C.c_int64), ("reload_over_full", C.c_double)]


class LoopMetrics(C.Structure):
    """vc_loop_metrics (SimMetrics, sim.hpp:52-74)."""
    _fields_ = [("throughput", C.c_double), ("warm_throughput", C.c_double), ("p50_latency_s", C.c_double),
                ("p99_latency_s", C.c_double), ("tokens", C.c_int64), ("iterations", C.c_int64),
                ("completed", C.c_int64), ("unserved", C.c_int64), ("clock_s", C.c_double),
                ("wall_ms", C.c_double), ("mean_batch", C.c_double), ("max_batch", C.c_int),
                ("peak_hbm_bytes", C.c_int64), ("full_batch_throughput", C.c_double)]


class ComposeStats(C.Structure):
    _fields_ = [("rounds", C.c_int64), ("verifies", C.c_int64), ("tokens", C.c_int64), ("draft_steps", C.c_int64),
                ("drafted", C.c_int64), ("aux_proposed", C.c_int64), ("aux_accepted", C.c_int64),
                ("mean_accept", C.c_double), ("ms", C.c_double)]



class RemoteDesc(C.Structure):
    _fields_ = [("x", C.c_int), ("K", C.c_int), ("baseline", C.c_int), ("link_queue", C.c_int),
                ("arrival_gap_ms", C.c_double), ("first_tokens", C.POINTER(C.c_int32)),
                ("payload_order", C.c_int)]


class RemoteStats(C.Structure):
    _fields_ = [("makespan_ms", C.c_double), ("wall_ms", C.c_double), ("tokens", C.c_int64),
                ("iterations", C.c_int64), ("link_waits", C.c_int64), ("verifies", C.c_int64),
                ("mean_accept", C.c_double), ("ttft_ms_mean", C.c_double), ("ttft_ms_max", C.c_double),
                ("compressed_ready_ms_mean", C.c_double), ("full_ready_ms_mean", C.c_double),
                ("h2d_bytes", C.c_double), ("h2d_ms", C.c_double)]


P = C.c_void_p
I, I64, U64, D, F = C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_float
PI, PI32, PI64, PU64, PD = (C.POINTER(C.c_int), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                            C.POINTER(C.c_uint64), C.POINTER(C.c_double))
PU16, PU32, PF = C.POINTER(C.c_uint16), C.POINTER(C.c_uint32), C.POINTER(C.c_float)
PPU16 = C.POINTER(PU16)

# name -> (restype, argtypes); every symbol include/vc_api.h declares.
SIGNATURES = {
    "vc_last_error": (C.c_char_p, []),
    "vc_version": (I, []),
    "vc_engine_create": (I, [C.POINTER(ModelDesc), C.POINTER(RuntimeDesc), I, C.POINTER(P)]),
    "vc_engine_destroy": (I, [P]),
    "vc_engine_init_weights": (I, [P, U64, F]),
    "vc_engine_init_weights_scaled": (I, [P, U64, F, F, F]),
    "vc_engine_load_weights": (I, [P, PU16, PPU16, PPU16, PPU16, PPU16, PPU16, PPU16, PPU16, PU16, PU16]),
    "vc_engine_stats": (I, [P, PU64, PU64]),
    "vc_engine_geometry": (I, [P, PI, PI]),
    "vc_engine_timing": (I, [P, PD, PI64, I]),
    "vc_kernel_bench": (I, [P, I, PI, I, I, PD, PD]),
    "vc_request_add_synthetic": (I, [P, I, I, C.c_int32, U64, I, F]),
    "vc_request_add_kv": (I, [P, I, I, C.c_int32, PU16, PU16]),
    "vc_request_prefill": (I, [P, I, PI32, I]),
    "vc_request_release": (I, [P, I]),
    "vc_request_state": (I, [P, I, C.POINTER(SeqState)]),
    "vc_request_history": (I, [P, I, PI32, I, PI]),
    "vc_compress": (I, [P, I, C.POINTER(CompressedMeta)]),
    "vc_compress_spec": (I, [P, I, C.POINTER(CompressorSpec), D, U64, C.POINTER(CompressedMeta)]),
    "vc_compressed_read": (I, [P, I, I, I, PU32, PU32, PU32, PU32, PU16, PU16]),
    "vc_compressed_geometry": (I, [P, PI, PI, PI, PI]),
    "vc_drop_kept": (I, [P, I, I, C.POINTER(C.c_int32), I, PI]),
    "vc_nccl_get_unique_id": (I, [C.POINTER(C.c_uint8)]),
    "vc_engine_attach_nccl": (I, [P, C.POINTER(C.c_uint8)]),
    "vc_tp_loopback_create": (I, [I, C.POINTER(P)]),
    "vc_tp_loopback_destroy": (I, [P]),
    "vc_engine_attach_loopback": (I, [P, P]),
    "vc_tp_collective_bench": (I, [P, I, I, PD]),
    "vc_drop_indices": (I64, [I, I, I, I64, D, U64, I, PI64]),
    "vc_update_window": (I, [I, I, I, I, PI64, PI64, PI64, PI64, PI64, I64, PI64]),
    "vc_topk_select": (I, [P, I, I, I, P, P]),
    "vc_key_scores": (I, [P, I, I, I, P, P, P]),
    "vc_pack_roundtrip": (I, [P, I, I, I, P, PI, P]),
    "vc_argmax_rows": (I, [P, I, I, P, P]),
    "vc_step": (I, [P, C.POINTER(StepItem), I, PI32, PF]),
    "vc_decode_step": (I, [P, PI, I, PI32]),
    "vc_draft_step": (I, [P, PI, I, PI32]),
    "vc_verify": (I, [P, PI, I, PI, PI32]),
    "vc_accept": (I, [PI32, PI32, I, PI32, PI, PI, PI]),
    "vc_accept_commit": (I, [P, I, PI32, I, PI32, PI]),
    "vc_swap_begin": (I, [P, I, I, PU64]),
    "vc_swap_poll": (I, [P, U64, PI]),
    "vc_stream_begin": (I, [P, I, PI]),
    "vc_stream_advance": (I, [P, I, PI, C.POINTER(C.c_int32)]),
    "vc_stream_accept": (I, [P, I, I, C.POINTER(C.c_int32), PI]),
    "vc_stream_abort": (I, [P, I]),
    "vc_engine_staging_bytes": (I, [P, C.POINTER(C.c_int64)]),
    "vc_drop_scores": (I, [P, I, I, PF, I]),
    "vc_obs_query": (I, [P, I, PU16]),
    "vc_run_decode": (I, [P, PI, I, I, PI32, PD]),
    "vc_run_speculative": (I, [P, PI, I, I, I, PI32, PI32, I, PI, PD]),
    "vc_run_speculative_ngram": (I, [P, PI, I, I, I, I, PI32, PI32, I, PI, PI, PD]),
    "vc_run_speculative_composed": (I, [P, PI, I, I, I, I, I, PI32, C.POINTER(ComposeStats)]),
    "vc_run_scheduled": (I, [P, PI, I, C.POINTER(SchedDesc), PI32, C.POINTER(SchedStats)]),
    "vc_prefix_store": (I, [P, I]),
    "vc_prefix_load": (I, [P, I, I, C.c_int32, PU64]),
    "vc_run_remote_prefix": (I, [P, PI, I, C.POINTER(RemoteDesc), PI32, C.POINTER(RemoteStats)]),
    "vc_run_decode_fifo": (I, [P, C.POINTER(RequestDesc), I, I, PI32, C.POINTER(LoopMetrics)]),
    "vc_reload_span": (I, [I64, D, D, PD, PI]),
    "vc_quant_kivi_slice": (I, [P, P, I, I, I, P, P, P, P, P]),
    "vc_attention_probe": (I, [P, I, I, I, P, I, I, PU16]),
    "vc_kv_read": (I, [P, I, I, I, I, I, I, PU16, PU16]),
    "vc_gemm_probe": (I, [P, I, I, P, I, P, P]),
    "vc_gemm_probe_epi": (I, [P, I, I, P, I, I, P, P]),
}

_lib = None


def load() -> C.CDLL:
    """Load libvericache.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `make -C paper_2605_17613_b200` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == VC_OK:
        return
    msg = load().vc_last_error().decode(errors="replace")
    cls = {VC_ERR_CONFIG: ConfigError, VC_ERR_CONTRACT: ContractError,
           VC_ERR_CUDA: CudaError}.get(rc, VcError)
    raise cls(rc, msg)
