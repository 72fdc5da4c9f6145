"""ctypes binding of libmtk.so (the C ABI in include/minitransfer/mtk.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2011_09463_b200/csrc``).  There is no fallback: if the shared
object is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MTK_LIB_PATH") or os.path.join(_HERE, "libmtk.so")  # override: A/B diagnostics

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for this path)")

lib = C.CDLL(LIB_PATH)

_vp = C.c_void_p
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)
_dpp = C.POINTER(_dp)
_u64p = C.POINTER(C.c_uint64)


class MtkStep(C.Structure):
    """mirrors mtk_step in mtk.h"""
    _fields_ = [
        ("X", _vp),
        ("y", _vp),
        ("w", _vp),
        ("B", C.c_int),
        ("src_rows", C.c_int),
        ("denom", C.c_double * 2),
        ("lr", C.c_double),
        ("frozen_layers", C.c_int),
        ("mmd_lambda", C.c_double),
        ("mmd_nb", C.c_int),
        ("mmd_mult", C.c_double * 8),
        ("optimizer", C.c_int),
        ("adam_beta1", C.c_double),
        ("adam_beta2", C.c_double),
        ("adam_eps", C.c_double),
    ]


class MtkSweepConfig(C.Structure):
    """mirrors mtk_sweep_config in mtk.h"""
    _fields_ = [
        ("paradigm", C.c_int),
        ("n_layers", C.c_int),
        ("dims", C.c_int * 9),
        ("n_shadows", C.c_int), ("pool", C.c_int), ("members", C.c_int), ("source_pool", C.c_int),
        ("source_per_model", C.c_int),
        ("batch", C.c_int), ("epochs", C.c_int), ("pretrain_epochs", C.c_int), ("frozen_layers", C.c_int),
        ("lr", C.c_double),
        ("optimizer", C.c_int),
        ("mmd_lambda", C.c_double), ("mu_scale", C.c_double), ("shift_scale", C.c_double),
        ("k", C.c_int), ("attack_hidden", C.c_int), ("attack_epochs", C.c_int), ("attack_batch", C.c_int),
        ("attack_lr", C.c_double),
        ("attack_optimizer", C.c_int),
        ("data_rng", C.c_int),
        ("seed", C.c_uint64),
    ]


class MtkSweepResult(C.Structure):
    """mirrors mtk_sweep_result in mtk.h"""
    _fields_ = [
        ("auc", C.c_double), ("accuracy", C.c_double),
        ("models", C.c_int), ("rank_model_begin", C.c_int), ("rank_model_end", C.c_int),
        ("n_queries", C.c_int64),
        ("seconds", C.c_double),
    ]


SIGNATURES = {
    "mtk_sweep_config_default": (None, [C.POINTER(MtkSweepConfig)]),
    "mtk_sweep_run": (C.c_int, [_vp, C.POINTER(MtkSweepConfig), _vp, C.POINTER(MtkSweepResult)]),
    "mtk_version": (C.c_int, []),
    "mtk_last_error": (C.c_char_p, []),
    "mtk_ctx_create": (C.c_int, [C.c_int, _vp, C.POINTER(_vp)]),
    "mtk_ctx_destroy": (C.c_int, [_vp]),
    "mtk_bank_reset_optimizer": (C.c_int, [_vp]),
    "mtk_bank_save": (C.c_int, [_vp, C.c_char_p]),
    "mtk_bank_load": (C.c_int, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "mtk_bank_info": (C.c_int, [_vp, _ip, _ip, _ip, _ip]),
    "mtk_sha256": (C.c_int, [_vp, C.c_size_t, _vp]),
    "mtk_philox4x64_fill": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                      C.c_int64, _vp]),
    "mtk_counter_normals": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, _vp]),
    "mtk_synth_counter": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int64, _vp,
                                    _vp, _vp, _vp]),
    "mtk_bank_grad_size": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "mtk_bank_compute_grads": (C.c_int, [_vp, C.POINTER(MtkStep), _vp, _dp, _dp]),
    "mtk_bank_dp_apply": (C.c_int, [_vp, C.POINTER(MtkStep), _vp, C.c_int, C.c_int64]),
    "mtk_bank_fingerprint": (C.c_int, [_vp, C.POINTER(C.c_uint64)]),
    "mtk_bank_train_epoch": (C.c_int, [_vp, C.POINTER(MtkStep), _vp, _vp, C.c_int64, _vp, _vp, _dp,
                                       C.c_int]),
    "mtk_gather_rows": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, _vp, C.c_int, C.c_int, _vp, C.c_int,
                                  C.c_int]),
    "mtk_ctx_synchronize": (C.c_int, [_vp]),
    "mtk_ctx_launch_count": (C.c_int, [_vp, _u64p]),
    "mtk_ctx_set_timing": (C.c_int, [_vp, C.c_int]),
    "mtk_ctx_phase_times": (C.c_int, [_vp, _dp, _u64p]),
    "mtk_rng_create": (C.c_int, [C.c_uint64, C.POINTER(_vp)]),
    "mtk_rng_destroy": (C.c_int, [_vp]),
    "mtk_rng_split": (C.c_int, [_vp, C.c_uint64, C.POINTER(_vp)]),
    "mtk_rng_next_u64": (C.c_uint64, [_vp]),
    "mtk_rng_uniform": (C.c_double, [_vp, C.c_double, C.c_double]),
    "mtk_rng_normal": (C.c_double, [_vp]),
    "mtk_rng_below": (C.c_uint64, [_vp, C.c_uint64]),
    "mtk_rng_permutation": (C.c_int, [_vp, C.c_uint64, _u64p]),
    "mtk_rng_fill_normal": (C.c_int, [_vp, _dp, C.c_uint64]),
    "mtk_synth": (C.c_int, [_vp, C.c_int, C.c_int, C.c_uint64, _dp, _dp, _dp, _vp, _vp]),
    "mtk_bank_create": (C.c_int, [_vp, C.c_int, C.c_int, _ip, C.c_int, C.POINTER(_vp)]),
    "mtk_bank_destroy": (C.c_int, [_vp]),
    "mtk_bank_set_params": (C.c_int, [_vp, C.c_int, _dpp, _dpp]),
    "mtk_bank_get_params": (C.c_int, [_vp, C.c_int, _dpp, _dpp]),
    "mtk_bank_init_params": (C.c_int, [_vp, C.c_int, _vp]),
    "mtk_bank_param_device": (C.c_int, [_vp, C.c_int, C.POINTER(_vp), C.POINTER(_vp)]),
    "mtk_bank_forward": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp]),
    "mtk_bank_train_step": (C.c_int, [_vp, C.POINTER(MtkStep), _dp, _dp]),
    "mtk_bank_train_step_host": (C.c_int, [_vp, C.POINTER(MtkStep), _vp, _vp, _vp, _dp, _dp]),
    "mtk_bank_train_step_host_async": (C.c_int, [_vp, C.POINTER(MtkStep), _vp, _vp, _vp]),
    "mtk_bank_step_result": (C.c_int, [_vp, C.c_int, _dp, _dp]),
    "mtk_bank_tc_layers": (C.c_int, [_vp, _ip]),
    "mtk_bank_set_keep_grads": (C.c_int, [_vp, C.c_int]),
    "mtk_bank_get_grads": (C.c_int, [_vp, C.c_int, _dpp, _dpp]),
    "mtk_mmd_gaussian": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int, _dp, C.c_int,
                                   C.c_double, _dp, _dp, _vp, _vp]),
    "mtk_mmd_gaussian_rows": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int, _dp,
                                        C.c_int, C.c_double, C.c_int64, C.c_int64, _dp, _vp,
                                        _vp]),
    "mtk_mmd_beta": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int, _dp]),
    "mtk_softmax": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, _vp]),
    "mtk_posterior_features": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, C.c_int, _vp, _vp]),
    "mtk_posterior_column": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, C.c_int, _vp]),
    "mtk_auc": (C.c_int, [_vp, _vp, _vp, C.c_int64, _dp, _dp]),
    "mtk_attack_auc": (C.c_int, [_vp, _vp, C.c_int64, C.c_int, _vp, _dp, _dp, _vp]),
    "mtk_mmd_gaussian_tiles": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int, _dp, C.c_int,
                                         C.c_double, C.c_int64, C.c_int64, _dp, _vp, _vp]),
    "mtk_mmd_value_from_tile_partials": (C.c_int, [_dp, C.c_int64, C.c_int64, C.c_int64, _dp]),
    "mtk_comm_unique_id": (C.c_int, [_vp]),
    "mtk_comm_init": (C.c_int, [C.c_int, C.c_int, _vp, C.POINTER(_vp)]),
    "mtk_comm_destroy": (C.c_int, [_vp]),
    "mtk_comm_info": (C.c_int, [_vp, _ip, _ip, _ip, _ip]),
    "mtk_allgather": (C.c_int, [_vp, _vp, _vp, _vp, C.c_size_t]),
    "mtk_diag_gemm_tf32x3": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       _vp, _vp, _vp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
