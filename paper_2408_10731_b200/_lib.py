"""ctypes binding of libtrajopt_b200.so (the C-ABI in include/trajopt_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2408_10731_b200/csrc``).  There is no CPU fallback: if the
library is missing, or no CUDA device is present, every compute entry point
raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int32, c_int64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# TRO_LIB_PATH selects a tuning variant built by `make variant` (tools/tune_alg1.py)
LIB_PATH = os.environ.get("TRO_LIB_PATH") or os.path.join(_HERE, "libtrajopt_b200.so")

TRO_F64 = 0
TRO_F32 = 1
TRO_CONVERGED = 1
TRO_FACTOR_FAILED = 2
TRO_FLAG_NO_SCHEDULE = 1
TRO_FLAG_NO_TMA = 2
TRO_LAYOUT_ANGLE = 0
TRO_LAYOUT_UNIT = 1
TRO_LAYOUT_HALF = 2
TRO_EINVAL = -1
TRO_REFIT_PRIEST = 0
TRO_REFIT_CEM = 1

# every symbol include/trajopt_b200.h declares (checked by tests/test_lib_exports.py)
EXPORTS = (
    "tro_alg1_prime",
    "tro_alg1_init",
    "tro_alg1_iterate",
    "tro_alg1_iterate_n",
    "tro_alg1_linear_terms",
    "tro_kkt_apply_f64",
    "tro_topk_stable_f64",
    "tro_topk_workspace_bytes",
    "tro_fastmath_eval",
    "tro_priest_project_f64",
    "tro_priest_cost_f64",
    "tro_elite_update_f64",
    "tro_normal_philox_f64",
    "tro_cholesky_f64",
    "tro_fp64_fma_probe",
    "tro_ma_run",
    "tro_ma_qp_ozaki",
    "tro_b2_run",
    "tro_validate_f64",
    "tro_predict_tracks_f64",
    "tro_mpc_advance_f64",
    "tro_mpc_compact",
    "tro_version",
    "tro_error_string",
)


class Alg1Dims(ctypes.Structure):
    _fields_ = [
        ("n_members", c_int32),
        ("n_obs", c_int32),
        ("n_p", c_int32),
        ("m", c_int32),
        ("dim", c_int32),
        ("n_eq", c_int32),
        ("n_levels", c_int32),
        ("groups", c_int32),
        ("layout", c_int32),
        ("reserved", c_int32),
    ]


class Alg1Consts(ctypes.Structure):
    _fields_ = [
        ("P", c_void_p),
        ("tracks", c_void_p),
        ("shape_a", c_void_p),
        ("shape_b", c_void_p),
        ("kinv", c_void_p),
        ("level_rho", c_void_p),
        ("level_ok", c_void_p),
        ("q", c_void_p),
        ("bvals", c_void_p),
        ("line_u", c_void_p),
        ("line_v", c_void_p),
        ("level0", c_void_p),
        ("track_lin", c_void_p),
    ]


class Alg1Params(ctypes.Structure):
    _fields_ = [
        ("tol", c_double),
        ("rho_growth", c_double),
        ("rho_cap", c_double),
        ("stall_improvement", c_double),
        ("stall_window", c_int32),
        ("d_mode", c_int32),
        ("max_hist", c_int32),
        ("flags", c_int32),
    ]


class Alg1State(ctypes.Structure):
    _fields_ = [
        ("state", c_void_p),
        ("d", c_void_p),
        ("copies", c_void_p),
        ("xi", c_void_p),
        ("pos", c_void_p),
        ("sums", c_void_p),
        ("rho", c_void_p),
        ("rho_o", c_void_p),
        ("ring", c_void_p),
        ("res_norm", c_void_p),
        ("res_max", c_void_p),
        ("hist", c_void_p),
        ("level", c_void_p),
        ("iteration", c_void_p),
        ("last_change", c_void_p),
        ("n_hist", c_void_p),
        ("status", c_void_p),
        ("n_changes", c_void_p),
        ("split_scratch", c_void_p),
        ("split_ticket", c_void_p),
        ("order", c_void_p),
        ("n_order", c_void_p),
        ("level_used", c_void_p),
    ]


class PriestDims(ctypes.Structure):
    _fields_ = [
        ("n_samples", c_int64),
        ("n_p", c_int32),
        ("m", c_int32),
        ("dim", c_int32),
        ("n_obs", c_int32),
        ("n_eq", c_int32),
        ("n_inner", c_int32),
    ]


class PriestConsts(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("P", "Pd", "Pdd", "tracks", "shape_a", "shape_b", "kinv", "FtF", "b_eq",
                                        "s_min", "s_max", "mu", "draw_L", "line")] + [
        ("v_max", c_double),
        ("a_max", c_double),
        ("rho", c_double),
        ("has_bounds", c_int32),
        ("static_tracks", c_int32),
        ("spheres", c_int32),
        ("reserved", c_int32),
    ]


class PriestIO(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("z", "samples", "samples_out", "xi", "scores", "history")]


class MaDims(ctypes.Structure):
    _fields_ = [(n, c_int32) for n in ("n_problems", "n_agents", "n_pairs", "n_static", "n_p", "m", "n_eq",
                                       "n_levels")]


class MaConsts(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("P", "kinv", "level_rho", "pair_i", "pair_j", "pair_s", "pair_a", "pair_b",
                                        "inc_ptr", "inc_pair", "b_eq", "statics", "line_u", "line_v", "bnd")]


class MaState(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("state", "xi", "sums", "ring", "res_norm", "res_max", "hist", "level",
                                        "iteration", "last_change", "n_hist", "status", "export_d", "export_ab")]


class OzakiWs(ctypes.Structure):
    _fields_ = [("a_slices", c_void_p), ("a_exp", c_void_p), ("b_slices", c_void_p), ("b_exp", c_void_p),
                ("n_slices", c_int32), ("n_col_tiles", c_int32)]


class MaParams(ctypes.Structure):
    _fields_ = [("tol_norm", c_double), ("stall_improvement", c_double), ("stall_window", c_int32),
                ("max_iter", c_int32), ("max_hist", c_int32), ("reserved", c_int32)]


class B2Dims(ctypes.Structure):
    _fields_ = [("n_members", c_int64)] + [(n, c_int32) for n in ("n_obs", "n_c", "n_p", "m", "n_levels",
                                                                  "max_hist")]


class B2Consts(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("PT", "Pr", "obs", "obs_ab", "offsets", "q", "b", "b_psi", "kinvT_xi",
                                        "kinvT_psi", "rho_chain", "rho_psi_chain", "desired")] + [
        (n, c_double) for n in ("v_max", "a_max", "w_smooth", "w_track")] + [("k_xi", c_void_p)]


class B2State(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("xi", "xi_psi", "lam", "lam_psi", "sums", "res_max", "res_norm", "ring",
                                        "hist", "level", "iteration", "last_change", "n_hist", "n_changes",
                                        "counter", "alpha_coll", "d_coll", "alpha_v", "alpha_a", "d_v", "d_a",
                                        "psi", "rank", "psi_targets", "shard", "shards_in")]


class B2Params(ctypes.Structure):
    _fields_ = [("tol", c_double), ("stall_improvement", c_double), ("stall_window", c_int32), ("flags", c_int32),
                ("member_offset", c_int64), ("n_shards", c_int32), ("reserved", c_int32)]


class ValDims(ctypes.Structure):
    _fields_ = [("n_members", c_int64)] + [(n, c_int32) for n in ("n_obs", "n_p", "m", "dim", "per_member_desired",
                                                                  "reserved")]


class ValConsts(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("P", "Pdd", "t", "centers", "velocities", "shape_a", "shape_b",
                                        "desired")] + [("margin", c_double)]


class ValIO(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("xi", "pos", "acc", "out")]


class TrackDims(ctypes.Structure):
    _fields_ = [(n, c_int32) for n in ("n_scen", "n_obs", "n_p", "dim", "layout", "shared_obstacles")]


class MpcDims(ctypes.Structure):
    _fields_ = [(n, c_int32) for n in ("n_members", "n_obs", "n_p", "m", "dim", "n_exec", "trace_cap", "ring_len")]


class MpcConsts(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("P", "Pdot", "Pddot", "frac", "goal", "centers", "velocities", "shape_a",
                                        "shape_b", "plan_a", "plan_b", "tracks", "t_exec")] + [
        ("goal_radius", c_double), ("w_track", c_double)]


class MpcIO(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("bvals", "q", "desired", "d", "trace", "n_trace", "flags", "res_out")]


TRO_MPC_COLLIDED = 1
TRO_MPC_REACHED = 2

TRO_B2_PSI_IN = 16
TRO_B2_GIVEN_AD = 32
TRO_B2_GIVEN_ALPHA = 64
TRO_B2_CIRCLES = 128
TRO_B2_SHARD = 256

_lib = None


def load() -> ctypes.CDLL:
    """Load the library (fails loudly: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libtrajopt_b200.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    sig = [POINTER(Alg1Dims), POINTER(Alg1Consts), POINTER(Alg1State), POINTER(Alg1Params), c_void_p]
    for name in ("tro_alg1_prime", "tro_alg1_init", "tro_alg1_iterate"):
        f = getattr(lib, name)
        f.argtypes = [c_int32] + sig
        f.restype = c_int32
    lib.tro_alg1_iterate_n.argtypes = [c_int32] + sig[:4] + [c_int32, c_void_p]
    lib.tro_alg1_iterate_n.restype = c_int32
    lib.tro_alg1_linear_terms.argtypes = [c_int64, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_double, c_void_p, c_void_p]
    lib.tro_alg1_linear_terms.restype = c_int32
    lib.tro_kkt_apply_f64.argtypes = [c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_void_p]
    lib.tro_kkt_apply_f64.restype = c_int32
    lib.tro_topk_stable_f64.argtypes = [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_int64, c_void_p]
    lib.tro_topk_stable_f64.restype = c_int32
    lib.tro_topk_workspace_bytes.argtypes = [c_int64, c_int32]
    lib.tro_topk_workspace_bytes.restype = c_int64
    lib.tro_priest_project_f64.argtypes = [POINTER(PriestDims), POINTER(PriestConsts), POINTER(PriestIO), c_void_p]
    lib.tro_priest_project_f64.restype = c_int32
    lib.tro_priest_cost_f64.argtypes = [POINTER(PriestDims), POINTER(PriestConsts), c_void_p, c_void_p, c_int64,
                                        c_void_p, c_double, c_double, c_double, c_void_p, c_void_p]
    lib.tro_priest_cost_f64.restype = c_int32
    lib.tro_elite_update_f64.argtypes = [c_void_p, c_int32, c_void_p, c_int32, c_void_p, c_double, c_double,
                                         c_int32, c_void_p, c_void_p, c_void_p]
    lib.tro_normal_philox_f64.argtypes = [ctypes.c_uint64, ctypes.c_uint64, c_int64, c_int64, c_int32, c_void_p,
                                          c_void_p]
    lib.tro_normal_philox_f64.restype = c_int32
    lib.tro_cholesky_f64.argtypes = [c_void_p, c_int32, c_void_p, c_void_p]
    lib.tro_cholesky_f64.restype = c_int32
    lib.tro_elite_update_f64.restype = c_int32
    lib.tro_fastmath_eval.argtypes = [c_int32, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]
    lib.tro_fastmath_eval.restype = c_int32
    lib.tro_ma_run.argtypes = [c_int32, POINTER(MaDims), POINTER(MaConsts), POINTER(MaState), POINTER(MaParams),
                               c_void_p]
    lib.tro_ma_run.restype = c_int32
    lib.tro_ma_qp_ozaki.argtypes = [POINTER(MaDims), POINTER(MaConsts), POINTER(MaState), POINTER(OzakiWs), c_void_p]
    lib.tro_ma_qp_ozaki.restype = c_int32
    lib.tro_b2_run.argtypes = [c_int32, POINTER(B2Dims), POINTER(B2Consts), POINTER(B2State), POINTER(B2Params),
                               c_void_p]
    lib.tro_b2_run.restype = c_int32
    lib.tro_validate_f64.argtypes = [POINTER(ValDims), POINTER(ValConsts), POINTER(ValIO), c_void_p]
    lib.tro_validate_f64.restype = c_int32
    lib.tro_predict_tracks_f64.argtypes = [POINTER(TrackDims), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                           c_void_p]
    lib.tro_predict_tracks_f64.restype = c_int32
    lib.tro_mpc_advance_f64.argtypes = [c_int32, POINTER(MpcDims), POINTER(MpcConsts), POINTER(Alg1State),
                                        POINTER(MpcIO), c_void_p]
    lib.tro_mpc_advance_f64.restype = c_int32
    lib.tro_mpc_compact.argtypes = [c_int32, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.tro_mpc_compact.restype = c_int32
    lib.tro_fp64_fma_probe.argtypes = [c_int64, c_int32, c_void_p, c_void_p]
    lib.tro_fp64_fma_probe.restype = c_int32
    lib.tro_version.argtypes = []
    lib.tro_version.restype = c_int32
    lib.tro_error_string.argtypes = [c_int32]
    lib.tro_error_string.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().tro_error_string(int(rc)).decode()
        raise RuntimeError(f"{what} failed: {msg} (code {rc})")


def require_cuda():
    """The compute path needs a CUDA device and the library; raise otherwise."""
    import torch

    load()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2408_10731_b200 needs a CUDA (sm_100a) device; no CPU fallback exists")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
