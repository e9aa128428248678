"""ctypes mirror of include/flume_b200.h and the library loader.

The CUDA library is required: importing the product path on a machine where
libflume_b200.so is missing raises immediately (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("FLUME_B200_LIB", _PKG / "libflume_b200.so"))

ABI_VERSION = 3  # include/flume_b200.h FLUME_B200_ABI_VERSION

FLUME_OK = 0
FLUME_E_ENGINE = 1
FLUME_E_SCENE = 2
FLUME_E_DEGENERATE = 3
FLUME_E_RIGIDITY = 4
FLUME_E_ADJOINT = 5
FLUME_E_SOLVER = 6
FLUME_E_CUDA = 7
FLUME_E_ARG = 8
FLUME_E_OTHER = 9

d3 = C.c_double * 3
d6 = C.c_double * 6
d9 = C.c_double * 9
i6 = C.c_int * 6


class Config(C.Structure):
    _fields_ = [("grid_resolution", C.c_int), ("domain", d3), ("dt_substep", C.c_double),
                ("substeps_per_step", C.c_int), ("gravity", d3), ("boundary_width", C.c_int),
                ("contact_eps_cells", C.c_double), ("cfl_fraction", C.c_double), ("mass_epsilon", C.c_double),
                ("hard_contact", C.c_int)]


class Material(C.Structure):
    _fields_ = [("kind", C.c_int), ("mu", C.c_double), ("lambda_", C.c_double), ("rho", C.c_double),
                ("theta_c", C.c_double), ("theta_s", C.c_double), ("sigma_y", C.c_double)]


class EffectorShape(C.Structure):
    _fields_ = [("shape_kind", C.c_int), ("radius", C.c_double), ("half_extents", d3), ("seg_a", d3),
                ("seg_b", d3), ("plane_normal", d3), ("plane_offset", C.c_double), ("half_height", C.c_double),
                ("shape_t", d3), ("shape_R", d9), ("friction_mu", C.c_double), ("action_mask", i6)]


class EffectorState(C.Structure):
    _fields_ = [("pose_t", d3), ("pose_R", d9), ("linear_velocity", d3), ("angular_velocity", d3)]


class RigidBody(C.Structure):
    _fields_ = [("body_id", C.c_int), ("n_members", C.c_long), ("members", C.POINTER(C.c_long)),
                ("rest_offsets", C.POINTER(C.c_double)), ("total_mass", C.c_double)]


class Emitter(C.Structure):
    _fields_ = [("particle", C.c_long), ("effector", C.c_int), ("local_pos", d3), ("local_vel", d3)]


class SceneDesc(C.Structure):
    _fields_ = [("config", Config), ("n_materials", C.c_int), ("materials", C.POINTER(Material)),
                ("n_effectors", C.c_int), ("effectors", C.POINTER(EffectorShape)), ("n_rigid", C.c_int),
                ("rigid", C.POINTER(RigidBody)), ("n_emitters", C.c_long), ("emitters", C.POINTER(Emitter)),
                ("n_particles", C.c_long), ("material_id", C.POINTER(C.c_int)), ("body_id", C.POINTER(C.c_int)),
                ("mass", C.POINTER(C.c_double)), ("volume0", C.POINTER(C.c_double)),
                ("activation_substep", C.POINTER(C.c_long))]


class StateView(C.Structure):
    _fields_ = [("time", C.c_double), ("substep_index", C.c_long), ("x", C.POINTER(C.c_double)),
                ("v", C.POINTER(C.c_double)), ("F", C.POINTER(C.c_double)), ("C", C.POINTER(C.c_double)),
                ("effectors", C.POINTER(EffectorState))]


class LossTerm(C.Structure):
    _fields_ = [("kind", C.c_int), ("body", C.c_int), ("weight", C.c_double), ("squared", C.c_int),
                ("final_only", C.c_int), ("goal", d3), ("n_goal_steps", C.c_int),
                ("goal_step_offsets", C.POINTER(C.c_long)), ("goal_points", C.POINTER(C.c_double))]


class LossDesc(C.Structure):
    _fields_ = [("n_terms", C.c_int), ("terms", C.POINTER(LossTerm)), ("attraction_body", C.c_int),
                ("attraction_weight", C.c_double), ("attraction_radius", C.c_double),
                ("attraction_tau", C.c_double), ("n_prev", C.c_long), ("prev_losses", C.POINTER(C.c_double))]


class Actions(C.Structure):
    _fields_ = [("n_segments", C.c_int), ("segment_length", C.c_int), ("values", C.POINTER(C.c_double))]


class ErrorInfo(C.Structure):
    _fields_ = [("code", C.c_int), ("particle_id", C.c_long), ("body_id", C.c_int), ("substep", C.c_long),
                ("message", C.c_char * 256)]


class Timing(C.Structure):
    _fields_ = [("forward_ms", C.c_double), ("backward_ms", C.c_double), ("substeps", C.c_long),
                ("particle_substeps", C.c_long), ("launches", C.c_long)]


# every symbol the header declares (checked by the CPU test suite)
EXPORTS = {
    "flume_abi_version": (C.c_int, []),
    "flume_scene_build_json": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "flume_scene_free": (C.c_int, [C.c_void_p]),
    "flume_scene_desc_get": (C.c_int, [C.c_void_p, C.POINTER(SceneDesc)]),
    "flume_scene_state_get": (C.c_int, [C.c_void_p, C.POINTER(StateView)]),
    "flume_scene_loss_get": (C.c_int, [C.c_void_p, C.POINTER(LossDesc)]),
    "flume_scene_optimizer_get": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                            C.POINTER(C.c_double)]),
    "flume_ctx_create": (C.c_int, [C.POINTER(SceneDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "flume_ctx_destroy": (C.c_int, [C.c_void_p]),
    "flume_group_create": (C.c_int, [C.POINTER(SceneDesc), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]),
    "flume_dist_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
    "flume_ctx_create_dist": (C.c_int, [C.POINTER(SceneDesc), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_ubyte),
                                        C.POINTER(C.c_void_p)]),
    "flume_slab_split": (C.c_int, [C.POINTER(C.c_double), C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "flume_slab_set_migration_capacity": (C.c_int, [C.c_void_p, C.c_int]),
    "flume_slab_migration_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_long)]),
    "flume_ipc_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
    "flume_slab_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), C.POINTER(C.c_long)]),
    "flume_set_mode": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "flume_last_error": (C.c_int, [C.c_void_p, C.POINTER(ErrorInfo)]),
    "flume_set_checkpoint_spill": (C.c_int, [C.c_void_p, C.c_int]),
    "flume_set_chamfer_mode": (C.c_int, [C.c_void_p, C.c_int]),
    "flume_set_incremental_sort": (C.c_int, [C.c_void_p, C.c_int]),
    "flume_ctx_create_replicas": (C.c_int, [C.POINTER(SceneDesc), C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "flume_replicas_rollout_loss": (C.c_int, [C.c_void_p, C.POINTER(Actions), C.POINTER(LossDesc), C.c_long,
                                              C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "flume_replicas_grad_trajectory": (C.c_int, [C.c_void_p, C.POINTER(Actions), C.POINTER(LossDesc), C.c_long,
                                                 C.c_long, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                 C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                 C.POINTER(C.c_long)]),
    "flume_replicas_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_long), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int)]),
    "flume_sort_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_long), C.POINTER(C.c_long)]),
    "flume_set_checkpoint_spill_dir": (C.c_int, [C.c_void_p, C.c_char_p]),
    "flume_get_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "flume_sync": (C.c_int, [C.c_void_p]),
    "flume_last_timing": (C.c_int, [C.c_void_p, C.POINTER(Timing)]),
    "flume_state_upload": (C.c_int, [C.c_void_p, C.POINTER(StateView)]),
    "flume_state_download": (C.c_int, [C.c_void_p, C.POINTER(StateView)]),
    "flume_store_order": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint), C.POINTER(C.c_uint), C.POINTER(C.c_long)]),
    "flume_store_sorted": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint), C.POINTER(C.c_uint), C.POINTER(C.c_float),
                                     C.POINTER(C.c_long)]),
    "flume_store_positions": (C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    "flume_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "flume_kernel_times": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_long), C.c_int]),
    "flume_timer_mark": (C.c_int, [C.c_void_p, C.c_int]),
    "flume_timer_elapsed": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "flume_substep": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_int]),
    "flume_stage_grid": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "flume_rollout_loss_final": (C.c_int, [C.c_void_p, C.POINTER(Actions), C.POINTER(LossDesc), C.c_long,
                                           C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "flume_loss_per_particle": (C.c_int, [C.c_void_p, C.POINTER(LossDesc), C.POINTER(C.c_double)]),
    "flume_rollout_loss": (C.c_int, [C.c_void_p, C.POINTER(Actions), C.POINTER(LossDesc), C.c_long,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "flume_grad_trajectory": (C.c_int, [C.c_void_p, C.POINTER(Actions), C.POINTER(LossDesc), C.c_long, C.c_long,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), C.POINTER(C.c_long)]),
    "flume_adjoint_substep": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}
EXTRA = {"flume_scene_error": (C.c_char_p, [C.c_void_p])}

_lib = None


def load() -> C.CDLL:
    """Load the CUDA library, failing loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(there is no CPU fallback for the MPM substep)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in {**EXPORTS, **EXTRA}.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.flume_abi_version() != ABI_VERSION:
        raise RuntimeError("libflume_b200.so ABI mismatch")
    _lib = lib
    return lib
