"""B200-native differentiable MLS-MPM substep (FluidLab / FluidEngine, arXiv 2303.02346).

The hot path -- P2G, grid update with SDF effector contact, G2P with
per-material return mapping, rigid shape matching and their adjoints -- runs
as hand-written sm_100a CUDA in libflume_b200.so behind the C ABI of
include/flume_b200.h.  This package is the host-side mirror of the reference's
scene / step / grad API (proj/include/flume)."""
from .api import (ActionTrajectory, AdjointError, AdjointState, DegenerateDeformation, DeviceError, EngineError,
                  GpuWorkspace, LossEvaluator, RigidityError, Scene, SceneError, SimState, SubstepRecord,
                  TrajectoryGrad, World, adjoint_substep, build_scene, dist_unique_id, grad_trajectory, ipc_unique_id, mpm_substep,
                  p2g_grid, rollout_loss, slab_split, WorkspacePool, rollout_loss_batch, ReplicaWorkspace,
                  rollout_loss_replicas, grad_trajectory_replicas,
                  grad_trajectory_batch, state_to_json, state_from_json, GradReport, grad_check,
                  finite_difference_gradient, optimizable_components)
from . import frames, scenes

__all__ = ["ActionTrajectory", "AdjointError", "AdjointState", "DegenerateDeformation", "DeviceError", "EngineError",
           "GpuWorkspace", "LossEvaluator", "RigidityError", "Scene", "SceneError", "SimState", "SubstepRecord",
           "TrajectoryGrad", "World", "adjoint_substep", "build_scene", "dist_unique_id", "grad_trajectory", "ipc_unique_id", "mpm_substep", "p2g_grid",
           "rollout_loss", "scenes", "slab_split", "WorkspacePool", "rollout_loss_batch", "grad_trajectory_batch",
           "ReplicaWorkspace", "rollout_loss_replicas", "grad_trajectory_replicas",
           "state_to_json", "state_from_json", "frames", "GradReport", "grad_check",
           "finite_difference_gradient", "optimizable_components"]
