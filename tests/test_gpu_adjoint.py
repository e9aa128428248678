"""Reverse-mode parity of the sm_100a adjoint against the reference engine.

Tolerances: action gradients by GradReport::rel_error (grad.hpp:162-169)
<= 1e-3 over short horizons; single-substep bars <= 1e-3
relative to each field's max; checkpoint stride leaves gradients bit-identical
(test_autodiff.cpp:153-178 asks <= 1e-12; deterministic kernels give 0).
"""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import grad_rel_error, pair, rel_err, spec_for

pytestmark = pytest.mark.gpu


def _grad_both(spec, nseg, seglen, stride=0):
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    vals = np.tile(w.init_action, (nseg, 1))
    acts = fl.ActionTrajectory(nseg, seglen, vals)
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    tg = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=stride, ws=ws)
    rg = r.grad_trajectory(vals, seglen, stride=max(stride, 1) if stride else 0)
    return tg, rg


@pytest.mark.parametrize("name,res,nseg,seglen", [("c1", None, 1, 10), ("c2", 32, 2, 4), ("c3", 32, 1, 8),
                                                  ("c5", 64, 2, 3)])
def test_grad_trajectory_parity(ref_available, name, res, nseg, seglen):
    tg, rg = _grad_both(spec_for(name, res), nseg, seglen)
    assert abs(tg.loss - rg["loss"]) <= 1e-5 * abs(rg["loss"])
    err = grad_rel_error(tg.action_grad, rg["grad"])
    assert err <= 1e-3, (tg.action_grad, rg["grad"], err)


def test_grad_c4_pool_loss(ref_available):
    spec = spec_for("c4", 32)
    spec["loss"] = {"kind": "target_point", "body": "pool", "goal": [0.3, 0.35, 0.5]}
    tg, rg = _grad_both(spec, 2, 4)
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3


def test_stride_invariance_and_snapshots(ref_available):
    spec = spec_for("c5", 64)
    w = fl.build_scene(spec)
    ws = fl.GpuWorkspace(w.scene)
    acts = fl.ActionTrajectory(3, 4, np.array([[0.3, 0.1, 0, 0, 0, 0], [-0.1, 0.2, 0.1, 0, 0, 0],
                                               [0.2, -0.2, 0, 0, 0, 0]]))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    g1 = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=1, ws=ws)
    g5 = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=5, ws=ws)
    g0 = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=0, ws=ws)
    assert np.array_equal(g1.action_grad, g5.action_grad)
    assert np.array_equal(g1.action_grad, g0.action_grad)
    assert g1.snapshots == 13 and g5.snapshots == 12 // 5 + 1 and g0.snapshots == 2


def test_adjoint_substep_parity(ref_available):
    spec = spec_for("c5", 64)
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    # advance a few substeps so F, C are non-trivial, on both engines
    fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=3)
    r.substep(w.init_action, 3)
    rs = r.state()
    w.state.x = rs["x"]
    w.state.v = rs["v"]
    w.state.F = rs["F"]
    w.state.C = rs["C"]
    rng = np.random.default_rng(0)
    n = w.scene.n_particles
    bars = [rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), rng.normal(size=(n, 3, 3)),
            rng.normal(size=(n, 3, 3))]
    adj = fl.AdjointState(*[b.copy() for b in bars], np.zeros((w.scene.n_effectors, 12)))
    abar = np.zeros(6)
    fl.adjoint_substep(w.scene, fl.SubstepRecord(3, w.init_action, w.state), adj, abar, ws)
    rx, rv, rF, rC, reb, rab = r.adjoint_substep(w.init_action, *bars)
    assert rel_err(adj.x_bar, rx) <= 1e-3
    assert rel_err(adj.v_bar, rv) <= 1e-3
    assert rel_err(adj.F_bar, rF) <= 1e-3
    assert rel_err(adj.C_bar, rC) <= 1e-3
    assert rel_err(abar, rab) <= 1e-3


def test_zero_cotangent_gives_zero(ref_available):
    """test_autodiff.cpp:31-45"""
    w = fl.build_scene(spec_for("c5", 64))
    ws = fl.GpuWorkspace(w.scene)
    adj = fl.AdjointState.init(w.state)
    abar = np.zeros(6)
    fl.adjoint_substep(w.scene, fl.SubstepRecord(0, [0.2, 0.1, 0, 0, 0, 0], w.state), adj, abar, ws)
    assert np.all(abar == 0)
    assert np.all(adj.x_bar == 0) and np.all(adj.v_bar == 0)


def test_grad_rerun_bit_identical(ref_available):
    spec = spec_for("c3", 32)
    w = fl.build_scene(spec)
    ws = fl.GpuWorkspace(w.scene)
    acts = fl.ActionTrajectory(1, 6, np.tile(w.init_action, (1, 1)))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    a = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    b = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    assert np.array_equal(a.action_grad, b.action_grad) and a.loss == b.loss


def test_long_rollouts_rerun_identical():
    """Many substeps in one context (work-counter pool wraps several times) give the
    same gradients as a fresh context, call after call."""
    spec = spec_for("c4", 32)
    out = []
    for fresh in (True, False, False):
        if fresh or not out:
            w = fl.build_scene(spec)
            ws = fl.GpuWorkspace(w.scene)
        acts = fl.ActionTrajectory(2, 45, np.tile(w.init_action, (2, 1)))
        loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
        g = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=30, ws=ws)
        out.append((g.loss, np.asarray(g.action_grad).copy()))
    for l, gr in out[1:]:
        assert l == out[0][0] and np.array_equal(gr, out[0][1])


def test_checkpoint_spill_to_host_identical():
    """Snapshots spilled to pinned host memory give bit-identical
    gradients and the same snapshot count as HBM snapshots."""
    spec = spec_for("c4", 32)
    out = []
    for spill in (False, True, True):
        w = fl.build_scene(spec)
        ws = fl.GpuWorkspace(w.scene)
        ws.set_checkpoint_spill(spill)
        acts = fl.ActionTrajectory(3, 7, np.tile(w.init_action, (3, 1)))
        loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
        g = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=4, ws=ws)
        out.append((g.loss, np.asarray(g.action_grad).copy(), g.snapshots))
    for l, gr, ns in out[1:]:
        assert l == out[0][0] and np.array_equal(gr, out[0][1]) and ns == out[0][2] == 21 // 4 + 1


def test_checkpoint_spill_to_file_identical(tmp_path):
    """The file tier (local NVMe) of the checkpoint store: snapshots written by a worker thread
    from pinned staging buffers, read back (the next older one prefetched) when the backward
    replays -- bit-identical gradients, same snapshot count, on repeated calls; and at the
    benchmark scene's size (c4, 1M particles, stride 5 over 2 x 10 substeps)."""
    for spec, nseg, seglen, stride in ((spec_for("c4", 32), 3, 7, 4), (spec_for("c4"), 2, 10, 5)):
        out = []
        for mode in ("hbm", "file", "file"):
            w = fl.build_scene(spec)
            ws = fl.GpuWorkspace(w.scene)
            if mode == "file":
                ws.set_checkpoint_spill_dir(tmp_path)
            acts = fl.ActionTrajectory(nseg, seglen, np.tile(w.init_action, (nseg, 1)))
            loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
            for _ in range(2 if mode == "file" else 1):  # a second call reuses the file tier
                g = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=stride, ws=ws)
            out.append((g.loss, np.asarray(g.action_grad).copy(), g.snapshots))
            ws.close()
        assert np.abs(out[0][1]).max() > 0
        for l, gr, ns in out[1:]:
            assert l == out[0][0] and np.array_equal(gr, out[0][1]) and ns == out[0][2]
    assert not list(tmp_path.iterdir())  # the spill file is anonymous


def test_grad_through_cfl_clamp(ref_available):
    """A blob faster than cfl * dx / dt: every G2P clamps |v| (mpm.hpp:322-328) and the
    adjoint zeroes v_raw_bar there (adjoint.hpp:281-365)."""
    from tests.test_gpu_kat import _free_blob
    spec = _free_blob(v=(400.0, 50.0, 0.0))
    spec["loss"] = {"kind": "target_point", "body": "blob", "goal": [0.8, 0.5, 0.5]}
    spec["effectors"] = spec_for("c1", 32)["effectors"]
    spec["action_bounds"] = spec_for("c1", 32)["action_bounds"]
    spec["optimizer"] = {"n_segments": 1, "segment_length": 6, "init": [0.5, 0.0, 0.0, 0, 0, 0]}
    tg, rg = _grad_both(spec, 1, 6)
    assert abs(tg.loss - rg["loss"]) <= 1e-5 * abs(rg["loss"])
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3, (tg.action_grad, rg["grad"])


@pytest.mark.parametrize("name,res", [("c1", None), ("c4", 32)])
def test_grad_hard_contact(ref_available, name, res):
    """hard_contact: the step contact weight instead of exp(-d) (mpm.hpp:120-128)."""
    spec = spec_for(name, res)
    spec["hard_contact"] = True
    tg, rg = _grad_both(spec, 1, 8)
    assert abs(tg.loss - rg["loss"]) <= 1e-5 * abs(rg["loss"])
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3, (tg.action_grad, rg["grad"])


@pytest.mark.parametrize("friction", ["sticky", 0.0])
def test_grad_effector_friction_modes(ref_available, friction):
    """Sticky (v_rel' = 0) and frictionless effectors (mpm.hpp:79-117, 146-161)."""
    spec = spec_for("c1", 32)
    spec["effectors"][0]["friction"] = friction
    tg, rg = _grad_both(spec, 1, 8)
    assert np.max(np.abs(rg["grad"])) > 0
    assert abs(tg.loss - rg["loss"]) <= 1e-5 * abs(rg["loss"])
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3, (tg.action_grad, rg["grad"])


SHAPES = {
    "sphere": {"type": "sphere", "radius": 0.09},
    "capsule": {"type": "capsule", "radius": 0.05, "a": [0.0, -0.12, 0.0], "b": [0.0, 0.12, 0.05]},
    "cylinder": {"type": "cylinder", "radius": 0.07, "half_height": 0.12, "axis_angle": [0.4, 0.0, 0.3]},
    "halfspace": {"type": "halfspace", "normal": [-1.0, 0.2, 0.0], "offset": -0.02},
}


@pytest.mark.parametrize("shape", list(SHAPES))
def test_grad_effector_shapes(ref_available, shape):
    """Every SDF shape (sdf.hpp:131-339): contact forward, normal and pose VJPs."""
    spec = spec_for("c1", 32)
    spec["effectors"][0]["shape"] = dict(SHAPES[shape], center=[0.0, 0.0, 0.0])
    spec["effectors"][0]["angular_velocity"] = [0.0, 0.0, 0.3]
    tg, rg = _grad_both(spec, 1, 10)
    assert np.max(np.abs(rg["grad"])) > 0  # the effector is in contact
    assert abs(tg.loss - rg["loss"]) <= 1e-5 * abs(rg["loss"])
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3, (tg.action_grad, rg["grad"])


def _rotating_box_spec():
    """test_autodiff.cpp:113-148: 3D elastic blob pushed by a rotating box effector."""
    return {
        "dim": 3, "grid_resolution": 16, "domain": [1.0, 1.0, 1.0], "dt_substep": 4e-4, "substeps_per_step": 5,
        "gravity": [0.0, -2.0, 0.0], "seed": 21,
        "materials": [{"name": "stuff", "kind": "elastic", "mu": 208.33, "lambda": 277.78, "rho": 1.0}],
        "bodies": [{"name": "blob", "material": "stuff",
                    "shape": {"type": "box", "half_extents": [0.1, 0.08, 0.1], "center": [0.45, 0.3, 0.5]},
                    "particles_per_cell_axis": 1, "jitter": 0.2}],
        "loss": {"kind": "target_point", "body": "blob", "goal": [0.6, 0.4, 0.55]},
        "effectors": [{"shape": {"type": "box", "half_extents": [0.07, 0.05, 0.07], "center": [0.0, 0.0, 0.0]},
                       "position": [0.33, 0.42, 0.5], "friction": 0.4,
                       "action_mask": [True, True, True, False, False, True]}],
    }


def test_grad_check_rotating_box(ref_available):
    """grad_check (grad.hpp:190-225) on the reference's 3D rotating-box case: the device
    adjoint gradient over the optimizable components matches the reference's adjoint and its
    fp64 finite differences (the test's own bar, 1e-3); the device's fp32 central differences
    audit its adjoint at a looser bar set by fp32 loss rounding."""
    spec = _rotating_box_spec()
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    vals = np.array([[0.4, -0.3, 0.2, 0, 0, 0.8], [-0.2, 0.3, -0.1, 0, 0, -0.5]])
    acts = fl.ActionTrajectory(2, 15, vals)
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    assert fl.optimizable_components(w.scene) == [0, 1, 2, 5]
    rep = fl.grad_check(w.scene, w.state, acts, loss, 10, 1e-3, ws=ws)
    ref = r.grad_check(vals, 15, 10, 1e-5)
    assert ref["max_rel_error"] <= 1e-3
    assert len(rep.gradient) == len(ref["gradient"]) == 8
    assert abs(rep.loss - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    assert fl.GradReport.rel_error(rep.gradient, ref["fd_gradient"]) <= 1e-3, (rep.gradient, ref["fd_gradient"])
    assert rep.max_rel_error <= 2e-2, (rep.gradient, rep.fd_gradient)
    no_fd = fl.grad_check(w.scene, w.state, acts, loss, 10, 1e-3, with_fd=False, ws=ws)
    assert no_fd.gradient == rep.gradient and no_fd.fd_gradient == []
