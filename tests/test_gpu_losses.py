"""Device point-set losses against the reference LossEvaluator
(losses.hpp:15-100, 474-551, compiled unmodified in oracle/_ref):
trajectory_chamfer (symmetric mean NN distance to per-segment goal sets) and
mixing_spread (-sum_ij |x_i - x_j|), alone and in a composite with target_point.

Tolerances: segment losses <= 1e-6 relative (fp32 state, fp64 loss arithmetic),
action gradients by GradReport::rel_error <= 1e-3.
"""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import grad_rel_error, pair, spec_for

pytestmark = pytest.mark.gpu


def _goal_sets(rng, n_steps, m):
    return [(np.array([0.5, 0.25, 0.5]) + 0.15 * rng.standard_normal((m, 3))).clip(0.1, 0.9).tolist()
            for _ in range(n_steps)]


def _run(spec, nseg, seglen, chamfer="auto"):
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    ws.set_chamfer_mode(chamfer)
    vals = np.tile(w.init_action, (nseg, 1))
    acts = fl.ActionTrajectory(nseg, seglen, vals)
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    per = []
    l = fl.rollout_loss(w.scene, w.state, acts, loss, per_segment=per, ws=ws)
    rl, rper = r.rollout_loss(vals, seglen)
    tg = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    rg = r.grad_trajectory(vals, seglen)
    return l, per, rl, rper, tg, rg


@pytest.mark.parametrize("mode", ["auto", "grid"])
@pytest.mark.parametrize("m", [1, 37, 700])
def test_trajectory_chamfer_parity(ref_available, m, mode):
    """mode "grid" forces the uniform-grid nearest-neighbour index (used above 2^24 pairs)."""
    rng = np.random.default_rng(m)
    spec = spec_for("c1", 16)
    spec["loss"] = {"kind": "trajectory_chamfer", "body": "column", "goal_trajectory": _goal_sets(rng, 2, m)}
    l, per, rl, rper, tg, rg = _run(spec, 3, 4, chamfer=mode)  # 3 segments, 2 goal sets: the last is reused
    np.testing.assert_allclose(per, rper, rtol=1e-6)
    assert abs(l - rl) <= 1e-6 * abs(rl)
    assert abs(tg.loss - rg["loss"]) <= 1e-6 * abs(rg["loss"])
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3, (tg.action_grad, rg["grad"])


def test_mixing_spread_parity(ref_available):
    spec = spec_for("c1", 16)
    spec["loss"] = {"kind": "mixing_spread", "body": "column", "weight": 1e-6}
    l, per, rl, rper, tg, rg = _run(spec, 2, 4)
    np.testing.assert_allclose(per, rper, rtol=1e-6)
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3, (tg.action_grad, rg["grad"])


def test_composite_point_and_target(ref_available):
    rng = np.random.default_rng(3)
    spec = spec_for("c1", 16)
    spec["loss"] = {"kind": "composite", "terms": [
        {"kind": "target_point", "body": "column", "goal": [0.7, 0.1, 0.5], "weight": 0.5},
        {"kind": "trajectory_chamfer", "body": "column", "goal_trajectory": _goal_sets(rng, 1, 64),
         "weight": 2.0, "eval": "final"}]}
    l, per, rl, rper, tg, rg = _run(spec, 2, 5)
    np.testing.assert_allclose(per, rper, rtol=1e-6)
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3


def _chamfer_run(spec, mode, nseg=2, seglen=3):
    w = fl.build_scene(spec)
    ws = fl.GpuWorkspace(w.scene)
    ws.set_chamfer_mode(mode)
    acts = fl.ActionTrajectory(nseg, seglen, np.tile(w.init_action, (nseg, 1)))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    per = []
    l = fl.rollout_loss(w.scene, w.state, acts, loss, per_segment=per, ws=ws)
    g = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    ws.close()
    return l, np.asarray(per), g.loss, np.asarray(g.action_grad).copy()


@pytest.mark.parametrize("body,m", [("column", 3000), ("column", 20)])
def test_chamfer_grid_index_equals_scan(body, m):
    """Both nearest-neighbour paths return the first-index minimum with the same rounding,
    so the loss, per-segment losses and action gradient are bit-identical (full c1:
    102,400 column particles against m goals, goals clustered and spread)."""
    rng = np.random.default_rng(11)
    spec = spec_for("c1")
    spec["loss"] = {"kind": "trajectory_chamfer", "body": body, "goal_trajectory": _goal_sets(rng, 2, m)}
    a = _chamfer_run(spec, "scan")
    b = _chamfer_run(spec, "grid")
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
    assert a[2] == b[2] and np.array_equal(a[3], b[3])


def test_chamfer_grid_full_scale():
    """trajectory_chamfer on c4's 1M-particle pool against a 300k-point goal set (3e11 pairs:
    grid index only), checked against exact nearest neighbours from a k-d tree on the host
    (scipy cKDTree over the device's own state after the substep)."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(12)
    spec = spec_for("c4")
    goals = (np.array([0.5, 0.08, 0.5]) + np.array([0.3, 0.05, 0.3]) * rng.uniform(-1, 1, (300_000, 3)))
    spec["loss"] = {"kind": "trajectory_chamfer", "body": "pool", "goal_trajectory": [goals.tolist()]}
    w = fl.build_scene(spec)
    ws = fl.GpuWorkspace(w.scene)
    acts = fl.ActionTrajectory(1, 1, w.init_action.reshape(1, 6))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    l = fl.rollout_loss(w.scene, w.state, acts, loss, ws=ws)
    st = w.state.copy()
    fl.mpm_substep(w.scene, st, w.init_action, ws, count=1)
    ws.close()
    body_id = int(w.loss_spec[0]["body"])
    pts = st.x[w.scene.body_id == body_id]
    g = np.asarray(goals, dtype=np.float64)
    da, _ = cKDTree(g).query(pts)
    dg, _ = cKDTree(pts).query(g)
    want = float(np.mean(da) + np.mean(dg))
    assert abs(l - want) <= 1e-10 * want, (l, want)


def test_chamfer_rerun_bit_identical():
    rng = np.random.default_rng(5)
    spec = spec_for("c1", 16)
    spec["loss"] = {"kind": "trajectory_chamfer", "body": "column", "goal_trajectory": _goal_sets(rng, 1, 200)}
    out = []
    for _ in range(2):
        w = fl.build_scene(spec)
        ws = fl.GpuWorkspace(w.scene)
        acts = fl.ActionTrajectory(2, 3, np.tile(w.init_action, (2, 1)))
        g = fl.grad_trajectory(w.scene, w.state, acts, fl.LossEvaluator(w.scene, w.loss_spec, w.state), ws=ws)
        out.append((g.loss, np.asarray(g.action_grad).copy()))
    assert out[0][0] == out[1][0] and np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("kind", ["target_point", "hold_initial", "trajectory_chamfer"])
def test_loss_on_emitter_body_at_activation_boundaries(ref_available, kind):
    """c2's stream body emits one particle per substep; segment boundaries fall on
    activation substeps, where the reference counts the not-yet-emitted particle as
    active at its parked position (types.hpp:109, losses.hpp gather)."""
    spec = spec_for("c2", 64)
    term = {"kind": kind, "body": "stream"}
    if kind == "target_point":
        term["goal"] = [0.5, 0.3, 0.5]
    if kind == "trajectory_chamfer":
        term["goal_trajectory"] = _goal_sets(np.random.default_rng(9), 2, 40)
    spec["loss"] = term
    l, per, rl, rper, tg, rg = _run(spec, 3, 5)
    np.testing.assert_allclose(per, rper, rtol=1e-6)
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3, (tg.action_grad, rg["grad"])


@pytest.mark.parametrize("name,res,body,tau", [("c1", 16, "column", 0.0), ("c1", 16, "column", 0.05),
                                               ("c2", 64, "stream", 0.0)])
def test_attraction_parity(ref_available, name, res, body, tau):
    """The optimizer's gradient-sharing surrogate (losses.hpp:104-218): enable_attraction,
    refresh_attraction from a rollout's final state (optimize.hpp:157-190), then loss and
    action gradient with the term active at every segment boundary.  c2's stream body has
    parked emitter particles, which the term includes at their parked positions."""
    spec = spec_for(name, res)
    spec["loss"] = {"kind": "target_point", "body": body, "goal": [0.5, 0.3, 0.5]}
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    nseg, seglen = 3, 4
    vals = np.tile(w.init_action, (nseg, 1))
    acts = fl.ActionTrajectory(nseg, seglen, vals)
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    radius = 3 * w.scene.dx
    loss.enable_attraction(-1, 1e-3, radius, tau)
    fs = w.state.copy()
    fl.rollout_loss(w.scene, w.state, acts, loss, final_state=fs, ws=ws)
    assert fs.substep_index == nseg * seglen
    # per_particle on the device == the reference's on the same positions
    pp = loss.per_particle(fs, ws)
    rpp = r.per_particle(fs.x)
    np.testing.assert_allclose(pp, rpp, rtol=1e-12, atol=1e-12)
    loss.refresh_attraction(fs, ws)
    r.set_attraction(-1, 1e-3, radius, tau, refresh_x=fs.x)
    body_id = int(w.loss_spec[0]["body"])
    assert loss.desc.n_prev == int(np.sum(w.scene.body_id == body_id)) >= 2
    per = []
    l = fl.rollout_loss(w.scene, w.state, acts, loss, per_segment=per, ws=ws)
    rl, rper = r.rollout_loss(vals, seglen)
    np.testing.assert_allclose(per, rper, rtol=1e-6)
    tg = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    rg = r.grad_trajectory(vals, seglen)
    assert abs(tg.loss - rg["loss"]) <= 1e-6 * abs(rg["loss"])
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-3, (tg.action_grad, rg["grad"])
    # the term is not negligible: switching it off changes the loss
    r.set_attraction(-1, 0.0, radius, tau)
    r0, _ = r.rollout_loss(vals, seglen)
    assert abs(rl - r0) > 1e-4 * abs(rl)


def test_attraction_size_mismatch_raises():
    spec = spec_for("c1", 16)
    w = fl.build_scene(spec)
    ws = fl.GpuWorkspace(w.scene)
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    loss.enable_attraction(-1, 1.0, 3 * w.scene.dx, 0.0)
    loss.set_attraction_prev(np.ones(5))
    acts = fl.ActionTrajectory(1, 2, w.init_action.reshape(1, 6))
    with pytest.raises(fl.EngineError, match="loss list size mismatch"):
        fl.rollout_loss(w.scene, w.state, acts, loss, ws=ws)
