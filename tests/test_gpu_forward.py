"""Forward-substep parity of the sm_100a path against the reference engine
(oracle/_ref = proj/include/flume compiled unmodified).

Tolerances (confirmed here for fp32 state): one substep from
identical inputs <= 1e-5 relative for x/dx, v/max|v|, F, C/max|C|; 20 substeps
<= 1e-4, except 5e-4 for v in scenes with SVD solids: with F stored in fp32 the
strain of a stiff solid (|F - R| ~ 1e-4) carries ~6e-8 absolute rounding, which
the corotated stress amplifies (measured: plastic 1.7e-4, elastic / von Mises
6e-5, liquids 6e-5, fp64 rigid members 2e-8 after 20 substeps of c5@64);
grid mass <= 1e-6 relative; cell keys and the canonical store order bit-exact
against a CPU recomputation on the GPU's own fp32 positions.
"""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import canonical_keys_cpu, grad_rel_error, pair, spec_for, state_errors

pytestmark = pytest.mark.gpu

SCENES = [("c1", None), ("c2", 32), ("c3", 32), ("c4", 32), ("c5", 64)]


@pytest.mark.parametrize("name,res", SCENES)
def test_one_substep_parity(ref_available, name, res):
    spec = spec_for(name, res)
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    act = w.init_action
    fl.mpm_substep(w.scene, w.state, act, ws)
    r.substep(act)
    e = state_errors(w.state, r.state(), w.scene.dx)
    assert e["x"] <= 1e-5 and e["v"] <= 1e-5 and e["F"] <= 1e-5 and e["C"] <= 1e-4, e


@pytest.mark.parametrize("name,res", SCENES)
def test_twenty_substeps_parity(ref_available, name, res):
    spec = spec_for(name, res)
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    act = w.init_action
    fl.mpm_substep(w.scene, w.state, act, ws, count=20)
    r.substep(act, 20)
    rs = r.state()
    e = state_errors(w.state, rs, w.scene.dx)
    assert w.state.substep_index == rs["substep"] == 20
    vtol = 5e-4 if name in ("c3", "c5") else 1e-4
    assert e["x"] <= 1e-4 and e["v"] <= vtol and e["F"] <= 1e-4 and e["C"] <= 1e-3, e
    # effector kinematics are fp64 on the host: identical to the reference
    np.testing.assert_allclose(w.state.effectors, r.effector_state(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("name,res", [("c1", None), ("c5", 64)])
def test_p2g_grid_parity(ref_available, name, res):
    spec = spec_for(name, res)
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    m, v = fl.p2g_grid(w.scene, w.state, ws)
    rm, _, rv = r.p2g_grid()
    assert abs(m.sum() - rm.sum()) <= 1e-6 * rm.sum()
    assert np.max(np.abs(m - rm)) <= 1e-6 * rm.max()
    massive = rm > 1e-12
    assert np.max(np.abs(v[massive] - rv[massive])) <= 1e-5 * max(np.abs(rv).max(), 1e-3)


def test_store_order_bit_exact(ref_available):
    w, _ = pair(spec_for("c1"))
    ws = fl.GpuWorkspace(w.scene)
    fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=5)
    keys, ids, na, x32 = ws.store_order(w.state)
    nd = w.scene.node_dims
    NB = tuple((d + 3) // 4 for d in nd)
    cpu = canonical_keys_cpu(x32[:, :na], w.scene.dx, nd, NB)
    assert np.array_equal(cpu, keys[:na].astype(np.uint64))
    comp = (keys[:na].astype(np.uint64) << np.uint64(32)) | ids[:na].astype(np.uint64)
    assert np.all(np.diff(comp.astype(np.float64)) > 0) or np.all(comp[1:] > comp[:-1])
    assert sorted(ids.tolist()) == list(range(w.scene.n_particles))


def test_rerun_bit_identical(ref_available):
    spec = spec_for("c5", 64)
    outs = []
    for _ in range(2):
        w = fl.build_scene(spec)
        ws = fl.GpuWorkspace(w.scene)
        fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=10)
        outs.append((w.state.x.copy(), w.state.v.copy(), w.state.F.copy(), w.state.C.copy()))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_rollout_loss_parity(ref_available):
    spec = spec_for("c1")
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    acts = fl.ActionTrajectory(2, 5, np.tile(w.init_action, (2, 1)))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    per = []
    l = fl.rollout_loss(w.scene, w.state, acts, loss, per_segment=per, ws=ws)
    rl, rper = r.rollout_loss(acts.values, 5)
    assert abs(l - rl) <= 1e-6 * abs(rl)
    np.testing.assert_allclose(per, rper, rtol=1e-6)


def test_store_order_oversized_blocks():
    """Blocks holding more particles than the per-block counting sort takes (1024) go
    through the bitonic fallback; the store order must still be canonical."""
    w = fl.build_scene(spec_for("c1", 32))
    x = w.state.x.copy()
    dx = w.scene.dx
    # squeeze every particle into 2x2x2 particle blocks around the domain centre
    lo = np.floor(0.5 / dx / 4) * 4 * dx
    x = lo + (x - x.min(0)) / (x.max(0) - x.min(0) + 1e-12) * (8 * dx - 1e-6)
    w.state.x = x
    ws = fl.GpuWorkspace(w.scene)
    keys, ids, na, x32 = ws.store_order(w.state)
    blocks, counts = np.unique(keys[:na] >> 6, return_counts=True)
    assert counts.max() > 1024
    nd = w.scene.node_dims
    NB = tuple((d + 3) // 4 for d in nd)
    cpu = canonical_keys_cpu(x32[:, :na], dx, nd, NB)
    assert np.array_equal(cpu, keys[:na].astype(np.uint64))
    comp = (keys[:na].astype(np.uint64) << np.uint64(32)) | ids[:na].astype(np.uint64)
    assert np.all(comp[1:] > comp[:-1])


def test_continue_from_reference_snapshot(ref_available):
    """A snapshot the reference wrote mid-run (io.hpp state_to_json) continues on the
    device with the same parity as a fresh scene."""
    spec = spec_for("c5", 32)
    w, r = pair(spec)
    r.substep(w.init_action, 6)
    fl.state_from_json(r.snapshot_dump(), w.scene, w.state)
    ws = fl.GpuWorkspace(w.scene)
    fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=5)
    r.substep(w.init_action, 5)
    rs = r.state()
    e = state_errors(w.state, rs, w.scene.dx)
    assert w.state.substep_index == rs["substep"] == 11
    assert e["x"] <= 1e-4 and e["v"] <= 5e-4 and e["F"] <= 1e-4 and e["C"] <= 1e-3, e


def test_rollout_loss_final_state_and_on_substep():
    """rollout_loss's final_state / on_substep (grad.hpp:15-41): the callback sees every
    substep's state and the final state is the one the loss was evaluated on."""
    w = fl.build_scene(spec_for("c1", 16))
    ws = fl.GpuWorkspace(w.scene)
    acts = fl.ActionTrajectory(2, 3, np.tile(w.init_action, (2, 1)))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    seen = []
    fs = w.state.copy()
    l1 = fl.rollout_loss(w.scene, w.state, acts, loss, ws=ws, final_state=fs,
                         on_substep=lambda st: seen.append((st.substep_index, st.x[0].copy())))
    assert [s for s, _ in seen] == list(range(1, 7)) and fs.substep_index == 6
    chain = w.state.copy()
    fl.mpm_substep(w.scene, chain, w.init_action, ws, count=6)
    assert np.array_equal(chain.x, fs.x) and np.array_equal(seen[-1][1], fs.x[0])
    assert fl.rollout_loss(w.scene, w.state, acts, loss, ws=ws) == l1


def test_empty_scene_advances_effectors_and_clock(ref_available, tmp_path):
    """A scene without bodies (test_cli.cpp:75-84): substeps move only the effectors and
    the clock, frames have no rows, the staged grid is empty."""
    from oracle.ref import RefWorld
    from paper_2303_02346_b200 import frames
    spec = {"dim": 3, "grid_resolution": 16, "domain": [1.0, 1.0, 1.0],
            "effectors": [{"shape": {"type": "sphere", "radius": 0.1, "center": [0.0, 0.0, 0.0]},
                           "position": [0.5, 0.5, 0.5], "action_mask": [True, True, True, False, False, True]}]}
    w = fl.build_scene(spec)
    assert w.scene.n_particles == 0
    ws = fl.GpuWorkspace(w.scene)
    act = np.array([0.2, -0.1, 0.05, 0.0, 0.0, 0.7])
    fl.mpm_substep(w.scene, w.state, act, ws, count=7)
    r = RefWorld(spec)
    r.substep(act, 7)
    rs = r.state()
    assert w.state.substep_index == rs["substep"] == 7 and w.state.time == rs["time"]
    np.testing.assert_array_equal(w.state.effectors, r.effector_state())
    m, v = fl.p2g_grid(w.scene, w.state, ws)
    assert not m.any() and not v.any()
    frames.write_frame_csv(tmp_path / "f.csv", w.scene, w.state, 1)
    assert (tmp_path / "f.csv").read_text().count("\n") == 2


def test_single_particle_carried_by_sticky_effector(ref_available):
    """test_autodiff.cpp:47-75 in 3D: one particle inside a sticky box effector moves with
    the commanded velocity, and d|x_T - goal|^2 / da = 2 (x_T - goal) T dt."""
    spec = {"dim": 3, "grid_resolution": 32, "domain": [1.0, 1.0, 1.0], "dt_substep": 1e-4,
            "substeps_per_step": 10, "gravity": [0.0, 0.0, 0.0],
            "materials": [{"name": "chip", "kind": "elastic", "mu": 10.0, "lambda": 10.0, "rho": 1.0}],
            "bodies": [{"name": "tracer", "material": "chip",
                        "shape": {"type": "box", "half_extents": [0.012, 0.012, 0.012], "center": [0.3, 0.4, 0.5]},
                        "particles_per_cell_axis": 1}],
            "effectors": [{"shape": {"type": "box", "half_extents": [0.08, 0.08, 0.08], "center": [0.0, 0.0, 0.0]},
                           "position": [0.3, 0.4, 0.5], "friction": "sticky",
                           "action_mask": [True, True, False, False, False, False]}],
            "loss": {"kind": "target_point", "body": "tracer", "goal": [0.5, 0.6, 0.5], "squared": True,
                     "eval": "final"},
            "optimizer": {"n_segments": 1, "segment_length": 100}}
    w, r = pair(spec)
    assert w.scene.n_particles == 1
    ws = fl.GpuWorkspace(w.scene)
    T, dt = 100, 1e-4
    a = np.array([[0.6, 0.4, 0.0, 0.0, 0.0, 0.0]])
    acts = fl.ActionTrajectory(1, T, a)
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    fs = w.state.copy()
    l = fl.rollout_loss(w.scene, w.state, acts, loss, ws=ws, final_state=fs)
    x0, xT = w.state.x[0], fs.x[0]
    np.testing.assert_allclose(xT[:2], x0[:2] + a[0, :2] * T * dt, rtol=0, atol=2e-6)
    tg = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    expect = (xT - np.array([0.5, 0.6, 0.5])) * (2.0 * T * dt)
    np.testing.assert_allclose(tg.action_grad[0, :2], expect[:2], rtol=2e-4)
    rg = r.grad_trajectory(a, T)
    assert abs(l - rg["loss"]) <= 1e-5 * abs(rg["loss"])
    assert grad_rel_error(tg.action_grad, rg["grad"]) <= 1e-4


def test_host_edits_of_a_resident_state_are_uploaded():
    """A state the workspace already holds is re-uploaded after any host access (the
    arrays may have been edited in place)."""
    w = fl.build_scene(spec_for("c1", 16))
    ws = fl.GpuWorkspace(w.scene)
    acts = fl.ActionTrajectory(1, 3, w.init_action.reshape(1, 6))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    l0 = fl.rollout_loss(w.scene, w.state, acts, loss, ws=ws)
    w.state.v[:] += 0.5  # in place, through the getter
    l1 = fl.rollout_loss(w.scene, w.state, acts, loss, ws=ws)
    w2 = fl.build_scene(spec_for("c1", 16))
    v = w2.state.v
    v += 0.5
    w2.state.v = v
    l2 = fl.rollout_loss(w2.scene, w2.state, acts, fl.LossEvaluator(w2.scene, w2.loss_spec, w2.state),
                         ws=fl.GpuWorkspace(w2.scene))
    assert l1 != l0 and l1 == l2


def test_final_state_keeps_state0_intact():
    w = fl.build_scene(spec_for("c1", 16))
    ws = fl.GpuWorkspace(w.scene)
    acts = fl.ActionTrajectory(2, 3, np.tile(w.init_action, (2, 1)))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=2)  # state0 now device-resident
    s0 = w.state.copy()
    fs = w.state.copy()
    l = fl.rollout_loss(w.scene, w.state, acts, loss, ws=ws, final_state=fs)
    assert np.array_equal(w.state.x, s0.x) and w.state.substep_index == s0.substep_index
    assert fs.substep_index == s0.substep_index + 6
    chain = s0.copy()
    fl.mpm_substep(w.scene, chain, w.init_action, ws, count=6)
    assert np.array_equal(chain.x, fs.x) and np.array_equal(chain.F, fs.F)
    assert fl.rollout_loss(w.scene, w.state, acts, loss, ws=ws) == l
