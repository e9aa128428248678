"""Known-answer checks in the style of the reference's own suite (proj/tests/test_mpm.cpp,
SURVEY.md 8(c)), run on the device path, with fp32 tolerances:
  * P2G conserves mass and momentum (test_mpm.cpp:58-72)
  * a uniform velocity field round-trips through the grid (74-101) and C stays ~0
  * momentum is conserved over many substeps away from walls, without gravity (340-370)
  * the CFL cap bounds |v| by cfl * dx / dt (386-393)
  * emitter particles activate at start + k * interval (395-430)
  * a resting body stays put (325-338); gravity and sticky effectors set the grid
    velocity exactly (103-113, 192-207); a head-on elastic collision conserves momentum
    and swaps the blocks' directions (340-370)
"""
import copy

import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import spec_for

pytestmark = pytest.mark.gpu


def _free_blob(res=32, v=(0.0, 0.0, 0.0), kind="liquid", mu=0.0):
    """A cube of material in the middle of the domain, no gravity, no effector."""
    spec = copy.deepcopy(spec_for("c1", res))
    spec["gravity"] = [0.0, 0.0, 0.0]
    spec["materials"] = [{"name": "m", "kind": kind, "mu": mu, "lambda": 277.78, "rho": 1.0}]
    spec["bodies"] = [{"name": "blob", "material": "m",
                       "shape": {"type": "box", "half_extents": [0.125] * 3, "center": [0.5] * 3},
                       "particles_per_cell_axis": 2, "jitter": 0.2, "velocity": list(v)}]
    spec["effectors"] = []
    spec["action_bounds"] = {"lo": [0] * 6, "hi": [0] * 6}
    spec["loss"] = {"kind": "target_point", "body": "blob", "goal": [0.5, 0.5, 0.5]}
    return spec


def test_p2g_conserves_mass_and_momentum():
    w = fl.build_scene(_free_blob(v=(0.3, -0.2, 0.1)))
    rng = np.random.default_rng(0)
    v = w.state.v + 0.05 * rng.standard_normal(w.state.v.shape)
    w.state.v = v
    ws = fl.GpuWorkspace(w.scene)
    m, vel = fl.p2g_grid(w.scene, w.state, ws)
    pm = w.scene.mass
    assert abs(m.sum() - pm.sum()) <= 1e-6 * pm.sum()
    # no gravity, no walls touched, no effectors: grid velocity = p / m
    p_grid = (m[..., None] * vel).reshape(-1, 3).sum(0)
    p_part = (pm[:, None] * v).sum(0)
    assert np.max(np.abs(p_grid - p_part)) <= 1e-5 * pm.sum() * np.abs(v).max()


def test_uniform_velocity_round_trip():
    u = np.array([0.4, -0.3, 0.2])
    w = fl.build_scene(_free_blob(v=tuple(u)))
    ws = fl.GpuWorkspace(w.scene)
    fl.mpm_substep(w.scene, w.state, np.zeros(6), ws)
    assert np.max(np.abs(w.state.v - u)) <= 2e-6 * np.abs(u).max()
    assert np.max(np.abs(w.state.C)) <= 1e-3  # k4 * dx * O(1e-7 |u|)


def test_momentum_conserved_over_many_substeps():
    w = fl.build_scene(_free_blob(v=(0.2, 0.1, -0.15)))
    rng = np.random.default_rng(1)
    v = w.state.v + 0.1 * rng.standard_normal(w.state.v.shape)
    w.state.v = v
    pm = w.scene.mass
    p0 = (pm[:, None] * v).sum(0)
    ws = fl.GpuWorkspace(w.scene)
    fl.mpm_substep(w.scene, w.state, np.zeros(6), ws, count=500)
    p1 = (pm[:, None] * w.state.v).sum(0)
    assert np.max(np.abs(p1 - p0)) <= 1e-4 * pm.sum() * np.abs(v).max()


def test_cfl_cap():
    w = fl.build_scene(_free_blob(v=(5000.0, 0.0, 0.0)))
    ws = fl.GpuWorkspace(w.scene)
    fl.mpm_substep(w.scene, w.state, np.zeros(6), ws)
    vmax = 0.9 * w.scene.dx / w.scene.dt_substep
    assert np.max(np.linalg.norm(w.state.v, axis=1)) <= vmax * (1 + 1e-6)


def test_emitter_activation_schedule():
    spec = spec_for("c2", 64)  # 63 emitter particles, one per substep
    w = fl.build_scene(spec)
    act = w.scene.activation_substep
    assert (act > 0).sum() > 20
    ws = fl.GpuWorkspace(w.scene)
    for _ in range(3):
        fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=9)
        t = w.state.substep_index
        _, _, na, _ = ws.store_order(w.state)
        # emitted at the start of substep a (mpm.hpp:435-449): in the store from then on
        assert na == int(np.sum(act < t)), (t, na)


def _single_particle(res=16, gravity=(0.0, 0.0, 0.0), effectors=()):
    return {"dim": 3, "grid_resolution": res, "domain": [1.0, 1.0, 1.0], "dt_substep": 1e-4,
            "gravity": list(gravity),
            "materials": [{"name": "m", "kind": "elastic", "mu": 10.0, "lambda": 10.0, "rho": 1.0}],
            "bodies": [{"name": "p", "material": "m",
                        "shape": {"type": "box", "half_extents": [0.012] * 3, "center": [0.5] * 3},
                        "particles_per_cell_axis": 1}],
            "effectors": list(effectors)}


def test_substep_identity_at_rest():
    """test_mpm.cpp:325-338: a resting liquid without gravity does not move."""
    spec = _free_blob(v=(0.0, 0.0, 0.0))
    w = fl.build_scene(spec)
    x0 = w.state.x.copy()
    ws = fl.GpuWorkspace(w.scene)
    fl.mpm_substep(w.scene, w.state, np.zeros(6), ws)
    assert w.state.substep_index == 1 and w.state.time == w.scene.dt_substep
    assert np.max(np.abs(w.state.x - x0)) <= 1e-7  # fp32 storage of the positions
    assert not w.state.v.any()


def test_gravity_increments_grid_velocity():
    """test_mpm.cpp:103-113: the node under a lone particle gets v = g dt."""
    w = fl.build_scene(_single_particle(gravity=(0.0, -9.8, 0.0)))
    assert w.scene.n_particles == 1
    ws = fl.GpuWorkspace(w.scene)
    m, v = fl.p2g_grid(w.scene, w.state, ws)
    dt = w.scene.dt_substep
    assert m[8, 8, 8] > 0
    np.testing.assert_allclose(v[8, 8, 8], [0.0, -9.8 * dt, 0.0], rtol=1e-6, atol=1e-12)


def test_sticky_effector_drives_contacted_nodes():
    """test_mpm.cpp:192-207: a node inside a sticky effector takes the effector velocity."""
    eff = {"shape": {"type": "box", "half_extents": [0.2] * 3, "center": [0.0] * 3}, "position": [0.5] * 3,
           "friction": "sticky", "action_mask": [True] * 6}
    w = fl.build_scene(_single_particle(effectors=[eff]))
    e = w.state.effectors
    e[0, 12:15] = [0.4, -0.7, 0.2]
    w.state.effectors = e
    ws = fl.GpuWorkspace(w.scene)
    m, v = fl.p2g_grid(w.scene, w.state, ws)
    assert m[8, 8, 8] > 0
    np.testing.assert_allclose(v[8, 8, 8], [0.4, -0.7, 0.2], rtol=1e-6)


def test_momentum_exchange_in_frictionless_collision():
    """test_mpm.cpp:340-370 in 3D: two equal elastic blocks collide head on; mass and
    momentum are conserved (fp32 state: relative 1e-5) and the blocks swap direction."""
    spec = {"dim": 3, "grid_resolution": 64, "domain": [1.0, 1.0, 1.0], "dt_substep": 1e-4,
            "substeps_per_step": 10, "gravity": [0.0, 0.0, 0.0],
            "materials": [{"name": "block", "kind": "elastic", "mu": 416.67, "lambda": 277.78, "rho": 1.0}],
            "bodies": [{"name": "left", "material": "block",
                        "shape": {"type": "box", "half_extents": [0.06] * 3, "center": [0.35, 0.5, 0.5]},
                        "velocity": [1.0, 0.0, 0.0]},
                       {"name": "right", "material": "block",
                        "shape": {"type": "box", "half_extents": [0.06] * 3, "center": [0.65, 0.5, 0.5]},
                        "velocity": [-1.0, 0.0, 0.0]}]}
    w = fl.build_scene(spec)
    pm = w.scene.mass
    v0 = w.state.v
    scale = float(np.sum(pm * np.linalg.norm(v0, axis=1)))
    p0 = (pm[:, None] * v0).sum(0)
    ws = fl.GpuWorkspace(w.scene)
    fl.mpm_substep(w.scene, w.state, np.zeros(6), ws, count=2500)
    v = w.state.v
    assert np.all(np.isfinite(v))
    p1 = (pm[:, None] * v).sum(0)
    assert np.linalg.norm(p1 - p0) <= 1e-5 * scale
    left = w.scene.body_id == 0
    vl = (pm[left, None] * v[left]).sum(0) / pm[left].sum()
    vr = (pm[~left, None] * v[~left]).sum(0) / pm[~left].sum()
    assert vl[0] < -0.2 and vr[0] > 0.2, (vl, vr)
