"""Error paths of the device engine map to the reference's exception types with their
context fields (core.hpp:18-48), and a context stays usable after an error:
  * a particle outside the clamped region -> EngineError at P2G (mpm.hpp:265-269,
    test_mpm.cpp:432-437)
  * det(F) <= 0 -> DegenerateDeformation(particle_id) (materials.hpp:20-32)
"""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import spec_for

pytestmark = pytest.mark.gpu


def test_escape_raises_and_context_recovers():
    w = fl.build_scene(spec_for("c1", 16))
    ws = fl.GpuWorkspace(w.scene)
    good = w.state.copy()
    x = w.state.x
    x[7] = [1.5, 0.5, 0.5]  # outside the domain: its stencil leaves the grid
    w.state.x = x
    with pytest.raises(fl.EngineError, match="escaped"):
        fl.mpm_substep(w.scene, w.state, w.init_action, ws)
    # the same workspace runs a good state afterwards, identically to a fresh one
    fl.mpm_substep(w.scene, good, w.init_action, ws, count=3)
    w2 = fl.build_scene(spec_for("c1", 16))
    ws2 = fl.GpuWorkspace(w2.scene)
    fl.mpm_substep(w2.scene, w2.state, w2.init_action, ws2, count=3)
    assert np.array_equal(good.x, w2.state.x) and np.array_equal(good.F, w2.state.F)


@pytest.mark.parametrize("name,res,material_kind", [("c5", 32, 0), ("c1", 16, 2)])
def test_inverted_F_raises_degenerate_with_particle_id(name, res, material_kind):
    w = fl.build_scene(spec_for(name, res))
    kinds = np.array([w.scene.materials[m].kind for m in w.scene.material_id])
    pid = int(np.nonzero(kinds == material_kind)[0][3])
    F = w.state.F
    F[pid] = np.diag([-1.0, 1.0, 1.0])  # det < 0
    w.state.F = F
    ws = fl.GpuWorkspace(w.scene)
    with pytest.raises(fl.DegenerateDeformation) as ei:
        fl.mpm_substep(w.scene, w.state, w.init_action, ws)
    assert ei.value.particle_id == pid


def test_nonfinite_cotangent_raises_adjoint_error_like_reference(ref_available):
    """AdjointState::check_finite (adjoint.hpp:34-45) -> AdjointError(substep): a NaN cotangent
    handed to adjoint_substep raises with the record's substep on both engines; the context
    then runs a finite adjoint identically to a fresh one."""
    from oracle.ref import RefError
    from tests._util import pair
    spec = spec_for("c5", 32)
    w, r = pair(spec)
    ws = fl.GpuWorkspace(w.scene)
    fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=2)
    r.substep(w.init_action, 2)
    n = w.scene.n_particles
    xb = np.zeros((n, 3))
    xb[11, 0] = np.nan
    zeros = [np.zeros((n, 3)), np.zeros((n, 3, 3)), np.zeros((n, 3, 3))]
    with pytest.raises(RefError) as er:
        r.adjoint_substep(w.init_action, xb, *zeros)
    adj = fl.AdjointState(xb.copy(), *[z.copy() for z in zeros], np.zeros((w.scene.n_effectors, 12)))
    with pytest.raises(fl.AdjointError) as eg:
        fl.adjoint_substep(w.scene, fl.SubstepRecord(2, w.init_action, w.state), adj, np.zeros(6), ws)
    assert eg.value.substep == er.value.substep == 2
    assert "non-finite adjoint at substep 2" in str(er.value) and "non-finite adjoint at substep 2" in str(eg.value)
    # recovery: a finite cotangent on the same workspace equals a fresh workspace's result
    rng = np.random.default_rng(1)
    xb2 = rng.normal(size=(n, 3))
    a1 = fl.AdjointState(xb2.copy(), *[z.copy() for z in zeros], np.zeros((w.scene.n_effectors, 12)))
    fl.adjoint_substep(w.scene, fl.SubstepRecord(2, w.init_action, w.state), a1, np.zeros(6), ws)
    ws2 = fl.GpuWorkspace(w.scene)
    a2 = fl.AdjointState(xb2.copy(), *[z.copy() for z in zeros], np.zeros((w.scene.n_effectors, 12)))
    fl.adjoint_substep(w.scene, fl.SubstepRecord(2, w.init_action, w.state), a2, np.zeros(6), ws2)
    assert np.array_equal(a1.x_bar, a2.x_bar) and np.array_equal(a1.F_bar, a2.F_bar)


def test_nonfinite_loss_raises_like_reference(ref_available):
    """grad.hpp:91-92: a non-finite forward loss raises EngineError before any backward."""
    from oracle.ref import RefError, RefWorld
    spec = spec_for("c1", 16)
    spec["loss"]["weight"] = 1e305  # the summed loss overflows to inf in fp64
    w = fl.build_scene(spec)
    r = RefWorld(spec)
    vals = np.tile(w.init_action, (2, 1))
    with pytest.raises(RefError, match="non-finite forward loss"):
        r.grad_trajectory(vals, 3, stride=2)
    ws = fl.GpuWorkspace(w.scene)
    with pytest.raises(fl.EngineError, match="non-finite forward loss"):
        fl.grad_trajectory(w.scene, w.state, fl.ActionTrajectory(2, 3, vals),
                           fl.LossEvaluator(w.scene, w.loss_spec, w.state), stride=2, ws=ws)


def test_collapsed_rigid_body_raises_rigidity_error_like_reference(ref_available):
    """rigid_shape_match (materials.hpp:178-192): every member of the brick at one point gives a
    zero covariance -> RigidityError(body_id) in the rigid pass of the first substep."""
    from oracle.ref import RefError
    from tests._util import pair
    w, r = pair(spec_for("c5", 32))
    rb = r.rigid_bodies()[0]
    x = w.state.x
    x[rb["members"]] = x[rb["members"]].mean(0)
    w.state.x = x
    r.set_state(x=x)
    with pytest.raises(RefError) as er:
        r.substep(w.init_action, 1)
    ws = fl.GpuWorkspace(w.scene)
    with pytest.raises(fl.RigidityError) as eg:
        fl.mpm_substep(w.scene, w.state, w.init_action, ws)
    assert eg.value.body_id == er.value.body_id == rb["body_id"] == 4
    assert "degenerate covariance" in str(eg.value)
