"""Parity at the benchmark horizons (SURVEY.md 8(c) tolerances), against fixtures the unmodified
reference produced (tests/golden/long/, tests/golden/make_golden_long.py).

  c1  full scene, 4 x 25 substeps: the SURVEY 8(c) golden loss/gradient rows (<= 1e-3 by
      GradReport::rel_error) and the state after 100 substeps (<= 1e-4)
  c4  full scene, the bench workload 10 x 50 = 500 substeps: loss and gradient (<= 1e-2, the
      SURVEY's 500-substep bound), the state after 500 substeps, and a pool-loss 2 x 25 gradient
      whose loss body touches the ladle's contact band (the scene's floater loss has an exactly
      zero gradient over a few substeps)
  c3  full scene (1M non-Newtonian particles), state after 100 substeps
  c2/c3/c5 at grid 64 (c5: every material kind + the rigid brick), 10 x 50 substeps
  c2 full (latte art, emitter active), state after 100 substeps
  c5 full (8M particles, 256^3, the scaling workload), 2 x 10 substeps: state, loss, gradient
  3D 512-substep checkpoint-stride invariance (proj/tests/acceptance_main.cpp:71-100)
"""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests import _long

pytestmark = pytest.mark.gpu

# measured errors (tools/parity_report.py -> profiles/r02_parity.json) sit below these.  The
# conditioning of each scene is in tests/golden/long/calib.json (tools/calibrate_fp32.py: the fp64
# reference from an fp32-rounded initial state): one rounding moves the state by ~2e-6 dx
# (c1, c2, c5) to 4e-6 dx (c3) over 100 substeps, and the device rounds every substep, so
# ~100x that is the fp32 floor.  SVD materials sit higher: c3's non-Newtonian return map
# (von Mises, a non-smooth projection) and c5's stiff solids get 5e-4 (c3's v: 1e-3).  c4
# over the bench's 500 substeps: one rounding moves x by 5.0e-6 dx, so 500 x that = 2.5e-3.
# c2 (full latte art, emitter active) over 100 substeps: one rounding moves x by 3.8e-6 dx, so
# 5e-4.  c5 at its full 256^3 (the scaling workload, 20 substeps): positions, F, loss and
# gradient sit at 6e-5 / 8e-6 / 2e-9 / 3e-6, but the stiff elastic and jelly bodies' velocities
# (and C) carry fp32 F's strain floor amplified by 256^3's 16x stress
# coefficient: v 9.2e-4, C 9.0e-3 of their maxima on particles at 2 % of the peak speed.
STATE_TOL = {"c1_4x25": 1e-4, "c3_fwd100": 5e-4, "c2_64_10x50": 1e-4, "c3_64_10x50": 5e-4,
             "c5_64_10x50": 5e-4, "c4_fwd500": 2.5e-3, "c2_fwd100": 5e-4, "c5_2x10": 1e-4}
V_TOL = {"c3_fwd100": 1e-3, "c3_64_10x50": 1e-3, "c5_2x10": 2e-3}
C_TOL = {"c5_2x10": 2e-2}
GRAD_TOL = {"c1_4x25": 1e-3, "c4pool_2x25": 1e-3, "c4_10x50": 1e-2, "c2_64_10x50": 1e-2, "c3_64_10x50": 1e-2,
            "c5_64_10x50": 1e-2, "c5_2x10": 1e-3}


def _need(name):
    if not _long.available(name):
        pytest.skip(f"fixture {name} not generated")


@pytest.mark.parametrize("name", sorted(STATE_TOL))
def test_state_long_horizon(name):
    _need(name)
    e = _long.run_case(name)
    tol = STATE_TOL[name]
    for k in ("x", "v", "F"):
        assert e[k] <= (V_TOL.get(name, tol) if k == "v" else tol), (k, e)
    assert e["C"] <= C_TOL.get(name, 10 * tol), e  # C = (4/dx^2) sum w v rel^T amplifies v's fp32 rounding
    assert e["centroid"] <= tol, e
    if name in GRAD_TOL:
        assert e["loss"] <= 1e-5, e
        assert e["grad"] <= GRAD_TOL[name], e
        assert e["snapshots"][0] == e["snapshots"][1], e


@pytest.mark.parametrize("name", ["c4_10x50", "c4pool_2x25"])
def test_c4_gradient_long_horizon(name):
    _need(name)
    e = _long.run_case(name)
    assert e["grad_scale"] > 0, e  # a vacuous (all-zero) reference gradient would prove nothing
    assert e["loss"] <= 1e-5 and e["per_segment"] <= 1e-5, e
    assert e["grad"] <= GRAD_TOL[name], e
    assert e["snapshots"][0] == e["snapshots"][1], e


def test_c1_survey_golden_rows():
    """c1, 4 segments x 25 substeps, stride 25 (the values quoted there)."""
    _need("c1_4x25")
    e = _long.run_case("c1_4x25")
    rows = np.array([[-132.81788010, 33.552360172, -59.127013822], [-80.276191988, 19.255038751, -27.877497774],
                     [-38.979694631, 7.9533831004, -11.721372240], [-11.752223729, 2.0727494979, -2.8341349106]])
    g = np.asarray(e["action_grad"])[:, :3]
    assert float(np.abs(g - rows).max() / np.abs(rows).max()) <= 1e-3, g
    assert e["snapshots"][0] == 5


def _elastic_512():
    """proj/tests/acceptance_main.cpp:71-100 in 3D: the gradcheck scene's elastic blob pushed by a
    box effector, 8 segments x 64 substeps, actions set on segments 0 and 3."""
    from tests.golden.make_golden import GRADCHECK_3D
    w = fl.build_scene(GRADCHECK_3D)
    return w, fl.ActionTrajectory(8, 64, _long.elastic512_actions())


def test_stride_invariance_512_substeps():
    w, acts = _elastic_512()
    ws = fl.GpuWorkspace(w.scene)
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    g1 = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=1, ws=ws)
    g8 = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=8, ws=ws)
    g64 = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=64, ws=ws)
    assert (g1.snapshots, g8.snapshots, g64.snapshots) == (513, 65, 9)
    scale = float(np.abs(g1.action_grad).max())
    assert scale > 0
    # the reference asks <= 1e-12 * scale; the device path is bit-identical across strides
    assert np.array_equal(g1.action_grad, g8.action_grad) and np.array_equal(g1.action_grad, g64.action_grad)
    assert g1.loss == g8.loss == g64.loss
    if _long.available("elastic512"):  # and the reference's own 512-substep gradient
        G, _ = _long.load("elastic512")
        assert abs(g1.loss - float(G["loss"])) <= 1e-5 * abs(float(G["loss"]))
        assert float(np.abs(g1.action_grad - G["grad"]).max() / np.abs(G["grad"]).max()) <= 1e-2
