"""Populations of independent rollouts on one GPU: a pool of
contexts evaluated concurrently gives exactly the per-candidate results of one
context evaluating them in turn."""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import spec_for

pytestmark = pytest.mark.gpu


def test_population_matches_sequential():
    spec = spec_for("c1", 32)
    w = fl.build_scene(spec)
    rng = np.random.default_rng(11)
    pop = [fl.ActionTrajectory(2, 5, np.tile(w.init_action, (2, 1)) + 0.2 * rng.standard_normal((2, 6)))
           for _ in range(7)]
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    ws = fl.GpuWorkspace(w.scene)
    seq_l = [fl.rollout_loss(w.scene, w.state, a, loss, ws=ws) for a in pop]
    seq_g = [fl.grad_trajectory(w.scene, w.state, a, loss, ws=ws) for a in pop]
    pool = fl.WorkspacePool(w.scene, 3)
    bl = fl.rollout_loss_batch(w.scene, w.state, pop, loss, pool)
    bg = fl.grad_trajectory_batch(w.scene, w.state, pop, loss, pool)
    pool.close()
    assert bl == seq_l
    for a, b in zip(seq_g, bg):
        assert a.loss == b.loss and np.array_equal(a.action_grad, b.action_grad)
