"""Replica contexts: a population of one scene in one grid, every kernel
launch covering all candidates (flume_ctx_create_replicas).  Each replica must evolve exactly
like a single context given that replica's actions: final states bit-identical, losses equal
up to the order of the fp64 loss sums (the replicas' particles sit at other store slots), and
gradients (grad_trajectory_replicas) up to the order of the fp64 effector-bar sums.

  c1        one liquid + a box effector, full size, 4 candidates
  c2 @ 64   emitters attached to an effector (activation per replica), 3 candidates
  c5 @ 32   every material kind + the rigid brick + a sphere effector, 4 candidates
"""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import spec_for

pytestmark = pytest.mark.gpu


def _population(w, R, nseg, seed=0):
    rng = np.random.default_rng(seed)
    base = np.asarray(w.init_action, dtype=np.float64)
    out = []
    for r in range(R):
        vals = np.tile(base, (nseg, 1)) + (0.0 if r == 0 else 0.3) * rng.standard_normal((nseg, 6))
        out.append(fl.ActionTrajectory(nseg, 0, vals))
    return out


@pytest.mark.parametrize("name,res,R,nseg,seglen", [("c1", None, 4, 2, 10), ("c2", 64, 3, 2, 10),
                                                    ("c5", 32, 4, 2, 5)])
def test_replicas_match_single_contexts(name, res, R, nseg, seglen):
    w = fl.build_scene(spec_for(name, res))
    pop = _population(w, R, nseg)
    for a in pop:
        a.segment_length = seglen
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    rws = fl.ReplicaWorkspace(w.scene, R)
    per_r, fin_r = [], []
    losses = fl.rollout_loss_replicas(w.scene, w.state, pop, loss, rws, per_segment=per_r, final_states=fin_r)
    rws.close()
    ws = fl.GpuWorkspace(w.scene)
    for r in range(R):
        per, fin = [], w.state.copy()
        l1 = fl.rollout_loss(w.scene, w.state.copy(), pop[r], loss, per_segment=per, ws=ws, final_state=fin)
        assert abs(losses[r] - l1) <= 1e-12 * abs(l1), (r, losses[r], l1)
        np.testing.assert_allclose(per_r[r], per, rtol=1e-12, atol=0)
        f = fin_r[r]
        for got, want in ((f.x, fin.x), (f.v, fin.v), (f.F, fin.F), (f.C, fin.C)):
            assert np.array_equal(got, want), r
        assert np.array_equal(f._eff, fin._eff)
        assert f.substep_index == fin.substep_index == nseg * seglen
    ws.close()
    # the candidates differ: the population is not R copies of one rollout
    assert len({round(l, 9) for l in losses}) > 1


@pytest.mark.parametrize("name,res,R,nseg,seglen,stride", [("c1", None, 3, 2, 10, 5), ("c5", 32, 3, 2, 5, 5),
                                                           ("c2", 64, 2, 2, 10, 10)])
def test_replica_gradients_match_single_contexts(name, res, R, nseg, seglen, stride):
    """grad_trajectory of a population in one replica context (records, checkpoint replays,
    effector bars of every replica's effectors) against single contexts: the particle
    cotangents are the same per block; only the fp64 effector-bar sums run in another order."""
    w = fl.build_scene(spec_for(name, res))
    pop = _population(w, R, nseg, seed=1)
    for a in pop:
        a.segment_length = seglen
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    rws = fl.ReplicaWorkspace(w.scene, R)
    gr = fl.grad_trajectory_replicas(w.scene, w.state, pop, loss, rws, stride=stride)
    rws.close()
    ws = fl.GpuWorkspace(w.scene)
    for r in range(R):
        g1 = fl.grad_trajectory(w.scene, w.state, pop[r], loss, stride=stride, ws=ws)
        assert abs(gr[r].loss - g1.loss) <= 1e-12 * abs(g1.loss), (r, gr[r].loss, g1.loss)
        np.testing.assert_allclose(gr[r].per_segment, g1.per_segment, rtol=1e-12, atol=0)
        scale = np.abs(g1.action_grad).max()
        assert scale > 0
        assert np.abs(gr[r].action_grad - g1.action_grad).max() <= 1e-9 * scale, (r, gr[r].action_grad, g1.action_grad)
        assert gr[r].snapshots == g1.snapshots
    ws.close()


def test_replica_context_rejects_single_scene_calls():
    w = fl.build_scene(spec_for("c1", 32))
    rws = fl.ReplicaWorkspace(w.scene, 2)
    acts = fl.ActionTrajectory(1, 2, w.init_action.reshape(1, 6))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    with pytest.raises(ValueError):
        fl.grad_trajectory(w.scene, rws.replicate(w.state), acts, loss, ws=rws)
    with pytest.raises(ValueError):
        fl.rollout_loss(w.scene, rws.replicate(w.state), acts, loss, ws=rws)
    rws.close()


def test_replicas_full_size_c4():
    """Two candidates of the benchmark scene (2 x 1,027,233 particles, 128^3 each) in one
    replica context: final states bit-identical to single contexts after 20 substeps."""
    w = fl.build_scene(spec_for("c4"))
    pop = _population(w, 2, 1, seed=3)
    for a in pop:
        a.segment_length = 20
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    rws = fl.ReplicaWorkspace(w.scene, 2)
    fin_r = []
    losses = fl.rollout_loss_replicas(w.scene, w.state, pop, loss, rws, final_states=fin_r)
    rws.close()
    ws = fl.GpuWorkspace(w.scene)
    for r in range(2):
        fin = w.state.copy()
        l1 = fl.rollout_loss(w.scene, w.state.copy(), pop[r], loss, ws=ws, final_state=fin)
        assert abs(losses[r] - l1) <= 1e-12 * abs(l1)
        for got, want in ((fin_r[r].x, fin.x), (fin_r[r].v, fin.v), (fin_r[r].F, fin.F), (fin_r[r].C, fin.C)):
            assert np.array_equal(got, want), r
    ws.close()


def test_replica_launches_do_not_scale_with_the_population():
    """One launch per kernel stage covers every candidate: a 4-candidate gradient issues the
    single context's launches plus only the per-replica loss evaluations at segment ends."""
    w = fl.build_scene(spec_for("c1", 32))
    acts = fl.ActionTrajectory(2, 5, np.tile(w.init_action, (2, 1)))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    ws = fl.GpuWorkspace(w.scene)
    fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    single = ws.last_timing().launches
    ws.close()
    R = 4
    rws = fl.ReplicaWorkspace(w.scene, R)
    fl.grad_trajectory_replicas(w.scene, w.state, [acts] * R, loss, rws)
    rep = rws.last_timing().launches
    rws.close()
    assert single <= rep <= single + 4 * (R - 1) * acts.n_segments, (single, rep)


def test_replica_gradients_full_size_c4():
    """Gradients of two benchmark-scene candidates (2 x 1M particles) in one replica context
    against single contexts, 2 segments x 10 substeps with a checkpoint replay."""
    w = fl.build_scene(spec_for("c4"))
    pop = _population(w, 2, 2, seed=5)
    for a in pop:
        a.segment_length = 10
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    rws = fl.ReplicaWorkspace(w.scene, 2)
    gr = fl.grad_trajectory_replicas(w.scene, w.state, pop, loss, rws, stride=10)
    rws.close()
    ws = fl.GpuWorkspace(w.scene)
    for r in range(2):
        g1 = fl.grad_trajectory(w.scene, w.state, pop[r], loss, stride=10, ws=ws)
        assert abs(gr[r].loss - g1.loss) <= 1e-12 * abs(g1.loss)
        scale = max(np.abs(g1.action_grad).max(), 1e-30)
        assert np.abs(gr[r].action_grad - g1.action_grad).max() <= 1e-9 * scale
    ws.close()


def test_batch_api_on_a_replica_workspace():
    """rollout_loss_batch / grad_trajectory_batch take a ReplicaWorkspace like a pool: a
    population of 5 runs as groups of 2 (the last padded) with the single-context results."""
    w = fl.build_scene(spec_for("c1", 32))
    pop = _population(w, 5, 2, seed=7)
    for a in pop:
        a.segment_length = 4
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    rws = fl.ReplicaWorkspace(w.scene, 2)
    lb = fl.rollout_loss_batch(w.scene, w.state, pop, loss, rws)
    gb = fl.grad_trajectory_batch(w.scene, w.state, pop, loss, rws, stride=4)
    rws.close()
    ws = fl.GpuWorkspace(w.scene)
    assert len(lb) == len(gb) == 5
    for r in range(5):
        l1 = fl.rollout_loss(w.scene, w.state, pop[r], loss, ws=ws)
        g1 = fl.grad_trajectory(w.scene, w.state, pop[r], loss, stride=4, ws=ws)
        assert abs(lb[r] - l1) <= 1e-12 * abs(l1) and abs(gb[r].loss - g1.loss) <= 1e-12 * abs(g1.loss)
        assert np.abs(gb[r].action_grad - g1.action_grad).max() <= 1e-9 * max(np.abs(g1.action_grad).max(), 1e-30)
    ws.close()
