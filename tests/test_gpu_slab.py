"""x-slab decomposition against one rank on the same device.

The slab ranks run in one process (flume_group_create, ThreadTransport); on a
single B200 they share the device, which exercises the same halo / migration /
all-reduce protocol the NCCL transport carries between GPUs.

Contract (include/flume_b200.h): particle states are bit-identical to one
rank's -- every grid node sums the same scatter tiles in the same order, rigid
fits are solved from all-reduced member positions (disjoint support, exact) --
while losses and action gradients differ only by the order of their final
cross-rank sums (<= 1e-12 relative for losses, 1e-9 for gradients).
"""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import spec_for

pytestmark = pytest.mark.gpu

SCENES = [("c1", 32), ("c2", 32), ("c3", 32), ("c4", 32), ("c5", 32)]


def _state(st):
    return [np.array(a, copy=True) for a in (st.x, st.v, st.F, st.C)]


def _run(spec, ranks, count, action=None):
    w = fl.build_scene(spec)
    ws = fl.GpuWorkspace(w.scene, ranks=ranks)
    fl.mpm_substep(w.scene, w.state, w.init_action if action is None else action, ws, count=count)
    out = _state(w.state)
    info = ws.slab_info()
    ws.close()
    return out, info


@pytest.mark.parametrize("name,res", SCENES)
@pytest.mark.parametrize("ranks", [2, 3])
def test_slab_forward_bit_identical(name, res, ranks):
    spec = spec_for(name, res)
    one, _ = _run(spec, 1, 20)
    many, info = _run(spec, ranks, 20)
    for a, b, f in zip(one, many, "xvFC"):
        assert np.array_equal(a, b), (f, float(np.max(np.abs(a - b))))
    # the slabs tile the x columns
    cols = [(s0, s1) for _, s0, s1, _ in info]
    assert cols[0][0] == 0 and all(cols[i][1] == cols[i + 1][0] for i in range(ranks - 1))
    assert all(s1 > s0 for s0, s1 in cols)


def test_slab_migration_happens_and_conserves():
    """A fast blob crosses slab faces: particles migrate, none are lost or duplicated."""
    spec = spec_for("c1", 32)
    w = fl.build_scene(spec)
    v = w.state.v
    v[:, 0] = 100.0  # 0.32 cells per substep along x at res 32 (CFL cap 281 m/s)
    w.state.v = v
    ref = fl.build_scene(spec)
    ref.state.v = v
    ws1 = fl.GpuWorkspace(ref.scene)
    ws3 = fl.GpuWorkspace(w.scene, ranks=3)
    ws3._upload(w.state)
    start = [n for *_, n in ws3.slab_info()]
    fl.mpm_substep(ref.scene, ref.state, ref.init_action, ws1, count=30)
    fl.mpm_substep(w.scene, w.state, w.init_action, ws3, count=30)
    end = [n for *_, n in ws3.slab_info()]
    assert sum(end) == sum(start) == w.scene.n_particles
    assert end[0] < start[0] and end[2] > start[2], (start, end)  # the blob moved up in x
    for a, b in zip(_state(ref.state), _state(w.state)):
        assert np.array_equal(a, b)


def test_slab_migration_overflow_reruns_larger():
    """Migration messages have a fixed capacity (counts stay on the device); a call whose
    migrants exceed it sets the overflow flag and is re-run from its start with 4x the
    capacity.  Forced here with 2 slots per message on the fast blob: the states are still
    one rank's bit for bit, for a mutating call (mpm_substep) and a pure one (grad_trajectory)."""
    spec = spec_for("c1", 32)
    w = fl.build_scene(spec)
    v = w.state.v
    v[:, 0] = 100.0
    w.state.v = v
    ref = fl.build_scene(spec)
    ref.state.v = v
    ws1 = fl.GpuWorkspace(ref.scene)
    ws3 = fl.GpuWorkspace(w.scene, ranks=3)
    ws3._upload(w.state)
    ws3.set_migration_capacity(2)
    fl.mpm_substep(ref.scene, ref.state, ref.init_action, ws1, count=12)
    fl.mpm_substep(w.scene, w.state, w.init_action, ws3, count=12)
    stats = ws3.migration_stats()
    assert all(n >= 1 and cap > 2 for cap, n in stats), stats
    for a, b in zip(_state(ref.state), _state(w.state)):
        assert np.array_equal(a, b)
    ws3.set_migration_capacity(2)
    acts = fl.ActionTrajectory(2, 4, np.tile(w.init_action, (2, 1)))
    g1 = fl.grad_trajectory(ref.scene, ref.state, acts, fl.LossEvaluator(ref.scene, ref.loss_spec, ref.state),
                            stride=2, ws=ws1)
    g3 = fl.grad_trajectory(w.scene, w.state, acts, fl.LossEvaluator(w.scene, w.loss_spec, w.state), stride=2,
                            ws=ws3)
    assert ws3.migration_stats()[0][1] > stats[0][1]
    assert abs(g1.loss - g3.loss) <= 1e-12 * abs(g1.loss)
    gg1, gg3 = np.asarray(g1.action_grad), np.asarray(g3.action_grad)
    assert np.max(np.abs(gg1 - gg3)) <= 1e-9 * np.max(np.abs(gg1)), (gg1, gg3)


@pytest.mark.parametrize("name,res,nseg,seglen,stride", [("c1", 32, 2, 5, 5), ("c2", 32, 2, 4, 3),
                                                         ("c5", 32, 2, 3, 2), ("c4", 32, 1, 6, 0)])
def test_slab_grad_trajectory_matches_one_rank(name, res, nseg, seglen, stride):
    spec = spec_for(name, res)
    res_ = []
    for ranks in (1, 2):
        w = fl.build_scene(spec)
        ws = fl.GpuWorkspace(w.scene, ranks=ranks)
        acts = fl.ActionTrajectory(nseg, seglen, np.tile(w.init_action, (nseg, 1)))
        loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
        res_.append(fl.grad_trajectory(w.scene, w.state, acts, loss, stride=stride, ws=ws))
        ws.close()
    a, b = res_
    assert abs(a.loss - b.loss) <= 1e-12 * abs(a.loss)
    assert a.snapshots == b.snapshots
    g1, g2 = np.asarray(a.action_grad), np.asarray(b.action_grad)
    assert np.max(np.abs(g1 - g2)) <= 1e-9 * max(np.max(np.abs(g1)), 1e-30), (g1, g2)


def test_slab_rollout_and_grid():
    spec = spec_for("c5", 32)
    out = []
    for ranks in (1, 3):
        w = fl.build_scene(spec)
        ws = fl.GpuWorkspace(w.scene, ranks=ranks)
        m, v = fl.p2g_grid(w.scene, w.state, ws)
        acts = fl.ActionTrajectory(2, 4, np.tile(w.init_action, (2, 1)))
        loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
        per = []
        l = fl.rollout_loss(w.scene, w.state, acts, loss, per_segment=per, ws=ws)
        out.append((m, v, l, per))
        ws.close()
    (m1, v1, l1, p1), (m3, v3, l3, p3) = out
    assert np.array_equal(m1, m3) and np.array_equal(v1, v3)
    assert abs(l1 - l3) <= 1e-12 * abs(l1)
    np.testing.assert_allclose(p1, p3, rtol=1e-12)


def test_nccl_transport_single_rank_matches_plain_context():
    """The NCCL transport (dlopen'ed libnccl, comm init, all-reduce, count exchange)
    on a one-rank group: the slab code path with one slab reproduces a plain context.
    (Multi-rank NCCL needs several GPUs; the protocol itself is covered above.)"""
    spec = spec_for("c5", 32)
    w1 = fl.build_scene(spec)
    ws1 = fl.GpuWorkspace(w1.scene)
    w2 = fl.build_scene(spec)
    ws2 = fl.GpuWorkspace.distributed(w2.scene, 0, 0, 1, fl.dist_unique_id())
    fl.mpm_substep(w1.scene, w1.state, w1.init_action, ws1, count=10)
    fl.mpm_substep(w2.scene, w2.state, w2.init_action, ws2, count=10)
    for a, b in zip(_state(w1.state), _state(w2.state)):
        assert np.array_equal(a, b)
    acts = fl.ActionTrajectory(2, 3, np.tile(w1.init_action, (2, 1)))
    g1 = fl.grad_trajectory(w1.scene, w1.state, acts, fl.LossEvaluator(w1.scene, w1.loss_spec, w1.state), ws=ws1)
    g2 = fl.grad_trajectory(w2.scene, w2.state, acts, fl.LossEvaluator(w2.scene, w2.loss_spec, w2.state), ws=ws2)
    assert g1.loss == g2.loss and np.array_equal(g1.action_grad, g2.action_grad)


def test_slab_full_c5_bit_identical():
    """The scaling target scene at full size (8M particles, 256^3): four
    slabs give one rank's particle states bit for bit after 5 substeps."""
    spec = spec_for("c5")
    one, _ = _run(spec, 1, 5)
    four, info = _run(spec, 4, 5)
    assert len(info) == 4 and all(s[3] > 1_000_000 for s in info), info
    for a, b in zip(one, four):
        assert np.array_equal(a, b)
