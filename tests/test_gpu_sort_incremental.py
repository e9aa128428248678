"""Incremental particle sort (csrc/fl_sort.cu header) against the full block sort.

Between chained substeps only the blocks a particle entered, left or moved inside are
re-sorted; the rest keep their order.  The canonical (cell key, id) order is unique, so the
store order, every state bit and every gradient bit must equal the full sort's.

  c1        one liquid (every block on the plain-liquid path)
  c2 @ 64   emitters: activation substeps fall back to the full sort
  c3 @ 64   non-Newtonian: every block on the SVD path
  c5 @ 64   every material kind + the rigid brick: block kinds change as materials mix
  c4        the benchmark scene at full size
  squeezed  c1 squeezed into 2x2x2 particle blocks: dirty blocks above the shared-memory
            counting sort's capacity take the bitonic path
"""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import canonical_keys_cpu, spec_for

pytestmark = pytest.mark.gpu


def _forward(spec, n, inc, x=None):
    w = fl.build_scene(spec)
    if x is not None:
        w.state.x = x
    ws = fl.GpuWorkspace(w.scene)
    ws.set_incremental_sort(inc)
    fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=n)
    stats = ws.sort_stats()[0]
    keys, ids, na, x32 = ws.store_order(w.state)  # (the next substep's sort: one more)
    state = [np.array(a, copy=True) for a in (w.state.x, w.state.v, w.state.F, w.state.C)]
    ws.close()
    return w, (keys, ids, na, x32), stats, state


def _check_same(a, b, w):
    (ka, ia, na, xa), (kb, ib, nb, xb) = a, b
    assert na == nb
    assert np.array_equal(ka, kb) and np.array_equal(ia, ib)
    assert np.array_equal(xa.view(np.uint32), xb.view(np.uint32))
    nd = w.scene.node_dims
    NB = tuple((d + 3) // 4 for d in nd)
    cpu = canonical_keys_cpu(xa[:, :na], w.scene.dx, nd, NB)
    assert np.array_equal(cpu, ka[:na].astype(np.uint64))
    comp = (ka[:na].astype(np.uint64) << np.uint64(32)) | ia[:na].astype(np.uint64)
    assert np.all(comp[1:] > comp[:-1])


@pytest.mark.parametrize("name,res,n", [("c1", None, 200), ("c2", 64, 100), ("c3", 64, 100), ("c5", 64, 100),
                                        ("c4", None, 20)])
def test_incremental_sort_matches_full(name, res, n):
    spec = spec_for(name, res)
    wa, oa, sa, sta = _forward(spec, n, True)
    wb, ob, sb, stb = _forward(spec, n, False)
    _check_same(oa, ob, wa)
    for a, b in zip(sta, stb):
        assert np.array_equal(a, b)
    assert sb[0] == 0 and sb[1] == n + 1  # upload + every substep
    assert sa[0] + sa[1] == n + 1
    if name != "c2":  # no activation: every substep chained, from the upload's sort on
        assert sa == (n, 1), sa


@pytest.mark.parametrize("name", ["c1", "c5"])
def test_incremental_sort_gradients_identical(name):
    """grad_trajectory (records, checkpoint replays at stride 5) gives the same bits."""
    spec = spec_for(name, None if name == "c1" else 64)
    out = []
    for inc in (True, False):
        w = fl.build_scene(spec)
        ws = fl.GpuWorkspace(w.scene)
        ws.set_incremental_sort(inc)
        acts = fl.ActionTrajectory(2, 10, np.tile(w.init_action, (2, 1)))
        loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
        g = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=5, ws=ws)
        out.append((g.loss, np.array(g.action_grad, copy=True), ws.sort_stats()[0]))
        ws.close()
    (la, ga, sa), (lb, gb, sb) = out
    assert la == lb and np.array_equal(ga, gb)
    assert np.any(ga != 0)
    assert sa[0] > 0 and sb[0] == 0


def test_incremental_sort_oversized_blocks():
    w0 = fl.build_scene(spec_for("c1", 32))
    x = w0.state.x.copy()
    dx = w0.scene.dx
    lo = np.floor(0.5 / dx / 4) * 4 * dx
    x = lo + (x - x.min(0)) / (x.max(0) - x.min(0) + 1e-12) * (8 * dx - 1e-6)
    spec = spec_for("c1", 32)
    wa, oa, sa, sta = _forward(spec, 4, True, x=x)
    wb, ob, sb, stb = _forward(spec, 4, False, x=x)
    keys, _, na, _ = oa
    assert np.unique(keys[:na] >> 6, return_counts=True)[1].max() > 1024
    _check_same(oa, ob, wa)
    for a, b in zip(sta, stb):
        assert np.array_equal(a, b)
    assert sa == (4, 1)


def test_incremental_sort_benchmark_horizon():
    """c4 over the bench's whole 500-substep horizon, where ~1,800 of ~2,800 blocks are dirty
    per substep late on (tools/dirty_probe.py): the same bits as the full sort."""
    spec = spec_for("c4")
    wa, oa, sa, sta = _forward(spec, 500, True)
    wb, ob, sb, stb = _forward(spec, 500, False)
    _check_same(oa, ob, wa)
    for a, b in zip(sta, stb):
        assert np.array_equal(a, b)
    assert sa == (500, 1) and sb == (0, 501)
