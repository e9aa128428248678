"""x-slabs across processes through the product's own transport.

Each rank runs in its own process (`GpuWorkspace.distributed`, the torchrun entry point of
`bench.py --gpus N`) with the CUDA-IPC transport (`ipc_unique_id`): device inboxes exported
with cudaIpcGetMemHandle, peer copies ordered by interprocess events, a host barrier in
POSIX shared memory.  On a one-GPU box the ranks share the device (no kernel waits on
another process: every wait is a stream-event wait or a host barrier).  Contract as in
tests/test_gpu_slab.py: particle states bit-identical to one rank, losses <= 1e-12 and
action gradients <= 1e-9 relative (the order of the final cross-rank sums).  The fast
blob (100 m/s along x) migrates across the slab faces every few substeps, and the
gradient runs with checkpoint replay (stride 2).
"""
import multiprocessing as mp
import os
from pathlib import Path

import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import spec_for

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _single(spec, fast_x):
    w = fl.build_scene(spec)
    if fast_x:
        v = w.state.v
        v[:, 0] = fast_x
        w.state.v = v
    ws = fl.GpuWorkspace(w.scene)
    fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=12)
    st = [np.array(a, copy=True) for a in (w.state.x, w.state.v, w.state.F, w.state.C)]
    acts = fl.ActionTrajectory(2, 4, np.tile(w.init_action, (2, 1)))
    g = fl.grad_trajectory(w.scene, w.state, acts, fl.LossEvaluator(w.scene, w.loss_spec, w.state), stride=2, ws=ws)
    ws.close()
    return st, g.loss, np.asarray(g.action_grad)


@pytest.mark.parametrize("name,res,fast_x,n", [("c1", 32, 100.0, 2), ("c1", 32, 100.0, 3), ("c5", 32, 0.0, 2)])
def test_processes_over_ipc_transport_match_one_rank(name, res, fast_x, n):
    from tests._mp_worker import run_rank
    spec = spec_for(name, res)
    os.environ["PYTHONPATH"] = str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", "")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = fl.ipc_unique_id()
    procs = [ctx.Process(target=run_rank, args=(r, n, uid, spec, fast_x, q)) for r in range(n)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(n):
            rank, status, *rest = q.get(timeout=300)
            assert status == "ok", (rank, rest[0])
            out[rank] = rest
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    st1, l1, g1 = _single(spec, fast_x)
    cols = sorted(out[r][3][0][1:3] for r in range(n))  # (rank, sx0, sx1, n_active) per process
    assert [out[r][3][0][0] for r in range(n)] == list(range(n))
    assert cols[0][0] == 0 and all(cols[i][1] == cols[i + 1][0] for i in range(n - 1))
    for r in range(n):
        st, l, g, _ = out[r]
        for a, b, f in zip(st1, st, "xvFC"):
            assert np.array_equal(a, b), (r, f, float(np.max(np.abs(a - b))))
        assert abs(l - l1) <= 1e-12 * abs(l1)
        assert np.max(np.abs(g - g1)) <= 1e-9 * np.max(np.abs(g1)), (r, g, g1)
