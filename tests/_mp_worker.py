"""Worker of tests/test_gpu_multiprocess.py: one slab rank in its own process (test
infrastructure; spawned, so it imports the package fresh)."""
from __future__ import annotations

import numpy as np


def run_rank(rank: int, n: int, uid: bytes, spec: dict, fast_x: float, q) -> None:
    try:
        import paper_2303_02346_b200 as fl
        w = fl.build_scene(spec)
        if fast_x:
            v = w.state.v
            v[:, 0] = fast_x
            w.state.v = v
        ws = fl.GpuWorkspace.distributed(w.scene, 0, rank, n, uid)
        fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=12)
        st = [np.array(a, copy=True) for a in (w.state.x, w.state.v, w.state.F, w.state.C)]
        info = ws.slab_info()
        acts = fl.ActionTrajectory(2, 4, np.tile(w.init_action, (2, 1)))
        loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
        g = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=2, ws=ws)
        q.put((rank, "ok", st, float(g.loss), np.asarray(g.action_grad).copy(), info))
        ws.close()
    except Exception as e:  # reported to the parent, which fails the test
        q.put((rank, "error", repr(e), None, None, None))
