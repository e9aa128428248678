"""A/B of the heavy/light concurrent launches (FL_DUAL_MODE): per-kernel-class device times and
the whole grad_trajectory of a scene over `horizon` substeps (CUDA events)."""
import ctypes as C
import json
import os
import sys

import numpy as np

import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import scenes

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
horizon = int(sys.argv[2]) if len(sys.argv) > 2 else 500
KERNELS = ["p2g", "grid_update", "g2p", "sort", "g2p_adjoint", "grid_adjoint", "p2g_adjoint", "rigid", "other",
           "slab_comm"]
w = fl.build_scene(scenes.load(name))
ws = fl.GpuWorkspace(w.scene)
lib, ctx = ws.lib, ws.ctx
seg = 50 if horizon % 50 == 0 else horizon
acts = fl.ActionTrajectory(horizon // seg, seg, np.tile(w.init_action, (horizon // seg, 1)))
loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
fl.grad_trajectory(w.scene, w.state, acts, loss, stride=horizon, ws=ws)
lib.flume_profile(ctx, 1)
g = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=horizon, ws=ws)
kms = (C.c_double * len(KERNELS))()
kcnt = (C.c_long * len(KERNELS))()
lib.flume_kernel_times(ctx, kms, kcnt, len(KERNELS))
lib.flume_profile(ctx, 0)
t = C.c_double()
lib.flume_sync(ctx)
lib.flume_timer_mark(ctx, 0)
for _ in range(3):
    g2 = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=horizon, ws=ws)
lib.flume_timer_mark(ctx, 1)
lib.flume_timer_elapsed(ctx, 0, 1, C.byref(t))
print(json.dumps({"scene": name, "dual_mode": os.environ.get("FL_DUAL_MODE", "default"), "ms_per_traj": t.value / 3,
                  "loss": g2.loss, "grad0": float(np.asarray(g2.action_grad).ravel()[0]),
                  "us_per_launch": {k: round(kms[i] * 1e3 / max(kcnt[i], 1), 2) for i, k in enumerate(KERNELS)
                                    if kcnt[i]}}))
