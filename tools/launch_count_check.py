"""Cross-check of the engine's launch counter (flume_timing.launches, bench.py's
gpu_launches) against the kernels a profiler sees: run under
  ncu --metrics gpu__time_duration.sum --csv --log-file L python tools/launch_count_check.py
and compare the printed count with the number of launches in L after the marker kernel."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_02346_b200 as fl  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402

w = fl.build_scene(scenes.load("c4"))
ws = fl.GpuWorkspace(w.scene)
acts = fl.ActionTrajectory(2, 2, np.tile(w.init_action, (2, 1)))
loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)  # upload + warm-up (not counted)
ws.lib.flume_sync(ws.ctx)
import torch  # noqa: E402
torch.cuda.synchronize()
torch.zeros(1, device="cuda").add_(1)  # marker kernel
torch.cuda.synchronize()
fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
print("engine launches:", ws.last_timing().launches)
