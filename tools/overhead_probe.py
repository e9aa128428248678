"""Per-substep fixed cost (launch latency, stream/event plumbing) of grad_trajectory:
time a tiny scene whose kernels do almost no work (python tools/overhead_probe.py)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_02346_b200 as fl  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402

for name, res in (("c1", 16), ("c4", 16), ("c4", 32)):
    w = fl.build_scene(scenes.scaled(name, res))
    ws = fl.GpuWorkspace(w.scene)
    T = 50
    acts = fl.ActionTrajectory(1, T, w.init_action.reshape(1, 6))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        g = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
        best = min(best, time.perf_counter() - t0)
    t = ws.last_timing()
    print(f"{name}@{res} N={w.scene.n_particles}: {1e6 * best / T:.1f} us/substep wall "
          f"(fwd {1e3 * g.forward_ms / T:.1f} + bwd {1e3 * g.backward_ms / T:.1f} us device), "
          f"{t.launches / T:.0f} launches/substep", flush=True)
