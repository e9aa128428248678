"""Throughput on every BASELINE config (SURVEY.md Appendix A scenes c1-c5, full size):
forward (mpm_substep chain) and forward+backward (grad_trajectory over one segment,
stride = segment).  python tools/config_sweep.py [T] [scenes...]"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_02346_b200 as fl  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 50
names = sys.argv[2:] or ["c1", "c2", "c3", "c4", "c5"]
print(f"| config | particles | grid | fwd p-s/s | fwd+bwd p-s/s | fwd ms/substep | fwd+bwd ms/substep |")
print("|---|---|---|---|---|---|---|")
for name in names:
    spec = scenes.load(name)
    w = fl.build_scene(spec)
    ws = fl.GpuWorkspace(w.scene)
    n = int(np.sum(w.scene.activation_substep <= 0))
    acts = fl.ActionTrajectory(1, T, w.init_action.reshape(1, 6))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    g = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)  # warm-up
    best = 1e30
    for _ in range(3):
        g = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
        best = min(best, g.forward_ms + g.backward_ms)
    st = w.state.copy()
    fl.mpm_substep(w.scene, st, w.init_action, ws, count=T)  # warm-up
    ws.lib.flume_sync(ws.ctx)
    fbest = 1e30
    for _ in range(3):
        st = w.state.copy()
        ws._upload(st)
        ws.lib.flume_sync(ws.ctx)
        t0 = time.perf_counter()
        fl.mpm_substep(w.scene, st, w.init_action, ws, count=T)
        ws.lib.flume_sync(ws.ctx)
        fbest = min(fbest, (time.perf_counter() - t0) * 1e3)
    res = w.scene.grid_resolution
    print(f"| {name} | {n} | {res}^3 | {n * T / (fbest / 1e3):.3e} | {n * T / (best / 1e3):.3e} | "
          f"{fbest / T:.3f} | {best / T:.3f} |", flush=True)
    ws.close()
    del w, ws
