"""Throughput of a population of independent rollouts (CMA-ES style) on one GPU:
one context in turn vs a WorkspacePool (python tools/population_probe.py [scene] [res])."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_02346_b200 as fl  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
res = int(sys.argv[2]) if len(sys.argv) > 2 else 0
spec = scenes.scaled(name, res) if res else scenes.load(name)
w = fl.build_scene(spec)
rng = np.random.default_rng(0)
P, T = 16, 50
pop = [fl.ActionTrajectory(1, T, w.init_action.reshape(1, 6) + 0.1 * rng.standard_normal((1, 6))) for _ in range(P)]
loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
ws = fl.GpuWorkspace(w.scene)
fl.grad_trajectory(w.scene, w.state, pop[0], loss, ws=ws)
t0 = time.perf_counter()
for a in pop:
    fl.grad_trajectory(w.scene, w.state, a, loss, ws=ws)
seq = time.perf_counter() - t0
print(f"{name}{'@' + str(res) if res else ''} N={w.scene.n_particles} population {P} x grad_trajectory(T={T}): "
      f"sequential {seq * 1e3:.1f} ms ({w.scene.n_particles * T * P / seq:.3e} p-s/s)", flush=True)
for k in (2, 4, 8):
    pool = fl.WorkspacePool(w.scene, k)
    fl.grad_trajectory_batch(w.scene, w.state, pop[:k], loss, pool)
    t0 = time.perf_counter()
    fl.grad_trajectory_batch(w.scene, w.state, pop, loss, pool)
    dt = time.perf_counter() - t0
    print(f"  pool of {k}: {dt * 1e3:.1f} ms ({w.scene.n_particles * T * P / dt:.3e} p-s/s, x{seq / dt:.2f})",
          flush=True)
    pool.close()
