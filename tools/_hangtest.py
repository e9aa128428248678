import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import scenes
spec = scenes.load("c4")
w = fl.build_scene(spec)
ws = fl.GpuWorkspace(w.scene)
for T in (4, 20, 50):
    acts = fl.ActionTrajectory(1, T, w.init_action.reshape(1, 6))
    loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
    t0 = time.time()
    g = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    print(T, "ok", time.time() - t0, g.loss, flush=True)
for i in range(6):
    t0 = time.time()
    g = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
    print("rep", i, time.time() - t0, flush=True)
