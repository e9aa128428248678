import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2303_02346_b200 as fl
from tests._util import spec_for
spec = spec_for("c1", 32)
def mk():
    w = fl.build_scene(spec); v = w.state.v; v[:, 0] = 100.0; w.state.v = v; return w
ref = mk(); ws1 = fl.GpuWorkspace(ref.scene)
acts = fl.ActionTrajectory(2, 4, np.tile(ref.init_action, (2, 1)))
g1 = fl.grad_trajectory(ref.scene, ref.state, acts, fl.LossEvaluator(ref.scene, ref.loss_spec, ref.state), stride=2, ws=ws1)
for cap in (100000, 2):
    for ranks in (2, 3):
        w = mk(); ws = fl.GpuWorkspace(w.scene, ranks=ranks); ws._upload(w.state); ws.set_migration_capacity(cap)
        g = fl.grad_trajectory(w.scene, w.state, acts, fl.LossEvaluator(w.scene, w.loss_spec, w.state), stride=2, ws=ws)
        d = np.max(np.abs(np.asarray(g.action_grad) - np.asarray(g1.action_grad))) / np.max(np.abs(g1.action_grad))
        print("cap", cap, "ranks", ranks, "stats", ws.migration_stats()[0], "loss", abs(g.loss - g1.loss) / abs(g1.loss), "grad", d, flush=True)
        ws.close()
