"""Population throughput: R candidate rollouts of one scene -- one after
another on one context, on a pool of concurrent contexts, and in one replica context
(every launch covering all R) -- and R gradients (grad_trajectory, one after another vs one
replica context).  Prints one JSON line per R with candidates/s and particle-substeps/s of
each mode (wall clock around synchronous calls, after a warm-up)."""
import json
import sys
import time

import numpy as np

import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import scenes

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
Rs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8,16").split(",")]
w = fl.build_scene(scenes.load(name))
nseg, seglen = 4, 25
rng = np.random.default_rng(0)
loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)


def pop(R):
    return [fl.ActionTrajectory(nseg, seglen, np.tile(w.init_action, (nseg, 1)) + 0.2 * rng.standard_normal((nseg, 6)))
            for _ in range(R)]


def timed(fn, reps=3):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


ws = fl.GpuWorkspace(w.scene)
pool = fl.WorkspacePool(w.scene, 4)
n = w.scene.n_particles
for R in Rs:
    P = pop(R)
    seq = timed(lambda: [fl.rollout_loss(w.scene, w.state, a, loss, ws=ws) for a in P])
    pl = timed(lambda: fl.rollout_loss_batch(w.scene, w.state, P, loss, pool))
    rws = fl.ReplicaWorkspace(w.scene, R)
    rep = timed(lambda: fl.rollout_loss_replicas(w.scene, w.state, P, loss, rws))
    gseq = timed(lambda: [fl.grad_trajectory(w.scene, w.state, a, loss, ws=ws) for a in P], reps=2)
    grep_ = timed(lambda: fl.grad_trajectory_replicas(w.scene, w.state, P, loss, rws), reps=2)
    rws.close()
    ps = R * n * nseg * seglen
    print(json.dumps({"scene": name, "replicas": R, "particles": n, "horizon": nseg * seglen,
                      "sequential_s": seq, "pool4_s": pl, "replica_s": rep,
                      "candidates_per_s": {"sequential": R / seq, "pool4": R / pl, "replica": R / rep},
                      "particle_substeps_per_s": {"sequential": ps / seq, "pool4": ps / pl, "replica": ps / rep},
                      "grad_s": {"sequential": gseq, "replica": grep_},
                      "grad_candidates_per_s": {"sequential": R / gseq, "replica": R / grep_}}),
          flush=True)
