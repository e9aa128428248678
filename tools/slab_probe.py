"""Cost of the x-slab protocol on ONE device: grad_trajectory of a scene with
1, 2, 4 in-process slab ranks sharing the GPU (python tools/slab_probe.py [scene] [T]).

The ranks split the same work, so on one device the ideal is "same time as one
rank"; the excess is the halo / migration / all-reduce protocol plus the host
synchronisation it adds.  (Multi-GPU numbers come from bench.py --gpus N.)
"""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_02346_b200 as fl  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    spec = scenes.load(name)
    for ranks in (1, 2, 4):
        w = fl.build_scene(spec)
        ws = fl.GpuWorkspace(w.scene, ranks=ranks)
        acts = fl.ActionTrajectory(1, T, w.init_action.reshape(1, 6))
        loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
        g = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)  # warm-up
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            g = fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        # rank 0's kernel classes (CUDA events on its stream; a separate, instrumented run)
        lib = ws.lib
        for c in ws.ctxs:
            lib.flume_profile(c, 1)
        fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)
        kms = (ctypes.c_double * 10)()
        kc = (ctypes.c_long * 10)()
        lib.flume_kernel_times(ws.ctxs[0], kms, kc, 10)
        for c in ws.ctxs:
            lib.flume_profile(c, 0)
        names = ["p2g", "grid", "g2p", "sort", "g2p_adj", "grid_adj", "p2g_adj", "rigid", "other", "comm"]
        print("   rank 0 ms/step: " + " ".join(f"{n} {kms[i]:.2f}" for i, n in enumerate(names)), flush=True)
        print(f"{name} T={T} ranks={ranks}: {1e3 * t:.2f} ms/step wall, fwd {g.forward_ms:.2f} ms + "
              f"bwd {g.backward_ms:.2f} ms (rank 0 device), {w.scene.n_particles * T / t:.3e} p-s/s, "
              f"loss {g.loss:.12e} grad {np.asarray(g.action_grad)[0, :3]} slabs {ws.slab_info()}", flush=True)
        ws.close()


if __name__ == "__main__":
    main()
