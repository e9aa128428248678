"""Is a scene launch-bound?  Compares, for a forward chain and a grad_trajectory,
the wall time per substep, the device time per substep (events around the call)
and the summed kernel time per substep (flume_profile).
usage: python tools/host_bound_probe.py [scene] [res]"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_02346_b200 as fl  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
res = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = fl.build_scene(scenes.load(name) if res is None else scenes.scaled(name, res))
ws = fl.GpuWorkspace(w.scene)
lib, ctx = ws.lib, ws.ctx
T = 50
acts = fl.ActionTrajectory(1, T, w.init_action.reshape(1, 6))
loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
a = np.ascontiguousarray(w.init_action, dtype=np.float64)
ap = a.ctypes.data_as(C.POINTER(C.c_double))


def kernel_sum(fn):
    lib.flume_profile(ctx, 1)
    fn()
    lib.flume_sync(ctx)
    kms = (C.c_double * 9)()
    kc = (C.c_long * 9)()
    lib.flume_kernel_times(ctx, kms, kc, 9)
    lib.flume_profile(ctx, 0)
    return sum(kms), sum(kc)


def fwd():
    lib.flume_substep(ctx, ap, T)


def fb():
    fl.grad_trajectory(w.scene, w.state, acts, loss, ws=ws)


ws._upload(w.state)
for label, fn in (("forward", fwd), ("fwd+bwd", fb)):
    fn()
    lib.flume_sync(ctx)
    best_wall, best_dev = 1e9, 1e9
    for _ in range(5):
        lib.flume_timer_mark(ctx, 0)
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        lib.flume_timer_mark(ctx, 1)
        lib.flume_sync(ctx)
        t2 = time.perf_counter()
        ms = C.c_double()
        lib.flume_timer_elapsed(ctx, 0, 1, C.byref(ms))
        best_wall = min(best_wall, t2 - t0)
        best_dev = min(best_dev, ms.value)
        enq = t1 - t0
    ksum, kcount = kernel_sum(fn)
    print(f"{name}{'' if res is None else '@%d' % res} N={w.scene.n_particles} {label}: wall {1e6 * best_wall / T:.1f} "
          f"us/substep, enqueue-return {1e6 * enq / T:.1f}, device {1e3 * best_dev / T:.1f}, "
          f"kernels {1e3 * ksum / T:.1f} ({kcount / T:.1f} timed launches/substep)", flush=True)

# device-only rate: hold the stream with a sleep kernel so the host finishes enqueueing
# the whole chain before the GPU starts it; (wall - sleep) / T is then the device time
# per substep without host starvation
import torch  # noqa: E402

sp = C.c_void_p()
lib.flume_get_stream(ctx, C.byref(sp))
xs = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", 0))
cyc = int(1.9e9 * 0.2)  # ~200 ms at ~1.9 GHz
for label, fn in (("forward", fwd), ("fwd+bwd", fb)):
    with torch.cuda.stream(xs):
        torch.cuda._sleep(cyc)
    lib.flume_timer_mark(ctx, 2)
    torch.cuda.synchronize()
    with torch.cuda.stream(xs):
        torch.cuda._sleep(cyc)
    lib.flume_timer_mark(ctx, 0)
    fn()
    lib.flume_timer_mark(ctx, 1)
    lib.flume_sync(ctx)
    ms = C.c_double()
    lib.flume_timer_elapsed(ctx, 0, 1, C.byref(ms))
    print(f"  {label}: device-only {1e3 * ms.value / T:.1f} us/substep (stream pre-blocked)", flush=True)
