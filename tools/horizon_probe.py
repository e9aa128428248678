"""Per-window kernel times over c4's horizon: how the per-substep cost evolves as the
lattice arrangement of t = 0 disorders (cells above 8 particles need a second staging
pass).  python tools/horizon_probe.py"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_02346_b200 as fl  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402

NAMES = ["p2g", "grid", "g2p", "sort", "adj_g2p", "adj_grid", "adj_p2g", "rigid", "other"]
w = fl.build_scene(scenes.load("c4"))
ws = fl.GpuWorkspace(w.scene)
lib, ctx = ws.lib, ws.ctx
a = np.ascontiguousarray(w.init_action, dtype=np.float64)
ap = a.ctypes.data_as(C.POINTER(C.c_double))
ws._upload(w.state)
t = 0
for t_end in (50, 100, 200, 300, 400, 500):
    lib.flume_profile(ctx, 1)
    lib.flume_substep(ctx, ap, t_end - t)
    lib.flume_sync(ctx)
    kms = (C.c_double * 9)()
    kc = (C.c_long * 9)()
    lib.flume_kernel_times(ctx, kms, kc, 9)
    lib.flume_profile(ctx, 0)
    n = t_end - t
    keys = np.zeros(w.scene.n_particles, np.uint32)
    na = C.c_long()
    lib.flume_store_order(ctx, keys.ctypes.data_as(C.POINTER(C.c_uint)), None, C.byref(na))
    k = keys[:na.value].astype(np.int64)
    cells, cc = np.unique(k, return_counts=True)
    blocks = np.unique(cells >> 6)
    maxc = np.zeros(len(blocks), np.int64)
    np.maximum.at(maxc, np.searchsorted(blocks, cells >> 6), cc)
    print(f"t {t:3d}-{t_end:3d}: " + " ".join(f"{NAMES[i]} {1e3 * kms[i] / max(kc[i], 1):.1f}" for i in range(4)) +
          f" us | blocks {len(blocks)}, 2-pass {int(np.sum(maxc > 8))}, max cell {int(cc.max())}", flush=True)
    t = t_end
