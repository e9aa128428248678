"""Per-material parity breakdown of the CUDA path vs the reference (diagnostic)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2303_02346_b200 as fl  # noqa: E402
from tests._util import pair, spec_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
res = int(sys.argv[2]) if len(sys.argv) > 2 else 64
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
w, r = pair(spec_for(name, res))
ws = fl.GpuWorkspace(w.scene)
for k in [1, steps]:
    pass
fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=steps)
r.substep(w.init_action, steps)
rs = r.state()
mat = w.scene.material_id
kinds = ["elastic", "plastic", "liquid", "viscous", "non_newtonian", "rigid"]
vmax = np.abs(rs["v"]).max()
print(f"{name}@{res} after {steps}: max|v| {vmax:.3e}")
for m in np.unique(mat):
    sel = mat == m
    kind = kinds[int(w.scene.materials[m].kind)]
    dv = np.abs(w.state.v[sel] - rs["v"][sel]).max()
    dx = np.abs(w.state.x[sel] - rs["x"][sel]).max() / w.scene.dx
    dF = np.abs(w.state.F[sel] - rs["F"][sel]).max()
    i = np.argmax(np.abs(w.state.v[sel] - rs["v"][sel]).max(axis=1))
    print(f"  mat {m} {kind:14s} n={sel.sum():7d} dv={dv:.3e} ({dv / vmax:.2e} rel) dx={dx:.2e} dF={dF:.2e} "
          f"|v| there={np.abs(rs['v'][sel][i]).max():.3e}")
