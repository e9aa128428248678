"""Generate the golden fixtures in tests/golden/ from the unmodified reference engine.

Runs oracle/_ref/libflume_ref.so (proj/include/flume compiled as-is by
oracle/Makefile) on small versions of the five benchmark scenes and on the 3D
gradient-check scene of proj/tests/test_autodiff.cpp:113-151, and stores the
states / grids / losses / gradients it produces.  Re-run with
    python tests/golden/make_golden.py
(needs /root/reference to build oracle/_ref; the fixtures then travel without it).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402

RES = 16

# proj/tests/test_autodiff.cpp:113-151 (3D rotating box effector), verbatim scene values
GRADCHECK_3D = {
    "dim": 3, "grid_resolution": 16, "domain": [1.0, 1.0, 1.0], "dt_substep": 4e-4, "substeps_per_step": 5,
    "gravity": [0.0, -2.0, 0.0], "seed": 21,
    "materials": [{"name": "stuff", "kind": "elastic", "mu": 208.33, "lambda": 277.78, "rho": 1.0}],
    "bodies": [{"name": "blob", "material": "stuff",
                "shape": {"type": "box", "half_extents": [0.1, 0.08, 0.1], "center": [0.45, 0.3, 0.5]},
                "particles_per_cell_axis": 1, "jitter": 0.2}],
    "loss": {"kind": "target_point", "body": "blob", "goal": [0.6, 0.4, 0.55]},
    "effectors": [{"shape": {"type": "box", "half_extents": [0.07, 0.05, 0.07], "center": [0.0, 0.0, 0.0]},
                   "position": [0.33, 0.42, 0.5], "friction": 0.4,
                   "action_mask": [True, True, True, False, False, True]}],
}
GRADCHECK_3D_ACTIONS = [[0.4, -0.3, 0.2, 0, 0, 0.8], [-0.2, 0.3, -0.1, 0, 0, -0.5]]


def scene_case(name):
    spec = scenes.scaled(name, RES)
    act = np.array(spec["optimizer"]["init"], dtype=np.float64)
    rw = ref.RefWorld(spec)
    s0 = rw.state()
    mass, mom, vel = rw.p2g_grid()
    rw.reset()
    rw.substep(act, 1)
    s1 = rw.state()
    rw.substep(act, 2)
    s3 = rw.state()
    rw.reset()
    g = rw.grad_trajectory(np.tile(act, (2, 1)), 3, stride=2)
    out = {f"{name}_x0": s0["x"], f"{name}_v0": s0["v"],
           f"{name}_grid_mass_sum": np.array(mass.sum()), f"{name}_grid_mom_sum": mom.reshape(-1, 3).sum(0),
           f"{name}_grid_vel": vel}
    for tag, s in (("s1", s1), ("s3", s3)):
        for k in ("x", "v", "F", "C"):
            out[f"{name}_{tag}_{k}"] = s[k]
    out[f"{name}_loss"] = np.array(g["loss"])
    out[f"{name}_grad"] = g["grad"]
    out[f"{name}_per_segment"] = g["per_segment"]
    return out, {"particles": int(rw.n), "action": act.tolist(), "grad_segments": 2, "segment_length": 3,
                 "stride": 2, "snapshots": g["snapshots"]}


def main():
    arrays, meta = {}, {"res": RES, "scenes": {}}
    for name in ("c1", "c2", "c3", "c4", "c5"):
        a, m = scene_case(name)
        arrays.update(a)
        meta["scenes"][name] = m
    rw = ref.RefWorld(GRADCHECK_3D)
    g = rw.grad_trajectory(np.array(GRADCHECK_3D_ACTIONS, dtype=np.float64), 15, stride=10)
    arrays["gradcheck3d_loss"] = np.array(g["loss"])
    arrays["gradcheck3d_grad"] = g["grad"]
    meta["gradcheck3d"] = {"scene": GRADCHECK_3D, "actions": GRADCHECK_3D_ACTIONS, "segment_length": 15,
                           "stride": 10, "snapshots": g["snapshots"]}
    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1))
    print("wrote", HERE / "golden.npz", sum(v.nbytes for v in arrays.values()), "bytes raw")


if __name__ == "__main__":
    main()
