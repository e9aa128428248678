"""Where does full-resolution c5 (256^3, dt 1e-4) stop being a valid simulation?

The jelly (mu 416.67, lambda 277.78, rho 0.5) has a P-wave speed sqrt((lambda + 2 mu)/rho)
= 47 m/s, i.e. 0.6 cells per substep at 128^3 but 1.2 at 256^3 -- beyond the explicit
stability limit, so its deformation grows until det(F) <= 0 and corotated_stress throws
DegenerateDeformation (materials.hpp:20-32), in the reference as on the device.
Runs the scene (or one body of it alone) on the GPU in chunks and prints the first substep
that raises, with the particle's body/material.

    python tools/c5_stability.py [--body jelly] [--res 256] [--max 500] [--chunk 10]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2303_02346_b200 as fl  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402


def spec_for(body=None, res=256, pool=True):
    spec = scenes.load("c5")
    spec["grid_resolution"] = res
    if body:
        keep = (body, "pool") if pool else (body,)
        spec["bodies"] = [b for b in spec["bodies"] if b["name"] in keep]
        if not pool:
            spec["loss"]["body"] = body
    return spec


def run(spec, max_sub, chunk):
    w = fl.build_scene(spec)
    ws = fl.GpuWorkspace(w.scene)
    st = w.state.copy()
    t = 0
    out = {"particles": w.scene.n_particles, "res": spec["grid_resolution"]}
    try:
        while t < max_sub:
            fl.mpm_substep(w.scene, st, w.init_action, ws, count=chunk)
            t += chunk
            f = st.F.reshape(-1, 9)
            det = np.linalg.det(st.F.reshape(-1, 3, 3))
            out.setdefault("trace", []).append([t, float(det.min()), float(np.abs(st.v).max())])
    except fl.EngineError as e:
        pid = getattr(e, "particle_id", -1)
        out["error"] = str(e)
        out["failed_in_chunk_ending"] = t + chunk
        if pid >= 0:
            out["particle"] = int(pid)
            out["body"] = int(w.scene.body_id[pid]) if hasattr(w.scene, "body_id") else None
    finally:
        ws.close()
    out["substeps_ok"] = t
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--body")
    ap.add_argument("--res", type=int, default=256)
    ap.add_argument("--max", type=int, default=500)
    ap.add_argument("--chunk", type=int, default=10)
    ap.add_argument("--no-pool", action="store_true")
    a = ap.parse_args()
    print(json.dumps(run(spec_for(a.body, a.res, not a.no_pool), a.max, a.chunk)))
