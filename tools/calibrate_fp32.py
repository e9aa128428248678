"""Conditioning of a scene over a horizon (SURVEY.md 8(c) "achievable-tolerance calibration"):
round only the initial state to fp32, run the unmodified fp64 reference (oracle/_ref) for the
fixture's substeps, and report the deviation from the fixture in the units of tests/_long.py.
The GPU's error budget at that horizon is set against this number (tests/golden/long/calib.json).

    python tools/calibrate_fp32.py c3_fwd100 [c5_64_10x50 ...]
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from tests import _long  # noqa: E402


def calibrate(name):
    G, meta = _long.load(name)
    spec = _long.spec_of(name)
    rw = ref.RefWorld(spec)
    s = rw.state()
    rw.set_state(x=s["x"].astype(np.float32).astype(np.float64), v=s["v"].astype(np.float32).astype(np.float64),
                 F=s["F"].astype(np.float32).astype(np.float64), C_=s["C"].astype(np.float32).astype(np.float64))
    rw.substep(np.array(meta["action"]), meta["state_substeps"])
    st = rw.state()
    ids = G["ids"]
    dx = 1.0 / spec["grid_resolution"] * spec["domain"][0]
    out = {"substeps": meta["state_substeps"],
           "x": float(np.abs(st["x"][ids] - G["s_x"]).max() / dx),
           "v": float(np.abs(st["v"][ids] - G["s_v"]).max() / float(G["s_vmax"])),
           "F": float(np.abs(st["F"][ids] - G["s_F"]).max() / np.abs(G["s_F"]).max()),
           "C": float(np.abs(st["C"][ids] - G["s_C"]).max() / float(G["s_Cmax"]))}
    return out


if __name__ == "__main__":
    path = _long.LONG / "calib.json"
    res = json.loads(path.read_text()) if path.exists() else {}
    for n in sys.argv[1:]:
        res[n] = calibrate(n)
        print(n, res[n], flush=True)
        path.write_text(json.dumps(res, indent=1))
