"""Conditioning probe (test infrastructure, SURVEY.md Appendix B `drift`): run the reference
engine twice on the same scene -- once from the exact fp64 initial state, once with x/v/F/C
rounded to fp32 -- and report how far the two states drift apart after K substeps on the
fixture's id sample, in the SURVEY 8(c) scales (x/dx, v/max|v|, F/max|F|, C/max|C|).  The
reference's own sensitivity to fp32 input rounding is the floor any fp32 device path sits on.

    python tools/drift_probe.py c3 100 [res]
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import ref  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402
from tests.golden.make_golden_long import sample_ids  # noqa: E402

name, K = sys.argv[1], int(sys.argv[2])
spec = scenes.load(name) if len(sys.argv) < 4 else scenes.scaled(name, int(sys.argv[3]))
act = np.array(spec["optimizer"]["init"], dtype=np.float64)
a, b = ref.RefWorld(spec), ref.RefWorld(spec)
s = b.state()
b.set_state(**{k: s[k].astype(np.float32).astype(np.float64) for k in ("x", "v", "F")},
            C_=s["C"].astype(np.float32).astype(np.float64))
a.substep(act, K)
b.substep(act, K)
sa, sb = a.state(), b.state()
ids = sample_ids(a.n)
dx = spec["domain"][0] / spec["grid_resolution"]
out = {"scene": name, "res": spec["grid_resolution"], "substeps": K,
       "x": float(np.abs(sa["x"][ids] - sb["x"][ids]).max() / dx),
       "v": float(np.abs(sa["v"][ids] - sb["v"][ids]).max() / np.abs(sa["v"]).max()),
       "F": float(np.abs(sa["F"][ids] - sb["F"][ids]).max() / np.abs(sa["F"][ids]).max()),
       "C": float(np.abs(sa["C"][ids] - sb["C"][ids]).max() / np.abs(sa["C"]).max()),
       "x_all": float(np.abs(sa["x"] - sb["x"]).max() / dx)}
print(json.dumps(out))
