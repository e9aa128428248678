"""The reference side of tools/c5_stability.py: the c5 jelly body (plus the pool, as on the
device) at 256^3 run by the unmodified reference (oracle/_ref) in 10-substep chunks; prints
min det(F), max |v| per chunk and the substep where DegenerateDeformation is raised.
Test infrastructure (imports oracle/)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from tools.c5_stability import spec_for  # noqa: E402


def main(body="jelly", res=256, max_sub=120, chunk=10, pool=True):
    spec = spec_for(body, res, pool)
    rw = ref.RefWorld(spec)
    act = np.array(spec["optimizer"]["init"], dtype=np.float64)
    out = {"particles": int(rw.n), "res": res, "trace": []}
    t = 0
    try:
        while t < max_sub:
            rw.substep(act, chunk)
            t += chunk
            s = rw.state()
            out["trace"].append([t, float(np.linalg.det(s["F"]).min()), float(np.abs(s["v"]).max())])
            print(json.dumps(out["trace"][-1]), flush=True)
    except Exception as e:  # the reference's DegenerateDeformation
        out["error"] = str(e)
        out["failed_in_chunk_ending"] = t + chunk
    out["substeps_ok"] = t
    print(json.dumps(out))


if __name__ == "__main__":
    main(pool="--no-pool" not in sys.argv)
