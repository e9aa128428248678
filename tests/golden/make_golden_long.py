"""Long-horizon golden fixtures from the unmodified reference engine (test infrastructure).

The round-1 fixtures (make_golden.py) stop at 3-substep states and 2x3-substep gradients.
These pin the CUDA path at the benchmark horizons of SURVEY.md 8(c)/8(d):

  c1_4x25      full c1 (102,400 particles), 4 segments x 25 substeps, stride 25: loss, per-segment
               losses and action_grad (SURVEY 8(c) quotes loss 2.536990744672e+05 and the 4 rows)
               + the state after 100 forward substeps on a fixed id sample
  c4_10x50     full c4 (1,027,233 particles), the bench workload: 10 x 50 substeps, the scene's
               own target_point loss on the floater (grad.hpp:61-134, stride 25 -- stride never
               changes the reference's result, test_autodiff.cpp:153-178)
  c4pool_2x25  full c4 with a `pool` target_point loss (the body in contact with the ladle's
               soft band), 2 x 25 substeps
  c4_fwd500    full c4 state after the bench's 500 forward substeps (id sample)
  c3_fwd100    full c3 (1,024,000 non-Newtonian particles) state after 100 substeps (id sample)
  c2_fwd100    full c2 (1,057,280 particles: liquid, viscous liquid, emitter) after 100 substeps
  c5_2x10      full c5 (8,044,544 particles, 256^3, every material + the rigid brick): the
               scaling workload -- state after 20 substeps, loss and gradient over 2 x 10
  elastic512   the 3D gradcheck scene (test_autodiff.cpp:113-151) over acceptance_main.cpp:71-100's
               8 x 64 substeps (the stride-invariance criterion's workload)
  c{2,3,5}_64_10x50  the scene at grid 64 (c5: 125,696 particles with every material kind and
               the rigid brick), 10 x 50 substeps: loss + action_grad, and the state after
               100 substeps (id sample)

Each case writes tests/golden/long/<case>.npz + <case>.json.  Run one case per process:
    python tests/golden/make_golden_long.py <case> [<case> ...]
(needs oracle/_ref built from /root/reference; c4_10x50 takes ~30 min on one core).
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = HERE / "long"
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_2303_02346_b200 import scenes  # noqa: E402

N_SAMPLE = 4096


def sample_ids(n: int) -> np.ndarray:
    """Fixed id sample (every particle kind is spread through the id range; seeded, sorted)."""
    rng = np.random.default_rng(12345)
    return np.sort(rng.choice(n, size=min(n, N_SAMPLE), replace=False)).astype(np.int64)


def state_sample(rw, ids):
    s = rw.state()
    out = {k: s[k][ids] for k in ("x", "v", "F", "C")}
    # whole-state summaries (size-independent): mass-weighted centroid and momentum, max |v|
    act = s["act"] <= s["substep"]
    m = s["mass"] * act
    out["centroid"] = (m[:, None] * s["x"]).sum(0) / m.sum()
    out["momentum"] = (m[:, None] * s["v"]).sum(0)
    out["vmax"] = np.array(np.abs(s["v"]).max())
    out["Cmax"] = np.array(np.abs(s["C"]).max())
    return out


def grad_case(spec, n_seg, seglen, stride, substeps_state=None):
    act = np.array(spec["optimizer"]["init"], dtype=np.float64)
    vals = np.tile(act, (n_seg, 1))
    rw = ref.RefWorld(spec)
    arrays, meta = {}, {"particles": int(rw.n), "action": act.tolist(), "segments": n_seg,
                        "segment_length": seglen, "stride": stride}
    if substeps_state:
        ids = sample_ids(rw.n)
        t0 = time.time()
        rw.substep(act, substeps_state)
        arrays.update({f"s_{k}": v for k, v in state_sample(rw, ids).items()})
        arrays["ids"] = ids
        meta["state_substeps"] = substeps_state
        meta["fwd_seconds"] = time.time() - t0
        rw.reset()
    if n_seg:
        t0 = time.time()
        g = rw.grad_trajectory(vals, seglen, stride=stride)
        meta["grad_seconds"] = time.time() - t0
        arrays["loss"] = np.array(g["loss"])
        arrays["full_loss"] = np.array(g["full_loss"])
        arrays["grad"] = g["grad"]
        arrays["per_segment"] = g["per_segment"]
        meta["snapshots"] = g["snapshots"]
    return arrays, meta


def case(name):
    if name == "c1_4x25":
        return grad_case(scenes.load("c1"), 4, 25, 25, substeps_state=100)
    if name == "c4_10x50":
        return grad_case(scenes.load("c4"), 10, 50, 25)
    if name == "c4pool_2x25":
        spec = scenes.load("c4")
        spec["loss"] = {"kind": "target_point", "body": "pool", "goal": [0.3, 0.35, 0.5]}
        return grad_case(spec, 2, 25, 25)
    if name == "c4_fwd500":
        return grad_case(scenes.load("c4"), 0, 0, 0, substeps_state=500)
    if name == "c3_fwd100":
        return grad_case(scenes.load("c3"), 0, 0, 0, substeps_state=100)
    if name == "c2_fwd100":  # full latte art: liquid + viscous liquid, the emitter active
        return grad_case(scenes.load("c2"), 0, 0, 0, substeps_state=100)
    if name == "c5_2x10":  # the scaling workload (8M particles, 256^3), its stable window
        return grad_case(scenes.load("c5"), 2, 10, 10, substeps_state=20)
    if name == "elastic512":
        from tests._long import elastic512_actions
        from tests.golden.make_golden import GRADCHECK_3D
        rw = ref.RefWorld(GRADCHECK_3D)
        g = rw.grad_trajectory(elastic512_actions(), 64, stride=64)
        return ({"loss": np.array(g["loss"]), "grad": g["grad"], "per_segment": g["per_segment"]},
                {"particles": int(rw.n), "segments": 8, "segment_length": 64, "stride": 64,
                 "snapshots": g["snapshots"]})
    if name.endswith("_64_10x50"):
        return grad_case(scenes.scaled(name[:2], 64), 10, 50, 25, substeps_state=100)
    raise SystemExit(f"unknown case {name}")


CASES = ["c1_4x25", "elastic512", "c4_10x50", "c4pool_2x25", "c4_fwd500", "c3_fwd100", "c2_64_10x50", "c3_64_10x50",
         "c5_64_10x50", "c2_fwd100", "c5_2x10"]


def main(argv):
    OUT.mkdir(exist_ok=True)
    for name in argv or CASES:
        t0 = time.time()
        arrays, meta = case(name)
        meta["wall_seconds"] = time.time() - t0
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1))
        print(name, json.dumps(meta), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
