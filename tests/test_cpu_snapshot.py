"""Versioned state snapshots in the reference's JSON format (io.hpp:144-240):
the snapshot this package writes equals the reference's own dump of the same
state, and each side loads the other's."""
import numpy as np

import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import scenes


def _same(a, b):
    assert a["version"] == b["version"] == 1 and a["dim"] == b["dim"] == 3
    assert a["time"] == b["time"] and a["substep_index"] == b["substep_index"]
    assert len(a["particles"]) == len(b["particles"])
    for pa, pb in zip(a["particles"], b["particles"]):
        assert pa == pb
    assert a["effectors"] == b["effectors"]


def test_snapshot_matches_reference_dump(ref_available):
    from oracle.ref import RefWorld
    spec = scenes.scaled("c2", 16)  # emitters (activation), two liquids, an effector
    w = fl.build_scene(spec)
    _same(fl.state_to_json(w.scene, w.state), RefWorld(spec).snapshot_dump())


def test_snapshot_roundtrip_both_ways(ref_available):
    from oracle.ref import RefWorld
    spec = scenes.scaled("c5", 16)
    w = fl.build_scene(spec)
    r = RefWorld(spec)
    rng = np.random.default_rng(2)
    snap = fl.state_to_json(w.scene, w.state)
    for p in snap["particles"]:  # perturb: a state that is not the scene's initial one
        p["v"] = (np.asarray(p["v"]) + rng.standard_normal(3) * 0.1).tolist()
    snap["time"], snap["substep_index"] = 0.25, 2500
    r.snapshot_load(snap)                     # reference reads ours
    back = r.snapshot_dump()
    _same(snap, back)
    w2 = fl.build_scene(spec)
    fl.state_from_json(back, w2.scene, w2.state)  # we read the reference's
    _same(fl.state_to_json(w2.scene, w2.state), back)
