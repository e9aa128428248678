"""On-disk frame and metric dumps in the reference's formats (io.hpp:18-130).

These write what the reference's run outputs hold, byte for byte, from a SimState
(pulled from the device if it is resident there):
  write_frame_csv   io.hpp:53-67   active particles, id, body, x, v in %.17g
  MetricsWriter     io.hpp:96-114  substep, time, particle_totals (mpm.hpp:486-496) per row
  actions_to_json / actions_from_json   io.hpp:251-273
"""
from __future__ import annotations

from pathlib import Path

import numpy as np

from .api import ActionTrajectory, EngineError, Scene, SimState


def format_real(v: float) -> str:
    """io.hpp:18-22 (snprintf "%.17g")."""
    return "%.17g" % float(v)


def _write_text(path, text: str) -> None:
    try:
        Path(path).write_bytes(text.encode())
    except OSError as e:
        raise EngineError(f"cannot write {path}") from e


def write_frame_csv(path, scene: Scene, state: SimState, manifest_hash: int) -> None:
    """write_frame_csv<3> (io.hpp:53-67): particles active at the state's substep."""
    state._pull()
    act = np.asarray(scene.activation_substep)
    body = np.asarray(scene.body_id)
    rows = ["# manifest %d\n" % int(manifest_hash), "id,body,x,y,z,vx,vy,vz\n"]
    for i in np.nonzero(act <= state.substep_index)[0]:
        x, v = state._x[i], state._v[i]
        rows.append("%d,%d,%s,%s,%s,%s,%s,%s\n" % (i, body[i], *(format_real(c) for c in x),
                                                   *(format_real(c) for c in v)))
    _write_text(path, "".join(rows))


def particle_totals(scene: Scene, state: SimState):
    """particle_totals<3> (mpm.hpp:486-496): (mass, momentum[3], kinetic energy) of the
    active particles, summed in particle order like the reference's loop."""
    state._pull()
    on = np.asarray(scene.activation_substep) <= state.substep_index
    m = np.asarray(scene.mass, dtype=np.float64)[on]
    v = state._v[on]
    if m.size == 0:
        return 0.0, np.zeros(3), 0.0
    seq = lambda a: float(np.add.accumulate(a)[-1])  # noqa: E731  (sequential, not pairwise)
    nsq = (v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1]) + v[:, 2] * v[:, 2]
    mom = np.array([seq(v[:, a] * m) for a in range(3)])
    return seq(m), mom, seq((0.5 * m) * nsq)


class MetricsWriter:
    """MetricsWriter<3> (io.hpp:96-114)."""

    def __init__(self, path, manifest_hash: int):
        self.path = path
        self.buf = ["# manifest %d\n" % int(manifest_hash), "substep,time,mass,px,py,pz,kinetic_energy\n"]

    def append(self, scene: Scene, state: SimState) -> None:
        mass, mom, ke = particle_totals(scene, state)
        self.buf.append("%d,%s,%s,%s,%s,%s,%s\n" % (state.substep_index, format_real(state.time), format_real(mass),
                                                   *(format_real(c) for c in mom), format_real(ke)))

    def flush(self) -> None:
        _write_text(self.path, "".join(self.buf))


def actions_to_json(a: ActionTrajectory) -> dict:
    """io.hpp:251-263."""
    return {"n_segments": a.n_segments, "segment_length": a.segment_length,
            "values": np.asarray(a.values, dtype=np.float64).reshape(-1, 6).tolist()}


def actions_from_json(j: dict) -> ActionTrajectory:
    """io.hpp:265-273."""
    ns, sl = int(j["n_segments"]), int(j["segment_length"])
    vals = j["values"]
    if len(vals) != ns:
        raise EngineError("trajectory file: segment count mismatch")
    return ActionTrajectory(ns, sl, np.asarray(vals, dtype=np.float64).reshape(ns, 6))
