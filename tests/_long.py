"""Long-horizon parity cases against tests/golden/long/*.npz (test infrastructure).

Each fixture was produced by the unmodified reference engine (tests/golden/make_golden_long.py).
`run_case(name)` runs the same workload through the CUDA path and returns the measured errors:
  loss      |L_gpu - L_ref| / |L_ref|
  grad      GradReport::rel_error (grad.hpp:162-169): max|g - g_ref| / max|g_ref|
  x v F C   state after `state_substeps` on the fixture's id sample, scaled as SURVEY.md 8(c):
            x / dx, v / max|v_ref|, F / max|F_ref|, C / max|C_ref| (maxima over the whole state)
tools/parity_report.py prints the same numbers into profiles/.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import scenes

LONG = Path(__file__).resolve().parent / "golden" / "long"


def elastic512_actions() -> np.ndarray:
    """acceptance_main.cpp:71-100: 8 x 64 substeps, actions on segments 0 and 3."""
    vals = np.zeros((8, 6))
    vals[0] = [0.3, 0.1, 0, 0, 0, 0]
    vals[3] = [-0.2, 0.25, 0, 0, 0, 0]
    return vals


def spec_of(name: str) -> dict:
    if name in ("c1_4x25",):
        return scenes.load("c1")
    if name in ("c4_10x50", "c4_fwd500"):
        return scenes.load("c4")
    if name == "c4pool_2x25":
        spec = scenes.load("c4")
        spec["loss"] = {"kind": "target_point", "body": "pool", "goal": [0.3, 0.35, 0.5]}
        return spec
    if name == "c3_fwd100":
        return scenes.load("c3")
    if name == "c2_fwd100":
        return scenes.load("c2")
    if name == "c5_2x10":
        return scenes.load("c5")
    if name.endswith("_64_10x50"):
        return scenes.scaled(name[:2], 64)
    raise KeyError(name)


def available(name: str) -> bool:
    return (LONG / f"{name}.npz").exists()


def load(name: str):
    return np.load(LONG / f"{name}.npz"), json.loads((LONG / f"{name}.json").read_text())


def run_case(name: str, stride: int | None = None) -> dict:
    G, meta = load(name)
    spec = spec_of(name)
    w = fl.build_scene(spec)
    ws = fl.GpuWorkspace(w.scene)
    act = np.array(meta["action"])
    out = {"particles": w.scene.n_particles}
    try:
        if meta.get("state_substeps"):
            st = w.state.copy()
            fl.mpm_substep(w.scene, st, act, ws, count=meta["state_substeps"])
            ids = G["ids"]
            vmax = float(G["s_vmax"])
            cmax = float(G["s_Cmax"])
            out["x"] = float(np.abs(st.x[ids] - G["s_x"]).max() / w.scene.dx)
            out["v"] = float(np.abs(st.v[ids] - G["s_v"]).max() / vmax)
            out["F"] = float(np.abs(st.F[ids] - G["s_F"]).max() / max(np.abs(G["s_F"]).max(), 1e-30))
            out["C"] = float(np.abs(st.C[ids] - G["s_C"]).max() / cmax)
            act_mask = w.scene.activation_substep <= st.substep_index
            m = w.scene.mass * act_mask
            cen = (m[:, None] * st.x).sum(0) / m.sum()
            out["centroid"] = float(np.abs(cen - G["s_centroid"]).max() / w.scene.dx)
        if meta.get("segments"):
            acts = fl.ActionTrajectory(meta["segments"], meta["segment_length"], np.tile(act, (meta["segments"], 1)))
            loss = fl.LossEvaluator(w.scene, w.loss_spec, w.state)
            tg = fl.grad_trajectory(w.scene, w.state, acts, loss, stride=meta["stride"] if stride is None else stride,
                                    ws=ws)
            gl = float(G["loss"])
            out["loss"] = abs(tg.loss - gl) / abs(gl)
            g, gr = np.asarray(tg.action_grad).ravel(), np.asarray(G["grad"]).ravel()
            out["grad"] = float(np.max(np.abs(g - gr)) / (np.max(np.abs(gr)) + 1e-12))
            out["grad_scale"] = float(np.max(np.abs(gr)))
            out["per_segment"] = float(np.max(np.abs(np.asarray(tg.per_segment) - G["per_segment"]) /
                                              np.abs(G["per_segment"])))
            out["snapshots"] = [tg.snapshots, meta["snapshots"]]
            out["action_grad"] = np.asarray(tg.action_grad).tolist()
    finally:
        ws.close()
    return out
