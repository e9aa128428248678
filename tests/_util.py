"""Shared helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import scenes


def spec_for(name: str, res: int | None = None) -> dict:
    return scenes.load(name) if res is None else scenes.scaled(name, res)


def pair(spec):
    """(World on the CUDA path, RefWorld on the reference) from the same scene JSON."""
    from oracle.ref import RefWorld
    w = fl.build_scene(spec)
    r = RefWorld(spec)
    return w, r


def rel_err(a, b, scale=None):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    s = np.max(np.abs(b)) if scale is None else scale
    return float(np.max(np.abs(a - b)) / max(s, 1e-30))


def state_errors(st: fl.SimState, rs: dict, dx: float):
    """max |dx|/dx, |dv|/max|v|, |dF|/max|F|, |dC|/max|C| (SURVEY.md 8(c) tolerance scales)."""
    return {
        "x": float(np.max(np.abs(st.x - rs["x"])) / dx),
        "v": rel_err(st.v, rs["v"]),
        "F": rel_err(st.F, rs["F"]),
        "C": rel_err(st.C, rs["C"]),
    }


def grad_rel_error(g, fd):
    """GradReport::rel_error (grad.hpp:162-169)."""
    g = np.asarray(g).ravel()
    fd = np.asarray(fd).ravel()
    return float(np.max(np.abs(g - fd)) / (np.max(np.abs(fd)) + 1e-12))


def canonical_keys_cpu(x32: np.ndarray, dx: float, nd, nbtot_dims):
    """CPU recomputation of the canonical cell key from fp32 positions
    (fl_layout.cuh: base = floor(x*inv_dx - 0.5) in fp32, block-major packing)."""
    inv_dx = np.float32(1.0 / dx)
    xs = (x32.astype(np.float32) * inv_dx).astype(np.float32)
    b = np.floor((xs - np.float32(0.5)).astype(np.float32)).astype(np.int64)
    NB = nbtot_dims
    blk = ((b[0] >> 2) * NB[1] + (b[1] >> 2)) * NB[2] + (b[2] >> 2)
    key = (blk << 6) | ((b[0] & 3) << 4) | ((b[1] & 3) << 2) | (b[2] & 3)
    return key.astype(np.uint64)
