"""The five 3D benchmark scenes of BASELINE.json, in the
reference's own scene-JSON schema (proj/include/flume/scene.hpp:161-408)."""
from __future__ import annotations

import json
from pathlib import Path

_DIR = Path(__file__).resolve().parent / "scenes_json"

NAMES = {
    "c1": "c1_dam_break",
    "c2": "c2_latte_art",
    "c3": "c3_ice_cream",
    "c4": "c4_scooping",
    "c5": "c5_multi_material",
}


def load(name: str) -> dict:
    """Scene spec by short name ("c1".."c5") or file stem."""
    stem = NAMES.get(name, name)
    return json.loads((_DIR / f"{stem}.json").read_text())


def text(name: str) -> str:
    return json.dumps(load(name))


def scaled(name: str, resolution: int) -> dict:
    """Same scene on a coarser grid (fewer particles) for fast parity tests."""
    spec = load(name)
    spec["grid_resolution"] = resolution
    return spec
