"""CPU tests of the drop-in boundary: the C-ABI library loads and exports every
symbol include/flume_b200.h declares, the ctypes mirror matches, and the
host-side scene builder reproduces the reference's build_scene<3>
(scene.hpp:161-408) bit-exactly.  No compute calls (no GPU here)."""
import ctypes as C
import json
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import _abi, scenes

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "flume_b200.h"
GOLD = np.load(ROOT / "tests" / "golden" / "golden.npz")
META = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())


def header_functions():
    txt = HEADER.read_text()
    return set(re.findall(r"^\s*(?:int|const char\*)\s+(flume_\w+)\s*\(", txt, flags=re.M))


def test_library_loads_and_abi_version():
    lib = _abi.load()
    assert lib.flume_abi_version() == 3


def test_every_declared_symbol_is_exported():
    declared = header_functions()
    assert len(declared) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(flume_\w+)", out))
    missing = declared - exported
    assert not missing, missing
    # the ctypes mirror covers the whole header
    assert declared <= set(_abi.EXPORTS) | set(_abi.EXTRA)


def test_ctypes_struct_sizes_match_c():
    """Compile a probe against the header and compare struct sizes with ctypes."""
    probe = ROOT / "paper_2303_02346_b200" / "_build" / "sizes_probe"
    src = probe.with_suffix(".c")
    src.parent.mkdir(exist_ok=True)
    names = ["flume_config", "flume_material", "flume_effector_shape", "flume_effector_state", "flume_rigid_body",
             "flume_emitter", "flume_scene_desc", "flume_state_view", "flume_loss_term", "flume_loss_desc",
             "flume_actions", "flume_error_info", "flume_timing"]
    src.write_text('#include <stdio.h>\n#include "flume_b200.h"\nint main(){' +
                   "".join(f'printf("%zu\\n", sizeof({n}));' for n in names) + "return 0;}\n")
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(probe)], check=True)
    sizes = [int(s) for s in subprocess.run([str(probe)], capture_output=True, text=True).stdout.split()]
    py = [_abi.Config, _abi.Material, _abi.EffectorShape, _abi.EffectorState, _abi.RigidBody, _abi.Emitter,
          _abi.SceneDesc, _abi.StateView, _abi.LossTerm, _abi.LossDesc, _abi.Actions, _abi.ErrorInfo, _abi.Timing]
    assert sizes == [C.sizeof(t) for t in py]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_scene_builder_matches_reference_bit_exact(name):
    """Jittered lattice sampling, exclusion, emitters and rigid rest shapes: identical bits
    to the reference's build_scene<3> output stored in the golden fixtures."""
    w = fl.build_scene(scenes.scaled(name, META["res"]))
    assert w.scene.n_particles == META["scenes"][name]["particles"]
    assert np.array_equal(w.state.x, GOLD[f"{name}_x0"])
    assert np.array_equal(w.state.v, GOLD[f"{name}_v0"])


def test_scene_builder_full_resolution_against_reference(ref_available):
    from oracle.ref import RefWorld
    spec = scenes.load("c4")
    w = fl.build_scene(spec)
    r = RefWorld(spec).state()
    assert np.array_equal(w.state.x, r["x"]) and np.array_equal(w.scene.mass, r["mass"])
    assert np.array_equal(w.scene.body_id, r["body"]) and np.array_equal(w.scene.material_id, r["material"])


def test_rigid_and_emitter_tables_match_reference(ref_available):
    from oracle.ref import RefWorld
    for name in ("c2", "c5"):
        spec = scenes.scaled(name, 32)
        w = fl.build_scene(spec)
        rw = RefWorld(spec)
        d = w.scene.desc
        rb = rw.rigid_bodies()
        assert d.n_rigid == len(rb)
        for i, b in enumerate(rb):
            r = d.rigid[i]
            mem = np.ctypeslib.as_array(r.members, (r.n_members,))
            rest = np.ctypeslib.as_array(r.rest_offsets, (r.n_members * 3,)).reshape(-1, 3)
            assert np.array_equal(mem, b["members"]) and np.array_equal(rest, b["rest"])
            assert r.total_mass == b["total_mass"]
        em = rw.emitters()
        assert d.n_emitters == len(em["particle"])
        for k in range(d.n_emitters):
            e = d.emitters[k]
            assert e.particle == em["particle"][k] and e.effector == em["effector"][k]
            assert list(e.local_pos) == list(em["local_pos"][k]) and list(e.local_vel) == list(em["local_vel"][k])
        assert np.array_equal(w.scene.activation_substep, rw.state()["act"])


@pytest.mark.parametrize("patch,msg", [
    ({"materials": [{"name": "w", "kind": "liquid", "mu": 1.0, "lambda": 1.0}]}, "liquid requires mu = 0"),
    ({"materials": [{"name": "w", "kind": "slime"}]}, "unknown material kind"),
    ({"grid_resolution": 2}, "grid_resolution too small"),
])
def test_scene_errors_like_reference(patch, msg):
    spec = scenes.scaled("c1", 16)
    spec.update(patch)
    with pytest.raises(fl.SceneError, match=msg):
        fl.build_scene(spec)


def test_canonical_key_cpu_rule():
    """The documented key rule (fl_layout.cuh) on hand-picked positions."""
    from tests._util import canonical_keys_cpu
    dx = 1.0 / 16
    nd = (17, 17, 17)
    NB = (5, 5, 5)
    x = np.array([[dx, dx, dx], [8 * dx, 8.6 * dx, 3.2 * dx]], dtype=np.float32).T
    k = canonical_keys_cpu(x, dx, nd, NB)
    base0 = (0, 0, 0)
    assert k[0] == ((0 * NB[1] + 0) * NB[2] + 0) << 6 | 0
    b = (7, 8, 2)  # floor(x/dx - 0.5)
    assert k[1] == (((b[0] >> 2) * NB[1] + (b[1] >> 2)) * NB[2] + (b[2] >> 2)) << 6 | (b[0] & 3) << 4 | (
        b[1] & 3) << 2 | (b[2] & 3)
    del base0
