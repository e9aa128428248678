"""Error paths of the device engine map to the reference's exception types with their
context fields (core.hpp:18-48), and a context stays usable after an error:
  * a particle outside the clamped region -> EngineError at P2G (mpm.hpp:265-269,
    test_mpm.cpp:432-437)
  * det(F) <= 0 -> DegenerateDeformation(particle_id) (materials.hpp:20-32)
"""
import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from tests._util import spec_for

pytestmark = pytest.mark.gpu


def test_escape_raises_and_context_recovers():
    w = fl.build_scene(spec_for("c1", 16))
    ws = fl.GpuWorkspace(w.scene)
    good = w.state.copy()
    x = w.state.x
    x[7] = [1.5, 0.5, 0.5]  # outside the domain: its stencil leaves the grid
    w.state.x = x
    with pytest.raises(fl.EngineError, match="escaped"):
        fl.mpm_substep(w.scene, w.state, w.init_action, ws)
    # the same workspace runs a good state afterwards, identically to a fresh one
    fl.mpm_substep(w.scene, good, w.init_action, ws, count=3)
    w2 = fl.build_scene(spec_for("c1", 16))
    ws2 = fl.GpuWorkspace(w2.scene)
    fl.mpm_substep(w2.scene, w2.state, w2.init_action, ws2, count=3)
    assert np.array_equal(good.x, w2.state.x) and np.array_equal(good.F, w2.state.F)


@pytest.mark.parametrize("name,res,material_kind", [("c5", 32, 0), ("c1", 16, 2)])
def test_inverted_F_raises_degenerate_with_particle_id(name, res, material_kind):
    w = fl.build_scene(spec_for(name, res))
    kinds = np.array([w.scene.materials[m].kind for m in w.scene.material_id])
    pid = int(np.nonzero(kinds == material_kind)[0][3])
    F = w.state.F
    F[pid] = np.diag([-1.0, 1.0, 1.0])  # det < 0
    w.state.F = F
    ws = fl.GpuWorkspace(w.scene)
    with pytest.raises(fl.DegenerateDeformation) as ei:
        fl.mpm_substep(w.scene, w.state, w.init_action, ws)
    assert ei.value.particle_id == pid
