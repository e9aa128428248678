"""The C++ drop-in adapter (include/flume/gpu.hpp) used from a program written
against the reference's own API (tests/cpp/shim_parity.cpp, built by
tests/cpp/Makefile against proj/include): flume::mpm_substep vs
flume::gpu::mpm_substep and the two grad_trajectory calls agree, and a two-candidate population
in a replica context (gpu::Workspace(..., gpu::Replicas{2}), gpu::rollout_loss_replicas) gives
the single-context losses."""
import json
import subprocess
from pathlib import Path

import pytest

from paper_2303_02346_b200 import scenes

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "shim_parity"


@pytest.mark.parametrize("name,res", [("c4", 32), ("c5", 32)])
def test_cpp_adapter_parity(tmp_path, name, res):
    if not BIN.exists():
        pytest.skip("tests/cpp/_build/shim_parity not built (make -C tests/cpp)")
    spec = tmp_path / "scene.json"
    spec.write_text(json.dumps(scenes.scaled(name, res)))
    r = subprocess.run([str(BIN), str(spec), "5"], capture_output=True, text=True, timeout=600)
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0 and line["ok"], (line, r.stderr[-2000:])
