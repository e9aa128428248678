"""Measured parity errors of the CUDA path against every long-horizon reference fixture
(tests/golden/long, made by tests/golden/make_golden_long.py), as JSON lines:
    python tools/parity_report.py [case ...] > profiles/r02_parity.jsonl
Scales as SURVEY.md 8(c): x/dx, v/max|v|, F/max|F|, C/max|C| on the fixture's id sample;
loss relative; grad = GradReport::rel_error."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from tests import _long  # noqa: E402
from tests.golden.make_golden_long import CASES  # noqa: E402

for name in sys.argv[1:] or CASES:
    if name == "elastic512" or not _long.available(name):
        continue
    t0 = time.time()
    e = _long.run_case(name)
    e.pop("action_grad", None)
    e["case"] = name
    e["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(e), flush=True)
