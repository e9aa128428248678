"""Run outputs in the reference's formats (io.hpp:18-130): frame CSV and metrics rows
written by this package are byte-identical to the reference's own writers for the
same state, including the active-particle filter with emitters; action trajectories
round-trip through the reference's JSON layout."""
import numpy as np

import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import frames, scenes


def _ref_state_as_ours(w, r):
    rs = r.state()
    return fl.SimState(rs["x"], rs["v"], rs["F"].reshape(-1, 9), rs["C"].reshape(-1, 9), r.effector_state(),
                       rs["time"], rs["substep"])


def test_frame_csv_and_metrics_match_reference(ref_available, tmp_path):
    from oracle.ref import RefWorld
    spec = scenes.scaled("c2", 16)  # emitters: the active set grows with the substep
    w = fl.build_scene(spec)
    r = RefWorld(spec)
    for k, steps in enumerate([0, 7, 20]):
        if steps:
            r.substep(w.init_action, steps)
        st = _ref_state_as_ours(w, r)
        h = 1234567890123 + k
        frames.write_frame_csv(tmp_path / "ours.csv", w.scene, st, h)
        r.write_frame_csv(tmp_path / "ref.csv", h)
        assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
        m = frames.MetricsWriter(tmp_path / "ours_m.csv", h)
        m.append(w.scene, st)
        m.flush()
        r.write_metrics(tmp_path / "ref_m.csv", h)
        assert (tmp_path / "ours_m.csv").read_bytes() == (tmp_path / "ref_m.csv").read_bytes()
    n_rows = len((tmp_path / "ours.csv").read_text().splitlines()) - 2
    assert 0 < n_rows == int(np.sum(w.scene.activation_substep <= 27))


def test_actions_json_matches_reference(ref_available):
    from oracle.ref import RefWorld
    spec = scenes.scaled("c1", 16)
    r = RefWorld(spec)
    vals = np.random.default_rng(0).standard_normal((3, 6))
    a = fl.ActionTrajectory(3, 5, vals)
    j = frames.actions_to_json(a)
    assert j == r.actions_json(vals, 5)
    b = frames.actions_from_json(j)
    assert b.n_segments == 3 and b.segment_length == 5 and np.array_equal(np.asarray(b.values), vals)


def test_format_real_is_shortest_roundtrip_17g():
    for v in [0.1, 1.0 / 3.0, -2.5e-300, 1e21, 0.0, 123456789.125]:
        s = frames.format_real(v)
        assert float(s) == v and s == "%.17g" % v
