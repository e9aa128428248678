"""CPU tests of the multi-rank (x-slab) host logic, SURVEY.md 8(e).

* the column split every rank computes at upload (flume_slab_split, the product's
  host code through the C ABI);
* the slab protocol itself -- two halo planes each way after P2G, grid update
  on owned + ghost planes, particle migration to the neighbour -- run by
  world_size-2 gloo ranks on the numpy restatement (tests/_slab_model.py) and
  compared with one process running the same substeps.  Only the order of the
  fp64 grid sums differs, so the states agree to ~1e-12.
"""
import multiprocessing as mp
import socket

import numpy as np
import pytest

import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import scenes


def test_slab_split_balanced_and_tiling():
    w = np.array([5, 0, 0, 30, 40, 30, 1, 1, 1, 1, 60, 2], dtype=np.float64)
    for ranks in (1, 2, 3, 4, 12):
        cuts = fl.slab_split(w, ranks)
        assert cuts[0] == 0 and cuts[-1] == len(w)
        assert all(cuts[i + 1] > cuts[i] for i in range(ranks))  # at least one column each
    cuts = fl.slab_split(w, 2)
    left = w[:cuts[1]].sum()
    # nearest cut to half the weight
    best = min(abs(w[:c].sum() - w.sum() / 2) for c in range(1, len(w)))
    assert abs(left - w.sum() / 2) == best
    with pytest.raises(ValueError):
        fl.slab_split(w[:2], 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_protocol_two_gloo_ranks_matches_one_process(ref_available, tmp_path):
    from oracle import restate
    from oracle.ref import RefWorld
    from tests import _slab_model

    spec = scenes.scaled("c1", 32)
    substeps, vx = 8, 100.0  # 0.32 cells per substep along x: particles cross the slab face
    out = tmp_path / "slab.npz"
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_slab_model.worker, args=(r, 2, port, spec, substeps, vx, str(out)))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]

    d = np.load(out)
    rows, migrated = d["rows"], int(d["migrated"])
    assert migrated > 0
    ids = rows[:, 0].astype(np.int64)
    sc, st, _ = restate.from_ref(RefWorld(spec))
    assert np.array_equal(np.sort(ids), np.arange(len(st.x)))  # every particle exactly once
    st.v[:, 0] = vx
    for _ in range(substeps):
        st = restate.mpm_substep(sc, st, np.zeros(6))
    order = np.argsort(ids)
    rows = rows[order]
    np.testing.assert_allclose(rows[:, 1:4], st.x, rtol=0, atol=1e-12)
    vs = np.max(np.abs(st.v))
    np.testing.assert_allclose(rows[:, 4:7], st.v, rtol=0, atol=1e-11 * vs)
    np.testing.assert_allclose(rows[:, 7:16], st.F.reshape(-1, 9), rtol=0, atol=1e-11)
    cs = np.max(np.abs(st.C))
    np.testing.assert_allclose(rows[:, 16:25], st.C.reshape(-1, 9), rtol=0, atol=1e-10 * cs)
