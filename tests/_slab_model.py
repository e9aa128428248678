"""CPU model of the x-slab protocol (test infrastructure).

Each gloo rank runs the numpy restatement of the substep (oracle/restate.py)
on the particles it owns and follows the same protocol as the CUDA path
(paper_2303_02346_b200/csrc/fl_slab.cu, Ctx::halo_exchange / Ctx::migrate):
  * columns split by paper_2303_02346_b200.slab_split (the product's host rule),
  * after P2G: node planes [4*sx0, 4*sx0+2) go down, [4*sx1, 4*sx1+2) go up,
    and the receiver adds them (its first owned planes / its ghost planes),
  * grid update on owned + ghost planes, G2P of the owned particles,
  * particles whose new base column left the slab move to the neighbour.
rank 0 gathers the final state by particle id into an .npz.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def _col(x, dx):
    return np.floor(x[:, 0] / dx - 0.5).astype(np.int64) >> 2


def _sendrecv(dist, torch, arr_down, arr_up, rank, world, shape_tail, dtype=np.float64):
    """Exchange with both neighbours: counts first, then payloads (gloo p2p)."""
    out = [None, None]
    reqs = []
    cnt_send = {}
    for d, arr, peer in ((0, arr_down, rank - 1), (1, arr_up, rank + 1)):
        if 0 <= peer < world:
            c = torch.tensor([arr.shape[0]], dtype=torch.int64)
            cnt_send[d] = c
            reqs.append(dist.isend(c, peer))
    cnt = {}
    for d, peer in ((0, rank - 1), (1, rank + 1)):
        if 0 <= peer < world:
            c = torch.zeros(1, dtype=torch.int64)
            dist.recv(c, peer)
            cnt[d] = int(c.item())
    for r in reqs:
        r.wait()
    reqs = []
    keep = []
    for d, arr, peer in ((0, arr_down, rank - 1), (1, arr_up, rank + 1)):
        if 0 <= peer < world and arr.shape[0]:
            t = torch.from_numpy(np.ascontiguousarray(arr, dtype=dtype))
            keep.append(t)
            reqs.append(dist.isend(t, peer))
    for d, peer in ((0, rank - 1), (1, rank + 1)):
        if 0 <= peer < world:
            t = torch.zeros((cnt[d],) + shape_tail, dtype=torch.float64 if dtype == np.float64 else torch.int64)
            if cnt[d]:
                dist.recv(t, peer)
            out[d] = t.numpy()
    for r in reqs:
        r.wait()
    return out


def worker(rank, world, port, spec, substeps, vx, out_path):
    sys.path.insert(0, str(ROOT))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2303_02346_b200 as fl
    from oracle import restate
    from oracle.ref import RefWorld

    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, st, _ = restate.from_ref(RefWorld(spec))
    st.v[:, 0] = vx
    dx = sc.dx
    ncol = (sc.nd[0] + 3) // 4
    w = np.bincount(_col(st.x, dx), minlength=ncol).astype(np.float64)
    cuts = fl.slab_split(w, world)
    sx0, sx1 = cuts[rank], cuts[rank + 1]
    ids = np.nonzero((_col(st.x, dx) >= sx0) & (_col(st.x, dx) < sx1))[0]
    action = np.zeros(6)
    migrated = 0
    for _ in range(substeps):
        loc = restate.State(st.x[ids], st.v[ids], st.F[ids], st.C[ids], st.eff, st.substep, st.time)
        lsc = restate.Scene(**{**sc.__dict__, "mass": sc.mass[ids], "vol0": sc.vol0[ids], "mat": sc.mat[ids],
                               "act": sc.act[ids], "rigid": [], "emitters": None})
        restate.advance_effectors(lsc, loc, action)
        mass, mom = restate.p2g(lsc, loc)
        grid = np.concatenate([mass[..., None], mom], -1)
        lo, hi = 4 * sx0, 4 * sx1
        down = grid[lo:lo + 2] if rank > 0 else np.zeros((0,) + grid.shape[1:])
        up = grid[hi:hi + 2] if rank + 1 < world else np.zeros((0,) + grid.shape[1:])
        rd, ru = _sendrecv(dist, torch, down, up, rank, world, grid.shape[1:])
        if rd is not None and rd.shape[0]:
            grid[lo:lo + 2] += rd  # the lower slab's spill into my first planes
        if ru is not None and ru.shape[0]:
            grid[hi:hi + 2] += ru  # the upper slab's bottom planes: my ghost planes
        vel = restate.grid_update(lsc, loc, grid[..., 0], grid[..., 1:])
        out = restate.g2p(lsc, loc, vel)
        out.substep, out.time = loc.substep + 1, loc.time + sc.dt
        # write back into the global arrays for my ids, then migrate
        st.x[ids], st.v[ids], st.F[ids], st.C[ids] = out.x, out.v, out.F, out.C
        st.eff, st.substep, st.time = out.eff, out.substep, out.time
        col = _col(st.x[ids], dx)
        go_dn, go_up = ids[col < sx0], ids[col >= sx1]
        migrated += len(go_dn) + len(go_up)
        pack = lambda sel: np.concatenate([sel[:, None].astype(np.float64), st.x[sel], st.v[sel],  # noqa: E731
                                           st.F[sel].reshape(-1, 9), st.C[sel].reshape(-1, 9)], 1)
        rd, ru = _sendrecv(dist, torch, pack(go_dn), pack(go_up), rank, world, (25,))
        ids = ids[(col >= sx0) & (col < sx1)]
        for arr in (rd, ru):
            if arr is None or not arr.shape[0]:
                continue
            got = arr[:, 0].astype(np.int64)
            st.x[got], st.v[got] = arr[:, 1:4], arr[:, 4:7]
            st.F[got], st.C[got] = arr[:, 7:16].reshape(-1, 3, 3), arr[:, 16:25].reshape(-1, 3, 3)
            ids = np.sort(np.concatenate([ids, got]))
    # gather by id on rank 0
    payload = np.concatenate([ids[:, None].astype(np.float64), st.x[ids], st.v[ids], st.F[ids].reshape(-1, 9),
                              st.C[ids].reshape(-1, 9)], 1)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([payload.shape[0]], dtype=torch.int64))
    mx = int(max(s.item() for s in sizes))
    buf = torch.zeros((mx, 25), dtype=torch.float64)
    buf[:payload.shape[0]] = torch.from_numpy(payload)
    allb = [torch.zeros((mx, 25), dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allb, buf)
    mig = torch.tensor([migrated], dtype=torch.int64)
    dist.all_reduce(mig)
    if rank == 0:
        rows = np.concatenate([allb[r][:int(sizes[r].item())].numpy() for r in range(world)], 0)
        np.savez(out_path, rows=rows, cuts=np.array(cuts), migrated=int(mig.item()))
    dist.destroy_process_group()
