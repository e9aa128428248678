"""How much of the store the incremental sort re-sorts: per substep, particles whose cell
key changed, those that changed block, and dirty / occupied particle blocks (sampled along
a forward chain)."""
import json
import sys

import numpy as np

import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import scenes

name = sys.argv[1]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 500
every = int(sys.argv[3]) if len(sys.argv) > 3 else 50
w = fl.build_scene(scenes.load(name))
ws = fl.GpuWorkspace(w.scene)


def keys_by_id():
    k, ids, na, _ = ws.store_order(w.state)
    out = np.full(w.scene.n_particles, 0xFFFFFFFF, np.uint64)
    out[ids[:na]] = k[:na]
    return out


rows = []
t = 0
while t < T:
    fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=every - 1)
    k0 = keys_by_id()
    fl.mpm_substep(w.scene, w.state, w.init_action, ws, count=1)
    k1 = keys_by_id()
    t += every
    act = (k0 != 0xFFFFFFFF) & (k1 != 0xFFFFFFFF)
    ch = act & (k0 != k1)
    bch = act & ((k0 >> 6) != (k1 >> 6))
    blocks = np.unique(k1[k1 != 0xFFFFFFFF] >> 6)
    dirty = np.unique(np.concatenate([k0[ch] >> 6, k1[ch] >> 6]))
    rows.append({"substep": t, "cell_changes": int(ch.sum()), "block_changes": int(bch.sum()),
                 "blocks": int(len(blocks)), "dirty_blocks": int(len(dirty))})
    print(json.dumps(rows[-1]), flush=True)
