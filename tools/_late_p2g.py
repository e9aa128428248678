import sys, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2303_02346_b200 as fl
from paper_2303_02346_b200 import scenes
w = fl.build_scene(scenes.load("c4"))
ws = fl.GpuWorkspace(w.scene)
a = np.ascontiguousarray(w.init_action, dtype=np.float64)
ws._upload(w.state)
ws.lib.flume_substep(ws.ctx, a.ctypes.data_as(C.POINTER(C.c_double)), int(sys.argv[1]))
ws.lib.flume_sync(ws.ctx)
