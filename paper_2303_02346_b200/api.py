"""Host-side mirror of the reference's scene / step / grad API (D = 3).

Names, argument meaning and error behaviour follow proj/include/flume:

    build_scene(spec)                               scene.hpp:161   -> World
    mpm_substep(scene, state, action, ws)           mpm.hpp:455
    p2g_grid(scene, state, ws)                      mpm.hpp:249 + :301 (p2g then grid_update)
    adjoint_substep(scene, rec, adj, action_bar, ws) adjoint.hpp:476
    rollout_loss(scene, state0, actions, loss, window, per_segment)   grad.hpp:15
    grad_trajectory(scene, state0, actions, loss, stride, window)     grad.hpp:61
    ActionTrajectory, LossEvaluator, TrajectoryGrad, AdjointState, SubstepRecord

`ws` is a GpuWorkspace (the MpmWorkspace analogue): it owns the device
context, and the SimState stays resident in HBM between calls -- host arrays
are only copied back when read.  Errors raise the reference's exception
types (core.hpp:18-48).
"""
from __future__ import annotations

import ctypes as C
import json as _json
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import load

# ---------------------------------------------------------------------------
# exceptions (core.hpp:18-48)
# ---------------------------------------------------------------------------


class EngineError(RuntimeError):
    pass


class SceneError(EngineError):
    pass


class DegenerateDeformation(EngineError):
    def __init__(self, msg, particle_id=-1):
        super().__init__(msg)
        self.particle_id = particle_id


class RigidityError(EngineError):
    def __init__(self, msg, body_id=-1):
        super().__init__(msg)
        self.body_id = body_id


class AdjointError(EngineError):
    def __init__(self, msg, substep=-1):
        super().__init__(msg)
        self.substep = substep


class SolverError(EngineError):
    pass


class DeviceError(EngineError):
    pass


def _raise(lib, ctx, rc):
    if rc == _abi.FLUME_OK:
        return
    info = _abi.ErrorInfo()
    lib.flume_last_error(ctx, C.byref(info))
    msg = info.message.decode(errors="replace")
    if rc == _abi.FLUME_E_SCENE:
        raise SceneError(msg)
    if rc == _abi.FLUME_E_DEGENERATE:
        raise DegenerateDeformation(msg, info.particle_id)
    if rc == _abi.FLUME_E_RIGIDITY:
        raise RigidityError(msg, info.body_id)
    if rc == _abi.FLUME_E_ADJOINT:
        raise AdjointError(msg, info.substep)
    if rc == _abi.FLUME_E_SOLVER:
        raise SolverError(msg)
    if rc == _abi.FLUME_E_CUDA:
        raise DeviceError(msg)
    if rc == _abi.FLUME_E_ARG:
        raise ValueError(msg)
    raise EngineError(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------------------
# data model
# ---------------------------------------------------------------------------

MATERIAL_KINDS = ["elastic", "plastic", "liquid", "viscous_liquid", "non_newtonian", "rigid"]
SHAPE_KINDS = ["sphere", "box", "capsule", "cylinder", "halfspace"]


class Scene:
    """Immutable scene data (types.hpp:227-235) as a flume_scene_desc.

    Owns the ctypes arrays the descriptor points to."""

    def __init__(self, desc: _abi.SceneDesc, keepalive):
        self.desc = desc
        self._keep = keepalive
        c = desc.config
        self.grid_resolution = c.grid_resolution
        self.domain = tuple(c.domain)
        self.dt_substep = c.dt_substep
        self.gravity = tuple(c.gravity)
        self.dx = c.domain[0] / c.grid_resolution
        self.n_particles = desc.n_particles
        n = desc.n_particles
        self.material_id = np.ctypeslib.as_array(desc.material_id, (n,)).copy()
        self.body_id = np.ctypeslib.as_array(desc.body_id, (n,)).copy()
        self.mass = np.ctypeslib.as_array(desc.mass, (n,)).copy()
        self.volume0 = np.ctypeslib.as_array(desc.volume0, (n,)).copy()
        self.activation_substep = np.ctypeslib.as_array(desc.activation_substep, (n,)).copy()
        self.materials = [desc.materials[i] for i in range(desc.n_materials)]
        self.n_effectors = desc.n_effectors
        self.action_masks = [[bool(desc.effectors[e].action_mask[k]) for k in range(6)]
                             for e in range(desc.n_effectors)]

    @property
    def node_dims(self):
        return tuple(int(round(self.domain[a] / self.dx)) + 1 for a in range(3))


class SimState:
    """SimState<3> (types.hpp:179-205) with lazy host/device synchronisation."""

    def __init__(self, x, v, F, C_, effectors, time=0.0, substep_index=0):
        self._x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
        self._v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 3)
        self._F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1, 3, 3)
        self._C = np.ascontiguousarray(C_, dtype=np.float64).reshape(-1, 3, 3)
        self._eff = np.ascontiguousarray(effectors, dtype=np.float64).reshape(-1, 18)
        self._time = float(time)
        self._substep = int(substep_index)
        self._ws: Optional["GpuWorkspace"] = None  # workspace holding the newer copy
        self._ver = 0  # bumped by every host access: a workspace re-uploads a state whose version moved

    # host views pull the device copy first and make the host authoritative
    def _pull(self):
        if self._ws is not None:
            self._ws._download(self)
            self._ws._resident = None
            self._ws = None

    def copy(self) -> "SimState":
        self._pull()
        return SimState(self._x.copy(), self._v.copy(), self._F.copy(), self._C.copy(), self._eff.copy(),
                        self._time, self._substep)

    # host access hands out the arrays themselves (callers may modify them in place), so
    # any access makes the host copy authoritative for the next upload
    def _touch(self):
        self._pull()
        self._ver += 1

    @property
    def n_particles(self):
        return self._x.shape[0]

    def _prop(name):  # noqa: N805
        def get(self):
            self._touch()
            return getattr(self, name)

        def set_(self, val):
            self._touch()
            getattr(self, name)[...] = val

        return property(get, set_)

    x = _prop("_x")
    v = _prop("_v")
    F = _prop("_F")
    C = _prop("_C")
    effectors = _prop("_eff")

    @property
    def time(self):
        return self._time

    @property
    def substep_index(self):
        return self._substep

    @substep_index.setter
    def substep_index(self, v):
        self._touch()
        self._substep = int(v)

    def active_particle_count(self, scene: Scene) -> int:
        return int(np.sum(scene.activation_substep <= self.substep_index))


@dataclass
class World:
    scene: Scene
    state: SimState
    loss_spec: list
    n_segments: int
    segment_length: int
    init_action: np.ndarray
    spec: dict


def build_scene(spec) -> World:
    """build_scene<3> (scene.hpp:161) through the library's JSON builder."""
    lib = load()
    text = spec if isinstance(spec, str) else _json.dumps(spec)
    h = C.c_void_p()
    rc = lib.flume_scene_build_json(text.encode(), C.byref(h))
    if rc != _abi.FLUME_OK:
        msg = lib.flume_scene_error(h).decode() if h else "scene error"
        lib.flume_scene_free(h)
        raise SceneError(msg)
    try:
        desc = _abi.SceneDesc()
        lib.flume_scene_desc_get(h, C.byref(desc))
        keep = _copy_desc(desc)
        view = _abi.StateView()
        lib.flume_scene_state_get(h, C.byref(view))
        n = desc.n_particles
        # (an empty scene hands out null arrays)
        grab = lambda p, k: np.ctypeslib.as_array(p, (n, k)).copy() if n else np.zeros((0, k))  # noqa: E731
        x, v, F, Cm = grab(view.x, 3), grab(view.v, 3), grab(view.F, 9), grab(view.C, 9)
        eff = np.zeros((desc.n_effectors, 18))
        for i in range(desc.n_effectors):
            e = view.effectors[i]
            eff[i] = list(e.pose_t) + list(e.pose_R) + list(e.linear_velocity) + list(e.angular_velocity)
        ld = _abi.LossDesc()
        lib.flume_scene_loss_get(h, C.byref(ld))
        terms = [_term_dict(ld.terms[i]) for i in range(ld.n_terms)]
        ns, sl = C.c_int(), C.c_int()
        init = np.zeros(6)
        lib.flume_scene_optimizer_get(h, C.byref(ns), C.byref(sl), _dp(init))
    finally:
        lib.flume_scene_free(h)
    scene = Scene(keep[0], keep)
    state = SimState(x, v, F, Cm, eff)
    return World(scene, state, terms, ns.value, sl.value, init,
                 spec if isinstance(spec, dict) else _json.loads(text))


_LOSS_KINDS = ["target_point", "hold_initial", "mixing_spread", "trajectory_chamfer"]


def _term_dict(t: _abi.LossTerm) -> dict:
    d = {"kind": _LOSS_KINDS[t.kind], "body": t.body, "weight": t.weight,
         "squared": bool(t.squared), "final_only": bool(t.final_only), "goal": list(t.goal)}
    if d["kind"] == "trajectory_chamfer":
        off = np.ctypeslib.as_array(t.goal_step_offsets, (t.n_goal_steps + 1,)).copy()
        pts = np.ctypeslib.as_array(t.goal_points, (int(off[-1]) * 3,)).reshape(-1, 3).copy()
        d["goal_trajectory"] = [pts[off[s]:off[s + 1]] for s in range(t.n_goal_steps)]
    return d


def _copy_desc(d: _abi.SceneDesc):
    """Deep-copy a descriptor into Python-owned ctypes arrays."""
    keep = []

    def arr(ctype, src, n):
        a = (ctype * max(n, 1))()
        if n:
            C.memmove(a, src, C.sizeof(ctype) * n)
        keep.append(a)
        return C.cast(a, C.POINTER(ctype))

    out = _abi.SceneDesc()
    out.config = d.config
    out.n_materials = d.n_materials
    out.materials = arr(_abi.Material, d.materials, d.n_materials)
    out.n_effectors = d.n_effectors
    out.effectors = arr(_abi.EffectorShape, d.effectors, d.n_effectors)
    out.n_rigid = d.n_rigid
    rbs = (_abi.RigidBody * max(d.n_rigid, 1))()
    for i in range(d.n_rigid):
        r = d.rigid[i]
        rbs[i].body_id = r.body_id
        rbs[i].n_members = r.n_members
        rbs[i].members = arr(C.c_long, r.members, r.n_members)
        rbs[i].rest_offsets = arr(C.c_double, r.rest_offsets, 3 * r.n_members)
        rbs[i].total_mass = r.total_mass
    keep.append(rbs)
    out.rigid = C.cast(rbs, C.POINTER(_abi.RigidBody))
    out.n_emitters = d.n_emitters
    out.emitters = arr(_abi.Emitter, d.emitters, d.n_emitters)
    n = d.n_particles
    out.n_particles = n
    out.material_id = arr(C.c_int, d.material_id, n)
    out.body_id = arr(C.c_int, d.body_id, n)
    out.mass = arr(C.c_double, d.mass, n)
    out.volume0 = arr(C.c_double, d.volume0, n)
    out.activation_substep = arr(C.c_long, d.activation_substep, n)
    return [out] + keep


@dataclass
class ActionTrajectory:
    """actions.hpp:13-39: one Action6 per segment."""
    n_segments: int = 1
    segment_length: int = 1
    values: np.ndarray = None

    def __post_init__(self):
        if self.values is None:
            self.values = np.zeros((self.n_segments, 6))
        self.values = np.ascontiguousarray(self.values, dtype=np.float64).reshape(self.n_segments, 6)

    def horizon(self) -> int:
        return self.n_segments * self.segment_length

    def segment_of(self, t: int) -> int:
        return t // self.segment_length

    def at_substep(self, t: int):
        return self.values[self.segment_of(t)]

    def _c(self):
        a = _abi.Actions()
        a.n_segments = self.n_segments
        a.segment_length = self.segment_length
        a.values = _dp(self.values)
        return a


class LossEvaluator:
    """Device-evaluable LossEvaluator (losses.hpp:306): target_point, hold_initial,
    mixing_spread and trajectory_chamfer terms, optionally composite."""

    def __init__(self, scene: Optional[Scene] = None, spec=None, state0: Optional[SimState] = None):
        terms = spec if isinstance(spec, list) else ([] if spec is None else self._parse(spec))
        if not terms:
            raise SceneError("scene has no loss specification")
        self.terms = terms
        self._arr = (_abi.LossTerm * len(terms))()
        self._keep = []
        for i, t in enumerate(terms):
            k = _LOSS_KINDS.index(t["kind"])
            self._arr[i].kind = k
            if t["kind"] == "trajectory_chamfer":
                steps = [np.asarray(s, dtype=np.float64).reshape(-1, 3) for s in t["goal_trajectory"]]
                off = np.zeros(len(steps) + 1, dtype=np.int64)
                off[1:] = np.cumsum([len(s) for s in steps])
                pts = np.ascontiguousarray(np.concatenate(steps, 0))
                self._keep += [off, pts]
                self._arr[i].n_goal_steps = len(steps)
                self._arr[i].goal_step_offsets = off.ctypes.data_as(C.POINTER(C.c_long))
                self._arr[i].goal_points = _dp(pts)
            self._arr[i].body = int(t["body"])
            self._arr[i].weight = float(t.get("weight", 1.0))
            self._arr[i].squared = int(bool(t.get("squared", False)))
            self._arr[i].final_only = int(bool(t.get("final_only", False)))
            g = t.get("goal", [0, 0, 0])
            for a in range(3):
                self._arr[i].goal[a] = float(g[a])
        self.desc = _abi.LossDesc(len(terms), C.cast(self._arr, C.POINTER(_abi.LossTerm)))
        self.desc.attraction_body = -1
        self._prev = None

    # -- the optimizer's gradient-sharing surrogate (losses.hpp:104-218, 348-363) --
    def enable_attraction(self, body: int, weight: float, radius: float, tau: float) -> None:
        """LossEvaluator::enable_attraction: body < 0 selects the first term's body."""
        self.desc.attraction_body = int(body) if body >= 0 else int(self.terms[0]["body"])
        self.desc.attraction_weight = float(weight)
        self.desc.attraction_radius = float(radius)
        self.desc.attraction_tau = float(tau)

    def set_attraction_prev(self, prev_losses) -> None:
        """prev_losses_ as refresh_attraction leaves it: per-particle losses of the body's
        members in particle-id order."""
        self._prev = np.ascontiguousarray(prev_losses, dtype=np.float64).reshape(-1)
        self.desc.n_prev = self._prev.size
        self.desc.prev_losses = _dp(self._prev)

    def per_particle(self, state: SimState, ws: "GpuWorkspace") -> np.ndarray:
        """LossEvaluator::per_particle (losses.hpp:367-390) of `state`, computed on the device."""
        ws._upload(state)
        out = np.zeros(ws.scene.n_particles)
        ws._check(ws.lib.flume_loss_per_particle(ws.ctx, C.byref(self.desc), _dp(out)))
        return out

    def refresh_attraction(self, state: SimState, ws: "GpuWorkspace") -> None:
        """LossEvaluator::refresh_attraction (losses.hpp:357-363)."""
        if not self.desc.attraction_weight > 0:
            return
        allp = self.per_particle(state, ws)
        body = np.asarray(ws.scene.body_id)
        self.set_attraction_prev(allp[body == self.desc.attraction_body])

    @staticmethod
    def _parse(spec: dict):
        def one(t):
            d = {"kind": t.get("kind", "target_point"), "body": t["body"], "weight": t.get("weight", 1.0),
                 "squared": t.get("squared", False), "final_only": t.get("eval", "per_step") == "final",
                 "goal": t.get("goal", [0, 0, 0])}
            if "goal_trajectory" in t:
                d["goal_trajectory"] = t["goal_trajectory"]
            return d
        if spec.get("kind") == "composite":
            return [one(t) for t in spec["terms"]]
        return [one(spec)]


@dataclass
class TrajectoryGrad:
    loss: float = 0.0
    full_loss: float = 0.0
    per_segment: List[float] = field(default_factory=list)
    action_grad: np.ndarray = None
    snapshots: int = 0
    forward_ms: float = 0.0
    backward_ms: float = 0.0

    def flatten(self):
        return self.action_grad.reshape(-1).tolist()


@dataclass
class AdjointState:
    """Cotangents of a SimState (adjoint.hpp:9-46), reference particle order."""
    x_bar: np.ndarray
    v_bar: np.ndarray
    F_bar: np.ndarray
    C_bar: np.ndarray
    eff_bars: np.ndarray  # n_eff x 12: t_bar[3], R_bar[9]

    @staticmethod
    def init(state: SimState) -> "AdjointState":
        n = state.n_particles
        return AdjointState(np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 3, 3)), np.zeros((n, 3, 3)),
                            np.zeros((state._eff.shape[0], 12)))


@dataclass
class SubstepRecord:
    index: int
    action: Sequence[float]
    pre_state: SimState


# ---------------------------------------------------------------------------
# workspace = device context
# ---------------------------------------------------------------------------


class GpuWorkspace:
    """Device context for one scene (MpmWorkspace analogue, mpm.hpp:223-238).

    ranks > 1: x-slab decomposition over `ranks` contexts in this process
    (SURVEY.md 8(e)); `devices` lists one CUDA device per rank (default: all on
    `device`).  Every call runs on all ranks concurrently, one thread each.
    """

    def __init__(self, scene: Scene, device: int = 0, ranks: int = 1, devices: Optional[Sequence[int]] = None):
        self.lib = load()
        self.scene = scene
        self.ctx = C.c_void_p()
        if ranks == 1 and devices is None:
            rc = self.lib.flume_ctx_create(C.byref(scene.desc), device, C.byref(self.ctx))
            if rc != _abi.FLUME_OK:
                _raise(self.lib, None, rc)
            self.ctxs = [self.ctx]
        else:
            devs = list(devices) if devices is not None else [device] * ranks
            arr = (C.c_void_p * len(devs))()
            rc = self.lib.flume_group_create(C.byref(scene.desc), len(devs), (C.c_int * len(devs))(*devs), arr)
            if rc != _abi.FLUME_OK:
                _raise(self.lib, None, rc)
            self.ctxs = [C.c_void_p(arr[i]) for i in range(len(devs))]
            self.ctx = self.ctxs[0]
        self._resident: Optional[SimState] = None
        self._resident_ver = -1
        self._ctx_time = 0.0
        self._ctx_substep = 0

    @classmethod
    def distributed(cls, scene: Scene, device: int, rank: int, n_ranks: int, uid: bytes) -> "GpuWorkspace":
        """This process's rank of an x-slab group spanning processes (one per GPU,
        NCCL); `uid` = dist_unique_id() of rank 0, shared by the launcher.  Every
        call is collective over the ranks."""
        self = cls.__new__(cls)
        self.lib = load()
        self.scene = scene
        self.ctx = C.c_void_p()
        u = (C.c_ubyte * 128).from_buffer_copy(uid)
        rc = self.lib.flume_ctx_create_dist(C.byref(scene.desc), device, rank, n_ranks, u, C.byref(self.ctx))
        if rc != _abi.FLUME_OK:
            _raise(self.lib, None, rc)
        self._dist = True
        self.ctxs = [self.ctx]
        self._resident = None
        self._resident_ver = -1
        self._ctx_time = 0.0
        self._ctx_substep = 0
        return self

    @property
    def ranks(self) -> int:
        return len(self.ctxs)

    def set_checkpoint_spill(self, host: bool = True):
        """grad_trajectory snapshots in pinned host memory instead of HBM (long horizons)."""
        self._collective(lambda r, c: self.lib.flume_set_checkpoint_spill(c, int(bool(host))))

    def set_checkpoint_spill_dir(self, directory: str):
        """grad_trajectory snapshots in a file under `directory` (local NVMe), read back when
        the backward replays their segment; results identical."""
        d = str(directory).encode()
        self._collective(lambda r, c: self.lib.flume_set_checkpoint_spill_dir(c, d))

    CHAMFER_MODES = {"auto": 0, "scan": 1, "grid": 2}

    def set_chamfer_mode(self, mode: str = "auto"):
        """trajectory_chamfer nearest-neighbour search: "auto", "scan" (brute force) or "grid"
        (uniform-grid index); identical results (the reference's first-index minimum)."""
        if mode not in self.CHAMFER_MODES:
            raise ValueError(f"chamfer mode must be one of {sorted(self.CHAMFER_MODES)}")
        self._collective(lambda r, c: self.lib.flume_set_chamfer_mode(c, self.CHAMFER_MODES[mode]))

    def set_incremental_sort(self, on: bool = True):
        """Sort only the blocks whose particles changed cell since the previous substep
        (default) or always run the full block sort; identical order and results."""
        self._collective(lambda r, c: self.lib.flume_set_incremental_sort(c, 1 if on else 0))

    def sort_stats(self):
        """[(incremental sorts, full sorts)] per rank."""
        out = []
        for c in self.ctxs:
            a, b = C.c_long(), C.c_long()
            self.lib.flume_sort_stats(c, C.byref(a), C.byref(b))
            out.append((a.value, b.value))
        return out

    def set_migration_capacity(self, capacity: int):
        """Slots per neighbour and substep of the fixed-size migration messages (slab
        workspaces); an overflowing call is re-run with 4x the capacity."""
        self._collective(lambda r, c: self.lib.flume_slab_set_migration_capacity(c, int(capacity)))

    def migration_stats(self):
        """[(capacity, re-runs)] per rank."""
        out = []
        for c in self.ctxs:
            cap, n = C.c_int(), C.c_long()
            self.lib.flume_slab_migration_stats(c, C.byref(cap), C.byref(n))
            out.append((cap.value, n.value))
        return out

    def slab_info(self):
        """[(rank, sx0, sx1, n_active)] -- the x-columns of 4 cells each rank owns."""
        out = []
        for c in self.ctxs:
            r, n, a, b, na = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_long()
            self.lib.flume_slab_info(c, C.byref(r), C.byref(n), C.byref(a), C.byref(b), C.byref(na))
            out.append((r.value, a.value, b.value, na.value))
        return out

    def _collective(self, fn):
        """fn(rank, ctx) -> status, on every rank concurrently (ctypes drops the GIL)."""
        if len(self.ctxs) == 1:
            self._check(fn(0, self.ctx))
            return
        rcs = [None] * len(self.ctxs)

        def run(i):
            rcs[i] = fn(i, self.ctxs[i])

        th = [threading.Thread(target=run, args=(i,)) for i in range(len(self.ctxs))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        bad = [i for i, rc in enumerate(rcs) if rc != _abi.FLUME_OK]
        if not bad:
            return
        # report the rank that failed first, not the peers it released
        for i in bad:
            info = _abi.ErrorInfo()
            self.lib.flume_last_error(self.ctxs[i], C.byref(info))
            if b"aborted by a failing rank" not in info.message:
                _raise(self.lib, self.ctxs[i], rcs[i])
        _raise(self.lib, self.ctxs[bad[0]], rcs[bad[0]])

    def close(self):
        if self.ctx:
            if self._resident is not None:
                self._resident._pull()
            for c in self.ctxs:
                self.lib.flume_ctx_destroy(c)
            self.ctx = C.c_void_p()
            self.ctxs = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        _raise(self.lib, self.ctx, rc)

    def _view(self, st: SimState, effs):
        v = _abi.StateView()
        v.time = st._time
        v.substep_index = st._substep
        v.x, v.v, v.F, v.C = _dp(st._x), _dp(st._v), _dp(st._F), _dp(st._C)
        v.effectors = effs
        return v

    @staticmethod
    def _eff_to_c(eff):
        arr = (_abi.EffectorState * max(len(eff), 1))()
        for i, e in enumerate(eff):
            arr[i].pose_t[:] = list(e[0:3])
            arr[i].pose_R[:] = list(e[3:12])
            arr[i].linear_velocity[:] = list(e[12:15])
            arr[i].angular_velocity[:] = list(e[15:18])
        return arr

    def _upload(self, st: SimState):
        if self._resident is st and self._resident_ver == st._ver:
            return
        if self._resident is not None:
            self._resident._pull()
        st._pull()
        effs = self._eff_to_c(st._eff)
        view = self._view(st, effs)
        self._collective(lambda r, c: self.lib.flume_state_upload(c, C.byref(view)))
        self._resident = st
        self._resident_ver = st._ver
        self._ctx_time = st._time
        self._ctx_substep = st._substep

    def _download(self, st: SimState):
        effs = (_abi.EffectorState * max(len(st._eff), 1))()
        v = self._view(st, effs)
        views, keep = [v], []
        for _ in range(1, len(self.ctxs)):  # every rank assembles the whole state; keep rank 0's
            sc = SimState.__new__(SimState)
            sc._time, sc._substep = st._time, st._substep
            sc._x, sc._v, sc._F, sc._C = (np.empty_like(a) for a in (st._x, st._v, st._F, st._C))
            e = (_abi.EffectorState * max(len(st._eff), 1))()
            keep.append((sc, e))
            views.append(self._view(sc, e))
        self._collective(lambda r, c: self.lib.flume_state_download(c, C.byref(views[r])))
        for i in range(len(st._eff)):
            e = effs[i]
            st._eff[i] = list(e.pose_t) + list(e.pose_R) + list(e.linear_velocity) + list(e.angular_velocity)
        st._time = v.time
        st._substep = v.substep_index

    def _mark_device_newer(self, st: SimState):
        st._ws = self
        self._resident = st
        self._resident_ver = st._ver

    def store_order(self, st: SimState):
        """Canonical store order (cell keys, particle ids, active count) + fp32 positions: the
        order the next substep's sort puts the state in (one rank; slab ranks: the store as
        it is)."""
        self._upload(st)
        n = self.scene.n_particles * getattr(self, "n_replicas", 1)
        keys = np.zeros(n, np.uint32)
        ids = np.zeros(n, np.uint32)
        na = C.c_long()
        xs = np.zeros(3 * n, np.float32)
        kp, ip = keys.ctypes.data_as(C.POINTER(C.c_uint)), ids.ctypes.data_as(C.POINTER(C.c_uint))
        xp = xs.ctypes.data_as(C.POINTER(C.c_float))
        if len(self.ctxs) == 1 and not getattr(self, "_dist", False):
            self._check(self.lib.flume_store_sorted(self.ctx, kp, ip, xp, C.byref(na)))
        else:
            self._check(self.lib.flume_store_order(self.ctx, kp, ip, C.byref(na)))
            self._check(self.lib.flume_store_positions(self.ctx, xp))
        return keys, ids, na.value, xs.reshape(3, n)

    def last_timing(self):
        t = _abi.Timing()
        self.lib.flume_last_timing(self.ctx, C.byref(t))
        return t


def slab_split(col_weight, n_ranks: int) -> list:
    """The x-column split of the slab ranks (flume_slab_split): rank r owns the
    4-cell columns [cuts[r], cuts[r+1]).  Host-only."""
    lib = load()
    w = np.ascontiguousarray(col_weight, dtype=np.float64)
    cuts = (C.c_int * (n_ranks + 1))()
    rc = lib.flume_slab_split(_dp(w), int(w.size), int(n_ranks), cuts)
    if rc != _abi.FLUME_OK:
        raise ValueError("slab_split: need at least one column per rank")
    return list(cuts)


def dist_unique_id() -> bytes:
    """NCCL unique id for GpuWorkspace.distributed (call on one rank, broadcast)."""
    lib = load()
    u = (C.c_ubyte * 128)()
    rc = lib.flume_dist_unique_id(u)
    if rc != _abi.FLUME_OK:
        _raise(lib, None, rc)
    return bytes(u)


def ipc_unique_id() -> bytes:
    """Group id for GpuWorkspace.distributed over CUDA IPC (the processes of one node,
    one or several ranks per GPU) instead of NCCL; call on one rank and share it."""
    lib = load()
    u = (C.c_ubyte * 128)()
    rc = lib.flume_ipc_unique_id(u)
    if rc != _abi.FLUME_OK:
        _raise(lib, None, rc)
    return bytes(u)


def _ws_for(scene: Scene, ws: Optional[GpuWorkspace]) -> GpuWorkspace:
    if ws is None:
        raise ValueError("a GpuWorkspace is required (MpmWorkspace analogue)")
    if ws.scene is not scene:
        raise ValueError("workspace belongs to a different scene")
    return ws


# ---------------------------------------------------------------------------
# API
# ---------------------------------------------------------------------------


def mpm_substep(scene: Scene, state: SimState, action, ws: GpuWorkspace, count: int = 1) -> None:
    """mpm.hpp:455-473 (count > 1 chains substeps without host round trips)."""
    ws = _ws_for(scene, ws)
    a = np.ascontiguousarray(action, dtype=np.float64).ravel()
    need = 6 * getattr(ws, "n_replicas", 1)  # a replica context takes one Action6 per replica
    if a.size != need:
        raise ValueError(f"mpm_substep: {need} action values expected, got {a.size}")
    ws._upload(state)
    ws._collective(lambda r, c: ws.lib.flume_substep(c, _dp(a), int(count)))
    t = state._time
    for _ in range(int(count)):  # the reference accumulates time += dt per substep (mpm.hpp:471)
        t += scene.dt_substep
    ws._ctx_time = t
    ws._ctx_substep = state._substep + count
    state._time, state._substep = ws._ctx_time, ws._ctx_substep
    ws._mark_device_newer(state)


def p2g_grid(scene: Scene, state: SimState, ws: GpuWorkspace):
    """p2g + grid_update on a state (mpm.hpp:249, :301); dense mass and velocity grids."""
    ws = _ws_for(scene, ws)
    ws._upload(state)
    nd = scene.node_dims
    mass = np.zeros(nd)
    vel = np.zeros(nd + (3,))
    # slab ranks write disjoint node planes of the same arrays
    ws._collective(lambda r, c: ws.lib.flume_stage_grid(c, _dp(mass), _dp(vel)))
    return mass, vel


def rollout_loss(scene: Scene, state0: SimState, actions: ActionTrajectory, loss: LossEvaluator,
                 window: int = 0, per_segment: Optional[list] = None, ws: Optional[GpuWorkspace] = None,
                 final_state: Optional[SimState] = None, on_substep=None) -> float:
    """grad.hpp:15-41.  final_state (the reference's out-pointer) receives the state after
    the whole horizon (the context continues from it: flume_rollout_loss_final), and
    on_substep(state) runs after every substep (metrics exports; the deterministic forward is
    re-run on the device from state0, host copies happen only if the callback reads host
    fields)."""
    ws = _ws_for(scene, ws)
    keep = final_state is not None and on_substep is None  # the context ends on the final state
    if keep:
        state0._pull()  # state0's host copy must survive the context moving on
    ws._upload(state0)
    outs = [C.c_double() for _ in ws.ctxs]
    pers = [np.zeros(actions.n_segments) for _ in ws.ctxs]
    a = actions._c()
    fn = ws.lib.flume_rollout_loss_final if keep else ws.lib.flume_rollout_loss
    ws._collective(lambda r, c: fn(c, C.byref(a), C.byref(loss.desc), int(window), C.byref(outs[r]),
                                   _dp(pers[r])))
    out, per = outs[0], pers[0]
    if per_segment is not None:
        per_segment[:] = per.tolist()
    if keep:
        ws._resident = None  # the context left state0
        final_state._pull()
        for name in ("_x", "_v", "_F", "_C", "_eff"):
            setattr(final_state, name, np.empty_like(getattr(state0, name)))
        ws._download(final_state)
        final_state._ver += 1
        ws._resident, ws._resident_ver = final_state, final_state._ver
        ws._ctx_time, ws._ctx_substep = final_state._time, final_state._substep
        return out.value
    if final_state is not None or on_substep is not None:
        st = state0.copy()
        for s in range(actions.n_segments):
            if on_substep is None:
                mpm_substep(scene, st, actions.values[s], ws, count=actions.segment_length)
                continue
            for _ in range(actions.segment_length):  # the callback sees every substep's state
                mpm_substep(scene, st, actions.values[s], ws)
                on_substep(st)
    if final_state is not None:
        st._pull()
        for name in ("_x", "_v", "_F", "_C", "_eff", "_time", "_substep"):
            setattr(final_state, name, getattr(st, name))
        final_state._ws = None
    return out.value


def grad_trajectory(scene: Scene, state0: SimState, actions: ActionTrajectory, loss: LossEvaluator,
                    stride: int = 0, window: int = 0, ws: Optional[GpuWorkspace] = None) -> TrajectoryGrad:
    """grad.hpp:61-134 (checkpoint stride semantics of checkpoint.hpp:11-50)."""
    ws = _ws_for(scene, ws)
    ws._upload(state0)
    R = len(ws.ctxs)
    gs = [np.zeros((actions.n_segments, 6)) for _ in range(R)]
    res = [(C.c_double(), C.c_double(), C.c_long()) for _ in range(R)]
    pers = [np.zeros(actions.n_segments) for _ in range(R)]
    a = actions._c()
    ws._collective(lambda r, c: ws.lib.flume_grad_trajectory(c, C.byref(a), C.byref(loss.desc), int(stride),
                                                             int(window), _dp(gs[r]), C.byref(res[r][0]),
                                                             C.byref(res[r][1]), _dp(pers[r]), C.byref(res[r][2])))
    g, per = gs[0], pers[0]
    lo, fl, snaps = res[0]
    t = ws.last_timing()
    return TrajectoryGrad(lo.value, fl.value, per.tolist(), g, snaps.value, t.forward_ms, t.backward_ms)


@dataclass
class GradReport:
    """grad.hpp:160-175."""
    gradient: List[float] = field(default_factory=list)
    fd_gradient: List[float] = field(default_factory=list)
    max_rel_error: float = 0.0
    wall_time: float = 0.0
    loss: float = 0.0

    @staticmethod
    def rel_error(g, fd) -> float:
        num = max((abs(a - b) for a, b in zip(g, fd)), default=0.0)
        den = max((abs(b) for b in fd), default=0.0)
        return num / (den + 1e-12)


def finite_difference_gradient(objective, params, eps: float) -> List[float]:
    """Central differences, two evaluations per parameter (grad.hpp:140-158)."""
    if eps <= 0:
        raise EngineError("finite_difference_gradient: eps must be positive")
    grad = []
    for i in range(len(params)):
        p, m = list(params), list(params)
        p[i] += eps
        m[i] -= eps
        fp, fm = objective(p), objective(m)
        if not (np.isfinite(fp) and np.isfinite(fm)):
            raise EngineError(f"finite_difference_gradient: non-finite objective at parameter {i}")
        grad.append((fp - fm) / (2 * eps))
    return grad


def optimizable_components(scene: Scene) -> List[int]:
    """Action components any effector accepts (grad.hpp:177-188)."""
    return [k for k in range(6) if any(m[k] for m in scene.action_masks)]


def grad_check(scene: Scene, state0: SimState, actions: ActionTrajectory, loss: LossEvaluator, stride: int,
               eps: float, with_fd: bool = True, ws: Optional[GpuWorkspace] = None) -> GradReport:
    """grad.hpp:190-225: the adjoint gradient over the optimizable components, audited by
    central differences of device rollouts.  The device computes in fp32, so eps must be
    large enough for the loss differences to clear fp32 rounding (about 1e-3 for O(1) actions)."""
    import time as _time
    t0 = _time.perf_counter()
    comps = optimizable_components(scene)
    rep = GradReport()
    tg = grad_trajectory(scene, state0, actions, loss, stride=stride, ws=ws)
    rep.loss = tg.loss
    rep.gradient = [float(tg.action_grad[s][k]) for s in range(actions.n_segments) for k in comps]
    if with_fd:
        base = np.asarray(actions.values, dtype=np.float64).reshape(actions.n_segments, 6)
        params = [float(base[s][k]) for s in range(actions.n_segments) for k in comps]

        def objective(p):
            v = base.copy()
            idx = 0
            for s in range(actions.n_segments):
                for k in comps:
                    v[s][k] = p[idx]
                    idx += 1
            return rollout_loss(scene, state0, ActionTrajectory(actions.n_segments, actions.segment_length, v), loss,
                                ws=ws)

        rep.fd_gradient = finite_difference_gradient(objective, params, eps)
        rep.max_rel_error = GradReport.rel_error(rep.gradient, rep.fd_gradient)
    rep.wall_time = _time.perf_counter() - t0
    return rep


def adjoint_substep(scene: Scene, rec: SubstepRecord, adj: AdjointState, action_bar: np.ndarray,
                    ws: GpuWorkspace) -> None:
    """adjoint.hpp:476-548: bars of the post-state -> bars of rec.pre_state (in place)."""
    ws = _ws_for(scene, ws)
    ws._upload(rec.pre_state)
    act = np.ascontiguousarray(rec.action, dtype=np.float64)
    for name in ("x_bar", "v_bar", "F_bar", "C_bar", "eff_bars"):
        setattr(adj, name, np.ascontiguousarray(getattr(adj, name), dtype=np.float64))
    ab = np.ascontiguousarray(action_bar, dtype=np.float64)
    eb = adj.eff_bars if adj.eff_bars.size else np.zeros((1, 12))
    ws._check(ws.lib.flume_adjoint_substep(ws.ctx, _dp(act), _dp(adj.x_bar), _dp(adj.v_bar), _dp(adj.F_bar),
                                           _dp(adj.C_bar), _dp(eb), _dp(ab)))
    action_bar[...] = ab


# ---------------------------------------------------------------------------
# populations: many independent rollouts of one scene, e.g. a
# CMA-ES population (optimize.hpp:383-418) or DP line-search candidates
# ---------------------------------------------------------------------------


class WorkspacePool:
    """K independent device contexts of one scene on one GPU.  Each context owns a
    stream, and the calls below run one host thread per context (ctypes releases the
    GIL), so the small scenes of a population overlap on the device instead of
    queueing behind each other's per-substep launch latency."""

    def __init__(self, scene: Scene, size: int, device: int = 0):
        self.scene = scene
        self.workspaces = [GpuWorkspace(scene, device=device) for _ in range(size)]

    def close(self):
        for ws in self.workspaces:
            ws.close()

    def _map(self, fn, items):
        out = [None] * len(items)
        errs = [None] * len(items)
        k = len(self.workspaces)

        def worker(w):
            for i in range(w, len(items), k):
                try:
                    out[i] = fn(self.workspaces[w], items[i])
                except Exception as e:  # noqa: BLE001 - re-raised below in item order
                    errs[i] = e

        th = [threading.Thread(target=worker, args=(w,)) for w in range(min(k, len(items)))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for e in errs:
            if e is not None:
                raise e
        return out


def _replica_groups(population, R):
    """The population in groups of a replica context's size (the last one padded with its last
    candidate) and each group's real count."""
    pop = list(population)
    for i in range(0, len(pop), R):
        grp = pop[i:i + R]
        yield grp + [grp[-1]] * (R - len(grp)), len(grp)


def rollout_loss_batch(scene: Scene, state0: SimState, population: Sequence[ActionTrajectory],
                       loss: LossEvaluator, pool, window: int = 0) -> List[float]:
    """rollout_loss (grad.hpp:15-41) for every action trajectory of a population, on a
    WorkspacePool (concurrent contexts) or a ReplicaWorkspace (one launch per stage for a
    group of its size; any population size)."""
    if getattr(pool, "n_replicas", None):
        out = []
        for grp, n in _replica_groups(population, pool.n_replicas):
            out += rollout_loss_replicas(scene, state0, grp, loss, pool, window=window)[:n]
        return out
    states = [state0.copy() for _ in pool.workspaces]
    idx = {id(ws): i for i, ws in enumerate(pool.workspaces)}
    return pool._map(lambda ws, a: rollout_loss(scene, states[idx[id(ws)]], a, loss, window=window, ws=ws),
                     list(population))


class ReplicaWorkspace(GpuWorkspace):
    """One device context holding `n_replicas` copies of a scene side by side in one grid
    (flume_ctx_create_replicas, the CMA-ES population of
    optimize.hpp:383-418): every kernel launch of a substep covers the whole population, so
    small scenes fill the GPU.  Positions stay replica-local and each replica's state
    evolves bit-identically to a single context's.  rollout_loss_replicas /
    grad_trajectory_replicas, or rollout_loss_batch / grad_trajectory_batch for populations
    of any size."""

    def __init__(self, scene: Scene, n_replicas: int, device: int = 0):
        self.lib = load()
        self.scene = scene
        self.n_replicas = int(n_replicas)
        self.ctx = C.c_void_p()
        rc = self.lib.flume_ctx_create_replicas(C.byref(scene.desc), self.n_replicas, device, C.byref(self.ctx))
        if rc != _abi.FLUME_OK:
            _raise(self.lib, None, rc)
        self.ctxs = [self.ctx]
        self._resident = None
        self._resident_ver = -1
        self._ctx_time = 0.0
        self._ctx_substep = 0

    def replicate(self, states) -> SimState:
        """The population state: one SimState per replica (or one, repeated), concatenated by
        particle id and effector index.  One repeated state is cached, so a population
        evaluated again from the same initial state (every CMA-ES generation) stays resident."""
        if isinstance(states, SimState):
            c = getattr(self, "_rep_cache", None)
            if c is not None and c[0] is states and c[1] == states._ver and c[2]._ws is None:
                return c[2]
            pop = self.replicate([states] * self.n_replicas)
            self._rep_cache = (states, states._ver, pop)
            return pop
        if len(states) != self.n_replicas:
            raise ValueError(f"need {self.n_replicas} states")
        for s in states:
            s._pull()
        t0, k0 = states[0]._time, states[0]._substep
        if any(s._time != t0 or s._substep != k0 for s in states):
            raise ValueError("replicas advance in lockstep: every state must be at the same substep")
        cat = lambda name: np.concatenate([getattr(s, name) for s in states])  # noqa: E731
        return SimState(cat("_x"), cat("_v"), cat("_F"), cat("_C"), cat("_eff"), t0, k0)

    def split(self, pop: SimState) -> List[SimState]:
        """Per-replica SimStates of a population state."""
        pop._pull()
        n1 = pop.n_particles // self.n_replicas
        e1 = pop._eff.shape[0] // self.n_replicas
        return [SimState(pop._x[r * n1:(r + 1) * n1].copy(), pop._v[r * n1:(r + 1) * n1].copy(),
                         pop._F[r * n1:(r + 1) * n1].copy(), pop._C[r * n1:(r + 1) * n1].copy(),
                         pop._eff[r * e1:(r + 1) * e1].copy(), pop._time, pop._substep)
                for r in range(self.n_replicas)]


def rollout_loss_replicas(scene: Scene, state0, population: Sequence[ActionTrajectory], loss: LossEvaluator,
                          ws: ReplicaWorkspace, window: int = 0, per_segment: Optional[list] = None,
                          final_states: Optional[list] = None) -> List[float]:
    """rollout_loss (grad.hpp:15-41) of a whole population in one replica context: one kernel
    launch per stage covers every candidate.  state0: the common initial SimState (or one per
    replica); per_segment / final_states (lists) receive each replica's per-segment losses
    and final state."""
    ws = _ws_for(scene, ws)
    st = ws.replicate(state0)
    ws._upload(st)
    a, vals, nseg = _replica_actions(ws, population)
    R = ws.n_replicas
    out = np.zeros(R)
    per = np.zeros(R * nseg)
    keep = final_states is not None
    ws._check(ws.lib.flume_replicas_rollout_loss(ws.ctx, C.byref(a), C.byref(loss.desc), int(window), int(keep),
                                                 _dp(out), _dp(per)))
    if per_segment is not None:
        per_segment[:] = [per[r * nseg:(r + 1) * nseg].copy() for r in range(R)]
    if keep:
        ws._resident = None
        ws._rep_cache = None  # st now holds the final states
        ws._download(st)
        final_states[:] = ws.split(st)
    return out.tolist()


def _replica_actions(ws, population):
    pop = list(population)
    R = ws.n_replicas
    if len(pop) != R:
        raise ValueError(f"the replica context holds {R} candidates, got {len(pop)}")
    nseg, seglen = pop[0].n_segments, pop[0].segment_length
    if any(a.n_segments != nseg or a.segment_length != seglen for a in pop):
        raise ValueError("every candidate needs the same segment layout")
    vals = np.ascontiguousarray(np.stack([a.values for a in pop], axis=1))  # (n_segments, R, 6)
    a = _abi.Actions()
    a.n_segments, a.segment_length, a.values = nseg, seglen, _dp(vals)
    return a, vals, nseg


def grad_trajectory_replicas(scene: Scene, state0, population: Sequence[ActionTrajectory], loss: LossEvaluator,
                             ws: ReplicaWorkspace, stride: int = 0, window: int = 0) -> List[TrajectoryGrad]:
    """grad_trajectory (grad.hpp:61-134) of every candidate in one replica context -- a
    population of independent gradient-based optimizations (optimize.hpp:180-239), every
    kernel launch of the forward and the backward covering all of them."""
    ws = _ws_for(scene, ws)
    st = ws.replicate(state0)
    ws._upload(st)
    a, vals, nseg = _replica_actions(ws, population)
    R = ws.n_replicas
    g = np.zeros((R, nseg, 6))
    lo, fu, per = np.zeros(R), np.zeros(R), np.zeros(R * nseg)
    snaps = C.c_long()
    ws._check(ws.lib.flume_replicas_grad_trajectory(ws.ctx, C.byref(a), C.byref(loss.desc), int(stride), int(window),
                                                    _dp(g), _dp(lo), _dp(fu), _dp(per), C.byref(snaps)))
    t = ws.last_timing()
    return [TrajectoryGrad(float(lo[r]), float(fu[r]), per[r * nseg:(r + 1) * nseg].tolist(), g[r].copy(),
                           snaps.value, t.forward_ms, t.backward_ms) for r in range(R)]


def grad_trajectory_batch(scene: Scene, state0: SimState, population: Sequence[ActionTrajectory],
                          loss: LossEvaluator, pool, stride: int = 0,
                          window: int = 0) -> List[TrajectoryGrad]:
    """grad_trajectory (grad.hpp:61-134) for every action trajectory of a population (a
    WorkspacePool or a ReplicaWorkspace, as rollout_loss_batch)."""
    if getattr(pool, "n_replicas", None):
        out = []
        for grp, n in _replica_groups(population, pool.n_replicas):
            out += grad_trajectory_replicas(scene, state0, grp, loss, pool, stride=stride, window=window)[:n]
        return out
    states = [state0.copy() for _ in pool.workspaces]
    idx = {id(ws): i for i, ws in enumerate(pool.workspaces)}
    return pool._map(lambda ws, a: grad_trajectory(scene, states[idx[id(ws)]], a, loss, stride=stride,
                                                   window=window, ws=ws), list(population))


# ---------------------------------------------------------------------------
# versioned state snapshots in the reference's JSON format (io.hpp:144-240), so
# states move between this engine and the reference (and on-disk parity dumps)
# ---------------------------------------------------------------------------


def state_to_json(scene: Scene, state: SimState) -> dict:
    """state_to_json<3> (io.hpp:144-190); pulls the state from the device if needed."""
    state._pull()
    parts = []
    for i in range(scene.n_particles):
        parts.append({"x": state._x[i].tolist(), "v": state._v[i].tolist(), "F": state._F[i].ravel().tolist(),
                      "C": state._C[i].ravel().tolist(), "material": int(scene.material_id[i]),
                      "body": int(scene.body_id[i]), "mass": float(scene.mass[i]),
                      "volume0": float(scene.volume0[i]), "activation": int(scene.activation_substep[i])})
    effs = [{"t": e[0:3].tolist(), "R": e[3:12].tolist(), "v": e[12:15].tolist(), "w": e[15:18].tolist()}
            for e in state._eff]
    return {"version": 1, "dim": 3, "time": state._time, "substep_index": state._substep, "particles": parts,
            "effectors": effs}


def state_from_json(snap: dict, scene: Scene, state: SimState) -> None:
    """state_from_json<3> (io.hpp:192-240) into `state`.  The per-particle constants
    (material, body, mass, volume0, activation) belong to the Scene here, so the
    snapshot must agree with them."""
    if snap.get("version", 0) != 1:
        raise EngineError("snapshot: unsupported version")
    if snap.get("dim", 0) != 3:
        raise EngineError("snapshot: dimension mismatch")
    parts = snap["particles"]
    if len(parts) != scene.n_particles:
        raise EngineError("snapshot: particle count mismatch")
    state._pull()
    for i, p in enumerate(parts):
        if (p["material"] != scene.material_id[i] or p["body"] != scene.body_id[i] or p["mass"] != scene.mass[i]
                or p["volume0"] != scene.volume0[i] or p["activation"] != scene.activation_substep[i]):
            raise EngineError(f"snapshot: particle {i} does not belong to this scene")
        state._x[i] = p["x"]
        state._v[i] = p["v"]
        state._F[i] = np.asarray(p["F"], dtype=np.float64).reshape(3, 3)
        state._C[i] = np.asarray(p["C"], dtype=np.float64).reshape(3, 3)
    for k, e in enumerate(snap["effectors"][:len(state._eff)]):
        state._eff[k] = list(e["t"]) + list(e["R"]) + list(e["v"]) + list(e["w"])
    state._time = float(snap["time"])
    state._substep = int(snap["substep_index"])
