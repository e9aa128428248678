"""oracle/ref.py -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper around oracle/_ref/libflume_ref.so: the unmodified reference
engine (proj/include/flume, compiled by oracle/Makefile from its own headers)
behind oracle/ref_capi.cpp.  Used by tests/ as the parity checker and by
bench.py's cpu_baseline / --impl reference arm as the timed CPU reference.
Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "_ref" / "libflume_ref.so"
_lib = None

D = C.POINTER(C.c_double)
I = C.POINTER(C.c_int)
L = C.POINTER(C.c_long)


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise RuntimeError(f"{LIB} missing (build with `make -C oracle`)")
        l = C.CDLL(str(LIB))
        sig = {
            "ref_last_error": (C.c_char_p, [L, L, L]),
            "ref_world_from_json": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
            "ref_world_free": (None, [C.c_void_p]),
            "ref_num_particles": (C.c_long, [C.c_void_p]),
            "ref_num_effectors": (C.c_int, [C.c_void_p]),
            "ref_num_materials": (C.c_int, [C.c_void_p]),
            "ref_num_rigid": (C.c_int, [C.c_void_p]),
            "ref_num_emitters": (C.c_long, [C.c_void_p]),
            "ref_config": (None, [C.c_void_p, I, D]),
            "ref_set_hard_contact": (None, [C.c_void_p, C.c_int]),
            "ref_set_gravity": (None, [C.c_void_p, D]),
            "ref_materials": (None, [C.c_void_p, D]),
            "ref_effectors": (None, [C.c_void_p, D]),
            "ref_rigid_members": (C.c_long, [C.c_void_p, C.c_int, L, D, I, D]),
            "ref_emitters": (None, [C.c_void_p, L, I, D, D]),
            "ref_loss_spec": (C.c_char_p, [C.c_void_p]),
            "ref_optimizer_spec": (C.c_char_p, [C.c_void_p]),
            "ref_snapshot_dump": (C.c_char_p, [C.c_void_p]),
            "ref_snapshot_load": (C.c_int, [C.c_void_p, C.c_char_p]),
            "ref_get_state": (None, [C.c_void_p, D, D, D, D, D, D, I, I, L, D, L]),
            "ref_set_state": (None, [C.c_void_p, D, D, D, D, D, D, I, I, L, D, L]),
            "ref_get_effector_state": (None, [C.c_void_p, D]),
            "ref_set_effector_state": (None, [C.c_void_p, D]),
            "ref_reset_state": (None, [C.c_void_p]),
            "ref_substep": (C.c_int, [C.c_void_p, D, C.c_int]),
            "ref_p2g_grid": (C.c_int, [C.c_void_p, D, D, D]),
            "ref_rollout_loss": (C.c_int, [C.c_void_p, C.c_int, C.c_int, D, C.c_long, D, D]),
            "ref_grad_trajectory": (C.c_int, [C.c_void_p, C.c_int, C.c_int, D, C.c_long, C.c_long, D, D, D, D, L]),
            "ref_adjoint_substep": (C.c_int, [C.c_void_p, D, D, D, D, D, D, D]),
            "ref_set_attraction": (None, [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double, D]),
            "ref_per_particle": (C.c_int, [C.c_void_p, D, D]),
            "ref_grad_check": (C.c_int, [C.c_void_p, C.c_int, C.c_int, D, C.c_long, C.c_double, C.c_int, D, D, L,
                                         D, D]),
            "ref_write_frame_csv": (C.c_int, [C.c_void_p, C.c_char_p, C.c_ulonglong]),
            "ref_write_metrics": (C.c_int, [C.c_void_p, C.c_char_p, C.c_ulonglong]),
            "ref_actions_json": (C.c_char_p, [C.c_int, C.c_int, D]),
        }
        for k, (r, a) in sig.items():
            f = getattr(l, k)
            f.restype = r
            f.argtypes = a
        _lib = l
    return _lib


def _p(a):
    if a is None:
        return None
    if a.dtype == np.float64:
        return a.ctypes.data_as(D)
    if a.dtype == np.int32:
        return a.ctypes.data_as(I)
    return a.ctypes.data_as(L)


class RefError(RuntimeError):
    def __init__(self, code, msg, pid, body, substep):
        super().__init__(f"[{code}] {msg}")
        self.code, self.particle_id, self.body_id, self.substep = code, pid, body, substep


class RefWorld:
    """build_scene<3> + a live SimState<3> in the reference engine."""

    def __init__(self, spec):
        self.l = lib()
        text = spec if isinstance(spec, str) else json.dumps(spec)
        h = C.c_void_p()
        self._check(self.l.ref_world_from_json(text.encode(), C.byref(h)))
        self.h = h
        self.n = self.l.ref_num_particles(h)
        self.n_eff = self.l.ref_num_effectors(h)

    def __del__(self):
        try:
            self.l.ref_world_free(self.h)
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            pid, body, sub = C.c_long(), C.c_long(), C.c_long()
            msg = self.l.ref_last_error(C.byref(pid), C.byref(body), C.byref(sub)).decode()
            raise RefError(rc, msg, pid.value, body.value, sub.value)

    def config(self):
        ints = np.zeros(8, np.int32)
        reals = np.zeros(12)
        self.l.ref_config(self.h, _p(ints), _p(reals))
        return {"res": int(ints[0]), "nd": tuple(int(v) for v in ints[1:4]), "bw": int(ints[4]),
                "hard": int(ints[5]), "dt": reals[0], "dx": reals[1], "domain": reals[2:5].copy(),
                "gravity": reals[5:8].copy(), "contact_eps": reals[8], "cfl": reals[9], "mass_eps": reals[10]}

    def state(self):
        n = self.n
        x, v = np.zeros((n, 3)), np.zeros((n, 3))
        F, Cm = np.zeros((n, 3, 3)), np.zeros((n, 3, 3))
        mass, vol0 = np.zeros(n), np.zeros(n)
        mat, body = np.zeros(n, np.int32), np.zeros(n, np.int32)
        act = np.zeros(n, np.int64)
        t, s = C.c_double(), C.c_long()
        self.l.ref_get_state(self.h, _p(x), _p(v), _p(F), _p(Cm), _p(mass), _p(vol0), _p(mat), _p(body), _p(act),
                             C.byref(t), C.byref(s))
        return {"x": x, "v": v, "F": F, "C": Cm, "mass": mass, "vol0": vol0, "material": mat, "body": body,
                "act": act, "time": t.value, "substep": s.value}

    def set_state(self, x=None, v=None, F=None, C_=None, substep=None, time=None):
        cv = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
        x, v, F, C_ = cv(x), cv(v), cv(F), cv(C_)
        s = C.c_long(substep) if substep is not None else None
        t = C.c_double(time) if time is not None else None
        self.l.ref_set_state(self.h, _p(x), _p(v), _p(F), _p(C_), None, None, None, None, None,
                             C.byref(t) if t is not None else None, C.byref(s) if s is not None else None)

    def effector_state(self):
        out = np.zeros((self.n_eff, 18))
        if self.n_eff:
            self.l.ref_get_effector_state(self.h, _p(out))
        return out

    def set_effector_state(self, e):
        e = np.ascontiguousarray(e, dtype=np.float64)
        if self.n_eff:
            self.l.ref_set_effector_state(self.h, _p(e))

    def set_gravity(self, g):
        self.l.ref_set_gravity(self.h, _p(np.asarray(g, dtype=np.float64)))

    def set_hard_contact(self, hard: bool):
        self.l.ref_set_hard_contact(self.h, int(hard))

    def reset(self):
        self.l.ref_reset_state(self.h)

    def substep(self, action, count=1):
        a = np.ascontiguousarray(action, dtype=np.float64)
        self._check(self.l.ref_substep(self.h, _p(a), int(count)))

    def p2g_grid(self):
        nd = self.config()["nd"]
        nn = nd[0] * nd[1] * nd[2]
        mass, mom, vel = np.zeros(nn), np.zeros(3 * nn), np.zeros(3 * nn)
        self._check(self.l.ref_p2g_grid(self.h, _p(mass), _p(mom), _p(vel)))
        return mass.reshape(nd), mom.reshape(nd + (3,)), vel.reshape(nd + (3,))

    def rollout_loss(self, values, seglen, window=0):
        values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1, 6)
        ns = values.shape[0]
        loss, per = C.c_double(), np.zeros(ns)
        self._check(self.l.ref_rollout_loss(self.h, ns, seglen, _p(values), window, C.byref(loss), _p(per)))
        return loss.value, per

    def grad_trajectory(self, values, seglen, stride=0, window=0):
        values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1, 6)
        ns = values.shape[0]
        g = np.zeros((ns, 6))
        loss, full, per, snaps = C.c_double(), C.c_double(), np.zeros(ns), C.c_long()
        self._check(self.l.ref_grad_trajectory(self.h, ns, seglen, _p(values), stride, window, _p(g),
                                               C.byref(loss), C.byref(full), _p(per), C.byref(snaps)))
        return {"grad": g, "loss": loss.value, "full_loss": full.value, "per_segment": per,
                "snapshots": snaps.value}

    def adjoint_substep(self, action, xb, vb, Fb, Cb, eff_bars=None, action_bar=None):
        a = np.ascontiguousarray(action, dtype=np.float64)
        xb, vb = np.array(xb, dtype=np.float64), np.array(vb, dtype=np.float64)
        Fb, Cb = np.array(Fb, dtype=np.float64), np.array(Cb, dtype=np.float64)
        eb = np.zeros((max(self.n_eff, 1), 12)) if eff_bars is None else np.array(eff_bars, dtype=np.float64)
        ab = np.zeros(6) if action_bar is None else np.array(action_bar, dtype=np.float64)
        self._check(self.l.ref_adjoint_substep(self.h, _p(a), _p(xb), _p(vb), _p(Fb), _p(Cb), _p(eb), _p(ab)))
        return xb, vb, Fb, Cb, eb, ab

    def set_attraction(self, body, weight, radius, tau, refresh_x=None):
        """enable_attraction + refresh_attraction(state with x = refresh_x) for later calls."""
        rx = None if refresh_x is None else np.ascontiguousarray(refresh_x, dtype=np.float64)
        self._att_keep = rx
        self.l.ref_set_attraction(self.h, int(body), float(weight), float(radius), float(tau), _p(rx))

    def per_particle(self, x=None):
        """LossEvaluator::per_particle of the live state (positions replaced by x if given)."""
        xs = None if x is None else np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(self.n)
        self._check(self.l.ref_per_particle(self.h, _p(xs), _p(out)))
        return out

    def grad_check(self, values, seglen, stride, eps, with_fd=True):
        """grad_check<3> (grad.hpp:190-225)."""
        values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1, 6)
        ns = values.shape[0]
        g, fd = np.zeros(ns * 6), np.zeros(ns * 6)
        n, mr, lo = C.c_long(), C.c_double(), C.c_double()
        self._check(self.l.ref_grad_check(self.h, ns, int(seglen), _p(values), int(stride), float(eps), int(with_fd),
                                          _p(g), _p(fd), C.byref(n), C.byref(mr), C.byref(lo)))
        k = n.value
        return {"gradient": g[:k], "fd_gradient": fd[:k] if with_fd else np.zeros(0), "max_rel_error": mr.value,
                "loss": lo.value}

    def write_frame_csv(self, path, manifest_hash):
        self._check(self.l.ref_write_frame_csv(self.h, str(path).encode(), int(manifest_hash)))

    def write_metrics(self, path, manifest_hash):
        """MetricsWriter<3> with one row for the live state."""
        self._check(self.l.ref_write_metrics(self.h, str(path).encode(), int(manifest_hash)))

    def actions_json(self, values, seglen):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1, 6)
        return json.loads(self.l.ref_actions_json(v.shape[0], int(seglen), _p(v)).decode())

    def loss_spec(self):
        return json.loads(self.l.ref_loss_spec(self.h).decode())

    def snapshot_dump(self) -> dict:
        """state_to_json<3> of the live state (io.hpp:144-190)."""
        return json.loads(self.l.ref_snapshot_dump(self.h).decode())

    def snapshot_load(self, snap: dict):
        """state_from_json<3> into the live state (io.hpp:192-240)."""
        if self.l.ref_snapshot_load(self.h, json.dumps(snap).encode()) != 0:
            raise RuntimeError("reference rejected the snapshot")

    def optimizer_spec(self):
        s = self.l.ref_optimizer_spec(self.h).decode()
        return json.loads(s) if s and s != "null" else {}

    def rigid_bodies(self):
        out = []
        for b in range(self.l.ref_num_rigid(self.h)):
            n = self.l.ref_rigid_members(self.h, b, None, None, None, None)
            mem = np.zeros(n, np.int64)
            rest = np.zeros((n, 3))
            bid, tm = C.c_int(), C.c_double()
            self.l.ref_rigid_members(self.h, b, _p(mem), _p(rest), C.byref(bid), C.byref(tm))
            out.append({"members": mem, "rest": rest, "body_id": bid.value, "total_mass": tm.value})
        return out

    def emitters(self):
        n = self.l.ref_num_emitters(self.h)
        p = np.zeros(n, np.int64)
        e = np.zeros(n, np.int32)
        lp, lv = np.zeros((n, 3)), np.zeros((n, 3))
        if n:
            self.l.ref_emitters(self.h, _p(p), _p(e), _p(lp), _p(lv))
        return {"particle": p, "effector": e, "local_pos": lp, "local_vel": lv}
