"""oracle/restate.py -- TEST INFRASTRUCTURE ONLY: a CPU restatement of the hot path.

A vectorised numpy (fp64) restatement of one MLS-MPM substep of the reference
engine, written from its behaviour (it is not linked into, or called by, the
product).  It is pinned against the unmodified reference (oracle/_ref) and
the committed golden vectors in tests/golden/ by tests/test_oracle.py; the
GPU parity tests use it (and oracle/_ref) as the checker.

Functions and the reference code they restate (all paths under /root/reference):
  quad_weights            proj/include/flume/mpm.hpp:55-71
  svd3 (one-sided Jacobi) proj/include/flume/svd.hpp:16-120
  polar_rotation          proj/include/flume/svd.hpp:130-134
  corotated_stress        proj/include/flume/materials.hpp:20-32
  box_yield_project       proj/include/flume/materials.hpp:55-63
  von_mises_project       proj/include/flume/materials.hpp:81-104
  liquid_project          proj/include/flume/materials.hpp:149-153
  sdf_eval (5 primitives) proj/include/flume/sdf.hpp:75-211, 307-315
  coulomb_project         proj/include/flume/mpm.hpp:79-87
  effector_contact        proj/include/flume/mpm.hpp:146-161
  p2g                     proj/include/flume/mpm.hpp:249-287
  grid_update             proj/include/flume/mpm.hpp:289-320
  g2p                     proj/include/flume/mpm.hpp:322-384
  rigid_body_pass         proj/include/flume/mpm.hpp:386-416, materials.hpp:171-202
  advance_effectors       proj/include/flume/mpm.hpp:418-433, core.hpp:380-433
  activate_emitted        proj/include/flume/mpm.hpp:435-449
  mpm_substep             proj/include/flume/mpm.hpp:455-473
  target_point loss       proj/include/flume/losses.hpp:66-76, 474-516
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# MaterialKind / ShapeKind numbering (types.hpp:12, sdf.hpp:24)
ELASTIC, PLASTIC, LIQUID, VISCOUS, NONNEWTONIAN, RIGID = range(6)
SPHERE, BOX, CAPSULE, CYLINDER, HALFSPACE = range(5)


# ---------------------------------------------------------------------------
# small linear algebra (batched over a leading axis)
# ---------------------------------------------------------------------------

def det3(a):
    return (a[..., 0, 0] * (a[..., 1, 1] * a[..., 2, 2] - a[..., 1, 2] * a[..., 2, 1])
            - a[..., 0, 1] * (a[..., 1, 0] * a[..., 2, 2] - a[..., 1, 2] * a[..., 2, 0])
            + a[..., 0, 2] * (a[..., 1, 0] * a[..., 2, 1] - a[..., 1, 1] * a[..., 2, 0]))


def cofactor3(a):
    """det(A) A^{-T} (core.hpp:324-336)."""
    c = np.empty_like(a)
    c[..., 0, 0] = a[..., 1, 1] * a[..., 2, 2] - a[..., 1, 2] * a[..., 2, 1]
    c[..., 0, 1] = a[..., 1, 2] * a[..., 2, 0] - a[..., 1, 0] * a[..., 2, 2]
    c[..., 0, 2] = a[..., 1, 0] * a[..., 2, 1] - a[..., 1, 1] * a[..., 2, 0]
    c[..., 1, 0] = a[..., 0, 2] * a[..., 2, 1] - a[..., 0, 1] * a[..., 2, 2]
    c[..., 1, 1] = a[..., 0, 0] * a[..., 2, 2] - a[..., 0, 2] * a[..., 2, 0]
    c[..., 1, 2] = a[..., 0, 1] * a[..., 2, 0] - a[..., 0, 0] * a[..., 2, 1]
    c[..., 2, 0] = a[..., 0, 1] * a[..., 1, 2] - a[..., 0, 2] * a[..., 1, 1]
    c[..., 2, 1] = a[..., 0, 2] * a[..., 1, 0] - a[..., 0, 0] * a[..., 1, 2]
    c[..., 2, 2] = a[..., 0, 0] * a[..., 1, 1] - a[..., 0, 1] * a[..., 1, 0]
    return c


def skew(w):
    k = np.zeros(w.shape[:-1] + (3, 3))
    k[..., 0, 1], k[..., 0, 2] = -w[..., 2], w[..., 1]
    k[..., 1, 0], k[..., 1, 2] = w[..., 2], -w[..., 0]
    k[..., 2, 0], k[..., 2, 1] = -w[..., 1], w[..., 0]
    return k


def exp_so3(w):
    """Rodrigues (core.hpp:380-392)."""
    w = np.asarray(w, dtype=np.float64)
    th = np.sqrt(np.sum(w * w))
    k = skew(w)
    if th < 1e-8:
        a, b = 1 - th * th / 6, 0.5 - th * th / 24
    else:
        a, b = np.sin(th) / th, (1 - np.cos(th)) / (th * th)
    return np.eye(3) + a * k + b * (k @ k)


def svd3(a, sweeps=30, tol=1e-15):
    """One-sided Jacobi SVD, sigma descending, det(U)=+1 (svd.hpp:16-120), batched."""
    a = np.asarray(a, dtype=np.float64)
    shp = a.shape[:-2]
    b = a.reshape(-1, 3, 3).copy()
    n = b.shape[0]
    v = np.tile(np.eye(3), (n, 1, 1))
    live = np.ones(n, dtype=bool)
    for _ in range(sweeps):
        if not live.any():
            break
        off = np.zeros(n)
        for p, q in ((0, 1), (0, 2), (1, 2)):
            bp, bq = b[:, :, p], b[:, :, q]
            apq = np.sum(bp * bq, axis=1)
            app = np.sum(bp * bp, axis=1)
            aqq = np.sum(bq * bq, axis=1)
            off = np.maximum(off, np.abs(apq) / (np.sqrt(app * aqq) + 1e-300))
            rot = live & (np.abs(apq) >= 1e-300)
            with np.errstate(divide="ignore", invalid="ignore"):
                tau = np.where(rot, (aqq - app) / (2 * np.where(rot, apq, 1.0)), 0.0)
                t = np.where(tau >= 0, 1.0, -1.0) / (np.abs(tau) + np.sqrt(1 + tau * tau))
            c = 1 / np.sqrt(1 + t * t)
            s = c * t
            c = np.where(rot, c, 1.0)[:, None]
            s = np.where(rot, s, 0.0)[:, None]
            nbp, nbq = c * bp - s * bq, s * bp + c * bq
            b[:, :, p], b[:, :, q] = nbp, nbq
            vp, vq = v[:, :, p].copy(), v[:, :, q].copy()
            v[:, :, p], v[:, :, q] = c * vp - s * vq, s * vp + c * vq
        live &= off >= tol
    sig = np.sqrt(np.sum(b * b, axis=1))
    order = np.argsort(-sig, axis=1, kind="stable")
    idx = np.arange(n)[:, None]
    sig_s = sig[idx, order]
    rows = np.arange(3)[None, :, None]
    V = v[idx[:, :, None], rows, order[:, None, :]]
    B = b[idx[:, :, None], rows, order[:, None, :]]
    with np.errstate(divide="ignore", invalid="ignore"):
        U = np.where(sig_s[:, None, :] > 1e-150, B / sig_s[:, None, :], 0.0)
    # (null-column rebuild of svd.hpp:88-106 is not needed by the scenes restated here)
    flip = det3(U) < 0
    U[flip, :, 2] *= -1
    V[flip, :, 2] *= -1
    return U.reshape(shp + (3, 3)), sig_s.reshape(shp + (3,)), V.reshape(shp + (3, 3))


def polar_rotation(a):
    U, _, V = svd3(a)
    return U @ np.swapaxes(V, -1, -2)


# ---------------------------------------------------------------------------
# constitutive models (materials.hpp)
# ---------------------------------------------------------------------------

def corotated_stress(F, mu, lam):
    J = det3(F)
    P = cofactor3(F) * (lam * (J - 1))[..., None, None]
    mu = np.broadcast_to(np.asarray(mu, dtype=np.float64), J.shape)
    nz = mu != 0
    if nz.any():
        R = polar_rotation(F[nz])
        P[nz] += (F[nz] - R) * (2 * mu[nz])[..., None, None]
    return P, J


def liquid_project(F):
    J = det3(F)
    return np.eye(3) * np.power(J, 1.0 / 3.0)[..., None, None], J


def box_yield_project(F, tc, ts):
    U, s, V = svd3(F)
    s = np.minimum(np.maximum(s, 1 - tc), 1 + ts)
    return (U * s[..., None, :]) @ np.swapaxes(V, -1, -2), det3(F)


def von_mises_project(F, sigma_y, mu):
    U, s, V = svd3(F)
    eps = np.log(s)
    mean = eps.sum(-1) / 3
    dev = eps - mean[..., None]
    dn = np.sqrt(np.sum(dev * dev, axis=-1))
    yield_ = 2 * mu * dn > sigma_y
    out = F.copy()
    if yield_.any():
        scale = sigma_y / (2 * mu * dn[yield_])
        s2 = np.exp(mean[yield_, None] + scale[:, None] * dev[yield_])
        out[yield_] = (U[yield_] * s2[:, None, :]) @ np.swapaxes(V[yield_], -1, -2)
    return out, s.min(-1)


# ---------------------------------------------------------------------------
# SDF primitives and contact (sdf.hpp, mpm.hpp:79-161)
# ---------------------------------------------------------------------------

def sdf_local(shape, q):
    k = shape["kind"]
    if k == SPHERE:
        n = np.linalg.norm(q, axis=-1)
        g = np.where(n[:, None] < 1e-12, np.array([1.0, 0, 0]), q / np.maximum(n, 1e-300)[:, None])
        return n - shape["radius"], g
    if k == BOX:
        h = np.asarray(shape["half"])
        a = np.abs(q) - h
        inside = a.max(-1)
        m = np.maximum(a, 0)
        out = np.sqrt(np.sum(m * m, -1))
        d = np.where(inside <= 0, inside, out)
        sgn = np.where(q >= 0, 1.0, -1.0)
        kk = np.argmax(a, axis=-1)
        gin = np.zeros_like(q)
        gin[np.arange(len(q)), kk] = sgn[np.arange(len(q)), kk]
        mn = np.linalg.norm(m, axis=-1)
        gout = np.where(mn[:, None] < 1e-12, np.array([1.0, 0, 0]), sgn * m / np.maximum(mn, 1e-300)[:, None])
        g = np.where((inside <= 0)[:, None], gin, gout)
        return d, g
    if k == CAPSULE:
        a_, b_ = np.asarray(shape["seg_a"]), np.asarray(shape["seg_b"])
        u = b_ - a_
        uu = u @ u
        t = np.clip((q - a_) @ u / uu, 0, 1) if uu > 0 else np.zeros(len(q))
        e = q - (a_ + t[:, None] * u)
        n = np.linalg.norm(e, axis=-1)
        g = np.where(n[:, None] < 1e-12, np.array([1.0, 0, 0]), e / np.maximum(n, 1e-300)[:, None])
        return n - shape["radius"], g
    if k == CYLINDER:
        rho = np.sqrt(q[:, 0] ** 2 + q[:, 1] ** 2)
        y1 = rho - shape["radius"]
        y2 = np.abs(q[:, 2]) - shape["half_height"]
        d = np.minimum(np.maximum(y1, y2), 0) + np.sqrt(np.maximum(y1, 0) ** 2 + np.maximum(y2, 0) ** 2)
        sz = np.where(q[:, 2] >= 0, 1.0, -1.0)
        radial = np.where((rho > 1e-12)[:, None],
                          np.stack([q[:, 0] / np.maximum(rho, 1e-300), q[:, 1] / np.maximum(rho, 1e-300),
                                    np.zeros_like(rho)], -1), np.array([1.0, 0, 0]))
        axial = np.stack([np.zeros_like(sz), np.zeros_like(sz), sz], -1)
        phi = np.sqrt(y1 * y1 + y2 * y2)
        corner = radial * (y1 / np.maximum(phi, 1e-300))[:, None] + axial * (y2 / np.maximum(phi, 1e-300))[:, None]
        corner = np.where((phi < 1e-12)[:, None], np.array([1.0, 0, 0]), corner)
        g = np.where(((y1 <= 0) & (y2 <= 0))[:, None], np.where((y1 > y2)[:, None], radial, axial),
                     np.where(((y1 > 0) & (y2 <= 0))[:, None], radial,
                              np.where(((y1 <= 0) & (y2 > 0))[:, None], axial, corner)))
        return d, g
    n = np.asarray(shape["normal"])
    return q @ n - shape["offset"], np.tile(n, (len(q), 1))


def sdf_eval(shape, wt, wR, p):
    q = (p - wt) @ wR  # R^T (p - t)
    d, g = sdf_local(shape, q)
    ng = g @ wR.T
    nn = np.linalg.norm(ng, axis=-1)
    n = np.where((nn < 1e-30)[:, None], np.array([1.0, 0, 0]), ng / np.maximum(nn, 1e-300)[:, None])
    return d, n


def coulomb_project(vrel, n, mu):
    vn = np.sum(vrel * n, -1)
    vt = vrel - n * vn[:, None]
    tn = np.linalg.norm(vt, axis=-1)
    with np.errstate(divide="ignore", invalid="ignore"):
        slide = vt * (1 + mu * vn / tn)[:, None]
    out = np.where((vn >= 0)[:, None], vrel, np.where((tn <= mu * (-vn))[:, None], 0.0, slide))
    return out


def effector_contact(eff, p, v, dx, eps_cells, hard):
    wt = eff["pose_t"] + eff["pose_R"] @ eff["shape_t"]
    wR = eff["pose_R"] @ eff["shape_R"]
    d, n = sdf_eval(eff["shape"], wt, wR, p)
    d = d / dx
    act = d < eps_cells
    if not act.any():
        return v
    r = p - eff["pose_t"]
    ve = eff["vlin"] + np.cross(eff["wang"], r)
    vrel = v - ve
    vp = np.zeros_like(vrel) if np.isinf(eff["mu"]) else coulomb_project(vrel, n, eff["mu"])
    vc = vp + ve
    if hard:
        a = np.where(d <= 0, 1.0, 0.0)
    else:
        a = np.where(d <= 0, 1.0, np.exp(-np.maximum(d, 0)))
    out = vc * a[:, None] + v * (1 - a)[:, None]
    return np.where(act[:, None], out, v)


# ---------------------------------------------------------------------------
# scene / state containers
# ---------------------------------------------------------------------------

@dataclass
class Scene:
    res: int
    nd: tuple
    dx: float
    dt: float
    domain: np.ndarray
    gravity: np.ndarray
    bw: int = 3
    eps_cells: float = 3.0
    cfl: float = 0.9
    mass_eps: float = 1e-12
    hard: bool = False
    materials: list = field(default_factory=list)  # dicts: kind, mu, lam, tc, ts, sy
    rigid: list = field(default_factory=list)  # dicts: members, rest, body_id
    emitters: dict = None  # particle, effector, local_pos, local_vel
    effector_shapes: list = field(default_factory=list)  # dicts: shape, shape_t, shape_R, mu, mask
    mass: np.ndarray = None
    vol0: np.ndarray = None
    mat: np.ndarray = None
    act: np.ndarray = None


@dataclass
class State:
    x: np.ndarray
    v: np.ndarray
    F: np.ndarray
    C: np.ndarray
    eff: list  # dicts: pose_t, pose_R, vlin, wang
    substep: int = 0
    time: float = 0.0

    def copy(self):
        return State(self.x.copy(), self.v.copy(), self.F.copy(), self.C.copy(),
                     [{k: np.array(v, copy=True) for k, v in e.items()} for e in self.eff], self.substep, self.time)


# ---------------------------------------------------------------------------
# the substep
# ---------------------------------------------------------------------------

def quad_weights(x, inv_dx):
    xs = x * inv_dx
    base = np.floor(xs - 0.5).astype(np.int64)
    fx = xs - base
    w = np.stack([0.5 * (1.5 - fx) ** 2, 0.75 - (fx - 1) ** 2, 0.5 * (fx - 0.5) ** 2], 0)  # (3, N, 3)
    return base, fx, w


class EscapeError(RuntimeError):
    pass


class DegenerateError(RuntimeError):
    def __init__(self, pid):
        super().__init__(f"degenerate deformation at particle {pid}")
        self.particle_id = pid


def _kinds(sc, idx):
    return np.array([sc.materials[m]["kind"] for m in sc.mat[idx]])


def p2g(sc: Scene, st: State):
    act = sc.act <= st.substep
    idx = np.nonzero(act)[0]
    x, v, F, C = st.x[idx], st.v[idx], st.F[idx], st.C[idx]
    inv_dx = 1.0 / sc.dx
    base, fx, w = quad_weights(x, inv_dx)
    bad = np.any((base < 0) | (base + 2 >= np.array(sc.nd)), axis=1)
    if bad.any():
        raise EscapeError(f"p2g: particle {idx[np.argmax(bad)]} escaped the clamped region")
    mats = sc.mat[idx]
    mu = np.array([sc.materials[m]["mu"] for m in mats])
    lam = np.array([sc.materials[m]["lam"] for m in mats])
    visc = _kinds(sc, idx) == VISCOUS
    Fs = F.copy()
    if visc.any():
        Fs[visc] = (np.eye(3) + C[visc] * sc.dt) @ F[visc]
    P, J = corotated_stress(Fs, mu, lam)
    if (J <= 0).any():
        raise DegenerateError(int(idx[np.argmax(J <= 0)]))
    smat = P @ np.swapaxes(Fs, -1, -2)
    m = sc.mass[idx]
    coeff = sc.dt * 4 * inv_dx * inv_dx
    affine = C * m[:, None, None] - smat * (coeff * sc.vol0[idx])[:, None, None]
    mass = np.zeros(sc.nd)
    mom = np.zeros(sc.nd + (3,))
    for ox in range(3):
        for oy in range(3):
            for oz in range(3):
                o = np.array([ox, oy, oz])
                wt = w[ox, :, 0] * w[oy, :, 1] * w[oz, :, 2]
                node = base + o
                rel = node * sc.dx - x
                contrib = v * m[:, None] + np.einsum("nij,nj->ni", affine, rel)
                np.add.at(mass, (node[:, 0], node[:, 1], node[:, 2]), wt * m)
                np.add.at(mom, (node[:, 0], node[:, 1], node[:, 2]), contrib * wt[:, None])
    return mass, mom


def grid_update(sc: Scene, st: State, mass, mom):
    vel = np.zeros_like(mom)
    ii = np.argwhere(mass > sc.mass_eps)
    m = mass[tuple(ii.T)]
    v = mom[tuple(ii.T)] / m[:, None] + sc.gravity * sc.dt
    nd = np.array(sc.nd)
    lo = ii <= sc.bw
    hi = ii >= nd - 1 - sc.bw
    v = np.where(lo & (v < 0), 0.0, v)
    v = np.where(hi & (v > 0), 0.0, v)
    p = ii * sc.dx
    for e, sh in zip(st.eff, sc.effector_shapes):
        eff = {**sh, **e}
        v = effector_contact(eff, p, v, sc.dx, sc.eps_cells, sc.hard)
    vel[tuple(ii.T)] = v
    return vel


def g2p(sc: Scene, st: State, vel):
    act = sc.act <= st.substep
    idx = np.nonzero(act)[0]
    x, F = st.x[idx], st.F[idx]
    inv_dx = 1.0 / sc.dx
    k4 = 4 * inv_dx * inv_dx
    base, fx, w = quad_weights(x, inv_dx)
    vnew = np.zeros_like(x)
    cnew = np.zeros_like(F)
    for ox in range(3):
        for oy in range(3):
            for oz in range(3):
                o = np.array([ox, oy, oz])
                wt = w[ox, :, 0] * w[oy, :, 1] * w[oz, :, 2]
                node = base + o
                gv = vel[node[:, 0], node[:, 1], node[:, 2]]
                rel = node * sc.dx - x
                vnew += gv * wt[:, None]
                cnew += np.einsum("ni,nj->nij", gv, rel) * (wt * k4)[:, None, None]
    vmax = sc.cfl * sc.dx / sc.dt
    vn = np.linalg.norm(vnew, axis=1)
    vnew = np.where((vn > vmax)[:, None], vnew * (vmax / np.maximum(vn, 1e-300))[:, None], vnew)
    xn = np.clip(x + vnew * sc.dt, sc.dx, sc.domain - sc.dx)
    ftr = (np.eye(3) + cnew * sc.dt) @ F
    kinds = _kinds(sc, idx)
    fnew = ftr.copy()
    for kind in np.unique(kinds):
        sel = kinds == kind
        mats = sc.mat[idx[sel]]
        if kind in (LIQUID, VISCOUS):
            fnew[sel], J = liquid_project(ftr[sel])
            bad = J <= 0
        elif kind == PLASTIC:
            tc = np.array([sc.materials[mm]["tc"] for mm in mats])[:, None]
            ts = np.array([sc.materials[mm]["ts"] for mm in mats])[:, None]
            fnew[sel], J = box_yield_project(ftr[sel], tc, ts)
            bad = J <= 0
        elif kind == NONNEWTONIAN:
            sy = np.array([sc.materials[mm]["sy"] for mm in mats])
            mu = np.array([sc.materials[mm]["mu"] for mm in mats])
            fnew[sel], smin = von_mises_project(ftr[sel], sy, mu)
            bad = smin <= 0
        else:
            continue
        if bad.any():
            raise DegenerateError(int(idx[sel][np.argmax(bad)]))
    out = st.copy()
    out.x[idx], out.v[idx], out.C[idx], out.F[idx] = xn, vnew, cnew, fnew
    return out


def rigid_body_pass(sc: Scene, st: State, start_x):
    for body in sc.rigid:
        mem = body["members"]
        if not np.all(sc.act[mem] <= st.substep):
            continue
        x = st.x[mem]
        m = sc.mass[mem]
        total = m.sum()
        c = (x * m[:, None]).sum(0) / total
        A = np.einsum("ni,nj->ij", (x - c) * m[:, None], body["rest"])
        U, s, V = svd3(A)
        if s[1] < 1e-12 * max(s[0], 1e-30):
            raise RuntimeError(f"rigid_shape_match: degenerate covariance (body {body['body_id']})")
        R = U @ V.T
        if det3(A) < 0:
            R = U @ np.diag([1.0, 1.0, -1.0]) @ V.T
        xn = np.clip(body["rest"] @ R.T + c, sc.dx, sc.domain - sc.dx)
        st.v[mem] = (xn - start_x[mem]) / sc.dt
        st.x[mem] = xn


def advance_effectors(sc: Scene, st: State, action):
    for e, sh in zip(st.eff, sc.effector_shapes):
        mask = sh["mask"]
        for a in range(3):
            if mask[a]:
                e["vlin"][a] = action[a]
            if mask[3 + a]:
                e["wang"][a] = action[3 + a]
        e["pose_t"] = e["pose_t"] + e["vlin"] * sc.dt
        e["pose_R"] = exp_so3(e["wang"] * sc.dt) @ e["pose_R"]


def activate_emitted(sc: Scene, st: State):
    em = sc.emitters
    if em is None or len(em["particle"]) == 0:
        return
    for k, pid in enumerate(em["particle"]):
        if sc.act[pid] != st.substep:
            continue
        e = em["effector"][k]
        if e >= 0:
            eff = st.eff[e]
            st.x[pid] = np.clip(eff["pose_R"] @ em["local_pos"][k] + eff["pose_t"], sc.dx, sc.domain - sc.dx)
            st.v[pid] = eff["pose_R"] @ em["local_vel"][k]
        else:
            st.x[pid] = np.clip(em["local_pos"][k], sc.dx, sc.domain - sc.dx)
            st.v[pid] = em["local_vel"][k]


def mpm_substep(sc: Scene, st: State, action) -> State:
    st = st.copy()
    advance_effectors(sc, st, np.asarray(action, dtype=np.float64))
    activate_emitted(sc, st)
    start = st.x.copy()
    mass, mom = p2g(sc, st)
    vel = grid_update(sc, st, mass, mom)
    out = g2p(sc, st, vel)
    rigid_body_pass(sc, out, start)
    out.substep = st.substep + 1
    out.time = st.time + sc.dt
    return out


def target_point_loss(sc: Scene, st: State, body_ids, body, goal, squared=False):
    sel = (body_ids == body) & (sc.act <= st.substep)
    d = np.linalg.norm(st.x[sel] - np.asarray(goal), axis=1)
    return float(np.sum(d * d if squared else d))


# ---------------------------------------------------------------------------
# construction from the reference engine (scene data is input, not restated)
# ---------------------------------------------------------------------------

def from_ref(rw) -> tuple[Scene, State, np.ndarray]:
    """Scene + initial state + body ids from an oracle.ref.RefWorld."""
    import ctypes as C

    from oracle import ref as _ref

    cfg = rw.config()
    st = rw.state()
    nmat = rw.l.ref_num_materials(rw.h)
    mats = np.zeros((max(nmat, 1), 7))
    rw.l.ref_materials(rw.h, mats.ctypes.data_as(_ref.D))
    materials = [{"kind": int(r[0]), "mu": r[1], "lam": r[2], "tc": r[4], "ts": r[5], "sy": r[6]} for r in mats[:nmat]]
    ne = rw.n_eff
    eff_raw = np.zeros((max(ne, 1), 64))
    if ne:
        rw.l.ref_effectors(rw.h, eff_raw.ctypes.data_as(_ref.D))
    shapes, effs = [], []
    for e in eff_raw[:ne]:
        shape = {"kind": int(e[0]), "radius": e[1], "half": e[2:5], "seg_a": e[5:8], "seg_b": e[8:11],
                 "normal": e[11:14], "offset": e[14], "half_height": e[15]}
        shapes.append({"shape": shape, "shape_t": e[16:19].copy(), "shape_R": e[19:28].reshape(3, 3).copy(),
                       "mu": e[46], "mask": e[47:53] != 0})
        effs.append({"pose_t": e[28:31].copy(), "pose_R": e[31:40].reshape(3, 3).copy(), "vlin": e[40:43].copy(),
                     "wang": e[43:46].copy()})
    rigid = [{"members": b["members"], "rest": b["rest"], "body_id": b["body_id"]} for b in rw.rigid_bodies()]
    em = rw.emitters()
    sc = Scene(res=cfg["res"], nd=cfg["nd"], dx=cfg["dx"], dt=cfg["dt"], domain=cfg["domain"],
               gravity=cfg["gravity"], bw=cfg["bw"], eps_cells=cfg["contact_eps"], cfl=cfg["cfl"],
               mass_eps=cfg["mass_eps"], hard=bool(cfg["hard"]), materials=materials, rigid=rigid, emitters=em,
               effector_shapes=shapes, mass=st["mass"], vol0=st["vol0"], mat=st["material"], act=st["act"])
    state = State(st["x"], st["v"], st["F"], st["C"], effs, st["substep"], st["time"])
    del C
    return sc, state, st["body"]
