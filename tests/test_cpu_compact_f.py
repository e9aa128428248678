"""CPU checks of the algebra behind the compact liquid F (fl_layout.cuh f_compact).

For (viscous) liquids the return map sets F = det(F)^(1/3) I (materials.hpp:147-153),
so the CUDA path stores c (F = c I) and the cotangent dL/dc = tr(F_bar).  These
tests verify, in fp64 with the numpy restatement of the reference (oracle/restate.py)
and finite differences, the identities the kernels rely on:
  * liquid_project's VJP depends on tr(F_post_bar) only;
  * for F = c I, the P2G stress term's cotangent is 3 lambda c^2 (2J - 1) tr(s_bar)
    (J = c^3), i.e. the trace of the reference's corotated_stress VJP (mu = 0);
  * the G2P chain F_trial = (I + dt C) c I gives the same dL/dc through the full
    3x3 VJP and through the compact formula.
"""
import numpy as np

from oracle import restate

rng = np.random.default_rng(7)


def liquid_project(F):
    return np.cbrt(np.linalg.det(F)) * np.eye(3)


def num_grad(f, x, eps=1e-6):
    g = np.zeros_like(x)
    it = np.nditer(x, flags=["multi_index"])
    for _ in it:
        i = it.multi_index
        xp, xm = x.copy(), x.copy()
        xp[i] += eps
        xm[i] -= eps
        g[i] = (f(xp) - f(xm)) / (2 * eps)
    return g


def test_liquid_project_vjp_depends_on_trace_only():
    F = np.eye(3) + 0.05 * rng.standard_normal((3, 3))
    A = rng.standard_normal((3, 3))
    B = A - np.trace(A) / 3 * np.eye(3) + np.trace(A) / 3 * np.eye(3)  # same trace
    B = B + np.array([[0, 1, 0], [-1, 0, 2], [0, -2, 0.0]])            # traceless change
    ga = num_grad(lambda f: np.sum(liquid_project(f) * A), F)
    gb = num_grad(lambda f: np.sum(liquid_project(f) * B), F)
    np.testing.assert_allclose(ga, gb, rtol=1e-7, atol=1e-9)
    # and the closed form used by liquid_project_vjp_c: cofactor(F) * tr(A) cbrt(J) / (3 J)
    J = np.linalg.det(F)
    cof = J * np.linalg.inv(F).T
    np.testing.assert_allclose(ga, cof * np.trace(A) * np.cbrt(J) / (3 * J), rtol=1e-6, atol=1e-9)


def test_pressure_stress_cotangent_for_isotropic_F():
    lam = 7.5
    for c in (0.93, 1.0, 1.07):
        s_bar = rng.standard_normal((3, 3))

        def stress_mat(cc):
            F = cc * np.eye(3)
            P, _ = restate.corotated_stress(F[None], np.array([0.0]), np.array([lam]))
            return np.sum((P[0] @ F.T) * s_bar)

        d = (stress_mat(c + 1e-6) - stress_mat(c - 1e-6)) / 2e-6
        J = c ** 3
        np.testing.assert_allclose(d, 3 * lam * c * c * (2 * J - 1) * np.trace(s_bar), rtol=1e-7)


def test_g2p_chain_compact_equals_full():
    dt = 1e-4
    C = rng.standard_normal((3, 3)) * 50
    c = 1.03
    Fpost_bar = rng.standard_normal((3, 3))

    def loss_c(cc):
        return np.sum(liquid_project((np.eye(3) + dt * C) @ (cc * np.eye(3))) * Fpost_bar)

    dc = (loss_c(c + 1e-7) - loss_c(c - 1e-7)) / 2e-7
    # compact path: F_trial_bar from tr(F_post_bar), then dL/dc = tr(ipc^T F_trial_bar)
    ipc = np.eye(3) + dt * C
    ftr = ipc * c
    J = np.linalg.det(ftr)
    ftr_bar = J * np.linalg.inv(ftr).T * (np.trace(Fpost_bar) * np.cbrt(J) / (3 * J))
    np.testing.assert_allclose(np.trace(ipc.T @ ftr_bar), dc, rtol=1e-6)
