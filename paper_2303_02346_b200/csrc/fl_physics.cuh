// fl_physics.cuh -- per-node contact and per-particle constitutive kernels.
//
//   coulomb_project(_vjp), contact_alpha(_deriv), effector_contact(_vjp)
//       restate proj/include/flume/mpm.hpp:79-217
//   corotated_stress(_vjp), box_yield_project(_vjp), von_mises_project(_vjp),
//   liquid_project(_vjp)
//       restate proj/include/flume/materials.hpp:20-161
// Everything is templated on the scalar; the kernels instantiate fp32.
#pragma once

#include "fl_sdf.cuh"

namespace fl {

// MaterialKind numbering (types.hpp:12)
enum MatKindId : int { MK_ELASTIC = 0, MK_PLASTIC = 1, MK_LIQUID = 2, MK_VISCOUS = 3, MK_NONNEWTONIAN = 4, MK_RIGID = 5 };

// A kinematic effector at one substep (stage-a pose), ready for node contact.
template <class T>
struct EffK {
    ShapeP<T> shape;
    V3<T> wt;   // world shape pose = compose(pose, sdf.pose)  (types.hpp:124)
    M3<T> wR;
    V3<T> pt;   // effector pose translation (contact lever arm, mpm.hpp:154)
    M3<T> shapeR;  // sdf.pose.R (for the R_bar chain, mpm.hpp:215)
    V3<T> shapet;  // sdf.pose.t
    V3<T> vlin;
    V3<T> wang;
    T mu;
    int sticky;
};

template <class T>
FL_HD V3<T> coulomb_project(V3<T> v_rel, V3<T> n, T mu) {
    T vn = dot(v_rel, n);
    if (vn >= T(0)) return v_rel;
    V3<T> vt = v_rel - n * vn;
    T tn = norm(vt);
    if (tn <= mu * (-vn)) return v3zero<T>();
    return vt * (T(1) + mu * vn / tn);
}

template <class T>
FL_HD void coulomb_project_vjp(V3<T> v_rel, V3<T> n, T mu, V3<T> out_bar, V3<T>& v_rel_bar, V3<T>& n_bar) {
    T vn = dot(v_rel, n);
    if (vn >= T(0)) {
        v_rel_bar += out_bar;
        return;
    }
    V3<T> vt = v_rel - n * vn;
    T tn = norm(vt);
    if (tn <= mu * (-vn)) return;
    T c = T(1) + mu * vn / tn;
    V3<T> th = vt * (T(1) / tn);
    T c_bar = dot(out_bar, vt);
    V3<T> vt_bar = out_bar * c;
    T vn_bar = mu * c_bar / tn;
    T tn_bar = -mu * vn * c_bar / (tn * tn);
    vt_bar += th * tn_bar;
    v_rel_bar += vt_bar;
    vn_bar += -dot(vt_bar, n);
    n_bar += vt_bar * (-vn);
    v_rel_bar += n * vn_bar;
    n_bar += v_rel * vn_bar;
}

template <class T> FL_HD T contact_alpha(T d, bool hard) {
    if (hard) return d <= T(0) ? T(1) : T(0);
    return d <= T(0) ? T(1) : exp(-d);
}
template <class T> FL_HD T contact_alpha_deriv(T d, bool hard) {
    if (hard || d <= T(0)) return T(0);
    return -exp(-d);
}

// mpm.hpp:146-161
template <class T>
FL_HD V3<T> effector_contact(const EffK<T>& e, T inv_dx, T eps_cells, bool hard, V3<T> p, V3<T> v_in,
                             bool* hit = nullptr) {
    // sdf_eval split: the normal is only needed inside the contact band, and most
    // nodes are far from every effector (same values as sdf_eval where it is used)
    const V3<T> q = tmul(e.wR, p - e.wt);
    T d = sdf_local_distance(e.shape, q) * inv_dx;
    if (hit) *hit = d < eps_cells;
    if (d >= eps_cells) return v_in;
    SdfSample<T> s;
    s.normal = normalized_or_x(e.wR * sdf_local_grad(e.shape, q), T(1e-30));
    V3<T> r = p - e.pt;
    V3<T> ve = e.vlin + cross(e.wang, r);
    V3<T> vrel = v_in - ve;
    V3<T> vrel_p = e.sticky ? v3zero<T>() : coulomb_project(vrel, s.normal, e.mu);
    V3<T> vc = vrel_p + ve;
    T a = contact_alpha(d, hard);
    return vc * a + v_in * (T(1) - a);
}

// Per-effector cotangents accumulated over nodes (mpm.hpp:137-143): t, R, vlin, w
template <class T>
struct EffBars {
    V3<T> t;
    M3<T> R;
    V3<T> vlin;
    V3<T> w;
};

// mpm.hpp:163-217.  Returns true when the node is inside the contact band
// (only then are effector bars touched).
template <class T>
FL_HD bool effector_contact_vjp(const EffK<T>& e, T dx, T inv_dx, T eps_cells, bool hard, V3<T> p, V3<T> v_in,
                                V3<T> out_bar, V3<T>& v_in_bar, EffBars<T>& eb) {
    SdfSample<T> s = sdf_eval(e.shape, e.wt, e.wR, p);
    T d = s.distance * inv_dx;
    if (d >= eps_cells) {
        v_in_bar += out_bar;
        return false;
    }
    V3<T> r = p - e.pt;
    V3<T> ve = e.vlin + cross(e.wang, r);
    V3<T> vrel = v_in - ve;
    V3<T> vrel_p = e.sticky ? v3zero<T>() : coulomb_project(vrel, s.normal, e.mu);
    V3<T> vc = vrel_p + ve;
    T a = contact_alpha(d, hard);
    T a_bar = dot(out_bar, vc - v_in);
    V3<T> vc_bar = out_bar * a;
    v_in_bar += out_bar * (T(1) - a);
    T d_bar = contact_alpha_deriv(d, hard) * a_bar;
    V3<T> ve_bar = vc_bar;
    V3<T> vrel_bar = v3zero<T>(), n_bar = v3zero<T>();
    if (!e.sticky) coulomb_project_vjp(vrel, s.normal, e.mu, vc_bar, vrel_bar, n_bar);
    v_in_bar += vrel_bar;
    ve_bar -= vrel_bar;
    eb.vlin += ve_bar;
    eb.w += cross(r, ve_bar);
    eb.t += cross(e.wang, ve_bar);
    V3<T> wt_bar = v3zero<T>();
    M3<T> wR_bar = mzero<T>();
    sdf_eval_pose_vjp(e.shape, e.wt, e.wR, p, d_bar / dx, n_bar, wt_bar, wR_bar);
    eb.t += wt_bar;
    eb.R += wR_bar * transpose(e.shapeR);
    eb.R += outer(wt_bar, e.shapet);
    return true;
}

// ---------------------------------------------------------------------------
// Constitutive models
// ---------------------------------------------------------------------------

// P(F) = 2 mu (F - R) + lambda (J - 1) cofactor(F); ok=false when J <= 0.
template <class T>
FL_HD M3<T> corotated_stress(const M3<T>& f, T mu, T lambda, bool& ok) {
    T j = det(f);
    ok = j > T(0);
    M3<T> p = cofactor(f) * (lambda * (j - T(1)));
    if (mu != T(0)) {
        M3<T> r = polar_R(svd3(f));
        p += (f - r) * (T(2) * mu);
    }
    return p;
}

// Same as corotated_stress but also returns the SVD so the VJP can reuse it.
template <class T>
FL_HD M3<T> corotated_stress_svd(const M3<T>& f, T mu, T lambda, bool& ok, Svd<T>& t) {
    T j = det(f);
    ok = j > T(0);
    M3<T> p = cofactor(f) * (lambda * (j - T(1)));
    if (mu != T(0)) {
        t = svd3(f);
        p += (f - polar_R(t)) * (T(2) * mu);
    }
    return p;
}

// materials.hpp:36-51
template <class T>
FL_HD M3<T> corotated_stress_vjp(const M3<T>& f, T mu, T lambda, const M3<T>& p_bar, const Svd<T>& t) {
    T j = det(f);
    M3<T> finv_t = transpose(inverse(f));
    M3<T> g = finv_t * j;
    T s = lambda * (j - T(1)) * j;
    M3<T> f_bar = g * (lambda * (T(2) * j - T(1)) * ddot(p_bar, finv_t));
    f_bar -= (finv_t * transpose(p_bar) * finv_t) * s;
    if (mu != T(0)) {
        f_bar += p_bar * (T(2) * mu);
        f_bar -= polar_rotation_vjp(t, p_bar) * (T(2) * mu);
    }
    return f_bar;
}

// the lambda (J-1) cofactor(F) part of corotated_stress_vjp alone (mu = 0 liquids)
template <class T>
FL_HD M3<T> pressure_stress_vjp(const M3<T>& f, T lambda, const M3<T>& p_bar) {
    T j = det(f);
    M3<T> finv_t = transpose(inverse(f));
    T s = lambda * (j - T(1)) * j;
    M3<T> f_bar = finv_t * (j * lambda * (T(2) * j - T(1)) * ddot(p_bar, finv_t));
    f_bar -= (finv_t * transpose(p_bar) * finv_t) * s;
    return f_bar;
}

// materials.hpp:55-63
template <class T>
FL_HD M3<T> box_yield_project(const M3<T>& f, T theta_c, T theta_s, bool& ok) {
    ok = det(f) > T(0);
    Svd<T> t = svd3(f);
    V3<T> s;
#pragma unroll
    for (int i = 0; i < 3; i++) s[i] = clamp_ref(t.s[i], T(1) - theta_c, T(1) + theta_s);
    return usv(t, s);
}

template <class T>
FL_HD M3<T> box_yield_project_vjp(const M3<T>& f, T theta_c, T theta_s, const M3<T>& out_bar) {
    Svd<T> t = svd3(f);
    double g[3], jg[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 3; i++) {
        T si = t.s[i];
        g[i] = double(clamp_ref(si, T(1) - theta_c, T(1) + theta_s));
        bool inside = si > T(1) - theta_c && si < T(1) + theta_s;
        jg[4 * i] = inside ? 1.0 : 0.0;
    }
    return spectral_map_vjp(t, g, jg, out_bar);
}

// materials.hpp:81-104
template <class T>
FL_HD M3<T> von_mises_project(const M3<T>& f, T sigma_y, T mu, bool& ok) {
    Svd<T> t = svd3(f);
    ok = t.s.x > T(0) && t.s.y > T(0) && t.s.z > T(0);
    T eps[3], mean = T(0);
#pragma unroll
    for (int i = 0; i < 3; i++) {
        eps[i] = log(t.s[i]);
        mean += eps[i];
    }
    mean /= T(3);
    T dev[3], dn2 = T(0);
#pragma unroll
    for (int i = 0; i < 3; i++) {
        dev[i] = eps[i] - mean;
        dn2 += dev[i] * dev[i];
    }
    T dn = sqrt(dn2);
    if (T(2) * mu * dn <= sigma_y) return f;
    T scale = sigma_y / (T(2) * mu * dn);
    V3<T> s;
#pragma unroll
    for (int i = 0; i < 3; i++) s[i] = exp(mean + scale * dev[i]);
    return usv(t, s);
}

// materials.hpp:106-145; the spectral Jacobian is formed in fp64.
template <class T>
FL_HD M3<T> von_mises_project_vjp(const M3<T>& f, T sigma_y, T mu, const M3<T>& out_bar) {
    Svd<T> t = svd3(f);
    double sd[3] = {double(t.s.x), double(t.s.y), double(t.s.z)};
    double eps[3], mean = 0;
#pragma unroll
    for (int i = 0; i < 3; i++) {
        eps[i] = log(sd[i]);
        mean += eps[i];
    }
    mean /= 3.0;
    double dev[3], dn2 = 0;
#pragma unroll
    for (int i = 0; i < 3; i++) {
        dev[i] = eps[i] - mean;
        dn2 += dev[i] * dev[i];
    }
    double dn = sqrt(dn2);
    double g[3], jg[9];
    double muD = double(mu), syD = double(sigma_y);
    if (2 * muD * dn <= syD) {
#pragma unroll
        for (int i = 0; i < 3; i++) g[i] = sd[i];
#pragma unroll
        for (int k = 0; k < 9; k++) jg[k] = (k % 4 == 0) ? 1.0 : 0.0;
    } else {
        double scale = syD / (2 * muD * dn);
#pragma unroll
        for (int i = 0; i < 3; i++) g[i] = exp(mean + scale * dev[i]);
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int k = 0; k < 3; k++) {
                double m = (i == k ? 1.0 : 0.0) - 1.0 / 3.0;
                double jeps = 1.0 / 3.0 + scale * (m - (dev[i] / dn) * (dev[k] / dn));
                jg[3 * i + k] = g[i] * jeps / sd[k];
            }
    }
    return spectral_map_vjp(t, g, jg, out_bar);
}

// materials.hpp:149-161
template <class T>
FL_HD M3<T> liquid_project(const M3<T>& f, bool& ok) {
    T j = det(f);
    ok = j > T(0);
    return meye<T>() * cbrt(j);
}
// the same with the output cotangent given compactly as dL/dc = tr(out_bar)
template <class T>
FL_HD M3<T> liquid_project_vjp_c(const M3<T>& f, T c_bar) {
    T j = det(f);
    return cofactor(f) * (c_bar * cbrt(j) / (T(3) * j));
}

template <class T>
FL_HD M3<T> liquid_project_vjp(const M3<T>& f, const M3<T>& out_bar) {
    T j = det(f);
    T c = trace(out_bar) * cbrt(j) / (T(3) * j);
    return cofactor(f) * c;
}

}  // namespace fl
