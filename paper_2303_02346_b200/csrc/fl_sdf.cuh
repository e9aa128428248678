// fl_sdf.cuh -- analytic SDF primitives for kinematic end-effectors.
//
// Restates the behaviour of proj/include/flume/sdf.hpp:75-339 (distance,
// gradient with +x fallback, Hessian-vector product, pose VJP) for the five
// reference primitives (sphere, box, capsule, cylinder, halfspace), templated
// on the scalar.  The shape-kind numbering matches ShapeKind (sdf.hpp:24).
#pragma once

#include "fl_math.cuh"

namespace fl {

enum ShapeKindId : int { SK_SPHERE = 0, SK_BOX = 1, SK_CAPSULE = 2, SK_CYLINDER = 3, SK_HALFSPACE = 4 };

template <class T>
struct ShapeP {
    int kind;
    T radius;
    V3<T> half;
    V3<T> seg_a, seg_b;
    V3<T> normal;
    T offset;
    T half_height;
};

template <class T> FL_HD T sgn_ge0(T x) { return x >= T(0) ? T(1) : T(-1); }

template <class T>
FL_HD void capsule_closest(const ShapeP<T>& s, V3<T> q, V3<T>& e, bool& interior) {
    V3<T> u = s.seg_b - s.seg_a;
    T uu = norm_sq(u);
    T t = uu > T(0) ? clamp_ref(dot(q - s.seg_a, u) / uu, T(0), T(1)) : T(0);
    interior = (t > T(0) && t < T(1));
    e = q - (s.seg_a + u * t);
}

// sdf.hpp:131-143
template <class T>
FL_HD T sdf_local_distance(const ShapeP<T>& s, V3<T> q) {
    switch (s.kind) {
        case SK_SPHERE: return norm(q) - s.radius;
        case SK_BOX: {
            T inside = -INFINITY;
            T out_sq = T(0);
            for (int i = 0; i < 3; i++) {
                T a = fabs(q[i]) - s.half[i];
                inside = inside > a ? inside : a;
                T m = a > T(0) ? a : T(0);
                out_sq += m * m;
            }
            if (inside <= T(0)) return inside;
            return sqrt(out_sq);
        }
        case SK_CAPSULE: {
            V3<T> e;
            bool in;
            capsule_closest(s, q, e, in);
            return norm(e) - s.radius;
        }
        case SK_CYLINDER: {
            T rho = sqrt(q.x * q.x + q.y * q.y);
            T y1 = rho - s.radius;
            T y2 = fabs(q.z) - s.half_height;
            T mx = y1 > y2 ? y1 : y2;
            T inside = mx < T(0) ? mx : T(0);
            T m1 = y1 > T(0) ? y1 : T(0), m2 = y2 > T(0) ? y2 : T(0);
            return inside + sqrt(m1 * m1 + m2 * m2);
        }
        case SK_HALFSPACE: return dot(s.normal, q) - s.offset;
    }
    return T(0);
}

// sdf.hpp:147-211
template <class T>
FL_HD V3<T> sdf_local_grad(const ShapeP<T>& s, V3<T> q) {
    const V3<T> fb = {T(1), T(0), T(0)};
    switch (s.kind) {
        case SK_SPHERE: {
            T n = norm(q);
            if (n < T(1e-12)) return fb;
            return q * (T(1) / n);
        }
        case SK_BOX: {
            V3<T> a, m;
            T inside = -INFINITY;
            int k = 0;
            bool out = false;
            for (int i = 0; i < 3; i++) {
                a[i] = fabs(q[i]) - s.half[i];
                m[i] = a[i] > T(0) ? a[i] : T(0);
                if (a[i] > T(0)) out = true;
                if (a[i] > inside) {
                    inside = a[i];
                    k = i;
                }
            }
            if (!out) {
                V3<T> g = v3zero<T>();
                g[k] = q[k] >= T(0) ? T(1) : T(-1);
                return g;
            }
            T mn = norm(m);
            if (mn < T(1e-12)) return fb;
            V3<T> g;
            for (int i = 0; i < 3; i++) g[i] = sgn_ge0(q[i]) * m[i] / mn;
            return g;
        }
        case SK_CAPSULE: {
            V3<T> e;
            bool in;
            capsule_closest(s, q, e, in);
            T n = norm(e);
            if (n < T(1e-12)) return fb;
            return e * (T(1) / n);
        }
        case SK_CYLINDER: {
            T rho = sqrt(q.x * q.x + q.y * q.y);
            T y1 = rho - s.radius;
            T y2 = fabs(q.z) - s.half_height;
            T sz = sgn_ge0(q.z);
            V3<T> radial = rho > T(1e-12) ? V3<T>{q.x / rho, q.y / rho, T(0)} : V3<T>{T(1), T(0), T(0)};
            V3<T> axial = {T(0), T(0), sz};
            if (y1 <= T(0) && y2 <= T(0)) return y1 > y2 ? radial : axial;
            if (y1 > T(0) && y2 <= T(0)) return radial;
            if (y1 <= T(0) && y2 > T(0)) return axial;
            T phi = sqrt(y1 * y1 + y2 * y2);
            if (phi < T(1e-12)) return fb;
            return radial * (y1 / phi) + axial * (y2 / phi);
        }
        case SK_HALFSPACE: return s.normal;
    }
    return fb;
}

// sdf.hpp:216-291
template <class T>
FL_HD V3<T> sdf_local_hess_vec(const ShapeP<T>& s, V3<T> q, V3<T> u) {
    switch (s.kind) {
        case SK_SPHERE: {
            T n = norm(q);
            if (n < T(1e-12)) return v3zero<T>();
            V3<T> qh = q * (T(1) / n);
            return (u - qh * dot(qh, u)) * (T(1) / n);
        }
        case SK_BOX: {
            V3<T> a, m;
            bool out = false;
            for (int i = 0; i < 3; i++) {
                a[i] = fabs(q[i]) - s.half[i];
                m[i] = a[i] > T(0) ? a[i] : T(0);
                if (a[i] > T(0)) out = true;
            }
            if (!out) return v3zero<T>();
            T mn = norm(m);
            if (mn < T(1e-12)) return v3zero<T>();
            T smu = T(0);
            for (int i = 0; i < 3; i++) smu += sgn_ge0(q[i]) * m[i] * u[i];
            V3<T> r;
            for (int i = 0; i < 3; i++) {
                T act = a[i] > T(0) ? T(1) : T(0);
                r[i] = act * u[i] / mn - sgn_ge0(q[i]) * m[i] * smu / (mn * mn * mn);
            }
            return r;
        }
        case SK_CAPSULE: {
            V3<T> e;
            bool interior;
            capsule_closest(s, q, e, interior);
            T n = norm(e);
            if (n < T(1e-12)) return v3zero<T>();
            V3<T> eh = e * (T(1) / n);
            V3<T> r = (u - eh * dot(eh, u)) * (T(1) / n);
            if (interior) {
                V3<T> ua = s.seg_b - s.seg_a;
                T un = norm(ua);
                if (un > T(1e-12)) {
                    V3<T> uh = ua * (T(1) / un);
                    r -= uh * (dot(uh, u) / n);
                }
            }
            return r;
        }
        case SK_CYLINDER: {
            T rho = sqrt(q.x * q.x + q.y * q.y);
            T y1 = rho - s.radius;
            T y2 = fabs(q.z) - s.half_height;
            T sz = sgn_ge0(q.z);
            if (rho < T(1e-12)) return v3zero<T>();
            V3<T> radial = {q.x / rho, q.y / rho, T(0)};
            V3<T> hrho_u = {u.x / rho, u.y / rho, T(0)};
            hrho_u -= radial * (dot(radial, u) / rho);
            bool side = (y1 > T(0) && y2 <= T(0)) || (y1 <= T(0) && y2 <= T(0) && y1 > y2);
            if (side) return hrho_u;
            if (y1 <= T(0) || y2 <= T(0)) return v3zero<T>();
            T phi = sqrt(y1 * y1 + y2 * y2);
            T yh0 = y1 / phi, yh1 = y2 / phi;
            T ju0 = dot(radial, u), ju1 = sz * u.z;
            T pr = yh0 * ju0 + yh1 * ju1;
            T hf0 = (ju0 - yh0 * pr) / phi, hf1 = (ju1 - yh1 * pr) / phi;
            V3<T> r = radial * hf0 + V3<T>{T(0), T(0), sz * hf1};
            r += hrho_u * (y1 / phi);
            return r;
        }
        case SK_HALFSPACE: return v3zero<T>();
    }
    return v3zero<T>();
}

// World-placed primitive: q = R^T (p - t)
template <class T>
struct SdfSample {
    T distance;
    V3<T> normal;
};

// sdf.hpp:307-315 -- normalized(R g) with +x fallback at 1e-30
template <class T>
FL_HD SdfSample<T> sdf_eval(const ShapeP<T>& s, V3<T> pt, const M3<T>& pr, V3<T> p) {
    V3<T> q = tmul(pr, p - pt);
    SdfSample<T> out;
    out.distance = sdf_local_distance(s, q);
    V3<T> g = sdf_local_grad(s, q);
    out.normal = normalized_or_x(pr * g, T(1e-30));
    return out;
}

// sdf.hpp:319-339
template <class T>
FL_HD void sdf_eval_pose_vjp(const ShapeP<T>& s, V3<T> pt, const M3<T>& pr, V3<T> p, T d_bar, V3<T> n_bar,
                             V3<T>& t_bar, M3<T>& r_bar) {
    V3<T> q = tmul(pr, p - pt);
    V3<T> g = sdf_local_grad(s, q);
    T gn = norm(g);
    V3<T> q_bar = g * d_bar;
    if (gn > T(1e-12)) {
        V3<T> ng = g * (T(1) / gn);
        V3<T> n = pr * ng;
        V3<T> nbp = (n_bar - n * dot(n, n_bar)) * (T(1) / gn);
        r_bar += outer(nbp, g);
        V3<T> g_bar = tmul(pr, nbp);
        q_bar += sdf_local_hess_vec(s, q, g_bar);
    }
    t_bar -= pr * q_bar;
    r_bar += outer(p - pt, q_bar);
}

}  // namespace fl
