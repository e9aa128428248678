// fl_math.cuh -- small fixed-size linear algebra for the MLS-MPM substep.
//
// Templated on the scalar so the same formulas run as fp32 inside the sm_100a
// kernels and as fp64 on the host (effector kinematics) and in the single-thread
// rigid-body solves.  Matrices are row-major 3x3 like the reference's Mat<N>
// (proj/include/flume/core.hpp:148-226).
#pragma once

#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define FL_HD __host__ __device__ __forceinline__
#else
#define FL_HD inline
#endif

namespace fl {

template <class T>
struct V3 {
    T x, y, z;
    FL_HD T& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
    FL_HD T operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};

template <class T> FL_HD V3<T> v3(T x, T y, T z) { return V3<T>{x, y, z}; }
template <class T> FL_HD V3<T> v3zero() { return V3<T>{T(0), T(0), T(0)}; }
template <class T> FL_HD V3<T> operator+(V3<T> a, V3<T> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class T> FL_HD V3<T> operator-(V3<T> a, V3<T> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class T> FL_HD V3<T> operator-(V3<T> a) { return {-a.x, -a.y, -a.z}; }
template <class T> FL_HD V3<T> operator*(V3<T> a, T s) { return {a.x * s, a.y * s, a.z * s}; }
template <class T> FL_HD V3<T> operator*(T s, V3<T> a) { return {a.x * s, a.y * s, a.z * s}; }
template <class T> FL_HD V3<T>& operator+=(V3<T>& a, V3<T> b) { a.x += b.x; a.y += b.y; a.z += b.z; return a; }
template <class T> FL_HD V3<T>& operator-=(V3<T>& a, V3<T> b) { a.x -= b.x; a.y -= b.y; a.z -= b.z; return a; }
template <class T> FL_HD T dot(V3<T> a, V3<T> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class T> FL_HD T norm_sq(V3<T> a) { return dot(a, a); }
template <class T> FL_HD T norm(V3<T> a) { return sqrt(norm_sq(a)); }
template <class T> FL_HD V3<T> cross(V3<T> a, V3<T> b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class T> FL_HD T clampv(T x, T lo, T hi) { return x < lo ? lo : (x > hi ? hi : x); }
// std::min(std::max(x, lo), hi) semantics of core.hpp:476 (NaN-free inputs)
template <class T> FL_HD T clamp_ref(T x, T lo, T hi) {
    T m = x > lo ? x : lo;
    return m < hi ? m : hi;
}

template <class T>
struct M3 {
    T m[9];
    FL_HD T& operator()(int r, int c) { return m[3 * r + c]; }
    FL_HD T operator()(int r, int c) const { return m[3 * r + c]; }
};

template <class T> FL_HD M3<T> mzero() {
    M3<T> r;
#pragma unroll
    for (int i = 0; i < 9; i++) r.m[i] = T(0);
    return r;
}
template <class T> FL_HD M3<T> meye() {
    M3<T> r = mzero<T>();
    r.m[0] = r.m[4] = r.m[8] = T(1);
    return r;
}
template <class T> FL_HD M3<T> mdiag(V3<T> d) {
    M3<T> r = mzero<T>();
    r.m[0] = d.x;
    r.m[4] = d.y;
    r.m[8] = d.z;
    return r;
}
template <class T> FL_HD M3<T> operator+(const M3<T>& a, const M3<T>& b) {
    M3<T> r;
#pragma unroll
    for (int i = 0; i < 9; i++) r.m[i] = a.m[i] + b.m[i];
    return r;
}
template <class T> FL_HD M3<T> operator-(const M3<T>& a, const M3<T>& b) {
    M3<T> r;
#pragma unroll
    for (int i = 0; i < 9; i++) r.m[i] = a.m[i] - b.m[i];
    return r;
}
template <class T> FL_HD M3<T> operator*(const M3<T>& a, T s) {
    M3<T> r;
#pragma unroll
    for (int i = 0; i < 9; i++) r.m[i] = a.m[i] * s;
    return r;
}
template <class T> FL_HD M3<T>& operator+=(M3<T>& a, const M3<T>& b) {
#pragma unroll
    for (int i = 0; i < 9; i++) a.m[i] += b.m[i];
    return a;
}
template <class T> FL_HD M3<T>& operator-=(M3<T>& a, const M3<T>& b) {
#pragma unroll
    for (int i = 0; i < 9; i++) a.m[i] -= b.m[i];
    return a;
}
template <class T> FL_HD M3<T> operator*(const M3<T>& a, const M3<T>& b) {
    M3<T> r;
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++)
            r.m[3 * i + j] = a.m[3 * i] * b.m[j] + a.m[3 * i + 1] * b.m[3 + j] + a.m[3 * i + 2] * b.m[6 + j];
    return r;
}
template <class T> FL_HD V3<T> operator*(const M3<T>& a, V3<T> v) {
    return {a.m[0] * v.x + a.m[1] * v.y + a.m[2] * v.z, a.m[3] * v.x + a.m[4] * v.y + a.m[5] * v.z,
            a.m[6] * v.x + a.m[7] * v.y + a.m[8] * v.z};
}
// a^T v
template <class T> FL_HD V3<T> tmul(const M3<T>& a, V3<T> v) {
    return {a.m[0] * v.x + a.m[3] * v.y + a.m[6] * v.z, a.m[1] * v.x + a.m[4] * v.y + a.m[7] * v.z,
            a.m[2] * v.x + a.m[5] * v.y + a.m[8] * v.z};
}
template <class T> FL_HD M3<T> transpose(const M3<T>& a) {
    M3<T> r;
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) r.m[3 * i + j] = a.m[3 * j + i];
    return r;
}
template <class T> FL_HD M3<T> outer(V3<T> a, V3<T> b) {
    M3<T> r;
    r.m[0] = a.x * b.x; r.m[1] = a.x * b.y; r.m[2] = a.x * b.z;
    r.m[3] = a.y * b.x; r.m[4] = a.y * b.y; r.m[5] = a.y * b.z;
    r.m[6] = a.z * b.x; r.m[7] = a.z * b.y; r.m[8] = a.z * b.z;
    return r;
}
template <class T> FL_HD T trace(const M3<T>& a) { return a.m[0] + a.m[4] + a.m[8]; }
template <class T> FL_HD T ddot(const M3<T>& a, const M3<T>& b) {
    T s = T(0);
#pragma unroll
    for (int i = 0; i < 9; i++) s += a.m[i] * b.m[i];
    return s;
}
template <class T> FL_HD T det(const M3<T>& a) {
    return a.m[0] * (a.m[4] * a.m[8] - a.m[5] * a.m[7]) - a.m[1] * (a.m[3] * a.m[8] - a.m[5] * a.m[6]) +
           a.m[2] * (a.m[3] * a.m[7] - a.m[4] * a.m[6]);
}
// cofactor(A) = det(A) A^{-T}  (core.hpp:324-336)
template <class T> FL_HD M3<T> cofactor(const M3<T>& a) {
    M3<T> r;
    r.m[0] = a.m[4] * a.m[8] - a.m[5] * a.m[7];
    r.m[1] = a.m[5] * a.m[6] - a.m[3] * a.m[8];
    r.m[2] = a.m[3] * a.m[7] - a.m[4] * a.m[6];
    r.m[3] = a.m[2] * a.m[7] - a.m[1] * a.m[8];
    r.m[4] = a.m[0] * a.m[8] - a.m[2] * a.m[6];
    r.m[5] = a.m[1] * a.m[6] - a.m[0] * a.m[7];
    r.m[6] = a.m[1] * a.m[5] - a.m[2] * a.m[4];
    r.m[7] = a.m[2] * a.m[3] - a.m[0] * a.m[5];
    r.m[8] = a.m[0] * a.m[4] - a.m[1] * a.m[3];
    return r;
}
template <class T> FL_HD M3<T> inverse(const M3<T>& a) {
    T d = det(a);
    return transpose(cofactor(a)) * (T(1) / d);
}
template <class T> FL_HD M3<T> skew(V3<T> w) {
    M3<T> r = mzero<T>();
    r.m[1] = -w.z; r.m[2] = w.y;
    r.m[3] = w.z;  r.m[5] = -w.x;
    r.m[6] = -w.y; r.m[7] = w.x;
    return r;
}
// <skew(u), M> = dot(u, ax(M))   (core.hpp:362-365)
template <class T> FL_HD V3<T> axv(const M3<T>& m) {
    return {m.m[7] - m.m[5], m.m[2] - m.m[6], m.m[3] - m.m[1]};
}
template <class T> FL_HD M3<T> col_flip_last(M3<T> a) {
    a.m[2] = -a.m[2];
    a.m[5] = -a.m[5];
    a.m[8] = -a.m[8];
    return a;
}

template <class T> FL_HD V3<T> normalized_or_x(V3<T> a, T eps) {
    T n = norm(a);
    if (n < eps) return {T(1), T(0), T(0)};
    return a * (T(1) / n);
}

// ---------------------------------------------------------------------------
// Rotations (core.hpp:379-457): Rodrigues exponential and its right Jacobian.
// ---------------------------------------------------------------------------
template <class T> FL_HD M3<T> exp_so3(V3<T> w) {
    T th = norm(w);
    M3<T> k = skew(w);
    T a, b;
    if (th < T(1e-8)) {
        a = T(1) - th * th / T(6);
        b = T(0.5) - th * th / T(24);
    } else {
        a = sin(th) / th;
        b = (T(1) - cos(th)) / (th * th);
    }
    return meye<T>() + k * a + (k * k) * b;
}

template <class T> FL_HD M3<T> right_jacobian_so3(V3<T> w) {
    T th = norm(w);
    M3<T> k = skew(w);
    T a, b;
    if (th < T(1e-6)) {
        a = T(0.5) - th * th / T(24);
        b = T(1) / T(6) - th * th / T(120);
    } else {
        a = (T(1) - cos(th)) / (th * th);
        b = (th - sin(th)) / (th * th * th);
    }
    return meye<T>() - k * a + (k * k) * b;
}

// ---------------------------------------------------------------------------
// SVD by one-sided Jacobi on the columns of B = A V (svd.hpp:16-120).
// sigma sorted descending (ties keep column order), near-null columns of U
// rebuilt orthogonal to the others, and det(U) = +1 enforced by flipping the
// last column of both factors.  fp32 runs a bounded sweep count with a
// relative off-diagonal stop at ~2.5 ulp; fp64 uses the reference's
// 30 sweeps / 1e-15.
// ---------------------------------------------------------------------------
template <class T> struct SvdTol;
template <> struct SvdTol<float> {
    static constexpr int sweeps = 8;
    static constexpr float stop = 3e-7f;
    static constexpr float null_sigma = 1e-30f;
    static constexpr float tiny = 1e-35f;
};
template <> struct SvdTol<double> {
    static constexpr int sweeps = 30;
    static constexpr double stop = 1e-15;
    static constexpr double null_sigma = 1e-150;
    static constexpr double tiny = 1e-300;
};

template <class T>
struct Svd {
    M3<T> U;
    V3<T> s;
    M3<T> V;
};

template <class T>
FL_HD void jacobi_rotate(M3<T>& b, M3<T>& v, int p, int q, T& off) {
    T apq = b.m[p] * b.m[q] + b.m[3 + p] * b.m[3 + q] + b.m[6 + p] * b.m[6 + q];
    T app = b.m[p] * b.m[p] + b.m[3 + p] * b.m[3 + p] + b.m[6 + p] * b.m[6 + p];
    T aqq = b.m[q] * b.m[q] + b.m[3 + q] * b.m[3 + q] + b.m[6 + q] * b.m[6 + q];
    T r = fabs(apq) / (sqrt(app * aqq) + SvdTol<T>::tiny);
    off = off > r ? off : r;
    if (fabs(apq) < SvdTol<T>::tiny) return;
    T tau = (aqq - app) / (T(2) * apq);
    T t = (tau >= T(0) ? T(1) : T(-1)) / (fabs(tau) + sqrt(T(1) + tau * tau));
    T c = T(1) / sqrt(T(1) + t * t);
    T sn = c * t;
#pragma unroll
    for (int i = 0; i < 3; i++) {
        T bp = b.m[3 * i + p], bq = b.m[3 * i + q];
        b.m[3 * i + p] = c * bp - sn * bq;
        b.m[3 * i + q] = sn * bp + c * bq;
        T vp = v.m[3 * i + p], vq = v.m[3 * i + q];
        v.m[3 * i + p] = c * vp - sn * vq;
        v.m[3 * i + q] = sn * vp + c * vq;
    }
}

template <class T>
FL_HD Svd<T> svd3(const M3<T>& a) {
    M3<T> b = a;
    M3<T> v = meye<T>();
    for (int sweep = 0; sweep < SvdTol<T>::sweeps; sweep++) {
        T off = T(0);
        jacobi_rotate(b, v, 0, 1, off);
        jacobi_rotate(b, v, 0, 2, off);
        jacobi_rotate(b, v, 1, 2, off);
        if (off < SvdTol<T>::stop) break;
    }
    // column norms, then a stable descending sort by swapping whole columns
    // (static indices only: no local-memory arrays)
    T s0 = sqrt(b.m[0] * b.m[0] + b.m[3] * b.m[3] + b.m[6] * b.m[6]);
    T s1 = sqrt(b.m[1] * b.m[1] + b.m[4] * b.m[4] + b.m[7] * b.m[7]);
    T s2 = sqrt(b.m[2] * b.m[2] + b.m[5] * b.m[5] + b.m[8] * b.m[8]);
    auto swap01 = [&]() {
        T t = s0; s0 = s1; s1 = t;
#pragma unroll
        for (int i = 0; i < 3; i++) {
            t = b.m[3 * i]; b.m[3 * i] = b.m[3 * i + 1]; b.m[3 * i + 1] = t;
            t = v.m[3 * i]; v.m[3 * i] = v.m[3 * i + 1]; v.m[3 * i + 1] = t;
        }
    };
    auto swap12 = [&]() {
        T t = s1; s1 = s2; s2 = t;
#pragma unroll
        for (int i = 0; i < 3; i++) {
            t = b.m[3 * i + 1]; b.m[3 * i + 1] = b.m[3 * i + 2]; b.m[3 * i + 2] = t;
            t = v.m[3 * i + 1]; v.m[3 * i + 1] = v.m[3 * i + 2]; v.m[3 * i + 2] = t;
        }
    };
    if (s1 > s0) swap01();
    if (s2 > s1) {
        swap12();
        if (s1 > s0) swap01();
    }
    Svd<T> out;
    out.s = V3<T>{s0, s1, s2};
    out.V = v;
#pragma unroll
    for (int jj = 0; jj < 3; jj++) {
        const T sj = jj == 0 ? s0 : (jj == 1 ? s1 : s2);
        const T inv = sj > SvdTol<T>::null_sigma ? T(1) / sj : T(0);
#pragma unroll
        for (int i = 0; i < 3; i++) out.U.m[3 * i + jj] = b.m[3 * i + jj] * inv;
    }
    // rebuild null columns of U (svd.hpp:88-106)
#pragma unroll
    for (int j = 0; j < 3; j++) {
        if (out.s[j] > SvdTol<T>::null_sigma) continue;
        for (int axis = 0; axis < 3; axis++) {
            V3<T> c = v3zero<T>();
            c[axis] = T(1);
            for (int k = 0; k < 3; k++) {
                if (k == j) continue;
                T proj = out.U.m[k] * c.x + out.U.m[3 + k] * c.y + out.U.m[6 + k] * c.z;
                c.x -= proj * out.U.m[k];
                c.y -= proj * out.U.m[3 + k];
                c.z -= proj * out.U.m[6 + k];
            }
            T n = norm(c);
            if (n > T(1e-8)) {
                out.U.m[j] = c.x / n;
                out.U.m[3 + j] = c.y / n;
                out.U.m[6 + j] = c.z / n;
                break;
            }
        }
    }
    if (det(out.U) < T(0)) {
        out.U = col_flip_last(out.U);
        out.V = col_flip_last(out.V);
    }
    return out;
}

// U diag(g) V^T
template <class T> FL_HD M3<T> usv(const Svd<T>& t, V3<T> g) {
    M3<T> r;
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++)
            r.m[3 * i + j] = t.U.m[3 * i] * g.x * t.V.m[3 * j] + t.U.m[3 * i + 1] * g.y * t.V.m[3 * j + 1] +
                             t.U.m[3 * i + 2] * g.z * t.V.m[3 * j + 2];
    return r;
}

template <class T> FL_HD M3<T> polar_R(const Svd<T>& t) { return t.U * transpose(t.V); }

// VJP of the full SVD (svd.hpp:140-162), K-matrix form with a clamped gap.
template <class T>
FL_HD M3<T> svd_vjp(const Svd<T>& t, const M3<T>& u_bar, V3<T> sig_bar, const M3<T>& v_bar, T gap_tol) {
    M3<T> bu = transpose(t.U) * u_bar;
    M3<T> bv = transpose(t.V) * v_bar;
    M3<T> inner = mdiag(sig_bar);
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) {
            if (i == j) continue;
            T si = t.s[i], sj = t.s[j];
            T den = sj * sj - si * si;
            if (fabs(den) < gap_tol) den = den >= T(0) ? gap_tol : -gap_tol;
            inner.m[3 * i + j] += (sj * (bu.m[3 * i + j] - bu.m[3 * j + i]) + si * (bv.m[3 * i + j] - bv.m[3 * j + i])) / den;
        }
    return t.U * inner * transpose(t.V);
}

// VJP of a spectral map Y = U g(sigma) V^T (svd.hpp:164-205).  The divided
// differences are formed in fp64 even for fp32 inputs: g_j - g_i loses all
// precision in fp32 when sigma_i ~ sigma_j (F near identity, the common case).
template <class T>
FL_HD M3<T> spectral_map_vjp(const Svd<T>& t, const double g[3], const double jg[9], const M3<T>& y_bar) {
    M3<T> q_bar = transpose(t.U) * y_bar * t.V;
    const double gap_tol = 1e-8;
    double s[3] = {double(t.s.x), double(t.s.y), double(t.s.z)};
    M3<T> p_bar = mzero<T>();
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) {
            if (i == j) continue;
            double sum = s[i] + s[j];
            sum = sum > 1e-300 ? sum : 1e-300;
            double diff = s[j] - s[i];
            double dd_g, dd_sg;
            if (fabs(diff) < gap_tol) {
                double gp = 0.5 * (jg[4 * i] + jg[4 * j] - jg[3 * i + j] - jg[3 * j + i]);
                dd_g = gp;
                dd_sg = 0.5 * (g[i] + g[j]) + 0.5 * (s[i] + s[j]) * gp;
            } else {
                dd_g = (g[j] - g[i]) / diff;
                dd_sg = (s[j] * g[j] - s[i] * g[i]) / diff;
            }
            double a = dd_sg / sum;
            double b = (s[i] * dd_g - g[i]) / sum;
            p_bar.m[3 * i + j] += T(a) * q_bar.m[3 * i + j];
            p_bar.m[3 * j + i] += T(b) * q_bar.m[3 * i + j];
        }
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int k = 0; k < 3; k++) p_bar.m[4 * k] += T(jg[3 * i + k]) * q_bar.m[4 * i];
    return t.U * p_bar * transpose(t.V);
}

// VJP of the polar rotation R = U V^T (svd.hpp:207-228):
// solve (tr(S) I - S) g = ax(R^T R_bar), A_bar = R skew(g).
template <class T>
FL_HD M3<T> polar_rotation_vjp(const Svd<T>& t, const M3<T>& r_bar) {
    M3<T> r = t.U * transpose(t.V);
    M3<T> s = t.V * mdiag(t.s) * transpose(t.V);
    M3<T> l = meye<T>() * trace(s) - s;
    V3<T> rhs = axv(transpose(r) * r_bar);
    V3<T> g = inverse(l) * rhs;
    return r * skew(g);
}

// R_new = Exp(w dt) R_old and its VJP (core.hpp:429-457)
template <class T> FL_HD M3<T> advance_rotation(const M3<T>& r_old, V3<T> w, T dt) {
    return exp_so3(w * dt) * r_old;
}
template <class T>
FL_HD void advance_rotation_vjp(const M3<T>& r_old, V3<T> w, T dt, const M3<T>& r_new_bar, M3<T>& r_old_bar,
                                V3<T>& w_bar) {
    M3<T> e = exp_so3(w * dt);
    r_old_bar += transpose(e) * r_new_bar;
    M3<T> jr = right_jacobian_so3(w * dt);
    V3<T> g = axv(transpose(e) * r_new_bar * transpose(r_old));
    V3<T> phi_bar = tmul(jr, g);
    w_bar += phi_bar * dt;
}

}  // namespace fl
