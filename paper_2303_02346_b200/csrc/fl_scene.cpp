// fl_scene.cpp -- scene JSON -> flume_scene_desc + initial state (3D).
//
// Restates build_scene<3> (proj/include/flume/scene.hpp:161-408) for the parts
// the hot path consumes: SimConfig, materials, effectors, bodies sampled on a
// jittered lattice (scene.hpp:114-147) with xoshiro256** seeded by splitmix64
// (rng.hpp:11-70), exclusion holes, emitters, rigid-body rest shapes and the
// target_point / hold_initial / composite loss specs.  Arithmetic follows the
// reference operation order so particle positions are bit-identical to the
// reference's on x86-64 (compiled without FMA contraction).  Gas sources are
// outside the GPU path and rejected.
#include <json.hpp>

#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/flume_b200.h"
#include "fl_math.cuh"
#include "fl_physics.cuh"

using nlohmann::json;
using fl::M3;
using fl::V3;
using V = V3<double>;
using M = M3<double>;

namespace {

struct SceneErr : std::runtime_error {
    explicit SceneErr(const std::string& m) : std::runtime_error(m) {}
};

class Xoshiro {
public:
    explicit Xoshiro(uint64_t seed) {
        uint64_t x = seed;
        for (auto& si : s_) {
            x += 0x9e3779b97f4a7c15ull;
            uint64_t z = x;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            si = z ^ (z >> 31);
        }
    }
    uint64_t next() {
        uint64_t r = rotl(s_[1] * 5, 7) * 9;
        uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return r;
    }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

private:
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t s_[4];
};

V vec3(const json& j, const char* what) {
    if (!j.is_array() || j.size() != 3) throw SceneErr(std::string(what) + ": expected an array of 3 numbers");
    return V{j[0].get<double>(), j[1].get<double>(), j[2].get<double>()};
}

// reference Mat*Vec accumulates s = 0; s += m[i][j] v[j]
V matvec(const M& m, const V& v) {
    V r;
    for (int i = 0; i < 3; i++) {
        double s = 0;
        for (int j = 0; j < 3; j++) s += m(i, j) * v[j];
        r[i] = s;
    }
    return r;
}

M matmul(const M& a, const M& b) {
    M r;
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0;
            for (int k = 0; k < 3; k++) s += a(i, k) * b(k, j);
            r(i, j) = s;
        }
    return r;
}

M exp_so3_ref(const V& w) {
    double th = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    M k = fl::skew(w);
    double a, b;
    if (th < 1e-8) {
        a = 1 - th * th / 6;
        b = 0.5 - th * th / 24;
    } else {
        a = std::sin(th) / th;
        b = (1 - std::cos(th)) / (th * th);
    }
    M kk = matmul(k, k);
    M r = fl::meye<double>();
    for (int q = 0; q < 9; q++) r.m[q] = (r.m[q] + a * k.m[q]) + b * kk.m[q];
    return r;
}

struct Pose {
    V t{0, 0, 0};
    M R = fl::meye<double>();
    V to_world(const V& q) const {
        V rq = matvec(R, q);
        return V{rq[0] + t[0], rq[1] + t[1], rq[2] + t[2]};
    }
};

Pose parse_pose(const json& j) {
    Pose p;
    if (j.contains("center")) p.t = vec3(j.at("center"), "center");
    if (j.contains("position")) p.t = vec3(j.at("position"), "position");
    if (j.contains("axis_angle")) p.R = exp_so3_ref(vec3(j.at("axis_angle"), "axis_angle"));
    return p;
}

fl::ShapeP<double> parse_shape(const json& j) {
    if (!j.contains("type")) throw SceneErr("shape: missing type");
    std::string type = j.at("type").get<std::string>();
    fl::ShapeP<double> s{};
    if (type == "sphere") {
        s.kind = fl::SK_SPHERE;
        s.radius = j.at("radius").get<double>();
        if (s.radius <= 0) throw SceneErr("sphere radius must be positive");
    } else if (type == "box") {
        s.kind = fl::SK_BOX;
        s.half = vec3(j.at("half_extents"), "box.half_extents");
        for (int a = 0; a < 3; a++)
            if (s.half[a] <= 0) throw SceneErr("box half extents must be positive");
    } else if (type == "capsule") {
        s.kind = fl::SK_CAPSULE;
        s.radius = j.at("radius").get<double>();
        s.seg_a = vec3(j.at("a"), "capsule.a");
        s.seg_b = vec3(j.at("b"), "capsule.b");
        if (s.radius <= 0) throw SceneErr("capsule radius must be positive");
    } else if (type == "cylinder") {
        s.kind = fl::SK_CYLINDER;
        s.radius = j.at("radius").get<double>();
        s.half_height = j.at("half_height").get<double>();
        if (s.radius <= 0 || s.half_height <= 0)
            throw SceneErr("cylinder radius and half height must be positive");
    } else if (type == "halfspace") {
        s.kind = fl::SK_HALFSPACE;
        V n = vec3(j.at("normal"), "halfspace.normal");
        double nn = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        if (nn < 1e-30)
            n = V{1, 0, 0};
        else
            n = n * (1.0 / nn);
        s.normal = n;
        s.offset = j.value("offset", 0.0);
    } else {
        throw SceneErr("shape: unknown type '" + type + "'");
    }
    return s;
}

int parse_kind(const std::string& k) {
    if (k == "elastic") return fl::MK_ELASTIC;
    if (k == "plastic") return fl::MK_PLASTIC;
    if (k == "liquid") return fl::MK_LIQUID;
    if (k == "viscous_liquid") return fl::MK_VISCOUS;
    if (k == "non_newtonian") return fl::MK_NONNEWTONIAN;
    if (k == "rigid") return fl::MK_RIGID;
    throw SceneErr("unknown material kind '" + k + "'");
}

void shape_bbox(const fl::ShapeP<double>& s, V& lo, V& hi) {
    switch (s.kind) {
        case fl::SK_SPHERE:
            lo = V{-s.radius, -s.radius, -s.radius};
            hi = V{s.radius, s.radius, s.radius};
            break;
        case fl::SK_BOX:
            lo = -s.half;
            hi = s.half;
            break;
        case fl::SK_CAPSULE:
            for (int a = 0; a < 3; a++) {
                lo[a] = std::min(s.seg_a[a], s.seg_b[a]) - s.radius;
                hi[a] = std::max(s.seg_a[a], s.seg_b[a]) + s.radius;
            }
            break;
        case fl::SK_CYLINDER:
            lo = V{-s.radius, -s.radius, -s.half_height};
            hi = V{s.radius, s.radius, s.half_height};
            break;
        default: throw SceneErr("halfspace cannot be particle-sampled");
    }
}

// scene.hpp:117-147 (axis 0 fastest)
std::vector<V> sample_shape(const fl::ShapeP<double>& shape, const Pose& pose, double dx, int ppc, double jitter,
                            Xoshiro& rng) {
    V lo, hi;
    shape_bbox(shape, lo, hi);
    double spacing = dx / ppc;
    int counts[3];
    V start;
    for (int a = 0; a < 3; a++) {
        counts[a] = std::max(1, int(std::round((hi[a] - lo[a]) / spacing)));
        start[a] = lo[a] + 0.5 * ((hi[a] - lo[a]) - counts[a] * spacing) + 0.5 * spacing;
    }
    std::vector<V> out;
    int it[3] = {0, 0, 0};
    for (;;) {
        V q;
        for (int a = 0; a < 3; a++) q[a] = start[a] + it[a] * spacing;
        V jq = q;
        if (jitter > 0)
            for (int a = 0; a < 3; a++) jq[a] += jitter * spacing * rng.uniform(-0.5, 0.5);
        if (fl::sdf_local_distance(shape, jq) <= 0) out.push_back(pose.to_world(jq));
        int a = 0;
        for (; a < 3; a++) {
            if (++it[a] < counts[a]) break;
            it[a] = 0;
        }
        if (a == 3) break;
    }
    return out;
}

}  // namespace

struct flume_scene {
    flume_config cfg{};
    std::vector<flume_material> mats;
    std::vector<flume_effector_shape> effs;
    std::vector<flume_effector_state> eff_state;
    std::vector<std::vector<long>> rb_members;
    std::vector<std::vector<double>> rb_rest;
    std::vector<flume_rigid_body> rigid;
    std::vector<flume_emitter> emitters;
    std::vector<int> mat_id, body_id;
    std::vector<double> mass, vol0;
    std::vector<long> act;
    std::vector<double> x, v, F, C;
    std::vector<flume_loss_term> loss_terms;
    std::vector<std::vector<long>> loss_goal_off;  // per term (trajectory_chamfer)
    std::vector<std::vector<double>> loss_goal_pts;
    int n_segments = 1, segment_length = 1;
    double init[6] = {0, 0, 0, 0, 0, 0};
    std::string error;
};

namespace {

void build(flume_scene& sc, const json& spec) {
    uint64_t seed = spec.value("seed", 0ull);
    Xoshiro rng(seed);
    if (spec.value("dim", 2) != 3) throw SceneErr("scene dim mismatch (the GPU path is 3D)");
    flume_config& c = sc.cfg;
    c.grid_resolution = spec.value("grid_resolution", 64);
    if (spec.value("gas_resolution", 0) > 0) throw SceneErr("gas fields are outside the GPU substep path");
    V dom{1, 1, 1};
    if (spec.contains("domain")) dom = vec3(spec.at("domain"), "domain");
    for (int a = 0; a < 3; a++) c.domain[a] = dom[a];
    c.dt_substep = spec.value("dt_substep", 1e-4);
    c.substeps_per_step = spec.value("substeps_per_step", 10);
    V g{0, 0, 0};
    if (spec.contains("gravity")) g = vec3(spec.at("gravity"), "gravity");
    for (int a = 0; a < 3; a++) c.gravity[a] = g[a];
    c.boundary_width = spec.value("boundary_width", 3);
    c.contact_eps_cells = spec.value("contact_eps_cells", 3.0);
    c.cfl_fraction = spec.value("cfl_fraction", 0.9);
    c.mass_epsilon = 1e-12;
    c.hard_contact = spec.value("hard_contact", false) ? 1 : 0;
    // SimConfig::validate (types.hpp:70-82)
    if (c.grid_resolution < 4) throw SceneErr("grid_resolution too small");
    if (c.dt_substep <= 0) throw SceneErr("dt_substep must be positive");
    if (c.substeps_per_step < 1) throw SceneErr("substeps_per_step must be >= 1");
    for (int a = 0; a < 3; a++)
        if (c.domain[a] <= 0) throw SceneErr("domain extent must be positive");
    const double dx = c.domain[0] / c.grid_resolution;
    for (int a = 1; a < 3; a++) {
        double cells = c.domain[a] / dx;
        if (std::abs(cells - std::round(cells)) > 1e-9)
            throw SceneErr("domain extent must be a whole number of cells per axis");
    }

    std::vector<std::string> mat_names;
    for (const json& jm : spec.value("materials", json::array())) {
        flume_material m{};
        std::string name = jm.value("name", "material_" + std::to_string(sc.mats.size()));
        m.kind = parse_kind(jm.value("kind", "elastic"));
        m.mu = jm.value("mu", 0.0);
        m.lambda = jm.value("lambda", 0.0);
        m.rho = jm.value("rho", 1.0);
        m.theta_c = jm.value("theta_c", 0.025);
        m.theta_s = jm.value("theta_s", 0.025);
        m.sigma_y = jm.value("sigma_y", 50.0);
        if (m.mu < 0 || m.lambda < 0) throw SceneErr("material " + name + ": negative Lame parameter");
        if (m.rho <= 0) throw SceneErr("material " + name + ": density must be positive");
        if (m.kind == fl::MK_LIQUID && m.mu != 0) throw SceneErr("material " + name + ": liquid requires mu = 0");
        if (m.kind == fl::MK_PLASTIC && (m.theta_c <= 0 || m.theta_c >= 1 || m.theta_s <= 0))
            throw SceneErr("material " + name + ": invalid box yield clamps");
        if (m.kind == fl::MK_NONNEWTONIAN && m.sigma_y <= 0)
            throw SceneErr("material " + name + ": yield stress must be positive");
        sc.mats.push_back(m);
        mat_names.push_back(name);
    }
    auto find_material = [&](const std::string& name) {
        for (size_t i = 0; i < mat_names.size(); i++)
            if (mat_names[i] == name) return int(i);
        throw SceneErr("unknown material '" + name + "'");
    };

    for (const json& je : spec.value("effectors", json::array())) {
        flume_effector_shape e{};
        flume_effector_state es{};
        fl::ShapeP<double> s = parse_shape(je.at("shape"));
        Pose sp = parse_pose(je.at("shape"));
        Pose ep = parse_pose(je);
        e.shape_kind = s.kind;
        e.radius = s.radius;
        for (int a = 0; a < 3; a++) {
            e.half_extents[a] = s.half[a];
            e.seg_a[a] = s.seg_a[a];
            e.seg_b[a] = s.seg_b[a];
            e.plane_normal[a] = s.normal[a];
            e.shape_t[a] = sp.t[a];
            es.pose_t[a] = ep.t[a];
        }
        e.plane_offset = s.offset;
        e.half_height = s.half_height;
        for (int q = 0; q < 9; q++) {
            e.shape_R[q] = sp.R.m[q];
            es.pose_R[q] = ep.R.m[q];
        }
        e.friction_mu = 0;
        if (je.contains("friction")) {
            const json& f = je.at("friction");
            if (f.is_string()) {
                if (f.get<std::string>() != "sticky") throw SceneErr("effector friction: number or \"sticky\"");
                e.friction_mu = std::numeric_limits<double>::infinity();
            } else {
                e.friction_mu = f.get<double>();
            }
            if (e.friction_mu < 0) throw SceneErr("effector friction must be >= 0");
        }
        if (je.contains("velocity")) {
            V vv = vec3(je.at("velocity"), "effector.velocity");
            for (int a = 0; a < 3; a++) es.linear_velocity[a] = vv[a];
        }
        if (je.contains("angular_velocity")) {
            V av = vec3(je.at("angular_velocity"), "effector.angular_velocity");
            for (int a = 0; a < 3; a++) es.angular_velocity[a] = av[a];
        }
        if (je.contains("action_mask")) {
            const json& jm = je.at("action_mask");
            if (!jm.is_array() || jm.size() != 6) throw SceneErr("effector action_mask must have 6 entries");
            for (int a = 0; a < 6; a++) e.action_mask[a] = jm[a].get<bool>() ? 1 : 0;
        }
        sc.effs.push_back(e);
        sc.eff_state.push_back(es);
    }

    int body = 0;
    std::vector<std::string> body_names;
    for (const json& jb : spec.value("bodies", json::array())) {
        std::string name = jb.value("name", "body_" + std::to_string(body));
        body_names.push_back(name);
        int mat = find_material(jb.at("material").get<std::string>());
        const flume_material& m = sc.mats[mat];
        fl::ShapeP<double> shape = parse_shape(jb.at("shape"));
        Pose pose = parse_pose(jb.at("shape"));
        int ppc = jb.value("particles_per_cell_axis", 2);
        double jitter = jb.value("jitter", 0.0);
        std::vector<V> pts = sample_shape(shape, pose, dx, ppc, jitter, rng);
        if (jb.contains("exclude")) {
            std::vector<std::pair<fl::ShapeP<double>, Pose>> holes;
            for (const json& jx : jb.at("exclude")) holes.push_back({parse_shape(jx), parse_pose(jx)});
            double margin = 0.5 * dx / ppc;
            std::vector<V> kept;
            for (const V& p : pts) {
                bool drop = false;
                for (const auto& h : holes) {
                    fl::SdfSample<double> ss = fl::sdf_eval(h.first, h.second.t, h.second.R, p);
                    if (ss.distance <= margin) drop = true;
                }
                if (!drop) kept.push_back(p);
            }
            pts.swap(kept);
        }
        if (pts.empty()) throw SceneErr("body '" + name + "': zero particles sampled");
        V v0{0, 0, 0}, w0{0, 0, 0};
        if (jb.contains("velocity")) v0 = vec3(jb.at("velocity"), "body.velocity");
        if (jb.contains("angular_velocity")) w0 = vec3(jb.at("angular_velocity"), "body.angular_velocity");
        double spacing = dx / ppc;
        double vol0 = std::pow(spacing, 3);
        bool rigid = m.kind == fl::MK_RIGID;
        const json* jem = jb.contains("emitter") ? &jb.at("emitter") : nullptr;
        long em_start = jem ? jem->value("start_substep", 0l) : 0;
        long em_interval = jem ? std::max(1l, jem->value("interval_substeps", 1l)) : 0;
        int em_eff = jem ? jem->value("effector", -1) : -1;
        V em_vel{0, 0, 0};
        if (jem && jem->contains("velocity")) em_vel = vec3(jem->at("velocity"), "emitter.velocity");
        if (rigid && jem) throw SceneErr("body '" + name + "': rigid emitters unsupported");
        std::vector<long> members;
        V centroid{0, 0, 0};
        double total = 0;
        for (size_t k = 0; k < pts.size(); k++) {
            V x = pts[k];
            for (int a = 0; a < 3; a++)
                if (x[a] < 0 || x[a] > c.domain[a]) throw SceneErr("body '" + name + "' extends outside the domain");
            for (int a = 0; a < 3; a++) x[a] = std::min(std::max(x[a], dx), c.domain[a] - dx);
            V r = pts[k] - pose.t;
            V vel = v0 + fl::cross(w0, r);
            long pid = long(sc.mat_id.size());
            sc.mat_id.push_back(mat);
            sc.body_id.push_back(body);
            sc.vol0.push_back(vol0);
            sc.mass.push_back(m.rho * vol0);
            sc.act.push_back(jem ? em_start + long(k) * em_interval : 0);
            for (int a = 0; a < 3; a++) {
                sc.x.push_back(x[a]);
                sc.v.push_back(vel[a]);
            }
            for (int q = 0; q < 9; q++) {
                sc.F.push_back(q % 4 == 0 ? 1.0 : 0.0);
                sc.C.push_back(0.0);
            }
            if (jem) {
                flume_emitter em{};
                em.particle = pid;
                em.effector = em_eff;
                V lp = em_eff >= 0 ? pts[k] - pose.t : pts[k];
                for (int a = 0; a < 3; a++) {
                    em.local_pos[a] = lp[a];
                    em.local_vel[a] = em_vel[a];
                }
                sc.emitters.push_back(em);
            }
            if (rigid) {
                members.push_back(pid);
                for (int a = 0; a < 3; a++) centroid[a] += x[a] * (m.rho * vol0);
                total += m.rho * vol0;
            }
        }
        if (rigid) {
            double inv = 1.0 / total;
            centroid = centroid * inv;
            std::vector<double> rest;
            for (long pid : members)
                for (int a = 0; a < 3; a++) rest.push_back(sc.x[3 * pid + a] - centroid[a]);
            sc.rb_members.push_back(members);
            sc.rb_rest.push_back(rest);
            flume_rigid_body rb{};
            rb.body_id = body;
            rb.total_mass = total;
            sc.rigid.push_back(rb);
        }
        body++;
    }
    for (size_t b = 0; b < sc.rigid.size(); b++) {
        sc.rigid[b].n_members = long(sc.rb_members[b].size());
        sc.rigid[b].members = sc.rb_members[b].data();
        sc.rigid[b].rest_offsets = sc.rb_rest[b].data();
    }

    auto resolve_body = [&](const json& jt) -> int {
        if (!jt.contains("body")) return -1;
        if (jt.at("body").is_number()) return jt.at("body").get<int>();
        std::string nm = jt.at("body").get<std::string>();
        for (size_t i = 0; i < body_names.size(); i++)
            if (body_names[i] == nm) return int(i);
        throw SceneErr("loss references unknown body '" + nm + "'");
    };
    auto add_term = [&](const json& jt) {
        flume_loss_term t{};
        std::string kind = jt.value("kind", "target_point");
        t.weight = jt.value("weight", 1.0);
        if (t.weight < 0) throw SceneErr("loss weights must be non-negative");
        t.squared = jt.value("squared", false) ? 1 : 0;
        t.final_only = jt.value("eval", "per_step") == std::string("final") ? 1 : 0;
        t.body = resolve_body(jt);
        if (kind == "target_point") {
            t.kind = FLUME_LOSS_TARGET_POINT;
            V gl = vec3(jt.at("goal"), "loss.goal");
            for (int a = 0; a < 3; a++) t.goal[a] = gl[a];
        } else if (kind == "hold_initial") {
            t.kind = FLUME_LOSS_HOLD_INITIAL;
        } else if (kind == "mixing_spread") {
            t.kind = FLUME_LOSS_MIXING_SPREAD;
        } else if (kind == "trajectory_chamfer") {
            t.kind = FLUME_LOSS_TRAJECTORY_CHAMFER;
            std::vector<long> off{0};
            std::vector<double> pts;
            for (const json& jstep : jt.at("goal_trajectory")) {
                for (const json& jp : jstep) {
                    V p = vec3(jp, "goal point");
                    for (int a = 0; a < 3; a++) pts.push_back(p[a]);
                }
                off.push_back(long(pts.size() / 3));
            }
            if (off.size() < 2) throw SceneErr("trajectory_chamfer: empty goal_trajectory");
            sc.loss_goal_off.resize(sc.loss_terms.size() + 1);
            sc.loss_goal_pts.resize(sc.loss_terms.size() + 1);
            sc.loss_goal_off.back() = std::move(off);
            sc.loss_goal_pts.back() = std::move(pts);
        } else {
            throw SceneErr("loss kind '" + kind + "' is outside the GPU path");
        }
        sc.loss_terms.push_back(t);
    };
    if (spec.contains("loss")) {
        const json& jl = spec.at("loss");
        if (jl.value("kind", "") == std::string("composite"))
            for (const json& jt : jl.at("terms")) add_term(jt);
        else
            add_term(jl);
    }
    if (spec.contains("optimizer")) {
        const json& jo = spec.at("optimizer");
        sc.n_segments = jo.value("n_segments", 1);
        sc.segment_length = jo.value("segment_length", 1);
        if (jo.contains("init"))
            for (int k = 0; k < 6 && k < int(jo.at("init").size()); k++) sc.init[k] = jo.at("init")[k].get<double>();
    }
}

}  // namespace

extern "C" {

int flume_scene_build_json(const char* text, flume_scene** out) {
    if (!text || !out) return FLUME_E_ARG;
    *out = nullptr;
    flume_scene* sc = new flume_scene();
    try {
        build(*sc, json::parse(text));
    } catch (const SceneErr& e) {
        static thread_local std::string msg;
        msg = e.what();
        sc->error = msg;
        *out = sc;
        return FLUME_E_SCENE;
    } catch (const std::exception& e) {
        sc->error = e.what();
        *out = sc;
        return FLUME_E_SCENE;
    }
    *out = sc;
    return FLUME_OK;
}

const char* flume_scene_error(const flume_scene* s) { return s ? s->error.c_str() : ""; }

int flume_scene_free(flume_scene* s) {
    delete s;
    return FLUME_OK;
}

int flume_scene_desc_get(const flume_scene* s, flume_scene_desc* d) {
    if (!s || !d) return FLUME_E_ARG;
    *d = flume_scene_desc{};
    d->config = s->cfg;
    d->n_materials = int(s->mats.size());
    d->materials = s->mats.data();
    d->n_effectors = int(s->effs.size());
    d->effectors = s->effs.data();
    d->n_rigid = int(s->rigid.size());
    d->rigid = s->rigid.data();
    d->n_emitters = long(s->emitters.size());
    d->emitters = s->emitters.data();
    d->n_particles = long(s->mat_id.size());
    d->material_id = s->mat_id.data();
    d->body_id = s->body_id.data();
    d->mass = s->mass.data();
    d->volume0 = s->vol0.data();
    d->activation_substep = s->act.data();
    return FLUME_OK;
}

int flume_scene_state_get(const flume_scene* s, flume_state_view* v) {
    if (!s || !v) return FLUME_E_ARG;
    v->time = 0;
    v->substep_index = 0;
    v->x = const_cast<double*>(s->x.data());
    v->v = const_cast<double*>(s->v.data());
    v->F = const_cast<double*>(s->F.data());
    v->C = const_cast<double*>(s->C.data());
    v->effectors = const_cast<flume_effector_state*>(s->eff_state.data());
    return FLUME_OK;
}

int flume_scene_loss_get(const flume_scene* s, flume_loss_desc* l) {
    if (!s || !l) return FLUME_E_ARG;
    // goal point sets live in the scene's own vectors; point the terms at them
    flume_scene* ms = const_cast<flume_scene*>(s);
    for (size_t k = 0; k < ms->loss_terms.size(); k++) {
        flume_loss_term& t = ms->loss_terms[k];
        if (t.kind != FLUME_LOSS_TRAJECTORY_CHAMFER || k >= ms->loss_goal_off.size()) continue;
        t.n_goal_steps = int(ms->loss_goal_off[k].size()) - 1;
        t.goal_step_offsets = ms->loss_goal_off[k].data();
        t.goal_points = ms->loss_goal_pts[k].data();
    }
    *l = flume_loss_desc{};
    l->n_terms = int(s->loss_terms.size());
    l->terms = s->loss_terms.data();
    l->attraction_body = -1;  // off until the optimizer enables it
    return FLUME_OK;
}

int flume_scene_optimizer_get(const flume_scene* s, int* n_segments, int* segment_length, double* init6) {
    if (!s) return FLUME_E_ARG;
    if (n_segments) *n_segments = s->n_segments;
    if (segment_length) *segment_length = s->segment_length;
    if (init6)
        for (int k = 0; k < 6; k++) init6[k] = s->init[k];
    return FLUME_OK;
}

}  // extern "C"
